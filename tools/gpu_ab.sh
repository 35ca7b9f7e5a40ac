# tests, then device-bench A/B over runtime switches given as arguments ("ENV=V ENV2=V2" per variant)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
i=0
for v in "$@"; do
  i=$((i+1))
  env $v timeout 600 python bench.py --no-cpu --no-fused > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
  python - "$v" gpurun_out/ab_$i.json <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
except Exception as e:
    print(sys.argv[1], 'FAILED', e); sys.exit(0)
print('==', sys.argv[1], 'value', round(d['value']), 'ms', round(d['ms_per_step'], 4), 'e2e', round(d['e2e']['value']))
for k, v in d['kernels'].items():
    print('  ', k, round(v['ms_per_step'], 4), v['launches'], round(v['gbs'], 1))
PY
done
