# A/B of runtime switches on the device bench: bash tools/gpu_env_ab.sh "ENV=V ..." ...
i=0
for v in "$@"; do
  i=$((i+1))
  env $v python bench.py --no-cpu --no-fused --steps 10 --warmup 3 > gpurun_out/env_$i.json 2> gpurun_out/env_$i.err || tail -3 gpurun_out/env_$i.err
  echo "== $v"; python tools/kern_ms.py gpurun_out/env_$i.json | cut -c1-200
done
