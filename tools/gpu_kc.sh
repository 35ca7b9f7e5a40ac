cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_stated_sizes.py -k "cfg4 or cfg3" -x -q > gpurun_out/kc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/kc_pytest.log
tail -5 gpurun_out/kc_pytest.log
for v in 1 0; do echo "== CONV_TC=$v"; HEGPU_CONV_TC=$v timeout 300 python tools/cfg3_kernels.py 16 2>&1 | tail -17; done > gpurun_out/kc_cfg3.log 2>&1
cat gpurun_out/kc_cfg3.log
for v in 1 0; do HEGPU_CONV_TC=$v timeout 300 python bench_configs.py --config 3 2>&1 | tail -2; done > gpurun_out/kc_bc3.log
cat gpurun_out/kc_bc3.log
timeout 300 python bench.py --no-cpu --no-fused > gpurun_out/kc_bench.json 2> gpurun_out/kc_bench.err
python -c "
import json; d=json.load(open('gpurun_out/kc_bench.json')); print('cfg2 ms', d['ms_per_step'], 'value', d['value'])
[print('  ', k, round(v['ms_per_step'],4), round(v['gbs'],1)) for k, v in d['kernels'].items()]"
