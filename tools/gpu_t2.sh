timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t2_pytest.log
timeout 600 python bench.py --no-cpu > gpurun_out/t2_bench.json 2> gpurun_out/t2_bench.err
HEGPU_HS_IMMA=0 timeout 600 python bench.py --no-cpu > gpurun_out/t2_bench_noimma.json 2>> gpurun_out/t2_bench.err
timeout 600 python bench_configs.py --config 3 > gpurun_out/t2_cfg3.json 2>> gpurun_out/t2_bench.err
tail -3 gpurun_out/t2_pytest.log
