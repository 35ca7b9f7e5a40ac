# refresh the committed evidence: tests, bench (+ reference arm), cfg sweeps, launch list, ncu of the top kernels
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/p_bench_ref.json 2> gpurun_out/p_bench_ref.err
timeout 600 python bench_configs.py --config 3 > gpurun_out/p_cfg3.json 2>> gpurun_out/p_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --graph 0 > gpurun_out/p_ncu_launch.log 2>&1
bash tools/gpu_ncu_k.sh "k_hs_imma(?!_tiles)" hsimma 0; bash tools/gpu_ncu_k.sh k_conv_pt conv 0; bash tools/gpu_ncu_k.sh "k_ks_inner_t" ksinner 20
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/traffic.csv python tools/one_step.py > gpurun_out/one_step.log 2>&1
bash tools/gpu_ncu_k.sh k_drop_ntt drop 40
bash tools/gpu_ncu_k.sh k_ks_modup modup 30
