# round evidence: tests, smoke, bench (both arms), configs 1/3/4, launch list of one step, traffic, ncu of the top kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/ev_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ev_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err
timeout 600 python bench_configs.py --config 3 > gpurun_out/ev_cfg3.json 2>> gpurun_out/ev_bench.err
timeout 900 python bench_configs.py --config 1 > gpurun_out/ev_cfg1.jsonl 2>> gpurun_out/ev_bench.err
timeout 900 python bench_configs.py --config 4 > gpurun_out/ev_cfg4.jsonl 2>> gpurun_out/ev_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-fused --graph 0 > gpurun_out/ev_ncu_launch.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/ev_traffic.csv python tools/one_step.py > gpurun_out/ev_one_step.log 2>&1
bash tools/gpu_ncu_k.sh k_ks_modup ev_modup 0
bash tools/gpu_ncu_k.sh k_drop_ntt ev_drop 0
bash tools/gpu_ncu_k.sh "k_hs_tc$" ev_hstc 0
bash tools/gpu_ncu_k.sh "k_conv_tc" ev_convtc 0
bash tools/gpu_ncu_k.sh "k_md_ntt" ev_mdntt 0
rm -f gpurun_out/*_source.csv
tail -2 gpurun_out/ev_pytest.log; tail -1 gpurun_out/ev_smoke.log; head -c 400 gpurun_out/ev_bench.json
