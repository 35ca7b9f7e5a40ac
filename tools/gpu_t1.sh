timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_core or hs_matvec" > gpurun_out/t1.log 2>&1; echo "rc=$?" >> gpurun_out/t1.log
tail -30 gpurun_out/t1.log
