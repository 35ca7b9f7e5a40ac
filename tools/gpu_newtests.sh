set -x
timeout 2400 python -m pytest tests/test_gpu_stated_sizes.py tests/test_cli.py -m gpu -x -q -v --durations=10 > gpurun_out/pytest_sizes.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sizes.log
tail -25 gpurun_out/pytest_sizes.log
