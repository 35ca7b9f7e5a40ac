# usage: bash tools/gpu_ncu_k.sh <kernel-regex> <tag> [launch-skip]
K="$1"; TAG="$2"; SKIP="${3:-0}"
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$K" -s "$SKIP" -c 1 -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i gpurun_out/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>&1
ncu -i gpurun_out/${TAG}_full.ncu-rep --page source --csv > gpurun_out/${TAG}_source.csv 2>&1
ncu -i gpurun_out/${TAG}_full.ncu-rep --page details > gpurun_out/${TAG}_details.txt 2>&1
