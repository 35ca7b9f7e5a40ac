# usage: bash tools/gpu_ncu_k.sh <kernel-regex> <tag> [launch-skip] [extra bench args]
# full ncu capture of one launch; the .ncu-rep stays in /tmp (size), the
# raw / source / details pages come back in gpurun_out/
K="$1"; TAG="$2"; SKIP="${3:-0}"; shift 3; EXTRA="$*"
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$K" -s "$SKIP" -c 1 -o /tmp/${TAG}_full -f python bench.py --steps 1 --warmup 3 --no-cpu --no-fused $EXTRA > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i /tmp/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>&1
ncu -i /tmp/${TAG}_full.ncu-rep --page source --csv > gpurun_out/${TAG}_source.csv 2>&1
ncu -i /tmp/${TAG}_full.ncu-rep --page details > gpurun_out/${TAG}_details.txt 2>&1
