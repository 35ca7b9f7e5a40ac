#!/bin/bash
# conv MAC time (cfg2 step kernel table + cfg3) per library variant
for L in "$@"; do
  a=$(HEGPU_LIB=$L python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['kernels']['k_conv_mac']['ms_per_step'],3))")
  b=$(HEGPU_LIB=$L python tools/cfg3_kernels.py 16 | grep conv | awk '{print $2}')
  echo "$(basename $L) cfg2: $a  cfg3 conv: $b"
done
