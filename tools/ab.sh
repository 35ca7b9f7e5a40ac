#!/bin/bash
# A/B timing of libhegpu variants on the GPU box:  tools/ab.sh LIB...
for L in "$@"; do
  HEGPU_LIB=$L python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$L'.split('/')[-1], round(d['value']), round(d['e2e']['value']), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items() if v['ms_per_step']>0.2})"
done
