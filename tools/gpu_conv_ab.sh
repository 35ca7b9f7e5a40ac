# A/B of the tcgen05 conv's tiles-per-CTA and A buffers (device bench, conv kernel time)
for v in "16 3" "8 3" "32 3" "16 4" "32 4" "64 4" "16 2"; do
  set -- $v
  HEGPU_TC_TILES=$1 HEGPU_TC_BUFS=$2 timeout 300 python bench.py --no-cpu --no-fused --steps 5 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernels']['k_conv_mac']; print('tiles $1 bufs $2', round(d['ms_per_step'],4), round(k['ms_per_step'],4), round(k['gbs']))"
done
