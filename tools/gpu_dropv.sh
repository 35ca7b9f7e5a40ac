# A/B of the drop-limb / fused ModDown build variants (HEGPU_DROP_V=<md><plain>)
for v in 10 12 20 22 11; do
  HEGPU_DROP_V=$v timeout 300 python bench.py --no-cpu --no-fused --steps 10 --warmup 3 > gpurun_out/dropv_$v.json 2> gpurun_out/dropv_$v.err
done
python tools/kern_ms.py gpurun_out/dropv_*.json
