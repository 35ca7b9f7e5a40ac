# A/B of library builds on the device bench: bash tools/gpu_lib_ab.sh [LIB ...] (the in-tree build first)
python bench.py --no-cpu --no-fused --steps 10 --warmup 3 > gpurun_out/ab_default.json 2> gpurun_out/ab_default.err
for L in "$@"; do
  HEGPU_LIB=$L python bench.py --no-cpu --no-fused --steps 10 --warmup 3 > gpurun_out/ab_$(basename $L .so).json 2> gpurun_out/ab_$(basename $L .so).err
done
python tools/kern_ms.py gpurun_out/ab_*.json
