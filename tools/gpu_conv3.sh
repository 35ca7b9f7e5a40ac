# tcgen05 conv A/B: "bufs kcb lag" (0 = default) on config 3 (75 taps, 32 maps) and the config-2 bench
timeout 600 python -m pytest tests/test_gpu_stated_sizes.py tests/test_gpu_parity.py -k "cfg4 or conv" -x -q 2>&1 | tail -1
for v in ${CFG3_SWEEP:-0_0_0 4_128_2 6_96_3 4_128_1}; do
  set -- $(echo $v | tr _ ' ')
  unset HEGPU_TC_BUFS HEGPU_TC_KCB HEGPU_TC_LAG
  [ "$1" != 0 ] && export HEGPU_TC_BUFS=$1; [ "$2" != 0 ] && export HEGPU_TC_KCB=$2; [ "$3" != 0 ] && export HEGPU_TC_LAG=$3
  echo "== bufs $1 kcb $2 lag $3: $(timeout 300 python tools/cfg3_kernels.py 16 2>&1 | grep k_conv_mac)"
done
for v in ${CFG2_SWEEP:-0_0 4_2 4_3 5_3 6_4 2_1}; do
  set -- $(echo $v | tr _ ' ')
  unset HEGPU_TC_BUFS HEGPU_TC_KCB HEGPU_TC_LAG
  [ "$1" != 0 ] && export HEGPU_TC_BUFS=$1; [ "$2" != 0 ] && export HEGPU_TC_LAG=$2
  timeout 300 python bench.py --no-cpu --no-fused --steps 5 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernels']['k_conv_mac']; print('cfg2 bufs $1 lag $2', round(d['ms_per_step'],4), round(k['ms_per_step'],4), round(k['gbs']))"
done
