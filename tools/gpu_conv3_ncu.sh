# one full ncu capture of the config-3 tcgen05 conv at batch 16 (args: env assignments)
export "$@"
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_conv_tc" -c 1 -o /tmp/c3_full -f python tools/cfg3_kernels.py 16 > gpurun_out/c3conv_ncu.log 2>&1
ncu -i /tmp/c3_full.ncu-rep --page raw --csv > gpurun_out/c3conv_raw.csv 2>&1
ncu -i /tmp/c3_full.ncu-rep --page source --csv > gpurun_out/c3conv_source.csv 2>&1
ncu -i /tmp/c3_full.ncu-rep --page details > gpurun_out/c3conv_details.txt 2>&1
