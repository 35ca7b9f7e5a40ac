timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_hs_imma(?!_tiles)" -c 1 -o gpurun_out/hs_imma_full python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/t3_ncu.log 2>&1
ncu -i gpurun_out/hs_imma_full.ncu-rep --page raw --csv > gpurun_out/hs_imma_raw.csv 2>&1
ncu -i gpurun_out/hs_imma_full.ncu-rep --page source --csv > gpurun_out/hs_imma_source.csv 2>&1
ncu -i gpurun_out/hs_imma_full.ncu-rep --page details > gpurun_out/hs_imma_details.txt 2>&1
tail -3 gpurun_out/t3_ncu.log
