rm -f /tmp/pm*.ncu-rep
python tools/merge_bench.py --set 70b --iters 1 > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"k_merge_nd1" -s 4 -c 1 -o /tmp/pm python tools/merge_bench.py --set 70b --iters 1 > gpurun_out/ncu_m.log 2>&1
ncu -i /tmp/pm.ncu-rep --page raw --csv > gpurun_out/raw_m.csv; ncu -i /tmp/pm.ncu-rep --page source --csv > gpurun_out/src_m.csv
