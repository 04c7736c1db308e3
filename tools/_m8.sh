rm -f /tmp/pf*.ncu-rep
python tools/micro.py --only bwd --iters 2 > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"k_tt_dg1m" -s 1 -c 1 -o /tmp/pfd python tools/micro.py --only bwd --iters 2 > gpurun_out/ncu_dm.log 2>&1
ncu -i /tmp/pfd.ncu-rep --page raw --csv > gpurun_out/raw_dm.csv; ncu -i /tmp/pfd.ncu-rep --page source --csv > gpurun_out/src_dm.csv
