rm -f /tmp/pr*.ncu-rep
python tools/micro.py --only fwd --iters 2 > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"k_aq_ring" -s 1 -c 1 -o /tmp/pr python tools/micro.py --only fwd --iters 2 > gpurun_out/ncu_r.log 2>&1
ncu -i /tmp/pr.ncu-rep --page raw --csv > gpurun_out/raw_r.csv; ncu -i /tmp/pr.ncu-rep --page source --csv > gpurun_out/src_r.csv
