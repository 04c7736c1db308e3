rm -f /tmp/pg*.ncu-rep
python tools/micro.py --only fwd --iters 2 > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"k_gemm_tc_2sm" -s 1 -c 1 -o /tmp/pg python tools/micro.py --only fwd --iters 2 > gpurun_out/ncu_g.log 2>&1
ncu -i /tmp/pg.ncu-rep --page source --csv > gpurun_out/src_g.csv; ncu -i /tmp/pg.ncu-rep --page raw --csv > gpurun_out/raw_g.csv
