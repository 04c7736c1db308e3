python tools/micro.py --only fwd --iters 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_aq_ -s 3 -c 1 -o /tmp/p_reg python tools/micro.py --only fwd --iters 2 > /dev/null 2>&1
QA_AQ_REG=0 ncu --set full --clock-control none --import-source on -k regex:k_aq_ -s 3 -c 1 -o /tmp/p_cta python tools/micro.py --only fwd --iters 2 > /dev/null 2>&1
for p in p_reg p_cta; do ncu -i /tmp/$p.ncu-rep --page raw --csv > gpurun_out/raw_$p.csv; ncu -i /tmp/$p.ncu-rep --page source --csv > gpurun_out/src_$p.csv; done
ls gpurun_out
