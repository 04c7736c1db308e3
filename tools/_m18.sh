rm -f /tmp/pd*.ncu-rep
python tools/decode_micro.py 1 > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:k_decode_prep -s 5 -c 1 -o /tmp/pd python tools/decode_micro.py 1 > /dev/null 2>&1
ncu -i /tmp/pd.ncu-rep --page source --csv > gpurun_out/src_pd.csv
