# Launch list + ncu --set full captures of the step's kernels; the .ncu-rep files are
# reduced to CSV on the box (gpurun brings back <= 64 MiB).
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1
echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 14 -c 14 -o /tmp/prof_gemm $B > gpurun_out/ncu2.log 2>&1
echo gemm rc=$?
ncu --set full --clock-control none --import-source on -k regex:"${SIDE_RE:-k_aq|k_tt_|k_mid|k_dequant}" -s ${SIDE_S:-45} -c ${SIDE_C:-45} -o /tmp/prof_side $B > gpurun_out/ncu3.log 2>&1
echo side rc=$?
for p in gemm side; do
  ncu -i /tmp/prof_$p.ncu-rep --page raw --csv > gpurun_out/raw_$p.csv 2>/dev/null
  ncu -i /tmp/prof_$p.ncu-rep --page details --csv > gpurun_out/details_$p.csv 2>/dev/null
done
python tools/measure_int8_peak.py > gpurun_out/int8_peak.log 2>&1; echo int8 rc=$?
ls -la gpurun_out
