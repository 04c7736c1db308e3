# Round profile: default bench line (+ reference arm), launch list of the timed steps, and
# ncu --set full captures of one step's GEMMs and side kernels, reduced to CSV on the box
# (gpurun brings back <= 64 MiB); plus the decode kernels and the config-4 decoder kernel shares.
python bench.py > gpurun_out/bench_full.log 2>&1; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-merge --no-decoder"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1
echo launches rc=$?
rm -f /tmp/prof_*.ncu-rep
ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s ${GEMM_S:-14} -c ${GEMM_C:-14} -o /tmp/prof_gemm $B > gpurun_out/ncu2.log 2>&1
echo gemm rc=$?
ncu --set full --clock-control none --import-source on -k regex:"${SIDE_RE:-k_aq|k_tt_|k_grad|k_dequant}" -s ${SIDE_S:-29} -c ${SIDE_C:-29} -o /tmp/prof_side $B > gpurun_out/ncu3.log 2>&1
echo side rc=$?
python tools/decode_micro.py 1 > gpurun_out/decode_micro.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_decode_prep|k_gemv" -s 10 -c 2 -o /tmp/prof_decode python tools/decode_micro.py 1 > gpurun_out/ncu4.log 2>&1
echo decode rc=$?
for p in gemm side decode; do
  ncu -i /tmp/prof_$p.ncu-rep --page raw --csv > gpurun_out/raw_$p.csv 2>/dev/null
done
python tools/decoder_profile.py > gpurun_out/decoder_prof.log 2>&1; echo decoder rc=$?
ls -la gpurun_out
