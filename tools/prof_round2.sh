# Round-2 profile set: default bench line + reference arm, launch list of one timed step (duration + DRAM bytes),
# ncu --set full of one step's GEMMs and side kernels, the merge (70B gate, fp32 and bf16 W'), the weight
# quantiser, the decode kernels and the smoke launch list; raw CSVs written on the box (gpurun brings <= 64 MiB).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2f
python bench.py > ${O}_bench.log 2>&1; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > ${O}_bench_ref.log 2>&1; echo ref rc=$?
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-merge --no-decoder"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file ${O}_launches.csv $B > ${O}_ncu_l.log 2>&1; echo launches rc=$?
rm -f /tmp/p_*.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 42 -c 14 -f -o /tmp/p_gemm $B > ${O}_ncu_g.log 2>&1; echo gemm rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_aq|k_tt_|k_grad|k_dequant|k_g1_frag|k_build_v" -s 60 -c 20 -f -o /tmp/p_side $B > ${O}_ncu_s.log 2>&1; echo side rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_merge_fast -s 12 -c 1 -f -o /tmp/p_merge32 python tools/merge_bench.py --set 70b --out f32 --iters 1 > ${O}_ncu_m.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_merge_fast -s 12 -c 1 -f -o /tmp/p_merge16 python tools/merge_bench.py --set 70b --out bf16 --iters 1 >> ${O}_ncu_m.log 2>&1; echo merge rc=$?
python tools/quant_micro.py > ${O}_quant.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_quantize_rows -s 3 -c 1 -f -o /tmp/p_quant python tools/quant_micro.py > ${O}_ncu_q.log 2>&1; echo quant rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_decode_prep|k_gemv" -s 10 -c 2 -f -o /tmp/p_decode python tools/decode_micro.py 1 > ${O}_ncu_d.log 2>&1; echo decode rc=$?
python tools/decode_timeline.py 1 > ${O}_decode_timeline.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo smoke rc=$?
for p in gemm side merge32 merge16 quant decode; do
  ncu -i /tmp/p_$p.ncu-rep --page raw --csv > ${O}_raw_$p.csv 2>/dev/null
done
ncu -i /tmp/p_side.ncu-rep --page details --csv > ${O}_det_side.csv 2>/dev/null
ls -la gpurun_out | tail -30
