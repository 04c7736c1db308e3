for v in main fold8 fold24; do
  if [ $v = main ]; then L=""; else L="QADAPTER_LIB=paper_2402_13533_b200/build/var/$v.so"; fi
  for K in 4096 11008; do env $L python tools/micro.py --only fwd --K $K --iters 30 2>&1 | grep -E "gemm_i8" | sed "s/^/$v K=$K /"; done
done
