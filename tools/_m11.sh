for v in main minb3 minb4; do
  if [ $v = main ]; then L=""; else L="QADAPTER_LIB=paper_2402_13533_b200/build/var/$v.so"; fi
  echo "== $v"; for K in 4096 11008; do env $L python tools/micro.py --only fwd --K $K 2>&1 | grep -E "quantize"; done
done
