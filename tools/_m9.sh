timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
for K in 4096 11008; do python tools/micro.py --only fwd --K $K 2>&1 | grep -E "quantize|per call"; QA_AQ_RING=0 python tools/micro.py --only fwd --K $K 2>&1 | grep -E "quantize"; done
python tools/micro.py --only bwd 2>&1 | grep -E "quantize"
