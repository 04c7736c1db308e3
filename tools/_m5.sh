timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
for K in 4096; do python tools/micro.py --only bwd --K $K 2>&1; QA_FUSED_BWD=0 python tools/micro.py --only bwd --K $K 2>&1 | grep -E "tt|per call"; done
python tools/micro.py --only bwd --N 11008 2>&1 | grep -E "tt|per call"
python tools/micro.py --only bwd --K 11008 2>&1 | grep -E "tt|per call"
