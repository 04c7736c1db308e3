timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for ts in 1 0; do for K in 4096 11008; do QA_GEMM_TMA_STORE=$ts python tools/micro.py --K $K --iters 30 2>&1 | grep -E "gemm" | sed "s/^/ts=$ts K=$K /"; done; done
