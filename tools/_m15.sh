timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for K in 4096 11008; do python tools/micro.py --only fwd --K $K --iters 30 2>&1 | grep -E "gemm" | sed "s/^/K=$K /"; done
python tools/micro.py --only fwd --N 11008 --iters 30 2>&1 | grep -E "gemm" | sed "s/^/N=11008 /"
