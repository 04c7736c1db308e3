for K in 4096 11008; do for pf in 1 0; do QA_GEMM_PREFETCH=$pf python tools/micro.py --only fwd --K $K --iters 30 2>&1 | grep -E "gemm_i8" | sed "s/^/K=$K pf=$pf /"; done; done
for pf in 1 0; do QA_GEMM_PREFETCH=$pf python tools/micro.py --only fwd --N 11008 --iters 30 2>&1 | grep -E "gemm_i8" | sed "s/^/N=11008 pf=$pf /"; done
