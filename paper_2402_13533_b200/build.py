"""Build the sm_100a C-ABI library in-tree: paper_2402_13533_b200/libqadapter.so.

    python -m paper_2402_13533_b200.build        (or __graft_entry__.build())

nvcc cross-compiles for sm_100a without a GPU.  cudart is linked statically; the
driver API entry point for TMA descriptors is resolved at run time
(cudaGetDriverEntryPoint), so the library needs nothing but libcuda on the box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libqadapter.so")
SOURCES = ["quant_kernels.cu", "tt_kernels.cu", "tt_dense.cu", "tt_fast.cu", "gemm_tc.cu", "gemv.cu", "optim.cu", "glue.cu", "qmm.cu", "timing.cu", "capi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "qadapter.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """defines / out: development variants (extra -D flags, another output path; see tools/)."""
    lib_path = out or LIB
    if not force and not defines and out is None and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build", "variant_" + "_".join(d.replace("=", "") for d in defines)) if defines \
        else os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    common = [nvcc(), "-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-fvisibility=hidden",
              "-Xptxas", "-v" if verbose else "-O3", "--expt-relaxed-constexpr", *["-D" + d for d in defines]]
    objs, cmds = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = common + ["-c", os.path.join(CSRC, src), "-o", obj]
        if src == "capi.cu":
            cmd.insert(1, "-DQA_EXPORTS")
        cmds.append(cmd)
        objs.append(obj)
    # translation units are independent: compile them concurrently
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as pool:
        for r in list(pool.map(lambda c: subprocess.run(c, check=True), cmds)):
            del r
    tmp = lib_path + ".tmp"
    subprocess.run([nvcc(), "-shared", *ARCH, "-o", tmp, *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"],
                   check=True)
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, out=outs[0] if outs else None))
