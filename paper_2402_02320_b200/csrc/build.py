"""Build libmpx.so in-tree with nvcc for sm_100a (no torch types cross the ABI).

    python -m paper_2402_02320_b200.csrc.build      (or __graft_entry__.build())
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(HERE)
REPO = os.path.dirname(PKG)
SOURCES = ["ring.cu", "beaver.cu", "gemm.cu", "gemm_tc.cu", "beaver_gemm.cu", "dealer.cu", "fused_ops.cu"]
OUT = os.path.join(PKG, "libmpx.so")


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def flags() -> list[str]:
    return ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC", "-Xptxas", "-v", f"-I{os.path.join(REPO, 'include')}",
            "--expt-relaxed-constexpr"] + os.environ.get("MPX_NVCC_EXTRA", "").split()


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(HERE, s) for s in SOURCES]
    deps = srcs + [os.path.join(HERE, "common.cuh"), os.path.join(REPO, "include", "mpx.h")]
    if not force and os.path.exists(OUT):
        newest = max(os.path.getmtime(p) for p in deps)
        if os.path.getmtime(OUT) >= newest:
            return OUT
    objdir = os.path.join(REPO, "build", "mpx")
    os.makedirs(objdir, exist_ok=True)
    objs, jobs = [], []
    hdrs = [os.path.join(HERE, "common.cuh"), os.path.join(REPO, "include", "mpx.h")]
    for src in srcs:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if not force and os.path.exists(obj) and \
                os.path.getmtime(obj) >= max(os.path.getmtime(p) for p in [src] + hdrs):
            continue  # object up to date
        jobs.append((src, obj, subprocess.Popen([nvcc(), "-c", src, "-o", obj] + flags(),
                                                stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    for src, obj, proc in jobs:  # translation units compile concurrently
        _, err = proc.communicate()
        if proc.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{err}")
        if verbose:
            print(err, file=sys.stderr)
        with open(obj + ".ptxas.txt", "w") as fh:
            fh.write(err)
    tmp = OUT + ".tmp"
    cmd = [nvcc(), "-shared", "-o", tmp] + objs + ["-gencode", "arch=compute_100a,code=sm_100a",
                                                   "-lcuda"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stderr}")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
