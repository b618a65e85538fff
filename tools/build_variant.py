"""Build an A/B variant of libmpx with extra nvcc defines (tuning sweeps):

    python tools/build_variant.py NAME -DMPX_LOG_MINB=4 [...]
    -> paper_2402_02320_b200/libmpx_NAME.so ; select it with MPX_LIB=<path>
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_02320_b200.csrc import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    objdir = os.path.join(B.REPO, "build", f"var_{name}")
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    for src in B.SOURCES:
        obj = os.path.join(objdir, src + ".o")
        objs.append(obj)
        procs.append(subprocess.Popen([B.nvcc(), "-c", os.path.join(B.HERE, src), "-o", obj] + B.flags() + defs,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    for p in procs:
        _, err = p.communicate()
        if p.returncode:
            raise SystemExit(err)
    out = os.path.join(B.PKG, f"libmpx_{name}.so")
    subprocess.run([B.nvcc(), "-shared", "-o", out] + objs + ["-gencode", "arch=compute_100a,code=sm_100a", "-lcuda"],
                   check=True)
    print(out)


if __name__ == "__main__":
    main()
