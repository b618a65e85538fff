"""GPU: the non-default party-split layouts of the sim-mode fused kernels
(csrc/fused_ops.cu, "party split") stay bit-exact against the per-round path
and the CPU oracle. The layout is chosen once per process from MPX_SPLIT4 /
MPX_SPLIT8, so each forced layout reruns tests/test_fused_ops.py's cases for
that party count in a child process."""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("env,n", [({"MPX_SPLIT8": "2"}, 8), ({"MPX_SPLIT8": "4"}, 8),
                                   ({"MPX_SPLIT4": "0"}, 4), ({"MPX_SPLIT4": "1"}, 4)],
                         ids=["n8-2lanes", "n8-4lanes", "n4-1lane", "n4-2lanes"])
def test_forced_split_layout_bit_exact(env, n):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    target = os.path.join(HERE, "test_fused_ops.py")
    col = subprocess.run([sys.executable, "-m", "pytest", target, "--collect-only", "-q", "-p", "no:cacheprovider"],
                         cwd=os.path.dirname(HERE), capture_output=True, text=True, timeout=300)
    ids = [ln.strip() for ln in col.stdout.splitlines() if f"[{n}-" in ln]
    assert ids, col.stdout[-2000:]
    res = subprocess.run([sys.executable, "-m", "pytest", "-m", "gpu", "-x", "-q", "-p", "no:cacheprovider"] + ids,
                         cwd=os.path.dirname(HERE), env={**os.environ, **env}, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
    assert " passed" in res.stdout, res.stdout[-2000:]
