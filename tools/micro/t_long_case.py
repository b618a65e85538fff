"""Run one mpx_beaver_tc_long case against the numpy restatement (debug aid):
    python tools/micro/t_long_case.py L M K N p0 xt"""
import sys
import os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np  # noqa: E402
from test_long_tc import _run  # noqa: E402

L, M, K, N, p0, xt = (int(v) for v in sys.argv[1:7])
got, want = _run(L, M, K, N, p0, bool(xt), 7)
print(sys.argv[1:7], "equal", np.array_equal(got, want))
