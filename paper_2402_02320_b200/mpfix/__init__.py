"""Reference-compatible facade: the ``mpfix`` API (``/root/reference/pkg/src/mpfix``
``__init__.py:5-45``) on the B200 engine.

Callers written against the reference keep their code: one
``PartySession(party, n, mesh, store)`` per party, ``AShare(np.uint64[...],
width, frac)`` / ``BShare(np.uint8[...])`` handles, numpy results from
``open_many``, ``memory_stores`` / ``DemandCounter`` / ``InProcHub`` /
``NullMesh`` for the ``tests/helpers.py:17-78`` harness pattern. Shares stay
in HBM between calls and every step runs in libmpx kernels; numpy copies
happen only where the reference API hands arrays back (``.values``,
``.bits``, openings).

``install()`` registers this package as ``mpfix`` in ``sys.modules`` so code
doing ``from mpfix.protocols import mul`` runs unmodified.

Out of scope: the scenario runner / config / report / CLI and
the TCP transport.
"""

from __future__ import annotations

import sys

from . import metrics, nn, nonlinear, preprocessing, protocols, ring, session, sharing, transport
from .metrics import CommMetrics, OpCounters
from .nn import (AttentionDims, LinearLayer, attention_block, fold_base2, linear_layer, maxcut, mlp_forward,
                 relu, softmax, softmax_parts)
from .nonlinear import (DEFAULT_PARAMS, ApproxParams, attention_exp, baseline_exp, exponentiation, logarithm,
                        reciprocal)
from .session import PartySession
from .sharing import AShare, BShare, reconstruct_arith, reconstruct_bits, share_arith, share_bits

__version__ = "0.1.0"

_SUBMODULES = ("ring", "sharing", "session", "preprocessing", "transport", "metrics", "protocols",
               "protocols.basic", "protocols.derived", "nonlinear", "nn")


def install(name: str = "mpfix") -> None:
    """Alias this package (and its submodules) as ``name`` in ``sys.modules``."""
    import importlib
    sys.modules[name] = sys.modules[__name__]
    for sub in _SUBMODULES:
        sys.modules[f"{name}.{sub}"] = importlib.import_module(f"{__name__}.{sub}")


__all__ = [
    "AShare", "BShare", "share_arith", "share_bits", "reconstruct_arith", "reconstruct_bits",
    "PartySession", "CommMetrics", "OpCounters", "ApproxParams", "DEFAULT_PARAMS",
    "reciprocal", "exponentiation", "logarithm", "baseline_exp", "attention_exp",
    "AttentionDims", "LinearLayer", "relu", "maxcut", "softmax", "softmax_parts",
    "attention_block", "linear_layer", "mlp_forward", "fold_base2", "install",
    "ring", "sharing", "session", "preprocessing", "transport", "metrics", "protocols", "nonlinear", "nn",
]
