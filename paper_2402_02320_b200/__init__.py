"""B200-native secret-shared fixed-point engine (arXiv 2402.02320 hot path).

Drop-in for the reference package ``mpfix``'s protocol API (sharing, opening,
Beaver mul/matmul, truncation, comparison, Reciprocal/Exp/Log, softmax and
attention) with every local step in hand-written sm_100a kernels
(``libmpx.so``, C ABI in ``include/mpx.h``) and openings as NCCL collectives
(one GPU per party) or on-device reductions (all parties on one GPU).
"""

__version__ = "0.1.0"

from . import _lib
from .metrics import CommMetrics, OpCounters
from .preprocessing import (DemandCounter, MaterialKey, MaterialStore, PreprocessingExhausted,
                            device_store)
from .session import PartySession, SimSession, dry_run, run_sim
from .sharing import AShare, BShare, add_public, public_ashare, xor_public
from .nonlinear import (DEFAULT_PARAMS, ApproxParams, attention_exp, baseline_exp, exponentiation,
                        logarithm, reciprocal)
from .nn import (AttentionDims, LinearLayer, attention_block, fold_base2, linear_layer, maxcut,
                 mlp_forward, relu, softmax, softmax_parts)

__all__ = [
    "AShare", "BShare", "PartySession", "SimSession", "run_sim", "dry_run",
    "CommMetrics", "OpCounters", "MaterialKey", "MaterialStore", "DemandCounter",
    "PreprocessingExhausted", "device_store", "add_public", "public_ashare", "xor_public",
    "ApproxParams", "DEFAULT_PARAMS", "reciprocal", "exponentiation", "logarithm",
    "baseline_exp", "attention_exp", "AttentionDims", "LinearLayer", "relu", "maxcut",
    "softmax", "softmax_parts", "attention_block", "linear_layer", "mlp_forward", "fold_base2",
]
