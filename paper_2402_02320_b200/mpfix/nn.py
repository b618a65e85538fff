"""``mpfix.nn`` (nn.py:48-206) over the engine: ReLU, MaxCut, softmax,
attention and public-weight linear layers."""

from .. import nn as _EN
from ..nn import AttentionDims, LinearLayer, fold_base2  # noqa: F401
from ._bridge import wrap_op

relu = wrap_op(_EN.relu, "relu")
maxcut = wrap_op(_EN.maxcut, "maxcut")
softmax_parts = wrap_op(_EN.softmax_parts, "softmax_parts")
softmax = wrap_op(_EN.softmax, "softmax")
attention_block = wrap_op(_EN.attention_block, "attention_block")
linear_layer = wrap_op(_EN.linear_layer, "linear_layer")
mlp_forward = wrap_op(_EN.mlp_forward, "mlp_forward")

__all__ = ["AttentionDims", "LinearLayer", "fold_base2", "relu", "maxcut", "softmax_parts", "softmax",
           "attention_block", "linear_layer", "mlp_forward"]
