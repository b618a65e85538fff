"""``mpfix.metrics`` (metrics.py:14-90): the same ledger classes the engine records into."""

from ..metrics import CommMetrics, OpCounters  # noqa: F401

__all__ = ["CommMetrics", "OpCounters"]
