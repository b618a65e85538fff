"""``mpfix.protocols.derived`` names (derived.py:20-170)."""

from . import (evaluate_poly, evaluate_square_completed, lmo, max_vec, scale_fixed,  # noqa: F401
               truncate, unsigned_truncate)
