"""InverseOracle: ||A^-1||_2 through LU factors (condest.hpp:109-152, lu.hpp).

Placeholder until the device factorisation lands; every entry point raises.
"""
from __future__ import annotations

from .errors import Unsupported


class InverseOracle:
    def __init__(self, factors):
        self.factors = factors

    def dimension(self) -> int:
        return self.factors.n


def _inverse_projected_adam(oracle, cfg, observer):
    raise Unsupported("InverseOracle is not available in this build yet")


def _inverse_estimate_norm(oracle, cfg, restarts):
    raise Unsupported("InverseOracle is not available in this build yet")
