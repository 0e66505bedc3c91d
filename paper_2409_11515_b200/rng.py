"""Seeded sampling, mirrored from condkit/rng.hpp through the C-ABI (host code in
the native library): mix_seed (rng.hpp:23-28) and random_unit_vector
(rng.hpp:68-77, mt19937_64 + Box-Muller), bit-identical to the reference."""
from __future__ import annotations

import numpy as np

from . import _lib


def mix_seed(base: int, stream: int) -> int:
    return int(_lib.load().ck_mix_seed(base & (2**64 - 1), stream & (2**64 - 1)))


def random_unit_vectors(seed: int, n: int, count: int = 1) -> np.ndarray:
    """`count` successive random_unit_vector(n, gen) draws of mt19937_64(seed)."""
    out = np.empty((count, n))
    _lib.check(_lib.load().ck_random_unit_vectors(seed & (2**64 - 1), n, count, _lib.dptr(out)),
               "ck_random_unit_vectors")
    return out


def random_unit_vector(n: int, seed: int) -> np.ndarray:
    return random_unit_vectors(seed, n, 1)[0]
