"""Seeded random streams, bit-compatible with the reference's spawn-key
scheme (`pkg/src/nidpipe/rng.py:13-33`) so that a given (seed, key) yields the
same gamma constants and embedding coefficients on both sides."""

from __future__ import annotations

import numpy as np

EMBED = 1
LIFT = 2
START_COEFFS = 3
GAMMA = 4
SQUARE = 5
# keys used only by this framework's synthetic configs (not in the reference)
CONFIG_COEFFS = 101
CONFIG_CANDIDATES = 102
CONFIG_SAMPLE = 103


def stream(seed: int, *key: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=key))


def unit_complex(gen: np.random.Generator, n: int | None = None):
    """exp(i*theta), theta ~ U[0, 2pi) (rng.py:24-27)."""
    return np.exp(1j * gen.uniform(0.0, 2.0 * np.pi, size=n))


def random_complex(gen: np.random.Generator, n: int | None = None):
    """Modulus ~ U(0.5, 1.5) times a unit direction (rng.py:30-33)."""
    r = gen.uniform(0.5, 1.5, size=n)
    return r * unit_complex(gen, n)


def gamma_for(seed: int, *extra: int) -> complex:
    """The gamma constant the reference draws for solve_top (cascade.py:226)
    and for cascade level d (cascade.py:309)."""
    return complex(unit_complex(stream(seed, GAMMA, *extra)))
