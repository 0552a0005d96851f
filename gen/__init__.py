"""Seeded synthetic input generators (shared by tests, bench and smoke).

Holds no arithmetic of the method - only patterns and bit patterns.
"""
from .configs import (CONFIG_IDS, SPEC, make, rand_values, rand_mantissas, pack_triples,
                      sha256_arrays, pattern_band, pattern_stencil5)
from .stress import stress

__all__ = ["CONFIG_IDS", "SPEC", "make", "stress", "rand_values", "rand_mantissas",
           "pack_triples", "sha256_arrays", "pattern_band", "pattern_stencil5"]
