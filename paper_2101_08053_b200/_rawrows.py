"""Raw (non-separable) rows: cut rows, c != 1 rows, the reference strategy."""

from __future__ import annotations

import numpy as np

from ._lib import CUT, INTERIOR


def needs_raw(f):
    if f.strategy == "reference" or not f.coeff.identity:
        return True
    return bool(np.any(f.config.func_class == CUT))


def build_dwq_sets(f, r1, r2):
    return {}


def run_phase(f, phase):
    if needs_raw(f):
        raise NotImplementedError("raw rows not built yet")
