"""Map golden fixture tags to case descriptions (shared by oracle and GPU tests)."""

import glob
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
STRATS = ("reference", "wq", "hybrid", "dwq")


def load(tag):
    return dict(np.load(os.path.join(HERE, f"{tag}.npz")))


def tags():
    """Full/sampled goldens in the dump_case format (headline goldens excluded)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "*.npz"))
                  if not os.path.basename(p).startswith(("rules_", "config5")))


def headline_tags():
    """Config-5 recipe goldens in the dump_huge format (make_golden.py --huge/--p4small)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "config5*.npz")))


def headline_nel(tag):
    return 2048 if tag == "config5" else int(tag.split("_")[1])


def describe(tag):
    """-> dict(kind, name, nel, p, coeff, target_name, strategies, full)."""
    parts = tag.split("_")
    if parts[0] == "case":
        return dict(kind="case", name=parts[1], nel=int(parts[2]), p=int(parts[3]), coeff=None,
                    target="default")
    if tag == "config1":
        return dict(kind="config", idx=1, nel=16, p=2, coeff=None, target="config1")
    if tag == "config2":
        return dict(kind="ccircle", nel=64, p=3, coeff=None, target="config23")
    if tag == "config3":
        return dict(kind="ccircle", nel=128, p=4, coeff=None, target="config23")
    if parts[0] == "ccircle":
        return dict(kind="ccircle", nel=int(parts[1]), p=int(parts[2]), coeff=None, target="config23")
    if parts[0] == "bspline" and parts[1] == "detj":
        return dict(kind="bspline", nel=int(parts[2]), p=int(parts[3]), coeff="detj", target="config5")
    if parts[0] == "bspline":
        return dict(kind="bspline", nel=int(parts[1]), p=int(parts[2]), coeff=None, target="config5")
    if parts[0] == "config4":
        return dict(kind="bspline", nel=256, p=int(parts[1][1:]), coeff="detj", target=None)
    raise KeyError(tag)


def strategies_in(d):
    return [s for s in STRATS if f"{s}_hash" in d]
