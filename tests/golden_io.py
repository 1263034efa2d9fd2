"""Readers for the committed golden fixtures (tests/golden/*.npz, made by make_golden.py)."""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def unpack(npz):
    """Inverse of make_golden.pack: a list of per-matrix dicts."""
    keys = [k for k in npz.files if not k.endswith("_off")]
    count = npz[keys[0] + "_off"].size - 1
    out = []
    for i in range(count):
        d = {}
        for k in keys:
            off = npz[k + "_off"]
            d[k] = npz[k][off[i]:off[i + 1]]
        out.append(d)
    return out


def spmv_suite(vdt="float64", idt="int32"):
    return unpack(load(f"spmv_suite_{vdt}_{idt}.npz"))


def solver_meta():
    with open(os.path.join(GOLDEN, "solvers.json")) as fh:
        return json.load(fh)
