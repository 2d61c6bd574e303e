"""Loaders for the committed fixtures in tests/golden/ (made by oracle/gen_golden.py)."""
import json
import os

import numpy as np

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def kats():
    return json.load(open(os.path.join(GOLD, "kats.json")))


def stage_cases():
    return json.load(open(os.path.join(GOLD, "stage_cases.json")))


def stage_small():
    return dict(np.load(os.path.join(GOLD, "stage_small.npz")))


def configs():
    return json.load(open(os.path.join(GOLD, "configs.json")))


def f32(h):
    return np.float32(float.fromhex(h))


def unit_mismatches(out, wl, name):
    """(b, h) units of a [B, H, L, d] f32 output whose valid rows do not hash to the
    live reference's digest in configs.json (or whose padding rows are not +0.0).
    Returns (bad units, units checked); raises KeyError if the config has no golden."""
    from cases import digest
    G = configs()[name]
    B, H = out.shape[:2]
    lens = wl.lengths()
    bad, u = [], 0
    for b in range(B):
        for h in range(H):
            n = int(lens[b])
            if digest(out[b, h, :n]) != G["unit_digests"][u] or out[b, h, n:].view(np.uint32).any():
                bad.append((b, h))
            u += 1
    return bad, u
