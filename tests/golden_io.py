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
