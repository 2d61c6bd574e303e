"""Seeded per-stage parity cases shared by oracle/gen_golden.py and the tests.

Each case regenerates identical f32 inputs from its parameters (numpy PCG64),
so the committed fixtures (tests/golden/stage_cases.json) hold only the case
parameters plus digests / scalars of the reference's per-stage outputs.
Edge cases follow SURVEY.md §4 / Appendix A: L = 1, L not a tile multiple,
all-zero heads (c_int = 2^52 clamp), planted +-0.5 ties, causal and random
masks with a fully masked row, both P formats, and the (b, c) range.
"""
from __future__ import annotations

import hashlib

import numpy as np


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()[:32]


def case_list():
    cases = []
    rng = np.random.default_rng(12345)
    dims = [1, 3, 16, 64, 128]
    scales = [1e-3, 1.0, 50.0]
    masks = ["none", "none", "causal", "random"]
    for i in range(60):
        cases.append(dict(
            seed=1000 + i,
            L=int(rng.integers(1, 161)),
            d=int(dims[i % len(dims)]),
            scale=float(scales[(i // 5) % 3]),
            mask=masks[i % len(masks)],
            b=5, c=6.6, p=255, special="none"))
    # fixed shapes that hit tile edges of the GPU kernels
    for j, (L, d) in enumerate([(128, 64), (129, 64), (197, 64), (256, 128),
                                (255, 128), (300, 32), (64, 96), (200, 80)]):
        cases.append(dict(seed=2000 + j, L=L, d=d, scale=1.0,
                          mask=["none", "causal"][j % 2], b=5, c=6.6, p=255,
                          special="none"))
    for j, (b, c, p) in enumerate([(2, 6.6, 255), (3, 6.6, 255), (4, 6.6, 255),
                                   (6, 6.6, 255), (7, 6.6, 255), (8, 6.6, 255),
                                   (5, 4.4, 255), (5, 8.8, 255), (5, 6.6, 127),
                                   (4, 5.5, 127), (8, 7.7, 127)]):
        cases.append(dict(seed=3000 + j, L=96 + 7 * j, d=64, scale=1.0,
                          mask=["none", "causal", "random"][j % 3], b=b, c=c, p=p,
                          special="none"))
    for j, sp in enumerate(["zero_q", "zero_k", "zero_all", "ties", "ties",
                            "one_hot", "L1", "L1", "big_d", "masked_rows"]):
        cases.append(dict(seed=4000 + j, L=[40, 33, 17, 64, 128, 50, 1, 1, 32, 90][j],
                          d=[64, 16, 8, 32, 64, 128, 64, 1, 300, 64][j], scale=1.0,
                          mask=["none", "causal", "none", "none", "random", "none",
                                "none", "none", "causal", "random"][j],
                          b=5, c=6.6, p=[255, 255, 255, 255, 127, 255, 255, 255, 255, 255][j],
                          special=sp))
    return cases


def case_inputs(case):
    """(q, k, v, mask|None) f32 [L, d] for a case dict."""
    rng = np.random.default_rng(case["seed"])
    L, d = case["L"], case["d"]
    s = np.float32(case["scale"])
    q = rng.standard_normal((L, d), dtype=np.float32) * s
    k = rng.standard_normal((L, d), dtype=np.float32) * s
    v = rng.standard_normal((L, d), dtype=np.float32) * s
    sp = case["special"]
    if sp in ("zero_q", "zero_all"):
        q[:] = 0
    if sp in ("zero_k", "zero_all"):
        k[:] = 0
    if sp == "zero_all":
        v[:] = 0
    if sp == "ties":
        # amax = 127 -> scale = 1.0 exactly; plant halves so x/scale ties at .5
        for x in (q, k, v):
            x[:] = np.round(rng.uniform(-120, 120, size=x.shape)).astype(np.float32)
            x += np.where(rng.random(x.shape) < 0.5, np.float32(0.5), np.float32(-0.5))
            x.flat[0] = np.float32(127.0)
    if sp == "one_hot":
        q[:] = 0
        q[np.arange(L), np.arange(L) % d] = 3.0
    mask = None
    if case["mask"] == "causal":
        mask = np.triu(np.ones((L, L), dtype=bool), 1)
    elif case["mask"] == "random":
        mask = rng.random((L, L)) < 0.3
        if L > 2:
            mask[L // 2, :] = True       # one fully masked row
    if sp == "masked_rows" and L > 4:
        mask[::7, :] = True
    return q, k, v, mask
