"""dataflow_audit parity: the (tag, dtype) stream of every audited call equals the
one the LIVE reference recorded (tests/golden/audit.json, oracle/gen_golden.py;
reference softmax.py:207-228, notes at :279-298, :394-398 and pipeline.py:248),
and the tensors between the QK^T GEMM and the P.V GEMM are integer-only
(SPEC.md:335)."""
import json
import os

import numpy as np
import pytest

from cases import audit_cases, run_audit_case

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "audit.json")


def _golden():
    return json.load(open(GOLD))


def test_audit_golden_covers_every_case():
    g = _golden()
    assert set(g) == set(audit_cases())
    for name, tags in g.items():
        for tag, dt in tags:
            assert tag in ("logits", "index_table", "lut", "mask", "prob", "pv_in", "surrogates")
            np.dtype(dt)


def test_audit_sink_restored_and_nested():
    import paper_2511_21513_b200 as ia
    from paper_2511_21513_b200 import softmax as sm
    outer, inner = [], []
    with ia.dataflow_audit(outer):
        sm._note("a", np.int32)
        with ia.dataflow_audit(inner):
            sm._note("b", np.uint8)
        sm._note("c", np.int8)
    sm._note("d", np.int32)  # no sink installed: dropped
    assert [t for t, _ in outer] == ["a", "c"] and [t for t, _ in inner] == ["b"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(audit_cases()))
def test_audit_stream_matches_reference(name):
    import paper_2511_21513_b200 as ia
    got = run_audit_case(audit_cases()[name], ia)
    assert got == _golden()[name]
    # integer-only dataflow between gemm_qk and gemm_pv
    for tag, dt in got:
        assert np.issubdtype(np.dtype(dt), np.integer), (tag, dt)
