"""Drop-in error behaviour: every call of tests/cases.py:error_cases() raises the same
exception class (or succeeds) here as in the reference (tests/golden/errors.json,
recorded from the live reference by oracle/gen_golden.py)."""
import json
import os

import pytest

import paper_2511_21513_b200 as ia
from cases import error_cases, run_error_case

pytestmark = pytest.mark.gpu
WANT = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "errors.json")))


@pytest.mark.parametrize("name", sorted(error_cases()))
def test_same_exception_as_reference(name):
    assert run_error_case(error_cases()[name], ia) == WANT[name]
