"""Pin the CPU oracle (oracle/fvb_oracle.c) against the reference's own outputs.

The golden vectors were produced by the reference (`fvbatch.kernel.update_patch_batch`,
cross-checked against `pkg/tests/oracle.py`) by tests/golden/make_golden.py.
"""

import numpy as np
import pytest

import oracle
from conftest import assert_bits_equal, load_golden


def _solution_cases():
    import json, os
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)["solution_cases"]


def _error_cases():
    import json, os
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)["error_cases"]


@pytest.mark.parametrize("case", _solution_cases(), ids=lambda c: c["name"])
def test_oracle_matches_reference_bitwise(case):
    b = load_golden(case["file"])
    qout, lam, st = oracle.update(case["dim"], case["p"], case["gamma"], b.QIn, b.cell_size, b.dt)
    assert st == 0
    assert_bits_equal(qout, b.QOut, case["name"] + " QOut")
    assert_bits_equal(lam, b.max_eigenvalue, case["name"] + " max_eigenvalue")


@pytest.mark.parametrize("case", _error_cases(), ids=lambda c: c["name"])
def test_oracle_error_semantics_match_reference(case):
    b = load_golden(case["file"])
    d, p = case["dim"], case["p"]
    info = oracle.locate(d, p, case["gamma"], b.QIn)
    _, _, st = oracle.update(d, p, case["gamma"], b.QIn, b.cell_size, b.dt)
    any_raise = any(e["raised"] for e in case["expect"])
    assert (st == 2) == any_raise
    for exp in case["expect"]:
        n = b.n_patches
        if exp["strategy"] == "seq":
            chunks = 1
        else:
            chunks = min(exp["workers"], n)
        ordering = 0 if exp["ordering"] == "patchwise" else 1
        got = oracle.first_error(d, p, info, ordering, chunks)
        if not exp["raised"]:
            assert got is None
            continue
        patch, box, lin, kind = got
        assert patch == exp["patch"], exp
        assert list(oracle.box_volume(d, p, box, lin)) == exp["volume"], exp
        msg = "non-positive density in pressure closure" if kind == 1 else \
            "negative pressure in eigenvalue evaluation"
        assert msg == exp["message"], exp


def _halo_cases():
    import json, os
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f).get("halo_cases", [])


@pytest.mark.parametrize("case", _halo_cases(), ids=lambda c: c["name"])
def test_oracle_halo_project_matches_reference(case):
    b = load_golden(case["file"])
    qin = oracle.halo_project(case["dim"], case["p"], b.QOut, case["grid"], case["periodic"])
    assert_bits_equal(qin, b.QIn, case["name"])
