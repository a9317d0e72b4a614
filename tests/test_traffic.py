"""Traffic oracle (paper_2205_01598_b200/traffic.py + csrc/traffic.cu) against
the reference's simulate_traffic (pkg/src/levelmpk/traffic.py:192-226): the
fixtures in tests/golden/golden_r2.* were produced by the reference itself
(tests/golden/make_golden_r2.py).  The replay is host code, so these run
without a GPU; the model cases follow pkg/tests/test_traffic.py."""

import json
import pathlib
import types

import numpy as np
import pytest

import paper_2205_01598_b200 as lm

GOLD = pathlib.Path(__file__).resolve().parent / "golden"
FACTS = json.loads((GOLD / "golden_r2.json").read_text())
ARR = np.load(GOLD / "golden_r2.npz")


def _plan(name, p_m):
    g = lambda k: ARR[f"traffic/{name}/{k}"]
    rp, col = g("row_ptr"), g("col")
    a = types.SimpleNamespace(row_ptr=rp, col=col, n_rows=rp.shape[0] - 1, n_nz=int(rp[-1]))
    return types.SimpleNamespace(a=a, p_m=p_m, row_start=g("row_start"), row_end=g("row_end"),
                                 power=g("power"), in_slot=g("in_slot"), out_slot=g("out_slot"))


@pytest.mark.parametrize("case", FACTS["traffic"], ids=lambda c: f"{c['plan']}-{c['cap']}-{c['line']}")
def test_report_equals_reference(case):
    rep = lm.simulate_traffic(_plan(case["plan"], case["p_m"]), lm.CacheModel(case["cap"], case["line"]))
    assert np.array_equal(rep.by_power, ARR[case["key"]])
    for k in ("matrix_bytes", "row_ptr_bytes", "vector_bytes", "n_accesses", "n_misses"):
        assert getattr(rep, k) == case[k], k
    assert rep.n_hits + rep.n_misses == rep.n_accesses
    assert rep.code_balance == case["code_balance"]


def test_zero_capacity_is_one_sweep_per_power():
    c = next(c for c in FACTS["traffic"] if c["plan"] == "base-3d8-p3" and c["cap"] == 0)
    rep = lm.simulate_traffic(_plan(c["plan"], c["p_m"]), lm.CacheModel(0))
    assert rep.matrix_bytes == c["p_m"] * 12 * c["n_nz"]
    assert rep.row_ptr_bytes == c["p_m"] * 4 * c["n_rows"]
    assert rep.n_misses == rep.n_accesses and rep.n_hits == 0


def test_lru_monotone_in_capacity():
    plan = _plan("p2p-3d8-p4", 4)
    totals = [lm.simulate_traffic(plan, lm.CacheModel(s)).total_bytes
              for s in (0, 4_096, 16_384, 65_536, 1 << 20, 1 << 26)]
    assert totals == sorted(totals, reverse=True)


def test_roofline_and_model_validation():
    assert lm.roofline_estimate(6.0, 116e9) == pytest.approx(19.33e9, rel=1e-3)
    assert lm.roofline_estimate(1.0, 1.0) == 1.0
    for bad in ((0.0, 1.0), (1.0, -5.0)):
        with pytest.raises(ValueError):
            lm.roofline_estimate(*bad)
    with pytest.raises(ValueError):
        lm.CacheModel(-1)
    with pytest.raises(ValueError):
        lm.CacheModel(100, line_bytes=7)


def test_bad_items_are_rejected():
    plan = _plan("base-3d8-p3", 3)
    plan.row_end = plan.row_end + 10_000
    with pytest.raises((ValueError, IndexError)):
        lm.simulate_traffic(plan, lm.CacheModel(1000))
