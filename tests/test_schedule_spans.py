"""Schedules of refined trees without a GPU: the level-group trees the
reference built (tests/golden/golden_r2.json) are reconstructed from their
JSON records and scheduled here; for p_m < 3 (no diamond halos,
groups.py:360-362) the flattened items need no dependency analysis, so the
whole item list must equal the reference's (plan.py:52-70)."""

import json
import pathlib

import numpy as np
import pytest

from paper_2205_01598_b200.groups import (HaloLevel, LevelGroup, LevelGroupTree, NeighborSplit, RefinedSpan,
                                          _flagged_runs, _merge_spans)
from paper_2205_01598_b200.levels import LevelSet
from paper_2205_01598_b200.plan import _flatten, _validate_coverage
from paper_2205_01598_b200.schedule import (DIAMOND, INPUT_ONLY, INSIDE, OUTPUT_ONLY, LpNode, SubgraphCall,
                                            build_schedule, classify_outer)

GOLD = pathlib.Path(__file__).resolve().parent / "golden"
FACTS = json.loads((GOLD / "golden_r2.json").read_text())["recursion"]
ARR = np.load(GOLD / "golden_r2.npz")


def tree_from_record(rec):
    groups = [LevelGroup(*g[:6], violates=g[6]) for g in rec["groups"]]
    tree = LevelGroupTree(stage=rec["stage"], groups=groups)
    for s in rec["spans"]:
        child = tree_from_record(s["tree"])

        def halo(h):
            if h is None:
                return None
            return NeighborSplit(h["side"], [tuple(g) for g in h["groups"]],
                                 {int(gi): [HaloLevel(lv["row_start"], lv["row_end"],
                                                      [tuple(p) for p in lv["portions"]], lv["keys"])
                                            for lv in lvs] for gi, lvs in h["levels"].items()})
        span = RefinedSpan(s["first_group"], s["last_group"], s["row_start"], s["row_end"],
                           LevelSet(np.array(s["level_ptr"]), s["root"]), child, halo(s["left"]), halo(s["right"]))
        for g in groups[span.first_group:span.last_group + 1]:
            g.children = child
        tree.spans.append(span)
    return tree


@pytest.mark.parametrize("key", sorted(k for k, r in FACTS.items() if r["p_m"] < 3))
def test_flat_items_without_halos_equal_reference(key):
    rec = FACTS[key]
    tree = tree_from_record(rec["tree"])
    sched = build_schedule(tree, rec["p_m"])
    items = _flatten(sched, tree, None)
    got = np.array([[it.row_start, it.row_end, it.power, it.stage, 0 if it.kind == "group" else 1,
                     it.boundary_end] for it in items], dtype=np.int64)
    assert np.array_equal(got, ARR[f"{key}/items"])
    assert [list(it.label) for it in items] == rec["labels"]


@pytest.mark.parametrize("key", sorted(FACTS))
def test_schedule_structure(key):
    """Every (group, power) node appears exactly once -- plain, inside a call
    or as a diamond node -- inputs precede their call, outputs follow it."""
    rec = FACTS[key]
    tree, p_m = tree_from_record(rec["tree"]), rec["p_m"]
    sched = build_schedule(tree, p_m)
    seen = set()
    for step, it in enumerate(sched.items):
        assert it.exec_step == step
        if isinstance(it, LpNode):
            assert (it.group, it.power) not in seen
            seen.add((it.group, it.power))
            span = next((s for s in tree.spans
                         if classify_outer(it.group, it.power, s.first_group, s.last_group, p_m)), None)
            if span is not None:
                call = next(c for c in sched.items if isinstance(c, SubgraphCall) and c.span is span)
                assert it.classification in (INPUT_ONLY, OUTPUT_ONLY)
                assert (it.exec_step < call.exec_step) == (it.classification == INPUT_ONLY)
        else:
            s = it.span
            inside = {(i, p) for i in range(s.first_group, s.last_group + 1) for p in range(1, p_m + 1)}
            dia = set(it.diamond_nodes)
            assert len(dia) == len(it.diamond_nodes) and not (inside | dia) & seen
            assert all(classify_outer(i, p, s.first_group, s.last_group, p_m) == DIAMOND for i, p in dia)
            seen |= inside | dia
    assert seen == {(i, p) for i in range(len(tree.groups)) for p in range(1, p_m + 1)}
    assert len([c for c in sched.items if isinstance(c, SubgraphCall)]) == len(tree.spans)


def test_span_merging_and_flagged_runs():
    g = lambda v: LevelGroup(0, 1, 1, 1, 0, 1, violates=v)
    groups = [g(v) for v in (0, 1, 1, 0, 0, 1, 0, 0, 0, 0, 0, 1, 1, 1)]
    runs = _flagged_runs(groups)
    assert runs == [(1, 2), (5, 5), (11, 13)]
    assert _merge_spans(runs, 1) == runs
    assert _merge_spans(runs, 2) == runs  # gaps 3 and 6 exceed 2 * (p_m - 1) = 2
    assert _merge_spans(runs, 3) == [(1, 5), (11, 13)]
    assert _merge_spans(runs, 4) == [(1, 13)]
    assert _merge_spans([], 4) == []
    assert classify_outer(3, 1, 4, 6, 5) == INPUT_ONLY and classify_outer(5, 2, 4, 6, 5) == INSIDE
    assert classify_outer(8, 5, 4, 6, 5) == OUTPUT_ONLY and classify_outer(0, 3, 4, 6, 4) is None
