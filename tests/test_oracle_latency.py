"""Pins for oracle O-3 (latency model, sec 3.4) and the partial/sequential DES.

Closed forms: SPEC.md:476-508 worked numbers for L_old / Eq. 2 / best case / Fig. 6;
Eq. 2 at n=2 for the paper's Fig. 1 shape (3 LLM rounds, 2 tool rounds, PAPER.md:44 --
durations are lost, so our illustrative numbers, R18); the DES reproduces
L_old exactly in sequential mode and always lands inside the Eq. 2 sandwich; the CodeGen
structure "lines 1-12 pipelined, only line 13 after decoding".
"""
import math
import random

import pytest
from hypothesis import given, settings, strategies as st

from oracle.latency import (Segment, best_case_improvement, curve, improvement, l_new_bounds,
                            l_old, reduction, request_latency, schedule_round)


def test_spec_worked_numbers():
    assert l_old([7], []) == 7
    assert l_old([10, 2], [10]) == 22
    assert l_old([5, 5, 5], [3, 7]) == 25
    assert l_new_bounds([10, 2], [10]) == (12, 22)
    assert l_new_bounds([10, 0], [1]) == (10, 11)
    assert l_new_bounds([4, 6], [0]) == (10, 10)
    assert best_case_improvement([10, 0], [10]) == pytest.approx(1.0)
    assert best_case_improvement([10, 0], [1000]) == pytest.approx(0.01)
    assert best_case_improvement([3, 3], [0]) == 0.0


def test_fig6_curve():
    assert curve(1.0) == pytest.approx(1.0)
    assert curve(0.01) == pytest.approx(0.01)
    assert curve(100.0) == pytest.approx(0.01)
    rs = [0.01 * 1.1 ** k for k in range(100)]
    for a, b in zip(rs, rs[1:]):
        if b <= 1:
            assert curve(b) >= curve(a)
        if a >= 1:
            assert curve(b) <= curve(a)
        assert curve(a) == pytest.approx(min(a, 1 / a))


def test_fig6_curve_equals_eq2_limit():
    # n rounds with t_i = r g_i and g_{n+1} -> 0 gives exactly f(r)
    for r in [0.05, 0.5, 1.0, 3.0, 40.0]:
        g = [1.0] * 5 + [0.0]
        t = [r] * 5
        assert best_case_improvement(g, t) == pytest.approx(curve(r))


def test_fig1_two_round_instantiation():
    """Fig. 1: 3 LLM rounds, 2 tool rounds.  Illustrative durations (ours)."""
    g, t = [300, 200, 100], [250, 400]
    assert l_old(g, t) == 1250
    lo, hi = l_new_bounds(g, t)
    assert (lo, hi) == (800, 1250)
    assert improvement(hi, lo) == pytest.approx(0.5625)
    assert reduction(hi, lo) == pytest.approx(0.36)
    # best-case partial schedule from the DES: each round's tool starts at its first token
    rounds = [{"g": 300, "segs": [Segment(0, 250)]}, {"g": 200, "segs": [Segment(0, 400)]},
              {"g": 100, "segs": []}]
    L_par, _ = request_latency(rounds, partial=True)
    L_seq, _ = request_latency(rounds, partial=False)
    assert (L_par, L_seq) == (800, 1250)


def test_improvement_vs_reduction_38_8():
    # the paper's "up to 38.8%" is L_old/L_new - 1 = 28.0% reduction
    L_new = 1.0
    L_old = 1.388
    assert reduction(L_old, L_new) == pytest.approx(0.2795, abs=1e-4)


rounds_strategy = st.lists(
    st.tuples(st.floats(0.1, 100), st.lists(st.tuples(st.floats(0, 1), st.floats(0, 50),
                                                       st.integers(0, 2)), max_size=6)),
    min_size=1, max_size=4)


@settings(max_examples=300, deadline=None)
@given(rounds_strategy, st.floats(0.1, 100))
def test_des_sandwich(rds, g_last):
    rounds = []
    for g, segs in rds:
        ss = sorted(((a * g, c, inst) for a, c, inst in segs), key=lambda x: x[0])
        rounds.append({"g": g, "segs": [Segment(a, c, inst) for a, c, inst in ss]})
    rounds.append({"g": g_last, "segs": []})
    L_par, per_p = request_latency(rounds, partial=True)
    L_seq, per_s = request_latency(rounds, partial=False)
    gs = [r["g"] for r in rounds]
    # per-round tool time t_i under sequential dispatch = makespan of the round's tools
    ts = [p[2] - p[0] for p in per_s[:-1]]
    lo, hi = l_new_bounds(gs, ts)
    assert L_seq == pytest.approx(hi)
    assert L_par <= L_seq + 1e-9
    # single-instance rounds: Eq. 2 lower bound holds
    if all(len({s.instance for s in r["segs"]}) <= 1 for r in rounds):
        assert L_par >= lo - 1e-9


def test_codegen_structure_only_last_line_after_decode():
    """13 lines decoded at a steady pace; each line's tool cost is less than one line's
    decode time except the last (render) line: in partial mode lines 1-12 finish before
    FINAL and only line 13 executes after it."""
    g = 13.0
    costs = [0.5] * 12 + [5.0]
    segs = [Segment(avail=i + 1.0, cost=c) for i, c in enumerate(costs)]
    E, starts, ends = schedule_round(segs, final_avail=g, partial=True)
    assert all(e <= g for e in ends[:12])
    assert starts[12] >= g - 1e-9 and E == pytest.approx(g + 5.0)
    E_seq, starts_s, _ = schedule_round(segs, final_avail=g, partial=False)
    assert all(s >= g for s in starts_s) and E_seq == pytest.approx(g + sum(costs))


def test_dag_dependencies_respected():
    segs = [Segment(1, 10, 0), Segment(2, 10, 1), Segment(3, 1, 2, deps=[0, 1]),
            Segment(4, 1, 3, deps=[2])]
    E, starts, ends = schedule_round(segs, final_avail=4, partial=True)
    assert starts[2] == max(ends[0], ends[1]) and starts[3] == ends[2]
    assert E == pytest.approx(14.0)
