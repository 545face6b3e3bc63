"""O-3: latency model and partial-vs-sequential schedule -- TEST INFRASTRUCTURE.

PAPER.md sec 3.4 (lines 158-171):
  g_i  token-generation time of round i (prefill + decode), t_i tool time of round i;
  L_old = sum_{i=1..n} (g_i + t_i) + g_{n+1}
  Eq. 1: max{g_i, t_i} <= L_i <= g_i + t_i
  Eq. 2: sum max{g_i, t_i} + g_{n+1} <= L_new <= L_old
  best-case improvement = L_old / (sum max{g_i,t_i} + g_{n+1}) - 1
  Fig. 6 curve: ratio r = t_i/g_i fixed, g_{n+1} negligible:
      f(r) = (1 + r)/max(1, r) - 1 = min(r, 1/r)
"Improvement" is the paper's L_old/L_new - 1; "reduction" is 1 - L_new/L_old
(R16).  The DES below is the plain schedule of SURVEY.md 8(c) O-3.
"""
from __future__ import annotations

from dataclasses import dataclass, field


def l_old(g, t) -> float:
    n = len(t)
    assert len(g) == n + 1
    return sum(g[i] + t[i] for i in range(n)) + g[n]


def l_new_bounds(g, t):
    n = len(t)
    assert len(g) == n + 1
    lower = sum(max(g[i], t[i]) for i in range(n)) + g[n]
    return lower, l_old(g, t)


def best_case_improvement(g, t) -> float:
    lower, upper = l_new_bounds(g, t)
    if lower <= 0:
        raise ZeroDivisionError("degenerate latency model (lower bound 0)")
    return upper / lower - 1.0


def improvement(l_seq: float, l_par: float) -> float:
    return l_seq / l_par - 1.0


def reduction(l_seq: float, l_par: float) -> float:
    return 1.0 - l_par / l_seq


def curve(r: float) -> float:
    """Fig. 6 theoretical improvement at tool/decode ratio r (> 0)."""
    return (1.0 + r) / max(1.0, r) - 1.0


@dataclass
class Segment:
    avail: float            # time the segment became available to the host
    cost: float             # tool execution time of the segment
    instance: int = 0       # tool instance; one instance executes its segments serially
    deps: list = field(default_factory=list)  # indices of earlier segments of the round


def schedule_round(segments: list[Segment], final_avail: float, partial: bool):
    """Start/end time of every segment.  Partial: start = max(avail, instance free, deps
    done).  Sequential ("tool invocation always happens after decoding to
    the EOS"): every avail := final_avail.  Returns (E, starts, ends) with E the time all
    tool work of the round is done (final_avail if there is none)."""
    inst_free: dict[int, float] = {}
    starts, ends = [], []
    for j, s in enumerate(segments):
        a = s.avail if partial else final_avail
        dep_done = max((ends[d] for d in s.deps), default=float("-inf"))
        st = max(a, inst_free.get(s.instance, float("-inf")), dep_done)
        en = st + s.cost
        starts.append(st)
        ends.append(en)
        inst_free[s.instance] = en
    E = max(ends, default=final_avail)
    return E, starts, ends


def request_latency(rounds, partial: bool, t0: float = 0.0):
    """rounds: list of dicts with keys g (generation time of the round, incl. injection
    prefill), segs (list of Segment with avail relative to the round start).  Round i+1
    starts when round i's decoding and tools are both done.  Returns
    (latency, per-round (g_i, t_i, L_i))."""
    t = t0
    per = []
    for rd in rounds:
        g = rd["g"]
        segs = [Segment(t + s.avail, s.cost, s.instance, list(s.deps)) for s in rd["segs"]]
        final = t + g
        E, _, _ = schedule_round(segs, final, partial)
        end = max(E, final)
        tool_time = sum(s.cost for s in segs)
        per.append((g, tool_time, end - t))
        t = end
    return t - t0, per
