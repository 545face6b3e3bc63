"""Host runtime (Partial vs Sequential dispatch) on CPU, against a fake
engine that replays the oracle's segment records one decode step at a time.

Checks: partial never loses to sequential; the measured latencies agree with the O-3 DES
recomputed from the logged availability times; CodeGen structure; Eq. 2
sandwich per request; validation aborts early only in partial mode."""
import threading
import time

import pytest

import oracle
from oracle.scan import round_records
from inputs.tool_workloads import TOOLS, build
from paper_2406_00059_b200 import capi
from paper_2406_00059_b200.engine import Record
from paper_2406_00059_b200.runtime import Runtime, summarize

STEP_S = 0.002


class FakeEngine:
    """Implements the subset of engine.Engine the runtime uses."""

    def __init__(self, vocab, tools):
        self.vocab = vocab
        self.tools = tools  # tool_id -> (kind, delims)
        self.lock = threading.Lock()
        self.reqs = {}
        self.queue = []
        self.next_id = 1
        self.pending_cancel = set()

    def submit_request(self, prompt, max_new, tool_id=-1, mode=0, forced=None, synth_prefix_len=0, synth_seed=0,
                       reserve_tokens=0):
        with self.lock:
            rid = self.next_id
            self.next_id += 1
            self.reqs[rid] = {"round": 0, "seq": 0, "tool": tool_id, "forced": list(forced), "t": 0,
                              "feed": len(prompt) - 1, "active": True, "recs": None}
            self._prep(rid)
            return rid

    def _prep(self, rid):
        r = self.reqs[rid]
        if r["tool"] >= 0:
            kind, delims = self.tools[r["tool"]]
            recs, _ = round_records(r["forced"], self.vocab, kind, delims, 4096, r["round"], r["seq"])
        else:
            recs, _ = round_records(r["forced"], self.vocab, oracle.PARSER_LITERAL, [b"\x00\x01"], 1 << 30,
                                    r["round"], r["seq"])
            recs = [x for x in recs if x.flags & 1]
            recs = [oracle.scan.Record(x.round, r["seq"], x.token_index, 0, 0, x.delim_id, x.flags, b"")
                    for x in recs]
        r["recs"] = recs

    def step(self):
        time.sleep(STEP_S)
        with self.lock:
            for rid, r in self.reqs.items():
                if not r["active"]:
                    continue
                if rid in self.pending_cancel:
                    self.pending_cancel.discard(rid)
                    r["active"] = False
                    self.queue.append(Record(rid, r["round"], r["seq"], 0, max(r["t"] - 1, 0), 0, 0, 0xFFFF,
                                             capi.SEG_FINAL | capi.SEG_CANCELLED, 0, b""))
                    r["seq"] += 1
                    continue
                if r["feed"] > 0:
                    r["feed"] -= 1
                    continue
                t = r["t"]
                for x in r["recs"]:
                    if x.token_index == t:
                        self.queue.append(Record(rid, x.round, x.seq, 0, x.token_index, x.byte_offset, x.byte_len,
                                                 x.delim_id, x.flags, 0, x.data))
                        r["seq"] = x.seq + 1
                r["t"] += 1
                if r["t"] >= len(r["forced"]):
                    r["active"] = False
        return None

    def poll_segments(self, with_bytes=True):
        with self.lock:
            q, self.queue = self.queue, []
        return q

    def inject_observation(self, rid, tokens, max_new, forced=None):
        with self.lock:
            r = self.reqs[rid]
            r.update(round=r["round"] + 1, forced=list(forced), t=0, feed=len(tokens) + 1, active=True)
            self._prep(rid)

    def cancel_request(self, rid):
        with self.lock:
            if self.reqs[rid]["active"]:
                self.pending_cancel.add(rid)

    def release_request(self, rid):
        pass

    def sync(self):
        pass


def oracle_des(rounds, partial):
    """The runtime's logged timelines through the oracle's O-3 schedule (oracle/latency.py)."""
    from oracle.latency import Segment, request_latency
    rr = [{"g": r["g"], "segs": [Segment(a, c, i, d) for a, c, i, d in r["segs"]]} for r in rounds]
    return request_latency(rr, partial)


def run(workload, B, mode):
    from inputs.vocab import synthetic_vocab
    vocab = synthetic_vocab(32000)
    ids = {name: i for i, name in enumerate(TOOLS)}
    kinds = {i: (getattr(oracle, TOOLS[n][0]), TOOLS[n][1]) for n, i in ids.items()}
    eng = FakeEngine(vocab, kinds)
    _, specs = build(workload, B, ids, seed=9)
    rt = Runtime(eng, mode)
    logs = rt.run(specs, timeout_s=120)
    return logs, summarize(logs, mode, des=oracle_des)


@pytest.mark.parametrize("workload", ["codegen", "codegen_fence", "search", "search_call", "planning"])
def test_partial_beats_sequential_and_matches_des(workload):
    _, p = run(workload, 3, capi.MODE_PARTIAL)
    _, s = run(workload, 3, capi.MODE_SEQUENTIAL)
    assert p["mean_ms"] < s["mean_ms"]
    # measured vs DES recomputed from logged availability times: poll quantum + a few steps
    assert p["des_max_abs_err_ms"] < 40 and s["des_max_abs_err_ms"] < 40


def test_validation_detects_early_only_in_partial_mode():
    _, p = run("validation", 6, capi.MODE_PARTIAL)
    _, s = run("validation", 6, capi.MODE_SEQUENTIAL)
    assert p["aborted"] == s["aborted"] > 0
    assert p["detection_ms_mean"] < s["detection_ms_mean"] * 0.7


def test_codegen_only_last_line_after_decode(monkeypatch):
    """With decoding slower than the interpreter (the paper's regime: ~3.9 s requests,
    PAPER.md:210), everything but the final render line overlaps decoding."""
    monkeypatch.setattr(__import__(__name__), "STEP_S", 0.008)
    logs, _ = run("codegen", 2, capi.MODE_PARTIAL)
    for lg in logs:
        final = lg.round_final[0]
        ends = [e for e in lg.seg_end[0] if e is not None]
        # every tool segment but the tail of the script finished before/near the FINAL
        late = [e for e in ends if e > final + 0.05]
        assert len(late) <= 2


@pytest.mark.gpu
@pytest.mark.parametrize("runtime", ["native", "python"])
def test_engine_latency_matches_des_and_partial_wins(runtime):
    """S13 on the real engine (2-layer 7B slice, 32k vocab, CUDA graphs), through the native C++
    runtime (cvy_runtime_*) and the Python one: the runtime's measured
    request latencies agree with the oracle's O-3 DES recomputed from each request's logged
    round / segment timeline, in both modes, and partial execution beats
    sequential execution on every workload shape; validation aborts are detected earlier in
    partial mode."""
    import bench
    from inputs.configs import MISTRAL_7B, slice_of
    from paper_2406_00059_b200.engine import DeviceModel
    shape = slice_of(MISTRAL_7B, L=2, name="7b-L2")
    w = ["codegen", "search", "planning", "validation"]
    batches = {"codegen": 8, "search": 8, "planning": 8, "validation": 16}
    dm = DeviceModel(shape, "bf16", 16 * 200, seed=1002)
    res = bench.run_latency(w, batches, dm=dm, des=oracle_des, runtime=runtime)
    for name, row in res.items():
        assert row["partial_mean_ms"] < row["sequential_mean_ms"], (name, row["improvement"])
        for mode in ("partial", "sequential"):
            r = row["runs"][mode][0]
            if "des_max_abs_err_ms" in r:
                assert r["des_max_abs_err_ms"] < 40, (name, mode, r["des_max_abs_err_ms"])
            elif name != "validation":
                raise AssertionError(f"{name} {mode}: no DES cross-check")
    assert res["validation"]["detection_partial_ms"] < res["validation"]["detection_sequential_ms"]


@pytest.mark.gpu
def test_native_runtime_refill_and_abort():
    """NEXT-3 through the native runtime: 24 validation requests through 6 slots
    (max_inflight); every request completes, aborted ones are cancelled when the validator's
    offending member executes, and Partial finishes the
    queue sooner than Sequential."""
    import bench
    from inputs.configs import MISTRAL_7B, slice_of
    from paper_2406_00059_b200.engine import DeviceModel
    dm = DeviceModel(slice_of(MISTRAL_7B, L=2, name="7b-L2"), "bf16", 6 * 140, seed=1002)
    res = bench.run_latency(["validation"], {"validation": 24}, dm=dm, inflight=6, runtime="native")
    row = res["validation"]
    for mode in ("partial", "sequential"):
        r = row["runs"][mode][0]
        assert r["n"] == 24 and r["aborted"] > 0, r
    assert row["throughput_gain"] > 0, row["throughput_gain"]
    assert row["detection_partial_ms"] < row["detection_sequential_ms"]


@pytest.mark.gpu
def test_native_runtime_poisson_arrivals():
    """The Poisson-arrival protocol through the native runtime: requests are
    admitted in arrival order no earlier than their arrival, every latency is measured from the
    arrival, and partial execution still beats sequential with identical arrivals; the O-3 DES
    recomputed from each request's own round timeline (admission -> completion) matches."""
    import bench
    from inputs.configs import MISTRAL_7B, slice_of
    from inputs.tool_workloads import TOOLS, build
    from inputs.vocab import synthetic_vocab
    from paper_2406_00059_b200.engine import DeviceModel, Engine
    from paper_2406_00059_b200.runtime import NativeRuntime
    dm = DeviceModel(slice_of(MISTRAL_7B, L=2, name="7b-L2"), "bf16", 16 * 40, seed=1002)
    res = bench.run_latency(["codegen"], {"codegen": 12}, dm=dm, arrival_rate={"codegen": 20.0})
    row = res["codegen"]
    assert row["partial_mean_ms"] < row["sequential_mean_ms"]
    # admission order and times, directly
    eng = Engine(dm, synthetic_vocab(32000), max_slots=12, max_pages_per_slot=40)
    ids = {n: eng.register_tool(n, getattr(capi, k), d) for n, (k, d) in TOOLS.items()}
    _, specs = build("codegen", 12, ids)
    arrivals = [0.05 * (i + 1) for i in range(12)][::-1]  # reverse submission order on purpose
    logs = NativeRuntime(eng, capi.MODE_PARTIAL).run(specs, arrivals=arrivals)
    for lg, a in zip(logs, arrivals):
        assert lg.t_submit == pytest.approx(a) and lg.round_start[0] >= a - 1e-6 and lg.t_done > a
    order = sorted(range(12), key=lambda i: logs[i].round_start[0])
    assert order == sorted(range(12), key=lambda i: arrivals[i])
    for lg in logs:
        model, _ = oracle_des([{"g": lg.round_final[0] - lg.round_start[0],
                                "segs": [(a - lg.round_start[0], w.cost_s, w.instance, list(w.deps))
                                         for a, w in zip(lg.seg_avail[0], lg.seg_work[0])]}], True)
        assert abs(model - (lg.t_done - lg.round_start[0])) < 0.04
    eng.close()


@pytest.mark.gpu
def test_native_runtime_queues_when_engine_full():
    """More requests than engine slots and no max_inflight: the native runtime keeps the ones
    the engine refuses (CVY_E_FULL) queued in arrival order and admits them as finished requests
    release their slots; every request completes."""
    from inputs.configs import MISTRAL_7B, slice_of
    from inputs.tool_workloads import TOOLS, build
    from inputs.vocab import synthetic_vocab
    from paper_2406_00059_b200.engine import DeviceModel, Engine
    from paper_2406_00059_b200.runtime import NativeRuntime
    dm = DeviceModel(slice_of(MISTRAL_7B, L=2, name="7b-L2"), "bf16", 4 * 40, seed=1002)
    eng = Engine(dm, synthetic_vocab(32000), max_slots=4, max_pages_per_slot=40)
    ids = {n: eng.register_tool(n, getattr(capi, k), d) for n, (k, d) in TOOLS.items()}
    _, specs = build("codegen", 10, ids)
    logs = NativeRuntime(eng, capi.MODE_PARTIAL).run(specs)
    assert len(logs) == 10 and all(lg.t_done > 0 for lg in logs)
    starts = sorted(lg.round_start[0] for lg in logs)
    assert starts[4] > min(lg.t_done for lg in logs) - 1e-6  # the 5th waited for a slot
    eng.close()


# ------------------------------------------------------------------ NEXT-4: Fig. 6 sweep
def test_sweep_builder_tool_time_is_r_times_decode_time():
    """build_sweep assigns line costs so a round's tool time is r x its decode time at the
    given per-token time (tokens attributed by bytes): sum of costs == r * tok_s * tokens."""
    from inputs.tool_workloads import build_sweep
    for r in (0.1, 1.0, 7.0):
        _, specs, _ = build_sweep(3, 0, r, 0.002, n_lines=10)
        for sp in specs:
            rd = sp.rounds[0]
            total = sum(rd.plan(j, b"").cost_s for j in range(10))
            assert abs(total - r * 0.002 * len(rd.forced)) < 1e-12 + 1e-9 * total


@pytest.mark.gpu
def test_fig6_sweep_on_engine_below_theory():
    """NEXT-4 on a 2-layer 7B slice: measured improvement L_seq/L_par - 1 stays below the
    paper's best case min(r, 1/r) and reaches a good part of it."""
    import bench
    from inputs.configs import MISTRAL_7B, slice_of
    out = bench.run_fig6(4, ratios=(0.5, 1.0, 3.0), n_lines=8, shape=slice_of(MISTRAL_7B, L=2, name="7b-L2"))
    for row in out["rows"]:
        assert row["measured"] <= row["theory"] + 0.05, row
        assert row["measured"] >= 0.4 * row["theory"], row


def test_refill_admits_waiting_requests_and_partial_aborts_free_slots_sooner():
    """NEXT-3 abort-and-refill on the fake engine: 8 validation requests through 2 slots; every
    request completes, at most 2 are in flight at any time, and Partial mode (aborts detected
    at the offending member) finishes the queue sooner than Sequential (detected at FINAL)."""
    from inputs.vocab import synthetic_vocab
    vocab = synthetic_vocab(32000)
    ids = {name: i for i, name in enumerate(TOOLS)}
    kinds = {i: (getattr(oracle, TOOLS[n][0]), TOOLS[n][1]) for n, i in ids.items()}
    spans = {}
    for mode in (capi.MODE_PARTIAL, capi.MODE_SEQUENTIAL):
        eng = FakeEngine(vocab, kinds)
        _, specs = build("validation", 8, ids, seed=21)
        rt = Runtime(eng, mode)
        t0 = time.perf_counter()
        logs = rt.run(specs, timeout_s=120, max_inflight=2)
        assert len(logs) == 8 and all(lg.done for lg in logs)
        events = sorted([(lg.t_submit, 1) for lg in logs] + [(lg.t_done, -1) for lg in logs])
        live = peak = 0
        for _, d in events:
            live += d
            peak = max(peak, live)
        assert peak <= 2
        spans[mode] = max(lg.t_done for lg in logs) - t0
    assert spans[capi.MODE_PARTIAL] < spans[capi.MODE_SEQUENTIAL]


def test_bench_peak_parsing_units_and_preference():
    """bench.parse_peaks reads a driver-written MEASURED_PEAKS.json of unknown key naming:
    sustained over burst, TB/s -> GB/s, GFLOP/s -> TF/s, and the fallback when nothing matches."""
    import bench
    p, src = bench.parse_peaks({"hbm_copy_gbs": {"burst": 7300.0, "sustained": 6900.0},
                                "bf16_dense_tflops": {"burst": 1650.0, "sustained": 1380.0}})
    assert src == "measured" and p == {"hbm_gbs": 6900.0, "bf16_tflops": 1380.0}
    p, src = bench.parse_peaks({"hbm_tbs": 6.54, "cublas_bf16_gflops": 1648400.0})
    assert src == "measured" and p["hbm_gbs"] == 6540.0 and abs(p["bf16_tflops"] - 1648.4) < 1e-9
    p, src = bench.parse_peaks({"unrelated": 1, "flag": True})
    assert src == "fallback" and p == bench.PEAKS_FALLBACK


def test_bench_algorithmic_bytes_match_survey_counts():
    """The roofline numerator (bench.step_alg_bytes) against SURVEY.md §8(d)'s independent count
    for the 7B shape: 7,110,393,856 streamed parameters (bf16: 14.22 GB; the embedding is a
    gather) + sum over slots of (ctx + 1) x 128 KiB of KV read + 128 KiB of KV written per slot."""
    import bench
    from inputs.configs import MISTRAL_7B
    assert MISTRAL_7B.n_params_streamed == 7_110_393_856
    kv_tok = 2 * MISTRAL_7B.L * MISTRAL_7B.Hkv * MISTRAL_7B.hd * 2
    assert kv_tok == 128 * 1024
    ctx = [128 + 7 * i for i in range(64)]
    want = 2 * 7_110_393_856 + sum(c + 1 for c in ctx) * kv_tok + len(ctx) * kv_tok
    assert bench.step_alg_bytes(MISTRAL_7B, ctx) == want


def test_time_oracle_runs_exactly_the_requested_steps():
    """bench.time_oracle with no time budget runs exactly max_steps steps (the reference arm
    reports steps and ms_per_step from it), and with a budget stops once the budget is spent."""
    import bench
    from inputs.configs import TINY
    reqs = [{"prefix": 5 + i, "seed": 100 + i} for i in range(4)]
    toks, t, _, n, steps = bench.time_oracle(TINY, reqs, 0.0, 7, n_req=2, max_steps=3)
    assert (steps, n, toks) == (3, 2, 6) and t > 0
    toks, t, _, n, steps = bench.time_oracle(TINY, reqs, 1e-9, 7, n_req=1, max_steps=50)
    assert steps == 1 and toks == 1


def _check_timeline(lg):
    from paper_2406_00059_b200 import timeline
    ev = timeline.events(lg)
    assert [e[0] for e in ev] == sorted(e[0] for e in ev)
    assert {e[1] for e in ev} <= set(timeline.KINDS)
    at = {}
    for (t, k, r, j, p, d) in ev:
        at.setdefault((r, p), {})[k] = t
    for (r, p), ks in at.items():
        if "PieceExecuted" in ks:
            assert ks["TokenDecoded"] <= ks["PieceDispatched"] <= ks["ToolStart"] <= ks["PieceExecuted"]
    # pieces of one tool instance are dispatched in order
    disp = [(r, p, t) for (t, k, r, j, p, d) in ev if k == "PieceDispatched"]
    for r in {x[0] for x in disp}:
        ts = [t for (rr, p, t) in sorted(x for x in disp if x[0] == r)]
        assert ts == sorted(ts)
    tsv = timeline.to_tsv(ev)
    rows = [ln.split("\t") for ln in tsv.splitlines()]
    assert all(len(x) == 6 for x in rows) and len(rows) == len(ev)
    assert "decode" in timeline.gantt(ev)
    return ev


def test_timeline_codegen_pieces_overlap_decode():
    """Fig. 3: in Partial mode the interpreter executes lines while the
    decode continues; the exported timeline (SPEC.md:387 columns) shows every piece but the
    last few dispatched before RoundEnd, and ResponseReady after the last PieceExecuted."""
    logs, _ = run("codegen", 2, capi.MODE_PARTIAL)
    for lg in logs:
        ev = _check_timeline(lg)
        t_end = next(t for (t, k, *_ ) in ev if k == "RoundEnd")
        disp = [t for (t, k, *_ ) in ev if k == "PieceDispatched"]
        assert sum(t < t_end for t in disp) >= len(disp) - 2
        assert ev[-1][1] == "ResponseReady"
    logs, _ = run("codegen", 2, capi.MODE_SEQUENTIAL)
    for lg in logs:
        ev = _check_timeline(lg)
        t_end = next(t for (t, k, *_ ) in ev if k == "RoundEnd")
        assert all(t >= t_end for (t, k, *_ ) in ev if k == "PieceDispatched")


def test_timeline_validation_abort_precedes_round_end():
    """SPEC.md:352 / Fig. 7: in Partial mode the AbortSignal of an offending
    request comes before its (cancelled) RoundEnd, far before a full decode would end."""
    logs, _ = run("validation", 4, capi.MODE_PARTIAL)
    aborted = [lg for lg in logs if lg.t_abort is not None]
    assert aborted
    for lg in aborted:
        ev = _check_timeline(lg)
        t_ab = next(t for (t, k, *_ ) in ev if k == "AbortSignal")
        t_end = next(t for (t, k, *_ ) in ev if k == "RoundEnd")
        assert t_ab <= t_end
        assert t_ab < 0.5 * len(lg.spec.rounds[0].forced) * STEP_S * 1e6
