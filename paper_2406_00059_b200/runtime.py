"""Host runtime above the C ABI: segment poller, tool executors, Partial vs Sequential dispatch.

PAPER.md:146 (Fig. 4): the scheduler (1) takes requests, (2) runs decoding iterations, and
(8) polls tool status; tools (6)/(7) run beside decoding and their outputs become the next
round's input (step (g)).  Here:
  * a driver thread calls cvy_step back to back (continuous batching);
  * a poller thread drains the pinned segment ring (cvy_poll_segments) while decoding
    continues -- Partial mode dispatches every segment the moment it is polled (tool partial
    execution), Sequential mode holds a round's segments until its FINAL record
    ("tool invocation always happens after decoding to the EOS", reading R15);
  * tool executors are event-driven stubs with seeded costs: segments of one tool instance
    run serially, instances run in parallel, DAG dependencies are honoured (planning) --
    the same rules as the O-3 schedule in oracle/latency.py, so measured latencies can be
    checked against the DES recomputed from the logged availability times;
  * when a round's FINAL is in and all its tool work is done, the observation is injected
    (cvy_inject_observation) and the next round decodes; the request completes after its
    last round (plus its tools, if any).  A validator may abort (cvy_cancel_request).
"""
from __future__ import annotations

import heapq
import threading
import time
from dataclasses import dataclass, field

from . import capi


@dataclass
class SegmentWork:
    cost_s: float
    instance: int = 0
    deps: list = field(default_factory=list)   # indices of earlier segments of the round
    abort: bool = False                        # validator verdict: abort the request


@dataclass
class Round:
    forced: list                 # teacher-forced generated tokens of the round
    tool_id: int                 # -1: no tool
    plan: object = None          # callable(seg_index, seg_bytes, flags) -> SegmentWork | None
    observation: list = field(default_factory=list)  # tokens injected before the next round


@dataclass
class RequestSpec:
    prompt: list
    rounds: list
    synth_prefix: int = 0
    synth_seed: int = 0


@dataclass
class RequestLog:
    spec: RequestSpec
    rid: int = 0
    t_submit: float = 0.0
    t_done: float = 0.0
    t_abort: float | None = None
    round: int = 0
    round_start: list = field(default_factory=list)
    round_final: list = field(default_factory=list)
    seg_avail: list = field(default_factory=list)    # per round: [t]
    seg_work: list = field(default_factory=list)     # per round: [SegmentWork]
    seg_end: list = field(default_factory=list)      # per round: [t]
    seg_disp: list = field(default_factory=list)     # per round: [t dispatched to the tool]
    seg_begin: list = field(default_factory=list)    # per round: [t the tool started it]
    seg_token: list = field(default_factory=list)    # per round: [token index of its last byte]
    held: list = field(default_factory=list)         # Sequential: segments waiting for FINAL
    pending_tools: int = 0
    final_seen: bool = False
    done: bool = False
    released: bool = False


class Runtime:
    """Drives one engine through a batch of multi-round tool-using requests."""

    def __init__(self, eng, mode: int):
        self.eng = eng
        self.mode = mode
        self.lock = threading.Lock()
        self.cv = threading.Condition(self.lock)
        self.events = []           # heap of (t, seq, callback)
        self.seq = 0
        self.inst_free = {}        # (req, round, instance) -> t
        self.by_rid = {}
        self.active = 0
        self.max_inflight = None
        self.waiting = []
        self.logs = []
        self.stop = False
        self.steps = 0
        self.poller_cpu_s = 0.0    # CPU time of the poller thread (polling + dispatch)
        self.dispatch_cpu_s = 0.0  # of which: handling polled records (parse plans, dispatch tools)

    # ---------------------------------------------------------------- tool clock
    def _schedule(self, t, cb):
        heapq.heappush(self.events, (t, self.seq, cb))
        self.seq += 1
        self.cv.notify_all()

    def _dispatch(self, log: RequestLog, rnd: int, j: int, t_avail: float):
        """Start segment j of round rnd at max(avail, instance free, deps done)."""
        work = log.seg_work[rnd][j]
        dep_ends = [log.seg_end[rnd][d] for d in work.deps]
        if any(e is None for e in dep_ends):
            return False  # retried when a dependency finishes
        key = (log.rid, rnd, work.instance)
        start = max(t_avail, self.inst_free.get(key, 0.0), max(dep_ends, default=0.0))
        end = start + work.cost_s
        self.inst_free[key] = end
        log.seg_end[rnd][j] = end
        log.seg_disp[rnd][j] = t_avail
        log.seg_begin[rnd][j] = start
        log.pending_tools += 1
        self._schedule(end, lambda lg=log, r=rnd, jj=j: self._tool_done(lg, r, jj))
        return True

    def _tool_done(self, log: RequestLog, rnd: int, j: int):
        log.pending_tools -= 1
        now = time.perf_counter()
        if log.seg_work[rnd][j].abort and log.t_abort is None and not log.done:
            log.t_abort = now
            self.eng.cancel_request(log.rid)
        # dependants waiting for this segment
        for k, w in enumerate(log.seg_work[rnd]):
            if log.seg_end[rnd][k] is None and j in w.deps and log.seg_avail[rnd][k] is not None:
                if self.mode == capi.MODE_PARTIAL or log.final_seen:
                    self._dispatch(log, rnd, k, max(now, log.seg_avail[rnd][k]))
        self._maybe_advance(log, now)

    def _maybe_advance(self, log: RequestLog, now: float):
        if log.done or not log.final_seen or log.pending_tools > 0:
            return
        if any(e is None for e in log.seg_end[log.round]):
            return
        rnd = log.round
        spec = log.spec
        if log.t_abort is not None or rnd + 1 >= len(spec.rounds):
            self._finish(log, now)
            return
        nxt = spec.rounds[rnd + 1]
        log.round = rnd + 1
        log.final_seen = False
        self._open_round(log, now)
        self.eng.inject_observation(log.rid, spec.rounds[rnd].observation, len(nxt.forced), forced=nxt.forced)

    def _finish(self, log: RequestLog, t_done: float):
        log.done = True
        log.t_done = t_done
        self.active -= 1
        if self.max_inflight is not None:
            # abort-and-refill (NEXT-3): the slot and its KV pages go back to the engine now
            # (applied at the next step boundary) and a waiting request takes them, so an
            # early abort ("saving the resources ... for decoding subsequent
            # tokens") turns into throughput
            self.eng.release_request(log.rid)
            log.released = True
            if self.waiting:
                self._submit(self.waiting.pop(0))
        self.cv.notify_all()

    def _submit(self, spec: RequestSpec):
        lg = RequestLog(spec)
        r0 = spec.rounds[0]
        lg.t_submit = time.perf_counter()
        lg.rid = self.eng.submit_request(spec.prompt, len(r0.forced), tool_id=r0.tool_id, mode=self.mode,
                                         forced=r0.forced, synth_prefix_len=spec.synth_prefix,
                                         synth_seed=spec.synth_seed,
                                         reserve_tokens=sum(len(rr.forced) + len(rr.observation) + 2
                                                            for rr in spec.rounds[1:]) + len(r0.observation))
        self._open_round(lg, lg.t_submit)
        self.by_rid[lg.rid] = lg
        self.logs.append(lg)
        return lg

    def _open_round(self, log: RequestLog, now: float):
        log.round_start.append(now)
        log.round_final.append(None)
        log.seg_avail.append([])
        log.seg_work.append([])
        log.seg_end.append([])
        log.seg_disp.append([])
        log.seg_begin.append([])
        log.seg_token.append([])
        log.held = []

    # ---------------------------------------------------------------- poller
    def _on_record(self, r, now):
        log = self.by_rid.get(r.req_id)
        if log is None or log.done:
            return
        rnd = log.round
        spec_round = log.spec.rounds[rnd]
        is_final = bool(r.flags & capi.SEG_FINAL)
        if not is_final or r.byte_len > 0:
            if spec_round.tool_id >= 0 and spec_round.plan is not None:
                j = len(log.seg_work[rnd])
                # plan(index, bytes, flags): region markers (CVY_SEG_OPEN / CLOSE) are passed
                # so a plan can ignore them (FENCE) or start the tool on them (CALL: "when
                # Conveyor identifies the function name of the tool")
                work = spec_round.plan(j, r.data, r.flags)
                if work is not None:
                    log.seg_work[rnd].append(work)
                    log.seg_avail[rnd].append(now)
                    log.seg_end[rnd].append(None)
                    log.seg_disp[rnd].append(None)
                    log.seg_begin[rnd].append(None)
                    log.seg_token[rnd].append(r.token_index)
                    if self.mode == capi.MODE_PARTIAL:
                        self._dispatch(log, rnd, j, now)
                    else:
                        log.held.append(j)
        if is_final:
            log.round_final[rnd] = now
            log.final_seen = True
            if r.flags & capi.SEG_CANCELLED:
                self._finish(log, now if log.t_abort is None else log.t_abort)
                return
            if self.mode == capi.MODE_SEQUENTIAL:
                for j in log.held:
                    self._dispatch(log, rnd, j, now)
                log.held = []
            # segments whose deps were not ready at dispatch time
            for k in range(len(log.seg_work[rnd])):
                if log.seg_end[rnd][k] is None:
                    self._dispatch(log, rnd, k, now)
            self._maybe_advance(log, now)

    def _poller(self):
        c0 = time.thread_time()
        try:
            self._poll_loop()
        finally:
            self.poller_cpu_s = time.thread_time() - c0

    def _poll_loop(self):
        while True:
            with self.lock:
                if self.stop:
                    return
            recs = self.eng.poll_segments(with_bytes=True)
            now = time.perf_counter()
            with self.lock:
                if recs:
                    d0 = time.thread_time()
                    for r in recs:
                        self._on_record(r, now)
                    self.dispatch_cpu_s += time.thread_time() - d0
                # fire due tool completions
                while self.events and self.events[0][0] <= now:
                    _, _, cb = heapq.heappop(self.events)
                    cb()
            if not recs:
                time.sleep(0.00005)

    # ---------------------------------------------------------------- driver
    def run(self, specs: list[RequestSpec], timeout_s: float = 600.0, max_inflight: int | None = None):
        """Run every request to completion.  max_inflight: admit at most this many at a time
        and refill a slot the moment its request completes or aborts (NEXT-3); None submits
        everything at t=0 and releases at the end."""
        self.logs = []
        self.max_inflight = max_inflight
        t0 = time.perf_counter()
        with self.lock:
            first = specs if max_inflight is None else specs[:max_inflight]
            self.waiting = [] if max_inflight is None else list(specs[max_inflight:])
            for spec in first:
                self._submit(spec)
            self.active = len(specs)
        logs = self.logs
        th = threading.Thread(target=self._poller, daemon=True)
        th.start()
        try:
            while True:
                with self.lock:
                    if self.active <= 0:
                        break
                    busy = any(not lg.done and (lg.round_final[lg.round] is None) for lg in logs)
                if busy:
                    self.eng.step()
                    self.steps += 1
                else:
                    # every live request waits on tools: idle until an injection is queued
                    with self.lock:
                        self.cv.wait(timeout=0.0005)
                if time.perf_counter() - t0 > timeout_s:
                    raise TimeoutError("latency run did not finish")
        finally:
            self.eng.sync()
            with self.lock:
                self.stop = True
            th.join()
        for lg in logs:
            if not lg.released:
                self.eng.release_request(lg.rid)
        return logs


class NativeRuntime:
    """The same scheduler in C++ behind the ABI (cvy_runtime_*, runtime.cpp): a native poller
    thread, n_workers executor threads (the plan's cost occupies a worker: a tool stub), the
    calling thread driving cvy_step.  Python is entered only through the plan callback, once
    per polled piece.  run() returns RequestLog objects like Runtime.run, so summarize /
    round_timelines / timeline.py work unchanged."""

    def __init__(self, eng, mode: int, n_workers: int | None = None, poll_sleep_us: int = 20):
        self.eng = eng
        self.mode = mode
        self.n_workers = n_workers
        self.poll_sleep_us = poll_sleep_us
        self.steps = 0
        self.poller_cpu_s = 0.0
        self.dispatch_cpu_s = 0.0
        self.stats = None

    def run(self, specs: list[RequestSpec], timeout_s: float = 600.0, max_inflight: int | None = None,
            arrivals: list[float] | None = None):
        """arrivals: per-request arrival times (seconds after the start; None: all at t = 0).
        With arrivals, a request's latency runs from its arrival (RequestLog.t_submit = the
        arrival), so admission waits count."""
        import ctypes
        from .capi import check
        L = capi.lib()
        errors = []

        def plan_cb(user, request, rnd, piece, data, n, flags, out):
            try:
                rd = specs[request].rounds[rnd]
                work = rd.plan(piece, ctypes.string_at(data, n) if n else b"", flags) if rd.plan else None
                o = out.contents
                if work is None:
                    o.skip = 1
                    return
                o.cost_ms = float(work.cost_s) * 1e3
                o.instance = int(work.instance)
                deps = list(work.deps)[:8]
                o.n_deps = len(deps)
                for k, d in enumerate(deps):
                    o.deps[k] = int(d)
                o.abort = 1 if work.abort else 0
            except Exception as exc:  # never unwind into C
                errors.append(exc)
                out.contents.skip = 1

        cb = capi.PLAN_FN(plan_cb)
        # executors: enough that tool capacity never binds (the paper's tools -- interpreter, web
        # search, validator -- run every call at once; the O-3 schedule assumes parallel instances)
        workers = self.n_workers or min(2048, max(64, 4 * len(specs)))
        cfg = capi.RuntimeConfig(self.mode, workers, max_inflight or 0, cb, None, self.poll_sleep_us)
        h = ctypes.c_void_p()
        check(L.cvy_runtime_create(self.eng.h, ctypes.byref(cfg), ctypes.byref(h)))
        keep = []
        reqs = (capi.RtRequest * len(specs))()
        for i, sp in enumerate(specs):
            arr = lambda xs: (ctypes.c_int32 * max(1, len(xs)))(*xs)
            rds = (capi.RoundDesc * len(sp.rounds))()
            for k, rd in enumerate(sp.rounds):
                f, o = arr(rd.forced), arr(rd.observation)
                keep += [f, o]
                rds[k] = capi.RoundDesc(f, len(rd.forced), rd.tool_id, o, len(rd.observation))
            pr = arr(sp.prompt)
            keep += [rds, pr]
            reqs[i] = capi.RtRequest(pr, len(sp.prompt), sp.synth_prefix, sp.synth_seed, rds, len(sp.rounds),
                                     float(arrivals[i]) if arrivals is not None else 0.0)
        try:
            check(L.cvy_runtime_run(h, reqs, len(specs), float(timeout_s)))
            if errors:
                raise errors[0]
            logs = []
            for i, sp in enumerate(specs):
                rl = capi.RtRequestLog()
                check(L.cvy_runtime_request_log(h, i, ctypes.byref(rl)))
                lg = RequestLog(sp, rid=rl.req_id, t_submit=rl.t_arrival if arrivals is not None else rl.t_submit,
                                t_done=rl.t_done,
                                t_abort=rl.t_abort if rl.aborted else None, done=True, released=True)
                for r in range(rl.n_rounds_run):
                    ro = capi.RtRoundLog()
                    check(L.cvy_runtime_round_log(h, i, r, ctypes.byref(ro)))
                    lg.round_start.append(ro.t_start)
                    lg.round_final.append(ro.t_final if ro.t_final >= 0 else None)
                    cols = ([], [], [], [], [], [])
                    for j in range(ro.n_pieces):
                        pl = capi.RtPieceLog()
                        check(L.cvy_runtime_piece_log(h, i, r, j, ctypes.byref(pl)))
                        cols[0].append(pl.t_avail)
                        cols[1].append(SegmentWork(pl.cost_ms / 1e3, pl.instance, [pl.deps[k] for k in range(pl.n_deps)]))
                        cols[2].append(pl.t_end if pl.t_end >= 0 else None)
                        cols[3].append(pl.t_dispatch if pl.t_dispatch >= 0 else None)
                        cols[4].append(pl.t_begin if pl.t_begin >= 0 else None)
                        cols[5].append(pl.token_index)
                    lg.seg_avail.append(cols[0])
                    lg.seg_work.append(cols[1])
                    lg.seg_end.append(cols[2])
                    lg.seg_disp.append(cols[3])
                    lg.seg_begin.append(cols[4])
                    lg.seg_token.append(cols[5])
                lg.round = max(0, rl.n_rounds_run - 1)
                lg.final_seen = True
                logs.append(lg)
            st = capi.RtStats()
            check(L.cvy_runtime_stats(h, ctypes.byref(st)))
            self.stats = {f: getattr(st, f) for f, _ in capi.RtStats._fields_}
            self.steps = st.steps
            self.poller_cpu_s = st.poller_cpu_s
            self.dispatch_cpu_s = st.dispatch_cpu_s
            return logs
        finally:
            L.cvy_runtime_destroy(h)
            del keep


def round_timelines(log: RequestLog):
    """Per round of one request: decode time g (round start -> FINAL polled) and the logged
    segments as (availability offset, cost, instance, deps) -- the inputs of the paper's
    latency model, for an external schedule cross-check."""
    rounds = []
    for i in range(len(log.round_start)):
        g = (log.round_final[i] - log.round_start[i]) if log.round_final[i] else 0.0
        segs = [(a - log.round_start[i], w.cost_s, w.instance, list(w.deps))
                for a, w in zip(log.seg_avail[i], log.seg_work[i])]
        rounds.append({"g": g, "segs": segs})
    return rounds


def summarize(logs, mode: int, des=None):
    """Per-request latency (submit -> completion) stats.  `des`, if given, is a schedule model
    callable(rounds, partial) -> (latency_s, detail) recomputing each request from its logged
    timeline (the tests pass the oracle's O-3 DES); the max deviation is reported."""
    import numpy as np
    lat = np.array([(lg.t_done - lg.t_submit) * 1e3 for lg in logs])
    out = {"n": len(logs), "mean_ms": float(lat.mean()), "std_ms": float(lat.std()),
           "p50_ms": float(np.percentile(lat, 50)), "p95_ms": float(np.percentile(lat, 95))}
    det = [((lg.t_abort - lg.t_submit) * 1e3) for lg in logs if lg.t_abort is not None]
    if det:
        out["detection_ms_mean"] = float(np.mean(det))
        out["aborted"] = len(det)
    if des is not None:
        errs = []
        for lg in logs:
            if lg.t_abort is not None:
                continue
            model, _ = des(round_timelines(lg), mode == capi.MODE_PARTIAL)
            errs.append(abs(model - (lg.t_done - lg.t_submit)))
        if errs:
            out["des_max_abs_err_ms"] = float(max(errs) * 1e3)
    return out
