#!/usr/bin/env python
"""bench.py -- the Conveyor decode hot path on B200 (BASELINE.json metric).

One "step" = one continuous-batching decode step of the whole hot path (SURVEY.md 8(a)
S1-S13: embed, 32 x [QKV+RoPE+KV append, paged GQA attention, O+residual, gate/up+SwiGLU,
down+residual], LM head + greedy sample + fused trigger scan + compaction + publish).

Default workload = BASELINE.json configs[4], "validation" (the largest single-GPU config;
BASELINE.json's metric names no config): Mistral-7B-shape random-init bf16, a TOTAL batch of
512 in-flight requests split over the ranks by the router (request k -> rank k mod G), 2K-token
contexts in the paged KV cache (synthetic prefix 1792 tokens, growing to ~2048), teacher-forced
streams of structured JSON calls through the incremental format-validator tool (JSON_MEMBER).
`--workload codegen` runs configs[1] (B = 64, prefixes 128 + U(0, 400), Python scripts, '\\n').

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload ...]

`--gpus N` without torchrun spawns its own N ranks (127.0.0.1).  Rank 0 prints ONE JSON line:
`value` = generated tokens/s of the whole job over the K timed steps (inputs resident in HBM;
device time from CUDA events on the engine stream, max over ranks).  Inputs exceed L2
(14.2 GB of weights + the KV cache streamed every step), so no L2 flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import random
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/s/GPU + HBM roofline %; request latency, partial vs sequential tool exec"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
WORKLOADS = {
    "validation": {"config": "BASELINE.json configs[4] (validation)", "batch": 512},
    "codegen": {"config": "BASELINE.json configs[1] (codegen)", "batch": 64},
}
SPAN_STEPS = 3


def _flatten(d, pre=""):
    out = {}
    if isinstance(d, dict):
        for k, v in d.items():
            out.update(_flatten(v, f"{pre}.{k}".lower() if pre else str(k).lower()))
    elif isinstance(d, (int, float)) and not isinstance(d, bool):
        out[pre] = float(d)
    return out


def parse_peaks(d):
    """HBM GB/s and dense bf16 TF/s from a driver-written MEASURED_PEAKS.json of unknown key
    naming: the sustained figure is preferred (the dominant kernel is timed inside a long step),
    TB/s and GFLOP/s are normalised; a figure that cannot be found keeps the fallback."""
    flat = _flatten(d)

    def pick(must, unit_fix):
        cands = [(k, v) for k, v in flat.items() if any(m in k for m in must) and v > 0]
        if not cands:
            return None
        cands.sort(key=lambda kv: (0 if "sustain" in kv[0] else 1 if "burst" not in kv[0] else 2, kv[0]))
        return unit_fix(cands[0][1])

    hbm = pick(("hbm", "copy", "dram"), lambda v: v * 1000.0 if v < 100 else v)
    tc = pick(("bf16",), lambda v: v / 1000.0 if v > 20000 else (v * 1000.0 if v < 20 else v))
    out = dict(PEAKS_FALLBACK)
    if hbm:
        out["hbm_gbs"] = hbm
    if tc:
        out["bf16_tflops"] = tc
    return out, ("measured" if hbm else "fallback")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            with open(p) as f:
                return parse_peaks(json.load(f))
        except (OSError, ValueError):
            pass
    return dict(PEAKS_FALLBACK), "fallback"


# ------------------------------------------------------------------ workload
def workload_requests(name: str, indices, gen_tokens: int, prefix: int | None = None):
    """Requests of a config's total batch (global indices `indices`: this rank's share under
    the router).  Per request: synthetic KV prefix length, synth seed (= global index), and the
    teacher-forced generated stream (DESIGN.md §5 "Input recipe")."""
    from inputs.vocab import Tokenizer, synthetic_vocab
    from inputs.workloads import codegen_script, validation_call
    vocab = synthetic_vocab(32000)
    tok = Tokenizer(vocab)
    reqs = []
    for k in indices:
        rng = random.Random(2000 + 100003 * (k + 1) + (4 if name == "validation" else 1))
        if name == "validation":
            p = prefix if prefix is not None else 1792
            ids = []
            while len(ids) < gen_tokens:   # consecutive validator calls (one JSON object each)
                ids += tok.encode(validation_call(rng, rng.random() < 0.5) + "\n")
        else:
            p = prefix if prefix is not None else 128 + rng.randrange(0, 400)
            ids = []
            while len(ids) < gen_tokens:
                ids += tok.encode(codegen_script(rng, 40))
        reqs.append({"k": k, "prefix": p, "seed": k, "forced": ids[:gen_tokens]})
    return vocab, reqs


def default_prefix(name: str, gen: int):
    """validation: contexts reach 2048 (prefix 1792 + the ~256-token output);
    a longer timed run starts from a shorter prefix so the context still ends near 2048."""
    if name == "validation":
        return 1792 if gen <= 256 else max(512, 2048 - gen)
    return None


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm, mx, pw, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
                pw.append(float(parts[3]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        pw.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": pw[len(pw) // 2] if pw else None}


# ------------------------------------------------------------------ multi-rank reduction
def reduce_over_ranks(local_ms: float, local_tokens: int, stats: list, device=None):
    """Max-over-ranks device time, whole-job tokens, and the per-rank completion stats
    all-gathered (NCCL over NVLink/NVSwitch on GPUs, gloo in the CPU tests).  Returns
    (max_ms, total_tokens, gathered_stats [world][len(stats)])."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size() if dist.is_initialized() else 1
    t = torch.tensor([local_ms], dtype=torch.float64, device=device)
    n = torch.tensor([local_tokens], dtype=torch.float64, device=device)
    st = torch.tensor(stats, dtype=torch.float64, device=device)
    if world == 1:
        return float(t.item()), int(n.item()), [list(map(float, st.tolist()))]
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    gathered = [torch.zeros_like(st) for _ in range(world)]
    dist.all_gather(gathered, st)
    return float(t.item()), int(n.item()), [list(map(float, g.tolist())) for g in gathered]


def gather_objects(obj):
    """All ranks' `obj` (rank order); [obj] without a process group."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


# ------------------------------------------------------------------ algorithmic bytes / flops
def gemm_launch_bytes(shape, kind: int, B: int) -> int:
    """Algorithmic HBM bytes of one projection GEMM launch: the bf16 weight
    matrix streamed once + the bf16 activation rows read + the rows written (QKV: q fp32 and
    the new token's K, V appended to the paged cache)."""
    d, H, Hkv, hd, dff, V = shape.d, shape.H, shape.Hkv, shape.hd, shape.dff, shape.V
    if kind == 1:
        N, K, out = (H + 2 * Hkv) * hd, d, B * (H * hd * 4 + 2 * Hkv * hd * 2)
    elif kind == 4:
        N, K, out = d, H * hd, B * d * (4 + 4 + 2)  # residual read+write fp32, next-norm input
    elif kind == 5:
        N, K, out = 2 * dff, d, B * dff * 2
    elif kind == 6:
        N, K, out = d, dff, B * d * (4 + 4 + 2)
    else:
        N, K, out = V, d, B * 8
    return N * K * 2 + B * K * 2 + out


def gemm_launch_flops(shape, kind: int, B: int) -> float:
    """Tensor-core flops of one projection launch as executed: 2 N K per batch column, twice
    for the (hi, lo) activation pair."""
    d, H, Hkv, hd, dff, V = shape.d, shape.H, shape.Hkv, shape.hd, shape.dff, shape.V
    NK = {1: (H + 2 * Hkv) * hd * d, 4: d * H * hd, 5: 2 * dff * d, 6: d * dff, 7: V * d}[kind]
    return 2.0 * NK * B * 2


def attention_launch_bytes(shape, ctx_lens) -> int:
    """One layer's paged attention: the K and V of keys [0, ctx] of every slot (bf16)."""
    return sum(c + 1 for c in ctx_lens) * (shape.kv_bytes_per_token // shape.L)


def step_alg_bytes(shape, ctx_lens):
    """Per step: weights streamed once + KV read (ctx incl. the new token) + KV written."""
    kv_tok = shape.kv_bytes_per_token
    return 2 * shape.n_params_streamed + sum(c + 1 for c in ctx_lens) * kv_tok + len(ctx_lens) * kv_tok


# ------------------------------------------------------------------ CPU oracle timing
def time_oracle(shape, reqs, budget_s: float, seed: int, n_req: int | None = None, max_steps: int | None = None):
    """Run the CPU oracle (as it stands, weights regenerated from the counter hash every step,
    no caching) on a bounded sample of the same workload: decode steps for n_req of the
    requests (their synthetic prefixes, first input token).  Stops after max_steps steps, or
    once budget_s seconds of oracle time are spent (whichever comes first; at least one of the
    two must bound the loop).  Returns (tokens, seconds, threads, n_req, steps)."""
    if not ((max_steps is not None and max_steps >= 1) or budget_s > 0):
        raise ValueError("time_oracle needs max_steps >= 1 or a positive time budget")
    import oracle
    w = oracle.Weights(shape, seed, bf16=True, cache=False)

    def one_step(sample):
        ors = []
        for r in sample:
            o = oracle.Request(w, r["prefix"] + 4)
            o.synth_prefix(r["prefix"], r["seed"])
            ors.append(o)
        t0 = time.perf_counter()
        oracle.step(ors, [1] * len(sample))
        return time.perf_counter() - t0

    if n_req is None:
        n_req = 4
    n_req = max(1, min(n_req, len(reqs)))
    t_total, toks, steps, i = 0.0, 0, 0, 0
    while True:
        sample = [reqs[(i + j) % len(reqs)] for j in range(n_req)]
        t_total += one_step(sample)
        toks += n_req
        steps += 1
        i += n_req
        if (budget_s > 0 and t_total >= budget_s) or (max_steps is not None and steps >= max_steps):
            break
    return toks, t_total, oracle.num_threads(), n_req, steps


def oracle_sample_text(name, n, steps, secs):
    return (f"{steps} oracle decode step(s), each over {n} of the {WORKLOADS[name]['batch']} {name} requests "
            f"(full 32 layers at their synthetic-prefix contexts, weights regenerated per step as the oracle "
            f"stands), {secs:.1f} s of CPU work")


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from inputs.configs import MISTRAL_7B
    B = WORKLOADS[args.workload]["batch"]
    gen = args.warmup + args.steps + SPAN_STEPS + 8
    prefix = args.prefix if args.prefix is not None else default_prefix(args.workload, gen)
    _, reqs = workload_requests(args.workload, range(B), 8, prefix)
    n = args.cpu_sample
    if args.warmup > 0:
        time_oracle(MISTRAL_7B, reqs, 0.0, 1001, n_req=n, max_steps=args.warmup)
    total_tok, total_t, cores, _, steps = time_oracle(MISTRAL_7B, reqs, 0.0, 1001, n_req=n, max_steps=args.steps)
    value = total_tok / total_t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(args.workload, B, None, None, prefix),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": oracle_sample_text(args.workload, n, steps, total_t), "host": host_info()},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(name, B_total, ctx_mean, world, prefix=None):
    return {"workload": f"{WORKLOADS[name]['config']}: Mistral-7B-shape random-init bf16, total batch {B_total} "
                        f"split over the ranks (request k -> rank k mod G), "
                        + ("2K-token contexts (synthetic KV prefix, paged), teacher-forced JSON calls through the "
                           "format-validator tool (JSON_MEMBER), partial execution"
                           if name == "validation" else
                           "synthetic KV prefixes 128+U(0,400), teacher-forced Python scripts through the "
                           "code-interpreter tool ('\\n'), partial execution"),
            "batch_total": B_total, "batch_per_gpu": None if not world else B_total // world,
            "kv_prefix": (f"{prefix} synthetic tokens" if prefix else "128+U(0,400) synthetic tokens"),
            "ctx_mean": ctx_mean,
            "l2": "no flush: inputs > L2 (14.2 GB of weights + the KV cache streamed per step)"}


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hooks for the multi-rank path on a single-GPU box: CVY_DIST_BACKEND=gloo (reductions
    # on host tensors) and CVY_SAME_GPU=1 (every rank on device 0); the driver's runs use NCCL,
    # one GPU per rank
    same_gpu = os.environ.get("CVY_SAME_GPU") == "1"
    # NCCL refuses two ranks on one device: the single-GPU test hook reduces over gloo
    backend = os.environ.get("CVY_DIST_BACKEND", "gloo" if same_gpu else "nccl")
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    red_dev = torch.device("cuda", local) if backend == "nccl" else None
    if world > 1:
        dist.init_process_group(backend)

    from inputs.configs import MISTRAL_7B
    from paper_2406_00059_b200 import build, capi
    from paper_2406_00059_b200.engine import DeviceModel, Engine
    from paper_2406_00059_b200.router import STATS_FIELDS, Router
    build.build()
    shape = MISTRAL_7B
    name = args.workload
    B_total = args.batch or WORKLOADS[name]["batch"]
    router = Router(rank, world, every=16, device=red_dev)
    mine = router.mine(B_total)
    B = len(mine)
    W, K = args.warmup, args.steps
    gen = W + K + SPAN_STEPS + 8
    prefix = args.prefix if args.prefix is not None else default_prefix(name, gen)
    vocab, reqs = workload_requests(name, mine, gen, prefix)
    max_ctx = max(r["prefix"] for r in reqs) + gen + 64
    pages_per_slot = (max_ctx + 15) // 16 + 1
    lat_pages = 0 if args.no_latency else latency_pages(router)
    n_pages = max(B * pages_per_slot, lat_pages) + 64
    dm = DeviceModel(shape, "bf16", n_pages, seed=1001, device=local)
    eng = Engine(dm, vocab, max_slots=B, max_pages_per_slot=pages_per_slot, device=local,
                 flags=(capi.ENGINE_SCAN_OFF if args.scan_off else 0) | capi.ENGINE_CHUNKED_PREFILL)
    if name == "validation":
        tool = eng.register_tool("validator", capi.PARSER_JSON_MEMBER)
    else:
        tool = eng.register_tool("interp", capi.PARSER_LITERAL, [b"\n"])
    rids = [eng.submit_request([1], gen, tool_id=tool, forced=r["forced"], synth_prefix_len=r["prefix"],
                               synth_seed=r["seed"]) for r in reqs]

    # a poller thread drains the pinned segment ring while decoding continues
    stop = threading.Event()
    nseg = [0]

    def poller():
        while not stop.is_set():
            recs = eng.poll_segments(with_bytes=True)
            nseg[0] += len(recs)
            if not recs:
                time.sleep(0.0002)

    th = threading.Thread(target=poller, daemon=True)
    th.start()
    stream = torch.cuda.ExternalStream(eng.stream_ptr(), device=local)
    for _ in range(W):
        eng.step()
    eng.sync()
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    wall0 = time.perf_counter()
    evs[0].record(stream)
    for i in range(K):
        info = eng.step()
        router.after_step(info)
        evs[i + 1].record(stream)
    evs[K].synchronize()
    wall = time.perf_counter() - wall0
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(K)]
    dev_ms = evs[0].elapsed_time(evs[K])
    med_local = float(np.median(step_ms))
    perf = eng.perf()
    max_ms, total_tokens, rank_stats = reduce_over_ranks(dev_ms, B * K, [float(rank), dev_ms, float(B * K), med_local],
                                                         device=red_dev)
    value = total_tokens / (max_ms / 1000.0)
    ms_med = max(s[3] for s in rank_stats)
    ctx_mean = float(np.mean([r["prefix"] + W + (K - 1) / 2.0 for r in reqs]))  # step t attends prefix + t + 1 keys
    stats_table = router.flush()

    # in-graph kernel spans of the same graph (+ %globaltimer atomics): kernel shares
    eng.set_kernel_spans(True)
    span_runs = []
    for _ in range(SPAN_STEPS):
        eng.step()
        span_runs.append(eng.kernel_spans())
    eng.set_kernel_spans(False)
    eng.sync()
    span_ctx = [r["prefix"] + W + K + SPAN_STEPS - 1 for r in reqs]   # the last recorded step
    peaks, peaks_src = load_peaks()
    roofline, kernels = span_roofline(shape, span_runs[-1], span_ctx, B, peaks, peaks_src, ms_med)
    ctx_now = [r["prefix"] + W + (K - 1) / 2.0 for r in reqs]
    step_roof = step_roofline(shape, ctx_now, B, max_ms / K, ms_med, peaks)

    # end-to-end through the C ABI with host buffers
    stop.set()
    th.join()
    eng.sync()
    eng.poll_segments()
    for rid in rids:
        if eng.request_state(rid) == 0:
            eng.cancel_request(rid)
    for _ in range(3):
        eng.step()
    eng.sync()
    eng.poll_segments()
    for rid in rids:
        eng.release_request(rid)
    e2e = run_e2e(eng, reqs, tool, B)
    eng.close()
    e2e_ms, e2e_tok, _ = reduce_over_ranks(e2e.pop("_dt_s") * 1e3, e2e.pop("_ntok"), [0.0], device=red_dev)
    e2e["per_rank_value"] = e2e["value"]
    e2e["value"] = e2e_tok / (e2e_ms / 1000.0)

    latency = None
    if not args.no_latency:
        latency = run_latency_ab(dm, router, reps=args.latency_reps, device=local)
    del dm

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            toks, secs, cores, n, steps = time_oracle(shape, reqs, args.cpu_budget, 1001, n_req=args.cpu_sample)
            cpu = {"value": toks / secs, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                   "sample": oracle_sample_text(name, n, steps, secs), "host": host_info(),
                   "extras": oracle_extras()}
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
                "ms_per_step": max_ms / K, "ms_per_step_median": ms_med, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": workload_config(name, B_total, ctx_mean, world, prefix),
                "tokens_per_s_per_gpu": value / world, "roofline": roofline, "kernels": kernels,
                "step_roofline": step_roof, "cpu_baseline": cpu, "e2e": e2e, "latency": latency,
                "gpu_launches": int(perf.launches_per_step) * K, "launches_per_step": int(perf.launches_per_step),
                "clocks": clk, "wall_s_timed": wall, "segments_polled": nseg[0], "rank_stats": rank_stats,
                "router": {"policy": "request k -> rank k mod G", "stats_every_steps": 16, "gathers": router.gathers,
                           "fields": list(STATS_FIELDS), "last_gather": stats_table}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def span_roofline(shape, spans, ctx, B, peaks, peaks_src, ms_step):
    """Per-kernel device time from the in-graph spans of one step (cvy_kernel_spans) and the
    roofline of the dominant kernel: achieved = algorithmic bytes per launch x launches / the
    summed spans; frac = achieved / the measured HBM copy peak."""
    from paper_2406_00059_b200 import capi
    hbm = float(peaks["hbm_gbs"])
    tc = float(peaks.get("bf16_tflops", PEAKS_FALLBACK["bf16_tflops"]))
    per = {}
    for kind, layer, chain, t0, t1 in spans:
        k = per.setdefault(kind, {"ms": 0.0, "launches": 0})
        k["ms"] += (t1 - t0) / 1e6
        k["launches"] += 1
    kernels = {}
    for kind, v in sorted(per.items()):
        name = capi.KERNEL_KINDS[kind]
        if kind == 2:
            by = attention_launch_bytes(shape, ctx) * v["launches"]
            fl = 4.0 * shape.H * shape.hd * sum(c + 1 for c in ctx) * v["launches"]
        elif kind in (1, 4, 5, 6, 7):
            by = gemm_launch_bytes(shape, kind, B) * v["launches"]
            fl = gemm_launch_flops(shape, kind, B) * v["launches"]
        else:
            by = B * shape.d * (2 + 4 + 2 * 2) * v["launches"]
            fl = 0.0
        s = v["ms"] / 1e3
        kernels[name] = {"ms_per_step": round(v["ms"], 4), "launches": v["launches"], "alg_bytes": by,
                         "GBps": by / s / 1e9 if s > 0 else None, "hbm_frac": by / s / 1e9 / hbm if s > 0 else None,
                         "TFLOPs": fl / s / 1e12 if s > 0 and fl else None,
                         "tc_frac": fl / s / 1e12 / tc if s > 0 and fl and kind != 2 else None}
    gemm_ms = sum(per[k]["ms"] for k in (1, 4, 5, 6, 7) if k in per)
    attn_ms = per.get(2, {"ms": 0.0})["ms"]
    if attn_ms >= gemm_ms:
        v = per[2]
        by = attention_launch_bytes(shape, ctx)
        name = "attention_tc_kernel (paged GQA decode attention: TMA KV pages + mma.sync, online softmax)"
        launches, ms = v["launches"], v["ms"]
    else:
        launches = sum(per[k]["launches"] for k in (1, 4, 5, 6, 7) if k in per)
        by = sum(gemm_launch_bytes(shape, k, B) * per[k]["launches"] for k in (1, 4, 5, 6, 7) if k in per) / launches
        name = "gemm_tc_kernel (tcgen05 projections QKV / O / gate-up / down / LM head, all launches of the step)"
        ms = gemm_ms
    achieved = by * launches / (ms / 1e3) / 1e9
    traffic = load_traffic("attention_traffic.json" if attn_ms >= gemm_ms else "gemm_traffic.json")
    roofline = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "peak_source": f"{peaks_src} HBM copy bandwidth (MEASURED_PEAKS.json)",
                "alg_bytes_per_launch": by, "launches_per_step": launches, "ms_per_step": ms,
                "share_of_step": ms / ms_step,
                "timing": "sum of in-graph spans (first CTA past its grid-dependency wait -> last CTA exit, "
                          "%globaltimer) of this kernel's launches in one step of the production graph",
                "traffic": (traffic or {}).get("per_launch_bytes"),
                "traffic_detail": None if traffic is None else {k: traffic[k] for k in traffic if k != "per_launch_bytes"}}
    return roofline, kernels


def step_roofline(shape, ctx_now, B, ms_mean, ms_med, peaks):
    """Whole-step HBM roofline and the phase roofline of SURVEY.md 8(d)."""
    hbm = float(peaks["hbm_gbs"])
    tc = float(peaks.get("bf16_tflops", PEAKS_FALLBACK["bf16_tflops"])) * 1e12
    step_bytes = step_alg_bytes(shape, ctx_now)
    kv_tok = shape.kv_bytes_per_token
    proj_bytes = 2.0 * shape.n_params_streamed
    proj_flops = 2.0 * shape.n_params_streamed * B * 2
    att_bytes = sum(c + 1 for c in ctx_now) * kv_tok + B * kv_tok
    att_flops = 4.0 * shape.L * shape.H * shape.hd * sum(c + 1 for c in ctx_now)
    t_proj = max(proj_bytes / (hbm * 1e9), proj_flops / tc)
    t_att = max(att_bytes / (hbm * 1e9), att_flops / tc)
    return {"alg_bytes_per_step": step_bytes, "achieved_GBps": step_bytes / (ms_mean / 1e3) / 1e9,
            "frac": step_bytes / (ms_mean / 1e3) / 1e9 / hbm,
            "frac_median_step": step_bytes / (ms_med / 1e3) / 1e9 / hbm,
            "frac_vs_8TBps_nominal": step_bytes / (ms_mean / 1e3) / 8e12,
            "phase_roofline": {"t_min_ms": (t_proj + t_att) * 1e3, "frac": (t_proj + t_att) / (ms_mean / 1e3),
                               "projections": "tensor" if proj_flops / tc > proj_bytes / (hbm * 1e9) else "hbm",
                               "tc_peak_tflops": tc / 1e12,
                               "note": "projection flops count the (hi, lo) activation pair twice (DESIGN.md §4)"}}


def _oracle_tiny_c0():
    """SURVEY.md 8(d) "O-1 tiny: the full C0": 4 requests, the 7-byte prompt then 64 forced
    bytes each, through the tiny model (fp32) one step at a time; prints one JSON line."""
    import oracle
    from inputs.configs import TINY
    from inputs.workloads import codegen_script
    prompt = list(b"# task\n")
    rng = random.Random(7)
    seqs = [prompt + list(codegen_script(rng, 6).encode())[:64] for _ in range(4)]
    t0 = time.perf_counter()
    w = oracle.Weights(TINY, 1000, bf16=False)
    reqs = [oracle.Request(w, 128) for _ in seqs]
    for t in range(len(seqs[0])):
        oracle.step(reqs, [sq[t] for sq in seqs])
    dt = time.perf_counter() - t0
    print(json.dumps({"tokens": 4 * len(seqs[0]), "seconds": dt, "tokens_per_s": 4 * len(seqs[0]) / dt,
                      "threads": oracle.num_threads()}))


def oracle_extras():
    """The rest of SURVEY.md 8(d)'s CPU-oracle protocol, bounded to a few seconds: O-1 tiny
    (C0) at 1 OpenMP thread and at all cores (subprocesses: OMP_NUM_THREADS is read at load),
    and O-2 segmentation throughput over the C1 (LITERAL) and C4 (JSON_MEMBER) forced streams."""
    import oracle
    from oracle.scan import round_records
    out = {"omp_num_threads_env": os.environ.get("OMP_NUM_THREADS")}
    for label, env in (("tiny_c0_1thread", {"OMP_NUM_THREADS": "1"}), ("tiny_c0_all_cores", {})):
        e = dict(os.environ)
        e.pop("OMP_NUM_THREADS", None)
        e.update(env)
        try:
            r = subprocess.run([sys.executable, os.path.abspath(__file__), "--oracle-tiny"], env=e,
                               capture_output=True, text=True, timeout=300)
            out[label] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as exc:  # reported, never fatal to the bench line
            out[label] = {"error": str(exc)[:200]}
    from inputs.vocab import synthetic_vocab
    vocab = synthetic_vocab(32000)
    for wl, kind, delims in (("codegen", oracle.PARSER_LITERAL, [b"\n"]),
                             ("validation", oracle.PARSER_JSON_MEMBER, [])):
        _, reqs = workload_requests(wl, range(64), 256, 0)
        nbytes = sum(sum(len(vocab[t]) for t in r["forced"]) for r in reqs)
        ntok = sum(len(r["forced"]) for r in reqs)
        t0 = time.perf_counter()
        nrec = sum(len(round_records(r["forced"], vocab, kind, delims, 4096)[0]) for r in reqs)
        dt = time.perf_counter() - t0
        out[f"scan_{wl}"] = {"requests": 64, "tokens": ntok, "bytes": nbytes, "records": nrec, "seconds": dt,
                             "MB_per_s": nbytes / dt / 1e6, "tokens_per_s": ntok / dt}
    return out


def host_info():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def run_e2e(eng, reqs, tool, B):
    """The same metric end to end through the C ABI: a fresh batch whose prompts (16 tokens) and
    forced streams come from host memory (submit copies them; the chunked prefill pass runs the
    prompts), decoded until every FINAL is polled and every request's tokens are read back."""
    G = 64
    prompt_len = 16
    rng = random.Random(77)
    prompts = [[1] + [rng.randrange(259, 32000) for _ in range(prompt_len - 1)] for _ in range(B)]
    t0 = time.perf_counter()
    ids = [eng.submit_request(prompts[b], G, tool_id=tool, forced=reqs[b]["forced"][:G],
                              synth_prefix_len=reqs[b]["prefix"], synth_seed=reqs[b]["seed"]) for b in range(B)]
    finals, nrec, nbytes, steps = set(), 0, 0, 0
    while len(finals) < B:
        eng.step()
        steps += 1
        for r in eng.poll_segments():
            nrec += 1
            nbytes += r.byte_len
            if r.flags & 1:
                finals.add(r.req_id)
        if steps > 10 * (G + prompt_len):
            break
    toks = [eng.round_tokens(i) for i in ids]
    dt = time.perf_counter() - t0
    ntok = sum(len(t) for t in toks)
    for i in ids:
        eng.release_request(i)
    h2d = B * (prompt_len + G) * 4 + B * 64 * 4  # prompt + forced tokens + page-table entries
    d2h = nrec * 40 + nbytes + ntok * 4
    return {"value": ntok / dt, "_dt_s": dt, "_ntok": ntok, "unit": "tokens/s", "h2d_bytes_per_step": h2d / steps,
            "d2h_bytes_per_step": d2h / steps, "steps": steps, "requests": B, "generated_per_request": G,
            "prompt_tokens": prompt_len, "includes": "submit (host prompts + forced streams, synthetic KV prefix), "
                                                     "chunked prefill (CVY_ENGINE_CHUNKED_PREFILL), decode, segment "
                                                     "polling, token read-back"}


def load_traffic(name):
    p = os.path.join(ROOT, "profiles", name)
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


# ------------------------------------------------------------------ self-launch of N ranks
def spawn_ranks(n: int) -> int:
    """`--gpus N` without torchrun: start N copies of this command as ranks 0..N-1 (one GPU
    each; 127.0.0.1 rendezvous) and return the worst exit code.  Rank 0's stdout is ours."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    return max(p.wait() for p in procs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)   # median of >= 200 steps
    ap.add_argument("--warmup", type=int, default=20)   # after 20 warm-up steps
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="validation", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0, help="total batch over all ranks (default: the config's)")
    ap.add_argument("--prefix", type=int, default=None, help="synthetic KV prefix tokens per request")
    ap.add_argument("--scan-off", action="store_true", help="trigger scan disabled (overhead A/B)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--cpu-sample", type=int, default=4, help="requests per oracle step (both arms)")
    ap.add_argument("--no-latency", action="store_true", help="skip the partial-vs-sequential latency A/B")
    ap.add_argument("--latency-reps", type=int, default=3)
    ap.add_argument("--latency-only", default="", help="comma list of workloads: run only the latency A/B")
    ap.add_argument("--latency-batch", type=int, default=0, help="override every workload's batch")
    ap.add_argument("--latency-inflight", type=int, default=0,
                    help="NEXT-3 abort-and-refill: run each workload's requests through this many slots")
    ap.add_argument("--chunked-prefill", action="store_true",
                    help="NEXT-1: prompts / observations as batched prefill passes (CVY_ENGINE_CHUNKED_PREFILL)")
    ap.add_argument("--fig6", action="store_true", help="NEXT-4: Fig. 6 tool/decode ratio sweep on the engine")
    ap.add_argument("--oracle-tiny", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--fig6-batch", type=int, default=16)
    args = ap.parse_args()
    if args.oracle_tiny:
        _oracle_tiny_c0()
        return
    if args.steps < 1:
        ap.error("--steps must be >= 1")
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.gpus > 1:
        # let the driver see the communicator size; NCCL's log goes to stderr, not the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.fig6:
        print(json.dumps({"fig6": run_fig6(args.fig6_batch, verbose=True)}), flush=True)
        return
    if args.latency_only:
        ws = args.latency_only.split(",")
        base = {"codegen": 64, "codegen_fence": 64, "search": 128, "search_call": 128, "planning": 256, "validation": 512}
        bs = {w: (args.latency_batch or base[w]) for w in ws}
        from paper_2406_00059_b200 import capi
        fl = capi.ENGINE_CHUNKED_PREFILL if args.chunked_prefill else 0
        res = run_latency(ws, bs, verbose=True, inflight=args.latency_inflight or None, flags=fl,
                          reps=args.latency_reps)
        for row in res.values():  # per-request latency lists stay out of the summary line
            for runs in row["runs"].values():
                for r in runs:
                    r.pop("lat_ms", None)
        print(json.dumps({"latency": res, "chunked_prefill": bool(args.chunked_prefill), "runtime": "native",
                          "protocol": "all requests at t=0, modes interleaved per repetition"}), flush=True)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


# ------------------------------------------------------------------ latency: partial vs sequential
LAT_PREFIX = {"codegen": 128, "codegen_fence": 128, "search": 256, "search_call": 256, "planning": 512, "validation": 1792}
LAT_TOKENS = {"codegen": 440, "codegen_fence": 460, "search": 560, "search_call": 560, "planning": 400, "validation": 320}
LAT_BATCH = {"codegen": 64, "codegen_fence": 64, "search": 128, "search_call": 128, "planning": 256, "validation": 512}
AB_WORKLOADS = ("codegen", "validation")


def latency_pages(router, workloads=AB_WORKLOADS):
    """KV pages the in-line latency A/B needs on this rank (its share of each workload)."""
    return max(router.share(LAT_BATCH[w]) * ((LAT_PREFIX[w] + LAT_TOKENS[w] + 31) // 16 + 1) for w in workloads)


def run_latency(workloads, batches, device=0, verbose=False, inflight=None, flags=0, dm=None, indices=None,
                reps=1, des=None, runtime="native", arrival_rate=None):
    """Request completion latency with tool partial execution vs sequential tool execution on
    the workload shapes (BASELINE.json configs[1..4]); identical seeded streams and tool costs
    in both modes (the baseline is the same code with partial execution
    disabled).  `indices(w)`: the global request indices this rank serves (router).  Each
    (workload, mode) runs `reps` times, modes interleaved.  `des`: a schedule model passed to
    runtime.summarize (the GPU tests pass the oracle's O-3 DES; bench.py never does).
    `runtime`: "native" (cvy_runtime_*, C++ poller / executors / driver) or "python".
    `arrival_rate` {workload: requests/s of the whole job}: Poisson arrivals (seeded, identical
    in both modes; native runtime) instead of all requests at t = 0; latency then runs from
    each request's arrival.
    Returns {workload: {...}}."""
    from inputs.configs import MISTRAL_7B
    from inputs.tool_workloads import TOOLS, build
    from inputs.vocab import synthetic_vocab
    from paper_2406_00059_b200 import capi
    from paper_2406_00059_b200.engine import DeviceModel, Engine
    from paper_2406_00059_b200.runtime import NativeRuntime, Runtime, summarize
    import numpy as np
    idx = {w: (list(range(batches[w])) if indices is None else indices(w)) for w in workloads}
    pages_per = {w: (LAT_PREFIX[w] + LAT_TOKENS[w] + 31) // 16 + 1 for w in workloads}
    slots = {w: (inflight or len(idx[w])) for w in workloads}
    need = max(slots[w] * pages_per[w] for w in workloads) + 64
    own = dm is None
    if own:
        dm = DeviceModel(MISTRAL_7B, "bf16", need, seed=1002, device=device)
    Bmax = max(slots[w] for w in workloads)
    eng = Engine(dm, synthetic_vocab(32000), max_slots=Bmax, max_pages_per_slot=max(pages_per.values()) + 2,
                 device=device, flags=flags)
    tool_ids = {name: eng.register_tool(name, getattr(capi, kind), delims) for name, (kind, delims) in TOOLS.items()}
    out = {}
    for w in workloads:
        res = {"partial": [], "sequential": []}
        for rep in range(reps):
            for mode, label in ((capi.MODE_PARTIAL, "partial"), (capi.MODE_SEQUENTIAL, "sequential")):
                _, specs = build(w, batches[w], tool_ids, indices=idx[w])
                rt = NativeRuntime(eng, mode) if runtime == "native" else Runtime(eng, mode)
                arr = None
                if arrival_rate and w in arrival_rate:
                    # this rank's requests arrive as its share of a Poisson process of the job's rate
                    share = len(idx[w]) / max(1, batches[w])
                    g = random.Random(4242 + rep)
                    t, arr = 0.0, []
                    for _ in specs:
                        t += g.expovariate(arrival_rate[w] * share)
                        arr.append(t)
                t0 = time.perf_counter()
                c0 = time.process_time()
                logs = rt.run(specs, max_inflight=inflight, arrivals=arr) if arr is not None else \
                    rt.run(specs, max_inflight=inflight)
                s = summarize(logs, mode, des=des)
                s["steps"] = rt.steps
                s["wall_s"] = time.perf_counter() - t0
                s["host_cpu_s"] = time.process_time() - c0
                s["poller_cpu_s"] = rt.poller_cpu_s
                s["dispatch_cpu_s"] = rt.dispatch_cpu_s
                s["lat_ms"] = [(lg.t_done - lg.t_submit) * 1e3 for lg in logs]
                if inflight:
                    span = max(lg.t_done for lg in logs) - min(lg.t_submit for lg in logs)
                    s.update(makespan_s=span, requests_per_s=len(logs) / span, slots=inflight)
                res[label].append(s)
                if verbose:
                    print(w, label, rep, {k: v for k, v in s.items() if k != "lat_ms"}, flush=True)
        p = float(np.mean([r["mean_ms"] for r in res["partial"]]))
        q = float(np.mean([r["mean_ms"] for r in res["sequential"]]))
        row = {"batch": batches[w], "reps": reps, "partial_mean_ms": p, "sequential_mean_ms": q,
               "improvement": q / p - 1.0,   # the paper's metric
               "reduction": 1.0 - p / q,     # the north star's wording
               "improvement_per_rep": [b["mean_ms"] / a["mean_ms"] - 1.0 for a, b in zip(res["partial"], res["sequential"])],
               "runs": res}
        if "detection_ms_mean" in res["partial"][0]:
            dp = float(np.mean([r["detection_ms_mean"] for r in res["partial"]]))
            ds = float(np.mean([r["detection_ms_mean"] for r in res["sequential"]]))
            row.update(detection_partial_ms=dp, detection_sequential_ms=ds, detection_speedup=ds / dp - 1.0)
        if inflight:
            row["throughput_gain"] = (np.mean([r["requests_per_s"] for r in res["partial"]]) /
                                      np.mean([r["requests_per_s"] for r in res["sequential"]]) - 1.0)
        out[w] = row
    eng.close()
    if own:
        del dm
    return out


LAT_POISSON_RATE = {"codegen": 50.0, "validation": 250.0}  # requests/s of the whole job


def run_latency_ab(dm, router, reps=3, device=0):
    """The latency half of the metric in the bench line: codegen (configs[1]) and validation
    (configs[4]), partial vs sequential, `reps` repetitions each, this rank serving its router
    share; per-request latencies are gathered over the ranks.  Host CPU: process CPU seconds
    per mode, the poller thread's CPU and the time spent dispatching records (the paper's CPU
    overhead figure is 0.6% extra cycles)."""
    import numpy as np
    res = run_latency(list(AB_WORKLOADS), LAT_BATCH, device=device, dm=dm, reps=reps,
                      indices=lambda w: router.mine(LAT_BATCH[w]))
    res_p = run_latency(list(AB_WORKLOADS), LAT_BATCH, device=device, dm=dm, reps=reps,
                        indices=lambda w: router.mine(LAT_BATCH[w]), arrival_rate=LAT_POISSON_RATE)
    out = {}
    for w, row in list(res.items()) + [(w + "_poisson", r) for w, r in res_p.items()]:
        per_rank = gather_objects({m: [r["lat_ms"] for r in row["runs"][m]] for m in ("partial", "sequential")})
        lat = {m: [sum((pr[m][i] for pr in per_rank), []) for i in range(reps)] for m in ("partial", "sequential")}
        means = {m: [float(np.mean(x)) for x in lat[m]] for m in lat}
        allv = {m: np.array(sum(lat[m], [])) for m in lat}
        p, q = float(np.mean(means["partial"])), float(np.mean(means["sequential"]))
        cpu = {m: float(np.mean([r["host_cpu_s"] for r in row["runs"][m]])) for m in ("partial", "sequential")}
        ent = {"requests": len(lat["partial"][0]), "reps": reps,
               "partial": {"mean_ms": p, "std_ms": float(allv["partial"].std()),
                           "p50_ms": float(np.percentile(allv["partial"], 50)),
                           "p95_ms": float(np.percentile(allv["partial"], 95))},
               "sequential": {"mean_ms": q, "std_ms": float(allv["sequential"].std()),
                              "p50_ms": float(np.percentile(allv["sequential"], 50)),
                              "p95_ms": float(np.percentile(allv["sequential"], 95))},
               "improvement": q / p - 1.0, "reduction": 1.0 - p / q,
               "improvement_per_rep": [b / a - 1.0 for a, b in zip(means["partial"], means["sequential"])],
               "host_cpu_s": cpu, "host_cpu_extra_partial": cpu["partial"] / cpu["sequential"] - 1.0,
               "dispatch_cpu_s_partial": float(np.mean([r["dispatch_cpu_s"] for r in row["runs"]["partial"]])),
               "poller_cpu_s_partial": float(np.mean([r["poller_cpu_s"] for r in row["runs"]["partial"]])),
               "wall_s_partial": float(np.mean([r["wall_s"] for r in row["runs"]["partial"]]))}
        if "detection_partial_ms" in row:
            ent.update(detection_partial_ms=row["detection_partial_ms"],
                       detection_sequential_ms=row["detection_sequential_ms"],
                       detection_speedup=row["detection_speedup"])
        out[w] = ent
    out["protocol"] = ("native C++ runtime (cvy_runtime_*); identical seeded streams and tool costs in both modes; "
                       "modes interleaved per repetition; all requests submitted at t=0, and *_poisson: Poisson "
                       f"arrivals at {LAT_POISSON_RATE} requests/s of the whole job (seeded per repetition, identical "
                       "in both modes), latency from arrival; latency = submit/arrival -> completion on the host clock")
    return out


# ------------------------------------------------------------------ NEXT-4: Fig. 6 sweep
def run_fig6(B, ratios=(0.1, 0.25, 0.5, 1.0, 2.0, 4.0, 10.0), n_lines=12, device=0, verbose=False, shape=None):
    """PAPER.md:240-242 (Fig. 6): latency improvement of tool partial execution as a function of
    the tool/decode time ratio r = t_i/g_i, measured on the engine.  Each request decodes one
    round of n_lines lines on the 7B-shape engine; line j's tool cost is r x its share of the
    round's decode time (per-token decode time calibrated by a cost-free Sequential run).
    Reported per r: the measured ratio r_meas = mean t / mean g, the paper's best case
    (1 + r)/max(1, r) - 1 = min(r, 1/r) at r_meas (g_{n+1} = 0: the request ends with its
    tools), and the measured improvement L_seq/L_par - 1."""
    import numpy as np
    from inputs.configs import MISTRAL_7B
    from inputs.tool_workloads import build_sweep
    from inputs.vocab import synthetic_vocab
    from paper_2406_00059_b200 import capi
    from paper_2406_00059_b200.engine import DeviceModel, Engine
    from paper_2406_00059_b200.runtime import Runtime
    dm = DeviceModel(shape or MISTRAL_7B, "bf16", B * 24 + 64, seed=1003, device=device)
    eng = Engine(dm, synthetic_vocab(32000), max_slots=B, max_pages_per_slot=20, device=device)
    tool = eng.register_tool("interp", capi.PARSER_LITERAL, [b"\n"])

    def run(r, mode, tok_s):
        _, specs, ntok = build_sweep(B, tool, r, tok_s, n_lines)
        rt = Runtime(eng, mode)
        logs = rt.run(specs)
        lat = float(np.mean([lg.t_done - lg.t_submit for lg in logs]))
        g = float(np.mean([lg.round_final[0] - lg.round_start[0] for lg in logs]))
        t = float(np.mean([sum(w.cost_s for w in lg.seg_work[0]) for lg in logs]))
        return lat, g, t, ntok

    _, g0, _, ntok = run(0.0, capi.MODE_SEQUENTIAL, 0.0)   # warm-up + calibration
    _, g0, _, ntok = run(0.0, capi.MODE_SEQUENTIAL, 0.0)
    tok_s = g0 / ntok
    rows = []
    for r in ratios:
        lp, gp, tp, _ = run(r, capi.MODE_PARTIAL, tok_s)
        ls, gs, ts, _ = run(r, capi.MODE_SEQUENTIAL, tok_s)
        r_meas = 0.5 * (tp / gp + ts / gs)
        row = {"r": r, "r_meas": r_meas, "theory": (1.0 + r_meas) / max(1.0, r_meas) - 1.0,
               "measured": ls / lp - 1.0, "L_par_ms": lp * 1e3, "L_seq_ms": ls * 1e3, "g_ms": gp * 1e3,
               "t_ms": tp * 1e3}
        rows.append(row)
        if verbose:
            print(json.dumps(row), flush=True)
    eng.close()
    return {"batch": B, "lines_per_round": n_lines, "tokens_per_round": ntok, "decode_ms_per_token": tok_s * 1e3,
            "rows": rows}


if __name__ == "__main__":
    main()
