#!/usr/bin/env python
"""bench.py -- decode throughput of the Conveyor hot path on B200 (BASELINE.json metric).

One "step" = one continuous-batching decode step of the whole hot path (SURVEY.md 8(a)
S1-S13: embed, 32 x [QKV+RoPE+KV append, paged GQA attention, O+residual, gate/up+SwiGLU,
down+residual], LM head + greedy sample + fused trigger scan + compaction + publish) for
the N=1 workload of BASELINE.json configs[1] ("codegen"): Mistral-7B-shape random-init
bf16, 64 in-flight requests per GPU, synthetic KV prefix 128 + U(0,400) tokens, teacher-
forced ~400-token Python-script streams through the code-interpreter tool ('\\n').

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  `value` = generated tokens/s of the whole job with inputs
resident in HBM (device time, CUDA events on the engine stream, max over ranks).  Inputs
are larger than L2 (14.2 GB of weights streamed every step), so no L2 flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import random
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/s/GPU + HBM roofline %; request latency, partial vs sequential tool exec"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


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
def codegen_workload(B: int, gen_tokens: int, seed: int = 2001, prefix_min: int = 128, prefix_spread: int = 400):
    """Per request: synthetic prefix length, synth seed, forced token stream (teacher forcing
    of codegen scripts)."""
    from inputs.vocab import Tokenizer, synthetic_vocab
    from inputs.workloads import codegen_script
    vocab = synthetic_vocab(32000)
    tok = Tokenizer(vocab)
    rng = random.Random(seed)
    reqs = []
    for b in range(B):
        prefix = prefix_min + (rng.randrange(0, prefix_spread) if prefix_spread > 0 else 0)
        ids = []
        while len(ids) < gen_tokens:
            ids += tok.encode(codegen_script(rng, 40))
        reqs.append({"prefix": prefix, "seed": b, "forced": ids[:gen_tokens]})
    return vocab, reqs


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
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


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


# ------------------------------------------------------------------ algorithmic bytes
def gemm_launch_bytes(shape, kind: int, B: int) -> int:
    """Algorithmic HBM bytes of one projection GEMM launch: the bf16
    weight matrix streamed once + the bf16 activation rows read + the rows written."""
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


def pk_launch_bytes(shape, ctx_lens):
    """Algorithmic HBM bytes of one persistent all-layers launch: every layer's QKV, O,
    gate/up and down weights streamed once (bf16) + the KV cache read (ctx incl. the new
    token) + the new token's K, V appended.  Activations are excluded (L2-resident)."""
    d, H, Hkv, hd, dff, L = shape.d, shape.H, shape.Hkv, shape.hd, shape.dff, shape.L
    layer_params = (H + 2 * Hkv) * hd * d + d * H * hd + 2 * dff * d + d * dff
    kv_tok = shape.kv_bytes_per_token
    return 2 * L * layer_params + sum(c + 1 for c in ctx_lens) * kv_tok + len(ctx_lens) * kv_tok


def step_alg_bytes(shape, ctx_lens):
    """Per step: weights streamed once + KV read (ctx incl. the new token) + KV written."""
    kv_tok = shape.kv_bytes_per_token
    return 2 * shape.n_params_streamed + sum(c + 1 for c in ctx_lens) * kv_tok + len(ctx_lens) * kv_tok


# ------------------------------------------------------------------ CPU oracle timing
def time_oracle(shape, reqs, budget_s: float, seed: int, n_req: int | None = None, max_steps: int | None = None):
    """Run the CPU oracle (as it stands, weights regenerated from the counter hash every step,
    no caching) on a bounded sample of the same workload: decode steps for a sample of the
    requests (their synthetic prefixes, first input token).  The sample size is calibrated
    so the total lands near budget_s.  Returns (tokens, seconds, threads, n_req, steps)."""
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
        t1 = one_step(reqs[:1])
        n_req = max(1, min(len(reqs), int(budget_s / 3 / max(t1, 1e-3))))
    t_total, toks, steps, i = 0.0, 0, 0, 0
    while True:
        sample = [reqs[(i + j) % len(reqs)] for j in range(n_req)]
        t_total += one_step(sample)
        toks += n_req
        steps += 1
        i += n_req
        # budget_s <= 0: no time budget (exactly max_steps steps, as the reference arm needs)
        if (budget_s > 0 and t_total >= budget_s) or (max_steps and steps >= max_steps):
            break
    return toks, t_total, oracle.num_threads(), n_req, steps


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from inputs.configs import MISTRAL_7B
    B = 64
    _, reqs = codegen_workload(B, 8)
    # calibrate: size each step (a sample of the 64 requests) to ~1 s of CPU work
    _, t1, cores, _, _ = time_oracle(MISTRAL_7B, reqs, 0.0, 1001, n_req=1, max_steps=1)
    n = max(1, min(B, int(1.0 / max(t1, 1e-3))))
    _, _, _, _, _ = time_oracle(MISTRAL_7B, reqs, 0.0, 1001, n_req=n, max_steps=args.warmup)
    total_tok, total_t, cores, _, _ = time_oracle(MISTRAL_7B, reqs, 0.0, 1001, n_req=n, max_steps=args.steps)
    value = total_tok / total_t
    sample = f"{n} of the 64 codegen requests per step (1 decode step each, full 32 layers, their synthetic prefixes)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(B, None),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(B, ctx_mean, prefix_min=128, prefix_spread=400):
    return {"workload": "codegen (BASELINE.json configs[1]): Mistral-7B-shape random-init, "
                        "teacher-forced Python-script streams, code-interpreter tool '\\n' (partial mode)"
                        if (B, prefix_min, prefix_spread) == (64, 128, 400) else
                        f"decode step at batch {B}, synthetic KV prefixes {prefix_min}+U(0,{prefix_spread}) "
                        "(Mistral-7B shape, codegen streams; SURVEY.md 8(d) config points)",
            "batch_per_gpu": B, "kv_prefix": f"{prefix_min}+U(0,{prefix_spread}) synthetic tokens",
            "ctx_mean": ctx_mean,
            "l2": "no flush: inputs > L2 (14.2 GB weights + KV streamed per step)"}


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
    backend = os.environ.get("CVY_DIST_BACKEND", "nccl")
    if os.environ.get("CVY_SAME_GPU") == "1":
        local = 0
    red_dev = "cuda" if backend == "nccl" else None
    if world > 1:
        dist.init_process_group(backend)
    torch.cuda.set_device(local)

    from inputs.configs import MISTRAL_7B
    from paper_2406_00059_b200 import build, capi
    from paper_2406_00059_b200.engine import DeviceModel, Engine
    build.build()
    shape = MISTRAL_7B
    B = args.batch
    W, K = args.warmup, args.steps
    gen = W + K + 8
    vocab, reqs = codegen_workload(B, gen, prefix_min=args.prefix_min, prefix_spread=args.prefix_spread)
    max_ctx = max(r["prefix"] for r in reqs) + gen + 64
    pages_per_slot = (max_ctx + 15) // 16 + 1
    n_pages = B * pages_per_slot + 64
    dm = DeviceModel(shape, "bf16", n_pages, seed=1001, device=local)
    # chunked prefill only changes requests with multi-token prompts: the timed decode batch
    # submits 1-token prompts (synthetic prefixes); the e2e leg's 16-token prompts use it
    eng = Engine(dm, vocab, max_slots=B, max_pages_per_slot=pages_per_slot, device=local,
                 flags=(capi.ENGINE_SCAN_OFF if args.scan_off else 0) | capi.ENGINE_CHUNKED_PREFILL)
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
    ctx_start = [r["prefix"] + 1 + W for r in reqs]  # positions at the first timed step
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.perf_counter()
    ev0.record(stream)
    for _ in range(K):
        eng.step()
    ev1.record(stream)
    ev1.synchronize()
    wall = time.perf_counter() - wall0
    torch.cuda.synchronize()
    clk = clocks.stop()
    dev_ms = ev0.elapsed_time(ev1)
    perf = eng.perf()
    max_ms, total_tokens, rank_stats = reduce_over_ranks(dev_ms, B * K, [float(rank), dev_ms, float(B * K)],
                                                         device=red_dev)
    value = total_tokens / (max_ms / 1000.0)
    ctx_mean = float(np.mean([c + K / 2 for c in ctx_start]))

    # per-kernel probe (timed graph variant: event pair per launch, no PDL): kernel shares
    eng.set_kernel_timing(True)
    for _ in range(3):
        eng.step()
    kt = eng.kernel_times()
    eng.set_kernel_timing(False)
    eng.sync()
    probe_ctx = [c + K + 2 for c in ctx_start]
    by_kind = {}
    gemm_ms, gemm_bytes = 0.0, 0
    for kind, layer, ms in kt:
        by_kind.setdefault(capi.KERNEL_KINDS[kind], [0.0, 0])
        by_kind[capi.KERNEL_KINDS[kind]][0] += ms
        by_kind[capi.KERNEL_KINDS[kind]][1] += 1
        if kind in (1, 4, 5, 6, 7):
            gemm_ms += ms
            gemm_bytes += gemm_launch_bytes(shape, kind, B)
    probe_ms = sum(ms for _, _, ms in kt)
    attn_ms = by_kind.get("attention", [0, 0])[0] + by_kind.get("attention_merge", [0, 0])[0]
    kv_bytes = sum(c + 1 for c in probe_ctx) * shape.kv_bytes_per_token
    peaks, peaks_src = load_peaks()
    hbm = float(peaks["hbm_gbs"])
    pk_ms = by_kind.get("layers_persistent", [0.0, 0])[0]
    if pk_ms > 0:
        # persistent all-layers kernel: one launch per step streams every layer's projection
        # weights once and reads / appends the KV cache
        pk_bytes = pk_launch_bytes(shape, probe_ctx)
        achieved = pk_bytes / (pk_ms / 1000.0) / 1e9
        traffic = load_traffic("pk_traffic.json")
        roofline = {"bound": "hbm",
                    "kernel": "layers_persistent_kernel (all 32 layers: tcgen05 stream-K projections + paged attention, 1 launch/step)",
                    "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "peak_source": f"{peaks_src} HBM copy bandwidth",
                    "alg_bytes_per_launch": pk_bytes,
                    "traffic": (traffic or {}).get("per_launch_bytes"),
                    "traffic_detail": None if traffic is None else {
                        "alg_per_launch_bytes": traffic["alg_per_launch_bytes"], "ratio": traffic["ratio"],
                        "source": "profiles/pk_traffic.json: " + traffic["source"]},
                    "share_of_step": pk_ms / probe_ms,
                    "kernels_ms_per_step": {k: round(v[0], 4) for k, v in by_kind.items()},
                    "probe_step_ms": probe_ms}
    else:
        achieved = gemm_bytes / (gemm_ms / 1000.0) / 1e9
        traffic = load_traffic()
        roofline = {"bound": "hbm", "kernel": "gemm_tc_kernel (tcgen05 projections, cluster split-K for narrow N, all 129 launches/step)",
                    "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "peak_source": f"{peaks_src} HBM copy bandwidth",
                    "traffic": (traffic or {}).get("per_launch_bytes"),
                    "traffic_detail": None if traffic is None else {
                        "alg_per_launch_bytes": traffic["alg_per_launch_bytes"], "ratio": traffic["ratio"],
                        "source": "profiles/gemm_traffic.json: " + traffic["source"]},
                    "share_of_step": gemm_ms / probe_ms,
                    "attention": {"achieved": kv_bytes / (attn_ms / 1000.0) / 1e9, "frac": kv_bytes / (attn_ms / 1000.0) / 1e9 / hbm,
                                  "ms_per_step": attn_ms},
                    "kernels_ms_per_step": {k: round(v[0], 4) for k, v in by_kind.items()},
                    "probe_step_ms": probe_ms}
    step_bytes = step_alg_bytes(shape, [c + K / 2 for c in ctx_start])
    step_roof = {"alg_bytes_per_step": step_bytes, "achieved_GBps": step_bytes / (max_ms / K / 1000.0) / 1e9,
                 "frac": step_bytes / (max_ms / K / 1000.0) / 1e9 / hbm}
    # phase roofline: t_min = sum over phases of max(bytes / HBM, flops / TC);
    # the projections' flops count the (hi, lo) activation pair twice
    tc = float(peaks.get("bf16_tflops", PEAKS_FALLBACK["bf16_tflops"])) * 1e12
    ctx_now = [c + K / 2 for c in ctx_start]
    proj_bytes = 2.0 * shape.n_params_streamed
    proj_flops = 2.0 * shape.n_params_streamed * B * 2
    kv_tok = shape.kv_bytes_per_token
    att_bytes = sum(c + 1 for c in ctx_now) * kv_tok + B * kv_tok
    att_flops = 4.0 * shape.L * shape.H * shape.hd * sum(c + 1 for c in ctx_now)
    t_proj = max(proj_bytes / (hbm * 1e9), proj_flops / tc)
    t_att = max(att_bytes / (hbm * 1e9), att_flops / tc)
    t_meas = max_ms / K / 1000.0
    step_roof["phase_roofline"] = {"t_min_ms": (t_proj + t_att) * 1e3, "frac": (t_proj + t_att) / t_meas,
                                   "projections": "tensor" if proj_flops / tc > proj_bytes / (hbm * 1e9) else "hbm",
                                   "tc_peak_tflops": tc / 1e12}

    # end-to-end through the C ABI with host buffers: release, then a fresh batch whose
    # prompts and forced streams come from host memory; timed until every FINAL is polled and
    # every request's generated tokens are read back to the host.
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
    # whole-job e2e at N GPUs: all ranks' generated tokens / the slowest rank's wall time
    e2e_ms, e2e_tok, _ = reduce_over_ranks(e2e.pop("_dt_s") * 1e3, e2e.pop("_ntok"), [0.0], device=red_dev)
    e2e["per_rank_value"] = e2e["value"]
    e2e["value"] = e2e_tok / (e2e_ms / 1000.0)

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            toks, secs, cores, n, steps = time_oracle(shape, reqs, args.cpu_budget, 1001)
            cpu = {"value": toks / secs, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                   "sample": f"{steps} decode step(s) x {n} of the 64 codegen requests (full 32 layers, their "
                             f"synthetic prefixes), {secs:.1f} s of CPU work"}
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
                "ms_per_step": max_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "bf16", "data": "synthetic", "config": workload_config(B, ctx_mean, args.prefix_min, args.prefix_spread),
                "tokens_per_s_per_gpu": value / world, "roofline": roofline, "step_roofline": step_roof,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(perf.launches_per_step) * K,
                "clocks": clk, "wall_s_timed": wall, "segments_polled": nseg[0],
                "rank_stats": rank_stats}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(eng, reqs, tool, B):
    import numpy as np
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
            "prompt_tokens": prompt_len, "includes": "submit (host prompts + forced streams), chunked prefill "
                                                     "(CVY_ENGINE_CHUNKED_PREFILL), decode, segment polling, "
                                                     "token read-back"}


def load_traffic(name="gemm_traffic.json"):
    p = os.path.join(ROOT, "profiles", name)
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--scan-off", action="store_true", help="trigger scan disabled (overhead A/B)")
    ap.add_argument("--prefix-min", type=int, default=128, help="synthetic KV prefix: min tokens")
    ap.add_argument("--prefix-spread", type=int, default=400, help="synthetic KV prefix: + U(0, spread)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--latency-only", default="", help="comma list of workloads: run only the latency A/B")
    ap.add_argument("--latency-batch", type=int, default=0, help="override every workload's batch")
    ap.add_argument("--latency-inflight", type=int, default=0,
                    help="NEXT-3 abort-and-refill: run each workload's requests through this many slots")
    ap.add_argument("--chunked-prefill", action="store_true",
                    help="NEXT-1: prompts / observations as batched prefill passes (CVY_ENGINE_CHUNKED_PREFILL)")
    ap.add_argument("--fig6", action="store_true", help="NEXT-4: Fig. 6 tool/decode ratio sweep on the engine")
    ap.add_argument("--fig6-batch", type=int, default=16)
    args = ap.parse_args()
    if args.fig6:
        print(json.dumps({"fig6": run_fig6(args.fig6_batch, verbose=True)}), flush=True)
        return
    if args.latency_only:
        ws = args.latency_only.split(",")
        base = {"codegen": 64, "codegen_fence": 64, "search": 128, "search_call": 128, "planning": 256, "validation": 512}
        bs = {w: (args.latency_batch or base[w]) for w in ws}
        from paper_2406_00059_b200 import capi
        fl = capi.ENGINE_CHUNKED_PREFILL if args.chunked_prefill else 0
        print(json.dumps({"latency": run_latency(ws, bs, verbose=True, inflight=args.latency_inflight or None,
                                                 flags=fl), "chunked_prefill": bool(args.chunked_prefill)}),
              flush=True)
        return
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)



# ------------------------------------------------------------------ latency: partial vs sequential
def run_latency(workloads, batches, device=0, verbose=False, inflight=None, flags=0):
    """Request completion latency with tool partial execution vs sequential tool execution on
    the four workload shapes (BASELINE.json configs[1..4]); identical seeded streams and tool
    costs in both modes (the baseline is the same code with partial execution
    disabled).  Returns {workload: {...}}."""
    from inputs.configs import MISTRAL_7B
    from inputs.tool_workloads import TOOLS, build
    from paper_2406_00059_b200 import capi
    from paper_2406_00059_b200.engine import DeviceModel, Engine
    import numpy as np
    from paper_2406_00059_b200.runtime import Runtime, summarize
    prefixes = {"codegen": 128, "codegen_fence": 128, "search": 256, "search_call": 256, "planning": 512, "validation": 1792}
    max_tokens = {"codegen": 440, "codegen_fence": 460, "search": 560, "search_call": 560, "planning": 400, "validation": 320}
    pages_per = {w: (prefixes[w] + max_tokens[w] + 31) // 16 + 1 for w in workloads}
    slots = {w: (inflight or batches[w]) for w in workloads}
    need = max(slots[w] * pages_per[w] for w in workloads) + 64
    dm = DeviceModel(MISTRAL_7B, "bf16", need, seed=1002, device=device)
    Bmax = max(slots[w] for w in workloads)
    from inputs.vocab import synthetic_vocab
    eng = Engine(dm, synthetic_vocab(32000), max_slots=Bmax, max_pages_per_slot=max(pages_per.values()) + 2,
                 device=device, flags=flags)
    tool_ids = {name: eng.register_tool(name, getattr(capi, kind), delims) for name, (kind, delims) in TOOLS.items()}
    out = {}
    for w in workloads:
        res = {}
        for mode, label in ((capi.MODE_PARTIAL, "partial"), (capi.MODE_SEQUENTIAL, "sequential")):
            _, specs = build(w, batches[w], tool_ids)
            rt = Runtime(eng, mode)
            t0 = time.perf_counter()
            logs = rt.run(specs, max_inflight=inflight)
            res[label] = summarize(logs, mode)
            res[label]["steps"] = rt.steps
            if inflight:
                # abort-and-refill (NEXT-3): makespan of the whole queue through `inflight` slots
                span = max(lg.t_done for lg in logs) - t0
                res[label].update(makespan_s=span, requests_per_s=len(logs) / span, slots=inflight,
                                  queue_latency_mean_ms=float(np.mean([lg.t_done - t0 for lg in logs])) * 1e3)
            if verbose:
                print(w, label, res[label], flush=True)
        p, s_ = res["partial"]["mean_ms"], res["sequential"]["mean_ms"]
        res["improvement"] = s_ / p - 1.0        # the paper's metric
        res["reduction"] = 1.0 - p / s_           # the north star's wording
        if "detection_ms_mean" in res["partial"]:
            d_p, d_s = res["partial"]["detection_ms_mean"], res["sequential"]["detection_ms_mean"]
            res["detection_speedup"] = d_s / d_p - 1.0  # PAPER.md:203 reports 376.4%
        res["batch"] = batches[w]
        if inflight:
            res["throughput_gain"] = res["partial"]["requests_per_s"] / res["sequential"]["requests_per_s"] - 1.0
        out[w] = res
    eng.close()
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
