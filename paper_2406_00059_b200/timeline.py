"""Per-request execution timelines of the host runtime (the paper's Fig. 3 / Fig. 7 views).

PAPER.md:116-121 (Fig. 3, CodeGen: "only line 13 needs to be executed after the decoding")
and PAPER.md:215-221 (Fig. 7, Validation: the abort lands long before the decode would end).
Events follow SPEC.md:339's TimelineEvent kinds -- RoundStart, TokenDecoded, PieceDispatched,
ToolStart, PieceExecuted, ToolDone, RoundEnd, AbortSignal, ResponseReady -- built from a
RequestLog of `runtime.Runtime`; the export is SPEC.md:387's tab-separated line
`t_us  kind  round  job  piece  detail`, and `gantt` renders SPEC.md:581's text chart (one lane
for the decode, one per tool instance).  Times are host monotonic, relative to the request's
submit.  TokenDecoded is observed at segment granularity: the token holding a piece's last byte,
at the moment its record was polled (the device publishes pieces, not single tokens).
"""
from __future__ import annotations

KINDS = ("RoundStart", "TokenDecoded", "PieceDispatched", "ToolStart", "PieceExecuted", "ToolDone",
         "RoundEnd", "AbortSignal", "ResponseReady")


def events(log):
    """[(t_us, kind, round, job, piece, detail)] of one request, sorted by time (stable)."""
    t0 = log.t_submit
    us = lambda t: int(round((t - t0) * 1e6))
    ev = []
    job = log.rid
    for r in range(len(log.round_start)):
        ev.append((us(log.round_start[r]), "RoundStart", r, job, -1, ""))
        last_end = None
        for j, w in enumerate(log.seg_work[r]):
            ev.append((us(log.seg_avail[r][j]), "TokenDecoded", r, job, j, f"token={log.seg_token[r][j]}"))
            if log.seg_disp[r][j] is not None:
                ev.append((us(log.seg_disp[r][j]), "PieceDispatched", r, job, j, f"instance={w.instance}"))
                ev.append((us(log.seg_begin[r][j]), "ToolStart", r, job, j, f"cost_ms={w.cost_s * 1e3:.3f}"))
                ev.append((us(log.seg_end[r][j]), "PieceExecuted", r, job, j, "abort" if w.abort else "ok"))
                last_end = max(last_end or 0.0, log.seg_end[r][j])
        if last_end is not None:
            ev.append((us(last_end), "ToolDone", r, job, -1, f"pieces={len(log.seg_work[r])}"))
        if log.round_final[r] is not None:
            ev.append((us(log.round_final[r]), "RoundEnd", r, job, -1, ""))
    if log.t_abort is not None:
        ev.append((us(log.t_abort), "AbortSignal", log.round, job, -1, ""))
    if log.done:
        ev.append((us(log.t_done), "ResponseReady", log.round, job, -1, ""))
    order = {k: i for i, k in enumerate(KINDS)}
    return sorted(ev, key=lambda e: (e[0], order[e[1]]))


def to_tsv(evs) -> str:
    return "".join(f"{t}\t{k}\t{r}\t{j}\t{p}\t{d}\n" for (t, k, r, j, p, d) in evs)


def write_tsv(logs, path: str):
    with open(path, "w") as f:
        f.write("t_us\tkind\tround\tjob\tpiece\tdetail\n")
        for lg in logs:
            f.write(to_tsv(events(lg)))


def gantt(evs, width: int = 100) -> str:
    """Text Gantt chart of one request: the decode lane (RoundStart -> RoundEnd per round) and one
    lane per tool piece (ToolStart -> PieceExecuted); '!' marks an AbortSignal."""
    if not evs:
        raise ValueError("empty timeline")
    t_end = max(e[0] for e in evs) or 1
    col = lambda t: min(width - 1, int(t * (width - 1) / t_end))
    rows = []
    dec = [" "] * width
    starts = {}
    for (t, k, r, j, p, d) in evs:
        if k == "RoundStart":
            starts[r] = t
        elif k == "RoundEnd":
            for c in range(col(starts.get(r, 0)), col(t) + 1):
                dec[c] = "="
        elif k == "AbortSignal":
            dec[col(t)] = "!"
    rows.append("decode   |" + "".join(dec) + "|")
    begin = {}
    for (t, k, r, j, p, d) in evs:
        if k == "ToolStart":
            begin[(r, p)] = t
        elif k == "PieceExecuted":
            lane = [" "] * width
            for c in range(col(begin.get((r, p), t)), col(t) + 1):
                lane[c] = "#"
            rows.append(f"r{r} p{p:<4}|" + "".join(lane) + "|")
    rows.append(f"0 us{' ' * (width - 8)}{t_end} us")
    return "\n".join(rows) + "\n"
