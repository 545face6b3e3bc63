"""The four tool-using workload shapes of BASELINE.json configs[1..4] as multi-round requests
with seeded tool-stub cost models (SURVEY.md 8(d) "Configs restated").

The paper gives no per-line or per-call tool costs (its Fig. 3 blocks are "not to scale",
PAPER.md:119); these distributions are calibration knobs, identical in both modes:
  codegen   : Python-interpreter stub, one serial instance (codegen_fence: the same inside a
              ```python block between prose, FENCE parser); a line costs U(50,300) ms if it
              imports, U(300,600) ms for the final render line, U(1,20) ms otherwise; a `:`
              block is buffered until its closing blank line.
  search    : 3 `search("...")` lines, each followed by the code drafted for that language
              ("the LLM decoding for the next search"), each search its own
              instance, U(200,1000) ms; observations are injected and a 100-token answer follows.
  planning  : 4 JSON stage objects (JSON_OBJECT parser), each after a short thought;
              searches U(200,1000) ms, calculator 1 ms after stages 1-2, formatter 1 ms after
              stage 3; answer 60 tokens.
  validation: one 12-member JSON call (JSON_MEMBER parser), validator 0.05 ms per member;
              a `location` member without ", ST" aborts the request.
  sweep     : NEXT-4 / Fig. 6: one round of n lines through the interpreter
              stub, each line costing r x (its share of the round's decode time), so that the
              round's tool time t = r x g for a chosen ratio r; one serial instance.
No method arithmetic lives here.
"""
from __future__ import annotations

import json
import random

from .vocab import Tokenizer, synthetic_vocab
from .workloads import codegen_script, plan_with_thoughts, prose, search_session, validation_call


def _codegen_plan(rng):
    state = {"pending": 0.0, "in_block": False}
    costs = {}

    def plan(j, data: bytes, flags: int = 0):
        from paper_2406_00059_b200.runtime import SegmentWork
        if flags & (8 | 16):
            return None  # FENCE markers (CVY_SEG_OPEN / CLOSE) are indicators, not code
        line = data.decode(errors="replace")
        body = line.strip()
        if j not in costs:
            if body.startswith("import"):
                costs[j] = rng.uniform(0.050, 0.300)
            elif "savefig" in body or "plt.show" in body or "plt.plot" in body:
                costs[j] = rng.uniform(0.300, 0.600)
            elif body == "":
                costs[j] = 0.0
            else:
                costs[j] = rng.uniform(0.001, 0.020)
        c = costs[j]
        if body.endswith(":"):
            state["in_block"] = True
            state["pending"] = c
            return SegmentWork(0.0, 0)
        if state["in_block"]:
            if body == "":
                c, state["pending"], state["in_block"] = state["pending"], 0.0, False
                return SegmentWork(c, 0)
            state["pending"] += c
            return SegmentWork(0.0, 0)
        return SegmentWork(c, 0)
    return plan


def _search_plan(rng):
    costs = [rng.uniform(0.2, 1.0) for _ in range(16)]
    seen = [0]

    def plan(j, data: bytes, flags: int = 0):
        from paper_2406_00059_b200.runtime import SegmentWork
        if not data.strip().startswith(b"search("):
            return None  # drafted code lines are not tool input
        k = seen[0]
        seen[0] += 1
        return SegmentWork(costs[k % 16], instance=k)
    return plan


def _search_call_plan(rng):
    """@call search {...} regions (CALL parser, R22): the OPEN record (function name decoded)
    starts the search tool's fixed setup (connection, U(100,300) ms) on a fresh instance; the
    argument fields arrive as pieces; the CLOSE record (object complete) runs the query
    (U(200,1000) ms) on the same instance, after its setup."""
    state = {"inst": -1}

    def plan(j, data: bytes, flags: int = 0):
        from paper_2406_00059_b200.runtime import SegmentWork
        if flags & 8:
            state["inst"] += 1
            return SegmentWork(rng.uniform(0.1, 0.3), instance=state["inst"])
        if flags & 16:
            return SegmentWork(rng.uniform(0.2, 1.0), instance=state["inst"])
        return SegmentWork(0.0, instance=max(state["inst"], 0))
    return plan


def _planning_plan(rng):
    costs = [rng.uniform(0.2, 1.0), rng.uniform(0.2, 1.0)]

    def plan(j, data: bytes, flags: int = 0):
        from paper_2406_00059_b200.runtime import SegmentWork
        txt = data.decode(errors="replace")
        try:
            st = json.loads(txt[txt.index("{"):].strip())
        except Exception:
            return None
        sid = int(st.get("id", j + 1)) - 1
        deps = [d - 1 for d in st.get("deps", []) if 0 <= d - 1 < j]
        tool = st.get("tool")
        cost = costs[sid] if tool == "search" and sid < 2 else 0.001
        return SegmentWork(cost, instance=j, deps=deps)
    return plan


def _validation_plan():
    def plan(j, data: bytes, flags: int = 0):
        from paper_2406_00059_b200.runtime import SegmentWork
        txt = data.decode(errors="replace")
        bad = False
        if '"location"' in txt:
            rest = txt.split('"location"', 1)[1].split('"')
            value = rest[1] if len(rest) > 1 else ""
            bad = ", " not in value  # "<City>, <ST>" required by the news API
        return SegmentWork(0.00005, instance=0, abort=bad)
    return plan


def build(workload: str, B: int, tool_ids: dict, seed: int = 2000, indices=None):
    """Returns (vocab, [RequestSpec]) for one workload shape: requests 0..B-1 of the config's
    total batch, or only the global indices given (a rank's share under the router)."""
    from paper_2406_00059_b200.runtime import RequestSpec, Round
    vocab = synthetic_vocab(32000)
    tok = Tokenizer(vocab)
    specs = []
    for b in (range(B) if indices is None else indices):
        rng = random.Random(seed * 100003 + b)
        if workload == "codegen":
            text = codegen_script(rng, 40)
            rounds = [Round(tok.encode(text)[:420], tool_ids["interp"], _codegen_plan(rng))]
            prefix = 128
        elif workload == "codegen_fence":
            # the paper's own indicators: prose, a ```python block, prose; the
            # FENCE parser (NEXT-2) sends only the block's lines to the interpreter
            text = ("Here is the script.\n```python\n" + codegen_script(rng, 36) + "```\n" +
                    "It draws the sine wave and saves the figure to sine.png.")
            rounds = [Round(tok.encode(text)[:440], tool_ids["interp_fence"], _codegen_plan(rng))]
            prefix = 128
        elif workload == "search":
            r0 = tok.encode(search_session(rng, 3))
            obs = tok.encode("\n[OBSERVATION search]\n" + prose(rng, 60) + "\n")[:96]
            r1 = tok.encode("The answer: " + prose(rng, 80))[:100]
            rounds = [Round(r0, tool_ids["search"], _search_plan(rng), obs), Round(r1, -1)]
            prefix = 256
        elif workload == "search_call":
            # the Search workload with @call syntax: each call is decoded as
            # "@call search {json args}" between drafted code lines
            parts = []
            for k in range(3):
                parts.append("@call search " + json.dumps({"q": "hello world in " + ["Python", "C++", "Java"][k],
                                                           "site": "stackoverflow.com", "n": 3}))
                parts.append(codegen_script(rng, 6).strip())
            r0 = tok.encode("\n".join(parts) + "\n")
            obs = tok.encode("\n[OBSERVATION search]\n" + prose(rng, 60) + "\n")[:96]
            r1 = tok.encode("The answer: " + prose(rng, 80))[:100]
            rounds = [Round(r0, tool_ids["search_call"], _search_call_plan(rng), obs), Round(r1, -1)]
            prefix = 256
        elif workload == "planning":
            r0 = tok.encode(plan_with_thoughts(rng))
            obs = tok.encode("\n[OBSERVATION plan]\n" + prose(rng, 30) + "\n")[:48]
            r1 = tok.encode("Result: " + prose(rng, 50))[:60]
            rounds = [Round(r0, tool_ids["planner"], _planning_plan(rng), obs), Round(r1, -1)]
            prefix = 512
        elif workload == "validation":
            bad = rng.random() < 0.5
            r0 = tok.encode(validation_call(rng, bad))[:300]
            rounds = [Round(r0, tool_ids["validator"], _validation_plan())]
            prefix = 1792
        else:
            raise ValueError(workload)
        specs.append(RequestSpec([1, rng.randrange(259, 32000)], rounds, synth_prefix=prefix, synth_seed=b))
    return vocab, specs


TOOLS = {"interp": ("PARSER_LITERAL", [b"\n"]), "interp_fence": ("PARSER_FENCE", [b"python"]),
         "search_call": ("PARSER_CALL", [b"search"]),
         "search": ("PARSER_LITERAL", [b"\n"]),
         "planner": ("PARSER_JSON_OBJECT", []), "validator": ("PARSER_JSON_MEMBER", [])}


def build_sweep(B: int, tool_id: int, r: float, tok_s: float, n_lines: int = 24, seed: int = 3000):
    """Fig. 6 sweep requests (NEXT-4): every request decodes n_lines lines; line j costs
    r * tok_s * (tokens attributed to line j), tokens attributed in proportion to bytes, so the
    round's tool time is r times its decode time at a per-token decode time tok_s (measured on
    the engine by the caller).  Returns (vocab, [RequestSpec], tokens_per_round)."""
    from paper_2406_00059_b200.runtime import RequestSpec, Round, SegmentWork
    vocab = synthetic_vocab(32000)
    tok = Tokenizer(vocab)
    specs = []
    n_tok = 0
    for b in range(B):
        rng = random.Random(seed * 100003 + b)
        lines = []
        for j in range(n_lines):
            v = "x%d" % rng.randrange(100)
            lines.append(rng.choice([f"{v} = compute({rng.randrange(1000)}, {rng.randrange(1000)})",
                                     f"print({v} + {rng.randrange(100)})",
                                     f"{v} = np.mean(data[{rng.randrange(64)}:])"]))
        text = "\n".join(lines) + "\n"
        ids = tok.encode(text)
        n_tok += len(ids)
        per_byte = tok_s * len(ids) / len(text.encode())
        costs = [r * per_byte * (len(ln) + 1) for ln in lines]

        def plan(j, data, flags=0, costs=costs):
            return SegmentWork(costs[j] if j < len(costs) else 0.0, 0)
        specs.append(RequestSpec([1, rng.randrange(259, 32000)], [Round(ids, tool_id, plan)], synth_prefix=64,
                                 synth_seed=b))
    return vocab, specs, n_tok / max(1, B)
