"""Seeded workload text generators shaped like the paper's workloads.

No figure content survives in PAPER.md, so these are synthetic streams with
the paper's *structure*: CodeGen = a Python script that runs line by line (imports,
tensor math, `:` blocks, one long final render line); Search =
three `search("...")` calls; Planning = a 4-stage LLMCompiler-style JSON
plan, one stage object per line; Validation = one JSON function-call
object with a `location` member that may lack the state.
Text only -- no method arithmetic lives here.
"""
from __future__ import annotations

import json
import random

_MODULES = ["torch", "numpy as np", "matplotlib.pyplot as plt", "math", "os", "time",
            "json", "random", "itertools", "collections"]
_VARS = ["x", "y", "t", "freq", "amp", "phase", "signal", "noise", "grid", "data", "vals",
         "acc", "total", "mean", "scale", "offset", "n", "k", "res", "out"]
_FUNCS = ["torch.sin", "torch.cos", "torch.exp", "torch.linspace", "torch.randn", "np.sqrt",
          "math.log", "torch.tanh", "np.abs", "torch.arange"]
_WORDS = ("the of and to in is for on with as by at from that this it be are or an was "
          "python code tensor plot value result search market cap apple microsoft ratio "
          "hello world program java news local city state weather report data table query "
          "answer step plan tool call function output error check format valid field").split()
_CITIES = [("Durham", "NC"), ("Austin", "TX"), ("Seattle", "WA"), ("Boston", "MA"),
           ("Denver", "CO"), ("Phoenix", "AZ"), ("Portland", "OR"), ("Atlanta", "GA"),
           ("Chicago", "IL"), ("Raleigh", "NC"), ("Madison", "WI"), ("Tucson", "AZ")]


def _expr(rng: random.Random) -> str:
    a, b = rng.choice(_VARS), rng.choice(_VARS)
    f = rng.choice(_FUNCS)
    forms = [f"{f}({a}) * {b}", f"{a} + {rng.randint(1, 99)} * {b}", f"{f}({a} / {rng.randint(2, 9)})",
             f"({a} - {b}) ** 2", f"{f}(torch.tensor([{rng.random():.3f}, {rng.random():.3f}]))"]
    return rng.choice(forms)


def codegen_script(rng: random.Random, n_lines: int = 40) -> str:
    """A Python script: 3-5 imports, assignments, `:` blocks with indented bodies and a
    blank line closing each block (the interpreter buffers a block until then,
    SPEC.md:178 / PAPER.md:148), and one long final render line."""
    lines = []
    for mod in rng.sample(_MODULES[:6], rng.randint(3, 5)):
        lines.append(f"import {mod}")
    while len(lines) < n_lines - 2:
        r = rng.random()
        if r < 0.15:
            v = rng.choice(_VARS)
            lines.append(f"for i in range({rng.randint(2, 50)}):")
            for _ in range(rng.randint(1, 3)):
                lines.append(f"    {v} = {_expr(rng)}")
            lines.append("")
        elif r < 0.22:
            fn = rng.choice(["step", "update", "normalize", "render"])
            lines.append(f"def {fn}({rng.choice(_VARS)}):")
            lines.append(f"    return {_expr(rng)}")
            lines.append("")
        else:
            lines.append(f"{rng.choice(_VARS)} = {_expr(rng)}")
    lines.append(f"plt.plot(x.numpy(), y.numpy(), label='sine wave', linewidth={rng.randint(1, 4)})")
    lines.append(f"plt.savefig('sine_{rng.randint(0, 999)}.png'); plt.show()")
    return "\n".join(lines) + "\n"


SINE_SCRIPT_13 = (
    "import torch\n"
    "import matplotlib.pyplot as plt\n"
    "x = torch.linspace(0, 4 * torch.pi, 1000)\n"
    "y = torch.sin(x)\n"
    "import numpy as np\n"
    "amp = 1.5\n"
    "y = amp * y\n"
    "fig, ax = plt.subplots()\n"
    "ax.set_title('Sine wave')\n"
    "ax.set_xlabel('x')\n"
    "ax.set_ylabel('sin(x)')\n"
    "ax.grid(True)\n"
    "ax.plot(x.numpy(), y.numpy()); plt.savefig('sine.png'); plt.show()\n"
)
"""Our own 13-line script with the paper's CodeGen shape (imports -> compute -> one long
final render line, PAPER.md:113-114).  The paper's Fig. 2 listing is elided (D5)."""


def search_calls(rng: random.Random, n: int = 3) -> str:
    langs = ["Python", "C++", "Java", "Rust", "Go", "Ruby"]
    out = []
    for lang in rng.sample(langs, n):
        out.append(f'search("hello world program in {lang} site:stackoverflow.com")')
    return "\n".join(out) + "\n"


def search_session(rng: random.Random, n: int = 3, code_lines: int = 12) -> str:
    """Search workload round: the model writes a Hello World program in
    several languages "consecutively, using tools to search online"; each `search(...)` line is
    followed by the code it drafts, so a search runs while the next part is decoded."""
    langs = ["Python", "C++", "Java", "Rust", "Go", "Ruby"]
    out = []
    for lang in rng.sample(langs, n):
        out.append(f'search("hello world program in {lang} site:stackoverflow.com")')
        out.append(f"# {lang} version, drafted while the search runs")
        for _ in range(code_lines):
            out.append(f"{rng.choice(_VARS)} = {_expr(rng)}")
    return "\n".join(out) + "\n"


def plan_with_thoughts(rng: random.Random, words: int = 30) -> str:
    """LLMCompiler/ReWOO-style plan: a short thought before each stage object (prose holds no
    brackets, so only the stage objects are JSON)."""
    stages = plan_stages(rng).strip().split("\n")
    out = []
    for st in stages:
        out.append("Thought: " + prose(rng, words))
        out.append(st)
    return "\n".join(out) + "\n"


def prose(rng: random.Random, n_words: int) -> str:
    return " ".join(rng.choice(_WORDS) for _ in range(n_words)) + "."


def plan_stages(rng: random.Random) -> str:
    """4 stages: two searches, a calculator over #E1/#E2, a formatter."""
    a, b = rng.sample(["MSFT", "AAPL", "GOOG", "AMZN", "NVDA"], 2)
    stages = [
        {"id": 1, "tool": "search", "args": {"q": f"{a} market cap"}, "deps": []},
        {"id": 2, "tool": "search", "args": {"q": f"{b} market cap"}, "deps": []},
        {"id": 3, "tool": "calculator", "args": {"expr": "#E1 / #E2"}, "deps": [1, 2]},
        {"id": 4, "tool": "format", "args": {"template": f"{a}/{b} ratio: #E3"}, "deps": [3]},
    ]
    return "\n".join(json.dumps(s, separators=(",", ":")) for s in stages) + "\n"


def validation_call(rng: random.Random, bad: bool) -> str:
    """One JSON object of 12 string members; member 2 is `location` = "<City>, <ST>"
    or, when bad, just "<City>"."""
    city, st = rng.choice(_CITIES)
    obj = {"function": "get_local_news", "topic": prose(rng, 3)[:-1],
           "location": city if bad else f"{city}, {st}"}
    for k in range(9):
        obj[f"field_{k}"] = prose(rng, rng.randint(8, 14))[:-1]
    return json.dumps(obj, separators=(", ", ": "))


def corpus(seed: int, n_docs: int = 120) -> str:
    """Text the synthetic vocabulary is learned from (all four workload shapes)."""
    rng = random.Random(seed)
    parts = []
    for i in range(n_docs):
        k = i % 4
        if k == 0:
            parts.append(codegen_script(rng))
        elif k == 1:
            parts.append(search_calls(rng) + prose(rng, 40))
        elif k == 2:
            parts.append(plan_stages(rng) + prose(rng, 20))
        else:
            parts.append(validation_call(rng, rng.random() < 0.5))
    return "\n".join(parts)
