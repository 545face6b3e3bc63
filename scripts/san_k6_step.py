"""A few decode steps of a 1-layer 7B-width slice with a 32k vocabulary and a JSON_MEMBER tool,
teacher-forced validator calls, B = 8: the LM-head GEMM + fused sample/scan/compaction/publish
(K6) under compute-sanitizer (scripts/sanitize.sh).  No graphs (every launch visible)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import random  # noqa: E402

from inputs.configs import MISTRAL_7B, slice_of  # noqa: E402
from inputs.vocab import Tokenizer, synthetic_vocab  # noqa: E402
from inputs.workloads import validation_call  # noqa: E402
from paper_2406_00059_b200 import capi  # noqa: E402
from paper_2406_00059_b200.engine import DeviceModel, Engine  # noqa: E402

shape = slice_of(MISTRAL_7B, L=1, name="7b-L1")
vocab = synthetic_vocab(32000)
tok = Tokenizer(vocab)
dm = DeviceModel(shape, "bf16", 256, seed=3)
eng = Engine(dm, vocab, max_slots=8, max_pages_per_slot=16, flags=capi.ENGINE_NO_GRAPH)
tool = eng.register_tool("validator", capi.PARSER_JSON_MEMBER)
rng = random.Random(1)
for i in range(8):
    ids = tok.encode(validation_call(rng, i % 2 == 0))[:40]
    eng.submit_request([1], len(ids), tool_id=tool, forced=ids, synth_prefix_len=20, synth_seed=i)
n = 0
for _ in range(12):
    eng.step()
    n += len(eng.poll_segments())
eng.sync()
n += len(eng.poll_segments())
eng.close()
print("k6 sanitizer run ok, records:", n)
