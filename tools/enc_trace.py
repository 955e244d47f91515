"""Per-step phase timings of the persistent encoder recurrence (ONMT_ENC_TRACE=1: CTA 0's
%globaltimer stamps of steps 8-11 of every layer, printed by the runtime) and the encode time
of a workload's batch (GPU box)."""
import os, sys, tempfile, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1805_11462_b200 as ob

wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
d = tempfile.mkdtemp()
path = synth.weights_file(wl, d)
ids, lens = synth.make_corpus(wl)
m = ob.Model(path, 0, "bf16")
for _ in range(3):
    m.encode(ids, lens)
import torch
torch.cuda.synchronize()
t0 = time.perf_counter()
n = 10
for _ in range(n):
    m.encode(ids, lens)
torch.cuda.synchronize()
print(f"{wl}: encode {1e3 * (time.perf_counter() - t0) / n:.3f} ms per batch (B={len(lens)}, S_max={int(lens.max())}, host wall)")
os.environ["ONMT_ENC_TRACE"] = "1"
m.encode(ids, lens)
