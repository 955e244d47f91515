"""Diagnostic: sentences whose token log-p disagree with the oracle (> 1e-4) for a batch size,
under runtime options name=value."""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1805_11462_b200 as ob  # noqa: E402
from oracle import OracleModel, load_model_tensors, score_sequence  # noqa: E402

wl, B, ML = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
opts = [kv.split("=") for kv in sys.argv[4:]]
cache = os.environ.get("ONMT_WEIGHT_CACHE", os.path.join(tempfile.gettempdir(), "onmt_weights"))
path = synth.weights_file(wl, cache)
w = synth.WORKLOADS[wl]
om = OracleModel(load_model_tensors(path, "bf16"))
ids, lens = synth.make_corpus(wl, B)
ids = np.ascontiguousarray(ids[:, :int(lens.max())])
m = ob.Model(path, 0, "bf16")
for k, v in opts:
    m.set_option(k, int(v))
out = m.translate(ids, lens, w.decode.beam, ML, w.decode.alpha)
bad = []
for b in range(B):
    src = [int(x) for x in ids[b, :lens[b]]]
    hyp = [int(x) for x in out["hyps"][b, :out["lens"][b]]]
    e = np.abs(np.array(score_sequence(om, src, hyp)) - out["token_logp"][b, :len(hyp)])
    if e.max() > 1e-4:
        bad.append((b, int(np.argmax(e > 1e-4)) + 1, float(e.max())))
print(f"{wl} B={B} R={B * w.decode.beam} opts={opts}: bad sentences (b, first t, err) {bad}", flush=True)
