"""Diagnostic: for the given batch size / max_len of a workload, the first token of the GPU's
returned hypothesis whose log-p differs from the oracle's teacher-forced log-p by > tol."""
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
sents = [int(x) for x in sys.argv[4].split(",")]
opts = [kv.split("=") for kv in sys.argv[5:]]
cache = os.environ.get("ONMT_WEIGHT_CACHE", os.path.join(tempfile.gettempdir(), "onmt_weights"))
path = synth.weights_file(wl, cache)
w = synth.WORKLOADS[wl]
om = OracleModel(load_model_tensors(path, "bf16"))
ids, lens = synth.make_corpus(wl, B)
m = ob.Model(path, 0, "bf16")
for k, v in opts:
    m.set_option(k, int(v))
S = int(lens.max())
out = m.translate(np.ascontiguousarray(ids[:, :S]), lens, w.decode.beam, ML, w.decode.alpha, trace=True)
for b in sents:
    src = [int(x) for x in ids[b, :lens[b]]]
    hyp = [int(x) for x in out["hyps"][b, :out["lens"][b]]]
    tf = np.array(score_sequence(om, src, hyp))
    d = np.abs(tf - out["token_logp"][b, :len(hyp)])
    bad = np.nonzero(d > 2e-3)[0]
    print(f"{wl} B={B} ML={ML} opts={opts} sent {b}: n={len(hyp)} max err {d.max():.3e} first bad t={bad[0] + 1 if len(bad) else None}"
          f" errs {np.array2string(d[max(0, (bad[0] if len(bad) else 0) - 2):(bad[0] if len(bad) else 0) + 4], precision=3)}",
          flush=True)
