"""Diagnostic: recurrent-split step vs the per-layer step vs the oracle (token log-p error of the
GPU hypotheses, hypothesis agreement), and the per-call device time of both."""
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1805_11462_b200 as ob  # noqa: E402
from oracle import OracleModel, load_model_tensors, score_sequence  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
ML = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cache = os.environ.get("ONMT_WEIGHT_CACHE", os.path.join(tempfile.gettempdir(), "onmt_weights"))
path = synth.weights_file(wl, cache)
w = synth.WORKLOADS[wl]
om = OracleModel(load_model_tensors(path, "bf16"))
ids, lens = synth.make_corpus(wl, int(sys.argv[3]) if len(sys.argv) > 3 else None)
ids = np.ascontiguousarray(ids[:, :int(lens.max())])
m = ob.Model(path, 0, "bf16")
outs = {}
for rs in (1, 0):
    m.set_option("rsplit", rs)
    out = m.translate(ids, lens, w.decode.beam, ML, w.decode.alpha)
    m.launches(reset=True)
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        out = m.translate(ids, lens, w.decode.beam, ML, w.decode.alpha)
    dt = (time.perf_counter() - t0) / 5
    nl = m.launches(reset=True) // 5
    errs = []
    for b in range(0, len(lens), max(1, len(lens) // 4)):
        src = [int(x) for x in ids[b, :lens[b]]]
        hyp = [int(x) for x in out["hyps"][b, :out["lens"][b]]]
        tf = np.array(score_sequence(om, src, hyp))
        errs.append(float(np.max(np.abs(tf - out["token_logp"][b, :len(hyp)]))))
    outs[rs] = out
    print(f"{wl} rsplit={rs}: {dt * 1e3:.3f} ms/call (host), {nl} launches, max token logp err {max(errs):.2e}", flush=True)
same = (outs[0]["hyps"] == outs[1]["hyps"]).all(axis=1)
dl = np.max(np.abs(outs[0]['token_logp'] - outs[1]['token_logp']), axis=1)
bad = np.nonzero(dl > 1e-4)[0]
for b in bad[:6]:
    src = [int(x) for x in ids[b, :lens[b]]]
    e = {}
    for rs in (0, 1):
        hyp = [int(x) for x in outs[rs]["hyps"][b, :outs[rs]["lens"][b]]]
        e[rs] = np.abs(np.array(score_sequence(om, src, hyp)) - outs[rs]["token_logp"][b, :len(hyp)])
    print(f"sentence {b} (rows {b * w.decode.beam}..): rsplit=1 err {e[1].max():.2e} first>1e-4 at t={np.argmax(e[1] > 1e-4) + 1}; rsplit=0 err {e[0].max():.2e}")
print(f"hypotheses identical for {same.sum()}/{len(same)} sentences; max |d logp| "
      f"{np.max(np.abs(outs[0]['token_logp'] - outs[1]['token_logp'])):.2e}")
