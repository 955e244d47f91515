"""Reading R34 evidence: how much the fp64 oracle's teacher-forced token log-probs
move under a relative perturbation of every weight by the working precision's unit roundoff
(fp32 2^-23, bf16 split activations 2^-18), on the toy models of the GPU parity suite and on c2.
Prints one line per (model, precision, sentence): max |d log p| per token and max |d cumulative|."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth  # noqa: E402
from oracle import OracleModel, beam_search, load_model_tensors  # noqa: E402
from parity import derived_tolerances  # noqa: E402


def bf16(t):
    import torch
    return {k: torch.from_numpy(v).to(torch.bfloat16).double().numpy() for k, v in t.items()}


def toy(bi, scale, peaky):
    cfg = synth.ModelConfig(2, 16, 32, 60, 40, bi, not bi)
    t = synth.random_model_tensors(cfg, 11, scale)
    if peaky:
        b = np.random.default_rng(0).uniform(0, 2, cfg.v_tgt).astype(np.float32)
        b[7] = 3.0
        b[synth.EOS] = 2.8
        t["gen.b"] = b
        t["attn.w_out"] = t["attn.w_out"] * 0.5
        t["gen.w"] = t["gen.w"] * 3.0
    return {k: v.astype(np.float64) for k, v in t.items()}


def main():
    rows = []
    for name, t in [("toy scale 1.5 uni", toy(False, 1.5, False)), ("toy scale 1.5 bi", toy(True, 1.5, False)),
                    ("toy scale 0.3 peaky uni", toy(False, 0.3, True)), ("toy scale 0.3 peaky bi", toy(True, 0.3, True))]:
        for prec in ("fp32", "bf16"):
            om = OracleModel(bf16(t) if prec == "bf16" else t)
            rng = np.random.default_rng(103)
            for b in range(4):
                src = [int(x) for x in rng.integers(4, 60, int(rng.integers(1, 12)))]
                hyp = beam_search(om, src, 3, 15, 0.6)["tokens"]
                _, _, d_tok, d_cum = derived_tolerances(om, src, hyp, prec)
                rows.append((name, prec, b, len(hyp), d_tok, d_cum))
    if "--c2" in sys.argv:
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            om = OracleModel(load_model_tensors(synth.weights_file("c2", d), "bf16"))
        ids, lens = synth.make_corpus("c2", 2)
        for b in range(2):
            src = [int(v) for v in ids[b, :lens[b]]]
            hyp = beam_search(om, src, 5, 100, 0.0)["tokens"]
            for prec in ("fp32", "bf16"):
                _, _, d_tok, d_cum = derived_tolerances(om, src, hyp, prec)
                rows.append(("c2 (bf16 weights)", prec, b, len(hyp), d_tok, d_cum))
    for r in rows:
        print(f"{r[0]:26s} {r[1]:5s} sent {r[2]} n={r[3]:3d}  max|d logp| {r[4]:.2e}  max|d cum| {r[5]:.2e}")


if __name__ == "__main__":
    main()
