import os, sys, tempfile
import numpy as np
sys.path.insert(0, "/root/repo")
import synth, paper_1805_11462_b200 as ob
from oracle import bf16_round
d = tempfile.mkdtemp()
cfg = synth.ModelConfig(2, 16, 32, 60, 40, False, True)
t = synth.random_model_tensors(cfg, 11, 0.3)
b = np.random.default_rng(0).uniform(0, 2, cfg.v_tgt).astype(np.float32); b[7] = 3.0; b[3] = 2.4
t["gen.b"] = b; t["gen.w"] = t["gen.w"] * 3.0
p = os.path.join(d, "k.mnmt"); synth.write_mnmt(p, t)
m = ob.Model(p, 0, "bf16")
W = bf16_round(t["gen.w"]).astype(np.float64); bb = bf16_round(t["gen.b"]).astype(np.float64)
for R, k in [(18, 3), (6, 3), (30, 5), (18, 1), (17, 16)]:
    h = np.tanh(np.random.default_rng(R).normal(size=(R, 32))).astype(np.float32)
    z = h.astype(np.float64) @ W.T + bb
    lse, tz, ti = m.test_gen(h, k)
    bad = 0
    for r in range(R):
        order = np.lexsort((np.arange(z.shape[1]), -z[r]))[:k]
        if not np.allclose(tz[r], z[r, order], atol=1e-4): bad += 1; print(R, k, r, tz[r], z[r, order], ti[r], order)
    print(R, k, "bad rows", bad, "lse err", np.abs(lse - (z.max(1) + np.log(np.exp(z - z.max(1, keepdims=True)).sum(1)))).max())
