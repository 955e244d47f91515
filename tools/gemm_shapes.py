import os, sys, tempfile
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_1805_11462_b200 as ob
d = tempfile.mkdtemp()
cfg = synth.ModelConfig(1, 40, 300, 500, 1000, False, True)
p = os.path.join(d, "k.mnmt"); synth.write_mnmt(p, synth.random_model_tensors(cfg, 3, 0.1))
m = ob.Model(p, 0, "bf16")
rng = np.random.default_rng(0)
for (M, N, K, S) in [(2000, 150, 64, 1), (2000, 150, 512, 0), (2000, 150, 1536, 0), (2000, 150, 1536, 4), (2000, 150, 1536, 16), (500, 150, 1024, 0)]:
    W = rng.uniform(-0.1, 0.1, (M, K)).astype(np.float32); X = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    for i in range(3):
        m.test_gemm(W, X, S)
