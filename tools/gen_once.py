import os, sys, tempfile
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_1805_11462_b200 as ob
d = tempfile.mkdtemp()
m = ob.Model(synth.weights_file("c2", d), 0, "bf16")
R = int(os.environ.get("GEN_ROWS", "150"))
h = np.tanh(np.random.default_rng(0).normal(size=(R, 500))).astype(np.float32)
for i in range(6):
    m.test_gen(h, 5)
