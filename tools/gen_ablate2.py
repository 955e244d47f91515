"""Generator timing vs rows (N) and ablation modes."""
import os, sys, tempfile
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_1805_11462_b200 as ob
d = tempfile.mkdtemp()
m = ob.Model(synth.weights_file("c2", d), 0, "bf16")
m.set_option("gen_multicast", 0)
m.set_option("profile", 1)
for R in (128, 150, 256):
    h = np.tanh(np.random.default_rng(0).normal(size=(R, 500))).astype(np.float32)
    for mode in ["0", "2", "5"]:
        os.environ["ONMT_GEN_EPI_MODE"] = mode
        for i in range(3):
            m.test_gen(h, 5)
        m.kernel_time("gen", reset=True)
        for i in range(20):
            m.test_gen(h, 5)
        ms, n = m.kernel_time("gen", reset=True)
        print(f"R={R} mode={mode}: {1000 * ms / n:.2f} us", flush=True)
