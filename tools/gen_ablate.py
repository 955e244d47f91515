"""Time the persistent generator alone on the c2 model (150 rows): epilogue ablations
(ONMT_GEN_EPI_MODE 0 full / 1 stage only / 2 drain only) x activation multicast on/off."""
import os, sys, tempfile
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1805_11462_b200 as ob
d = tempfile.mkdtemp()
m = ob.Model(synth.weights_file("c2", d), 0, "bf16")
h = np.tanh(np.random.default_rng(0).normal(size=(150, 500))).astype(np.float32)
ref = None
for mc in (0,):
    m.set_option("gen_multicast", mc)
    for mode in ["0", "1", "2", "3", "4", "5"]:
        os.environ["ONMT_GEN_EPI_MODE"] = mode
        m.set_option("profile", 1)
        for i in range(3):
            out = m.test_gen(h, 5)
        if mode == "0":
            if ref is None:
                ref = out
            else:
                assert np.allclose(ref[0], out[0], atol=2e-6), "LSE changed"
                assert np.array_equal(ref[1], out[1]) and np.array_equal(ref[2], out[2]), "top-k changed"
                print("multicast results match (LSE within 2e-6, top-k identical)")
        m.kernel_time("gen", reset=True)
        for i in range(20):
            m.test_gen(h, 5)
        ms, n = m.kernel_time("gen", reset=True)
        print(f"multicast={mc} epi_mode={mode}: gen avg {1000 * ms / n:.2f} us over {n}", flush=True)
