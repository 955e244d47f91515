"""The generator's scheduling modes change only when and where tiles are
computed - the K-outer batches, their TMEM columns, the staging overlay - never what: every
mode must produce bit-identical translations.  ONMT_GEN_OVL is read once per process, so each
mode runs in its own subprocess on the same c2 weights and corpus."""
import os
import subprocess
import sys

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import synth, paper_1805_11462_b200 as ob
m = ob.Model({path!r}, 0, "bf16")
ids, lens = synth.make_corpus("c2")
out = m.translate(ids, lens, 5, 40, 0.0)
np.savez({dst!r}, hyps=out["hyps"], lens=out["lens"], scores=out["scores"], logp=out["token_logp"])
"""


def _run(path, mode, dst):
    env = dict(os.environ, ONMT_GEN_OVL=str(mode))
    code = _SCRIPT.format(root=ROOT, path=path, dst=dst)
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(dst)


def test_generator_modes_bit_identical(weight_cache, tmp_path):
    """Single K-outer batch (ONMT_GEN_OVL=0), batches of one tile (1) and the default (2)."""
    path = synth.weights_file("c2", weight_cache)
    outs = {mode: _run(path, mode, str(tmp_path / f"m{mode}.npz")) for mode in (0, 1, 2)}
    ref = outs[2]
    for mode in (0, 1):
        for key in ("hyps", "lens", "scores", "logp"):
            assert np.array_equal(outs[mode][key], ref[key]), (mode, key)


def test_regrouped_gate_gemm_bit_identical(weight_cache):
    """c4's single-split decoder gate GEMMs run in 160-row groups (128 CTAs) instead of the
    operand's 224-row groups (96 CTAs) (option regroup): every output is the
    same K-ordered tensor-core sum, so translations must be bit-identical."""
    import paper_1805_11462_b200 as ob
    path = synth.weights_file("c4", weight_cache)
    ids, lens = synth.make_corpus("c4")
    outs = {}
    for v in (1, 0):
        with ob.Model(path, 0, "bf16") as m:
            m.set_option("regroup", v)
            outs[v] = m.translate(ids, lens, 5, 16, 0.6)
    for key in ("hyps", "lens", "scores", "token_logp"):
        assert np.array_equal(outs[0][key], outs[1][key]), key
