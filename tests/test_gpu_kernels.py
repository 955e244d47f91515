"""Kernel-level GPU tests through the C-ABI test entry points (tcgen05 GEMM, SIMT GEMM,
fused generator/log-softmax/top-k) against fp64 numpy."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def models(tmp_path_factory):
    import paper_1805_11462_b200 as ob
    d = tmp_path_factory.mktemp("k")
    cfg = synth.ModelConfig(1, 40, 300, 500, 1000, False, True)
    t = synth.random_model_tensors(cfg, 3, 0.1)
    p = str(d / "k.mnmt")
    synth.write_mnmt(p, t)
    mb = ob.Model(p, 0, "bf16")
    mf = ob.Model(p, 0, "fp32")
    yield mb, mf, t
    mb.close(); mf.close()


def bf16(x):
    from oracle import bf16_round
    return bf16_round(np.asarray(x, np.float32)).astype(np.float64)


@pytest.mark.parametrize("M,N,K,splits", [(128, 16, 64, 1), (300, 150, 500, 0), (2000, 150, 1500, 0),
                                          (256, 160, 128, 2), (130, 300, 200, 3), (512, 7, 1000, 8),
                                          (1000, 1536, 500, 1), (64, 33, 40, 1)])
def test_tc_gemm_vs_numpy(models, M, N, K, splits):
    mb, _, _ = models
    rng = np.random.default_rng(M + N + K)
    W = rng.uniform(-0.1, 0.1, (M, K)).astype(np.float32)
    X = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    got = mb.test_gemm(W, X, splits).astype(np.float64)
    ref = X.astype(np.float64) @ bf16(W).T
    # split-bf16 activations: |err| <~ 2^-17 * sum|w x|
    bound = 2.0 ** -15 * (np.abs(X).astype(np.float64) @ np.abs(bf16(W)).T) + 1e-6
    assert np.all(np.abs(got - ref) <= bound), float(np.max(np.abs(got - ref) / bound))


@pytest.mark.parametrize("M,N,K,splits", [(128, 16, 64, 1), (300, 150, 500, 0), (130, 300, 200, 3)])
def test_simt_gemm_fp32_vs_numpy(models, M, N, K, splits):
    _, mf, _ = models
    rng = np.random.default_rng(7 + M)
    W = rng.uniform(-0.1, 0.1, (M, K)).astype(np.float32)
    X = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    got = mf.test_gemm(W, X, splits).astype(np.float64)
    ref = X.astype(np.float64) @ W.astype(np.float64).T
    np.testing.assert_allclose(got, ref, atol=2e-6 * K ** 0.5, rtol=0)


@pytest.mark.parametrize("R,k", [(1, 1), (6, 3), (150, 5), (160, 10), (17, 16), (300, 5)])
@pytest.mark.parametrize("which", ["bf16", "fp32"])
def test_gen_lse_topk(models, R, k, which):
    mb, mf, t = models
    m = mb if which == "bf16" else mf
    rng = np.random.default_rng(R * 31 + k)
    h = np.tanh(rng.normal(size=(R, 300))).astype(np.float32)
    W = bf16(t["gen.w"]) if which == "bf16" else t["gen.w"].astype(np.float64)
    b = bf16(t["gen.b"]) if which == "bf16" else t["gen.b"].astype(np.float64)
    z = h.astype(np.float64) @ W.T + b
    lse_ref = z.max(1) + np.log(np.exp(z - z.max(1, keepdims=True)).sum(1))
    lse, tz, ti = m.test_gen(h, k)
    tol = 1e-5 if which == "bf16" else 2e-6
    np.testing.assert_allclose(lse, lse_ref, atol=tol)
    for r in range(R):
        order = np.lexsort((np.arange(z.shape[1]), -z[r]))[:k]
        # ids must agree except inside near-ties; z values must agree everywhere
        np.testing.assert_allclose(tz[r], z[r, order], atol=tol)
        for i in range(k):
            if ti[r, i] != order[i]:
                assert abs(z[r, ti[r, i]] - z[r, order[i]]) < 2 * tol
