"""Trainer.  No reference
trainer code exists, so the SPEC's properties pin it: finite-difference
gradients, lr = 0 identity, zero-loss fixed point, L2 shrinkage, determinism,
selection rules; a trained (non-Lorenzo) model must round-trip bit-exactly
against the oracle through the general predictor path of the kernels."""
import numpy as np
import pytest

from paper_2309_09778_b200 import training as T
from paper_2309_09778_b200.errors import ConfigError, SweepExhausted
from paper_2309_09778_b200.predictor import PerceptronModel, init_model


def _rep(cr, err):
    return T.ValidationReport(cr, err, 0.99, 10)


def test_select_best_rules():
    hc = [T.HyperConfig(1e-3, 0.0), T.HyperConfig(1e-4, 0.0), T.HyperConfig(1e-3, 1e-2), T.HyperConfig(1e-4, 1e-4)]
    res = [(hc[0], "a", _rep(0.25, 1e-2), None), (hc[1], "b", _rep(0.20, 1e-2), None),
           (hc[2], "c", _rep(0.10, 9e-2), None), (hc[3], "d", None, RuntimeError())]
    assert T.select_best(res, 1e-2).model == "b"            # argmin CR within the bound
    tie = [(hc[2], "x", _rep(0.2, 0.0), None), (hc[0], "y", _rep(0.2, 0.0), None), (hc[1], "z", _rep(0.2, 0.0), None)]
    assert T.select_best(tie, 1e-2).model == "z"             # smaller l2, then smaller lr
    with pytest.raises(SweepExhausted):
        T.select_best([(hc[2], "c", _rep(0.1, 1.0), None)], 1e-2)


def test_grid_and_config_validation():
    assert len(T.default_grid()) == 6
    assert T.parse_grid("lr:1e-3;l2:0,1e-2") == [T.HyperConfig(1e-3, 0.0), T.HyperConfig(1e-3, 1e-2)]
    with pytest.raises(ConfigError):
        T.HyperConfig(0.0, 0.0)
    with pytest.raises(ConfigError):
        T.HyperConfig(1e-3, -1.0)


def _batch(rng, n):
    import torch
    s = rng.normal(0, 3, (n, 3))
    t = rng.normal(0, 3, n)
    return T.TrainBatch(torch.tensor(s, device="cuda"), torch.tensor(t, device="cuda"))


def _lorenzo(s):
    h = s[:, 0] + s[:, 1] - s[:, 2]
    return np.where(h < 0, 0.01 * h, h)


@pytest.mark.gpu
def test_gradient_vs_finite_differences():
    rng = np.random.default_rng(0)
    for trial in range(5):
        m = PerceptronModel(rng.normal(0, 1, (4, 2)), rng.normal(0, 1, 2))
        b = _batch(rng, 4000)
        sums = T.batch_sums(m, b)
        grad = np.concatenate([sums[:8], sums[8:10]])
        w = T._weights(m)
        h = 1e-6
        for i in range(10):
            wp, wm = w.copy(), w.copy()
            wp[i] += h
            wm[i] -= h
            lp = T.batch_sums(PerceptronModel(wp[:8], wp[8:]), b)[10]
            lm = T.batch_sums(PerceptronModel(wm[:8], wm[8:]), b)[10]
            fd = (lp - lm) / (2 * h)
            assert abs(fd - grad[i]) <= 1e-5 * max(1.0, abs(grad[i])), (trial, i, fd, grad[i])


@pytest.mark.gpu
def test_step_identities_and_shrinkage():
    import torch
    rng = np.random.default_rng(1)
    m0 = init_model(3)
    b = _batch(rng, 2000)
    m1, _ = T.train_step(m0, b, 0.0, 0.0)                       # lr = 0: unchanged
    assert np.array_equal(T._weights(m1), T._weights(m0))
    # integer surfaces: init-model predictions are exact, so the loss is 0
    s = rng.integers(-50, 50, (3000, 3)).astype(np.float64)
    zb = T.TrainBatch(torch.tensor(s, device="cuda"), torch.tensor(_lorenzo(s), device="cuda"))
    m2, loss = T.train_step(m0, zb, 1e-3, 0.0)                  # zero-gradient fixed point
    assert loss == 0.0 and np.array_equal(T._weights(m2), T._weights(m0))
    m3, _ = T.train_step(m0, zb, 1e-3, 1e-2)                    # L2 shrinkage
    w0, w3 = T._weights(m0), T._weights(m3)
    nz = w0 != 0
    assert np.all(np.abs(w3[nz]) < np.abs(w0[nz])) and np.all(w3[~nz] == 0)
    a1, a2 = T.batch_sums(m0, b), T.batch_sums(m0, b)           # determinism
    assert np.array_equal(a1, a2)


@pytest.mark.gpu
def test_sweep_select_and_trained_model_parity(oracle):
    import torch
    import paper_2309_09778_b200 as P
    from paper_2309_09778_b200 import synthetic
    x = synthetic.generate("C2", shape=(600, 800)).numpy()
    codec = P.Codec("cuda:0")
    cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.5)
    xd = torch.from_numpy(x).cuda()
    res = T.sweep(codec, xd, cfg)
    assert len(res) == 6 and all(r is not None for _, _, r, _ in res)
    res2 = T.sweep(codec, xd, cfg)                               # reproducible sweep
    assert [T._weights(mm).tolist() for _, mm, _, _ in res] == [T._weights(mm).tolist() for _, mm, _, _ in res2]
    out = T.select_best(res, 1e-2)
    assert out.report.max_rel_error <= 1.5e-2 and 0 < out.report.compression_ratio
    # the chosen (non-Lorenzo) weights through the general predictor: bit-exact vs the oracle
    mdl = out.model
    assert not np.array_equal(T._weights(mdl), T._weights(init_model(3)))
    buf, info = codec.compress_device(xd, P.CompressConfig(rel_error=1e-2, repair_factor=1.5, model=mdl))
    ref, _ = oracle.compress(x, oracle.OracleConfig(b_r=1e-2, repair_factor=1.5, w1=mdl.w1, w2=mdl.w2))
    assert buf.cpu().numpy().tobytes() == ref
    y = P.decompress(ref, device="cuda:0")
    assert np.array_equal(y.view(np.uint32), oracle.decompress(ref).view(np.uint32))
