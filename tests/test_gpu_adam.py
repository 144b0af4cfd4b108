"""SURVEY §8(f) row f1 on the GPU: vks_adam_step (through the C ABI) vs the oracle's fp64 Adam
(SPEC S:252-259), element by element.

Both sides take the hyperparameters the kernel receives (fp32 values: the oracle is fed the
fp32-rounded betas, eps and learning rates).  Tolerance: the kernel computes in
fp32 with IEEE division and square root, the oracle in fp64 rounded once; each moment is a sum of
two rounded products, so |m - m_ref| <= 2^-22 (|b1 m0| + |(1 - b1) g|) (likewise v); the update
u = lr m_hat / (sqrt(v_hat) + eps) inherits that error through m_hat plus a few roundings, so
|p - p_ref| <= 2^-23 |p_ref| + 4e-6 lr (|b1 m0| + |(1 - b1) g|) / (1 - b1^t) / (sqrt(v_hat) + eps);
re-normalised quaternions to 1e-6 absolute."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

f32 = lambda x: float(np.float32(x))  # noqa: E731
LR = dict(means=1.6e-4, log_scales=5e-3, quats=1e-3, opacity_logits=5e-2, sh=(2.5e-3, 1.25e-4))
LR32 = {k: (tuple(f32(x) for x in v) if isinstance(v, tuple) else f32(v)) for k, v in LR.items()}
B1, B2, EPS = f32(0.9), f32(0.999), f32(1e-8)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _state(n, K, seed):
    rng = np.random.default_rng(seed)
    shapes = dict(means=(n, 3), log_scales=(n, 3), quats=(n, 4), opacity_logits=(n,), sh=(n, K, 3))
    p = {k: rng.normal(0, 1, s).astype(np.float32) for k, s in shapes.items()}
    p["quats"] /= np.linalg.norm(p["quats"], axis=1, keepdims=True)
    # gradients over several decades, moments of an earlier step
    g = {k: (rng.normal(0, 1, s) * 10.0 ** rng.uniform(-6, 0, s)).astype(np.float32) for k, s in shapes.items()}
    m = {k: (rng.normal(0, 1e-3, s)).astype(np.float32) for k, s in shapes.items()}
    v = {k: (np.abs(rng.normal(0, 1e-6, s))).astype(np.float32) for k, s in shapes.items()}
    return p, g, m, v


def _gpu_step(p, g, m, v, lr, step, zero_m=False):
    import torch
    import paper_2605_00219_b200 as P
    G = oracle.ADAM_GROUPS
    tp = [torch.from_numpy(p[k].copy()).cuda() for k in G]
    tg = [torch.from_numpy(g[k].copy()).cuda() for k in G]
    tm = [torch.from_numpy(m[k].copy()).cuda() for k in G]
    tv = [torch.from_numpy(v[k].copy()).cuda() for k in G]
    P.vks_adam_step(P.make_adam_config(lr, step=step), tp, tg, tm, tv)
    torch.cuda.synchronize()
    return ({k: t.cpu().numpy() for k, t in zip(G, tp)}, {k: t.cpu().numpy() for k, t in zip(G, tm)},
            {k: t.cpu().numpy() for k, t in zip(G, tv)})


@pytest.mark.parametrize("n,K,step", [(1, 16, 1), (1001, 16, 7), (4099, 9, 300), (2, 1, 2)])
def test_adam_matches_oracle(n, K, step):
    """Ragged group sizes (3n, n and 3Kn not multiples of 4: the kernel's scalar tails) and SH
    widths 16 / 9 / 1, the SH coefficient-0 / rest learning-rate split, steps 1 to 300."""
    p, g, m, v = _state(n, K, seed=n + K + step)
    Pg, Mg, Vg = _gpu_step(p, g, m, v, LR, step)
    Po, Mo, Vo = oracle.adam_step(p, g, m, v, LR32, beta1=B1, beta2=B2, eps=EPS, step=step)
    bc1, bc2 = 1.0 - B1 ** step, 1.0 - B2 ** step
    for k in oracle.ADAM_GROUPS:
        g64, m0, v0 = (a.astype(np.float64) for a in (g[k], m[k], v[k]))
        m_mass = np.abs(B1 * m0) + np.abs((1.0 - B1) * g64)
        v_mass = B2 * v0 + (1.0 - B2) * g64 * g64
        assert np.all(np.abs(Mg[k] - Mo[k].astype(np.float64)) <= 2.0 ** -22 * m_mass + 1e-38), k
        assert np.all(np.abs(Vg[k] - Vo[k].astype(np.float64)) <= 2.0 ** -22 * v_mass + 1e-38), k
        if k == "quats":
            assert np.all(np.abs(Pg[k].astype(np.float64) - Po[k]) <= 1e-6), k
            continue
        lr = LR32[k]
        if k == "sh":
            lr = np.where((np.arange(g64.size).reshape(g64.shape) // 3) % K == 0, LR32["sh"][0], LR32["sh"][1])
        vhat = Vo[k].astype(np.float64) / bc2
        u_mass = lr * m_mass / bc1 / (np.sqrt(vhat) + EPS)
        tol = 2.0 ** -23 * np.abs(Po[k].astype(np.float64)) + 4e-6 * u_mass + 1e-38
        bad = np.abs(Pg[k].astype(np.float64) - Po[k]) > tol
        assert not bad.any(), (k, int(bad.sum()), np.argwhere(bad)[:4].tolist())


def test_adam_zero_gradients_and_spec_example():
    """zero gradients from zero moments leave the parameters bit-identical (quaternions to
    one rounding); g = 1, lr = 0.1 from zero moments moves a parameter by -0.1/(1+1e-8)."""
    n, K = 37, 16
    p, _, _, _ = _state(n, K, seed=5)
    z = {k: np.zeros_like(a) for k, a in p.items()}
    Pg, Mg, Vg = _gpu_step(p, z, z, z, LR, 3)
    for k in oracle.ADAM_GROUPS:
        if k == "quats":
            assert np.allclose(Pg[k], p[k], atol=2e-7, rtol=0)
        else:
            assert np.array_equal(Pg[k], p[k]), k
        assert not Mg[k].any() and not Vg[k].any()
    ones = {k: np.ones_like(a) for k, a in p.items()}
    zp = {k: np.zeros_like(a) for k, a in p.items()}
    lr = dict(means=0.1, log_scales=0.1, quats=0.1, opacity_logits=0.1, sh=(0.1, 0.1))
    Pg, Mg, Vg = _gpu_step(zp, ones, z, z, lr, 1)
    assert np.all(Pg["means"] == np.float32(-0.1 / (1 + 1e-8)))
    # the moments hold (1 - beta) g with the config's fp32 betas; the bias correction divides
    # the same (1 - beta) back out, so the update is exactly the worked example's
    assert np.all(Mg["means"] == np.float32(1) - np.float32(0.9))
    assert np.all(Vg["means"] == np.float32(1) - np.float32(0.999))


def test_adam_late_step():
    """t = 10^4: the bias corrections are ~1 (1 - b1^t underflows to 1); same bounds."""
    n, K, step = 3001, 16, 10000
    p, g, m, v = _state(n, K, seed=99)
    Pg, Mg, Vg = _gpu_step(p, g, m, v, LR, step)
    Po, Mo, Vo = oracle.adam_step(p, g, m, v, LR32, beta1=B1, beta2=B2, eps=EPS, step=step)
    for k in oracle.ADAM_GROUPS:
        if k == "quats":
            assert np.all(np.abs(Pg[k].astype(np.float64) - Po[k]) <= 1e-6)
            continue
        d = np.abs(Pg[k].astype(np.float64) - Po[k])
        upd = np.abs(p[k].astype(np.float64) - Po[k])
        assert np.all(d <= 2.0 ** -23 * np.abs(Po[k]) + 4e-6 * np.maximum(upd, 1e-3 * LR32["means"])), k
