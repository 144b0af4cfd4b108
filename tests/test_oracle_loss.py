"""Pins of the oracle's loss gradient:
loss = (1 - lambda) mean|r - t| + lambda (1 - SSIM), SSIM over valid 11x11 Gaussian windows."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _pair(H, W, seed, noise=0.1):
    rng = np.random.default_rng(seed)
    t = rng.random((H, W, 3)).astype(np.float32)
    r = np.clip(t + rng.normal(0, noise, t.shape), 0, 1).astype(np.float32)
    return r, t


def test_identical_images():
    """render == target -> loss 0 and gradient 0 (lambda = 0 and 0.2; SSIM(a, a) = 1)."""
    _, t = _pair(20, 17, 1)
    for lam in (0.0, 0.2):
        loss, g, ss = oracle.loss_grad(t, t, lam)
        assert abs(loss) <= 1e-15 and ss == pytest.approx(1.0, abs=1e-15)
        assert np.abs(g).max() <= 1e-15


def test_l1_spec_example():
    """lambda = 0, one channel differs by +0.5 -> loss 0.5/(3N), gradient 1/(3N) there."""
    G = GOLD["loss_l1_one_channel"]
    H, W = 8, 6
    t = np.full((H, W, 3), 0.25, np.float32)
    r = t.copy()
    r[3, 2, 1] += G["diff"]
    loss, g, _ = oracle.loss_grad(r, t, 0.0)
    N = H * W
    assert loss * 3 * N == pytest.approx(G["loss_times_3N"], rel=1e-12)
    assert g[3, 2, 1] * 3 * N == pytest.approx(G["grad_times_3N"], rel=1e-12)
    g[3, 2, 1] = 0
    assert not g.any()


def test_ssim_matches_scipy_gaussian_filter():
    """S:482 / S:487: the oracle's SSIM equals an independent implementation (scipy.ndimage
    gaussian_filter with sigma 1.5 truncated at radius 5, valid centres only) and is symmetric."""
    from scipy.ndimage import gaussian_filter
    for seed in range(3):
        r, t = _pair(31, 40, seed)
        _, _, ss = oracle.loss_grad(r, t, 0.2)
        _, _, ss2 = oracle.loss_grad(t, r, 0.2)
        x, y = r.astype(np.float64), t.astype(np.float64)
        f = lambda a: gaussian_filter(a, sigma=1.5, truncate=5 / 1.5, axes=(0, 1), mode="constant")  # noqa: E731
        mx, my = f(x), f(y)
        sx2, sy2, sxy = f(x * x) - mx * mx, f(y * y) - my * my, f(x * y) - mx * my
        C1, C2 = GOLD["ssim_definition"]["C1"], GOLD["ssim_definition"]["C2"]
        S = (2 * mx * my + C1) * (2 * sxy + C2) / ((mx * mx + my * my + C1) * (sx2 + sy2 + C2))
        ref = S[5:-5, 5:-5].mean()
        assert ss == pytest.approx(ref, abs=1e-12)
        assert ss == pytest.approx(ss2, abs=1e-12)


def test_gradient_matches_central_differences():
    """lambda = 0.2, random 16x16 pair: the analytic gradient matches central finite
    differences within 1e-4 relative (fp64 loss; perturbations taken as the fp32-representable
    steps, on channels away from the L1 kink)."""
    r, t = _pair(16, 16, 7, noise=0.2)
    loss, g, _ = oracle.loss_grad(r, t, 0.2)
    rng = np.random.default_rng(3)
    checked = 0
    for _ in range(200):
        i, j, c = rng.integers(16), rng.integers(16), rng.integers(3)
        h = 1e-3
        if abs(float(r[i, j, c]) - float(t[i, j, c])) < 4 * h:
            continue
        rp, rm = r.copy(), r.copy()
        rp[i, j, c] = np.float32(r[i, j, c] + h)
        rm[i, j, c] = np.float32(r[i, j, c] - h)
        d = float(rp[i, j, c]) - float(rm[i, j, c])
        fd = (oracle.loss_grad(rp, t, 0.2)[0] - oracle.loss_grad(rm, t, 0.2)[0]) / d
        assert fd == pytest.approx(g[i, j, c], rel=1e-4, abs=1e-9), (i, j, c)
        checked += 1
    assert checked > 100
