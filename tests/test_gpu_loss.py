"""SURVEY §8(f) row f2 on the GPU: vks_loss_grad (through the C ABI) vs the oracle's fp64 loss
gradient, element by element.

Tolerance: the kernels sum the windows and form the SSIM partials in fp64 from
the same fp32 pixels, so the per-pixel gradient differs from the oracle's only by summation
order and the final fp32 rounding: with G = 3 H W dL (an O(1) quantity),
|G - G_ref| <= 1e-6 |G_ref| + 1e-9; the loss within 1e-6 relative (fp32 output)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _pair(H, W, seed, noise=0.1):
    rng = np.random.default_rng(seed)
    t = rng.random((H, W, 3)).astype(np.float32)
    r = np.clip(t + rng.normal(0, noise, t.shape), 0, 1).astype(np.float32)
    r[: H // 3, : W // 4] = t[: H // 3, : W // 4]  # a region where render == target (sign(0) = 0)
    return r, t


def _gpu(r, t, lam):
    import torch
    import paper_2605_00219_b200 as P
    H, W = r.shape[:2]
    rr, tt = torch.from_numpy(r).cuda(), torch.from_numpy(t).cuda()
    dL = torch.empty_like(rr)
    loss = torch.empty(1, device="cuda")
    ws = torch.empty(P.vks_loss_workspace_bytes(W, H), dtype=torch.uint8, device="cuda")
    P.vks_loss_grad(rr, tt, dL, loss, ws, lam=lam)
    torch.cuda.synchronize()
    return float(loss.item()), dL.cpu().numpy()


@pytest.mark.parametrize("H,W,lam", [(11, 11, 0.2), (48, 64, 0.2), (150, 200, 0.2), (37, 53, 0.0),
                                     (822, 1237, 0.2)])
def test_loss_grad_matches_oracle(H, W, lam):
    """Single window (11x11), several tiles with ragged edges (150x200, 37x53), pure L1 (lambda 0)
    and the bicycle resolution 1237x822 (the size bench.py's e2e leg runs)."""
    r, t = _pair(H, W, seed=H * W)
    loss, g = _gpu(r, t, lam)
    lo, go, _ = oracle.loss_grad(r, t, lam)
    assert loss == pytest.approx(lo, rel=1e-6, abs=1e-9)
    G, Go = g.astype(np.float64) * 3 * H * W, go * 3 * H * W
    err = np.abs(G - Go)
    bad = err > 1e-6 * np.abs(Go) + 1e-9
    assert not bad.any(), (int(bad.sum()), np.argwhere(bad)[:4].tolist(), float(err.max()))


def test_identical_images_zero_gradient():
    """render == target gives loss 0 and gradient 0 (SSIM = 1 exactly: every partial pair
    cancels in fp64 up to rounding)."""
    _, t = _pair(40, 30, 2)
    loss, g = _gpu(t, t, 0.2)
    assert abs(loss) <= 1e-7 and np.abs(g).max() * 3 * 40 * 30 <= 1e-9


@pytest.mark.parametrize("H,W,lam", [(11, 40, 1.0), (40, 11, 0.5), (33, 70, 1.0)])
def test_loss_grad_pure_ssim_and_thin_images(H, W, lam):
    """lambda = 1 (pure D-SSIM) and images one window thick in one dimension."""
    r, t = _pair(H, W, seed=7 * H + W)
    loss, g = _gpu(r, t, lam)
    lo, go, _ = oracle.loss_grad(r, t, lam)
    assert loss == pytest.approx(lo, rel=1e-6, abs=1e-9)
    G, Go = g.astype(np.float64) * 3 * H * W, go * 3 * H * W
    assert np.all(np.abs(G - Go) <= 1e-6 * np.abs(Go) + 1e-9)


@pytest.mark.parametrize("H,W", [(42, 42), (43, 75), (74, 74), (75, 106), (12, 300)])
def test_loss_grad_tile_seams(H, W):
    """Centre-tile seams of the fused kernel (32x32 centre tiles, each reaching a 42x42 pixel
    region; a pixel gets the partials of 1, 2 or 4 tiles): one tile exactly (42x42), a ragged
    second tile (43x75), 2x2 tiles whose regions overlap by 10 pixels (74x74: Wv = 64) and one past
    it (75x106), and a strip two centres high (12x300)."""
    r, t = _pair(H, W, seed=11 * H + W)
    loss, g = _gpu(r, t, 0.2)
    lo, go, _ = oracle.loss_grad(r, t, 0.2)
    assert loss == pytest.approx(lo, rel=1e-6, abs=1e-9)
    G, Go = g.astype(np.float64) * 3 * H * W, go * 3 * H * W
    err = np.abs(G - Go)
    bad = err > 1e-6 * np.abs(Go) + 1e-9
    assert not bad.any(), (int(bad.sum()), np.argwhere(bad)[:4].tolist(), float(err.max()))
