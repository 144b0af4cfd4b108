"""Pins of the oracle's default densification (
readings R6-R9 of DESIGN.md §4.7): screen-gradient statistics, clone / split / prune."""
import numpy as np
import pytest

import oracle
import synth


def _scene(n, seed):
    s = synth.make_scene(n, "outdoor", seed)
    s["opacity_logits"] = np.maximum(s["opacity_logits"], -3.0).astype(np.float32)  # nobody prunable
    return s


def test_stats_accumulate_visible_norms():
    """R6: |dL/dmean2d| is added, and the view counted, only where the view rasterised the Gaussian."""
    rng = np.random.default_rng(0)
    g = rng.normal(size=(100, 2)).astype(np.float32)
    radii = np.where(rng.random((100, 1)) < 0.5, 3, 0).repeat(2, 1).astype(np.int32)
    a, d = oracle.densify_stats(g, radii, np.zeros(100, np.float32), np.zeros(100, np.float32))
    vis = radii[:, 0] > 0
    assert np.allclose(a[vis], np.hypot(g[vis, 0], g[vis, 1]), rtol=1e-6) and not a[~vis].any()
    assert np.array_equal(d, vis.astype(np.float32))


def test_nothing_over_threshold_is_identity():
    """no Gaussian over the gradient threshold and none under the prune opacity -> unchanged."""
    s = _scene(500, 1)
    acc, den = np.full(500, 1e-5, np.float32), np.ones(500, np.float32)
    out, n2, _, _ = oracle.densify(s, acc, den, 2e-4, 0.01)
    assert n2 == 500
    for k in out:
        assert np.array_equal(out[k], s[k]), k


def test_clone_split_prune():
    """one small high-gradient Gaussian -> count + 1, the copy shares every parameter and has
    zero moments; a large one splits into two children with log-scales - ln 1.6 replacing it; a
    low-opacity one is removed (only sub-threshold opacities are pruned)."""
    s = _scene(10, 2)
    n, K = 10, s["sh"].shape[1]
    F = 11 + 3 * K
    s["log_scales"][:] = np.log(0.001)
    s["log_scales"][5] = np.log(0.05)               # large -> split
    s["opacity_logits"][7] = -7.0                   # rho ~ 9e-4 -> pruned
    acc, den = np.full(n, 1e-5, np.float32), np.ones(n, np.float32)
    acc[[2, 5]] = 1e-3                              # over the threshold
    m = np.arange(n * F, dtype=np.float32) + 1.0
    out, n2, om, ov = oracle.densify(s, acc, den, 2e-4, 0.01, m=m, v=m.copy(), seed=4)
    assert n2 == n + 1 + 1 - 1
    # emitted order: 0 1 2 2' 3 4 5a 5b 6 8 9
    src = [0, 1, 2, 2, 3, 4, 5, 5, 6, 8, 9]
    for o, i in enumerate(src):
        for k in ("quats", "opacity_logits", "sh"):
            assert np.array_equal(out[k][o], s[k][i]), (o, k)
    assert np.array_equal(out["means"][3], s["means"][2]) and np.array_equal(out["log_scales"][3], s["log_scales"][2])
    for o in (6, 7):
        assert np.allclose(out["log_scales"][o], s["log_scales"][5] - np.log(1.6), atol=1e-6)
        assert not np.array_equal(out["means"][o], s["means"][5])
    offs_in = np.cumsum([0, 3 * n, 3 * n, 4 * n, n])
    offs_out = np.cumsum([0, 3 * n2, 3 * n2, 4 * n2, n2])
    wid = [3, 3, 4, 1, 3 * K]
    for o, i in enumerate(src):
        fresh = o in (3, 6, 7)
        for oi, oo, w in zip(offs_in, offs_out, wid):
            got = om[oo + w * o: oo + w * (o + 1)]
            assert (not got.any()) if fresh else np.array_equal(got, m[oi + w * i: oi + w * (i + 1)]), (o, i)


def test_split_children_sample_the_parent():
    """R8: the children's offsets from the parent mean are Rq diag(s) eps: over 20000 split parents
    their covariance is R diag(s^2) R^T and their mean 0 (sampling error)."""
    n = 10000
    q = np.float32([0.8, -0.2, 0.4, 0.1])
    q /= np.linalg.norm(q)
    s = dict(means=np.zeros((n, 3), np.float32), log_scales=np.tile(np.log(np.float32([0.5, 1.0, 2.0])), (n, 1)),
             quats=np.tile(q, (n, 1)), opacity_logits=np.zeros(n, np.float32), sh=np.zeros((n, 1, 3), np.float32))
    out, n2, _, _ = oracle.densify(s, np.ones(n, np.float32), np.ones(n, np.float32), 0.5, 0.1, seed=8)
    assert n2 == 2 * n
    d = out["means"].astype(np.float64)
    w, x, y, z = q.astype(np.float64)
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    assert np.allclose(np.cov(d.T), R @ np.diag([0.25, 1.0, 4.0]) @ R.T, atol=0.15)
    assert np.abs(d.mean(0)).max() < 0.05


def test_capacity_reports_the_new_count():
    """R9: when n' exceeds the output capacity nothing is written and n' is returned (the caller
    grows its buffers, x1.5 by default, and repeats)."""
    s = _scene(100, 3)
    out, n2, _, _ = oracle.densify(s, np.ones(100, np.float32), np.ones(100, np.float32), 0.5, 10.0, cap=150)
    assert out is None and n2 == 200
