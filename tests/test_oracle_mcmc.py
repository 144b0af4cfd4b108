"""Pins of the oracle's MCMC densification (readings R1-R5 of
DESIGN.md §4.7): fixed budget, relocation targets drawn in proportion to opacity, appearance-
conserving opacity split, gated positional noise."""
import numpy as np
import pytest

import oracle
import synth


def _scene(n, seed, dead_frac=0.2):
    s = synth.make_scene(n, "indoor", seed)
    rng = np.random.default_rng(seed)
    dead = rng.random(n) < dead_frac
    s["opacity_logits"][dead] = -8.0  # rho ~ 3e-4 < 0.005
    return s, dead


def test_rng_is_uniform_and_counter_based():
    """R1/R2: the generator is a pure function of (seed, stream, counter); its 24-bit uniforms have
    mean 1/2 and variance 1/12 over 2^16 counters, and streams / seeds are decorrelated."""
    a = np.array([oracle.rng(7, 1, i) >> 40 for i in range(1 << 16)], np.float64) / 2**24
    assert abs(a.mean() - 0.5) < 0.005 and abs(a.var() - 1 / 12) < 0.002
    assert oracle.rng(7, 1, 123) == oracle.rng(7, 1, 123) != oracle.rng(7, 2, 123) != oracle.rng(8, 1, 123)
    b = np.array([oracle.rng(7, 2, i) >> 40 for i in range(1 << 16)], np.float64) / 2**24
    assert abs(np.corrcoef(a, b)[0, 1]) < 0.02


def test_budget_and_no_dead_identity():
    """the count is the budget before and after; with no dead Gaussians and noise scale 0
    nothing moves."""
    s, _ = _scene(2000, 1, dead_frac=0.0)
    s["opacity_logits"] = np.maximum(s["opacity_logits"], -4.0)  # rho > 0.017: nobody dead
    out, tg, dead, _, _ = oracle.mcmc_relocate(s, seed=3)
    assert dead == 0 and (tg == -1).all()
    for k in out:
        assert out[k].shape == s[k].shape and np.array_equal(out[k], s[k])
    assert np.array_equal(oracle.mcmc_noise(s, 1e-3, 0.0, seed=3), s["means"])


def test_relocation_frequencies_follow_opacity():
    """over 10^5 draws the target frequencies match the opacity distribution (chi-square
    against the exact probabilities w_j / sum w, and every frequency within 1% absolute)."""
    n_alive, n_dead = 50, 100000
    rng = np.random.default_rng(0)
    rho = rng.uniform(0.02, 0.99, n_alive)
    s = dict(means=np.zeros((n_alive + n_dead, 3), np.float32), log_scales=np.zeros((n_alive + n_dead, 3), np.float32),
             quats=np.tile(np.float32([1, 0, 0, 0]), (n_alive + n_dead, 1)),
             opacity_logits=np.concatenate([np.log(rho / (1 - rho)), np.full(n_dead, -9.0)]).astype(np.float32),
             sh=np.zeros((n_alive + n_dead, 1, 3), np.float32))
    _, tg, dead, _, _ = oracle.mcmc_relocate(s, seed=11)
    assert dead == n_dead and tg[:n_alive].max() == -1 and tg[n_alive:].min() >= 0 and tg.max() < n_alive
    r32 = (1 / (1 + np.exp(-s["opacity_logits"][:n_alive].astype(np.float64)))).astype(np.float32)
    w = np.floor(r32.astype(np.float64) * 2**24)
    p = w / w.sum()
    f = np.bincount(tg[n_alive:], minlength=n_alive) / n_dead
    chi2 = n_dead * ((f - p) ** 2 / p).sum()
    assert chi2 < 100.0  # 49 degrees of freedom: P(chi2 > 100) ~ 2e-5
    assert np.abs(f - p).max() < 0.01


def test_relocated_copies_conserve_appearance():
    """R4: a target j chosen k times ends with its k copies at opacity rho' with
    (1 - rho')^(k+1) = 1 - rho_j, and the copies carry j's other parameters and zero moments."""
    s, dead = _scene(3000, 2)
    n, K = 3000, s["sh"].shape[1]
    F = 11 + 3 * K
    m = np.random.default_rng(1).random(n * F).astype(np.float32)
    out, tg, nd, mo, vo = oracle.mcmc_relocate(s, seed=5, m=m, v=m.copy())
    rho = 1 / (1 + np.exp(-s["opacity_logits"].astype(np.float64)))
    assert nd == (rho.astype(np.float32) < np.float32(0.005)).sum() >= dead.sum()
    rho2 = 1 / (1 + np.exp(-out["opacity_logits"].astype(np.float64)))
    k = np.bincount(tg[tg >= 0], minlength=n)
    for j in np.nonzero(k)[0][:200]:
        assert (1 - rho2[j]) ** (k[j] + 1) == pytest.approx(1 - rho[j], rel=1e-5)
        for i in np.nonzero(tg == j)[0]:
            assert rho2[i] == rho2[j]
            for key in ("means", "log_scales", "quats", "sh"):
                assert np.array_equal(out[key][i], s[key][j])
    i = np.nonzero(tg >= 0)[0][0]
    offs = [0, 3 * n, 6 * n, 10 * n, 11 * n]
    wid = [3, 3, 4, 1, 3 * K]
    for o, wdt in zip(offs, wid):
        assert not mo[o + wdt * i: o + wdt * (i + 1)].any()
    u = np.nonzero(tg < 0)[0][0]  # an untouched row keeps its moments
    for o, wdt in zip(offs, wid):
        assert np.array_equal(mo[o + wdt * u: o + wdt * (u + 1)], m[o + wdt * u: o + wdt * (u + 1)])


def test_noise_gate_and_covariance():
    """R5: the displacement is lr * scale * gate(rho) * Rq diag(s) eps: the sample covariance of
    20000 identical Gaussians matches (lr * scale * gate)^2 R diag(s^2) R^T within sampling error
    (gate(rho ~ 6e-6) = sigmoid(100 (0.005 - rho)) ~ 0.62); for rho >> 0.005 the gate closes
    (|displacement| < 1e-12)."""
    n = 20000
    q = np.float32([0.9, 0.1, -0.3, 0.2])
    q /= np.linalg.norm(q)
    s = dict(means=np.zeros((n, 3), np.float32), log_scales=np.tile(np.log(np.float32([0.5, 1.0, 2.0])), (n, 1)),
             quats=np.tile(q, (n, 1)), opacity_logits=np.full(n, -12.0, np.float32), sh=np.zeros((n, 1, 3), np.float32))
    rho = 1 / (1 + np.exp(12.0))
    gate = 1 / (1 + np.exp(-100 * (0.005 - rho)))
    d = oracle.mcmc_noise(s, 0.01, 10.0, seed=4, step=3).astype(np.float64) / (0.1 * gate)
    w, x, y, z = q.astype(np.float64)
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    cov = R @ np.diag([0.25, 1.0, 4.0]) @ R.T
    assert np.allclose(np.cov(d.T), cov, atol=0.08 * 4)
    assert np.abs(d.mean(0)).max() < 0.05
    s["opacity_logits"][:] = 2.0
    assert np.abs(oracle.mcmc_noise(s, 0.01, 10.0, seed=4, step=3)).max() < 1e-12
