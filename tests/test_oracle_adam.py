"""Pins of the oracle's optimizer step: Adam with
bias correction per parameter group, quaternions re-normalised after the step.  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))["adam_one_step"]


def _groups(n, K, rng, zero=False):
    shapes = dict(means=(n, 3), log_scales=(n, 3), quats=(n, 4), opacity_logits=(n,), sh=(n, K, 3))
    f = (lambda s: np.zeros(s, np.float32)) if zero else (lambda s: rng.normal(0, 1, s).astype(np.float32))
    return {k: f(s) for k, s in shapes.items()}


def _one(p, g, m, v, lr, b1, b2, eps, t):
    import ctypes as C
    L = oracle.lib()
    L.vko_adam_group.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                 C.c_double, C.c_double, C.c_double, C.c_int32]
    arrs = [np.array(x, np.float32).reshape(-1) for x in (p, m, v, g)]
    L.vko_adam_group(arrs[0].size, *(a.ctypes.data_as(C.c_void_p) for a in arrs), lr, b1, b2, eps, t)
    return arrs[0], arrs[1], arrs[2]


def test_spec_worked_example():
    """g = 1 from m = v = 0 at t = 1 gives the update -lr / (1 + eps) (bias corrections
    make m_hat = 1, v_hat = 1)."""
    G = GOLD
    p, m, v = _one([0.0], [G["g"]], [0.0], [0.0], G["lr"], G["beta1"], G["beta2"], G["eps"], G["step"])
    assert p[0] == np.float32(G["update"])
    assert m[0] == np.float32(G["m"]) and v[0] == np.float32(G["v"])


def test_zero_gradient_identity():
    """S:258 / S:283: zero gradients from zero moments leave the parameters unchanged; quaternions
    that are already unit stay unit (up to one rounding)."""
    rng = np.random.default_rng(0)
    n, K = 257, 16
    params = _groups(n, K, rng)
    params["quats"] /= np.linalg.norm(params["quats"], axis=1, keepdims=True)
    z = _groups(n, K, rng, zero=True)
    lr = dict(means=1e-3, log_scales=5e-3, quats=1e-3, opacity_logits=5e-2, sh=(2.5e-3, 1.25e-4))
    P, M, V = oracle.adam_step(params, z, z, z, lr, step=5)
    for k in oracle.ADAM_GROUPS:
        if k == "quats":
            assert np.allclose(P[k], params[k], atol=2e-7, rtol=0)
        else:
            assert np.array_equal(P[k], params[k]), k
        assert not M[k].any() and not V[k].any()


@pytest.mark.parametrize("g", [0.3, -2.5, 1e-4])
def test_constant_gradient_closed_form(g):
    """With a constant gradient g from m = v = 0, the bias corrections give m_hat = g and
    v_hat = g^2 exactly at every step, so p_t = p_0 - t lr g / (|g| + eps).  A missing bias
    correction, swapped betas or a wrong sign breaks it at t = 1 or t > 1."""
    lr, b1, b2, eps = 0.01, 0.9, 0.999, 1e-8
    p, m, v = np.array([0.5], np.float32), np.zeros(1, np.float32), np.zeros(1, np.float32)
    p64 = 0.5
    for t in range(1, 8):
        p, m, v = _one(p, [g], m, v, lr, b1, b2, eps, t)
        p64 -= lr * g / (abs(g) + eps)
        assert abs(float(p[0]) - p64) <= 1e-6 * t, (t, float(p[0]), p64)
        assert abs(float(m[0]) - (1 - b1 ** t) * g) <= 1e-6 * abs(g)
        assert abs(float(v[0]) - (1 - b2 ** t) * g * g) <= 1e-6 * g * g


def test_x_squared_decreases():
    """100 Adam steps on f(x) = x^2 from x = 1 strictly decrease f."""
    x, m, v = np.array([1.0], np.float32), np.zeros(1, np.float32), np.zeros(1, np.float32)
    f = [1.0]
    for t in range(1, 101):
        x, m, v = _one(x, [2.0 * float(x[0])], m, v, 0.01, 0.9, 0.999, 1e-8, t)
        f.append(float(x[0]) ** 2)
    assert all(b < a for a, b in zip(f, f[1:]))


def test_quaternions_renormalised_and_sh_lr_split():
    """rotations re-normalised after the step; the SH group's coefficient 0 and the
    others take their own learning rates (a lr of 0 freezes them)."""
    rng = np.random.default_rng(3)
    n, K = 64, 16
    params, grads = _groups(n, K, rng), _groups(n, K, rng)
    z = _groups(n, K, rng, zero=True)
    lr = dict(means=1e-3, log_scales=5e-3, quats=0.1, opacity_logits=5e-2, sh=(0.0, 1e-2))
    P, _, _ = oracle.adam_step(params, grads, z, z, lr, step=1)
    assert np.allclose(np.linalg.norm(P["quats"].astype(np.float64), axis=1), 1.0, atol=1e-6)
    assert np.array_equal(P["sh"][:, 0], params["sh"][:, 0])
    assert not np.array_equal(P["sh"][:, 1:], params["sh"][:, 1:])
