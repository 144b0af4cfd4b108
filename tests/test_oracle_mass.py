"""Pins of the oracle's condition measure (the "mass" of SURVEY §8c.9 P4/P5) — CPU only.

The GPU parity tests classify an element that misses the 1e-3 rule but lies within 1e-5 of its
mass as "condition-limited" (tests/gpu_helpers.py).  That escape is only as good as the mass, so
the mass is pinned here against things other than itself:

* Definition ("mass = sum |terms| per gradient entry").  For the projection backward
  the terms are those of the chain rule of SURVEY §8c.6 / DESIGN.md §4.5, stage by stage.  This
  test rebuilds that chain independently: every stage of the forward projection (SURVEY §8c.2 steps
  1-12) is written again here in torch fp64, its local Jacobian taken by autograd, and the masses
  propagated back with |J|^T — except the two normalisations, whose backward is WRITTEN as a
  difference of two terms (dq = (dq^ - q^<q^,dq^>)/|q|, §8c.6; the same for the SH direction d^),
  so their sum of |terms| is (|I| + |q^||q^|^T)/|q|.  vko_project_bwd_mass must equal this to
  rounding (1e-9 relative).  A dropped or extra path, a wrong coefficient or a transposed operand
  fails it.
* Bound property: the chain is linear in the 2D gradients, so for any signed input g with
  |g| <= m elementwise, |project_bwd(g)| <= mass(m) (triangle inequality).  Checked with random
  signs and one-hot inputs; a mass computed without one path (the colour path) is shown to fail it.
* The raster-backward mass (oracle.render(want_mass=True)) obeys the same bound, equals |gradient|
  exactly when one term contributes (one Gaussian, one pixel), and adds over pixels.
"""
import numpy as np
import pytest
import torch

import synth

F64 = torch.float64  # every tensor here is fp64 (explicitly: the default dtype is left alone)

GRADS = ("dmeans", "dlog_scales", "dquats", "dopacity_logits", "dsh")
IN2D = ("dmeans2d", "dconics", "dcolors", "dopacities")

# 3DGS real-SH constants
C0 = 0.28209479177387814
C1 = 0.4886025119029199
C2 = [1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792, 0.5462742152960396]
C3 = [-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
      -0.4570457994644658, 1.445305721320277, -0.5900435899266435]


def sh_basis(d):
    x, y, z = d[0], d[1], d[2]
    xx, yy, zz = x * x, y * y, z * z
    return torch.stack([
        0 * x + C0,
        -C1 * y, C1 * z, -C1 * x,
        C2[0] * x * y, C2[1] * y * z, C2[2] * (2 * zz - xx - yy), C2[3] * x * z, C2[4] * (xx - yy),
        C3[0] * y * (3 * xx - yy), C3[1] * x * y * z, C3[2] * y * (4 * zz - xx - yy),
        C3[3] * z * (2 * zz - 3 * xx - 3 * yy), C3[4] * x * (4 * zz - xx - yy), C3[5] * z * (xx - yy),
        C3[6] * x * (xx - 3 * yy)])


def jac(f, *xs):
    """Local Jacobian blocks of stage f at xs (autograd, fp64): list over inputs of [out, in]."""
    J = torch.autograd.functional.jacobian(f, tuple(xs))
    out = []
    for j, x in zip(J, xs):
        out.append(j.reshape(-1, x.numel()))
    return out


def chain_mass(cfg, cam, mu, ls, q, o, sh, flags, m2d):
    """sum |terms| of the SURVEY §8c.6 chain for one visible Gaussian, rebuilt from local Jacobians.
    m2d = (m_mean2d[2], m_conic[3], m_colour[3], m_rho) non-negative.  Returns the five masses."""
    import oracle
    R = torch.tensor(np.asarray(cam["R"], np.float64)).reshape(3, 3)
    tc = torch.tensor(np.asarray(cam["t"], np.float64))
    fx, fy, cx, cy = (float(cam[k]) for k in ("fx", "fy", "cx", "cy"))
    W, H = float(cam["width"]), float(cam["height"])
    K = cfg["sh_degree"] + 1
    K = K * K
    mu, ls, q = (torch.tensor(np.asarray(a, np.float64)) for a in (mu, ls, q))
    f = torch.tensor(np.asarray(sh, np.float64)[:K])          # [K, 3]
    m_uv, m_con, m_col, m_rho = (torch.tensor(np.asarray(a, np.float64)) for a in m2d)
    # forward decisions (FOV clamp, colour clamp) from the oracle's fp32 projection flags
    clx = bool(flags & (oracle.F_FOVX_HI | oracle.F_FOVX_LO))
    cly = bool(flags & (oracle.F_FOVY_HI | oracle.F_FOVY_LO))
    Lx = ((W - cx) / fx + 0.3 * (0.5 * W / fx)) if flags & oracle.F_FOVX_HI else -(cx / fx + 0.3 * (0.5 * W / fx))
    Ly = ((H - cy) / fy + 0.3 * (0.5 * H / fy)) if flags & oracle.F_FOVY_HI else -(cy / fy + 0.3 * (0.5 * H / fy))
    col_on = torch.tensor([0.0 if flags & (oracle.F_CLAMP_R << ch) else 1.0 for ch in range(3)], dtype=F64)

    # ---- the forward stages, each a function of the previous stage's outputs
    st_t = lambda mu_: R @ mu_ + tc                                                     # step 1

    def st_uvJ(t):                                                                        # steps 6, 7, 9
        tx, ty, tz = t[0], t[1], t[2]
        txc = tz * Lx if clx else tx
        tyc = tz * Ly if cly else ty
        return torch.stack([fx * tx / tz + cx, fy * ty / tz + cy,
                            fx / tz, -fx * txc / (tz * tz), fy / tz, -fy * tyc / (tz * tz)])

    def st_Rq(qh):                                                                        # step 3
        w, x, y, z = qh[0], qh[1], qh[2], qh[3]
        return torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                            2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                            2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)])
    st_s = lambda ls_: torch.exp(ls_)                                                     # step 4
    st_M = lambda Rq, s: (Rq.reshape(3, 3) * s[None, :]).reshape(9)                       # step 4
    st_Mc = lambda M: (R @ M.reshape(3, 3)).reshape(9)                                    # step 5

    def st_K(Jv, Mc):                                                                     # step 7
        Mc = Mc.reshape(3, 3)
        return torch.cat([Jv[0] * Mc[0] + Jv[1] * Mc[2], Jv[2] * Mc[1] + Jv[3] * Mc[2]])

    def st_ABC(Kv):                                                                       # step 8
        K0, K1 = Kv[:3], Kv[3:]
        return torch.stack([K0 @ K0 + 0.3, K0 @ K1, K1 @ K1 + 0.3])

    def st_conic(abc):                                                                    # step 8
        A, B, C = abc[0], abc[1], abc[2]
        det = A * C - B * B
        return torch.stack([C / det, -B / det, A / det])

    st_col = lambda Y, fv: Y[:K] @ fv                                                     # step 12

    # forward values
    t = st_t(mu)
    uvJ = st_uvJ(t)
    qn = torch.linalg.norm(q)
    qh = q / qn
    Rq = st_Rq(qh)
    s = st_s(ls)
    M = st_M(Rq, s)
    Mc = st_Mc(M)
    Kv = st_K(uvJ[2:], Mc)
    abc = st_ABC(Kv)
    campos = -(R.T @ tc)
    d = mu - campos
    dn = torch.linalg.norm(d)
    dh = d / dn
    Y = sh_basis(dh)
    rho = 1.0 / (1.0 + torch.exp(-torch.as_tensor(float(o), dtype=F64)))

    # ---- reverse accumulation with |local Jacobian|^T
    (Jc,) = jac(st_conic, abc)
    m_abc = Jc.abs().T @ m_con
    (JK,) = jac(st_ABC, Kv)
    m_K = JK.abs().T @ m_abc
    JKJ, JKM = jac(st_K, uvJ[2:], Mc)
    m_J, m_Mc = JKJ.abs().T @ m_K, JKM.abs().T @ m_K
    (JMc,) = jac(st_Mc, M)
    m_M = JMc.abs().T @ m_Mc
    JMR, JMs = jac(st_M, Rq, s)
    m_Rq, m_s = JMR.abs().T @ m_M, JMs.abs().T @ m_M
    (Js,) = jac(st_s, ls)
    m_ls = Js.abs().T @ m_s
    (JRq,) = jac(st_Rq, qh)
    m_qh = JRq.abs().T @ m_Rq
    # dq = (dq^ - q^ <q^, dq^>) / |q|: two terms, sum of their magnitudes
    m_q = (m_qh + qh.abs() * (qh.abs() @ m_qh)) / qn
    (Jt,) = jac(st_uvJ, t)
    m_t = Jt.abs().T @ torch.cat([m_uv, m_J])
    (Jmu,) = jac(st_t, mu)
    m_mu = Jmu.abs().T @ m_t
    # colour: (Y, f) -> colour on unclamped channels; d^ -> Y; d -> d^ written as two terms
    mce = m_col * col_on
    JY, Jf = jac(st_col, Y, f)
    m_Y, m_f = JY.abs().T @ mce, Jf.abs().T @ mce
    (JdY,) = jac(sh_basis, dh)
    m_dh = JdY[:K].abs().T @ m_Y[:K]
    m_mu = m_mu + (m_dh + dh.abs() * (dh.abs() @ m_dh)) / dn
    m_logit = m_rho * rho * (1 - rho)
    return dict(dmeans=m_mu.numpy(), dlog_scales=m_ls.numpy(), dquats=m_q.numpy(),
                dopacity_logits=float(m_logit), dsh=m_f.reshape(K, 3).numpy())


def _cases():
    out = []
    # FD fixtures: seeds 5, 9, 13, 17 carry a visible FOV-clamped Gaussian, seeds 0, 6, 9, 12, 13,
    # 14, 17 a colour-clamped channel
    for seed in (0, 3, 5, 6, 9, 12, 13, 14, 17):
        scene, cam, cfg, _ = synth.fd_fixture(seed, footprint=seed % 2)
        out.append((f"fd{seed}", scene, cam, cfg))
    tiny = synth.CONFIGS["tiny"]
    sc = synth.make_scene(400, tiny.kind, 7)
    cam = synth.ring_cameras(64, 64, tiny.kind, 8)[3]
    out.append(("tiny_d3", sc, cam, synth.default_render_config(3)))
    sc1 = dict(sc, sh=np.ascontiguousarray(sc["sh"][:, :4]))
    out.append(("tiny_d1", sc1, cam, synth.default_render_config(1)))
    return out


def _random_m2d(rng, n, onehot=None):
    m = dict(dmeans2d=rng.uniform(0.1, 2.0, (n, 2)), dconics=rng.uniform(0.1, 2.0, (n, 3)),
             dcolors=rng.uniform(0.1, 2.0, (n, 3)), dopacities=rng.uniform(0.1, 2.0, n))
    if onehot is not None:  # one input component only: (group, column)
        for k in m:
            m[k] = np.zeros_like(m[k])
        k, c = onehot
        if m[k].ndim == 1:
            m[k][:] = 1.0
        else:
            m[k][:, c] = 1.0
    return m


@pytest.mark.parametrize("case", range(len(_cases())))
def test_project_mass_equals_abs_chain(oracle_lib, case):
    name, scene, cam, cfg = _cases()[case]
    n = scene["means"].shape[0]
    rng = np.random.default_rng(100 + case)
    m2d = _random_m2d(rng, n)
    mass = oracle_lib.project_bwd_mass(cfg, cam, scene, m2d)
    proj = oracle_lib.project_fwd(cfg, cam, scene)
    vis = np.nonzero(proj["tiles_touched"] > 0)[0]
    assert len(vis) > 0, name
    if name in ("fd5", "fd9", "fd13", "fd17"):
        clamped = proj["flags"][vis] & (oracle_lib.F_FOVX_HI | oracle_lib.F_FOVX_LO)
        assert clamped.any(), name  # the FOV-clamp branch is exercised
    checked = 0
    for i in vis[:60]:
        ref = chain_mass(cfg, cam, scene["means"][i], scene["log_scales"][i], scene["quats"][i],
                         scene["opacity_logits"][i], scene["sh"][i], int(proj["flags"][i]),
                         (m2d["dmeans2d"][i], m2d["dconics"][i], m2d["dcolors"][i], m2d["dopacities"][i]))
        for k in GRADS:
            got = np.asarray(mass[k][i], np.float64).reshape(-1)
            want = np.asarray(ref[k], np.float64).reshape(-1)
            got = got[: want.size]
            assert np.allclose(got, want, rtol=1e-9, atol=1e-300), (name, i, k, got, want)
        checked += 1
    # rows the chain never reaches have zero mass
    hid = proj["tiles_touched"] == 0
    for k in GRADS:
        assert not np.any(mass[k][hid]), (name, k)
    assert checked > 0


def _bound_ok(oracle_lib, cfg, cam, scene, m2d, g2d, mass=None):
    g = oracle_lib.project_bwd(cfg, cam, scene, g2d)
    if mass is None:
        mass = oracle_lib.project_bwd_mass(cfg, cam, scene, m2d)
    worst = 0.0
    for k in GRADS:
        lhs = np.abs(g[k]).reshape(-1)
        rhs = mass[k].reshape(-1) * (1 + 1e-9) + 1e-300
        worst = max(worst, float(np.max(lhs / rhs)) if lhs.size else 0.0)
    return worst


@pytest.mark.parametrize("case", range(len(_cases())))
def test_project_mass_bounds_the_chain(oracle_lib, case):
    """|project_bwd(g)| <= mass(|g|) for random signs and for every one-hot input component."""
    name, scene, cam, cfg = _cases()[case]
    n = scene["means"].shape[0]
    rng = np.random.default_rng(200 + case)
    for trial in range(4):
        m2d = _random_m2d(rng, n)
        g2d = {k: v * rng.choice([-1.0, 1.0], v.shape) for k, v in m2d.items()}
        assert _bound_ok(oracle_lib, cfg, cam, scene, m2d, g2d) <= 1.0, (name, trial)
    for oh in [("dmeans2d", 0), ("dmeans2d", 1), ("dconics", 0), ("dconics", 1), ("dconics", 2),
               ("dcolors", 0), ("dcolors", 2), ("dopacities", 0)]:
        m2d = _random_m2d(rng, n, onehot=oh)
        w = _bound_ok(oracle_lib, cfg, cam, scene, m2d, m2d)
        assert w <= 1.0, (name, oh, w)


def test_project_mass_without_a_path_is_caught(oracle_lib):
    """A mass that drops the colour path under-estimates: the bound check above flags it."""
    scene, cam, cfg, _ = synth.fd_fixture(2)
    n = scene["means"].shape[0]
    m2d = _random_m2d(np.random.default_rng(3), n)
    bad = oracle_lib.project_bwd_mass(cfg, cam, scene, dict(m2d, dcolors=np.zeros_like(m2d["dcolors"])))
    assert _bound_ok(oracle_lib, cfg, cam, scene, m2d, m2d, mass=bad) > 1.0
    half = {k: 0.5 * v for k, v in oracle_lib.project_bwd_mass(cfg, cam, scene, m2d).items()}
    assert _bound_ok(oracle_lib, cfg, cam, scene, m2d, m2d, mass=half) > 1.0


def test_project_mass_is_linear(oracle_lib):
    scene, cam, cfg, _ = synth.fd_fixture(4)
    n = scene["means"].shape[0]
    rng = np.random.default_rng(4)
    a, b = _random_m2d(rng, n), _random_m2d(rng, n)
    ma, mb = (oracle_lib.project_bwd_mass(cfg, cam, scene, x) for x in (a, b))
    mab = oracle_lib.project_bwd_mass(cfg, cam, scene, {k: 2 * a[k] + 3 * b[k] for k in a})
    for k in GRADS:
        assert np.allclose(mab[k], 2 * ma[k] + 3 * mb[k], rtol=1e-12, atol=0), k


def test_render_mass_bounds_and_single_term(oracle_lib):
    """The raster-backward mass: |grad| <= mass for random upstream signs; with one Gaussian and one
    pixel carrying upstream gradient every entry has a single term, so mass == |grad|."""
    scene, cam, cfg, dL = synth.fd_fixture(6)
    r = oracle_lib.render(cfg, cam, scene, dL=dL, want_mass=True)
    cols = {"dmeans2d": [0, 1], "dconics": [2, 3, 4], "dcolors": [5, 6, 7], "dopacities": [8]}
    for k, c in cols.items():
        g = np.abs(r[k]).reshape(len(r["mass"]), -1)
        assert np.all(g <= r["mass"][:, c] * (1 + 1e-12) + 1e-300), k
    one = {k: v[:1].copy() for k, v in scene.items()}
    one["means"][0] = [0.05, -0.03, 3.0]
    one["opacity_logits"][0] = 0.0
    w = np.zeros_like(dL)
    w[8, 9] = [0.3, -0.7, 0.5]
    r1 = oracle_lib.render(cfg, cam, one, dL=w, want_mass=True)
    assert r1["mass"][0].max() > 0
    for k, c in cols.items():
        assert np.allclose(np.abs(r1[k]).reshape(-1), r1["mass"][0, c], rtol=1e-12, atol=0), k
    # additivity over pixels: the mass of two pixels' upstream is the sum of each pixel's mass
    w2 = np.zeros_like(dL)
    w2[5, 4] = [-0.2, 0.4, 0.1]
    ra = oracle_lib.render(cfg, cam, one, dL=w2, want_mass=True)
    rb = oracle_lib.render(cfg, cam, one, dL=w + w2, want_mass=True)
    assert np.allclose(rb["mass"], r1["mass"] + ra["mass"], rtol=1e-12, atol=1e-300)
