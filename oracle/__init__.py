"""CPU oracle for the VkSplat hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2605_00219_b200``) never imports it; the two share no code.

Thin ctypes wrapper over ``oracle/libvko.so`` (plain C, see vko.h / vko.c for the
citations of every formula).  numpy in, numpy out.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libvko.so")
_lib = None


class Camera(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32)]


class Config(C.Structure):
    _fields_ = [("sh_degree", C.c_int32), ("sh_coeffs", C.c_int32), ("near_plane", C.c_float),
                ("bg", C.c_float * 3), ("fov_clamp", C.c_int32), ("footprint", C.c_int32)]


F_PROJECTABLE, F_VISIBLE = 1, 2
F_CLAMP_R, F_CLAMP_G, F_CLAMP_B = 4, 8, 16
F_FOVX_HI, F_FOVX_LO, F_FOVY_HI, F_FOVY_LO = 32, 64, 128, 256


def build(force: bool = False) -> str:
    """Compile libvko.so with gcc (no fast-math, no FP contraction)."""
    src = [os.path.join(_HERE, f) for f in ("vko.c", "vko_generic.inc", "vko.h")]
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= max(os.path.getmtime(s) for s in src)):
        return _LIB_PATH
    import subprocess
    cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-pthread", "-Wall", "-Wno-unused-function", "-o", _LIB_PATH,
           os.path.join(_HERE, "vko.c"), "-lm"]
    subprocess.check_call(cmd)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.vko_scan_offsets.restype = C.c_int64
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def make_camera(cam: dict) -> Camera:
    c = Camera()
    c.R[:] = [float(x) for x in np.asarray(cam["R"], np.float32).reshape(9)]
    c.t[:] = [float(x) for x in np.asarray(cam["t"], np.float32).reshape(3)]
    c.fx, c.fy, c.cx, c.cy = (float(np.float32(cam[k])) for k in ("fx", "fy", "cx", "cy"))
    c.width, c.height = int(cam["width"]), int(cam["height"])
    return c


def make_config(cfg: dict) -> Config:
    c = Config()
    c.sh_degree = int(cfg["sh_degree"])
    c.sh_coeffs = int(cfg["sh_coeffs"])
    c.near_plane = float(cfg["near_plane"])
    c.bg[:] = [float(b) for b in cfg["bg"]]
    c.fov_clamp = int(cfg["fov_clamp"])
    c.footprint = int(cfg["footprint"])
    return c


def _scene32(scene):
    return [np.ascontiguousarray(scene[k], np.float32) for k in
            ("means", "log_scales", "quats", "opacity_logits", "sh")]


def _scene64(scene):
    return [np.ascontiguousarray(scene[k], np.float64) for k in
            ("means", "log_scales", "quats", "opacity_logits", "sh")]


def n_tiles(cam):
    return ((cam["width"] + 15) // 16) * ((cam["height"] + 15) // 16)


def project_fwd(cfg, cam, scene, nthreads=0, f64=False):
    """O1 (fp32) or O2 (fp64) projection forward.  Returns a dict of arrays."""
    n = scene["means"].shape[0]
    dt = np.float64 if f64 else np.float32
    out = dict(means2d=np.zeros((n, 2), dt), conics=np.zeros((n, 3), dt), depths=np.zeros(n, dt),
               radii=np.zeros((n, 2), np.int32), tiles_touched=np.zeros(n, np.int32),
               colors=np.zeros((n, 3), dt), opacities=np.zeros(n, dt), cov2d=np.zeros((n, 3), dt),
               flags=np.zeros(n, np.int32))
    args = [C.byref(make_config(cfg)), C.byref(make_camera(cam)), C.c_int64(n)]
    args += [_p(a) for a in (_scene64(scene) if f64 else _scene32(scene))]
    args += [_p(out[k]) for k in ("means2d", "conics", "depths", "radii", "tiles_touched", "colors",
                                  "opacities", "cov2d", "flags")]
    if f64:
        lib().vko_project_fwd_f64(*args)
    else:
        lib().vko_project_fwd_f32(*args, C.c_int(nthreads))
    return out


def scan_offsets(tiles_touched):
    t = np.ascontiguousarray(tiles_touched, np.int32)
    off = np.zeros(t.shape[0], np.uint32)
    m = lib().vko_scan_offsets(C.c_int64(t.shape[0]), _p(t), _p(off))
    return off, int(m)


def gen_keys(cam, proj, offsets, m):
    n = proj["depths"].shape[0]
    keys = np.zeros(max(m, 0), np.uint64)
    vals = np.zeros(max(m, 0), np.uint32)
    lib().vko_gen_keys(C.byref(make_camera(cam)), C.c_int64(n),
                       _p(np.ascontiguousarray(proj["means2d"], np.float32)),
                       _p(np.ascontiguousarray(proj["radii"], np.int32)),
                       _p(np.ascontiguousarray(proj["depths"], np.float32)),
                       _p(np.ascontiguousarray(proj["tiles_touched"], np.int32)),
                       _p(np.ascontiguousarray(offsets, np.uint32)), _p(keys), _p(vals))
    return keys, vals


def sort_pairs(keys, vals):
    k = np.array(keys, np.uint64, copy=True)
    v = np.array(vals, np.uint32, copy=True)
    lib().vko_sort_pairs(C.c_int64(k.shape[0]), _p(k), _p(v))
    return k, v


def tile_ranges(sorted_keys, ntiles):
    k = np.ascontiguousarray(sorted_keys, np.uint64)
    to = np.zeros(ntiles + 1, np.uint32)
    lib().vko_tile_ranges(C.c_int64(k.shape[0]), _p(k), C.c_int32(ntiles), _p(to))
    return to


def bin_sort(cfg, cam, proj):
    """Index offsets -> keys -> stable sort -> tile ranges."""
    off, m = scan_offsets(proj["tiles_touched"])
    keys_u, vals_u = gen_keys(cam, proj, off, m)
    keys, vals = sort_pairs(keys_u, vals_u)
    to = tile_ranges(keys, n_tiles(cam))
    return dict(offsets=off, num_isects=m, keys_unsorted=keys_u, vals_unsorted=vals_u,
                keys=keys, vals=vals, tile_offsets=to)


def render(cfg, cam, scene, dL=None, row_mask=None, brute=False, want_mass=False, nthreads=0):
    """O1 forward (+ fp64 backward when dL is given), untiled."""
    n = scene["means"].shape[0]
    H, W = cam["height"], cam["width"]
    out = dict(image=np.zeros((H, W, 3), np.float32), T_final=np.zeros((H, W), np.float32),
               last_id=np.zeros((H, W), np.int32), fragile=np.zeros((H, W), np.uint8),
               stats=np.zeros(8, np.int64))
    if dL is not None:
        for k, s in (("dmeans2d", 2), ("dconics", 3), ("dcolors", 3)):
            out[k] = np.zeros((n, s), np.float64)
        out["dopacities"] = np.zeros(n, np.float64)
        if want_mass:
            out["mass"] = np.zeros((n, 9), np.float64)
    dLa = None if dL is None else np.ascontiguousarray(dL, np.float32)
    rm = None if row_mask is None else np.ascontiguousarray(row_mask, np.uint8)
    lib().vko_render_f32(C.byref(make_config(cfg)), C.byref(make_camera(cam)), C.c_int64(n),
                         *[_p(a) for a in _scene32(scene)], _p(dLa), _p(rm), C.c_int(int(brute)),
                         _p(out["image"]), _p(out["T_final"]), _p(out["last_id"]),
                         _p(out["fragile"]), _p(out["stats"]), _p(out.get("dmeans2d")),
                         _p(out.get("dconics")), _p(out.get("dcolors")), _p(out.get("dopacities")),
                         _p(out.get("mass")), C.c_int(nthreads))
    st = out["stats"]
    out["footprint_violations"], out["evaluations"], out["composited"] = int(st[0]), int(st[1]), int(st[2])
    out["fragile_pixels"], out["candidates"], out["rows"] = int(st[3]), int(st[4]), int(st[5])
    return out


def render_f64(cfg, cam, scene, dL=None):
    """O2: fp64 forward (brute force), decision hashes, optional fp64 backward."""
    n = scene["means"].shape[0]
    H, W = cam["height"], cam["width"]
    out = dict(image=np.zeros((H, W, 3), np.float64), decision_hash=np.zeros((H, W), np.uint64),
               proj_flags=np.zeros(n, np.int32))
    if dL is not None:
        for k, s in (("dmeans2d", 2), ("dconics", 3), ("dcolors", 3)):
            out[k] = np.zeros((n, s), np.float64)
        out["dopacities"] = np.zeros(n, np.float64)
    dLa = None if dL is None else np.ascontiguousarray(dL, np.float64)
    lib().vko_render_f64(C.byref(make_config(cfg)), C.byref(make_camera(cam)), C.c_int64(n),
                         *[_p(a) for a in _scene64(scene)], _p(dLa), _p(out["image"]),
                         _p(out["decision_hash"]), _p(out["proj_flags"]), _p(out.get("dmeans2d")),
                         _p(out.get("dconics")), _p(out.get("dcolors")), _p(out.get("dopacities")))
    return out


def project_bwd(cfg, cam, scene, g2d, nthreads=0, f64=False):
    """O2 projection backward.  g2d: dict dmeans2d [n,2], dconics [n,3],
    dcolors [n,3], dopacities [n] (any float dtype).  Returns fp64 parameter gradients."""
    n = scene["means"].shape[0]
    S = scene["sh"].shape[1]
    out = dict(dmeans=np.zeros((n, 3)), dlog_scales=np.zeros((n, 3)), dquats=np.zeros((n, 4)),
               dopacity_logits=np.zeros(n), dsh=np.zeros((n, S, 3)))
    gi = [np.ascontiguousarray(g2d[k], np.float64) for k in ("dmeans2d", "dconics", "dcolors", "dopacities")]
    args = [C.byref(make_config(cfg)), C.byref(make_camera(cam)), C.c_int64(n)]
    args += [_p(a) for a in (_scene64(scene) if f64 else _scene32(scene))]
    args += [_p(a) for a in gi]
    args += [_p(out[k]) for k in ("dmeans", "dlog_scales", "dquats", "dopacity_logits", "dsh")]
    if f64:
        lib().vko_project_bwd_f64(*args)
    else:
        lib().vko_project_bwd(*args, C.c_int(nthreads))
    return out


def project_bwd_mass(cfg, cam, scene, m2d, nthreads=0):
    """Running-error mass of the projection backward for non-negative 2D-gradient masses m2d
    (dict dmeans2d/dconics/dcolors/dopacities).  Returns fp64 masses shaped like the gradients."""
    n = scene["means"].shape[0]
    S = scene["sh"].shape[1]
    out = dict(dmeans=np.zeros((n, 3)), dlog_scales=np.zeros((n, 3)), dquats=np.zeros((n, 4)),
               dopacity_logits=np.zeros(n), dsh=np.zeros((n, S, 3)))
    gi = [np.ascontiguousarray(np.abs(m2d[k]), np.float64) for k in ("dmeans2d", "dconics", "dcolors", "dopacities")]
    lib().vko_project_bwd_mass(C.byref(make_config(cfg)), C.byref(make_camera(cam)), C.c_int64(n),
                               *[_p(a) for a in _scene32(scene)], *[_p(a) for a in gi],
                               *[_p(out[k]) for k in ("dmeans", "dlog_scales", "dquats", "dopacity_logits", "dsh")],
                               C.c_int(nthreads))
    return out


def full_backward(cfg, cam, scene, dL, row_mask=None, want_mass=False, nthreads=0):
    """End-to-end oracle: render (O1 fwd + O2 bwd) then O2 projection backward."""
    r = render(cfg, cam, scene, dL=dL, row_mask=row_mask, want_mass=want_mass, nthreads=nthreads)
    pb = project_bwd(cfg, cam, scene, r, nthreads=nthreads)
    r.update(pb)
    return r


# ---- the optimizer step (Adam with bias correction) -------------------
ADAM_GROUPS = ("means", "log_scales", "quats", "opacity_logits", "sh")


def adam_step(params, grads, m, v, lr, beta1=0.9, beta2=0.999, eps=1e-8, step=1):
    """One Adam step on every parameter group (vko_adam_group), then the quaternion
    re-normalisation (vko_quat_renorm).  params/grads/m/v: dicts of fp32 arrays keyed by
    ADAM_GROUPS; lr: dict with a learning rate per group, where "sh" may be a pair (lr of SH
    coefficient 0, lr of the others).  Returns new (params, m, v) dicts (inputs untouched)."""
    L = lib()
    L.vko_adam_group.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                 C.c_double, C.c_double, C.c_double, C.c_int32]
    L.vko_quat_renorm.argtypes = [C.c_int64, C.c_void_p]
    P, M, Vv = {}, {}, {}
    for k in ADAM_GROUPS:
        p = np.ascontiguousarray(params[k], np.float32).copy()
        mm = np.ascontiguousarray(m[k], np.float32).copy()
        vv = np.ascontiguousarray(v[k], np.float32).copy()
        g = np.ascontiguousarray(grads[k], np.float32)
        lk = lr[k]
        if k == "sh" and isinstance(lk, (tuple, list)):  # coefficient 0 and the rest: two groups
            n = p.shape[0]
            p3, m3, v3, g3 = (a.reshape(n, -1, 3) for a in (p, mm, vv, g))
            for sl, lrs in ((slice(0, 1), lk[0]), (slice(1, None), lk[1])):
                ps, ms, vs, gs = (np.ascontiguousarray(a[:, sl]) for a in (p3, m3, v3, g3))
                L.vko_adam_group(ps.size, _p(ps), _p(ms), _p(vs), _p(gs), lrs, beta1, beta2, eps, step)
                p3[:, sl], m3[:, sl], v3[:, sl] = ps, ms, vs
        else:
            L.vko_adam_group(p.size, _p(p), _p(mm), _p(vv), _p(g), float(lk), beta1, beta2, eps, step)
        if k == "quats":
            L.vko_quat_renorm(p.shape[0], _p(p))
        P[k], M[k], Vv[k] = p, mm, vv
    return P, M, Vv


# ---- the loss gradient (L1 + lambda D-SSIM) ------------------
def loss_grad(render, target, lam=0.2):
    """(loss, dL/drender fp64 [H, W, 3], ssim) of vko_loss_grad for HWC fp32 images."""
    L = lib()
    L.vko_loss_grad.restype = C.c_double
    L.vko_loss_grad.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    r = np.ascontiguousarray(render, np.float32)
    t = np.ascontiguousarray(target, np.float32)
    H, W = r.shape[:2]
    g = np.zeros((H, W, 3), np.float64)
    ss = C.c_double(0)
    loss = L.vko_loss_grad(W, H, lam, _p(r), _p(t), _p(g), C.byref(ss))
    return float(loss), g, float(ss.value)


# ---- MCMC densification (DESIGN.md §4.7 readings R1-R5) ------------------
def _mcmc_lib():
    L = lib()
    L.vko_rng.restype = C.c_uint64
    L.vko_rng.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64]
    L.vko_mcmc_relocate.restype = C.c_int64
    L.vko_mcmc_relocate.argtypes = [C.c_int64, C.c_int32, C.c_float, C.c_uint64] + [C.c_void_p] * 8
    L.vko_mcmc_noise.argtypes = [C.c_int64, C.c_float, C.c_float, C.c_uint64, C.c_uint32] + [C.c_void_p] * 4
    return L


def rng(seed, stream, i):
    return int(_mcmc_lib().vko_rng(seed, stream, i))


def mcmc_relocate(scene, dead_opacity=0.005, seed=0, m=None, v=None):
    """Relocation of the dead Gaussians (vko_mcmc_relocate) on copies of the scene arrays (and of
    the flat Adam moments m, v if given).  Returns (new scene dict, targets, n_dead, m, v)."""
    L = _mcmc_lib()
    sc = {k: np.ascontiguousarray(scene[k], np.float32).copy() for k in ("means", "log_scales", "quats",
                                                                          "opacity_logits", "sh")}
    n, K = sc["means"].shape[0], sc["sh"].shape[1]
    mm = None if m is None else np.ascontiguousarray(m, np.float32).copy()
    vv = None if v is None else np.ascontiguousarray(v, np.float32).copy()
    tg = np.zeros(n, np.int64)
    dead = L.vko_mcmc_relocate(n, K, dead_opacity, seed, _p(sc["means"]), _p(sc["log_scales"]), _p(sc["quats"]),
                               _p(sc["opacity_logits"]), _p(sc["sh"]), _p(mm), _p(vv), _p(tg))
    return sc, tg, int(dead), mm, vv


def mcmc_noise(scene, lr_pos, noise_scale, seed=0, step=0):
    """Positional noise (vko_mcmc_noise) on a copy of the means; returns the new means."""
    L = _mcmc_lib()
    means = np.ascontiguousarray(scene["means"], np.float32).copy()
    ls = np.ascontiguousarray(scene["log_scales"], np.float32)
    q = np.ascontiguousarray(scene["quats"], np.float32)
    o = np.ascontiguousarray(scene["opacity_logits"], np.float32)
    L.vko_mcmc_noise(means.shape[0], lr_pos, noise_scale, seed, step, _p(means), _p(ls), _p(q), _p(o))
    return means


# ---- default densification (DESIGN.md §4.7 readings R6-R9) -----------
def _densify_lib():
    L = _mcmc_lib()
    L.vko_densify_stats.argtypes = [C.c_int64] + [C.c_void_p] * 4
    L.vko_densify.restype = C.c_int64
    L.vko_densify.argtypes = ([C.c_int64, C.c_int32] + [C.c_void_p] * 9 + [C.c_float, C.c_float, C.c_float, C.c_uint64,
                              C.c_int64] + [C.c_void_p] * 7)
    return L


def densify_stats(dmeans2d, radii, accum, denom):
    """Returns updated copies of (accum, denom) after one view (vko_densify_stats)."""
    L = _densify_lib()
    a = np.ascontiguousarray(accum, np.float32).copy()
    d = np.ascontiguousarray(denom, np.float32).copy()
    g = np.ascontiguousarray(dmeans2d, np.float32)
    r = np.ascontiguousarray(radii, np.int32)
    L.vko_densify_stats(a.shape[0], _p(g), _p(r), _p(a), _p(d))
    return a, d


def densify(scene, accum, denom, grad_threshold, size_threshold, prune_opacity=0.005, seed=0, m=None, v=None,
            cap=None):
    """One densification event (vko_densify).  Returns (new scene dict, n', m', v') — n' only (and
    None for the rest) when n' > cap."""
    L = _densify_lib()
    sc = {k: np.ascontiguousarray(scene[k], np.float32) for k in ("means", "log_scales", "quats", "opacity_logits", "sh")}
    n, K = sc["means"].shape[0], sc["sh"].shape[1]
    F = 11 + 3 * K
    cap = 2 * n if cap is None else cap
    out = dict(means=np.zeros((cap, 3), np.float32), log_scales=np.zeros((cap, 3), np.float32),
               quats=np.zeros((cap, 4), np.float32), opacity_logits=np.zeros(cap, np.float32),
               sh=np.zeros((cap, K, 3), np.float32))
    om = np.zeros(max(cap, 1) * F, np.float32) if m is not None else None
    ov = np.zeros(max(cap, 1) * F, np.float32) if v is not None else None
    mm = None if m is None else np.ascontiguousarray(m, np.float32)
    vv = None if v is None else np.ascontiguousarray(v, np.float32)
    a = np.ascontiguousarray(accum, np.float32)
    d = np.ascontiguousarray(denom, np.float32)
    np_ = L.vko_densify(n, K, _p(sc["means"]), _p(sc["log_scales"]), _p(sc["quats"]), _p(sc["opacity_logits"]),
                        _p(sc["sh"]), _p(mm), _p(vv), _p(a), _p(d), grad_threshold, size_threshold, prune_opacity,
                        seed, cap, _p(out["means"]), _p(out["log_scales"]), _p(out["quats"]),
                        _p(out["opacity_logits"]), _p(out["sh"]), _p(om), _p(ov))
    if np_ > cap:
        return None, int(np_), None, None
    out = {k: a_[:np_] for k, a_ in out.items()}
    if om is not None:  # the flat group-major moments of n' rows are the first n' F entries
        om, ov = om[:np_ * F], ov[:np_ * F]
    return out, int(np_), om, ov
