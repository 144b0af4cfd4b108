"""ctypes binding of libvks.so — argument marshalling only.

Every function here has the name of the C entry point it wraps (include/vks.h) and does nothing
but check tensor dtype / device / contiguity, pass raw device pointers and the current CUDA
stream, and raise on a non-OK status.  All computation happens in the CUDA kernels.  If the
library is missing or cannot load, importing this module raises: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# VKS_DEBUG_CHECKS=1: the debug build with device-side bounds / invariant checks (_build.py);
# VKS_LIB_VARIANT=<name>: libvks_<name>.so, an in-tree build variant (measurement experiments)
_variant = os.environ.get("VKS_LIB_VARIANT")
LIB_PATH = os.path.join(_HERE, "libvks_debug.so" if os.environ.get("VKS_DEBUG_CHECKS") == "1" else
                        (f"libvks_{_variant}.so" if _variant else "libvks.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python paper_2605_00219_b200/_build.py` "
                      "(or __graft_entry__.build()); the CUDA path has no fallback")
_lib = C.CDLL(LIB_PATH)

(VKS_OK, VKS_ERR_INVALID_ARG, VKS_ERR_CAPACITY, VKS_ERR_WORKSPACE, VKS_ERR_CUDA, VKS_ERR_UNSUPPORTED,
 VKS_ERR_NONFINITE, VKS_ERR_UNSORTED) = range(8)
FOOTPRINT_SUPPORT, FOOTPRINT_3SIGMA = 0, 1
FLAG_GRAD_OVERWRITE = 1
FLAG_VALIDATE = 2

EXPORTS = ("vks_status_string", "vks_version", "vks_last_cuda_error", "vks_project_fwd",
           "vks_bin_sort_workspace_bytes", "vks_bin_sort", "vks_raster_fwd", "vks_raster_fwd_stats",
           "vks_raster_bwd", "vks_project_bwd", "vks_project_fwd_batch", "vks_project_bwd_batch",
           "vks_adam_step", "vks_loss_workspace_bytes", "vks_loss_grad", "vks_mcmc_workspace_bytes",
           "vks_mcmc_relocate", "vks_mcmc_noise", "vks_densify_stats", "vks_densify_workspace_bytes",
           "vks_densify", "vks_bin_sort_check", "vks_bin_sort_async")


class VksCamera(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32)]


class VksConfig(C.Structure):
    _fields_ = [("sh_degree", C.c_int32), ("sh_coeffs", C.c_int32), ("near_plane", C.c_float),
                ("bg", C.c_float * 3), ("fov_clamp", C.c_int32), ("footprint", C.c_int32),
                ("flags", C.c_uint32)]


class VksAdamConfig(C.Structure):
    _fields_ = [("lr", C.c_float * 6), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("step", C.c_int32)]


ADAM_GROUPS = ("means", "log_scales", "quats", "opacity_logits", "sh")


def make_adam_config(lr, beta1=0.9, beta2=0.999, eps=1e-8, step=1) -> VksAdamConfig:
    """lr: dict keyed by ADAM_GROUPS ("sh" may be a pair: coefficient 0, the others) or 6 floats."""
    a = VksAdamConfig()
    if isinstance(lr, dict):
        sh = lr["sh"] if isinstance(lr["sh"], (tuple, list)) else (lr["sh"], lr["sh"])
        vals = [lr["means"], lr["log_scales"], lr["quats"], lr["opacity_logits"], sh[0], sh[1]]
    else:
        vals = list(lr)
    a.lr[:] = [float(x) for x in vals]
    a.beta1, a.beta2, a.eps, a.step = float(beta1), float(beta2), float(eps), int(step)
    return a


_P = C.c_void_p
_lib.vks_status_string.restype = C.c_char_p
_lib.vks_status_string.argtypes = [C.c_int]
_lib.vks_last_cuda_error.restype = C.c_char_p
_lib.vks_version.restype = C.c_int
_lib.vks_bin_sort_workspace_bytes.restype = C.c_size_t
_lib.vks_bin_sort_workspace_bytes.argtypes = [C.c_int64, C.c_int64, C.c_int32]
_lib.vks_project_fwd.argtypes = [_P, _P, C.c_int64] + [_P] * 14
_lib.vks_bin_sort.argtypes = [_P, C.c_int64] + [_P] * 5 + [C.c_int64] + [_P] * 8 + [C.c_size_t, _P]
_lib.vks_raster_fwd.argtypes = [_P, _P, C.c_int64] + [_P] * 13
_lib.vks_bin_sort_async.argtypes = [_P, C.c_int64] + [_P] * 5 + [C.c_int64] + [_P] * 5 + [_P, C.c_size_t, _P]
_lib.vks_bin_sort_check.argtypes = [_P, C.c_int64] + [_P] * 5 + [C.c_int64, _P]
_lib.vks_raster_bwd.argtypes = [_P, _P, C.c_int64] + [_P] * 17
_lib.vks_raster_fwd_stats.argtypes = [_P, _P, C.c_int64] + [_P] * 11
_lib.vks_project_bwd.argtypes = [_P, _P, C.c_int64] + [_P] * 17
_lib.vks_project_bwd_batch.argtypes = [_P, C.c_int32, _P, C.c_int64] + [_P] * 17
_lib.vks_project_fwd_batch.argtypes = [_P, C.c_int32, _P, C.c_int64] + [_P] * 15
_lib.vks_adam_step.argtypes = [_P, C.c_int64, C.c_int32, _P, _P, _P, _P, _P]
_lib.vks_loss_workspace_bytes.restype = C.c_size_t
_lib.vks_loss_workspace_bytes.argtypes = [C.c_int32, C.c_int32]
_lib.vks_loss_grad.argtypes = [C.c_int32, C.c_int32, C.c_float, _P, _P, _P, _P, _P, C.c_size_t, _P]
_lib.vks_loss_grad.restype = C.c_int
_lib.vks_mcmc_workspace_bytes.restype = C.c_size_t
_lib.vks_mcmc_workspace_bytes.argtypes = [C.c_int64]
_lib.vks_mcmc_relocate.argtypes = [C.c_int64, C.c_int32, C.c_float, C.c_uint64] + [_P] * 10 + [C.c_size_t, _P]
_lib.vks_mcmc_relocate.restype = C.c_int
_lib.vks_mcmc_noise.argtypes = [C.c_int64, C.c_float, C.c_float, C.c_uint64, C.c_uint32] + [_P] * 5
_lib.vks_mcmc_noise.restype = C.c_int
_lib.vks_densify_stats.argtypes = [C.c_int64] + [_P] * 5
_lib.vks_densify_stats.restype = C.c_int
_lib.vks_densify_workspace_bytes.restype = C.c_size_t
_lib.vks_densify_workspace_bytes.argtypes = [C.c_int64]
_lib.vks_densify.argtypes = ([C.c_int64, C.c_int32] + [_P] * 5 + [C.c_float, C.c_float, C.c_float, C.c_uint64,
                             C.c_int64] + [_P] * 5 + [C.c_size_t, _P])
_lib.vks_densify.restype = C.c_int
for _f in ("vks_project_fwd", "vks_bin_sort", "vks_raster_fwd", "vks_raster_fwd_stats", "vks_raster_bwd",
           "vks_project_bwd", "vks_project_fwd_batch", "vks_project_bwd_batch", "vks_adam_step"):
    getattr(_lib, _f).restype = C.c_int


class VksError(RuntimeError):
    def __init__(self, fn: str, status: int):
        msg = _lib.vks_status_string(status).decode()
        if status == VKS_ERR_CUDA:
            msg += ": " + _lib.vks_last_cuda_error().decode()
        super().__init__(f"{fn}: {msg} (status {status})")
        self.status = status


def make_camera(cam: dict) -> VksCamera:
    c = VksCamera()
    R = cam["R"].reshape(-1).tolist() if hasattr(cam["R"], "reshape") else list(cam["R"])
    c.R[:] = [float(x) for x in R]
    t = cam["t"].reshape(-1).tolist() if hasattr(cam["t"], "reshape") else list(cam["t"])
    c.t[:] = [float(x) for x in t]
    c.fx, c.fy, c.cx, c.cy = (float(cam[k]) for k in ("fx", "fy", "cx", "cy"))
    c.width, c.height = int(cam["width"]), int(cam["height"])
    return c


def make_config(cfg: dict) -> VksConfig:
    c = VksConfig()
    c.sh_degree = int(cfg["sh_degree"])
    c.sh_coeffs = int(cfg.get("sh_coeffs", (c.sh_degree + 1) ** 2))
    c.near_plane = float(cfg.get("near_plane", 0.01))
    c.bg[:] = [float(b) for b in cfg.get("bg", (0.0, 0.0, 0.0))]
    c.fov_clamp = int(cfg.get("fov_clamp", 1))
    c.footprint = int(cfg.get("footprint", FOOTPRINT_SUPPORT))
    c.flags = int(cfg.get("flags", 0))
    return c


def _ptr(t, dtype, name):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_cuda:
        raise ValueError(f"{name}: expected a CUDA tensor (libvks takes device pointers)")
    if not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous tensor")
    return t.data_ptr() if t.numel() else None


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _check(fn, st):
    if st != VKS_OK:
        raise VksError(fn, st)


def _cfgcam(cfg, cam):
    c = cfg if isinstance(cfg, VksConfig) else make_config(cfg)
    k = cam if isinstance(cam, VksCamera) else make_camera(cam)
    return c, k


f32, i32, u32, u64 = torch.float32, torch.int32, torch.uint32, torch.uint64


def vks_project_fwd(cfg, cam, means, log_scales, quats, opacity_logits, sh, means2d, conics, depths,
                    radii, tiles_touched, colors, opacities, stream=None, records=None):
    """records (optional, fp32 [n, 12], 16-byte aligned): the packed raster records of the visible
    Gaussians, for vks_raster_fwd / vks_raster_bwd (include/vks.h)."""
    c, k = _cfgcam(cfg, cam)
    n = means.shape[0]
    st = _lib.vks_project_fwd(C.byref(c), C.byref(k), n, _ptr(means, f32, "means"),
                              _ptr(log_scales, f32, "log_scales"), _ptr(quats, f32, "quats"),
                              _ptr(opacity_logits, f32, "opacity_logits"), _ptr(sh, f32, "sh"),
                              _ptr(means2d, f32, "means2d"), _ptr(conics, f32, "conics"),
                              _ptr(depths, f32, "depths"), _ptr(radii, i32, "radii"),
                              _ptr(tiles_touched, i32, "tiles_touched"), _ptr(colors, f32, "colors"),
                              _ptr(opacities, f32, "opacities"), _ptr(records, f32, "records"), _stream(stream))
    _check("vks_project_fwd", st)


def vks_bin_sort_workspace_bytes(n, capacity, n_tiles) -> int:
    return int(_lib.vks_bin_sort_workspace_bytes(n, capacity, n_tiles))


def vks_bin_sort(cam, means2d, radii, depths, tiles_touched, offsets, keys, vals, tile_offsets,
                 workspace, keys_unsorted=None, vals_unsorted=None, stream=None, raise_capacity=True,
                 tile_order=None):
    """Returns M (num_isects).  Capacity = vals.numel(); keys (u64, same capacity) may be None.
    tile_order (u32 [n_tiles], optional) receives the rasterizer's tile schedule.
    On VKS_ERR_CAPACITY returns -M when raise_capacity is False."""
    k = cam if isinstance(cam, VksCamera) else make_camera(cam)
    n = means2d.shape[0]
    m = C.c_int64(0)
    st = _lib.vks_bin_sort(C.byref(k), n, _ptr(means2d, f32, "means2d"), _ptr(radii, i32, "radii"),
                           _ptr(depths, f32, "depths"), _ptr(tiles_touched, i32, "tiles_touched"),
                           _ptr(offsets, u32, "offsets"), vals.numel(), _ptr(keys, u64, "keys"),
                           _ptr(vals, u32, "vals"), _ptr(keys_unsorted, u64, "keys_unsorted"),
                           _ptr(vals_unsorted, u32, "vals_unsorted"), _ptr(tile_offsets, u32, "tile_offsets"),
                           _ptr(tile_order, u32, "tile_order"), C.byref(m), _ptr(workspace, torch.uint8, "workspace"), workspace.numel(),
                           _stream(stream))
    if st == VKS_ERR_CAPACITY and not raise_capacity:
        return -int(m.value)
    _check("vks_bin_sort", st)
    return int(m.value)


def vks_bin_sort_async(cam, means2d, radii, depths, tiles_touched, offsets, vals, tile_offsets, workspace,
                       num_isects, status, tile_order=None, stream=None):
    """Host-sync-free binning (include/vks.h): capacity = vals.numel(); M and the status land in the
    device tensors num_isects (int64 [1]) and status (int32 [1]); nothing is returned."""
    k = cam if isinstance(cam, VksCamera) else make_camera(cam)
    n = means2d.shape[0]
    st = _lib.vks_bin_sort_async(C.byref(k), n, _ptr(means2d, f32, "means2d"), _ptr(radii, i32, "radii"),
                                 _ptr(depths, f32, "depths"), _ptr(tiles_touched, i32, "tiles_touched"),
                                 _ptr(offsets, u32, "offsets"), vals.numel(), _ptr(vals, u32, "vals"),
                                 _ptr(tile_offsets, u32, "tile_offsets"), _ptr(tile_order, u32, "tile_order"),
                                 _ptr(num_isects, torch.int64, "num_isects"), _ptr(status, i32, "status"),
                                 _ptr(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream))
    _check("vks_bin_sort_async", st)


def vks_bin_sort_check(cam, means2d, radii, depths, vals, tile_offsets, num_isects, stream=None) -> int:
    """Debug verification of a binning (include/vks.h): returns the status (VKS_OK or
    VKS_ERR_UNSORTED) instead of raising on it; other failures raise."""
    k = cam if isinstance(cam, VksCamera) else make_camera(cam)
    st = _lib.vks_bin_sort_check(C.byref(k), means2d.shape[0], _ptr(means2d, f32, "means2d"), _ptr(radii, i32, "radii"),
                                 _ptr(depths, f32, "depths"), _ptr(vals, u32, "vals"),
                                 _ptr(tile_offsets, u32, "tile_offsets"), int(num_isects), _stream(stream))
    if st not in (VKS_OK, VKS_ERR_UNSORTED):
        _check("vks_bin_sort_check", st)
    return st


def vks_raster_fwd(cfg, cam, means2d, conics, colors, opacities, radii, vals, tile_offsets, image, T_final,
                   n_contrib, stream=None, tile_order=None, records=None):
    """records (optional): vks_project_fwd's packed raster records; when given, the kernel stages
    them with cp.async instead of gathering the separate arrays (same results)."""
    c, k = _cfgcam(cfg, cam)
    st = _lib.vks_raster_fwd(C.byref(c), C.byref(k), means2d.shape[0], _ptr(means2d, f32, "means2d"),
                             _ptr(conics, f32, "conics"), _ptr(colors, f32, "colors"),
                             _ptr(opacities, f32, "opacities"), _ptr(radii, i32, "radii"),
                             _ptr(records, f32, "records"), _ptr(vals, u32, "vals"),
                             _ptr(tile_offsets, u32, "tile_offsets"), _ptr(tile_order, u32, "tile_order"),
                             _ptr(image, f32, "image"),
                             _ptr(T_final, f32, "T_final"), _ptr(n_contrib, i32, "n_contrib"),
                             _stream(stream))
    _check("vks_raster_fwd", st)


def vks_raster_fwd_stats(cfg, cam, means2d, conics, colors, opacities, radii, vals, tile_offsets, stats, stream=None,
                         tile_order=None, records=None):
    """Diagnostic: accumulate [visited, composited, evaluated, replayed, warp_entries,
    warp_entries_composited] counts into the int64 CUDA tensor `stats` (6 entries)."""
    if stats.numel() < 6:
        raise ValueError("stats needs 6 int64 entries")
    c, k = _cfgcam(cfg, cam)
    st = _lib.vks_raster_fwd_stats(C.byref(c), C.byref(k), means2d.shape[0], _ptr(means2d, f32, "means2d"),
                                   _ptr(conics, f32, "conics"), _ptr(colors, f32, "colors"),
                                   _ptr(opacities, f32, "opacities"), _ptr(radii, i32, "radii"),
                                   _ptr(records, f32, "records"), _ptr(vals, u32, "vals"),
                                   _ptr(tile_offsets, u32, "tile_offsets"), _ptr(tile_order, u32, "tile_order"),
                                   _ptr(stats, torch.int64, "stats"),
                                   _stream(stream))
    _check("vks_raster_fwd_stats", st)


def vks_raster_bwd(cfg, cam, means2d, conics, colors, opacities, radii, vals, tile_offsets, T_final, n_contrib,
                   dL_dimage, dmeans2d, dconics, dcolors, dopacities, stream=None, tile_order=None, records=None):
    c, k = _cfgcam(cfg, cam)
    st = _lib.vks_raster_bwd(C.byref(c), C.byref(k), means2d.shape[0], _ptr(means2d, f32, "means2d"),
                             _ptr(conics, f32, "conics"), _ptr(colors, f32, "colors"),
                             _ptr(opacities, f32, "opacities"), _ptr(radii, i32, "radii"),
                             _ptr(records, f32, "records"), _ptr(vals, u32, "vals"),
                             _ptr(tile_offsets, u32, "tile_offsets"), _ptr(tile_order, u32, "tile_order"),
                             _ptr(T_final, f32, "T_final"),
                             _ptr(n_contrib, i32, "n_contrib"), _ptr(dL_dimage, f32, "dL_dimage"),
                             _ptr(dmeans2d, f32, "dmeans2d"), _ptr(dconics, f32, "dconics"),
                             _ptr(dcolors, f32, "dcolors"), _ptr(dopacities, f32, "dopacities"),
                             _stream(stream))
    _check("vks_raster_bwd", st)


def vks_project_bwd(cfg, cam, means, log_scales, quats, opacity_logits, sh, colors, radii, dmeans2d, dconics,
                    dcolors, dopacities, dmeans, dlog_scales, dquats, dopacity_logits, dsh, stream=None):
    c, k = _cfgcam(cfg, cam)
    st = _lib.vks_project_bwd(C.byref(c), C.byref(k), means.shape[0], _ptr(means, f32, "means"),
                              _ptr(log_scales, f32, "log_scales"), _ptr(quats, f32, "quats"),
                              _ptr(opacity_logits, f32, "opacity_logits"), _ptr(sh, f32, "sh"),
                              _ptr(colors, f32, "colors"), _ptr(radii, i32, "radii"), _ptr(dmeans2d, f32, "dmeans2d"),
                              _ptr(dconics, f32, "dconics"), _ptr(dcolors, f32, "dcolors"),
                              _ptr(dopacities, f32, "dopacities"), _ptr(dmeans, f32, "dmeans"),
                              _ptr(dlog_scales, f32, "dlog_scales"), _ptr(dquats, f32, "dquats"),
                              _ptr(dopacity_logits, f32, "dopacity_logits"), _ptr(dsh, f32, "dsh"),
                              _stream(stream))
    _check("vks_project_bwd", st)


def vks_project_fwd_batch(cfg, cams, means, log_scales, quats, opacity_logits, sh, means2d, conics, depths, radii,
                          tiles_touched, colors, opacities, g2d_zero=None, stream=None, records=None):
    """Batched projection forward: `cams` and the per-view outputs (means2d, conics, depths, radii,
    tiles_touched, colors) are equal-length sequences; `opacities` is one tensor for the batch;
    g2d_zero (optional): per view a [9n] fp32 tensor of 2D-gradient accumulators to zero;
    records (optional): per view an fp32 [n, 12] tensor receiving the packed raster records."""
    nv = len(cams)
    per_view = (means2d, conics, depths, radii, tiles_touched, colors)
    if any(len(x) != nv for x in per_view):
        raise ValueError("per-view sequences must all have len(cams) entries")
    c = make_config(cfg) if isinstance(cfg, dict) else cfg
    karr = (VksCamera * max(nv, 1))(*[k if isinstance(k, VksCamera) else make_camera(k) for k in cams])
    dts = (f32, f32, f32, i32, i32, f32)
    names = ("means2d", "conics", "depths", "radii", "tiles_touched", "colors")
    arrs = [(C.c_void_p * max(nv, 1))(*[_ptr(t, dt, nm) for t in seq]) for seq, dt, nm in zip(per_view, dts, names)]
    # (conics may be a sequence of None when records are written)
    st = _lib.vks_project_fwd_batch(C.byref(c), nv, karr, means.shape[0], _ptr(means, f32, "means"),
                                    _ptr(log_scales, f32, "log_scales"), _ptr(quats, f32, "quats"),
                                    _ptr(opacity_logits, f32, "opacity_logits"), _ptr(sh, f32, "sh"), *arrs,
                                    _ptr(opacities, f32, "opacities"),
                                    None if g2d_zero is None else (C.c_void_p * max(nv, 1))(
                                        *[_ptr(t, f32, "g2d_zero") for t in g2d_zero]),
                                    None if records is None else (C.c_void_p * max(nv, 1))(
                                        *[_ptr(t, f32, "records") for t in records]),
                                    _stream(stream))
    _check("vks_project_fwd_batch", st)


def vks_project_bwd_batch(cfg, cams, means, log_scales, quats, opacity_logits, sh, colors, radii, dmeans2d,
                          dconics, dcolors, dopacities, dmeans, dlog_scales, dquats, dopacity_logits, dsh,
                          stream=None):
    """Batched projection backward: `cams` and the per-view tensors (colors, radii, dmeans2d,
    dconics, dcolors, dopacities) are equal-length sequences, one entry per view."""
    nv = len(cams)
    per_view = (colors, radii, dmeans2d, dconics, dcolors, dopacities)
    if any(len(x) != nv for x in per_view):
        raise ValueError("per-view sequences must all have len(cams) entries")
    c = make_config(cfg) if isinstance(cfg, dict) else cfg
    karr = (VksCamera * max(nv, 1))(*[k if isinstance(k, VksCamera) else make_camera(k) for k in cams])
    dts = (f32, i32, f32, f32, f32, f32)
    names = ("colors", "radii", "dmeans2d", "dconics", "dcolors", "dopacities")
    arrs = [(C.c_void_p * max(nv, 1))(*[_ptr(t, dt, nm) for t in seq]) for seq, dt, nm in zip(per_view, dts, names)]
    st = _lib.vks_project_bwd_batch(C.byref(c), nv, karr, means.shape[0], _ptr(means, f32, "means"),
                                    _ptr(log_scales, f32, "log_scales"), _ptr(quats, f32, "quats"),
                                    _ptr(opacity_logits, f32, "opacity_logits"), _ptr(sh, f32, "sh"),
                                    *arrs, _ptr(dmeans, f32, "dmeans"), _ptr(dlog_scales, f32, "dlog_scales"),
                                    _ptr(dquats, f32, "dquats"), _ptr(dopacity_logits, f32, "dopacity_logits"),
                                    _ptr(dsh, f32, "dsh"), _stream(stream))
    _check("vks_project_bwd_batch", st)


def vks_adam_step(acfg, params, grads, m, v, stream=None):
    """Adam step: params / grads / m / v are 5-sequences of fp32 tensors in
    ADAM_GROUPS order (means [n,3], log_scales [n,3], quats [n,4], opacity_logits [n],
    sh [n,K,3]); params, m and v are updated in place.  acfg: VksAdamConfig or a dict of
    make_adam_config's keyword arguments."""
    a = acfg if isinstance(acfg, VksAdamConfig) else make_adam_config(**acfg)
    seqs = (params, grads, m, v)
    if any(len(x) != 5 for x in seqs):
        raise ValueError("params, grads, m, v: one tensor per parameter group (5)")
    n, K = params[0].shape[0], params[4].shape[1]
    for seq in seqs:
        for q, t in enumerate(seq):
            rows = (3, 3, 4, 1, 3 * K)[q]
            if t.numel() != n * rows:
                raise ValueError(f"group {ADAM_GROUPS[q]}: expected {n * rows} elements, got {t.numel()}")
    arrs = [(C.c_void_p * 5)(*[_ptr(t, f32, f"{nm}[{ADAM_GROUPS[q]}]") for q, t in enumerate(seq)])
            for seq, nm in zip(seqs, ("params", "grads", "m", "v"))]
    st = _lib.vks_adam_step(C.byref(a), n, K, *arrs, _stream(stream))
    _check("vks_adam_step", st)


def vks_loss_workspace_bytes(width: int, height: int) -> int:
    return int(_lib.vks_loss_workspace_bytes(int(width), int(height)))


def vks_loss_grad(render, target, dL_dimage, loss, workspace, lam=0.2, stream=None):
    """Loss gradient: render / target / dL_dimage [H, W, 3] fp32 device tensors,
    loss a 1-element fp32 device tensor (or None), workspace a uint8 device tensor of at least
    vks_loss_workspace_bytes(W, H) bytes."""
    H, W = render.shape[0], render.shape[1]
    for t, nm in ((render, "render"), (target, "target"), (dL_dimage, "dL_dimage")):
        if tuple(t.shape) != (H, W, 3):
            raise ValueError(f"{nm}: expected shape {(H, W, 3)}, got {tuple(t.shape)}")
    st = _lib.vks_loss_grad(W, H, float(lam), _ptr(render, f32, "render"), _ptr(target, f32, "target"),
                            _ptr(dL_dimage, f32, "dL_dimage"), _ptr(loss, f32, "loss"),
                            _ptr(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream))
    _check("vks_loss_grad", st)


def vks_mcmc_workspace_bytes(n: int) -> int:
    return int(_lib.vks_mcmc_workspace_bytes(int(n)))


def vks_mcmc_relocate(params, workspace, dead_opacity=0.005, seed=0, m=None, v=None, targets=None, n_dead=None,
                      stream=None):
    """MCMC relocation: params = GaussianParams-like (means, log_scales, quats,
    opacity_logits, sh tensors, updated in place); m, v: 5-sequences of Adam moment tensors (or
    None); targets: int64 [n] device tensor (or None); n_dead: int64 [1] device tensor (or None)."""
    n, K = params.means.shape[0], params.sh.shape[1]
    if (m is None) != (v is None):
        raise ValueError("pass both m and v, or neither")
    ma = None if m is None else (C.c_void_p * 5)(*[_ptr(t, f32, "m") for t in m])
    va = None if v is None else (C.c_void_p * 5)(*[_ptr(t, f32, "v") for t in v])
    st = _lib.vks_mcmc_relocate(n, K, float(dead_opacity), int(seed), _ptr(params.means, f32, "means"),
                                _ptr(params.log_scales, f32, "log_scales"), _ptr(params.quats, f32, "quats"),
                                _ptr(params.opacity_logits, f32, "opacity_logits"), _ptr(params.sh, f32, "sh"), ma, va,
                                _ptr(targets, torch.int64, "targets"), _ptr(n_dead, torch.int64, "n_dead"),
                                _ptr(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream))
    _check("vks_mcmc_relocate", st)


def vks_mcmc_noise(params, lr_pos, noise_scale, seed=0, step=0, stream=None):
    """Positional noise after an optimizer step: params.means updated in place."""
    st = _lib.vks_mcmc_noise(params.means.shape[0], float(lr_pos), float(noise_scale), int(seed), int(step),
                             _ptr(params.means, f32, "means"), _ptr(params.log_scales, f32, "log_scales"),
                             _ptr(params.quats, f32, "quats"), _ptr(params.opacity_logits, f32, "opacity_logits"),
                             _stream(stream))
    _check("vks_mcmc_noise", st)


def vks_densify_stats(dmeans2d, radii, accum, denom, stream=None):
    """Screen-gradient statistics of one view: accum / denom updated in place."""
    st = _lib.vks_densify_stats(accum.shape[0], _ptr(dmeans2d, f32, "dmeans2d"), _ptr(radii, i32, "radii"),
                                _ptr(accum, f32, "accum"), _ptr(denom, f32, "denom"), _stream(stream))
    _check("vks_densify_stats", st)


def vks_densify_workspace_bytes(n: int) -> int:
    return int(_lib.vks_densify_workspace_bytes(int(n)))


def vks_densify(params, accum, denom, out_params, workspace, grad_threshold, size_threshold, prune_opacity=0.005,
                seed=0, m=None, v=None, out_m=None, out_v=None, stream=None) -> int:
    """One densification event.  params / out_params (/ m, v, out_m, out_v):
    5-sequences of fp32 tensors in ADAM_GROUPS order; the outputs' first dimension is the capacity.
    Returns n'; raises VksError(VKS_ERR_CAPACITY) when n' exceeds it (VksError.n_out holds n')."""
    n, K = params[0].shape[0], params[4].shape[1]
    cap = out_params[0].shape[0]
    arr = lambda seq, nm: None if seq is None else (C.c_void_p * 5)(*[_ptr(t, f32, nm) for t in seq])  # noqa: E731
    n_out = C.c_int64(0)
    st = _lib.vks_densify(n, K, arr(params, "params"), arr(m, "m"), arr(v, "v"), _ptr(accum, f32, "accum"),
                          _ptr(denom, f32, "denom"), float(grad_threshold), float(size_threshold),
                          float(prune_opacity), int(seed), cap, arr(out_params, "out_params"), arr(out_m, "out_m"),
                          arr(out_v, "out_v"), C.byref(n_out), _ptr(workspace, torch.uint8, "workspace"),
                          workspace.numel(), _stream(stream))
    if st != VKS_OK:
        err = VksError("vks_densify", st)
        err.n_out = int(n_out.value)
        raise err
    return int(n_out.value)


def vks_version() -> int:
    return int(_lib.vks_version())


def exported_symbols():
    """Names of include/vks.h entry points resolvable in the loaded library."""
    return [name for name in EXPORTS if hasattr(_lib, name)]
