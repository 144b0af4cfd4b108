"""CPU-only checks of the C-ABI library: it loads, exports every entry point include/vks.h declares,
validates arguments synchronously, and has no CPU fallback (no compute without a GPU)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "vks.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vks_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2605_00219_b200 as P
    lib = C.CDLL(os.path.join(ROOT, "paper_2605_00219_b200", "libvks.so"))
    syms = header_symbols()
    assert len(syms) >= 9
    for s in syms:
        assert hasattr(lib, s), s
    assert set(P.EXPORTS) == set(syms)
    assert P.vks_version() == 1


def test_no_unresolved_library_symbols():
    """Every launcher the entry points call is defined in the library (a declaration / definition
    mismatch would otherwise only surface as an undefined symbol at load time on the GPU box)."""
    import shutil
    import subprocess
    nm = shutil.which("nm")
    if not nm:
        pytest.skip("nm not available")
    out = subprocess.run([nm, "-D", "--undefined-only", "-C", os.path.join(ROOT, "paper_2605_00219_b200", "libvks.so")],
                         capture_output=True, text=True).stdout
    assert "vks::" not in out and "vks_" not in out, out


def test_cuda_objects_are_sm100a():
    """The library carries sm_100a SASS (cuobjdump lists the ELF arch)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", os.path.join(ROOT, "paper_2605_00219_b200", "libvks.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _lib():
    from paper_2605_00219_b200 import _vks
    return _vks._lib, _vks


def test_status_strings_and_workspace():
    lib, V = _lib()
    for st in range(6):
        assert lib.vks_status_string(st)
    assert V.vks_bin_sort_workspace_bytes(1000, 5000, 16) > 5000 * 12
    assert V.vks_bin_sort_workspace_bytes(-1, 10, 16) == 0
    assert V.vks_bin_sort_workspace_bytes(10, 10, 0) == 0


def test_argument_validation_is_synchronous():
    lib, V = _lib()
    cfg = V.make_config(dict(sh_degree=3, sh_coeffs=16))
    cam = V.make_camera(dict(R=[1, 0, 0, 0, 1, 0, 0, 0, 1], t=[0, 0, 0], fx=100, fy=100, cx=32, cy=32,
                             width=64, height=64))
    # null camera / negative n / bad degree / bad footprint -> errors before any CUDA call
    assert lib.vks_project_fwd(C.byref(cfg), None, 0, *([None] * 14)) == V.VKS_ERR_INVALID_ARG
    assert lib.vks_project_fwd(C.byref(cfg), C.byref(cam), -1, *([None] * 14)) == V.VKS_ERR_INVALID_ARG
    bad = V.make_config(dict(sh_degree=4, sh_coeffs=25))
    assert lib.vks_project_fwd(C.byref(bad), C.byref(cam), 0, *([None] * 14)) == V.VKS_ERR_UNSUPPORTED
    bad = V.make_config(dict(sh_degree=3, sh_coeffs=9))
    assert lib.vks_project_fwd(C.byref(bad), C.byref(cam), 0, *([None] * 14)) == V.VKS_ERR_INVALID_ARG
    bad = V.make_config(dict(sh_degree=3, sh_coeffs=16, footprint=7))
    assert lib.vks_raster_fwd(C.byref(bad), C.byref(cam), 0, *([None] * 13)) == V.VKS_ERR_UNSUPPORTED
    wide = V.make_camera(dict(R=[1, 0, 0, 0, 1, 0, 0, 0, 1], t=[0, 0, 0], fx=100, fy=100, cx=32, cy=32,
                              width=70000, height=64))
    assert lib.vks_raster_bwd(C.byref(cfg), C.byref(wide), 0, *([None] * 17)) == V.VKS_ERR_INVALID_ARG
    arr = (C.c_void_p * 1)(None)
    cams = (V.VksCamera * 1)(cam)
    for nv in (0, 17):  # batch size outside [1, 16]
        assert lib.vks_project_bwd_batch(C.byref(cfg), nv, cams, 0, *([None] * 5), *([arr] * 6),
                                         *([None] * 5), None) == V.VKS_ERR_INVALID_ARG
    # Adam: step < 1, beta outside [0, 1), sh_coeffs outside [1, 64], unaligned pointer
    five = (C.c_void_p * 5)(*([256] * 5))
    a = V.make_adam_config([1e-3] * 6, step=0)
    assert lib.vks_adam_step(C.byref(a), 4, 16, five, five, five, five, None) == V.VKS_ERR_INVALID_ARG
    a = V.make_adam_config([1e-3] * 6, beta1=1.0)
    assert lib.vks_adam_step(C.byref(a), 4, 16, five, five, five, five, None) == V.VKS_ERR_INVALID_ARG
    a = V.make_adam_config([1e-3] * 6)
    assert lib.vks_adam_step(C.byref(a), 4, 65, five, five, five, five, None) == V.VKS_ERR_INVALID_ARG
    odd = (C.c_void_p * 5)(*([256] * 4 + [260]))
    assert lib.vks_adam_step(C.byref(a), 4, 16, five, odd, five, five, None) == V.VKS_ERR_INVALID_ARG
    # loss gradient: SSIM needs 11x11 images, lambda in [0, 1], workspace size
    P = C.c_void_p(256)
    assert lib.vks_loss_grad(10, 64, C.c_float(0.2), P, P, P, None, P, 1 << 30, None) == V.VKS_ERR_INVALID_ARG
    assert lib.vks_loss_grad(64, 64, C.c_float(1.5), P, P, P, None, P, 1 << 30, None) == V.VKS_ERR_INVALID_ARG
    assert lib.vks_loss_grad(64, 64, C.c_float(0.2), P, P, P, None, P, 16, None) == V.VKS_ERR_WORKSPACE
    # one fp64 42x42 partial slot per 32x32 centre tile and channel: > 3 x 8 B per valid centre
    assert lib.vks_loss_workspace_bytes(1237, 822) > 3 * 8 * 1227 * 812
    # MCMC: dead_opacity outside [0, 1), only one of m / v, workspace too small
    assert lib.vks_mcmc_relocate(4, 16, C.c_float(1.0), 0, *([P] * 5), None, None, None, None, P, 1 << 20,
                                 None) == V.VKS_ERR_INVALID_ARG
    assert lib.vks_mcmc_relocate(4, 16, C.c_float(0.005), 0, *([P] * 5), five, None, None, None, P, 1 << 20,
                                 None) == V.VKS_ERR_INVALID_ARG
    assert lib.vks_mcmc_relocate(4, 16, C.c_float(0.005), 0, *([P] * 5), None, None, None, None, P, 8,
                                 None) == V.VKS_ERR_WORKSPACE
    m = C.c_int64(0)
    assert lib.vks_bin_sort(C.byref(cam), 5, *([None] * 5), 0, *([None] * 4), None, None, C.byref(m), None, 0,
                            None) == V.VKS_ERR_INVALID_ARG
    # async binning: device M / status words required, capacity below 2^30
    assert lib.vks_bin_sort_async(C.byref(cam), 0, *([None] * 5), 0, *([None] * 3), None, None, P, 1 << 20,
                                  None) == V.VKS_ERR_INVALID_ARG


def test_no_cpu_fallback():
    """Without a CUDA device a well-formed call reports VKS_ERR_CUDA instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib, V = _lib()
    cfg = V.make_config(dict(sh_degree=3, sh_coeffs=16))
    cam = V.make_camera(dict(R=[1, 0, 0, 0, 1, 0, 0, 0, 1], t=[0, 0, 0], fx=100, fy=100, cx=32, cy=32,
                             width=64, height=64))
    st = lib.vks_raster_fwd(C.byref(cfg), C.byref(cam), 0, None, None, None, None, None, None, None, C.c_void_p(16),
                            None, C.c_void_p(16), C.c_void_p(16), C.c_void_p(16), None)
    assert st == V.VKS_ERR_CUDA
    assert b"no CUDA device" in lib.vks_last_cuda_error()


def test_binding_rejects_host_tensors():
    import torch
    import paper_2605_00219_b200 as P
    x = torch.zeros(4, 3)
    with pytest.raises((ValueError, TypeError)):
        P.vks_project_fwd(dict(sh_degree=0), dict(R=[1, 0, 0, 0, 1, 0, 0, 0, 1], t=[0, 0, 0], fx=1, fy=1,
                                                   cx=0, cy=0, width=4, height=4),
                          x, x, torch.zeros(4, 4), torch.zeros(4), torch.zeros(4, 1, 3), *([x] * 7))
