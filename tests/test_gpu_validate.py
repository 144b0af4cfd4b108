"""VKS_FLAG_VALIDATE and vks_bin_sort_check (SURVEY §8(b) "Errors"; include/vks.h), through the C ABI:
SPEC S:119 NonFiniteParameter -> VKS_ERR_NONFINITE, S:52 ZeroQuaternion -> VKS_ERR_NONFINITE,
S:155 UnsortedInput -> VKS_ERR_UNSORTED; the M >= 2^30 hard limit -> VKS_ERR_UNSUPPORTED.  Clean
inputs pass and give bit-identical outputs with and without the flag."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_00219_b200 as P
    return P


def _tiny():
    c = synth.CONFIGS["tiny"]
    scene = synth.make_scene(c.n, c.kind, c.seed)
    cam = synth.ring_cameras(c.width, c.height, c.kind, 8)[0]
    dL = synth.upstream_grad(c.height, c.width, c.seed + 1000)
    return scene, cam, dL


def _render(P, scene, cam, cfg):
    params = P.GaussianParams.from_host(scene)
    r = P.ViewRenderer(params.n, cam["width"], cam["height"])
    r.forward(cfg, cam, params)
    return params, r


def test_validate_clean_inputs_pass_and_match(P):
    import torch
    scene, cam, dL = _tiny()
    cfg = synth.default_render_config()
    cfg_v = dict(cfg, flags=P.FLAG_VALIDATE)
    p0, r0 = _render(P, scene, cam, cfg)
    p1, r1 = _render(P, scene, cam, cfg_v)
    for k in ("image", "T_final", "n_contrib", "radii", "means2d"):
        assert torch.equal(getattr(r0, k), getattr(r1, k)), k
    dLt = torch.from_numpy(dL).cuda()
    r0.backward(cfg, cam, p0, dLt)
    r1.backward(cfg_v, cam, p1, dLt)
    torch.cuda.synchronize()
    # gradients: same computation, fp32 atomics sum in a run-dependent order
    for a, b in ((r0.g2d, r1.g2d), (p0.grad_flat, p1.grad_flat)):
        assert torch.allclose(a, b, rtol=1e-4, atol=1e-6 * float(a.abs().max()))
    assert P.vks_bin_sort_check(cam, r1.means2d, r1.radii, r1.depths, r1.vals, r1.tile_offsets,
                                r1.num_isects) == P.VKS_OK


@pytest.mark.parametrize("field,index,value", [("means", (5, 1), np.nan), ("log_scales", (9, 2), np.inf),
                                               ("quats", (3,), 0.0), ("opacity_logits", (7,), -np.inf),
                                               ("sh", (11, 15, 2), np.nan)])
def test_validate_nonfinite_parameters(P, field, index, value):
    import torch
    scene, cam, _ = _tiny()
    bad = {k: v.copy() for k, v in scene.items()}
    bad[field][index] = value  # quats row 3 = 0: a zero quaternion
    params = P.GaussianParams.from_host(bad)
    r = P.ViewRenderer(params.n, cam["width"], cam["height"])
    cfg = synth.default_render_config()
    r.means2d.fill_(123.0)
    with pytest.raises(P.VksError) as ei:
        P.vks_project_fwd(dict(cfg, flags=P.FLAG_VALIDATE), cam, params.means, params.log_scales, params.quats,
                          params.opacity_logits, params.sh, r.means2d, r.conics, r.depths, r.radii, r.tiles,
                          r.colors, r.opacities)
    assert ei.value.status == P.VKS_ERR_NONFINITE
    torch.cuda.synchronize()
    assert bool((r.means2d == 123.0).all())  # nothing written
    # without the flag the Gaussian is culled, never an error
    P.vks_project_fwd(cfg, cam, params.means, params.log_scales, params.quats, params.opacity_logits, params.sh,
                      r.means2d, r.conics, r.depths, r.radii, r.tiles, r.colors, r.opacities)
    torch.cuda.synchronize()
    assert int(r.tiles[index[0]].item()) == 0
    # the batched projection checks the same
    with pytest.raises(P.VksError) as ei:
        P.vks_project_fwd_batch(dict(cfg, flags=P.FLAG_VALIDATE), [cam], params.means, params.log_scales,
                                params.quats, params.opacity_logits, params.sh, [r.means2d], [r.conics], [r.depths],
                                [r.radii], [r.tiles], [r.colors], r.opacities)
    assert ei.value.status == P.VKS_ERR_NONFINITE


def test_validate_nonfinite_gradients(P):
    import torch
    scene, cam, dL = _tiny()
    cfg = synth.default_render_config()
    cfg_v = dict(cfg, flags=P.FLAG_VALIDATE)
    params, r = _render(P, scene, cam, cfg)
    bad = dL.copy()
    bad[10, 20, 1] = np.nan
    r.g2d.zero_()
    with pytest.raises(P.VksError) as ei:
        P.vks_raster_bwd(cfg_v, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals, r.tile_offsets,
                         r.T_final, r.n_contrib, torch.from_numpy(bad).cuda(), r.dmeans2d, r.dconics, r.dcolors,
                         r.dopacities)
    assert ei.value.status == P.VKS_ERR_NONFINITE
    torch.cuda.synchronize()
    assert not bool(r.g2d.any())  # nothing accumulated
    P.vks_raster_bwd(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals, r.tile_offsets,
                     r.T_final, r.n_contrib, torch.from_numpy(dL).cuda(), r.dmeans2d, r.dconics, r.dcolors,
                     r.dopacities)
    r.dconics[17, 1] = float("inf")
    g = params.grads()
    with pytest.raises(P.VksError) as ei:
        P.vks_project_bwd(cfg_v, cam, params.means, params.log_scales, params.quats, params.opacity_logits,
                          params.sh, r.colors, r.radii, r.dmeans2d, r.dconics, r.dcolors, r.dopacities, g["dmeans"],
                          g["dlog_scales"], g["dquats"], g["dopacity_logits"], g["dsh"])
    assert ei.value.status == P.VKS_ERR_NONFINITE


def test_bin_sort_check_detects_unsorted_lists(P):
    import torch
    scene, cam, _ = _tiny()
    cfg = synth.default_render_config()
    _, r = _render(P, scene, cam, cfg)
    m = r.num_isects
    args = (cam, r.means2d, r.radii, r.depths)
    assert P.vks_bin_sort_check(*args, r.vals, r.tile_offsets, m) == P.VKS_OK
    to = r.tile_offsets.view(torch.int32).cpu().numpy().view(np.uint32).astype(np.int64)
    t = int(np.argmax(np.diff(to)))  # the longest list
    b = int(to[t])
    def i32(x):  # uint32 tensors edited through their int32 view
        return x.clone().view(torch.int32)

    # two entries of a tile swapped: out of (depth, id) order
    v = i32(r.vals)
    v[b], v[b + 1] = v[b + 1].clone(), v[b].clone()
    assert P.vks_bin_sort_check(*args, v.view(torch.uint32), r.tile_offsets, m) == P.VKS_ERR_UNSORTED
    # an id out of range
    v = i32(r.vals)
    v[b] = scene["means"].shape[0] + 5
    assert P.vks_bin_sort_check(*args, v.view(torch.uint32), r.tile_offsets, m) == P.VKS_ERR_UNSORTED
    # a CSR that decreases, and one that does not end at M
    o = i32(r.tile_offsets)
    o[t + 1] = o[t] - 1
    assert P.vks_bin_sort_check(*args, r.vals, o.view(torch.uint32), m) == P.VKS_ERR_UNSORTED
    assert P.vks_bin_sort_check(*args, r.vals, r.tile_offsets, m + 1) == P.VKS_ERR_UNSORTED
    # an entry whose Gaussian's tile rect misses its tile: that Gaussian's mean moved far off-image
    g = int(r.vals.view(torch.int32)[b].item())
    m2 = r.means2d.clone()
    m2[g] = torch.tensor([-5000.0, -5000.0], device="cuda")
    assert P.vks_bin_sort_check(cam, m2, r.radii, r.depths, r.vals, r.tile_offsets, m) == P.VKS_ERR_UNSORTED
    # the raster passes under VKS_FLAG_VALIDATE reject a corrupted CSR before compositing
    o = i32(r.tile_offsets)
    o[t + 1] = 0
    with pytest.raises(P.VksError) as ei:
        P.vks_raster_fwd(dict(cfg, flags=P.FLAG_VALIDATE), cam, r.means2d, r.conics, r.colors, r.opacities, r.radii,
                         r.vals, o.view(torch.uint32), r.image, r.T_final, r.n_contrib)
    assert ei.value.status == P.VKS_ERR_UNSORTED


def test_bin_sort_hard_limit_is_unsupported(P):
    """M >= 2^30 keys cannot be sorted at any capacity (30-bit look-back counts): the call returns
    VKS_ERR_UNSUPPORTED (not the regrow request VKS_ERR_CAPACITY) after writing M."""
    import ctypes as C
    import torch
    W, H = 2474, 1644  # 155 x 103 = 15,965 tiles
    n = 68_000         # each Gaussian covers every tile: M = 1.086e9 >= 2^30
    cam = dict(R=np.eye(3, dtype=np.float32), t=np.zeros(3, np.float32), fx=np.float32(1000.0), fy=np.float32(1000.0),
               cx=np.float32(W / 2), cy=np.float32(H / 2), width=W, height=H)
    dev = "cuda"
    means2d = torch.full((n, 2), 0.0, device=dev)
    means2d[:, 0], means2d[:, 1] = W / 2, H / 2
    radii = torch.full((n, 2), 4000, dtype=torch.int32, device=dev)
    depths = torch.linspace(1.0, 2.0, n, device=dev)
    tiles = torch.full((n,), 15965, dtype=torch.int32, device=dev)
    offsets = torch.empty(n, dtype=torch.uint32, device=dev)
    vals = torch.empty(1024, dtype=torch.uint32, device=dev)
    tile_offsets = torch.empty(15966, dtype=torch.uint32, device=dev)
    ws = torch.empty(P.vks_bin_sort_workspace_bytes(n, 1024, 15965), dtype=torch.uint8, device=dev)
    from paper_2605_00219_b200 import _vks as V
    mm = C.c_int64(0)
    st = V._lib.vks_bin_sort(C.byref(V.make_camera(cam)), n, means2d.data_ptr(), radii.data_ptr(), depths.data_ptr(),
                             tiles.data_ptr(), offsets.data_ptr(), 1024, None, vals.data_ptr(), None, None,
                             tile_offsets.data_ptr(), None, C.byref(mm), ws.data_ptr(), ws.numel(), None)
    assert st == P.VKS_ERR_UNSUPPORTED == 5
    assert mm.value == n * 15965
