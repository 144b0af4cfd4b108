"""vks_bin_sort_async (include/vks.h) on the GPU: the host-sync-free binning gives the same tile
lists, offsets and M as vks_bin_sort (which P2 pins bit-exactly to the oracle, tests/
test_gpu_parity.py), reports overflow through its device status word with every list emptied,
handles empty scenes, and runs inside a captured CUDA graph."""
import numpy as np
import pytest

import synth
from gpu_helpers import to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _project(scene, cam, cfg):
    import paper_2605_00219_b200 as P
    params = P.GaussianParams.from_host(scene)
    r = P.ViewRenderer(params.n, cam["width"], cam["height"])
    r.forward(cfg, cam, params)  # the synchronous binning (P2-pinned) into r.vals / r.tile_offsets
    return params, r


def _async(r, cam, capacity=None, stream=None):
    import torch
    import paper_2605_00219_b200 as P
    cap = capacity if capacity is not None else r.capacity
    vals = torch.empty(cap, dtype=torch.uint32, device="cuda")
    tile_offsets = torch.empty(r.n_tiles + 1, dtype=torch.uint32, device="cuda")
    tile_order = torch.empty(r.n_tiles, dtype=torch.uint32, device="cuda")
    offsets = torch.empty(r.n, dtype=torch.uint32, device="cuda")
    ws = torch.empty(P.vks_bin_sort_workspace_bytes(r.n, cap, r.n_tiles), dtype=torch.uint8, device="cuda")
    m = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    st = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    P.vks_bin_sort_async(cam, r.means2d, r.radii, r.depths, r.tiles, offsets, vals, tile_offsets, ws, m, st,
                         tile_order=tile_order, stream=stream)
    return dict(vals=vals, tile_offsets=tile_offsets, tile_order=tile_order, offsets=offsets, m=m, st=st, ws=ws)


@pytest.mark.parametrize("name,view", [("tiny", 0), ("mcmc", 3), ("bicycle", 0)])
def test_async_equals_sync(name, view):
    """Same M, index offsets, tile ranges and sorted ids as the synchronous binning; the tile schedule
    is a permutation of the tiles (its order within a length class is arbitrary)."""
    import torch
    c = synth.CONFIGS[name]
    scene = synth.make_scene(c.n, c.kind, c.seed)
    cam = synth.ring_cameras(c.width, c.height, c.kind, 8)[view]
    cfg = synth.default_render_config()
    _, r = _project(scene, cam, cfg)
    a = _async(r, cam)
    torch.cuda.synchronize()
    m = r.num_isects
    assert int(a["st"].item()) == 0 and int(a["m"].item()) == m
    assert np.array_equal(to_np(a["offsets"]), to_np(r.offsets))
    assert np.array_equal(to_np(a["tile_offsets"]), to_np(r.tile_offsets))
    assert np.array_equal(to_np(a["vals"][:m]), to_np(r.vals[:m]))
    assert np.array_equal(np.sort(to_np(a["tile_order"])), np.arange(r.n_tiles, dtype=np.uint32))


def test_async_overflow_reports_and_empties_lists():
    """capacity < M: status VKS_ERR_CAPACITY, M reported, every tile list empty (tile_offsets 0), and
    nothing written past the capacity."""
    import torch
    import paper_2605_00219_b200 as P
    c = synth.CONFIGS["tiny"]
    scene = synth.make_scene(c.n, c.kind, c.seed)
    cam = synth.ring_cameras(c.width, c.height, c.kind, 8)[0]
    _, r = _project(scene, cam, synth.default_render_config())
    m = r.num_isects
    cap = m // 2
    a = _async(r, cam, capacity=cap)
    torch.cuda.synchronize()
    assert int(a["st"].item()) == P.VKS_ERR_CAPACITY and int(a["m"].item()) == m
    assert not to_np(a["tile_offsets"]).any()


def test_async_empty_scene():
    """Every Gaussian behind the camera: M = 0, status ok, empty lists."""
    import torch
    c = synth.CONFIGS["tiny"]
    scene = synth.make_scene(c.n, c.kind, c.seed)
    cam = synth.ring_cameras(c.width, c.height, c.kind, 8)[0]
    cam = dict(cam, t=cam["t"] + np.array([0.0, 0.0, -1e4], np.float32))  # the scene behind the camera
    _, r = _project(scene, cam, synth.default_render_config())
    assert r.num_isects == 0
    a = _async(r, cam, capacity=1024)
    torch.cuda.synchronize()
    assert int(a["st"].item()) == 0 and int(a["m"].item()) == 0
    assert not to_np(a["tile_offsets"]).any()


def test_async_binning_in_a_cuda_graph():
    """The binning and both raster passes captured into one CUDA graph and replayed give the image and
    gradients of the eager calls (the launch sequence depends only on n, capacity and the camera)."""
    import torch
    import paper_2605_00219_b200 as P
    c = synth.CONFIGS["mcmc"]
    scene = synth.make_scene(200000, c.kind, c.seed)
    cam = synth.ring_cameras(640, 480, c.kind, 8)[2]
    cfg = synth.default_render_config()
    params, r = _project(scene, cam, cfg)
    dL = torch.from_numpy(synth.upstream_grad(480, 640, 3)).cuda()
    cap = int(r.num_isects * 1.25) + 1024
    s = torch.cuda.Stream()
    bufs = _async(r, cam, capacity=cap, stream=s)  # allocates (outside the capture)
    image, T, nc = torch.empty_like(r.image), torch.empty_like(r.T_final), torch.empty_like(r.n_contrib)
    g2d = torch.zeros(9 * params.n, device="cuda")

    def body():
        P.vks_bin_sort_async(cam, r.means2d, r.radii, r.depths, r.tiles, bufs["offsets"], bufs["vals"],
                             bufs["tile_offsets"], bufs["ws"], bufs["m"], bufs["st"], tile_order=bufs["tile_order"])
        P.vks_raster_fwd(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, bufs["vals"],
                         bufs["tile_offsets"], image, T, nc, tile_order=bufs["tile_order"], records=r.records)
        g2d.zero_()
        n = params.n
        P.vks_raster_bwd(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, bufs["vals"],
                         bufs["tile_offsets"], T, nc, dL, g2d[:2 * n].view(n, 2), g2d[2 * n:5 * n].view(n, 3),
                         g2d[5 * n:8 * n].view(n, 3), g2d[8 * n:], tile_order=bufs["tile_order"], records=r.records)

    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        body()  # eager, on the capture stream
    torch.cuda.synchronize()
    ref_img, ref_g = image.clone(), g2d.clone()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        body()
    image.zero_()
    g2d.fill_(float("nan"))
    graph.replay()
    torch.cuda.synchronize()
    assert int(bufs["st"].item()) == 0
    assert torch.equal(image, ref_img)
    scale = ref_g.abs().max().item()
    assert torch.allclose(g2d, ref_g, rtol=1e-4, atol=1e-6 * scale)
