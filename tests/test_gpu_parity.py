"""GPU path (through the C ABI) vs the CPU oracle — the parity gate.

  P1 projection        bit-exact on every output of visible rows, radii / tiles_touched on all rows
  P2 binning           bit-exact M, offsets, unsorted + sorted keys/vals, tile_offsets
  P3 raster forward    |image - O1| <= 1e-5 and |T - O1| <= 1e-5, last contributor exact, on
                       non-fragile pixels; zero footprint violations
  P4 raster backward   per element |g - ref| <= max(1e-3 |ref|, 1e-6) (ref = fp64 oracle), with
                       upstream dL/dimage ~ U(-1,1) zeroed on fragile pixels; cancellation-limited
                       elements (|g - ref| <= 1e-5 * sum|terms|) reported separately
  P5 projection bwd    same rule, stage-isolated (oracle fed the GPU's 2D grads) and end-to-end
Large configs (MCMC 1M, bicycle 5.8M) run in the bench's launch configuration with the oracle on
sampled rows (every 8th tile row, dL nonzero only there); binning and projection in full."""
import json
import os

import numpy as np
import pytest

import synth
from gpu_helpers import check_rule, grad_rule, to_np, last_id_from_ncontrib, run_gpu, sampled_rows, scene_for

pytestmark = pytest.mark.gpu

REPORT_DIR = os.environ.get("VKS_PARITY_REPORT")


def report(name, payload):
    if REPORT_DIR:
        os.makedirs(REPORT_DIR, exist_ok=True)
        with open(os.path.join(REPORT_DIR, f"parity_{name}.json"), "w") as f:
            json.dump(payload, f, indent=1, default=lambda o: o.tolist() if hasattr(o, "tolist") else str(o))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def check_projection(o, g, tag):
    assert np.array_equal(o["radii"], g["radii"]), tag
    assert np.array_equal(o["tiles_touched"], g["tiles_touched"]), tag
    vis = o["tiles_touched"] > 0
    for k in ("means2d", "conics", "depths", "colors", "opacities"):
        a, b = o[k][vis], g[k][vis]
        same = (a.view(np.uint32) == b.view(np.uint32))
        assert same.all(), (tag, k, int((~same).sum()), np.nonzero(~same.reshape(len(a), -1).all(1))[0][:5])
    return int(vis.sum())


def check_binning(oracle_lib, cam, g, tag):
    proj = {k: g[k] for k in ("means2d", "radii", "depths", "tiles_touched")}
    ob = oracle_lib.bin_sort(None, cam, proj)
    assert g["num_isects"] == ob["num_isects"], tag
    assert np.array_equal(g["offsets"], ob["offsets"]), tag
    if "keys_unsorted" in g:
        assert np.array_equal(g["keys_unsorted"], ob["keys_unsorted"]), tag
        assert np.array_equal(g["vals_unsorted"], ob["vals_unsorted"]), tag
    assert np.array_equal(g["keys"], ob["keys"]), tag
    assert np.array_equal(g["vals"], ob["vals"]), tag
    assert np.array_equal(g["tile_offsets"], ob["tile_offsets"]), tag
    if "tile_order" in g:  # the raster schedule: a permutation of the tiles, longest lists first
        order = g["tile_order"].astype(np.int64)
        n_tiles = len(ob["tile_offsets"]) - 1
        assert np.array_equal(np.sort(order), np.arange(n_tiles)), tag
        lens = np.diff(ob["tile_offsets"].astype(np.int64))[order]
        octave = np.where(lens > 0, np.floor(np.log2(np.maximum(lens, 1))), -1)
        assert np.all(np.diff(octave) <= 0), tag
    return ob["num_isects"]


def oracle_reference(oracle_lib, scene, cam, cfg, dL, row_mask=None):
    fwd = oracle_lib.render(cfg, cam, scene, row_mask=row_mask)
    keep = (fwd["fragile"] == 0)
    if row_mask is not None:
        keep &= row_mask.astype(bool)[:, None]
    dL_eff = (dL * keep[..., None]).astype(np.float32)
    ref = oracle_lib.full_backward(cfg, cam, scene, dL_eff, row_mask=row_mask, want_mass=True)
    return fwd, ref, dL_eff, keep


def check_raster_fwd(o, g, cam, keep, tag):
    d_img = np.abs(g["image"].astype(np.float64) - o["image"]).max(axis=2)
    d_T = np.abs(g["T_final"].astype(np.float64) - o["T_final"])
    lid = last_id_from_ncontrib(g, cam)
    bad = keep & ((d_img > 1e-5) | (d_T > 1e-5) | (lid != o["last_id"]))
    stats = dict(pixels=int(keep.sum()), fragile=int(o["fragile_pixels"]), bad=int(bad.sum()),
                 max_img=float(d_img[keep].max()) if keep.any() else 0.0,
                 max_T=float(d_T[keep].max()) if keep.any() else 0.0,
                 footprint_violations=o["footprint_violations"])
    assert o["footprint_violations"] == 0, (tag, stats)
    assert stats["bad"] == 0, (tag, stats, np.argwhere(bad)[:5])
    return stats


def check_grads(oracle_lib, scene, cam, cfg, ref, g, iso):
    """P4 on the 2D grads (mass = oracle's sum|terms|); P5 on the parameter grads end-to-end
    (mass propagated from the 2D masses) and stage-isolated (oracle chain on the GPU's 2D grads,
    mass propagated from |2D grads|)."""
    out = {}
    mass = ref["mass"]
    cols = {"dmeans2d": [0, 1], "dconics": [2, 3, 4], "dcolors": [5, 6, 7], "dopacities": [8]}
    m2d = {k: mass[:, c].reshape(ref[k].shape) for k, c in cols.items()}
    for k in cols:
        out[k] = grad_rule(g[k], ref[k], m2d[k])
    m_e2e = oracle_lib.project_bwd_mass(cfg, cam, scene, m2d)
    m_iso = oracle_lib.project_bwd_mass(cfg, cam, scene, {k: g[k] for k in cols})
    for k in ("dmeans", "dlog_scales", "dquats", "dopacity_logits", "dsh"):
        out[k] = grad_rule(g[k], ref[k], m_e2e[k])
        out[k + "_isolated"] = grad_rule(g[k], iso[k], m_iso[k])
    return out


def run_case(oracle_lib, name, scene, cam, cfg, dL, row_mask=None, capacity=None):
    g = run_gpu(scene, cam, cfg, dL=None, capacity=capacity, debug_unsorted=True)
    o_proj = oracle_lib.project_fwd(cfg, cam, scene)
    nvis = check_projection(o_proj, g, name)
    m = check_binning(oracle_lib, cam, g, name)
    fwd, ref, dL_eff, keep = oracle_reference(oracle_lib, scene, cam, cfg, dL, row_mask)
    rstats = check_raster_fwd(fwd, g, cam, keep, name)
    gb = run_gpu(scene, cam, cfg, dL=dL_eff, capacity=capacity)
    iso = oracle_lib.project_bwd(cfg, cam, scene, {k: gb[k] for k in ("dmeans2d", "dconics", "dcolors", "dopacities")})
    gstats = check_grads(oracle_lib, scene, cam, cfg, ref, gb, iso)
    rep = dict(case=name, visible=nvis, num_isects=m, raster=rstats,
               grads={k: {kk: vv for kk, vv in v.items() if kk != "bad_idx"} for k, v in gstats.items()})
    report(name, rep)
    for k, v in gstats.items():
        # P4/P5: every element passes, or is condition-limited (at most 1e-5 of the field)
        check_rule(name, k, v)
    return rep


# ------------------------------------------------------------------ configs of BASELINE.json

def test_tiny_full(oracle_lib):
    scene, cam, dL = scene_for("tiny")
    run_case(oracle_lib, "tiny", scene, cam, synth.default_render_config(), dL)


@pytest.mark.parametrize("view", [1, 5])
def test_tiny_other_views_bg(oracle_lib, view):
    scene, cam, dL = scene_for("tiny", view)
    cam = synth.ring_cameras(64, 64, "outdoor", 8)[view]
    run_case(oracle_lib, f"tiny_v{view}", scene, cam, synth.default_render_config(bg=(0.2, 0.5, 0.9)), dL)


def test_mcmc_sampled(oracle_lib):
    scene, cam, dL = scene_for("mcmc")
    run_case(oracle_lib, "mcmc", scene, cam, synth.default_render_config(), dL, row_mask=sampled_rows(cam))


def test_bicycle_sampled(oracle_lib):
    scene, cam, dL = scene_for("bicycle")
    run_case(oracle_lib, "bicycle", scene, cam, synth.default_render_config(), dL, row_mask=sampled_rows(cam))


def test_garden_sampled_other_view(oracle_lib):
    """Garden-shaped 5.0M @ 1297x840, a different ring view (3), sampled rows."""
    c = synth.CONFIGS["garden"]
    scene = synth.make_scene(c.n, c.kind, c.seed)
    cam = synth.ring_cameras(c.width, c.height, c.kind, 8)[3]
    dL = synth.upstream_grad(c.height, c.width, c.seed + 1003)
    run_case(oracle_lib, "garden_v3", scene, cam, synth.default_render_config(), dL, row_mask=sampled_rows(cam, 16))


@pytest.mark.slow
def test_stress_20m_sampled(oracle_lib):
    """Stress config (BASELINE.json configs[4]): 20M Gaussians @ 2474x1644 — projection and binning
    bit-exact in full, raster and gradients on every 32nd tile row."""
    c = synth.CONFIGS["stress"]
    scene = synth.make_scene(c.n, c.kind, c.seed)
    cam = synth.ring_cameras(c.width, c.height, c.kind, 8)[0]
    dL = synth.upstream_grad(c.height, c.width, c.seed + 1000)
    run_case(oracle_lib, "stress", scene, cam, synth.default_render_config(), dL, row_mask=sampled_rows(cam, 32))


# ------------------------------------------------------------------ edge cases

def test_ragged_sizes_and_3sigma(oracle_lib):
    s = synth.make_scene(20000, "outdoor", 31)
    for W, H in ((83, 61), (17, 200), (1, 1)):
        cam = synth.ring_cameras(W, H, "outdoor", 8)[2]
        dL = synth.upstream_grad(H, W, 7)
        for fp in (0, 1):
            run_case(oracle_lib, f"ragged_{W}x{H}_fp{fp}", s, cam, synth.default_render_config(footprint=fp), dL)


@pytest.mark.parametrize("deg,coeffs", [(0, 1), (1, 4), (2, 9), (3, 16), (1, 16), (2, 16)])
def test_sh_degrees(oracle_lib, deg, coeffs):
    s = synth.make_scene(5000, "indoor", 40 + deg, sh_degree=3)
    s["sh"] = np.ascontiguousarray(s["sh"][:, :coeffs])
    cam = synth.ring_cameras(96, 72, "indoor", 8)[deg]
    cfg = synth.default_render_config(deg, sh_coeffs=coeffs, bg=(0.3, 0.3, 0.3))
    run_case(oracle_lib, f"sh{deg}_{coeffs}", s, cam, cfg, synth.upstream_grad(72, 96, 3))


def test_empty_scene():
    """All Gaussians behind the camera: M = 0, image = bg, T = 1, n_contrib = 0, zero grads."""
    s = synth.make_scene(3000, "outdoor", 50)
    cam = synth.ring_cameras(64, 48)[0]
    eye = -cam["R"].astype(np.float64).T @ cam["t"].astype(np.float64)
    behind = eye - 5.0 * cam["R"][2].astype(np.float64)
    s["means"] = (behind[None, :] + 0.01 * s["means"]).astype(np.float32)
    cfg = synth.default_render_config(bg=(0.25, 0.5, 0.75))
    dL = synth.upstream_grad(48, 64, 1)
    g = run_gpu(s, cam, cfg, dL=dL)
    assert g["num_isects"] == 0
    assert (g["tiles_touched"] == 0).all()
    assert np.all(g["image"] == np.float32([0.25, 0.5, 0.75]))
    assert np.all(g["T_final"] == 1) and np.all(g["n_contrib"] == 0)
    assert np.all(g["tile_offsets"] == 0)
    for k in ("dmeans", "dlog_scales", "dquats", "dopacity_logits", "dsh", "dmeans2d"):
        assert not np.any(g[k]), k


def test_zero_gaussians():
    s = {k: v[:0] for k, v in synth.make_scene(10, "outdoor", 1).items()}
    cam = synth.ring_cameras(40, 40)[0]
    cfg = synth.default_render_config(bg=(0.1, 0.1, 0.1))
    g = run_gpu(s, cam, cfg, dL=synth.upstream_grad(40, 40, 1))
    assert g["num_isects"] == 0 and np.all(g["image"] == np.float32(0.1))


def test_capacity_regrow(oracle_lib):
    """A too-small key capacity returns VKS_ERR_CAPACITY with M; the binding regrows and retries."""
    scene, cam, dL = scene_for("tiny")
    run_case(oracle_lib, "tiny_regrow", scene, cam, synth.default_render_config(), dL, capacity=16)


def test_deterministic_integer_stages():
    """Keys, order, offsets, ranges, image and n_contrib are bitwise identical across runs."""
    scene, cam, dL = scene_for("tiny")
    cfg = synth.default_render_config()
    a = run_gpu(scene, cam, cfg)
    b = run_gpu(scene, cam, cfg)
    for k in ("keys", "vals", "offsets", "tile_offsets", "image", "T_final", "n_contrib", "means2d"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("coeffs,deg", [(16, 3), (9, 2), (4, 1), (1, 0), (16, 1)])
def test_grad_overwrite_equals_accumulate_into_zero(coeffs, deg):
    """VKS_FLAG_GRAD_OVERWRITE writes what += into a zeroed buffer gives (same 2D grads), including
    exact zero rows for Gaussians the view does not see, over a NaN-filled buffer."""
    import torch
    import paper_2605_00219_b200 as P
    s = synth.make_scene(3001, "outdoor", 60)  # odd n: ragged last warp
    s["sh"] = np.ascontiguousarray(s["sh"][:, :coeffs])
    cam = synth.ring_cameras(80, 64)[1]
    cfg = synth.default_render_config(deg, sh_coeffs=coeffs)
    params = P.GaussianParams.from_host(s)
    r = P.ViewRenderer(params.n, 80, 64)
    r.forward(cfg, cam, params)
    dL = torch.from_numpy(synth.upstream_grad(64, 80, 9)).cuda()
    params.grad_flat.zero_()
    r.backward(cfg, cam, params, dL)
    acc = params.grad_flat.clone()
    params.grad_flat.fill_(float("nan"))
    g = params.grads()
    ocfg = dict(cfg, flags=P.FLAG_GRAD_OVERWRITE)
    P.vks_project_bwd(ocfg, cam, params.means, params.log_scales, params.quats, params.opacity_logits, params.sh,
                      r.colors, r.radii, r.dmeans2d, r.dconics, r.dcolors, r.dopacities, g["dmeans"], g["dlog_scales"],
                      g["dquats"], g["dopacity_logits"], g["dsh"])
    torch.cuda.synchronize()
    vis = (r.radii != 0).any(dim=1)
    for k, v in g.items():
        ref = P.GaussianParams(params.means, params.log_scales, params.quats, params.opacity_logits, params.sh,
                               acc).grads()[k]
        assert torch.isfinite(v).all(), k                         # every row written
        assert (v[~vis] == 0).all(), k                            # unseen Gaussians: exact zeros
        # seen Gaussians: same arithmetic up to FMA contraction choices of the two instantiations
        assert torch.allclose(v[vis], ref[vis], rtol=1e-5, atol=1e-6 * ref.abs().max().item()), k


# ------------------------------------------------------------------ raster variants

def _stats(cfg, cam, scene):
    import torch
    import paper_2605_00219_b200 as P
    params = P.GaussianParams.from_host(scene)
    r = P.ViewRenderer(params.n, cam["width"], cam["height"])
    r.forward(cfg, cam, params)
    st = torch.zeros(6, dtype=torch.int64, device="cuda")
    P.vks_raster_fwd_stats(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals, r.tile_offsets, st)
    return [int(x) for x in st.tolist()]


@pytest.mark.parametrize("fp", [0, 1])
def test_patch_culling_and_ppt_variants_agree(fp, monkeypatch):
    """Patch culling only skips (warp, entry) pairs that cannot composite, and the pixel-per-thread
    layout does not change any pixel's sequence: every variant (no culling / support box /
    exact ellipse, 1, 2 or 4 pixels per thread) gives the identical image, T and n_contrib, and the
    same gradients up to atomic summation order."""
    s = synth.make_scene(200000, "indoor", 70)
    cam = synth.ring_cameras(400, 300, "indoor", 8)[3]
    cfg = synth.default_render_config(footprint=fp)
    dL = synth.upstream_grad(300, 400, 5)
    variants = [("2", "2", "0"), ("2", "2", "2"), ("4", "4", "2"), ("1", "1", "2"), ("2", "2", "1")]
    if fp == 1:
        variants = variants[:4]  # the box test needs the support footprint
    runs, stats = {}, {}
    for fw, bw, cull in variants:
        monkeypatch.setenv("VKS_RASTER_FWD_PPT", fw)
        monkeypatch.setenv("VKS_RASTER_BWD_PPT", bw)
        monkeypatch.setenv("VKS_RASTER_CULL", cull)
        runs[(fw, bw, cull)] = run_gpu(s, cam, cfg, dL=dL)
        stats[(fw, bw, cull)] = _stats(cfg, cam, s)
    base = runs[variants[0]]
    assert base["num_isects"] > 100000
    for v in variants[1:]:
        g = runs[v]
        for k in ("image", "T_final", "n_contrib"):
            assert np.array_equal(g[k], base[k]), (v, k)
        for k in ("dmeans2d", "dconics", "dcolors", "dopacities"):
            scale = np.abs(base[k]).max()
            assert np.allclose(g[k], base[k], rtol=1e-4, atol=1e-6 * scale), (v, k)
    s0, s2 = stats[variants[0]], stats[variants[1]]
    assert s2[1] == s0[1]  # composited pairs
    assert s2[0] == s0[0] and s2[3] == s0[3]  # visited / replayed do not depend on culling
    assert s2[2] < s0[2] and s2[4] < s0[4]    # ellipse culling removes evaluations
    report(f"cull_fp{fp}", dict(stats={"/".join(k): v for k, v in stats.items()}))


@pytest.mark.parametrize("kind,n,W,H,view", [("indoor", 200000, 400, 300, 3), ("outdoor", 60001, 333, 211, 5),
                                              ("outdoor", 777, 64, 48, 1)])
def test_records_path_agrees_with_gather(kind, n, W, H, view):
    """The packed raster records (vks_project_fwd `records`) hold exactly the projection's outputs
    of every visible row — (u, v, a/2, b), (c/2, rho, c0, c1), (c2, id, 0, 0), bit for bit — and
    both raster passes staging them with cp.async give the identical image, T and n_contrib as the
    gather path, and the same 2D gradients up to atomic summation order (ragged 333x211 image, a
    ragged last warp of rows, a scene smaller than one block)."""
    s = synth.make_scene(n, kind, 72)
    cam = synth.ring_cameras(W, H, kind, 8)[view]
    cfg = synth.default_render_config()
    dL = synth.upstream_grad(H, W, 6)
    rec = run_gpu(s, cam, cfg, dL=dL, records=True)
    gat = run_gpu(s, cam, cfg, dL=dL, records=False)
    vis = rec["tiles_touched"] > 0
    assert vis.sum() > n // 20
    R = rec["records"][vis].reshape(-1, 12)
    ids = np.nonzero(vis)[0]
    want = np.stack([rec["means2d"][vis, 0], rec["means2d"][vis, 1], 0.5 * rec["conics"][vis, 0],
                     rec["conics"][vis, 1], 0.5 * rec["conics"][vis, 2], rec["opacities"][vis],
                     rec["colors"][vis, 0], rec["colors"][vis, 1], rec["colors"][vis, 2]], 1).astype(np.float32)
    assert np.array_equal(R[:, :9].view(np.uint32), want.view(np.uint32))
    assert np.array_equal(R[:, 9].view(np.uint32), ids.astype(np.uint32))
    culled = rec["records"][~vis]
    assert not culled.any()  # culled rows: zeros
    for k in ("image", "T_final", "n_contrib", "vals", "tile_offsets"):
        assert np.array_equal(rec[k], gat[k]), k
    for k in ("dmeans2d", "dconics", "dcolors", "dopacities"):
        scale = np.abs(gat[k]).max()
        assert np.allclose(rec[k], gat[k], rtol=1e-4, atol=1e-6 * scale), k
    # the raster statistics (bench roofline counts) are the same through either staging
    import torch
    import paper_2605_00219_b200 as P
    params = P.GaussianParams.from_host(s)
    r = P.ViewRenderer(params.n, W, H)
    r.forward(cfg, cam, params)
    st = [torch.zeros(6, dtype=torch.int64, device="cuda") for _ in range(2)]
    for t, recs in zip(st, (None, r.records)):
        P.vks_raster_fwd_stats(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals, r.tile_offsets,
                               t, tile_order=r.tile_order, records=recs)
    assert st[0].tolist() == st[1].tolist()


def test_batched_projection_records_match_single_view():
    """vks_project_fwd_batch writes every view's records bit-identical to vks_project_fwd's."""
    import torch
    import paper_2605_00219_b200 as P
    s = synth.make_scene(50001, "outdoor", 73)
    cams = synth.ring_cameras(320, 240, "outdoor", 8)[:3]
    cfg = synth.default_render_config()
    params = P.GaussianParams.from_host(s)
    n = params.n
    e = lambda *sh, dt=torch.float32: torch.empty(*sh, dtype=dt, device="cuda")
    outs = [dict(m=e(n, 2), c=e(n, 3), d=e(n), r=e(n, 2, dt=torch.int32), t=e(n, dt=torch.int32), col=e(n, 3),
                 rec=torch.full((n, 12), float("nan"), device="cuda")) for _ in cams]
    op = e(n)
    P.vks_project_fwd_batch(cfg, cams, params.means, params.log_scales, params.quats, params.opacity_logits, params.sh,
                            [o["m"] for o in outs], [o["c"] for o in outs], [o["d"] for o in outs],
                            [o["r"] for o in outs], [o["t"] for o in outs], [o["col"] for o in outs], op,
                            records=[o["rec"] for o in outs])
    # the records carry the conics: conics may be omitted (the bench's configuration)
    rec2 = [torch.full((n, 12), float("nan"), device="cuda") for _ in cams]
    P.vks_project_fwd_batch(cfg, cams, params.means, params.log_scales, params.quats, params.opacity_logits, params.sh,
                            [o["m"] for o in outs], [None] * len(cams), [o["d"] for o in outs],
                            [o["r"] for o in outs], [o["t"] for o in outs], [o["col"] for o in outs], op,
                            records=rec2)
    for o, r2 in zip(outs, rec2):
        assert torch.equal(o["rec"].view(torch.int32), r2.view(torch.int32))
    for cam, o in zip(cams, outs):
        r = P.ViewRenderer(n, cam["width"], cam["height"])
        r.records.fill_(float("nan"))
        P.vks_project_fwd(cfg, cam, params.means, params.log_scales, params.quats, params.opacity_logits, params.sh,
                          r.means2d, r.conics, r.depths, r.radii, r.tiles, r.colors, r.opacities, records=r.records)
        torch.cuda.synchronize()
        vis = (r.tiles > 0).cpu().numpy()
        assert vis.sum() > 1000
        a, b = to_np(o["rec"])[vis], to_np(r.records)[vis]
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("lanes", ["0", "4", "32"])
def test_raster_bwd_sparse_path_agrees(lanes, monkeypatch, oracle_lib):
    """The raster backward's sparse-entry path (per-lane atomics for entries composited by few
    lanes of a warp, skip of entries no lane composited) regroups the same sums: the 2D gradients
    equal the butterfly-only kernel's up to summation order, and pass the P4 rule against the
    oracle, with the threshold at 0 (never), 4 (default) and 32 (always)."""
    s = synth.make_scene(200000, "indoor", 71)
    cam = synth.ring_cameras(400, 300, "indoor", 8)[5]
    cfg = synth.default_render_config()
    _, ref, dL, _ = oracle_reference(oracle_lib, s, cam, cfg, synth.upstream_grad(300, 400, 6))
    monkeypatch.setenv("VKS_RASTER_BWD_SPARSE", "0")
    base = run_gpu(s, cam, cfg, dL=dL)
    monkeypatch.setenv("VKS_RASTER_BWD_SPARSE", "1")
    monkeypatch.setenv("VKS_RASTER_SPARSE", lanes)
    g = run_gpu(s, cam, cfg, dL=dL)
    for k in ("dmeans2d", "dconics", "dcolors", "dopacities"):
        scale = np.abs(base[k]).max()
        assert np.allclose(g[k], base[k], rtol=1e-4, atol=1e-6 * scale), (lanes, k)
    cols = {"dmeans2d": [0, 1], "dconics": [2, 3, 4], "dcolors": [5, 6, 7], "dopacities": [8]}
    for k, c in cols.items():
        check_rule(f"sparse{lanes}", k, grad_rule(g[k], ref[k], ref["mass"][:, c].reshape(ref[k].shape)))


@pytest.mark.parametrize("W,H", [(16, 16), (200, 150), (1600, 1000), (2000, 1600), (4200, 4000)])
def test_binning_tile_pass_counts(oracle_lib, W, H):
    """Binning bit-exact for 1 tile (trivial pass), 130 tiles (one 8-bit pass), 6,300 and 12,500
    tiles (two 7-bit passes) and 65,750 tiles (three 6-bit passes), with a few Gaussians large
    enough that one Gaussian's keys span several 4096-slot key blocks."""
    s = synth.make_scene(30000, "outdoor", 80)
    cam = synth.ring_cameras(W, H, "outdoor", 8)[6]
    eye = -cam["R"].astype(np.float64).T @ cam["t"].astype(np.float64)
    fwd = cam["R"][2].astype(np.float64)
    for j in range(4):  # big, opaque Gaussians right in front of the camera
        s["means"][j] = (eye + (1.0 + 0.3 * j) * fwd).astype(np.float32)
        s["log_scales"][j] = np.log(0.6)
        s["opacity_logits"][j] = 4.0
    cfg = synth.default_render_config()
    g = run_gpu(s, cam, cfg, debug_unsorted=True)
    o_proj = oracle_lib.project_fwd(cfg, cam, s)
    check_projection(o_proj, g, f"bin_{W}x{H}")
    m = check_binning(oracle_lib, cam, g, f"bin_{W}x{H}")
    assert m > 0
    if W * H > 10**6:
        assert int(g["tiles_touched"].max()) > 4096  # one Gaussian's keys span key blocks


@pytest.mark.parametrize("case", ["equal_depths", "wide_range"])
def test_binning_depth_ranges(oracle_lib, case):
    """The depth sort uses as many digit passes as the visible depth-bit range needs: all depths
    equal (one trivial pass: ties keep id order) and a range of ~2^31 depth bits (4 passes)."""
    s = synth.make_scene(20000, "outdoor", 90)
    cam = dict(R=np.eye(3, dtype=np.float32), t=np.zeros(3, np.float32), fx=200.0, fy=200.0, cx=96.0, cy=64.0,
               width=192, height=128)
    rng = np.random.default_rng(5)
    if case == "equal_depths":
        z = np.full(len(s["means"]), 5.0)
    else:
        z = np.exp(rng.uniform(np.log(0.02), np.log(5e4), len(s["means"])))
    s["means"] = np.stack([rng.uniform(-0.45, 0.45, len(z)) * z, rng.uniform(-0.3, 0.3, len(z)) * z, z],
                          1).astype(np.float32)
    s["log_scales"] = (np.log(0.01 * z)[:, None] + rng.normal(0, 0.3, (len(z), 3))).astype(np.float32)
    cfg = synth.default_render_config()
    g = run_gpu(s, cam, cfg, debug_unsorted=True)
    o_proj = oracle_lib.project_fwd(cfg, cam, s)
    check_projection(o_proj, g, case)
    assert check_binning(oracle_lib, cam, g, case) > 1000
    d = g["depths"][g["tiles_touched"] > 0].view(np.uint32).astype(np.int64)
    spread = int(d.max() - d.min())
    assert (spread == 0) if case == "equal_depths" else (spread > 2**27)


# ------------------------------------------------------------------ batched projection backward

@pytest.mark.parametrize("coeffs,deg,nv", [(16, 3, 4), (9, 2, 3), (16, 1, 1), (4, 1, 2), (1, 0, 2)])
def test_project_bwd_batch_equals_sum_of_views(oracle_lib, coeffs, deg, nv):
    """vks_project_bwd_batch over a batch of views = the per-view vks_project_bwd summed (first view
    overwriting, the others accumulating), up to the regrouped summation; exact zeros for
    Gaussians no view sees; accumulate mode adds onto the existing gradients."""
    import torch
    import paper_2605_00219_b200 as P
    s = synth.make_scene(20001, "outdoor", 70 + nv)
    s["sh"] = np.ascontiguousarray(s["sh"][:, :coeffs])
    cams = synth.ring_cameras(160, 120, "outdoor", 8)[:nv]
    cfg = synth.default_render_config(deg, sh_coeffs=coeffs)
    params = P.GaussianParams.from_host(s)
    views = []
    for v, cam in enumerate(cams):
        r = P.ViewRenderer(params.n, 160, 120)
        r.forward(cfg, cam, params)
        r.g2d.zero_()
        dL = torch.from_numpy(synth.upstream_grad(120, 160, 11 + v)).cuda()
        P.vks_raster_bwd(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals, r.tile_offsets,
                         r.T_final, r.n_contrib, dL, r.dmeans2d, r.dconics, r.dcolors, r.dopacities,
                         tile_order=r.tile_order)
        views.append(r)
    g = params.grads()
    ocfg = dict(cfg, flags=P.FLAG_GRAD_OVERWRITE)
    for v, (cam, r) in enumerate(zip(cams, views)):
        P.vks_project_bwd(ocfg if v == 0 else cfg, cam, params.means, params.log_scales, params.quats,
                          params.opacity_logits, params.sh, r.colors, r.radii, r.dmeans2d, r.dconics, r.dcolors,
                          r.dopacities, g["dmeans"], g["dlog_scales"], g["dquats"], g["dopacity_logits"], g["dsh"])
    torch.cuda.synchronize()
    ref = params.grad_flat.clone()

    def batch(c):
        P.vks_project_bwd_batch(c, cams, params.means, params.log_scales, params.quats, params.opacity_logits,
                                params.sh, [r.colors for r in views], [r.radii for r in views],
                                [r.dmeans2d for r in views], [r.dconics for r in views], [r.dcolors for r in views],
                                [r.dopacities for r in views], g["dmeans"], g["dlog_scales"], g["dquats"],
                                g["dopacity_logits"], g["dsh"])
        torch.cuda.synchronize()
        return params.grad_flat.clone()

    params.grad_flat.fill_(float("nan"))
    got = batch(ocfg)
    seen = torch.zeros(params.n, dtype=torch.bool, device="cuda")
    for r in views:
        seen |= (r.radii != 0).any(dim=1)
    G = P.GaussianParams(params.means, params.log_scales, params.quats, params.opacity_logits, params.sh, got).grads()
    Rf = P.GaussianParams(params.means, params.log_scales, params.quats, params.opacity_logits, params.sh, ref).grads()
    # against the oracle: its fp64 projection backward of each view (fed that view's GPU 2D
    # gradients, stage-isolated as P5) summed over the batch; same per-element rule and mass
    ref_o, mass_o = None, None
    for cam, r in zip(cams, views):
        g2 = {k: to_np(getattr(r, k)) for k in ("dmeans2d", "dconics", "dcolors", "dopacities")}
        iso = oracle_lib.project_bwd(cfg, cam, s, g2)
        ms = oracle_lib.project_bwd_mass(cfg, cam, s, g2)
        ref_o = iso if ref_o is None else {k: ref_o[k] + iso[k] for k in ref_o}
        mass_o = ms if mass_o is None else {k: mass_o[k] + ms[k] for k in mass_o}
    for k in ("dmeans", "dlog_scales", "dquats", "dopacity_logits", "dsh"):
        assert torch.isfinite(G[k]).all(), k
        assert (G[k][~seen] == 0).all(), k
        rule = grad_rule(to_np(G[k]), ref_o[k], mass=mass_o[k])
        check_rule("batch", k, rule)
        # and against the per-view kernels summed (the same chains, regrouped): the rule with the
        # sequential sum as reference
        rule = grad_rule(to_np(G[k]), to_np(Rf[k]), mass=mass_o[k], rel=1e-4)
        check_rule("batch vs per-view", k, rule)
    # accumulate mode: += onto existing rows (the batch result itself)
    got2 = batch(cfg)
    G2 = P.GaussianParams(params.means, params.log_scales, params.quats, params.opacity_logits, params.sh, got2).grads()
    for k in G:
        rule = grad_rule(to_np(G2[k]), 2 * to_np(G[k]).astype(np.float64), mass=2 * mass_o[k], rel=1e-4)
        check_rule("batch accumulate", k, rule)


@pytest.mark.parametrize("coeffs,deg,nv,fp", [(16, 3, 5, 0), (9, 2, 3, 0), (4, 1, 2, 1), (1, 0, 1, 0)])
def test_project_fwd_batch_bit_exact(oracle_lib, coeffs, deg, nv, fp):
    """vks_project_fwd_batch: every view's outputs bit-identical to vks_project_fwd for that view
    and to the oracle's O1 (P1), the opacities equal for every visible row; the optional
    2D-gradient blocks (g2d_zero) come back zeroed (every row, culled or not)."""
    import torch
    import paper_2605_00219_b200 as P
    s = synth.make_scene(30001, "outdoor", 90 + nv)
    s["sh"] = np.ascontiguousarray(s["sh"][:, :coeffs])
    cams = synth.ring_cameras(200, 150, "outdoor", 8)[:nv]
    cfg = synth.default_render_config(deg, sh_coeffs=coeffs, footprint=fp)
    params = P.GaussianParams.from_host(s)
    n = params.n
    e = lambda *sh, dt=torch.float32: torch.empty(*sh, dtype=dt, device="cuda")
    outs = [dict(means2d=e(n, 2), conics=e(n, 3), depths=e(n), radii=e(n, 2, dt=torch.int32),
                 tiles=e(n, dt=torch.int32), colors=e(n, 3)) for _ in range(nv)]
    opac = e(n)
    g2d = [torch.full((9 * n,), float("nan"), device="cuda") for _ in range(nv)]
    P.vks_project_fwd_batch(cfg, cams, params.means, params.log_scales, params.quats, params.opacity_logits, params.sh,
                            [o["means2d"] for o in outs], [o["conics"] for o in outs], [o["depths"] for o in outs],
                            [o["radii"] for o in outs], [o["tiles"] for o in outs], [o["colors"] for o in outs], opac,
                            g2d_zero=g2d)
    torch.cuda.synchronize()
    assert all(bool((t == 0).all()) for t in g2d)
    for v, (cam, o) in enumerate(zip(cams, outs)):
        g = {k: to_np(t) for k, t in o.items()}
        g["tiles_touched"] = g.pop("tiles")
        g["opacities"] = to_np(opac)
        ref = oracle_lib.project_fwd(cfg, cam, s)
        nvis = check_projection(ref, g, f"fwd_batch_v{v}")
        assert nvis > 1000
