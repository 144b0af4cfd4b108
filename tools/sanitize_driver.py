"""Every kernel of libvks once: for compute-sanitizer where it runs, and with VKS_DEBUG_CHECKS=1
(libvks_debug.so: device-side bounds / invariant checks that trap) where it does not
(tests/test_gpu_debug_checks.py).  usage: python tools/sanitize_driver.py [config] [n_override]

Runs on one view of the config: the single-view and batched projection forward, bin sort (with the
debug unsorted keys), vks_bin_sort_check, raster forward (+ stats), raster backward (sparse-entry and
butterfly-only variants), the single-view and batched projection backward, VALIDATE checks, the
Adam step, the loss gradient, MCMC relocation + noise and default densification."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_00219_b200 as P  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
c = synth.CONFIGS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else c.n
cfg = synth.default_render_config(3)
scene = synth.make_scene(n, c.kind, c.seed)
cams = synth.ring_cameras(c.width, c.height, c.kind, 8)
cam = cams[0]
params = P.GaussianParams.from_host(scene)
dL = torch.from_numpy(synth.upstream_grad(c.height, c.width, c.seed + 1000)).cuda()
r = P.ViewRenderer(params.n, c.width, c.height)
r.forward(cfg, cam, params, want_keys=True)
ku = torch.empty(r.capacity, dtype=torch.uint64, device="cuda")
vu = torch.empty(r.capacity, dtype=torch.uint32, device="cuda")
r.forward(dict(cfg, flags=P.FLAG_VALIDATE), cam, params, ku, vu, want_keys=True)
assert P.vks_bin_sort_check(cam, r.means2d, r.radii, r.depths, r.vals, r.tile_offsets, r.num_isects) == 0
st = torch.zeros(6, dtype=torch.int64, device="cuda")
P.vks_raster_fwd_stats(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals, r.tile_offsets, st,
                       tile_order=r.tile_order)
for sparse in ("1", "0"):
    os.environ["VKS_RASTER_BWD_SPARSE"] = sparse
    r.backward(dict(cfg, flags=P.FLAG_VALIDATE), cam, params, dL, accumulate=False)
# batched projection (2 views) + backward
views = [P.ViewRenderer(params.n, c.width, c.height, capacity=2 * r.capacity) for _ in range(2)]
vc = cams[:2]
P.vks_project_fwd_batch(cfg, vc, params.means, params.log_scales, params.quats, params.opacity_logits, params.sh,
                        [v.means2d for v in views], [v.conics for v in views], [v.depths for v in views],
                        [v.radii for v in views], [v.tiles for v in views], [v.colors for v in views],
                        views[0].opacities, g2d_zero=[v.g2d for v in views])
for v, cv in zip(views, vc):
    v.opacities.copy_(views[0].opacities)
    m = P.vks_bin_sort(cv, v.means2d, v.radii, v.depths, v.tiles, v.offsets, None, v.vals, v.tile_offsets,
                       v.workspace, tile_order=v.tile_order)
    P.vks_raster_fwd(cfg, cv, v.means2d, v.conics, v.colors, v.opacities, v.radii, v.vals, v.tile_offsets, v.image,
                     v.T_final, v.n_contrib, tile_order=v.tile_order)
    P.vks_raster_bwd(cfg, cv, v.means2d, v.conics, v.colors, v.opacities, v.radii, v.vals, v.tile_offsets, v.T_final,
                     v.n_contrib, dL, v.dmeans2d, v.dconics, v.dcolors, v.dopacities, tile_order=v.tile_order)
g = params.grads()
P.vks_project_bwd_batch(dict(cfg, flags=P.FLAG_GRAD_OVERWRITE), vc, params.means, params.log_scales, params.quats,
                        params.opacity_logits, params.sh, [v.colors for v in views], [v.radii for v in views],
                        [v.dmeans2d for v in views], [v.dconics for v in views], [v.dcolors for v in views],
                        [v.dopacities for v in views], g["dmeans"], g["dlog_scales"], g["dquats"],
                        g["dopacity_logits"], g["dsh"])
# optimizer, loss, MCMC, densification
groups = [params.means, params.log_scales, params.quats, params.opacity_logits, params.sh]
grads = [g[k] for k in ("dmeans", "dlog_scales", "dquats", "dopacity_logits", "dsh")]
mom, vel = [torch.zeros_like(t) for t in groups], [torch.zeros_like(t) for t in groups]
lrs = dict(means=1.6e-4, log_scales=5e-3, quats=1e-3, opacity_logits=5e-2, sh=(2.5e-3, 1.25e-4))
P.vks_adam_step(P.make_adam_config(lrs, step=1), groups, grads, mom, vel)
if c.width >= 11 and c.height >= 11:
    ws = torch.empty(P.vks_loss_workspace_bytes(c.width, c.height), dtype=torch.uint8, device="cuda")
    dLd, loss = torch.empty_like(r.image), torch.empty(1, device="cuda")
    P.vks_loss_grad(r.image, torch.rand_like(r.image), dLd, loss, ws, lam=0.2)
mws = torch.empty(P.vks_mcmc_workspace_bytes(params.n), dtype=torch.uint8, device="cuda")
P.vks_mcmc_relocate(params, mws, dead_opacity=0.05, seed=3)
P.vks_mcmc_noise(params, 1.6e-4, 5e5, seed=3, step=1)
acc, den = torch.zeros(params.n, device="cuda"), torch.zeros(params.n, device="cuda")
P.vks_densify_stats(r.dmeans2d, r.radii, acc, den)
dst = [torch.empty((2 * params.n,) + tuple(t.shape[1:]), device="cuda") for t in groups]
dws = torch.empty(P.vks_densify_workspace_bytes(params.n), dtype=torch.uint8, device="cuda")
n_new = P.vks_densify(groups, acc, den, dst, dws, 1e-4, 0.05, 0.005, seed=1)
torch.cuda.synchronize()
print(f"sanitize driver ok: {name} n={params.n} M={r.num_isects} densified to {n_new} "
      f"lib={os.path.basename(P._vks.LIB_PATH)}")
