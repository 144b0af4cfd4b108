"""CUDA-event medians of every stage of the single-view (batch-1) path on one view, through the C
ABI: vks_project_fwd, vks_bin_sort, vks_raster_fwd, vks_raster_bwd, vks_project_bwd.
usage: python tools/time_stages.py [config] [reps] [VAR=value ...]   (env overrides per run)"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

for a in sys.argv[1:]:
    if "=" in a:
        k, v = a.split("=", 1)
        os.environ[k] = v
args = [a for a in sys.argv[1:] if "=" not in a]

import torch  # noqa: E402

import paper_2605_00219_b200 as P  # noqa: E402
import synth  # noqa: E402

name = args[0] if args else "bicycle"
reps = int(args[1]) if len(args) > 1 else 20
c = synth.CONFIGS[name]
cfg = synth.default_render_config(3)
params = P.GaussianParams.from_host(synth.make_scene(c.n, c.kind, c.seed))
cams = synth.ring_cameras(c.width, c.height, c.kind, 8)
dL = torch.from_numpy(synth.upstream_grad(c.height, c.width, c.seed + 1000)).cuda()
r = P.ViewRenderer(params.n, c.width, c.height)
for cam in cams:
    r.forward(cfg, cam, params)
r._alloc_capacity(int(r.capacity * 1.1))
g = params.grads()
names = ["project_fwd", "bin_sort", "raster_fwd", "raster_bwd", "project_bwd"]
ts = {k: [] for k in names}
for i in range(reps + 3):
    cam = cams[i % 8]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    r.g2d.zero_()
    ev[0].record()
    P.vks_project_fwd(cfg, cam, params.means, params.log_scales, params.quats, params.opacity_logits, params.sh,
                      r.means2d, r.conics, r.depths, r.radii, r.tiles, r.colors, r.opacities)
    ev[1].record()
    m = P.vks_bin_sort(cam, r.means2d, r.radii, r.depths, r.tiles, r.offsets, None, r.vals, r.tile_offsets,
                       r.workspace, tile_order=r.tile_order)
    ev[2].record()
    P.vks_raster_fwd(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals, r.tile_offsets,
                     r.image, r.T_final, r.n_contrib, tile_order=r.tile_order)
    ev[3].record()
    P.vks_raster_bwd(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals, r.tile_offsets,
                     r.T_final, r.n_contrib, dL, r.dmeans2d, r.dconics, r.dcolors, r.dopacities,
                     tile_order=r.tile_order)
    ev[4].record()
    P.vks_project_bwd(dict(cfg, flags=P.FLAG_GRAD_OVERWRITE), cam, params.means, params.log_scales, params.quats,
                      params.opacity_logits, params.sh, r.colors, r.radii, r.dmeans2d, r.dconics, r.dcolors,
                      r.dopacities, g["dmeans"], g["dlog_scales"], g["dquats"], g["dopacity_logits"], g["dsh"])
    ev[5].record()
    torch.cuda.synchronize()
    if i >= 3:
        for q, k in enumerate(names):
            ts[k].append(ev[q].elapsed_time(ev[q + 1]))
med = {k: statistics.median(v) for k, v in ts.items()}
tot = sum(med.values())
print(" ".join(f"{k}={v:.4f}" for k, v in med.items()), f"sum={tot:.4f} ms -> {1e3 / tot:.1f} it/s",
      f"|img|={float(r.image.abs().sum()):.6e} |g2d|={float(r.g2d.abs().sum()):.6e}")
