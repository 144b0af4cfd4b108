"""The bench step's kernels between cudaProfilerStart/Stop, for `ncu --profile-from-start off ...`:
one batched projection forward (8 ring views), view 0's binning, raster forward and raster
backward, and one batched projection backward (views 1-7 rendered and raster-backpropagated
before the profiled range, so the batch has all of its 2D gradients).  Bicycle-shaped scene."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_00219_b200 as P  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bicycle"
B = 8
c = synth.CONFIGS[name]
cfg = synth.default_render_config(3)
ocfg = dict(cfg, flags=P.FLAG_GRAD_OVERWRITE)
params = P.GaussianParams.from_host(synth.make_scene(c.n, c.kind, c.seed))
cams = synth.ring_cameras(c.width, c.height, c.kind, 8)
views = [P.ViewRenderer(params.n, c.width, c.height) for _ in range(B)]
dLs = [torch.from_numpy(synth.upstream_grad(c.height, c.width, c.seed + 1000 + v)).cuda() for v in range(B)]
g = params.grads()


def fwd_batch():
    P.vks_project_fwd_batch(cfg, cams[:B], params.means, params.log_scales, params.quats, params.opacity_logits,
                            params.sh, [r.means2d for r in views], [None for r in views],  # records carry the conics
                            [r.depths for r in views], [r.radii for r in views], [r.tiles for r in views],
                            [r.colors for r in views], views[0].opacities, g2d_zero=[r.g2d for r in views],
                            records=[r.records for r in views])


def view(v):
    r = views[v]
    r.num_isects = P.vks_bin_sort(cams[v], r.means2d, r.radii, r.depths, r.tiles, r.offsets, None, r.vals,
                                  r.tile_offsets, r.workspace, tile_order=r.tile_order)
    P.vks_raster_fwd(cfg, cams[v], r.means2d, r.conics, r.colors, views[0].opacities, r.radii, r.vals,
                     r.tile_offsets, r.image, r.T_final, r.n_contrib, tile_order=r.tile_order, records=r.records)
    P.vks_raster_bwd(cfg, cams[v], r.means2d, r.conics, r.colors, views[0].opacities, r.radii, r.vals,
                     r.tile_offsets, r.T_final, r.n_contrib, dLs[v], r.dmeans2d, r.dconics, r.dcolors,
                     r.dopacities, tile_order=r.tile_order, records=r.records)


def bwd_batch():
    P.vks_project_bwd_batch(ocfg, cams[:B], params.means, params.log_scales, params.quats, params.opacity_logits,
                            params.sh, [r.colors for r in views], [r.radii for r in views],
                            [r.dmeans2d for r in views], [r.dconics for r in views], [r.dcolors for r in views],
                            [r.dopacities for r in views], g["dmeans"], g["dlog_scales"], g["dquats"],
                            g["dopacity_logits"], g["dsh"])


for r in views:  # size the key capacities (regrow outside the profiled range)
    for v in range(B):
        r.forward(cfg, cams[v], params)
fwd_batch()
for v in range(B):
    view(v)
bwd_batch()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
fwd_batch()
view(0)
bwd_batch()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("M", views[0].num_isects)
