"""CUDA-event medians of one batch's projection forward and backward (vks_project_fwd_batch /
vks_project_bwd_batch, overwrite) after 8 ring views are rendered and raster-backpropagated.
usage: python tools/time_batch.py [config] [B]   (VKS_LIB_VARIANT=name: a tools/build_variant.py build)"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_00219_b200 as P  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bicycle"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
c = synth.CONFIGS[name]
cfg = synth.default_render_config(3)
params = P.GaussianParams.from_host(synth.make_scene(c.n, c.kind, c.seed))
cams = synth.ring_cameras(c.width, c.height, c.kind, 8)
views = []
for v in range(B):
    r = P.ViewRenderer(params.n, c.width, c.height)
    cam = cams[v % 8]
    r.forward(cfg, cam, params)
    r.g2d.zero_()
    dL = torch.from_numpy(synth.upstream_grad(c.height, c.width, c.seed + 1000 + v)).cuda()
    P.vks_raster_bwd(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals, r.tile_offsets,
                     r.T_final, r.n_contrib, dL, r.dmeans2d, r.dconics, r.dcolors, r.dopacities, tile_order=r.tile_order)
    views.append(r)
g = params.grads()
ocfg = dict(cfg, flags=P.FLAG_GRAD_OVERWRITE)


def batch():
    P.vks_project_bwd_batch(ocfg, [cams[v % 8] for v in range(B)], params.means, params.log_scales, params.quats,
                            params.opacity_logits, params.sh, [r.colors for r in views], [r.radii for r in views],
                            [r.dmeans2d for r in views], [r.dconics for r in views], [r.dcolors for r in views],
                            [r.dopacities for r in views], g["dmeans"], g["dlog_scales"], g["dquats"],
                            g["dopacity_logits"], g["dsh"])


def fwd_batch():
    P.vks_project_fwd_batch(cfg, [cams[v % 8] for v in range(B)], params.means, params.log_scales, params.quats,
                            params.opacity_logits, params.sh, [r.means2d for r in views], [r.conics for r in views],
                            [r.depths for r in views], [r.radii for r in views], [r.tiles for r in views],
                            [r.colors for r in views], views[0].opacities,
                            g2d_zero=[r.g2d for r in views], records=[r.records for r in views])


def med(fn, reps=15):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(4_000_000)  # the GPU busy while the host marshals the call: device time only
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts[2:])


print(f"{name} B={B} lib={os.environ.get('VKS_LIB_VARIANT', 'default')}: project_fwd_batch {med(fwd_batch):.4f} ms  "
      f"project_bwd_batch {med(batch):.4f} ms", flush=True)
