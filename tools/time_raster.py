"""CUDA-event time of vks_raster_bwd on the bicycle view 0, for each value of an optional kernel
selector environment variable.  usage: python tools/time_raster.py [config] [VAR v1 v2 ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_00219_b200 as P  # noqa: E402
import synth  # noqa: E402

c = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "bicycle"]
cfg = synth.default_render_config(3)
params = P.GaussianParams.from_host(synth.make_scene(c.n, c.kind, c.seed))
cam = synth.ring_cameras(c.width, c.height, c.kind, 8)[0]
dL = torch.from_numpy(synth.upstream_grad(c.height, c.width, c.seed + 1000)).cuda()
r = P.ViewRenderer(params.n, c.width, c.height)
r.forward(cfg, cam, params)


var = sys.argv[2] if len(sys.argv) > 2 else None
for pair in (sys.argv[3:] if var else ["-"]):
    if var:
        os.environ[var] = pair
    ts = []
    for i in range(23):
        r.g2d.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        P.vks_raster_bwd(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals, r.tile_offsets,
                         r.T_final, r.n_contrib, dL, r.dmeans2d, r.dconics, r.dcolors, r.dopacities,
                         tile_order=r.tile_order)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    ts.sort()
    g = r.g2d.clone()
    print(f"raster_bwd {var}={pair}: median {ts[len(ts) // 2]:.4f} ms  min {ts[0]:.4f}  |g|={float(g.abs().sum()):.6e}")
