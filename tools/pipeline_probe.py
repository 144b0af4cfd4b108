"""Throughput probe: views in flight on S streams (one ViewRenderer per stream), gradients of all
views accumulated into one buffer (project_bwd of consecutive views serialised by events, since it
read-modify-writes the gradient rows).  Prints views/s for S = 1 and S = 2.
usage: python tools/pipeline_probe.py [config] [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_00219_b200 as P  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bicycle"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 64
c = synth.CONFIGS[name]
cfg = synth.default_render_config(3)
params = P.GaussianParams.from_host(synth.make_scene(c.n, c.kind, c.seed))
cams = synth.ring_cameras(c.width, c.height, c.kind, 8)
dLs = [torch.from_numpy(synth.upstream_grad(c.height, c.width, c.seed + 1000 + v)).cuda() for v in range(8)]


def run(S):
    rends = [P.ViewRenderer(params.n, c.width, c.height) for _ in range(S)]
    streams = [torch.cuda.Stream() for _ in range(S)]
    for r in rends:
        for v in range(8):
            r.forward(cfg, cams[v], params)
        r._alloc_capacity(int(r.capacity * 1.1))
    torch.cuda.synchronize()
    bwd_done = [None]

    def view(i):
        k = i % S
        st = streams[k]
        r, cam = rends[k], cams[i % 8]
        with torch.cuda.stream(st):
            r.forward(cfg, cam, params)
            r.g2d.zero_()
            P.vks_raster_bwd(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals, r.tile_offsets,
                             r.T_final, r.n_contrib, dLs[i % 8], r.dmeans2d, r.dconics, r.dcolors, r.dopacities,
                             tile_order=r.tile_order)
            if bwd_done[0] is not None:
                st.wait_event(bwd_done[0])  # gradient rows: one project_bwd at a time
            g = params.grads()
            P.vks_project_bwd(cfg, cam, params.means, params.log_scales, params.quats, params.opacity_logits,
                              params.sh, r.colors, r.radii, r.dmeans2d, r.dconics, r.dcolors, r.dopacities,
                              g["dmeans"], g["dlog_scales"], g["dquats"], g["dopacity_logits"], g["dsh"])
            ev = torch.cuda.Event()
            ev.record(st)
            bwd_done[0] = ev

    for i in range(8):
        view(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        view(i)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return steps / dt


for S in (1, 2, 3):
    print(f"streams={S}: {run(S):.1f} views/s")
