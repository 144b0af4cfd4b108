"""CUDA-event medians of vks_raster_fwd and vks_raster_bwd on one bicycle-shaped view, staging the
packed records (cp.async) vs gathering the separate arrays, optionally for each value of a kernel
selector environment variable.
usage: python tools/time_raster_ab.py [config] [view] [VAR v1 v2 ...]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_00219_b200 as P  # noqa: E402
import synth  # noqa: E402

c = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "bicycle"]
view = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = synth.default_render_config(3)
params = P.GaussianParams.from_host(synth.make_scene(c.n, c.kind, c.seed))
cam = synth.ring_cameras(c.width, c.height, c.kind, 8)[view]
dL = torch.from_numpy(synth.upstream_grad(c.height, c.width, c.seed + 1000 + view)).cuda()
r = P.ViewRenderer(params.n, c.width, c.height)
r.forward(cfg, cam, params)


def med(fn, reps=21):
    ts = []
    for i in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts[2:])


ORDER = None if os.environ.get("VKS_TOOL_NO_ORDER") == "1" else r.tile_order  # LPT schedule or tile id order


def run(rec):
    fwd = med(lambda: P.vks_raster_fwd(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals,
                                       r.tile_offsets, r.image, r.T_final, r.n_contrib, tile_order=ORDER,
                                       records=rec))

    def bwd():
        P.vks_raster_bwd(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals, r.tile_offsets,
                         r.T_final, r.n_contrib, dL, r.dmeans2d, r.dconics, r.dcolors, r.dopacities,
                         tile_order=ORDER, records=rec)
    bwd_ms = med(bwd)
    return fwd, bwd_ms


var = sys.argv[3] if len(sys.argv) > 3 else None
for val in (sys.argv[4:] if var else ["-"]):
    if var:
        os.environ[var] = val
    for name, rec in (("gather", None), ("records", r.records)):
        f, b = run(rec)
        print(f"{c.name} view {view} {var or ''}={val} {name:8s} raster_fwd {f:.4f} ms  raster_bwd {b:.4f} ms", flush=True)

if os.environ.get("VKS_TOOL_WORK_ORDER") == "1":
    # the backward scheduled by its own work estimate from the forward: per tile the sum over its
    # four 8x8 warp patches of the patch's largest n_contrib (the replay range), heaviest first
    H, W = c.height, c.width
    TX, TY = (W + 15) // 16, (H + 15) // 16
    nc = torch.zeros(TY * 16, TX * 16, dtype=torch.int32, device="cuda")
    nc[:H, :W] = r.n_contrib
    patch = nc.view(TY * 2, 8, TX * 2, 8).amax(dim=(1, 3)).to(torch.int64)  # [2TY, 2TX]
    work = patch.view(TY, 2, TX, 2).sum(dim=(1, 3)).reshape(-1)
    order_w = torch.argsort(work, descending=True).to(torch.int32).view(torch.uint32).contiguous()

    def bwd_w():
        P.vks_raster_bwd(cfg, cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals, r.tile_offsets,
                         r.T_final, r.n_contrib, dL, r.dmeans2d, r.dconics, r.dcolors, r.dopacities,
                         tile_order=order_w, records=r.records)
    print(f"{c.name} view {view} backward with the work order: {med(bwd_w):.4f} ms", flush=True)
