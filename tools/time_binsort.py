"""CUDA-event time of vks_bin_sort alone on the bicycle view 0 (projection done once, untimed).
usage: python tools/time_binsort.py [config] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_00219_b200 as P  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bicycle"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = synth.CONFIGS[name]
cfg = synth.default_render_config(3)
params = P.GaussianParams.from_host(synth.make_scene(c.n, c.kind, c.seed))
cam = synth.ring_cameras(c.width, c.height, c.kind, 8)[0]
r = P.ViewRenderer(params.n, c.width, c.height)
r.forward(cfg, cam, params)
torch.cuda.synchronize()
ts = []
for i in range(reps + 3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    P.vks_bin_sort(cam, r.means2d, r.radii, r.depths, r.tiles, r.offsets, None, r.vals, r.tile_offsets,
                   r.workspace, tile_order=r.tile_order)
    b.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b))
ts.sort()
print(f"bin_sort {name}: median {ts[len(ts) // 2]:.4f} ms  min {ts[0]:.4f} ms  (M = {r.num_isects})")

if os.environ.get("PLACE_PROF"):
    import ctypes as C
    lib = P._vks._lib
    buf = (C.c_ulonglong * 8)()
    lib.vks_debug_place_prof(buf, 1)
    P.vks_bin_sort(cam, r.means2d, r.radii, r.depths, r.tiles, r.offsets, None, r.vals, r.tile_offsets,
                   r.workspace, tile_order=r.tile_order)
    torch.cuda.synchronize()
    lib.vks_debug_place_prof(buf, 0)
    nw = 4 * ((r.num_isects + 16383) // 16384)
    names = ["setup+owner", "phaseA count", "phaseB prefix", "stage", "positions", "stores"]
    for i, nm in enumerate(names):
        print(f"{nm:14s} {buf[i] / nw:10.0f} cycles per warp")
