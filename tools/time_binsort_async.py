"""CUDA-event medians of vks_bin_sort (host-synchronising) and vks_bin_sort_async on one view.
usage: python tools/time_binsort_async.py [config] [reps]"""
import os
import statistics
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
cap = int(r.num_isects * 1.2) + 1024
vals = torch.empty(cap, dtype=torch.uint32, device="cuda")
ws = torch.empty(P.vks_bin_sort_workspace_bytes(r.n, cap, r.n_tiles), dtype=torch.uint8, device="cuda")
m = torch.zeros(1, dtype=torch.int64, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")


def med(fn):
    ts = []
    for i in range(reps + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


t_sync = med(lambda: P.vks_bin_sort(cam, r.means2d, r.radii, r.depths, r.tiles, r.offsets, None, r.vals,
                                    r.tile_offsets, r.workspace, tile_order=r.tile_order))
t_async = med(lambda: P.vks_bin_sort_async(cam, r.means2d, r.radii, r.depths, r.tiles, r.offsets, vals,
                                           r.tile_offsets, ws, m, st, tile_order=r.tile_order))
print(f"bin_sort {name}: sync {t_sync:.4f} ms  async {t_async:.4f} ms (capacity {cap}, M {int(m.item())}, "
      f"status {int(st.item())})")
