"""One warm step of the hot path between cudaProfilerStart/Stop, for
`ncu --profile-from-start off --set full ...` (see profiles/README.md)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_00219_b200 as P  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bicycle"
c = synth.CONFIGS[name]
cfg = synth.default_render_config(3)
params = P.GaussianParams.from_host(synth.make_scene(c.n, c.kind, c.seed))
cam = synth.ring_cameras(c.width, c.height, c.kind, 8)[0]
dL = torch.from_numpy(synth.upstream_grad(c.height, c.width, c.seed + 1000)).cuda()
r = P.ViewRenderer(params.n, c.width, c.height)
for _ in range(2):
    r.forward(cfg, cam, params)
    r.backward(cfg, cam, params, dL, accumulate=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
r.forward(cfg, cam, params)
r.backward(cfg, cam, params, dL, accumulate=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("M", r.num_isects)
