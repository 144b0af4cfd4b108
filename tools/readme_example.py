"""The README's Python usage example, runnable (checks that it works as written)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_00219_b200 as P  # noqa: E402
import synth  # noqa: E402

scene = synth.make_scene(1_000_000, "indoor", seed=1)
cam = synth.ring_cameras(1559, 1039, "indoor", 8)[0]
cfg = synth.default_render_config(3)
params = P.GaussianParams.from_host(scene)
view = P.ViewRenderer(params.n, cam["width"], cam["height"])

image = view.forward(cfg, cam, params)
dL = torch.rand_like(image) * 2 - 1
params.grad_flat.zero_()
view.backward(cfg, cam, params, dL)
grads = params.grads()
torch.cuda.synchronize()
print("image", tuple(image.shape), float(image.mean()), "M", view.num_isects,
      {k: float(v.abs().sum()) for k, v in grads.items()})
