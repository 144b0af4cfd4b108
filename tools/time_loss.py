"""CUDA-event time of vks_loss_grad at a config's resolution.  usage: python tools/time_loss.py [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_00219_b200 as P  # noqa: E402
import synth  # noqa: E402

c = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "bicycle"]
r = torch.rand(c.height, c.width, 3, device="cuda")
t = torch.rand(c.height, c.width, 3, device="cuda")
dL = torch.empty_like(r)
loss = torch.empty(1, device="cuda")
ws = torch.empty(P.vks_loss_workspace_bytes(c.width, c.height), dtype=torch.uint8, device="cuda")
ts = []
for i in range(23):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    P.vks_loss_grad(r, t, dL, loss, ws, lam=0.2)
    b.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b))
ts.sort()
print(f"loss_grad {c.width}x{c.height}: median {ts[len(ts) // 2]:.4f} ms")
