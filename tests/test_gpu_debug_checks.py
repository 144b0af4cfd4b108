"""The debug build (libvks_debug.so, -DVKS_DEBUG_CHECKS) through every kernel — the stand-in for
compute-sanitizer memcheck, which this GPU pool refuses to run (profiles/r2_sanitizer_unavailable.txt).
Its device-side checks guard the indexed accesses (raster list ids < n and tile ranges ordered, radix
scatter destinations inside [0, n), expanded key slots inside their block and tile ids in range,
tile rects inside the grid, MCMC relocation targets in [0, n), densification output rows below n').
The driver runs the tiny, MCMC-shaped (1M) and bicycle-shaped (5.8M) configurations without a trap,
and a corrupted tile range is shown to trap (the checks are live)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "paper_2605_00219_b200", "libvks_debug.so")


def _run(args, timeout=900):
    env = dict(os.environ, VKS_DEBUG_CHECKS="1")
    return subprocess.run([sys.executable, *args], cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


@pytest.fixture(scope="module", autouse=True)
def _need():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(DEBUG_LIB):
        pytest.fail("libvks_debug.so missing: __graft_entry__.build() builds it")


@pytest.mark.parametrize("config", ["tiny", "mcmc", "bicycle"])
def test_every_kernel_passes_the_debug_checks(config):
    r = _run([os.path.join("tools", "sanitize_driver.py"), config])
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    assert "sanitize driver ok" in r.stdout and "lib=libvks_debug.so" in r.stdout
    assert "VKS_DCHECK failed" not in r.stdout + r.stderr


CORRUPT = r'''
import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth, paper_2605_00219_b200 as P
c = synth.CONFIGS["tiny"]
params = P.GaussianParams.from_host(synth.make_scene(c.n, c.kind, c.seed))
cam = synth.ring_cameras(c.width, c.height, c.kind, 8)[0]
r = P.ViewRenderer(params.n, c.width, c.height)
r.forward(synth.default_render_config(), cam, params)
o = r.tile_offsets.clone().view(torch.int32)
o[3] = o[4] + 5  # tile 3's range ends before it starts
P.vks_raster_fwd(synth.default_render_config(), cam, r.means2d, r.conics, r.colors, r.opacities, r.radii, r.vals,
                 o.view(torch.uint32), r.image, r.T_final, r.n_contrib)
torch.cuda.synchronize()
print("no trap")
'''


def test_debug_checks_are_live():
    r = _run(["-c", CORRUPT], timeout=300)
    assert r.returncode != 0 and "no trap" not in r.stdout
    assert "VKS_DCHECK failed" in r.stdout + r.stderr
