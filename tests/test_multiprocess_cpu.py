"""World-size-2 gloo test of the view-sharded gradient path on CPU: per-view
gradients (from the oracle, standing in for one GPU each) are accumulated per rank into the flat
buffer layout of GaussianParams and all-reduced; the result equals the single-process sum over
all views."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

N_VIEWS = 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _flat_grads(scene, views):
    import oracle
    from paper_2605_00219_b200.pipeline import GaussianParams
    n, K = scene["means"].shape[0], scene["sh"].shape[1]
    offs, total = GaussianParams.layout(n, K)
    flat = np.zeros(total, np.float64)
    cams = synth.ring_cameras(48, 40, "outdoor", 8)
    cfg = synth.default_render_config()
    for v in views:
        dL = synth.upstream_grad(40, 48, 100 + v)
        r = oracle.full_backward(cfg, cams[v], scene, dL)
        for (o, sz), k in zip(offs, ("dmeans", "dlog_scales", "dquats", "dopacity_logits", "dsh")):
            flat[o:o + sz] += r[k].reshape(-1)
    return flat


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_00219_b200.shard import allreduce_grads, views_for_rank
    scene = synth.make_scene(400, "outdoor", 3)
    mine = views_for_rank(rank, world, N_VIEWS)
    buf = torch.from_numpy(_flat_grads(scene, mine))
    allreduce_grads(buf)
    out[rank] = buf.numpy().copy()
    dist.barrier()
    dist.destroy_process_group()


def test_views_for_rank_partition():
    from paper_2605_00219_b200.shard import views_for_rank
    for world in (1, 2, 3, 4, 8):
        got = sorted(v for r in range(world) for v in views_for_rank(r, world, 8))
        assert got == list(range(8))


def test_gloo_world2_allreduce_equals_sequential_sum():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    scene = synth.make_scene(400, "outdoor", 3)
    ref = _flat_grads(scene, range(N_VIEWS))
    assert np.abs(ref).max() > 0
    for r in range(2):
        np.testing.assert_allclose(out[r], ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    np.testing.assert_array_equal(out[0], out[1])
