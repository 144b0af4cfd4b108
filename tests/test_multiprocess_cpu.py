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


# ---- partitions, chunked all-reduce and the sharded optimizer ----------

def test_partition_views_strong_and_weak():
    from paper_2605_00219_b200.shard import partition_views
    for world in (1, 2, 4, 8):
        # strong: one global batch of 8 ring views, each rendered by exactly one rank
        got = [partition_views(r, world, 8, "strong") for r in range(world)]
        assert all(ring == 8 for _, ring in got)
        assert sorted(v for vs, _ in got for v in vs) == list(range(8))
        assert all(len(vs) == 8 // world for vs, _ in got)
        # weak: 8 distinct views per rank from a ring of 8 * world cameras, none rendered twice
        got = [partition_views(r, world, 8, "weak") for r in range(world)]
        assert all(ring == 8 * world for _, ring in got)
        assert sorted(v for vs, _ in got for v in vs) == list(range(8 * world))
        assert all(len(vs) == 8 for vs, _ in got)
    with pytest.raises(ValueError):
        partition_views(0, 16, 8, "strong")


def test_row_chunks_cover_rows():
    from paper_2605_00219_b200.shard import row_chunks
    for n, c in ((0, 4), (1, 4), (1000, 1), (1000, 3), (5_800_000, 4), (257, 8)):
        ch = row_chunks(n, c)
        assert ch[0][0] == 0 and ch[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(ch, ch[1:]))
        assert all(r0 % 256 == 0 for r0, _ in ch)
        assert len(ch) <= max(1, c)


N_ROWS = 203  # not a multiple of the world size: exercises the padded shards
LRS = dict(means=1.6e-4, log_scales=5e-3, quats=1e-3, opacity_logits=5e-2, sh=(2.5e-3, 1.25e-4))


def _rank_params(rank, world):
    """Replicated parameters (same seed on every rank) and this rank's own gradients."""
    from paper_2605_00219_b200.pipeline import GaussianParams
    scene = synth.make_scene(N_ROWS, "outdoor", 11)
    p = GaussianParams.from_host(scene, device="cpu", pad_to=world)
    rng = np.random.default_rng(1000 + rank)
    for g in p.grads().values():
        g.copy_(torch.from_numpy(rng.standard_normal(tuple(g.shape)).astype(np.float32)))
    return p


def _oracle_adam_fn(step, prm, grd, m, v):
    """CPU stand-in for vks_adam_step (the oracle's Adam, test-only)."""
    import oracle
    G = oracle.ADAM_GROUPS
    P_, M_, V_ = oracle.adam_step({k: t.numpy() for k, t in zip(G, prm)}, {k: t.numpy() for k, t in zip(G, grd)},
                                  {k: t.numpy() for k, t in zip(G, m)}, {k: t.numpy() for k, t in zip(G, v)},
                                  LRS, step=step)
    for k, a, b, c in zip(G, prm, m, v):
        a.copy_(torch.from_numpy(P_[k]))
        b.copy_(torch.from_numpy(M_[k]))
        c.copy_(torch.from_numpy(V_[k]))


def _shard_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_00219_b200.shard import GradientSync, ShardedAdam, allreduce_grads
    # (1) chunked all-reduce == one all-reduce of the whole buffer
    p = _rank_params(rank, world)
    ref = p.grad_flat.clone()
    allreduce_grads(ref)
    sync = GradientSync(p, n_chunks=3, align=64)
    assert len(sync.chunks()) > 1
    for r0, r1 in sync.chunks():
        sync.launch(r0, r1)
    sync.finish()
    out[f"chunk_equal_{rank}"] = bool(torch.equal(p.grad_flat, ref))
    # (2) sharded Adam (reduce-scatter, Adam on 1/world of the rows, all-gather), two steps
    p = _rank_params(rank, world)
    opt = ShardedAdam(p, LRS, rank, world, adam_fn=_oracle_adam_fn)
    assert opt.m[0].shape[0] == p.n_rows // world  # moments for this rank's rows only
    for t in (1, 2):
        opt.step(t)
    out[f"params_{rank}"] = [x.clone().numpy() for x in (p.means, p.log_scales, p.quats, p.opacity_logits, p.sh)]
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_chunked_allreduce_and_sharded_adam():
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert out["chunk_equal_0"] and out["chunk_equal_1"]
    # reference: replicated optimizer on the all-reduced gradients (single process, oracle Adam)
    ps = [_rank_params(r, world) for r in range(world)]
    gsum = {k: sum(p.grads()[k] for p in ps) for k in ps[0].grads()}
    G = oracle.ADAM_GROUPS
    prm = {k: t.numpy() for k, t in zip(G, (ps[0].means, ps[0].log_scales, ps[0].quats, ps[0].opacity_logits,
                                            ps[0].sh))}
    grd = {k: gsum[g].numpy() for k, g in zip(G, ("dmeans", "dlog_scales", "dquats", "dopacity_logits", "dsh"))}
    m = {k: np.zeros_like(a) for k, a in prm.items()}
    v = {k: np.zeros_like(a) for k, a in prm.items()}
    for t in (1, 2):
        prm, m, v = oracle.adam_step(prm, grd, m, v, LRS, step=t)
    for r in range(world):
        for k, got in zip(G, out[f"params_{r}"]):
            # the reduce-scatter sums in a different order than the reference's sum: a few ulp
            np.testing.assert_allclose(got, prm[k], rtol=2e-6, atol=1e-7, err_msg=f"rank {r} {k}")
    for a, b in zip(out["params_0"], out["params_1"]):
        np.testing.assert_array_equal(a, b)  # every rank ends with identical parameters
