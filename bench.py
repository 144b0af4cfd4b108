#!/usr/bin/env python
"""Benchmark of the VkSplat hot path on B200 (BASELINE.json metric:
"fwd+bwd rasterize iters/sec @5.8M Gaussians 1237x822; sort Gkeys/s; HBM GB/s").

A step = one training step's hot path per rank: a batch of ring views
of the synthetic bicycle-shaped scene — one batched projection forward, then index offsets + keys
+ radix sort + tile ranges, raster forward and raster backward per view, one batched projection
backward — plus (N > 1) the all-reduce of the per-Gaussian gradient buffer, chunked by Gaussian rows
and overlapped with the projection backward (row a9).  Views are sharded across ranks:
`--scaling strong` (default) splits one global batch of `--views` views (BASELINE config 4: "a
batch of 8 views sharded across 1/2/4/8"); `--scaling weak` gives every rank `--views` distinct
views of a ring of views x N cameras.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config bicycle]
                    [--scaling strong|weak] [--views 8] [--streams 4] [--split bin-high]
                    [--binning sync|async] [--graph] [--no-records]

Every view of the batch is in flight (`--streams`, 8 slots), each slot with a binning stream of high
priority and a raster stream (`--split`); the raster passes stage the projection's packed records
(`--no-records`: gather the separate arrays); `--binning async --graph` runs the host-sync-free
binning and replays the whole step as one CUDA graph (measured no faster).

Beside the step (not in `value`): `batch1` (the paper's iteration: one view at a time through the
single-view entry points), `train_step` (the step plus the optimizer, row f1: sharded
reduce-scatter / Adam / all-gather), the loss gradient, MCMC and densification rows.
Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (the reference arm of
this tier) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd rasterize iters/sec @5.8M Gaussians 1237x822; sort Gkeys/s; HBM GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="bicycle")
    ap.add_argument("--views", type=int, default=8,
                    help="views per step: the global batch (strong scaling) or per rank (weak scaling)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--ar-chunks", type=int, default=4,
                    help="N > 1: gradient all-reduce chunks, each overlapped with the next projection-bwd chunk")
    ap.add_argument("--no-batch1", action="store_true")
    ap.add_argument("--binning", default="sync", choices=["sync", "async"],
                    help="vks_bin_sort (one host sync per view) or vks_bin_sort_async (device-side counts)")
    ap.add_argument("--graph", action="store_true",
                    help="capture the whole step in a CUDA graph and replay it (needs --binning async)")
    ap.add_argument("--no-records", action="store_true",
                    help="raster passes gather the separate projection arrays instead of staging packed records")
    ap.add_argument("--streams", type=int, default=8, help="views in flight per rank")
    ap.add_argument("--split", default="bin-high", choices=["none", "bin-high", "raster-high", "same"],
                    help="binning and raster passes of a view on separate streams (with these priorities)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rows-every", type=int, default=8, help="oracle raster sample: every k-th tile row")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm_gbs=float(d["hbm_gbs"]), sm_max_mhz=float(d.get("sm_max_mhz", 1965.0)), src="measured")
    return dict(hbm_gbs=6650.0, sm_max_mhz=1965.0, src="fallback")


# ----------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["nvidia-smi unavailable"], samples=0)
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 9]
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return dict(sm_mhz=statistics.median(sm) if sm else None, sm_max_mhz=max(mx) if mx else None,
                    reasons=reasons, samples=len(rows))


# ----------------------------------------------------------------------------------- algorithmic work
def algorithmic_bytes(n, vis, m, dpasses=4, batch=1, K=16, records=True):
    """Per-view algorithmic HBM bytes of the HBM-bound stages, for the algorithms as built
    (DESIGN.md §6).  Parameters are fp32; sh has K coefficients per channel."""
    sh = 12 * K
    return dict(
        # batched forward, per view: the parameter rows (44 B geometry + opacity, the SH row) read
        # and the opacity (4 B) written once per batch of `batch` views (SH for all n: upper bound
        # of the Gaussians some view shows); radii + tiles written for all (12 B), the other 36 B
        # of outputs for the visible
        # ... plus the 36 B of 2D-gradient accumulators zeroed per Gaussian and view (g2d_zero)
        # ... plus, with records, the 48-B packed raster record of every visible Gaussian
        project_fwd=(44 + sh) * n / batch + 4 * n / batch + 12 * n + 36 * vis + 36 * n + (48 * vis if records else 0),
        # id-order scan (read tiles twice, write offsets) + compaction of the visible (read depth,
        # means2d, radii; write depth key, id, rect code) + `dpasses` depth passes over V (count
        # 4 B, scatter 8 B in / 8 B out) + depth-order scan (ids + gathered rect codes in, rect
        # codes out; rect codes in, slots out) + rect difference array (8 B) + key-pass count
        # (rect code + slot) + key-pass scatter (rect code, slot, id in; 8 B per key out) + the
        # last tile pass (count 4 B, scatter 8 B in, 4 B out per key)
        bin_sort=(12 * n + (20 + 16) * vis + dpasses * 20 * vis + (12 + 8) * vis + (8 + 4) * vis + 8 * vis
                  + 12 * vis + 16 * vis + 8 * m + (4 + 8 + 4) * m),
        # batched projection backward, per view: the parameter rows (236 B) read and the gradient
        # rows (236 B) written once per batch of `batch` views (all n rows: upper bound of the
        # Gaussians some view sees), radii of every row and 2D gradients + colours of the visible
        project_bwd=(40 + sh) * 2 * n / batch + 8 * n + (36 + 12) * vis,
    )


def raster_flops(visited, composited, replayed):
    """Algorithmic fp32 operations: per visited (pixel, Gaussian) pair 12 (sigma 9,
    exp 1, rho*G 1, clamp 1), per composited pair 9 more in the forward (3 fma + 3); the backward
    re-evaluates the replayed pairs (12) and spends 50 per composited pair on the 9 gradient terms."""
    return dict(raster_fwd=12 * visited + 9 * composited, raster_bwd=12 * replayed + 50 * composited)


def measured_traffic(stage, key="dram_bytes_per_launch"):
    """DRAM bytes (read + write) per launch of the stage's dominant kernel (or, key="issue_active",
    its issue-slot utilisation) from the newest committed `ncu --set full` capture (profiles/
    rNN_traffic.json, written by tools/traffic_from_ncu.py), or None when no capture is committed."""
    import glob
    cands = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))  # the newest round's capture
    path = cands[-1] if cands else ""
    try:
        with open(path) as f:
            t = json.load(f)
        return t["kernels"][stage][key]
    except (OSError, KeyError, ValueError):
        return None


# The paper's RTX 3090 stage times, bicycle, default densification (seconds per
# training run; the iteration count is not stated, 30k assumed (A28)): context only —
# another GPU, and N grows over training there while it is fixed at 5.8M here.
PAPER_CONTEXT = dict(
    source="PAPER.md P:61-76, RTX 3090, bicycle, default densification, seconds per training run",
    seconds=dict(project_fwd=32.6, index_offset=5.6, generate_keys=8.5, sorting=14.6, tile_ranges=0.5,
                 raster_fwd=31.9, raster_bwd=163.0, proj_bwd_plus_optimizer=236.2),
    ms_per_iter_at_30k_iters=dict(project_fwd=1.087, bin_sort=0.973, raster_fwd=1.063, raster_bwd=5.433,
                                  proj_bwd_plus_optimizer=7.873),
    note="iteration count not stated in the paper (30k assumed); N grows during training there")


# ----------------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2605_00219_b200 as P
    import synth
    from paper_2605_00219_b200.shard import GradientSync, ShardedAdam, partition_views

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} != --gpus {args.gpus}", file=sys.stderr)
    # VKS_BENCH_BACKEND=gloo with more ranks than GPUs: a functional check of the N > 1 code path
    # (partitions, chunked all-reduce, sharded optimizer) on a smaller box — not a measurement
    backend = os.environ.get("VKS_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    # launched by torchrun (even with one rank): the NCCL process group, barriers, max-over-ranks
    # timing and the gradient allreduce all run
    distributed = "WORLD_SIZE" in os.environ
    if distributed:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    c = synth.CONFIGS[args.config]
    cfg = synth.default_render_config(3)
    scene = synth.make_scene(c.n, c.kind, c.seed)
    # the views this rank renders every step (strong: its share of one global batch; weak: its own
    # batch of distinct views) and the ring they come from
    my_views, ring = partition_views(rank, world, args.views, args.scaling)
    views_per_step = args.views if args.scaling == "strong" else args.views * world  # all ranks
    cams = synth.ring_cameras(c.width, c.height, c.kind, ring)
    params = P.GaussianParams.from_host(scene, pad_to=world)  # equal row shards for the sharded optimizer
    del scene
    n = params.n
    B, S = len(my_views), max(1, args.streams)
    gsync = GradientSync(params, n_chunks=args.ar_chunks if world > 1 else 1)
    host_dL = {v: torch.from_numpy(synth.upstream_grad(c.height, c.width, c.seed + 1000 + v)) for v in set(my_views)}
    dLs = {v: t.cuda() for v, t in host_dL.items()}
    use_rec = not args.no_records
    rends = [P.ViewRenderer(n, c.width, c.height, records=use_rec) for _ in range(S)]
    for r in rends:  # size the key capacity once (untimed)
        for v in set(my_views):
            r.forward(cfg, cams[v], params)
        r._alloc_capacity(int(r.capacity * 1.1))
    main = torch.cuda.current_stream()
    streams = [torch.cuda.Stream() for _ in range(S)]
    # --split: per slot a binning stream and a raster stream (the view's raster waits for its
    # binning; the slot's next binning waits for the slot's previous raster: the buffers are shared)
    pb = {"bin-high": -1, "raster-high": 0, "same": 0}.get(args.split, 0)  # priorities (lower = higher)
    pr = {"bin-high": 0, "raster-high": -1, "same": 0}.get(args.split, 0)
    bin_streams = [torch.cuda.Stream(priority=pb) for _ in range(S)] if args.split != "none" else None
    ras_streams = [torch.cuda.Stream(priority=pr) for _ in range(S)] if args.split != "none" else None
    cfg_ow = dict(cfg, flags=P.FLAG_GRAD_OVERWRITE)
    # stage boundaries (CUDA events on the launching stream); the 2D-gradient accumulators that
    # raster_bwd adds into are zeroed by the batched projection forward (g2d_zero)
    stages = ["project_fwd", "bin_sort", "raster_fwd", "raster_bwd", "project_bwd"]

    copy_stream = torch.cuda.Stream()

    # per-view outputs that live until the batch's projection backward: colours and radii of the
    # projection, the 2D gradients of the raster backward (everything else is per-stream scratch)
    vbuf = []
    for _ in range(B):
        g2d = torch.zeros(9 * n, dtype=torch.float32, device="cuda")
        vbuf.append(dict(means2d=torch.empty(n, 2, device="cuda"),
                         conics=None if use_rec else torch.empty(n, 3, device="cuda"),  # the records carry them
                         depths=torch.empty(n, device="cuda"), tiles=torch.empty(n, dtype=torch.int32, device="cuda"),
                         colors=torch.empty(n, 3, device="cuda"),
                         radii=torch.empty(n, 2, dtype=torch.int32, device="cuda"), g2d=g2d,
                         dm2=g2d[: 2 * n].view(n, 2), dcon=g2d[2 * n: 5 * n].view(n, 3),
                         dcol=g2d[5 * n: 8 * n].view(n, 3), dop=g2d[8 * n:],
                         rec=torch.empty(n, 12, device="cuda") if use_rec else None,
                         m_dev=torch.zeros(1, dtype=torch.int64, device="cuda"),     # vks_bin_sort_async:
                         st_dev=torch.zeros(1, dtype=torch.int32, device="cuda")))   # M and status words
    opac = torch.empty(n, device="cuda")  # view-independent

    def project_fwd_batch(vcams, st):
        """The batch's projection forward: one pass over the parameters for all its views (row a1)."""
        nb = len(vcams)
        with torch.cuda.stream(st):
            P.vks_project_fwd_batch(cfg, vcams, params.means, params.log_scales, params.quats, params.opacity_logits,
                                    params.sh, [vbuf[j]["means2d"] for j in range(nb)],
                                    [vbuf[j]["conics"] for j in range(nb)], [vbuf[j]["depths"] for j in range(nb)],
                                    [vbuf[j]["radii"] for j in range(nb)], [vbuf[j]["tiles"] for j in range(nb)],
                                    [vbuf[j]["colors"] for j in range(nb)], opac,
                                    g2d_zero=[vbuf[j]["g2d"] for j in range(nb)],
                                    records=[vbuf[j]["rec"] for j in range(nb)] if use_rec else None)

    st_done_prev = [None] * S  # --split: the event after each slot's last raster pass

    def view_path(rend, vb, cam, dL, st, ev=None, copies=None, split_k=None):
        """One view's forward and raster backward on stream `st` (S views in flight, one stream
        each, or with split_k a binning and a raster stream per slot).  copies = (host target image, slot, loss slot): the e2e variant — the view's target
        image comes in from pinned host memory on a copy stream ("Copy Image to Device"),
        vks_loss_grad turns the rendered image and the target into the loss and dL/dimage on the
        device ("Loss Gradient"), and raster_bwd consumes that."""
        if copies is not None:
            host_src, slot, loss_out = copies  # loss_out None: the path's e2e (dL in, image out)
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(slot["in_free"])      # the slot's previous consumer is done
                slot["in"].copy_(host_src, non_blocking=True)
                slot["in_ready"].record(copy_stream)
        bst = st
        if split_k is not None:  # binning on the slot's binning stream, the raster passes on its raster stream
            bst, st = bin_streams[split_k], ras_streams[split_k]
            bst.wait_event(st_done_prev[split_k])
        with torch.cuda.stream(bst):
            if copies is not None and loss_out is None:
                bst.wait_event(slot["img_free"])             # the previous image has left rend.image
            if ev is not None: ev[1].record(bst)
            if args.binning == "async":  # no host sync: M and the status stay on the device
                P.vks_bin_sort_async(cam, vb["means2d"], vb["radii"], vb["depths"], vb["tiles"], rend.offsets,
                                     rend.vals, rend.tile_offsets, rend.workspace, vb["m_dev"], vb["st_dev"],
                                     tile_order=rend.tile_order)
                m = None
            else:
                m = P.vks_bin_sort(cam, vb["means2d"], vb["radii"], vb["depths"], vb["tiles"], rend.offsets, None,
                                   rend.vals, rend.tile_offsets, rend.workspace, tile_order=rend.tile_order)
                rend.num_isects = m
            if ev is not None: ev[2].record(bst)
        if bst is not st:
            bdone = torch.cuda.Event()
            bdone.record(bst)
            st.wait_event(bdone)
        with torch.cuda.stream(st):
            P.vks_raster_fwd(cfg, cam, vb["means2d"], vb["conics"], vb["colors"], opac, vb["radii"],
                             rend.vals, rend.tile_offsets, rend.image, rend.T_final, rend.n_contrib,
                             tile_order=rend.tile_order, records=vb["rec"])
            if copies is not None and loss_out is None:  # dL/dimage from the host, the image out
                slot["img_done"].record(st)
                with torch.cuda.stream(copy_stream):
                    copy_stream.wait_event(slot["img_done"])
                    slot["img_host"].copy_(rend.image, non_blocking=True)
                    slot["img_free"].record(copy_stream)
                st.wait_event(slot["in_ready"])
                dL = slot["in"]
            elif copies is not None:  # the target from the host, loss + dL/dimage on the device
                st.wait_event(slot["in_ready"])
                P.vks_loss_grad(rend.image, slot["in"], slot["dL"], loss_out, slot["ws"], lam=0.2)
                slot["in_free"].record(st)
                dL = slot["dL"]
            if ev is not None: ev[3].record(st)
            P.vks_raster_bwd(cfg, cam, vb["means2d"], vb["conics"], vb["colors"], opac, vb["radii"],
                             rend.vals, rend.tile_offsets, rend.T_final, rend.n_contrib, dL, vb["dm2"], vb["dcon"],
                             vb["dcol"], vb["dop"], tile_order=rend.tile_order, records=vb["rec"])
            if ev is not None: ev[4].record(st)
            if copies is not None and loss_out is None:
                slot["in_free"].record(st)
            done = torch.cuda.Event()
            done.record(st)
        if split_k is not None:
            st_done_prev[split_k] = done
        return m, done

    def project_bwd_batch(vcams, st, sync=None):
        """The batch's projection backward: one pass over the parameters for all its views,
        overwriting the gradient buffer (row a8).  With `sync` (N > 1), in Gaussian-row chunks,
        each chunk's gradient all-reduce (row a9) started as soon as its rows are written."""
        g = params.grads()
        nb = len(vcams)
        chunks = sync.chunks() if sync is not None else [(0, n)]
        with torch.cuda.stream(st):
            for r0, r1 in chunks:
                P.vks_project_bwd_batch(cfg_ow, vcams, params.means[r0:r1], params.log_scales[r0:r1],
                                        params.quats[r0:r1], params.opacity_logits[r0:r1], params.sh[r0:r1],
                                        [vbuf[j]["colors"][r0:r1] for j in range(nb)],
                                        [vbuf[j]["radii"][r0:r1] for j in range(nb)],
                                        [vbuf[j]["dm2"][r0:r1] for j in range(nb)],
                                        [vbuf[j]["dcon"][r0:r1] for j in range(nb)],
                                        [vbuf[j]["dcol"][r0:r1] for j in range(nb)],
                                        [vbuf[j]["dop"][r0:r1] for j in range(nb)], g["dmeans"][r0:r1],
                                        g["dlog_scales"][r0:r1], g["dquats"][r0:r1], g["dopacity_logits"][r0:r1],
                                        g["dsh"][r0:r1])
                if sync is not None:
                    sync.launch(r0, r1)
            if sync is not None:
                sync.finish()

    def step(s, copies=None, main=main):
        """One training step's hot path: a batch of B views per rank — one batched projection
        forward (row a1), then binning, raster forward and raster backward per view, alternating
        over S streams, one batched projection backward (row a8) and the allreduce (row a9; no-op
        at N = 1).  The batch starts after the previous step's allreduce (an optimizer would run
        there)."""
        vviews = my_views
        vcams = [cams[v] for v in vviews]
        project_fwd_batch(vcams, main)  # after the previous step's allreduce (main stream order)
        start = torch.cuda.Event()
        start.record(main)
        for st in streams:
            st.wait_event(start)
        if bin_streams is not None:
            for k in range(S):
                st_done_prev[k] = start
        m = 0
        for j, v in enumerate(vviews):
            k = j % S
            cp = None
            if copies is not None:
                cp = (copies[0][v], copies[1][k], None if copies[2] is None else copies[2][j:j + 1])
            m, done = view_path(rends[k], vbuf[j], cams[v], dLs[v], streams[k], copies=cp,
                                split_k=k if bin_streams is not None else None)
            main.wait_event(done)
        project_bwd_batch(vcams, main, gsync if world > 1 else None)  # + the chunked all-reduce (row a9)
        if copies is not None and copies[2] is not None:
            copies[3].copy_(copies[2], non_blocking=True)  # the batch's losses to pinned host memory
        elif copies is not None:
            main.wait_stream(copy_stream)  # every image of the batch has reached the host
        return m

    def timed(fn, nsteps):
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(main)
        for s in range(nsteps):
            fn(args.warmup + s)
        t1.record(main)
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        ms = t0.elapsed_time(t1)
        if distributed:
            tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        return ms

    for s in range(args.warmup):
        step(s)
    torch.cuda.synchronize()
    run_step = step
    if args.graph:
        if args.binning != "async":
            raise SystemExit("--graph needs --binning async (vks_bin_sort synchronises the host)")
        # the whole step captured once (project fwd batch, per view async binning + raster passes on
        # S forked streams, project bwd batch) and replayed: no host launches in the timed region
        graph = torch.cuda.CUDAGraph()
        cap_stream = torch.cuda.Stream()
        cap_stream.wait_stream(main)
        with torch.cuda.graph(graph, stream=cap_stream):
            step(0, main=cap_stream)
        torch.cuda.synchronize()

        def run_step(s):
            graph.replay()
    clocks = ClockSampler(local)
    clocks.start()
    ncu_range = bool(os.environ.get("VKS_NCU_RANGE"))  # `ncu --profile-from-start off`: timed steps only
    if ncu_range:
        torch.cuda.cudart().cudaProfilerStart()
    elapsed_ms = timed(run_step, args.steps)
    if ncu_range:
        torch.cuda.cudart().cudaProfilerStop()
    clk = clocks.stop()
    if args.binning == "async":  # every view's binning fitted its capacity (device status words)
        bad = [int(vb["st_dev"].item()) for vb in vbuf if int(vb["st_dev"].item()) != 0]
        if bad:
            raise SystemExit(f"vks_bin_sort_async status {bad}: capacity too small")
    views_total = views_per_step * args.steps
    value = views_total / (elapsed_ms / 1e3)

    # --- batch 1: the paper's iteration — one view at a time through
    # the single-view entry points (vks_project_fwd, vks_bin_sort, vks_raster_fwd, vks_raster_bwd,
    # vks_project_bwd) on one stream, CUDA events between them; views cycle over the rank's views
    batch1 = None
    if not args.no_batch1:
        rb = rends[0]
        rb_con = None if rb.records is not None else rb.conics  # the records carry the conics
        gb = params.grads()
        nb1 = max(24, args.steps)
        b1ev = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(nb1 + 3)]
        for i in range(nb1 + 3):
            cam = cams[my_views[i % B]]
            dLv = dLs[my_views[i % B]]
            e = b1ev[i]
            e[0].record(main)
            P.vks_project_fwd(cfg, cam, params.means, params.log_scales, params.quats, params.opacity_logits,
                              params.sh, rb.means2d, rb_con, rb.depths, rb.radii, rb.tiles, rb.colors,
                              rb.opacities, records=rb.records)
            e[1].record(main)
            P.vks_bin_sort(cam, rb.means2d, rb.radii, rb.depths, rb.tiles, rb.offsets, None, rb.vals,
                           rb.tile_offsets, rb.workspace, tile_order=rb.tile_order)
            e[2].record(main)
            P.vks_raster_fwd(cfg, cam, rb.means2d, rb_con, rb.colors, rb.opacities, rb.radii, rb.vals,
                             rb.tile_offsets, rb.image, rb.T_final, rb.n_contrib, tile_order=rb.tile_order,
                             records=rb.records)
            e[3].record(main)
            rb.g2d.zero_()  # the raster backward accumulates the view's 2D gradients
            P.vks_raster_bwd(cfg, cam, rb.means2d, rb_con, rb.colors, rb.opacities, rb.radii, rb.vals,
                             rb.tile_offsets, rb.T_final, rb.n_contrib, dLv, rb.dmeans2d, rb.dconics, rb.dcolors,
                             rb.dopacities, tile_order=rb.tile_order, records=rb.records)
            e[4].record(main)
            P.vks_project_bwd(cfg_ow, cam, params.means, params.log_scales, params.quats, params.opacity_logits,
                              params.sh, rb.colors, rb.radii, rb.dmeans2d, rb.dconics, rb.dcolors, rb.dopacities,
                              gb["dmeans"], gb["dlog_scales"], gb["dquats"], gb["dopacity_logits"], gb["dsh"])
            e[5].record(main)
        torch.cuda.synchronize()
        b1 = b1ev[3:]
        b1_total = b1[0][0].elapsed_time(b1[-1][5])
        b1_stage = {name: statistics.median([e[q].elapsed_time(e[q + 1]) for e in b1])
                    for q, name in enumerate(stages)}
        b1_vis = int((rb.tiles > 0).sum().item())
        batch1 = dict(value=round(len(b1) / (b1_total / 1e3), 3), unit="iters/s",
                      ms_per_iter=round(b1_total / len(b1), 4),
                      stages_ms={k: round(v, 4) for k, v in b1_stage.items()}, _vis=b1_vis, _m=rb.num_isects,
                      note=("the paper's iteration: one view at a time through the single-view entry points "
                            "on one stream (P:59, P:67-76; S:614-616), projection backward writing the "
                            "gradients (overwrite), the 2D-gradient memset inside raster_bwd; "
                            f"{len(b1)} timed views after 3 warm-up views"))

    # --- per-stage breakdown (its own timed region): views one at a time on one stream, CUDA
    # events between the entry points; medians over the views
    nv = max(B, min(64, (args.steps // B + 1) * B))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(stages))] for _ in range(nv)]
    pb_ms, pf_ms = [], []
    torch.cuda.synchronize()
    for i in range(nv):
        v = my_views[i % len(my_views)]
        if i % B == 0:  # the batch's projection forward, per view
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main)
            project_fwd_batch([cams[my_views[q % len(my_views)]] for q in range(i, i + B)], main)
            e1.record(main)
            pf_ms.append((e0, e1))
        view_path(rends[0], vbuf[i % B], cams[v], dLs[v], main, ev=evs[i])
        if i % B == B - 1:  # the batch's projection backward, per view
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main)
            project_bwd_batch([cams[my_views[q % len(my_views)]] for q in range(i - B + 1, i + 1)], main)
            e1.record(main)
            pb_ms.append((e0, e1))
    torch.cuda.synchronize()
    st_ms = {name: statistics.median([evs[i][q].elapsed_time(evs[i][q + 1]) for i in range(nv)])
             for q, name in enumerate(stages[:-1]) if q > 0}
    st_ms["project_fwd"] = statistics.median([a.elapsed_time(b) for a, b in pf_ms]) / B
    # the optimizer after the path (not part of the step or of `value`): one
    # Adam step over every parameter group per batch, timed on its own
    groups = [params.means, params.log_scales, params.quats, params.opacity_logits, params.sh]
    gr = params.grads()
    grads = [gr[k] for k in ("dmeans", "dlog_scales", "dquats", "dopacity_logits", "dsh")]
    mom = [torch.zeros_like(t) for t in groups]
    vel = [torch.zeros_like(t) for t in groups]
    lrs = dict(means=1.6e-4, log_scales=5e-3, quats=1e-3, opacity_logits=5e-2, sh=(2.5e-3, 1.25e-4))
    adam_ev = []
    for t in range(1, 6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        P.vks_adam_step(P.make_adam_config(lrs, step=t), groups, grads, mom, vel)
        e1.record(main)
        adam_ev.append((e0, e1))
    torch.cuda.synchronize()
    adam_ms = statistics.median([a.elapsed_time(b) for a, b in adam_ev[1:]])
    del mom, vel
    # the loss gradient before the path (in the e2e leg, not in `value`)
    tgt = torch.rand(c.height, c.width, 3, device="cuda")
    dl_tmp = torch.empty_like(tgt)
    loss_tmp = torch.empty(1, device="cuda")
    lws = torch.empty(P.vks_loss_workspace_bytes(c.width, c.height), dtype=torch.uint8, device="cuda")
    loss_ev = []
    for t in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        P.vks_loss_grad(rends[0].image, tgt, dl_tmp, loss_tmp, lws, lam=0.2)
        e1.record(main)
        loss_ev.append((e0, e1))
    torch.cuda.synchronize()
    loss_ms = statistics.median([a.elapsed_time(b) for a, b in loss_ev[1:]])
    del tgt, dl_tmp, lws
    # MCMC densification on a copy of the parameters: one relocation (every
    # 100 iterations in training) and one noise step (every iteration), timed on their own
    import copy as _copy
    pc = _copy.copy(params)
    pc.means, pc.log_scales, pc.quats = params.means.clone(), params.log_scales.clone(), params.quats.clone()
    pc.opacity_logits, pc.sh = params.opacity_logits.clone(), params.sh.clone()
    mws = torch.empty(P.vks_mcmc_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    ndead = torch.zeros(1, dtype=torch.int64, device="cuda")
    rel_ev, noi_ev = [], []
    for t in range(4):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(main)
        P.vks_mcmc_relocate(pc, mws, dead_opacity=0.005, seed=100 + t, n_dead=ndead)
        e1.record(main)
        P.vks_mcmc_noise(pc, 1.6e-4, 5e5, seed=100 + t, step=t)
        e2.record(main)
        rel_ev.append((e0, e1))
        noi_ev.append((e1, e2))
    torch.cuda.synchronize()
    mcmc = dict(row="f3 (SURVEY 8f): vks_mcmc_relocate + vks_mcmc_noise on the bench scene; not in value",
                relocate_ms=round(statistics.median([a.elapsed_time(b) for a, b in rel_ev[1:]]), 4),
                noise_ms=round(statistics.median([a.elapsed_time(b) for a, b in noi_ev[1:]]), 4),
                dead_last=int(ndead.item()))
    # default densification (row f4): the statistics of the batch's 8 views, then one event (out of
    # place into buffers with room for 2n), thresholds chosen so that ~5% of the Gaussians grow
    acc, den = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for j in range(B):
        P.vks_densify_stats(vbuf[j]["dm2"], vbuf[j]["radii"], acc, den)
    e1.record(main)
    torch.cuda.synchronize()
    stats_ms = e0.elapsed_time(e1) / B
    mg = (acc / den.clamp(min=1)).float()
    gthr = float(torch.quantile(mg[den > 0][:1 << 24].float(), 0.95).item()) if bool((den > 0).any()) else 1.0
    sthr = float(torch.quantile(params.log_scales.max(1).values.exp()[:1 << 24], 0.5).item())
    src = [params.means, params.log_scales, params.quats, params.opacity_logits, params.sh]
    dst = [torch.empty((2 * n,) + tuple(t.shape[1:]), device="cuda") for t in src]
    dws = torch.empty(P.vks_densify_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    dens_ev, n_new = [], 0
    for t in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        n_new = P.vks_densify(src, acc, den, dst, dws, gthr, sthr, 0.005, seed=t)
        e1.record(main)
        dens_ev.append((e0, e1))
    torch.cuda.synchronize()
    densify = dict(row="f4 (SURVEY 8f): vks_densify_stats per view + one vks_densify event; not in value",
                   stats_ms_per_view=round(stats_ms, 4),
                   densify_ms=round(statistics.median([a.elapsed_time(b) for a, b in dens_ev[1:]]), 4),
                   n_before=n, n_after=n_new)
    del pc, mws, dst, dws, acc, den
    st_ms["project_bwd"] = statistics.median([a.elapsed_time(b) for a, b in pb_ms]) / B
    st_ms = {k: st_ms[k] for k in stages}
    rend = rends[0]

    # --- workload statistics (untimed): visible count, M, raster pair counts of the last view
    vl = vbuf[(nv - 1) % B]  # the last view's projection outputs
    vis = int((vl["tiles"] > 0).sum().item())
    if args.binning == "async":
        rend.num_isects = int(vl["m_dev"].item())
    m_last = rend.num_isects
    stats = torch.zeros(6, dtype=torch.int64, device="cuda")
    P.vks_raster_fwd_stats(cfg, cams[my_views[(nv - 1) % len(my_views)]], vl["means2d"],
                           vl["conics"], vl["colors"], opac, vl["radii"], rend.vals, rend.tile_offsets, stats,
                           tile_order=rend.tile_order, records=vl["rec"])
    visited, composited, evaluated, replayed, warp_entries, warp_entries_comp = (int(x) for x in stats.tolist())
    # depth passes the sort ran: <= 8-bit digits over the visible depth-bit range
    dvis = vl["depths"][vl["tiles"] > 0].view(torch.int32).to(torch.int64)
    drange = int(dvis.max().item() - dvis.min().item()) if dvis.numel() else 0
    dpasses = max(1, (drange.bit_length() + 7) // 8)
    ab = algorithmic_bytes(n, vis, m_last, dpasses, batch=B, records=use_rec)
    fl = raster_flops(visited, composited, replayed)
    pk = peaks()
    clock_mhz = clk["sm_mhz"] or pk["sm_max_mhz"]
    fp32_peak_tflops = 148 * 128 * 2 * clock_mhz * 1e6 / 1e12
    per_stage = {}
    for k in ("project_fwd", "bin_sort", "project_bwd"):
        gbs = ab[k] / (st_ms[k] * 1e-3) / 1e9
        per_stage[k] = dict(ms=st_ms[k], bound="hbm", achieved=gbs, peak=pk["hbm_gbs"], unit="GB/s",
                            frac=gbs / pk["hbm_gbs"], algorithmic_bytes=ab[k])
    per_stage["bin_sort"]["gkeys_per_s"] = m_last / (st_ms["bin_sort"] * 1e-3) / 1e9
    adam_bytes = 28 * n * (11 + 3 * params.sh.shape[1])  # p, g, m, v in; p, m, v out (fp32)
    optimizer = dict(row="f1 (SURVEY 8f): vks_adam_step, once per step after the allreduce; not in value",
                     ms_per_step=round(adam_ms, 4), bound="hbm", algorithmic_bytes=adam_bytes,
                     achieved=round(adam_bytes / (adam_ms * 1e-3) / 1e9, 1), peak=pk["hbm_gbs"], unit="GB/s",
                     frac=round(adam_bytes / (adam_ms * 1e-3) / 1e9 / pk["hbm_gbs"], 4))
    loss_bytes = 36 * c.width * c.height  # render + target in, dL/dimage out (fp32 RGB)
    loss_grad = dict(row="f2 (SURVEY 8f): vks_loss_grad (L1 + 0.2 D-SSIM), once per view in the e2e leg; "
                         "not in value", ms_per_view=round(loss_ms, 4), algorithmic_bytes=loss_bytes,
                     achieved_gbs=round(loss_bytes / (loss_ms * 1e-3) / 1e9, 1),
                     note="fp64 window sums; the fp64 partial maps (72 B per pixel) round-trip through L2")
    per_stage["bin_sort"]["depth_passes"] = dpasses
    for k in ("raster_fwd", "raster_bwd"):
        tf = fl[k] / (st_ms[k] * 1e-3) / 1e12
        per_stage[k] = dict(ms=st_ms[k], bound="alu", achieved=tf, peak=fp32_peak_tflops, unit="TFLOP/s",
                            frac=tf / fp32_peak_tflops, algorithmic_flops=fl[k])
    # the batched projection forward's fraction without the 2D-gradient zeroing it performs for the
    # raster backward (36 B per Gaussian and view: a memset moved into the kernel, not projection work)
    pf_bytes_proj = ab["project_fwd"] - 36 * n
    per_stage["project_fwd"]["frac_without_g2d_zero"] = (pf_bytes_proj / (st_ms["project_fwd"] * 1e-3) / 1e9
                                                         / pk["hbm_gbs"])
    # the dominant KERNEL: the longest of the single-kernel stages (bin_sort is a chain of ~25 short
    # kernels; its stage roofline is reported in stage_roofline)
    dom = max(("project_fwd", "raster_fwd", "raster_bwd", "project_bwd"), key=lambda k: per_stage[k]["ms"])
    d = per_stage[dom]
    # the raster kernels are issue-bound: beside the flop model, their warp-instruction
    # rate against the issue peak (4 schedulers x 148 SMs x the sampled clock), from the ncu-counted
    # instructions of one launch (committed capture, bicycle view 0) and this run's live launch time
    issue = {}
    for k, units in (("raster_fwd", ("evaluated_pairs", evaluated)), ("raster_bwd", ("replayed_pairs", replayed))):
        wi = measured_traffic(k, "warp_instructions_per_launch")
        if wi:
            ipk = 4 * 148 * clock_mhz * 1e6
            issue[k] = dict(warp_instructions_per_launch_ncu=int(wi),
                            achieved=round(wi / (st_ms[k] * 1e-3) / 1e9, 1), peak=round(ipk / 1e9, 1),
                            unit="G warp-instructions/s", frac=round(wi / (st_ms[k] * 1e-3) / ipk, 4),
                            lane_instructions_per_pair=round(32 * wi / max(1, units[1]), 2), per=units[0],
                            warp_instructions_per_warp_entry=round(wi / max(1, warp_entries), 1))
            per_stage[k]["issue"] = issue[k]
    roofline = dict(kernel=dom, bound=d["bound"], achieved=round(d["achieved"], 3), peak=round(d["peak"], 3),
                    unit=d["unit"], frac=round(d["frac"], 4), traffic=measured_traffic(dom),
                    issue_active_ncu=measured_traffic(dom, "issue_active"), issue=issue.get(dom),
                    peak_source=(pk["src"] + " HBM copy (MEASURED_PEAKS.json)" if d["bound"] == "hbm" else
                                 f"derived (no measured FP32 figure in MEASURED_PEAKS.json): 148 SM x 128 FP32 "
                                 f"lanes x 2 flop x {clock_mhz:.0f} MHz (median SM clock sampled in the timed "
                                 f"region)"))
    # our kernels per view: bin_sort = id scan (2) + dpasses x (count, scan, scatter) + depth-order
    # scan (2) + rect diff + tile count + tile passes x 3; raster fwd; raster bwd; plus one batched
    # project fwd and one chunked batched project bwd per step
    tp = max(1, ((rend.n_tiles - 1).bit_length() + 7) // 8)
    # (async binning: always four 8-bit depth passes, plus its status kernel)
    bin_launches = (2 + 3 * dpasses + 2 + 1 + 1 + 3 * tp) if args.binning == "sync" else (2 + 3 * 4 + 2 + 1 + 1 + 3 * tp + 1)
    gpu_launches = ((bin_launches + 1 + 1) * B + 1 + len(gsync.chunks() if world > 1 else [0])) * args.steps
    if batch1 is not None:
        # stage rooflines of the single-view kernels (DESIGN.md §6.3 per-unit bytes): projection
        # forward 60 B per Gaussian (geometry + opacity read, radii + tiles written) + 232 B per
        # visible one (SH row read, outputs written); projection backward with overwrite 244 B per
        # Gaussian (radii read, gradient row written) + 280 B per visible one (parameters, 2D
        # gradients and colour read); binning as in the step
        v1, m1 = batch1.pop("_vis"), batch1.pop("_m")
        b1_bytes = dict(project_fwd=60 * n + (232 + (48 if use_rec else 0)) * v1,
                        bin_sort=algorithmic_bytes(n, v1, m1, dpasses)["bin_sort"],
                        project_bwd=244 * n + 280 * v1)
        b1_roof = {}
        for k, b in b1_bytes.items():
            gbs = b / (batch1["stages_ms"][k] * 1e-3) / 1e9
            b1_roof[k] = dict(bound="hbm", achieved=round(gbs, 1), peak=pk["hbm_gbs"], unit="GB/s",
                              frac=round(gbs / pk["hbm_gbs"], 4), algorithmic_bytes=int(b))
        for k in ("raster_fwd", "raster_bwd"):
            tf = fl[k] / (batch1["stages_ms"][k] * 1e-3) / 1e12
            b1_roof[k] = dict(bound="alu", achieved=round(tf, 3), peak=round(fp32_peak_tflops, 3), unit="TFLOP/s",
                              frac=round(tf / fp32_peak_tflops, 4))
        b1_roof["bin_sort"]["gkeys_per_s"] = round(m1 / (batch1["stages_ms"]["bin_sort"] * 1e-3) / 1e9, 3)
        batch1["stage_roofline"] = b1_roof
        batch1["gpu_launches_per_iter"] = (2 + 3 * dpasses + 2 + 1 + 1 + 3 * tp) + 4

    out = dict(metric=METRIC, value=round(value, 3), unit="iters/s", n_gpus=world, steps=args.steps,
               warmup=args.warmup, ms_per_step=round(elapsed_ms / args.steps, 4), higher_is_better=True,
               scaling=args.scaling, vs_baseline=None, dtype="f32", data="synthetic",
               config=dict(workload=c.description + ", fwd+bwd", n_gaussians=n, width=c.width,
                           height=c.height, sh_degree=3, footprint="support", views_per_step=views_per_step,
                           raster_staging=("packed 48-B records, cp.async double-buffered per warp" if use_rec
                                           else "gather of the separate arrays"),
                           views_per_rank_per_step=B, streams=S, visible=vis, num_isects=m_last,
                           l2="inputs larger than L2 (params 1.37 GB, keys+vals 0.22 GB per view), no flush",
                           parallelism=f"view-sharded dp{world} ({args.scaling} scaling)",
                           step=(f"{B} ring views per rank ({views_per_step} per step in all): one batched projection "
                                 f"forward, binning and both raster passes per view ({S} views in flight"
                                 + (f"; per slot a binning stream and a raster stream, {args.split}" if args.split != "none"
                                    else ", one stream each") + "), one batched projection backward"
                                 + (f" in {len(gsync.chunks())} Gaussian-row chunks, each chunk's gradient "
                                    f"all-reduce (NCCL) overlapping the next chunk" if world > 1 else "")
                                 + "; unit = views")),
               stages_ms={k: round(v, 4) for k, v in st_ms.items()},
               stage_roofline={k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                               for k, v in per_stage.items()},
               sort_gkeys_per_s=round(per_stage["bin_sort"]["gkeys_per_s"], 3),
               hbm_gbs={k: round(per_stage[k]["achieved"], 1) for k in ("project_fwd", "bin_sort", "project_bwd")},
               raster_work=dict(visited_pairs=visited, composited_pairs=composited, evaluated_pairs=evaluated,
                                replayed_pairs=replayed, warp_entries=warp_entries,
                                warp_entries_composited=warp_entries_comp),
               roofline=roofline, gpu_launches=gpu_launches, clocks=clk, batch1=batch1, optimizer=optimizer,
               loss_grad=loss_grad, mcmc=mcmc, densify=densify, paper_context=PAPER_CONTEXT)

    if not args.no_e2e:
        # (1) the path end to end: each view's dL/dimage copied in from pinned host memory and its
        # rendered image copied out to pinned host memory, on a copy stream overlapping compute
        nbytes = c.height * c.width * 3 * 4
        wsb = P.vks_loss_workspace_bytes(c.width, c.height)

        def make_slots(loss_leg):
            out_slots = []
            for _ in range(S):
                sl = {"in": torch.empty(c.height, c.width, 3, device="cuda")}
                if loss_leg:
                    sl["dL"] = torch.empty(c.height, c.width, 3, device="cuda")
                    sl["ws"] = torch.empty(wsb, dtype=torch.uint8, device="cuda")
                else:
                    sl["img_host"] = torch.empty(c.height, c.width, 3, pin_memory=True)
                for e in ("in_free", "in_ready", "img_done", "img_free"):
                    sl[e] = torch.cuda.Event()
                    sl[e].record(main)
                out_slots.append(sl)
            return out_slots

        pinned = {v: t.pin_memory() for v, t in host_dL.items()}
        copies = (pinned, make_slots(False), None, None)
        for s in range(min(args.warmup, 3)):
            step(s, copies)
        ms = timed(lambda s: step(s, copies), args.steps)
        out["e2e"] = dict(value=round(world * B * args.steps / (ms / 1e3), 3), unit="iters/s",
                          h2d_bytes_per_step=B * nbytes, d2h_bytes_per_step=B * nbytes,
                          ms_per_step=round(ms / args.steps, 4),
                          note=("per view: dL/dimage in from pinned host memory and the rendered image out to "
                                "pinned host memory, on a copy stream overlapping compute, inside the timed region"))
        # (2) as a training iteration sees it: the target image in ("Copy Image to Device"),
        # loss + dL/dimage on the device (vks_loss_grad, L1 + 0.2 D-SSIM: SURVEY 8(f) row f2), the
        # batch's losses out
        import numpy as np
        targets = {v: torch.from_numpy(np.random.default_rng(c.seed + 3000 + v).random(
            (c.height, c.width, 3), dtype=np.float32)).pin_memory() for v in set(my_views)}
        losses, losses_host = torch.zeros(B, device="cuda"), torch.zeros(B, pin_memory=True)
        copies = (targets, make_slots(True), losses, losses_host)
        for s in range(min(args.warmup, 3)):
            step(s, copies)
        ms = timed(lambda s: step(s, copies), args.steps)
        out["e2e_with_loss"] = dict(value=round(world * B * args.steps / (ms / 1e3), 3), unit="iters/s",
                                    h2d_bytes_per_step=B * nbytes, d2h_bytes_per_step=B * 4,
                                    ms_per_step=round(ms / args.steps, 4), loss_view0=round(float(losses_host[0]), 6),
                                    note=("per view: the target image in from pinned host memory, loss + dL/dimage "
                                          "computed on the device (row f2), the batch's losses out; inside the "
                                          "timed region"))
    # --- the training step (beside `value`): the step plus the optimizer (row f1) in its sharded
    # form — reduce-scatter of the gradients, Adam on this rank's 1/N of the rows, all-gather of the
    # parameters (at N = 1: Adam on every row).  Last, because it moves the parameters.
    opt = ShardedAdam(params, lrs, rank, world)
    tcount = [0]

    def train(s):
        step(s)
        tcount[0] += 1
        opt.step(tcount[0])

    for s in range(2):
        train(s)
    tr_ms = timed(train, args.steps)
    out["train_step"] = dict(
        row="a1-a9 + f1: the step plus the sharded optimizer; not in value", value=round(
            views_per_step * args.steps / (tr_ms / 1e3), 3), unit="iters/s", ms_per_step=round(tr_ms / args.steps, 4),
        optimizer=("reduce-scatter + vks_adam_step on 1/%d of the rows + all-gather" % world if world > 1 else
                   "vks_adam_step on every row"),
        moments_bytes_per_rank=int(sum(t.numel() for t in opt.m) * 8))
    del opt
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, c, cfg)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------------- oracle (CPU)
def oracle_view_sample(c, cfg, view, rows_every, band_offset=0):
    """The oracle on one view: projection + binning in full, raster fwd+bwd on every `rows_every`-th
    tile row (starting at band_offset), projection backward in full.  Returns (seconds, estimate of
    the full-view seconds, description)."""
    import numpy as np

    import oracle
    import synth
    scene = synth.make_scene(c.n, c.kind, c.seed)
    cam = synth.ring_cameras(c.width, c.height, c.kind, 8)[view]
    dL = synth.upstream_grad(c.height, c.width, c.seed + 1000 + view)
    ty = np.arange(c.height) // 16
    rm = (((ty - band_offset) % rows_every) == 0).astype(np.uint8)
    t = {}
    t0 = time.perf_counter()
    proj = oracle.project_fwd(cfg, cam, scene)
    t["project_fwd"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.bin_sort(cfg, cam, proj)
    t["bin_sort"] = time.perf_counter() - t0
    # the oracle's rasterizer has a per-call part independent of the rows rendered (projection of
    # every Gaussian, the global depth order, candidate lists): timed with no rows, then only the
    # per-row remainder of the sampled call is scaled to the full image
    t0 = time.perf_counter()
    oracle.render(cfg, cam, scene, dL=dL, row_mask=np.zeros_like(rm))
    t["raster_fixed"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    r = oracle.render(cfg, cam, scene, dL=dL, row_mask=rm)
    t["raster_fwd_bwd_sampled"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.project_bwd(cfg, cam, scene, r)
    t["project_bwd"] = time.perf_counter() - t0
    frac = float(rm.sum()) / c.height
    per_row = max(0.0, t["raster_fwd_bwd_sampled"] - t["raster_fixed"])
    full = t["project_fwd"] + t["bin_sort"] + t["raster_fixed"] + per_row / frac + t["project_bwd"]
    return sum(t.values()), full, t, frac


def cpu_baseline(args, c, cfg):
    cores = os.cpu_count()
    secs, full, t, frac = oracle_view_sample(c, cfg, 0, args.cpu_rows_every)
    return dict(value=round(1.0 / full, 5), unit="iters/s", cores=cores, kind="oracle",
                sample=(f"{c.name} view 0: projection, binning and projection-bwd in full; raster fwd+bwd on "
                        f"every {args.cpu_rows_every}th tile row ({frac:.3f} of pixels; the per-row time scaled "
                        f"by 1/{frac:.3f}, the rasterizer's per-call part timed separately); {secs:.1f} s of "
                        f"CPU wall time on {cores} threads"),
                stage_seconds={k: round(v, 3) for k, v in t.items()})


def run_reference(args):
    """Reference arm of this tier: the CPU oracle, as it stands, on the host cores."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    c = synth.CONFIGS[args.config]
    cfg = synth.default_render_config(3)
    cores = os.cpu_count()
    budget_s = 240.0
    fulls, walls = [], []
    total = args.warmup + args.steps
    done = 0
    t_start = time.perf_counter()
    rows_every = 8  # one band in 8 per step (rotating), bounded per-step sample
    for s in range(total):
        secs, full, _, frac = oracle_view_sample(c, cfg, s % 8, rows_every, band_offset=s % rows_every)
        done += 1
        if s >= args.warmup or (s == total - 1 and not fulls):
            fulls.append(full)
            walls.append(secs)
        if time.perf_counter() - t_start > budget_s and fulls:
            break
    value = len(fulls) / sum(fulls)
    out = dict(metric=METRIC, value=round(value, 5), unit="iters/s", n_gpus=world, steps=args.steps,
               warmup=args.warmup, ms_per_step=round(1e3 * sum(fulls) / len(fulls), 2), higher_is_better=True,
               scaling="weak", vs_baseline=None, dtype="f32", data="synthetic", impl="reference",
               config=dict(workload=c.description + ", fwd+bwd", n_gaussians=c.n, width=c.width, height=c.height,
                           sh_degree=3, footprint="support", parallelism="cpu oracle (rank 0 only)"),
               cpu_baseline=dict(value=round(value, 5), unit="iters/s", cores=cores, kind="oracle",
                                 sample=(f"per step one ring view (unit: views/s, as ours); projection, binning, "
                                         f"projection-bwd in full, raster fwd+bwd on 1 of every {rows_every} tile "
                                         f"rows (rotating), its per-row time scaled to the full view; "
                                         f"{len(fulls)} timed steps run (240 s budget), {sum(walls):.1f} s wall")),
               e2e=dict(value=round(value, 5), unit="iters/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0),
               gpu_launches=0)
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
