"""Per-view orchestration of the five C-ABI calls (buffer management only; no arithmetic).

`GaussianParams` holds the device-resident parameters and their gradient buffer (one flat fp32
buffer of 59 floats per Gaussian at SH degree 3, sliced into the five gradient views, so the
multi-GPU allreduce is a single call).  `ViewRenderer` owns the per-view scratch buffers (projection
outputs, binning, image/aux, 2D gradients) sized for one camera resolution and regrows the
intersection capacity on VKS_ERR_CAPACITY.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _vks as V


GRAD_NAMES = ("dmeans", "dlog_scales", "dquats", "dopacity_logits", "dsh")


@dataclass
class GaussianParams:
    means: torch.Tensor
    log_scales: torch.Tensor
    quats: torch.Tensor
    opacity_logits: torch.Tensor
    sh: torch.Tensor
    grad_flat: torch.Tensor
    # storage rows (>= n): every parameter tensor is the first n rows of a zero-padded [rows, ...]
    # tensor and every gradient group spans `rows` rows, so that the groups split into equal
    # per-rank shards for the sharded optimizer (shard.ShardedAdam).  0 = n (no padding).
    rows: int = 0
    storage: tuple | None = None  # the padded parameter tensors (None when rows == n)

    @property
    def n(self) -> int:
        return self.means.shape[0]

    @property
    def n_rows(self) -> int:
        return self.rows or self.n

    @staticmethod
    def layout(n: int, K: int):
        """(offset, numel) of each gradient group inside grad_flat for n (storage) rows; groups
        start 256-byte aligned."""
        sizes = [3 * n, 3 * n, 4 * n, n, 3 * K * n]
        offs, o = [], 0
        for s in sizes:
            offs.append((o, s))
            o += (s + 63) // 64 * 64
        return offs, o

    @staticmethod
    def from_host(scene: dict, device="cuda", pad_to: int = 1) -> "GaussianParams":
        """pad_to: storage rows rounded up to a multiple of this (the world size of a sharded
        optimizer); the padding rows are zero and never rendered."""
        t = {k: torch.as_tensor(v).to(device=device, dtype=torch.float32).contiguous() for k, v in scene.items()}
        n, K = t["means"].shape[0], t["sh"].shape[1]
        rows = -(-n // pad_to) * pad_to if pad_to > 1 else n
        names = ("means", "log_scales", "quats", "opacity_logits", "sh")
        storage = None
        if rows != n:
            storage = tuple(torch.zeros((rows,) + tuple(t[k].shape[1:]), dtype=torch.float32, device=device)
                            for k in names)
            for st, k in zip(storage, names):
                st[:n].copy_(t[k])
            t = {k: st[:n] for st, k in zip(storage, names)}
        _, total = GaussianParams.layout(rows, K)
        g = torch.zeros(total, dtype=torch.float32, device=device)
        return GaussianParams(t["means"], t["log_scales"], t["quats"], t["opacity_logits"], t["sh"], g,
                              rows=rows if rows != n else 0, storage=storage)

    def _group_shapes(self, rows):
        K = self.sh.shape[1]
        return [(rows, 3), (rows, 3), (rows, 4), (rows,), (rows, K, 3)]

    def grads(self) -> dict:
        """Views into grad_flat: [dmeans | dlog_scales | dquats | dlogit | dsh] (group-major), n rows."""
        return {nm: g.view(*sh) for nm, g, sh in zip(GRAD_NAMES, self.grad_groups(0, self.n),
                                                      self._group_shapes(self.n))}

    def grad_groups(self, r0: int = 0, r1: int | None = None) -> list:
        """The five gradient groups restricted to storage rows [r0, r1) (flat views into grad_flat)."""
        r1 = self.n_rows if r1 is None else r1
        offs, _ = GaussianParams.layout(self.n_rows, self.sh.shape[1])
        cols = [3, 3, 4, 1, 3 * self.sh.shape[1]]
        return [self.grad_flat[o + r0 * c:o + r1 * c] for (o, _), c in zip(offs, cols)]

    def param_groups(self, r0: int = 0, r1: int | None = None) -> list:
        """The five parameter tensors restricted to storage rows [r0, r1) (padding rows included)."""
        full = self.storage if self.storage is not None else (self.means, self.log_scales, self.quats,
                                                              self.opacity_logits, self.sh)
        r1 = self.n_rows if r1 is None else r1
        return [t[r0:r1] for t in full]


class ViewRenderer:
    """Scratch buffers for one resolution; `forward` then `backward` run one view's hot path."""

    def __init__(self, n: int, width: int, height: int, device="cuda", capacity: int | None = None,
                 records: bool = True):
        """records: the projection also writes the packed raster records and both raster passes
        stage them with cp.async (include/vks.h); False: the rasterizer gathers the separate
        arrays (same results)."""
        self.device = device
        self.n, self.W, self.H = n, width, height
        self.TX, self.TY = (width + 15) // 16, (height + 15) // 16
        self.n_tiles = self.TX * self.TY
        e = lambda *s, dt=torch.float32: torch.empty(*s, dtype=dt, device=device)
        self.means2d, self.conics, self.depths = e(n, 2), e(n, 3), e(n)
        self.radii, self.tiles = e(n, 2, dt=torch.int32), e(n, dt=torch.int32)
        self.colors, self.opacities = e(n, 3), e(n)
        self.records = e(n, 12) if records else None
        self.offsets = e(n, dt=torch.uint32)
        self.tile_offsets = e(self.n_tiles + 1, dt=torch.uint32)
        self.tile_order = e(self.n_tiles, dt=torch.uint32)  # raster schedule (heaviest tiles first)
        self.image, self.T_final = e(height, width, 3), e(height, width)
        self.n_contrib = e(height, width, dt=torch.int32)
        self.g2d = torch.zeros(n * 9, dtype=torch.float32, device=device)
        self.dmeans2d = self.g2d[: 2 * n].view(n, 2)
        self.dconics = self.g2d[2 * n: 5 * n].view(n, 3)
        self.dcolors = self.g2d[5 * n: 8 * n].view(n, 3)
        self.dopacities = self.g2d[8 * n:]
        self.capacity = 0
        self._alloc_capacity(capacity if capacity is not None else max(1024, 4 * n))
        self.num_isects = 0

    def _alloc_capacity(self, cap: int):
        self.capacity = int(cap)
        self.keys = torch.empty(self.capacity, dtype=torch.uint64, device=self.device)
        self.vals = torch.empty(self.capacity, dtype=torch.uint32, device=self.device)
        ws = V.vks_bin_sort_workspace_bytes(self.n, self.capacity, self.n_tiles)
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=self.device)

    def forward(self, cfg, cam, P: GaussianParams, keys_unsorted=None, vals_unsorted=None, want_keys=False):
        """want_keys: also write the sorted u64 (tile|depth) keys (verification only; the
        rasterizer needs the sorted ids and the tile ranges)."""
        V.vks_project_fwd(cfg, cam, P.means, P.log_scales, P.quats, P.opacity_logits, P.sh, self.means2d,
                          self.conics, self.depths, self.radii, self.tiles, self.colors, self.opacities,
                          records=self.records)
        for attempt in range(2):
            m = V.vks_bin_sort(cam, self.means2d, self.radii, self.depths, self.tiles, self.offsets,
                               self.keys if want_keys else None,
                               self.vals, self.tile_offsets, self.workspace, keys_unsorted, vals_unsorted,
                               raise_capacity=False, tile_order=self.tile_order)
            if m >= 0:
                break
            if attempt == 1:  # the call is idempotent: a regrown capacity always fits the same M
                raise RuntimeError(f"vks_bin_sort: {-m} intersections exceed the regrown capacity {self.capacity}")
            self._alloc_capacity(int(-m * 1.25) + 1024)
        self.num_isects = m
        V.vks_raster_fwd(cfg, cam, self.means2d, self.conics, self.colors, self.opacities, self.radii, self.vals,
                         self.tile_offsets, self.image, self.T_final, self.n_contrib, tile_order=self.tile_order,
                         records=self.records)
        return self.image

    def backward(self, cfg, cam, P: GaussianParams, dL_dimage: torch.Tensor, zero_2d: bool = True,
                 accumulate: bool = True):
        """accumulate=False: this view's parameter gradients overwrite P.grad_flat (first view of a
        batch; rows of Gaussians this view does not see are zeroed) — no memset needed."""
        if zero_2d:
            self.g2d.zero_()
        if not accumulate:
            cfg = dict(cfg, flags=int(cfg.get("flags", 0)) | V.FLAG_GRAD_OVERWRITE)
        V.vks_raster_bwd(cfg, cam, self.means2d, self.conics, self.colors, self.opacities, self.radii, self.vals,
                         self.tile_offsets, self.T_final, self.n_contrib, dL_dimage, self.dmeans2d, self.dconics,
                         self.dcolors, self.dopacities, tile_order=self.tile_order, records=self.records)
        g = P.grads()
        V.vks_project_bwd(cfg, cam, P.means, P.log_scales, P.quats, P.opacity_logits, P.sh, self.colors, self.radii,
                          self.dmeans2d, self.dconics, self.dcolors, self.dopacities, g["dmeans"],
                          g["dlog_scales"], g["dquats"], g["dopacity_logits"], g["dsh"])
