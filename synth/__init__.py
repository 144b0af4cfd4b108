"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no projection, binning,
compositing or gradients): it only draws Gaussian clouds, cameras and upstream
gradients with the shapes and statistics of the paper's workloads
(Mip-NeRF-360-shaped scenes, P:7; sizes from BASELINE.json configs), following
the recipe in SURVEY.md §8(d) / DESIGN.md §5.  Everything is numpy with
``np.random.default_rng(seed)``, so both sides of a parity test receive
identical bytes.

Layouts (all float32, C-contiguous):
  means [N,3], log_scales [N,3], quats [N,4] (w,x,y,z, unnormalised allowed),
  opacity_logits [N], sh [N,K,3] with K = (D+1)^2 stored coefficients.
Camera: dict(R=[3,3] world->camera rows (OpenCV: x right, y down, z forward),
  t=[3], fx, fy, cx, cy, width, height).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "SceneConfig", "CONFIGS", "make_scene", "ring_cameras", "upstream_grad",
    "fd_fixture", "default_render_config", "scene_to_f64",
]


@dataclass(frozen=True)
class SceneConfig:
    name: str
    n: int
    width: int
    height: int
    kind: str          # "outdoor" | "indoor"
    n_views: int
    seed: int
    description: str


# BASELINE.json "configs" (index = scene seed, SURVEY §8d "Seeds")
CONFIGS = {
    "tiny": SceneConfig("tiny", 1_000, 64, 64, "outdoor", 1, 0,
                        "tiny synthetic scene: 1,000 random Gaussians, one 64x64 view"),
    "mcmc": SceneConfig("mcmc", 1_000_000, 1559, 1039, "indoor", 1, 1,
                        "MCMC-shaped scene: 1M Gaussians, bonsai-like indoor view 1559x1039"),
    "bicycle": SceneConfig("bicycle", 5_800_000, 1237, 822, "outdoor", 8, 2,
                           "bicycle-shaped: 5.8M Gaussians, 1237x822 outdoor view"),
    "garden": SceneConfig("garden", 5_000_000, 1297, 840, "outdoor", 8, 3,
                          "garden-shaped: 5.0M Gaussians, 1297x840, batch of 8 views"),
    "stress": SceneConfig("stress", 20_000_000, 2474, 1644, "outdoor", 8, 4,
                          "stress: 20M Gaussians at 2474x1644"),
}


def default_render_config(sh_degree: int = 3, sh_coeffs: int | None = None, bg=(0.0, 0.0, 0.0),
                          footprint: int = 0, fov_clamp: int = 1, near_plane: float = 0.01) -> dict:
    """Render configuration (DESIGN.md §4 readings A1-A16)."""
    K = (sh_degree + 1) ** 2
    return dict(sh_degree=sh_degree, sh_coeffs=K if sh_coeffs is None else sh_coeffs,
                near_plane=near_plane, bg=tuple(float(b) for b in bg),
                fov_clamp=fov_clamp, footprint=footprint)


def _unit_ball(rng, n):
    v = rng.standard_normal((n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    r = rng.random(n) ** (1.0 / 3.0)
    return v * r[:, None]


def make_scene(n: int, kind: str = "outdoor", seed: int = 0, sh_degree: int = 3) -> dict:
    """Mip-NeRF-360-shaped Gaussian cloud (SURVEY §8d "Synthetic scene generator").

    60% object (unit ball), 25% ground disk (r=4, z=-0.6, sigma_z=0.02),
    15% background (outdoor: upper-hemisphere shell, log-uniform radius in
    [5,30]; indoor: faces of the box [+-5,+-5,+-2.5]).  Log-scales are
    log(0.5*spacing) + N(0, 0.5^2) with spacing = (region measure / count)^(1/d).
    Order is randomly permuted (training appends Gaussians in no spatial order).
    """
    rng = np.random.default_rng(seed)
    n_obj = int(round(0.60 * n))
    n_gnd = int(round(0.25 * n))
    n_bg = n - n_obj - n_gnd

    pos_obj = _unit_ball(rng, n_obj)
    sp_obj = np.full(n_obj, (4.19 / max(n_obj, 1)) ** (1.0 / 3.0))

    r = 4.0 * np.sqrt(rng.random(n_gnd))
    th = 2 * np.pi * rng.random(n_gnd)
    pos_gnd = np.stack([r * np.cos(th), r * np.sin(th), -0.6 + 0.02 * rng.standard_normal(n_gnd)], 1)
    sp_gnd = np.full(n_gnd, (math.pi * 16 * 0.04 / max(n_gnd, 1)) ** (1.0 / 3.0))

    if kind == "outdoor":
        d = rng.standard_normal((n_bg, 3))
        d[:, 2] = 0.5 * np.abs(d[:, 2])
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        rad = np.exp(rng.uniform(np.log(5.0), np.log(30.0), n_bg))
        pos_bg = d * rad[:, None]
        sp_bg = rad * math.sqrt(2 * math.pi / max(n_bg, 1)) * 0.5
    elif kind == "indoor":
        half = np.array([5.0, 5.0, 2.5])
        face = rng.integers(0, 6, n_bg)
        p = rng.uniform(-1, 1, (n_bg, 3)) * half
        axis = face // 2
        sign = np.where(face % 2 == 0, -1.0, 1.0)
        p[np.arange(n_bg), axis] = sign * half[axis]
        pos_bg = p
        sp_bg = np.full(n_bg, math.sqrt(400.0 / max(n_bg, 1)) * 0.5)
    else:
        raise ValueError(kind)

    means = np.concatenate([pos_obj, pos_gnd, pos_bg], 0)
    spacing = np.concatenate([sp_obj, sp_gnd, sp_bg], 0)
    log_scales = np.log(0.5 * spacing)[:, None] + 0.5 * rng.standard_normal((n, 3))
    perm = rng.permutation(n)
    means = means[perm]
    log_scales = log_scales[perm]

    quats = rng.standard_normal((n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    opacity_logits = 2.0 * rng.standard_normal(n)
    K = (sh_degree + 1) ** 2
    # f0 ~ N(0, 0.6^2); f1..f15 uniform with std 0.1 (a uniform draw is 3x cheaper than a normal
    # one at 5.8M x 45 samples and only shapes the view-dependent colour)
    sh = rng.random((n, K, 3), dtype=np.float32)
    sh -= np.float32(0.5)
    sh *= np.float32(0.2 * math.sqrt(3.0))
    sh[:, 0, :] = 0.6 * rng.standard_normal((n, 3), dtype=np.float32)
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    return dict(means=f32(means), log_scales=f32(log_scales), quats=f32(quats),
                opacity_logits=f32(opacity_logits), sh=f32(sh))


def look_at(eye, target, up=(0.0, 0.0, 1.0)):
    """World->camera (R, t) for an OpenCV camera at `eye` looking at `target`."""
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd], 0)
    t = -R @ eye
    return R, t


def ring_cameras(width: int, height: int, kind: str = "outdoor", n_views: int = 8,
                 hfov_deg: float = 56.0) -> list:
    """8 cameras on a ring (angle 2*pi*k/8, radius 3.0 outdoor / 2.5 indoor, z=0.8), looking at
    the origin, fx=fy=W/(2 tan(HFOV/2)), principal point at the image centre."""
    radius = 3.0 if kind == "outdoor" else 2.5
    f = width / (2.0 * math.tan(math.radians(hfov_deg) / 2.0))
    cams = []
    for k in range(n_views):
        a = 2 * math.pi * k / n_views
        R, t = look_at((radius * math.cos(a), radius * math.sin(a), 0.8), (0.0, 0.0, 0.0))
        cams.append(dict(R=R.astype(np.float32), t=t.astype(np.float32), fx=np.float32(f),
                         fy=np.float32(f), cx=np.float32(width / 2.0), cy=np.float32(height / 2.0),
                         width=int(width), height=int(height)))
    return cams


def upstream_grad(height: int, width: int, seed: int) -> np.ndarray:
    """Synthetic dL/dimage ~ U(-1,1) per channel, [H,W,3] float32."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, (height, width, 3)).astype(np.float32)


def fd_fixture(seed: int, n: int = 8, footprint: int = 0):
    """Finite-difference fixture: <=8 Gaussians, one 16x16 tile,
    camera at the origin looking +z, fx=fy=20, cx=cy=8.  On seeds with seed % 4 == 1 one Gaussian
    sits at x/z ~ +-0.6 so the FOV clamp fires; bg=(0.1,0.2,0.3) on odd seeds."""
    rng = np.random.default_rng(10_000 + seed)
    depth = rng.uniform(2.0, 5.0, n)
    xz = rng.uniform(-0.5, 0.5, n)
    yz = rng.uniform(-0.5, 0.5, n)
    if seed % 4 == 1:
        xz[0] = 0.6 * (1 if rng.random() < 0.5 else -1) + rng.uniform(-0.02, 0.02)
    means = np.stack([xz * depth, yz * depth, depth], 1)
    log_scales = np.log(rng.uniform(0.05, 0.4, (n, 3)))
    quats = rng.standard_normal((n, 4))           # unnormalised: exercises the normalisation Jacobian
    opacity_logits = 1.5 * rng.standard_normal(n)
    sh = 0.3 * rng.standard_normal((n, 16, 3))
    sh[:, 0, :] += 1.0
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    scene = dict(means=f32(means), log_scales=f32(log_scales), quats=f32(quats),
                 opacity_logits=f32(opacity_logits), sh=f32(sh))
    cam = dict(R=np.eye(3, dtype=np.float32), t=np.zeros(3, np.float32), fx=np.float32(20.0),
               fy=np.float32(20.0), cx=np.float32(8.0), cy=np.float32(8.0), width=16, height=16)
    bg = (0.1, 0.2, 0.3) if seed % 2 == 1 else (0.0, 0.0, 0.0)
    cfg = default_render_config(3, bg=bg, footprint=footprint)
    dL = upstream_grad(16, 16, 20_000 + seed)
    return scene, cam, cfg, dL


def scene_to_f64(scene: dict) -> dict:
    return {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in scene.items()}
