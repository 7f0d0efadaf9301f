"""Seeded synthetic RGB-D scenes with the shapes BASELINE.json names.

The reference's own generator (taskgen: shapes.cpp + sdf_render.cpp) renders
CSG categories from a hemisphere camera ring and is out of scope (SURVEY.md
G7); BASELINE's scenes differ (sphere / box unions, Fibonacci cameras). This
module keeps the reference conventions that matter to the train step:
  * depth = distance along the unit ray, 0 = missing (image.hpp:25,
    render.cpp:80-83);
  * mask = instance id (1 for the object, 0 background) (image.hpp:26);
  * pixel rays use integer pixel coordinates through
    Camera::pixel_direction (render.hpp:20-22, render.cpp:75);
  * camera pose is camera -> world with +z forward, x right, y down.
Vectorised numpy; a 50 x 256^2 box-union scene takes well under a second.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .trainer import Camera, FieldArch, Pose

SIGMA_PRIOR_SCALE = 50.0  # sigma [1/m] of a fully occupied prior voxel


@dataclass
class Scene:
    cams: list
    rgb: np.ndarray  # [n][H][W][3] f32
    depth: np.ndarray  # [n][H][W] f32
    mask: np.ndarray  # [n][H][W] u8
    box_min: np.ndarray
    box_max: np.ndarray
    obj_pose: Pose
    boxes: list | None = None  # [(lo, hi, albedo)] for box unions


def fibonacci_cameras(n: int, radius: float, width: int, height: int, fx: float, fy: float | None = None):
    """n cameras at Fibonacci-sphere positions looking at the origin."""
    fy = fx if fy is None else fy
    cams = []
    golden = np.pi * (3.0 - np.sqrt(5.0))
    for i in range(n):
        z = 1.0 - 2.0 * (i + 0.5) / n
        r = np.sqrt(max(0.0, 1.0 - z * z))
        th = golden * i
        pos = radius * np.array([r * np.cos(th), r * np.sin(th), z])
        fwd = -pos / np.linalg.norm(pos)
        up = np.array([0.0, 0.0, 1.0]) if abs(fwd[2]) < 0.95 else np.array([0.0, 1.0, 0.0])
        right = np.cross(fwd, up)
        right /= np.linalg.norm(right)
        down = np.cross(fwd, right)
        R = np.stack([right, down, fwd], axis=1).astype(np.float32)  # columns: cam axes in world
        cams.append(Camera(fx=float(fx), fy=float(fy), cx=width / 2.0, cy=height / 2.0, width=width,
                           height=height, pose=Pose(R=R, t=pos.astype(np.float32))))
    return cams


def _pixel_rays(cam: Camera):
    """World-frame origins/unit directions of every pixel (render.hpp:20-22)."""
    v, u = np.meshgrid(np.arange(cam.height, dtype=np.float32), np.arange(cam.width, dtype=np.float32),
                       indexing="ij")
    d = np.stack([(u - cam.cx) / cam.fx, (v - cam.cy) / cam.fy, np.ones_like(u)], -1)
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    dw = d @ np.asarray(cam.pose.R, np.float32).T
    return np.asarray(cam.pose.t, np.float32), dw


def _finish(rng, t_hit, albedo, depth_noise, missing_frac):
    hit = np.isfinite(t_hit)
    depth = np.where(hit, t_hit, 0.0).astype(np.float32)
    if depth_noise > 0:
        depth = np.where(hit, depth + rng.normal(0.0, depth_noise, depth.shape), 0.0).astype(np.float32)
    if missing_frac > 0:
        depth = np.where(rng.random(depth.shape) < missing_frac, 0.0, depth).astype(np.float32)
    rgb = np.where(hit[..., None], albedo, 0.0).astype(np.float32)
    return rgb, depth, hit.astype(np.uint8)


def sphere_scene(n_views=24, res=128, radius=0.35, cam_radius=1.5, fx=128.0, depth_noise=0.005,
                 missing_frac=0.0, seed=0) -> Scene:
    """BASELINE config 1: sphere r=0.35, albedo sin(7 xyz) * 0.5 + 0.5."""
    rng = np.random.default_rng(seed)
    cams = fibonacci_cameras(n_views, cam_radius, res, res, fx)
    rgbs, deps, masks = [], [], []
    for cam in cams:
        o, d = _pixel_rays(cam)
        b = d @ o
        c = o @ o - radius * radius
        disc = b * b - c
        t = -b - np.sqrt(np.maximum(disc, 0.0))
        t = np.where((disc > 0) & (t > 0), t, np.inf)
        p = o + d * np.where(np.isfinite(t), t, 0.0)[..., None]
        rgb, dep, m = _finish(rng, t, np.sin(7.0 * p) * 0.5 + 0.5, depth_noise, missing_frac)
        rgbs.append(rgb), deps.append(dep), masks.append(m)
    return Scene(cams, np.stack(rgbs), np.stack(deps), np.stack(masks),
                 np.full(3, -0.5, np.float32), np.full(3, 0.5, np.float32), Pose())


def random_boxes(rng, n_min=3, n_max=6, size_lo=0.05, size_hi=0.4, centre=0.3):
    n = int(rng.integers(n_min, n_max + 1))
    boxes = []
    for _ in range(n):
        size = rng.uniform(size_lo, size_hi, 3)
        ctr = rng.uniform(-centre, centre, 3)
        albedo = rng.uniform(0.1, 0.95, 3)
        boxes.append(((ctr - size / 2).astype(np.float32), (ctr + size / 2).astype(np.float32),
                      albedo.astype(np.float32)))
    return boxes


def box_union_scene(n_views=50, res=256, cam_radius=1.5, fx=None, depth_noise=0.0, missing_frac=0.0,
                    seed=0, boxes=None) -> Scene:
    """BASELINE configs 2-5: union of 3-6 random axis-aligned boxes with per-box albedo."""
    rng = np.random.default_rng(seed)
    boxes = boxes if boxes is not None else random_boxes(rng)
    fx = float(res) if fx is None else fx
    cams = fibonacci_cameras(n_views, cam_radius, res, res, fx)
    rgbs, deps, masks = [], [], []
    for cam in cams:
        o, d = _pixel_rays(cam)
        inv = 1.0 / np.where(np.abs(d) < 1e-12, 1e-12, d)
        t_best = np.full(d.shape[:2], np.inf, np.float32)
        alb = np.zeros(d.shape, np.float32)
        for lo, hi, a in boxes:
            ta, tb = (lo - o) * inv, (hi - o) * inv
            t0 = np.minimum(ta, tb).max(-1)
            t1 = np.maximum(ta, tb).min(-1)
            hit = (t0 <= t1) & (t1 > 0)
            t = np.where(hit, np.maximum(t0, 0.0), np.inf)
            better = t < t_best
            t_best = np.where(better, t, t_best)
            alb = np.where(better[..., None], a, alb)
        rgb, dep, m = _finish(rng, t_best, alb, depth_noise, missing_frac)
        rgbs.append(rgb), deps.append(dep), masks.append(m)
    return Scene(cams, np.stack(rgbs), np.stack(deps), np.stack(masks),
                 np.full(3, -0.5, np.float32), np.full(3, 0.5, np.float32), Pose(), boxes)


def box_union_mesh(boxes):
    """Ground-truth surface of a box union for the genome evaluation's Chamfer metric:
    every box's 12 outward triangles (faces inside other boxes are kept -- a
    surface-sampling target, not a watertight union). Returns (vertices [8n,3], triangles [12n,3])."""
    verts, tris = [], []
    quads = [(0, 2, 3, 1), (4, 5, 7, 6), (0, 1, 5, 4), (2, 6, 7, 3), (0, 4, 6, 2), (1, 3, 7, 5)]
    for b, (lo, hi, _) in enumerate(boxes):
        base = 8 * b
        for k in range(8):
            verts.append([hi[0] if k & 1 else lo[0], hi[1] if k & 2 else lo[1], hi[2] if k & 4 else lo[2]])
        for a, c, d, e in quads:
            tris.append([base + a, base + c, base + d])
            tris.append([base + a, base + d, base + e])
    return np.asarray(verts, np.float32), np.asarray(tris, np.int32)


def occupancy_prior(boxes, R=32, box_min=-0.5, box_max=0.5, dilate=1, blur=1, k=SIGMA_PRIOR_SCALE):
    """sigma-valued R^3 prior grid = k * blur(dilate(occupancy)) at vertices
    (i,j,k)/(R-1) of the normalised box, x-fastest (density_grid.hpp:15-35)."""
    g = np.linspace(box_min, box_max, R, dtype=np.float32)
    Z, Y, X = np.meshgrid(g, g, g, indexing="ij")  # index [k][j][i] -> x fastest in memory
    occ = np.zeros((R, R, R), np.float32)
    for lo, hi, _ in boxes:
        occ = np.maximum(occ, ((X >= lo[0]) & (X <= hi[0]) & (Y >= lo[1]) & (Y <= hi[1]) & (Z >= lo[2])
                               & (Z <= hi[2])).astype(np.float32))
    for _ in range(dilate):
        p = np.pad(occ, 1)
        occ = np.max(np.stack([p[a:a + R, b:b + R, c:c + R] for a in range(3) for b in range(3) for c in range(3)]),
                     axis=0)
    for _ in range(blur):
        p = np.pad(occ, 1, mode="edge")
        occ = np.mean(np.stack([p[a:a + R, b:b + R, c:c + R] for a in range(3) for b in range(3) for c in range(3)]),
                      axis=0)
    return (k * occ).astype(np.float32)


# BASELINE.json architectures.
def cfg1_arch() -> FieldArch:
    return FieldArch(hash_levels=8, features_per_level=2, log2_table_size=15, base_resolution=16,
                     per_level_scale=FieldArch.scale_for(16, 256, 8), hidden_width=32, hidden_layers=2)


def cfg2_arch(width: int = 64) -> FieldArch:
    return FieldArch(hash_levels=16, features_per_level=2, log2_table_size=19, base_resolution=16,
                     per_level_scale=FieldArch.scale_for(16, 1024, 16), hidden_width=width, hidden_layers=2)


def cfg4_arch() -> FieldArch:
    return FieldArch(hash_levels=16, features_per_level=2, log2_table_size=18, base_resolution=16,
                     per_level_scale=FieldArch.scale_for(16, 1024, 16), hidden_width=64, hidden_layers=2)
