"""Reconstruction metric of the genome evaluation: surface
sampling and Chamfer distance, as evaluate_genome (search.cpp:230-270) scores a
baked mesh against ground truth.

* ``sample_surface`` restates mesh.cpp:70-104 exactly, including its
  std::mt19937 stream (a bit-exact MT19937 + libstdc++ generate_canonical
  replica), so the same mesh and seed give the reference's points bit for bit.
  It is O(n log T) host bookkeeping on a mesh already copied out.
* ``chamfer`` (metrics.cpp:14-22): the O(|a|·|b|) nearest-neighbour search runs
  on the GPU (prenom_nearest_sq: brute force, squared distances in the
  reference's float operation order, exact minimum -- the kd-tree's pruning is
  exact, so its minima are these); the two means are then summed in the
  reference's sequential double order on the host. Bit-exact vs the reference.
* ``transformed`` (mesh.cpp:56-60) with the identity rotation the evaluation uses.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .trainer import DataError, _check, _f32, fptr

_TWO32 = float(2 ** 32)
_TWO64 = float(2 ** 64)


class _StdMt19937Canonical:
    """std::mt19937 seeded with a uint32 + std::uniform_real_distribution<double>(0, 1)
    as libstdc++ implements it: generate_canonical<double, 53> draws two 32-bit
    words, sum = w0 + w1 * 2^32 (double), u = sum / 2^64 (1 -> nextafter(1, 0))."""

    def __init__(self, seed32: int):
        self.bg = np.random.MT19937()
        self.bg._legacy_seeding(int(seed32) & 0xFFFFFFFF)  # init_genrand, as std::mt19937(seed)

    def uniforms(self, n: int) -> np.ndarray:
        w = self.bg.random_raw(2 * n).astype(np.float64).reshape(n, 2)
        u = (w[:, 0] + w[:, 1] * _TWO32) / _TWO64
        return np.where(u >= 1.0, np.nextafter(1.0, 0.0), u)


def triangle_areas(vertices, triangles) -> np.ndarray:
    """mesh.cpp:16-19 per triangle: 0.5 * sqrt(double(dot(n, n))), n = cross(b - a, c - a) in float."""
    v = _f32(vertices).reshape(-1, 3)
    t = np.asarray(triangles).reshape(-1, 3)
    a, b, c = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    u, w = b - a, c - a
    nx = u[:, 1] * w[:, 2] - u[:, 2] * w[:, 1]
    ny = u[:, 2] * w[:, 0] - u[:, 0] * w[:, 2]
    nz = u[:, 0] * w[:, 1] - u[:, 1] * w[:, 0]
    d = (nx * nx + ny * ny) + nz * nz  # float32, left to right
    return 0.5 * np.sqrt(d.astype(np.float64))


def sample_surface(vertices, triangles, n: int, seed: int) -> np.ndarray:
    """mesh.cpp:70-104: n area-weighted surface points [n, 3] float32."""
    v = _f32(vertices).reshape(-1, 3)
    t = np.asarray(triangles).reshape(-1, 3)
    if len(t) == 0:
        raise DataError("sample_surface: empty mesh")
    cumulative = np.cumsum(triangle_areas(v, t))  # sequential: total += area
    total = float(cumulative[-1])
    if not total > 0.0:
        raise DataError("sample_surface: degenerate mesh")
    rng = _StdMt19937Canonical((seed ^ (seed >> 32)) & 0xFFFFFFFF)
    u3 = rng.uniforms(3 * n).reshape(n, 3)  # per point: pick, r1, r2 (in draw order)
    idx = np.minimum(np.searchsorted(cumulative, u3[:, 0] * total, side="left"), len(t) - 1)
    r1 = u3[:, 1].astype(np.float32)
    r2 = u3[:, 2].astype(np.float32)
    flip = (r1 + r2) > np.float32(1.0)
    r1 = np.where(flip, np.float32(1.0) - r1, r1)
    r2 = np.where(flip, np.float32(1.0) - r2, r2)
    tri = t[idx]
    a, b, c = v[tri[:, 0]], v[tri[:, 1]], v[tri[:, 2]]
    return ((a + (b - a) * r1[:, None]) + (c - a) * r2[:, None]).astype(np.float32)


def transformed(vertices, scale, t) -> np.ndarray:
    """mesh.cpp:56-60 with Pose{identity, t}: v * scale (componentwise) + t, in float."""
    v = _f32(vertices).reshape(-1, 3)
    return (v * _f32(scale).reshape(1, 3) + _f32(t).reshape(1, 3)).astype(np.float32)


def nearest_sq(ctx, queries, points) -> np.ndarray:
    """Per query point, the minimum squared distance to `points` (device brute force)."""
    q, p = _f32(queries).reshape(-1, 3), _f32(points).reshape(-1, 3)
    out = np.zeros(len(q), np.float32)
    _check(ctx.lib.prenom_nearest_sq(ctx.h, len(q), fptr(q), len(p), fptr(p), fptr(out)))
    return out


def chamfer(ctx, a, b) -> float:
    """metrics.cpp:14-22: 0.5 * (mean_a dist(a, B) + mean_b dist(b, A))."""
    a, b = _f32(a).reshape(-1, 3), _f32(b).reshape(-1, 3)
    if len(a) == 0 or len(b) == 0:
        raise DataError("chamfer: empty cloud")
    dab = np.sqrt(nearest_sq(ctx, a, b)).astype(np.float64)  # float sqrt, then widened
    dba = np.sqrt(nearest_sq(ctx, b, a)).astype(np.float64)
    s_ab = float(np.add.accumulate(dab)[-1])  # sequential double sums, reference order
    s_ba = float(np.add.accumulate(dba)[-1])
    return 0.5 * (s_ab / float(len(a)) + s_ba / float(len(b)))


__all__ = ["sample_surface", "triangle_areas", "transformed", "nearest_sq", "chamfer", "C"]
