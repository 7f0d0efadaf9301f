"""Seeded density grids for the mesh-extraction parity tests (shared by the
golden generator and tests/test_mesh.py). Grids are [R][R][R] = (z, y, x)."""
import numpy as np


def _lattice(R):
    ax = np.arange(R, dtype=np.float32) / np.float32(R - 1)
    return np.meshgrid(ax, ax, ax, indexing="ij")  # z, y, x


def GRIDS():
    rng = np.random.default_rng(20261019)
    out = {}
    z, y, x = _lattice(24)
    d2 = (x - 0.45) ** 2 + (y - 0.5) ** 2 + (z - 0.55) ** 2
    out["blob24"] = ((60.0 * np.exp(-d2 / 0.03)).astype(np.float32), None)  # iso = choose_iso
    z, y, x = _lattice(20)
    two = 40 * np.exp(-((x - 0.3) ** 2 + (y - 0.3) ** 2 + (z - 0.4) ** 2) / 0.01) + \
        40 * np.exp(-((x - 0.7) ** 2 + (y - 0.6) ** 2 + (z - 0.6) ** 2) / 0.02)
    out["two_blobs20"] = (two.astype(np.float32), 12.5)
    out["random10"] = (rng.uniform(0, 10, (10, 10, 10)).astype(np.float32), 5.0)  # every configuration family
    # values exactly at iso: vertices at t = 0 / 1, coincident vertices, zero-area triangles (cleanup_mesh)
    out["steps12"] = (rng.choice(np.float32([0, 5, 10]), (12, 12, 12)).astype(np.float32), 5.0)
    out["single_cell"] = (np.float32([[[0, 9], [9, 0]], [[9, 0], [0, 9]]]), 4.0)  # R = 2, ambiguous cell
    out["empty"] = (np.zeros((6, 6, 6), np.float32), 5.0)
    out["full"] = (np.full((6, 6, 6), 7.0, np.float32), 5.0)
    return out
