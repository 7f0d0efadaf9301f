"""Generate tests/golden/ref_mesh_golden.npz from the REFERENCE ITSELF:
marching_cubes (marching_cubes.cpp:125-180, incl. cleanup_mesh) and
choose_iso (density_grid.cpp:134-136) of the unmodified reference sources
(oracle/_ref/libnoma_ref.so) on small seeded grids. tests/test_mesh.py checks
the CUDA extraction against these where the compiled reference is absent.
Re-run: python tests/golden/make_golden_mesh.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import pyoracle  # noqa: E402
from mesh_grids import GRIDS  # noqa: E402


def main():
    pyoracle.build_oracle(ref=True)
    ref = pyoracle.Ref()
    out = {}
    for name, (grid, iso) in GRIDS().items():
        if iso is None:
            iso = ref.choose_iso(grid)
        v, t = ref.marching_cubes(grid, iso)
        out[f"{name}/grid"] = grid
        out[f"{name}/iso"] = np.float32(iso)
        out[f"{name}/vertices"] = v
        out[f"{name}/triangles"] = t
    out["case_table"] = np.array([np.pad(ref.cube_case_triangles(c).reshape(-1), (0, 48 - ref.cube_case_triangles(c).size),
                                         constant_values=-1) for c in range(256)], np.int32)
    np.savez_compressed(Path(__file__).with_name("ref_mesh_golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
