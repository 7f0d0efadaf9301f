"""Time the density query (refresh_grid lattice) through the C ABI: R^3 points/s."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_01582_b200 import Context, ObjectTrainer, scenes  # noqa: E402

ctx = Context(0)
for W in (64, 32):
    arch = scenes.cfg2_arch(W)
    ob = ObjectTrainer.create(ctx, arch, grid_res=8, seed=1)
    for R in (32, 128, 256):
        ob.density_query(R)
        ctx.synchronize()
        t = time.perf_counter()
        reps = 3
        for _ in range(reps):
            ob.density_query(R)
        ctx.synchronize()
        dt = (time.perf_counter() - t) / reps
        print(f"W{W} R={R}: {dt * 1e3:.3f} ms  {R ** 3 / dt:.3e} points/s")
    ob.close()
