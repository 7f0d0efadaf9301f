"""evaluate_genome on box-union tasks: CD for a few genomes + wall time."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_01582_b200 import Context, scenes  # noqa: E402
from paper_2503_01582_b200.prior import Genome  # noqa: E402
from paper_2503_01582_b200.search import EvalTask, SearchConfig, evaluate_genome  # noqa: E402


def task(seed):
    sc = scenes.box_union_scene(n_views=20, res=128, seed=seed)
    v, t = scenes.box_union_mesh(sc.boxes)
    return EvalTask(scene=sc, gt_vertices=v, gt_triangles=t)


ctx = Context(0)
train, test = [task(100 + i) for i in range(4)], [task(200 + i) for i in range(3)]
cfg = SearchConfig()  # reference defaults: 64 rays x 16 samples, 60 adapt iters, 32^3 grid, 2048 samples
for g in (Genome(), Genome(hash_levels=8, log2_table_size=14, hidden_width=32, meta_steps=60, inner_iters=15),
          Genome(hash_levels=2, log2_table_size=8, features_per_level=1, hidden_width=8, hidden_layers=1,
                 meta_steps=15, inner_iters=5)):
    t0 = time.perf_counter()
    ev = evaluate_genome(ctx, g, train, test, eval_seed=1, cfg=cfg)
    print(f"L{g.hash_levels} T{g.log2_table_size} W{g.hidden_width} N{g.meta_steps} q{g.inner_iters}: "
          f"cd={ev.cd:.4f} per-task={[round(c, 4) for c in ev.per_task_cd]} time_per_iter={ev.time_per_iter:.3e} "
          f"wall={time.perf_counter() - t0:.2f}s")
