"""Host enqueue cost vs device time of the train step (is the host ever the bottleneck?).

  python scripts/host_enqueue.py   -> JSON: per step host enqueue us and device us, cfg2 and cfg3
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_01582_b200 import Context  # noqa: E402
from paper_2503_01582_b200.trainer import train_many  # noqa: E402

out = {}
for wl_name in ("cfg2", "cfg3"):
    sys.argv = ["bench.py", "--workload", wl_name, "--mlp", "bf16x3"]
    args = bench.parse()
    ctx = Context(0)
    wl = bench.WORKLOADS[wl_name](args, ctx, 0, 1)
    wl.step(5)
    ctx.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream)
    res = {}
    for k in (2, 5, 20, 50):  # short calls: pure enqueue; long ones fill the launch queue and wait on the GPU
        l0 = ctx.launch_count()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        t0 = time.perf_counter()
        wl.step(k)
        t_host = time.perf_counter() - t0
        b.record(stream)
        ctx.synchronize()
        t_dev = a.elapsed_time(b) / 1e3
        res[k] = {"host_enqueue_us_per_step": round(t_host / k * 1e6, 1), "device_us_per_step": round(t_dev / k * 1e6, 1),
                  "launches_per_step": round((ctx.launch_count() - l0) / k, 1)}
    out[wl_name] = res
    for o in wl.objs:
        o.close()
    ctx.close()
print(json.dumps(out))
