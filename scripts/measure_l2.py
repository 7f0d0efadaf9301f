"""L2 bandwidth peak on this B200 ("the L2 peak must be measured on the box").

Device-to-device copies of buffers that fit the 126 MB L2 (read + write bytes per copy),
and a read-only reduction, each repeated back to back after a warm-up and timed with CUDA
events; the best of several sizes is the L2 figure the encode kernels' lts__t_bytes rates
are compared against. Writes profiles/<tag>_l2_peak.json (or prints)."""
import json
import sys

import torch

tag = sys.argv[1] if len(sys.argv) > 1 else None
torch.cuda.init()
res = {"copy": {}, "read": {}}
for mb in (4, 8, 16, 24, 32, 48):
    n = mb * 2**20 // 4
    a = torch.randn(n, device="cuda")
    b = torch.empty_like(a)
    for _ in range(20):
        b.copy_(a)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 400
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        b.copy_(a)
    e.record()
    torch.cuda.synchronize()
    res["copy"][mb] = round(2 * n * 4 * reps / (s.elapsed_time(e) / 1e3) / 1e9, 1)
    out = torch.empty(1, device="cuda")
    for _ in range(20):
        torch.sum(a)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        torch.sum(a)
    e.record()
    torch.cuda.synchronize()
    res["read"][mb] = round(n * 4 * reps / (s.elapsed_time(e) / 1e3) / 1e9, 1)
big = torch.randn(1 << 28, device="cuda")  # 1 GiB: HBM for comparison
big2 = torch.empty_like(big)
big2.copy_(big)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
s.record()
for _ in range(10):
    big2.copy_(big)
e.record()
torch.cuda.synchronize()
res["hbm_copy_1GiB"] = round(2 * big.numel() * 4 * 10 / (s.elapsed_time(e) / 1e3) / 1e9, 1)
# the library's own probe: one launch re-reading an L2-resident buffer (no launch overheads)
import ctypes as C  # noqa: E402
import os  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01582_b200 import Context  # noqa: E402

ctx = Context(0)
res["kernel_read"] = {}
for mb in (16, 32, 48, 64, 96):
    g = C.c_double()
    ctx.lib.prenom_debug_l2_read(ctx.h, mb, 50, C.byref(g))
    res["kernel_read"][mb] = round(g.value, 1)
res["l2_peak_gbs"] = max(max(res["copy"].values()), max(res["read"].values()), max(res["kernel_read"].values()))
res["how"] = ("torch copy_ (read+write bytes) and sum (read bytes) of L2-resident fp32 buffers, 400 back-to-back "
              "launches after 20 warm-up; prenom_debug_l2_read: one launch re-reading an L2-resident buffer 50x "
              "(float4 __ldcg, 8 CTAs x 512 threads per SM); CUDA events; l2_peak_gbs = the best of all")
line = json.dumps(res)
print(line)
if tag:
    open(f"gpurun_out/{tag}_l2_peak.json", "w").write(line)
