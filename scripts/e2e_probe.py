import sys, time, ctypes as C
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2503_01582_b200 import Context, ObjectTrainer
class A: pass
args = A(); args.width = 64; args.rays = 8192; args.samples = 96; args.mlp = "bf16"
ctx = Context(0)
sc, grid, arch, cfg = bench.make_workload(args, 0)
obj = ObjectTrainer.create(ctx, arch, theta=None, grid=grid, seed=7, cfg=cfg, box_min=sc.box_min, box_max=sc.box_max)
obj.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
obj.train_step(20, stats=False); ctx.synchronize()
rgb_h = torch.from_numpy(np.ascontiguousarray(sc.rgb)).pin_memory()
dep_h = torch.from_numpy(np.ascontiguousarray(sc.depth)).pin_memory()
npx = sc.rgb.shape[1] * sc.rgb.shape[2]
fptr = C.POINTER(C.c_float)
lib = ctx.lib
stream = torch.cuda.ExternalStream(ctx.stream)
def upload(step):
    f = obj.frame_at(step)
    lib.prenom_object_upload_frame(obj.h, f, C.cast(rgb_h.data_ptr() + f * npx * 12, fptr), C.cast(dep_h.data_ptr() + f * npx * 4, fptr), None)
def run(n, do_upload, do_wait, prefetch=True):
    ctx.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0 = obj.step()
    a.record(stream)
    prev = None
    for i in range(n):
        if do_upload: upload(s0 + i + 1)
        tk = obj.train_step_async(1, prefetch_next=prefetch)
        if do_wait and prev is not None: obj.wait_stats(prev)
        prev = tk
    obj.wait_stats(prev)
    b.record(stream); ctx.synchronize()
    return a.elapsed_time(b) / n
def run_batch(n):
    ctx.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream); obj.train_step(n, stats=False); b.record(stream); ctx.synchronize()
    return a.elapsed_time(b) / n
for r in range(2):
    print("batch(100)          ", round(run_batch(100), 4))
    print("async no-up no-wait ", round(run(100, False, False), 4))
    print("async no-up wait    ", round(run(100, False, True), 4))
    print("async up wait       ", round(run(100, True, True), 4))
    print("async up wait nopref", round(run(100, True, True, False), 4))
