"""Reference-shaped Python host API over the C ABI (include/prenom/prenom_gpu.h).

Names and argument meaning follow the reference's object-trainer surface in
/root/reference/proj/core (namespace ``noma``):

==========================  ==============================================
this module                 reference
==========================  ==============================================
``FieldArch``               ``noma::FieldArch``      field.hpp:20-31
``Camera`` / ``Pose``       ``noma::Camera`` / ``Pose`` render.hpp:13-23, geom.hpp:120-131
``TrainConfig``             ``MapperConfig`` hot keys mapper.hpp:80-103
``ObjectTrainer.create``    train_track CREATE block  mapper.cpp:133-143
``ObjectTrainer.train_step`` train_track loop body    mapper.cpp:150-184
``ObjectTrainer.render``    field_eval + composite    render.hpp:79
``ObjectTrainer.density_query`` refresh_grid          density_grid.cpp:119-132
``UsageError`` etc.         errors.hpp:9-24
==========================  ==============================================

Every compute call goes through the CUDA library; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
import weakref
from dataclasses import dataclass, field, fields

import numpy as np

from . import _capi
from ._capi import BoxC, CameraC, FieldArchC, PoseC, StepStatsC, TrainCfgC, fptr, iptr, u8ptr, u32ptr


# --------------------------------------------------------------- errors
class PrenomError(RuntimeError):
    code = -1


class UsageError(PrenomError):  # noma::UsageError
    code = _capi.PRENOM_USAGE


class DataError(PrenomError):  # noma::DataError
    code = _capi.PRENOM_DATA


class NumericError(PrenomError):  # noma::NumericError
    code = _capi.PRENOM_NUMERIC


class CudaError(PrenomError):
    code = _capi.PRENOM_CUDA


_ERRORS = {c.code: c for c in (UsageError, DataError, NumericError, CudaError)}


def _check(status: int):
    if status != 0:
        msg = _capi.load().prenom_last_error()
        msg = msg.decode() if msg else ""
        raise _ERRORS.get(status, PrenomError)(msg)


# ---------------------------------------------------------- value types
@dataclass
class FieldArch:
    """noma::FieldArch (field.hpp:20-31); defaults are the reference's."""

    hash_levels: int = 8
    features_per_level: int = 2
    log2_table_size: int = 14
    base_resolution: int = 4
    per_level_scale: float = 1.45
    hidden_width: int = 32
    hidden_layers: int = 2
    density_activation: int = _capi.ACT_EXP_CLAMPED

    def to_c(self) -> FieldArchC:
        return FieldArchC(*[getattr(self, f.name) for f in fields(self)])

    # field.cpp:122-139
    def hash_param_count(self) -> int:
        return self.hash_levels * self.features_per_level * (1 << self.log2_table_size)

    def mlp_param_count(self) -> int:
        n, i = 0, self.hash_levels * self.features_per_level
        for _ in range(self.hidden_layers):
            n += self.hidden_width * i + self.hidden_width
            i = self.hidden_width
        return n + 4 * i + 4

    def param_count(self) -> int:
        return self.hash_param_count() + self.mlp_param_count()

    def level_resolution(self, level: int) -> int:
        """field.cpp:113-116 (double pow over the float scale)."""
        r = self.base_resolution * math.pow(float(np.float32(self.per_level_scale)), level)
        return max(1, int(r))

    @staticmethod
    def scale_for(base: int, max_res: int, levels: int) -> float:
        """Per-level scale reaching max_res at the top level."""
        s = float(np.float32((max_res / base) ** (1.0 / (levels - 1))))
        # nudge up one float ulp at a time until the top level is not truncated below max_res
        while FieldArch(hash_levels=levels, base_resolution=base, per_level_scale=s).level_resolution(levels - 1) < max_res:
            s = float(np.nextafter(np.float32(s), np.float32(2.0)))
        return s


def _mat_rowmajor(R) -> list:
    return [float(x) for x in np.asarray(R, np.float32).reshape(9)]


@dataclass
class Pose:
    """noma::Pose: world = R @ local + t (geom.hpp:120-131)."""

    R: np.ndarray = field(default_factory=lambda: np.eye(3, dtype=np.float32))
    t: np.ndarray = field(default_factory=lambda: np.zeros(3, np.float32))

    def to_c(self) -> PoseC:
        p = PoseC()
        p.R[:] = _mat_rowmajor(self.R)
        p.t[:] = [float(x) for x in np.asarray(self.t, np.float32)]
        return p


@dataclass
class Camera:
    """noma::Camera (render.hpp:13-23); pose is camera -> world."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    pose: Pose = field(default_factory=Pose)

    def to_c(self) -> CameraC:
        c = CameraC()
        c.fx, c.fy, c.cx, c.cy = self.fx, self.fy, self.cx, self.cy
        c.width, c.height = self.width, self.height
        c.R[:] = _mat_rowmajor(self.pose.R)
        c.t[:] = [float(x) for x in np.asarray(self.pose.t, np.float32)]
        return c


@dataclass
class TrainConfig:
    """Hot keys of MapperConfig/InnerOptions/LossWeights (mapper.hpp:80-103,
    meta.hpp:14-19, render.hpp:93-96). Defaults are the mapper's."""

    rays_per_iter: int = 128
    bg_fraction: float = 0.25
    samples_per_ray: int = 24
    lambda_d: float = 0.1
    lambda_sigma: float = 1e-4
    coarse_samples: int = 32
    escape_eps: float = 1e-4
    grid_refresh_every: int = 50
    eta: float = 1e-2
    prior_sampling: int = 1
    band_px: int = 8
    mlp_precision: int = _capi.MLP_FP32
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8

    def to_c(self) -> TrainCfgC:
        return TrainCfgC(*[getattr(self, f.name) for f in fields(self)])


def mix_seed(base: int, salt: int) -> int:
    """mapper.cpp:20-26 (per-track seed derivation)."""
    M = (1 << 64) - 1
    s = (base * 0x9E3779B97F4A7C15 + salt * 0xC2B2AE3D27D4EB4F + 1) & M
    s ^= s >> 31
    s = (s * 0x94D049BB133111EB) & M
    s ^= s >> 29
    return (s ^ (s >> 32)) & 0xFFFFFFFF


def derive_seed(base: int, salt: int) -> int:
    """meta.cpp:14-20 (per-meta-step seed derivation)."""
    M = (1 << 64) - 1
    s = (base * 0x9E3779B97F4A7C15 + salt * 0xBF58476D1CE4E5B9 + 1) & M
    s ^= s >> 31
    s = (s * 0x94D049BB133111EB) & M
    s ^= s >> 29
    return (s ^ (s >> 32)) & 0xFFFFFFFF


MAX_GRID_RES = 1024  # prenom_object_create / prenom_set_grid / prenom_density_query

# -------------------------------------------------------------- context
class Context:
    """One per GPU (prenom_ctx_create)."""

    def __init__(self, device: int = 0):
        self.lib = _capi.load()
        h = C.c_void_p()
        _check(self.lib.prenom_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self._objects = weakref.WeakSet()  # live ObjectTrainers: destroyed before the context

    def close(self):
        if getattr(self, "h", None):
            for o in list(self._objects):
                o.close()
            self.lib.prenom_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(self.lib.prenom_ctx_stream(self.h, C.byref(s)))
        return s.value or 0

    def synchronize(self):
        _check(self.lib.prenom_ctx_synchronize(self.h))

    def set_grouping(self, enable: bool):
        """Grouped launches for same-arch objects in train_many (prenom_ctx_set_grouping)."""
        _check(self.lib.prenom_ctx_set_grouping(self.h, int(bool(enable))))

    def launch_count(self) -> int:
        n = C.c_int64()
        _check(self.lib.prenom_ctx_launch_count(self.h, C.byref(n)))
        return n.value

    def init_comm(self, nranks: int, rank: int, unique_id: bytes):
        """Bind an NCCL communicator (prenom_ctx_init_comm) for prenom_reptile_step."""
        if len(unique_id) != _capi.COMM_ID_BYTES:
            raise UsageError("NCCL unique id must be 128 bytes")
        buf = (C.c_uint8 * _capi.COMM_ID_BYTES).from_buffer_copy(unique_id)
        _check(self.lib.prenom_ctx_init_comm(self.h, nranks, rank, buf))

    def comm_info(self) -> tuple[int, int, int]:
        """(nranks or 0 when unbound, rank, NCCL version code)."""
        n, r, v = C.c_int32(), C.c_int32(), C.c_int32()
        _check(self.lib.prenom_ctx_comm_info(self.h, C.byref(n), C.byref(r), C.byref(v)))
        return n.value, r.value, v.value


def comm_unique_id() -> bytes:
    """ncclGetUniqueId on this process (rank 0), as bytes to broadcast."""
    lib = _capi.load()
    buf = (C.c_uint8 * _capi.COMM_ID_BYTES)()
    _check(lib.prenom_comm_unique_id(buf))
    return bytes(buf)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# --------------------------------------------------------------- trainer
class ObjectTrainer:
    """A per-object NeRF (hash grid + MLP + density grid + Adam) resident on one GPU."""

    def __init__(self, ctx: Context, handle, arch: FieldArch, cfg: TrainConfig, grid_res: int):
        self.ctx, self.h, self.arch, self.cfg, self.grid_res = ctx, handle, arch, cfg, grid_res
        self.lib = ctx.lib
        ctx._objects.add(self)

    @classmethod
    def create(cls, ctx: Context, arch: FieldArch, theta=None, grid=None, grid_res: int = 48,
               seed: int = 0, cfg: TrainConfig | None = None, box_min=(-0.5, -0.5, -0.5),
               box_max=(0.5, 0.5, 0.5)) -> "ObjectTrainer":
        """Create from a category prior (theta, grid) or from init_params(seed)."""
        cfg = cfg or TrainConfig()
        if grid is not None:
            grid = _f32(grid)
            grid_res = int(round(len(grid.reshape(-1)) ** (1 / 3)))
        th = None if theta is None else _f32(theta)
        h = C.c_void_p()
        a = arch.to_c()
        c = cfg.to_c()
        _check(ctx.lib.prenom_object_create(ctx.h, C.byref(a), fptr(th),
                                            fptr(None if grid is None else grid.reshape(-1)), grid_res, seed,
                                            C.byref(c), fptr(_f32(box_min)), fptr(_f32(box_max)), C.byref(h)))
        return cls(ctx, h, arch, cfg, grid_res)

    @classmethod
    def from_prior(cls, ctx: Context, prior, seed: int = 0, cfg: TrainConfig | None = None,
                   box_min=(-0.5, -0.5, -0.5), box_max=(0.5, 0.5, 0.5)) -> "ObjectTrainer":
        """Create from a category prior (a prior.PriorBundle, e.g. from load_prior):
        arch, θ and the density grid come from the bundle (mapper.cpp:133-137).
        Deviation: load_prior accepts grids up to 4096^3 (prior_bundle.cpp); the device
        sampler's grids are limited to 1024^3 (32-bit lattice indices), larger ones are a
        DataError here rather than a silent resample."""
        R = int(np.asarray(prior.grid).shape[0])
        if R > MAX_GRID_RES:
            raise DataError(f"from_prior: {R}^3 prior grid exceeds the device sampler's {MAX_GRID_RES}^3 limit")
        return cls.create(ctx, prior.arch, theta=prior.theta, grid=prior.grid, seed=seed, cfg=cfg,
                          box_min=box_min, box_max=box_max)

    def close(self):
        if getattr(self, "h", None):
            self.lib.prenom_object_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_frames(self, cams, rgb, depth, mask, instance_value: int = 1, obj_pose: Pose | None = None):
        arr = (CameraC * len(cams))()
        for i, c in enumerate(cams):
            arr[i] = c.to_c() if isinstance(c, Camera) else c
        pose = (obj_pose or Pose()).to_c()
        _check(self.lib.prenom_object_set_frames(self.h, len(cams), arr, fptr(_f32(rgb)), fptr(_f32(depth)),
                                                 u8ptr(np.ascontiguousarray(mask, np.uint8)), instance_value,
                                                 C.byref(pose)))
        self._frame_hw = (arr[0].height, arr[0].width)

    def synth_frames(self, cams, boxes, depth_noise: float = 0.0, missing_frac: float = 0.0, seed: int = 0,
                     obj_pose: Pose | None = None):
        """Render a box-union scene's views on the device into this object's frames
        (prenom_object_synth_frames). boxes: [(lo[3], hi[3], albedo[3])]."""
        cc = (CameraC * len(cams))(*[c.to_c() for c in cams])
        bb = (BoxC * len(boxes))()
        for i, (lo, hi, alb) in enumerate(boxes):
            bb[i].lo[:] = [float(x) for x in lo]
            bb[i].hi[:] = [float(x) for x in hi]
            bb[i].albedo[:] = [float(x) for x in alb]
        pose = (obj_pose or Pose()).to_c()
        _check(self.lib.prenom_object_synth_frames(self.h, len(cams), cc, len(boxes), bb, depth_noise, missing_frac,
                                                   seed, C.byref(pose)))
        self._frame_hw = (cams[0].height, cams[0].width)

    def get_frame(self, frame: int):
        """(rgb [H,W,3], depth [H,W], object pixel list, band pixel list) of one frame."""
        H, W = self._frame_hw
        rgb, dep = np.zeros((H, W, 3), np.float32), np.zeros((H, W), np.float32)
        no, nb = C.c_int32(), C.c_int32()
        _check(self.lib.prenom_object_get_frame(self.h, frame, None, None, C.byref(no), C.byref(nb), None, None))
        op, bp = np.zeros(no.value, np.int32), np.zeros(nb.value, np.int32)
        _check(self.lib.prenom_object_get_frame(self.h, frame, fptr(rgb), fptr(dep), C.byref(no), C.byref(nb),
                                                iptr(op), iptr(bp)))
        return rgb, dep, op, bp

    def upload_frame(self, frame: int, rgb, depth, mask):
        _check(self.lib.prenom_object_upload_frame(self.h, frame, fptr(rgb), fptr(depth), u8ptr(mask)))

    def train_step(self, n_steps: int = 1, stats: bool = True):
        """n_steps iterations; returns per-step loss dicts (or None when stats=False: async)."""
        if not stats:
            _check(self.lib.prenom_train_step(self.h, n_steps, None))
            return None
        out = (StepStatsC * n_steps)()
        _check(self.lib.prenom_train_step(self.h, n_steps, out))
        return [_stats(s) for s in out]

    def train_step_async(self, n_steps: int = 1, prefetch_next: bool = True) -> int:
        """Streaming step (prenom_train_step_async): returns a ticket for wait_stats."""
        t = C.c_uint64()
        _check(self.lib.prenom_train_step_async(self.h, n_steps, int(prefetch_next), C.byref(t)))
        self._async_n = getattr(self, "_async_n", {})
        self._async_n[t.value] = n_steps
        return t.value

    def wait_stats(self, ticket: int):
        """Per-step loss dicts of one train_step_async call (waits for that call only)."""
        n = self._async_n.pop(ticket, 1)
        out = (StepStatsC * n)()
        _check(self.lib.prenom_wait_stats(self.h, ticket, out))
        return [_stats(s) for s in out]

    def frame_at(self, step: int) -> int:
        f = C.c_int32()
        _check(self.lib.prenom_object_frame_at(self.h, step, C.byref(f)))
        return f.value

    def last_stats(self, n: int = 1):
        out = (StepStatsC * n)()
        _check(self.lib.prenom_object_last_stats(self.h, n, out))
        return [_stats(s) for s in out]

    def step(self) -> int:
        s = C.c_int64()
        _check(self.lib.prenom_object_step(self.h, C.byref(s)))
        return s.value

    def check(self):
        _check(self.lib.prenom_object_check(self.h))

    def render(self, origins, dirs):
        o, d = _f32(origins).reshape(-1, 3), _f32(dirs).reshape(-1, 3)
        n = len(o)
        rgb, dep = np.zeros((n, 3), np.float32), np.zeros(n, np.float32)
        _check(self.lib.prenom_render(self.h, n, fptr(o), fptr(d), fptr(rgb), fptr(dep)))
        return rgb, dep

    def density_query(self, R: int, update_sampling_grid: bool = False):
        out = np.zeros((R, R, R), np.float32)
        _check(self.lib.prenom_density_query(self.h, R, fptr(out.reshape(-1)), int(update_sampling_grid)))
        return out

    def extract_mesh(self, R: int, iso: float | None = None, iso_floor: float = 5.0):
        """train_track's tail on the device (mapper.cpp:186-187): density query at R,
        choose_iso unless `iso` is given, marching_cubes. Returns (vertices [V,3] in the
        unit cube, triangles [T,3] int32, iso used)."""
        nv, nt, used = C.c_int64(), C.c_int64(), C.c_float()
        _check(self.lib.prenom_extract_mesh(self.h, R, float("nan") if iso is None else iso, iso_floor,
                                            C.byref(used), C.byref(nv), C.byref(nt)))
        v = np.zeros((nv.value, 3), np.float32)
        t = np.zeros((nt.value, 3), np.int32)
        _check(self.lib.prenom_get_mesh(self.h, fptr(v), iptr(t)))
        return v, t, used.value

    def get_mesh_grid(self):
        """The R^3 σ lattice the last extract_mesh ran on (bake_prior's grid)."""
        R = C.c_int32()
        _check(self.lib.prenom_get_mesh_grid(self.h, C.byref(R), None))
        g = np.zeros((R.value,) * 3, np.float32)
        _check(self.lib.prenom_get_mesh_grid(self.h, C.byref(R), fptr(g.reshape(-1))))
        return g

    def extract_mesh_counts(self, R: int, iso: float | None = None, iso_floor: float = 5.0) -> int:
        """extract_mesh without the host copy (the mesh stays on the device); returns
        the triangle count."""
        nv, nt, used = C.c_int64(), C.c_int64(), C.c_float()
        _check(self.lib.prenom_extract_mesh(self.h, R, float("nan") if iso is None else iso, iso_floor,
                                            C.byref(used), C.byref(nv), C.byref(nt)))
        return nt.value

    def field_eval(self, xyz):
        x = _f32(xyz).reshape(-1, 3)
        n = len(x)
        sig, rgb = np.zeros(n, np.float32), np.zeros((n, 3), np.float32)
        _check(self.lib.prenom_field_eval(self.h, n, fptr(x), fptr(sig), fptr(rgb)))
        return sig, rgb

    def get_params(self):
        out = np.zeros(self.arch.param_count(), np.float32)
        _check(self.lib.prenom_get_params(self.h, fptr(out)))
        return out

    def set_params(self, theta):
        _check(self.lib.prenom_set_params(self.h, fptr(_f32(theta))))

    def get_grid(self):
        r = C.c_int32()
        _check(self.lib.prenom_get_grid(self.h, C.byref(r), None))
        out = np.zeros((r.value,) * 3, np.float32)
        _check(self.lib.prenom_get_grid(self.h, C.byref(r), fptr(out.reshape(-1))))
        return out

    def set_grid(self, grid):
        g = _f32(grid)
        _check(self.lib.prenom_set_grid(self.h, g.shape[0], fptr(g.reshape(-1))))

    def get_adam(self):
        P = self.arch.param_count()
        m, v = np.zeros(P, np.float32), np.zeros(P, np.float32)
        s = C.c_int64()
        _check(self.lib.prenom_get_adam(self.h, fptr(m), fptr(v), C.byref(s)))
        return m, v, s.value

    def set_adam(self, m, v, step: int):
        """Restore a checkpointed Adam state (resume; see checkpoint()/restore())."""
        _check(self.lib.prenom_set_adam(self.h, fptr(_f32(m)), fptr(_f32(v)), int(step)))

    def checkpoint(self) -> dict:
        """Everything a resumed object needs: θ, Adam (m, v, step), the sampling grid."""
        m, v, step = self.get_adam()
        return dict(theta=self.get_params(), m=m, v=v, step=step, grid=self.get_grid())

    def restore(self, ck: dict):
        self.set_params(ck["theta"])
        self.set_grid(ck["grid"])
        self.set_adam(ck["m"], ck["v"], ck["step"])

    def reset_adam(self):
        _check(self.lib.prenom_reset_adam(self.h))

    def copy_params_from(self, other: "ObjectTrainer"):
        """params <- other's params (device to device) and a fresh Adam (meta.cpp:31-34)."""
        _check(self.lib.prenom_object_copy_params(self.h, other.h))

    def set_seed(self, seed: int):
        _check(self.lib.prenom_object_set_seed(self.h, seed))

    def reptile_update(self, adapted: "ObjectTrainer", beta: float):
        """self <- (1-beta)*self + beta*adapted (meta.cpp:83-92), on the device."""
        _check(self.lib.prenom_reptile_update(self.h, adapted.h, beta))

    def debug_generate_rays(self, frame: int, step: int):
        n = self.cfg.rays_per_iter
        out = dict(origins=np.zeros((n, 3), np.float32), dirs=np.zeros((n, 3), np.float32),
                   kinds=np.zeros(n, np.int32), target_rgb=np.zeros((n, 3), np.float32),
                   target_depth=np.zeros(n, np.float32), pick_px=np.zeros(n, np.int32))
        _check(self.lib.prenom_debug_generate_rays(self.h, frame, step, fptr(out["origins"]), fptr(out["dirs"]),
                                                   iptr(out["kinds"]), fptr(out["target_rgb"]),
                                                   fptr(out["target_depth"]), iptr(out["pick_px"])))
        return out


def train_many(objs, n_steps: int = 1):
    arr = (C.c_void_p * len(objs))(*[o.h for o in objs])
    _check(objs[0].lib.prenom_train_step_many(arr, len(objs), n_steps))


def reptile_delta(meta: ObjectTrainer, adapted: ObjectTrainer, delta_ptr: int):
    _check(meta.lib.prenom_reptile_delta(meta.h, adapted.h, C.c_void_p(delta_ptr)))


def reptile_apply(meta: ObjectTrainer, delta_ptr: int, n_tasks: int, beta: float):
    _check(meta.lib.prenom_reptile_apply(meta.h, C.c_void_p(delta_ptr), n_tasks, beta))


def reptile_step(meta: ObjectTrainer, adapted: list, n_tasks: int, beta: float):
    """prenom_reptile_step: this rank's task deltas summed, all-reduced over the context's
    NCCL communicator (if bound), reptile_update(meta, mean adapted, beta) applied."""
    arr = (C.c_void_p * max(1, len(adapted)))(*[a.h for a in adapted])
    _check(meta.lib.prenom_reptile_step(meta.h, arr, len(adapted), n_tasks, beta))


def _stats(s: StepStatsC) -> dict:
    return dict(total=s.total, color=s.color_term, depth=s.depth_term, sigma=s.sigma_term,
                n_samples=s.n_samples, escaped=s.n_rays_escaped, frame=s.frame_index)


# ------------------------------------------------ single-stage debug calls
def debug_philox(ctx: Context, ctr_key):
    ck = np.ascontiguousarray(ctr_key, np.uint32).reshape(-1, 6)
    out = np.zeros((len(ck), 4), np.uint32)
    _check(ctx.lib.prenom_debug_philox(ctx.h, len(ck), u32ptr(ck), u32ptr(out)))
    return out


def debug_hash_encode(ctx: Context, arch: FieldArch, params, xyz):
    x = _f32(xyz).reshape(-1, 3)
    out = np.zeros((len(x), arch.hash_levels * arch.features_per_level), np.float32)
    a = arch.to_c()
    _check(ctx.lib.prenom_debug_hash_encode(ctx.h, C.byref(a), fptr(_f32(params)), len(x), fptr(x), fptr(out)))
    return out


def debug_field_eval(ctx: Context, arch: FieldArch, params, xyz, precision: int = _capi.MLP_FP32):
    x = _f32(xyz).reshape(-1, 3)
    n = len(x)
    sig, rgb, raw = np.zeros(n, np.float32), np.zeros((n, 3), np.float32), np.zeros((n, 4), np.float32)
    a = arch.to_c()
    _check(ctx.lib.prenom_debug_field_eval(ctx.h, C.byref(a), fptr(_f32(params)), n, fptr(x), fptr(sig), fptr(rgb),
                                           fptr(raw), precision))
    return sig, rgb, raw


def debug_field_backward(ctx: Context, arch: FieldArch, params, xyz, d_sigma, d_rgb,
                         precision: int = _capi.MLP_FP32):
    x = _f32(xyz).reshape(-1, 3)
    g = np.zeros(arch.param_count(), np.float32)
    a = arch.to_c()
    _check(ctx.lib.prenom_debug_field_backward(ctx.h, C.byref(a), fptr(_f32(params)), len(x), fptr(x),
                                               fptr(_f32(d_sigma)), fptr(_f32(d_rgb).reshape(-1)), fptr(g),
                                               precision))
    return g


def debug_adam(ctx: Context, params, grads, m, v, step, lr=1e-2, b1=0.9, b2=0.999, eps=1e-8):
    p, mm, vv = _f32(params).copy(), _f32(m).copy(), _f32(v).copy()
    s = C.c_int64(step)
    _check(ctx.lib.prenom_debug_adam(ctx.h, len(p), fptr(p), fptr(_f32(grads)), fptr(mm), fptr(vv), C.byref(s),
                                     lr, b1, b2, eps))
    return p, mm, vv, s.value


def debug_sample_rays(ctx: Context, origins, dirs, box_min, box_max, prior: bool, grid, n_coarse: int,
                      n_fine: int, eps: float, seed: int, step: int):
    o, d = _f32(origins).reshape(-1, 3), _f32(dirs).reshape(-1, 3)
    n = len(o)
    g = None if grid is None else _f32(grid)
    R = 0 if g is None else g.shape[0]
    out = dict(depths=np.zeros((n, n_fine), np.float32), deltas=np.zeros((n, n_fine), np.float32),
               positions=np.zeros((n, n_fine, 3), np.float32), count=np.zeros(n, np.int32),
               t_entry=np.zeros(n, np.float32), t_exit=np.zeros(n, np.float32))
    _check(ctx.lib.prenom_debug_sample_rays(ctx.h, n, fptr(o), fptr(d), fptr(_f32(box_min)), fptr(_f32(box_max)),
                                            int(prior), R, fptr(None if g is None else g.reshape(-1)), n_coarse,
                                            n_fine, eps, seed, step, fptr(out["depths"]), fptr(out["deltas"]),
                                            fptr(out["positions"]), iptr(out["count"]), fptr(out["t_entry"]),
                                            fptr(out["t_exit"])))
    return out


def debug_batch_loss(ctx: Context, S: int, kind, target_rgb, target_depth, count, deltas, depths, sigma, rgb,
                     bg_colors, lambda_d=0.1, lambda_sigma=1e-4):
    kind = np.ascontiguousarray(kind, np.int32)
    n = len(kind)
    terms = np.zeros(4, np.float64)
    ds, dr = np.zeros(n * S, np.float32), np.zeros((n * S, 3), np.float32)
    col, dep = np.zeros((n, 3), np.float32), np.zeros(n, np.float32)
    _check(ctx.lib.prenom_debug_batch_loss(ctx.h, n, S, iptr(kind), fptr(_f32(target_rgb).reshape(-1)),
                                           fptr(_f32(target_depth)), iptr(np.ascontiguousarray(count, np.int32)),
                                           fptr(_f32(deltas).reshape(-1)), fptr(_f32(depths).reshape(-1)),
                                           fptr(_f32(sigma).reshape(-1)), fptr(_f32(rgb).reshape(-1)),
                                           fptr(_f32(bg_colors).reshape(-1)), lambda_d, lambda_sigma,
                                           terms.ctypes.data_as(C.POINTER(C.c_double)), fptr(ds), fptr(dr),
                                           fptr(col), fptr(dep)))
    return dict(terms=terms, d_sigma=ds, d_rgb=dr, color=col, depth=dep)


def debug_umma_gemm(ctx: Context, A, B, a_mn: bool = False, b_mn: bool = False):
    """D = A @ B.T on one tcgen05 tile (bf16 in, fp32 out)."""
    A, B = _f32(A), _f32(B)
    M, K = A.shape
    N = B.shape[0]
    D = np.zeros((M, N), np.float32)
    _check(ctx.lib.prenom_debug_umma_gemm(ctx.h, M, N, K, int(a_mn), int(b_mn), fptr(A), fptr(B), fptr(D)))
    return D


def debug_marching_cubes(ctx: Context, grid, iso: float):
    """marching_cubes (marching_cubes.cpp:125-180) of a host grid [R][R][R] (z, y, x) on the device."""
    g = _f32(grid)
    R = g.shape[0]
    nv, nt = C.c_int64(), C.c_int64()
    _check(ctx.lib.prenom_debug_marching_cubes(ctx.h, R, fptr(g.reshape(-1)), iso, C.byref(nv), C.byref(nt)))
    v = np.zeros((nv.value, 3), np.float32)
    t = np.zeros((nt.value, 3), np.int32)
    _check(ctx.lib.prenom_debug_mesh_get(ctx.h, fptr(v), iptr(t)))
    return v, t


def mc_case_triangles(config: int):
    """The host case table (cube_case_triangles, marching_cubes.cpp:115-117) as edge triples."""
    out = np.zeros(16 * 3, np.int32)
    n = _capi.load().prenom_mc_case_triangles(config, iptr(out))
    if n < 0:
        raise ValueError("config out of range")
    return out[:3 * n].reshape(-1, 3)
