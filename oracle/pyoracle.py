"""TEST INFRASTRUCTURE ONLY: numpy-facing ctypes wrappers for

* ``Oracle`` -- oracle/_oracle/libprenom_oracle.so, the plain-C restatement
  with Philox draws (the bit-exact checker of the CUDA path), and
* ``Ref``    -- oracle/_ref/libnoma_ref.so, the unmodified reference sources
  behind oracle/ref_shim.cpp (pins the restatement; CPU baseline).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

from paper_2503_01582_b200._capi import (
    CameraC,
    FieldArchC,
    PoseC,
    StepStatsC,
    TrainCfgC,
    dptr,
    fptr,
    iptr,
    u8ptr,
    u32ptr,
)

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_oracle" / "libprenom_oracle.so"
REF_SO = HERE / "_ref" / "libnoma_ref.so"
REF_DIR = Path("/root/reference/proj")

f32p, f64p = C.POINTER(C.c_float), C.POINTER(C.c_double)
i32p, i64p = C.POINTER(C.c_int32), C.POINTER(C.c_int64)


def i64ptr(a):
    return a.ctypes.data_as(i64p)
u8p, u32p = C.POINTER(C.c_uint8), C.POINTER(C.c_uint32)
archp = C.POINTER(FieldArchC)


def build_oracle(ref: bool | None = None) -> None:
    """Compile the C oracle, and the reference library when its sources exist."""
    subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)
    if ref is None:
        ref = (REF_DIR / "core" / "src" / "field.cpp").exists()
    if ref:
        subprocess.run(["make", "-s", "-j8", "-C", str(HERE), "ref"], check=True)


def f32(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


def zeros(*shape):
    return np.zeros(shape, dtype=np.float32)


class RefArch(C.Structure):
    _fields_ = FieldArchC._fields_


class RefCamera(C.Structure):
    _fields_ = CameraC._fields_


class RefTrainCfg(C.Structure):
    _fields_ = [
        ("rays_per_iter", C.c_int32),
        ("bg_fraction", C.c_float),
        ("samples_per_ray", C.c_int32),
        ("lambda_d", C.c_float),
        ("lambda_sigma", C.c_float),
        ("coarse_samples", C.c_int32),
        ("escape_eps", C.c_float),
        ("grid_refresh_every", C.c_int32),
        ("eta", C.c_float),
        ("prior_sampling", C.c_int32),
    ]


def arch_c(arch) -> FieldArchC:
    if isinstance(arch, FieldArchC):
        return arch
    return arch.to_c()


def cams_c(cams):
    arr = (CameraC * len(cams))()
    for i, c in enumerate(cams):
        arr[i] = c if isinstance(c, CameraC) else c.to_c()
    return arr


class _Lib:
    def __init__(self, path: Path, sigs: dict):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing; build with oracle.pyoracle.build_oracle()")
        self.lib = C.CDLL(str(path))
        for name, (res, args) in sigs.items():
            fn = getattr(self.lib, name)
            fn.restype = res
            fn.argtypes = args


# --------------------------------------------------------------------------
class Oracle(_Lib):
    """The C restatement (Philox draws)."""

    def __init__(self):
        P = C.c_void_p
        sz = C.c_size_t
        sigs = {
            "po_philox": (None, [u32p, u32p, u32p]),
            "po_u01": (C.c_float, [C.c_uint32]),
            "po_det_exp": (C.c_double, [C.c_double]),
            "po_pick": (C.c_uint32, [C.c_uint32, C.c_uint32]),
            "po_level_resolution": (C.c_int, [archp, C.c_int]),
            "po_param_count": (sz, [archp]),
            "po_hash_param_count": (sz, [archp]),
            "po_vertex_table_row": (C.c_uint32, [archp, C.c_int, C.c_uint32, C.c_uint32, C.c_uint32]),
            "po_hash_encode": (None, [archp, f32p, f32p, f32p, u32p, f32p]),
            "po_field_eval": (C.c_int, [archp, f32p, f32p, f32p, f32p, f32p, f32p, f32p, f32p, u32p, f32p]),
            "po_field_backward": (None, [archp, f32p, f32p, C.c_float, f32p, f32p]),
            "po_adam_step": (None, [sz, f32p, f32p, f32p, f32p, i64p, C.c_float, C.c_float, C.c_float, C.c_float]),
            "po_uniform_samples": (C.c_int, [f32p, f32p, f32p, f32p, C.c_int, f32p, f32p, f32p, f32p, f32p]),
            "po_composite": (None, [C.c_int, f32p, f32p, f32p, f32p, f32p, f32p, f32p]),
            "po_composite_backward": (None, [C.c_int, f32p, f32p, f32p, f32p, f32p, C.c_float, f32p, f32p]),
            "po_batch_loss": (C.c_int, [C.c_int, i32p, f32p, f32p, i32p, i32p, f32p, f32p, f32p, f32p, f32p,
                                        C.c_float, C.c_float, f64p, f32p, f32p, f32p, f32p]),
            "po_dilation_band": (None, [C.c_int, C.c_int, u8p, C.c_uint8, C.c_int, u8p]),
            "po_generate_rays": (C.c_int, [C.POINTER(CameraC), f32p, f32p, u8p, C.c_uint8, C.POINTER(PoseC),
                                           C.c_int, C.c_float, C.c_int, u32p, f32p, f32p, i32p, f32p, f32p,
                                           i32p, i32p]),
            "po_generate_rays_philox": (C.c_int, [C.POINTER(CameraC), f32p, f32p, u8p, C.c_uint8,
                                                  C.POINTER(PoseC), C.c_int, C.c_float, C.c_int, C.c_uint64,
                                                  C.c_int64, f32p, f32p, i32p, f32p, f32p, i32p]),
            "po_trilerp": (C.c_float, [C.c_int, f32p, f32p]),
            "po_build_ray_cdf": (C.c_int, [C.c_int, f32p, C.c_int, f32p, f32p, C.c_float, f32p, f32p]),
            "po_inverse_transform_sample": (None, [f32p, f32p, f32p, f32p, C.c_float, C.c_float, C.c_int, f32p,
                                                   f32p, f32p, C.c_int, f32p, f32p, f32p, f32p]),
            "po_sample_ray": (C.c_int, [C.c_int, f32p, f32p, f32p, f32p, f32p, C.c_int, C.c_int, C.c_float,
                                        f32p, f32p, f32p, f32p, f32p, f32p]),
            "po_sample_ray_philox": (C.c_int, [C.c_int, f32p, f32p, f32p, f32p, f32p, C.c_int, C.c_int,
                                               C.c_float, C.c_uint64, C.c_uint32, C.c_int64, C.c_uint32,
                                               f32p, f32p, f32p, f32p, f32p]),
            "po_refresh_grid": (C.c_int, [archp, f32p, C.c_int, f32p]),
            "po_reptile_update": (None, [sz, f32p, f32p, C.c_float, f32p]),
            "po_object_create": (P, [archp, f32p, f32p, C.c_int, C.c_uint64, C.POINTER(TrainCfgC), f32p, f32p]),
            "po_object_destroy": (None, [P]),
            "po_object_set_frames": (C.c_int, [P, C.c_int, C.POINTER(CameraC), f32p, f32p, u8p, C.c_uint8,
                                               C.POINTER(PoseC)]),
            "po_object_train_step": (C.c_int, [P, C.c_int, C.POINTER(StepStatsC)]),
            "po_object_get_params": (None, [P, f32p]),
            "po_object_get_grid": (None, [P, f32p]),
            "po_object_step": (C.c_int64, [P]),
        }
        super().__init__(ORACLE_SO, sigs)

    # -- RNG
    def philox(self, ctr, key):
        c = np.ascontiguousarray(ctr, dtype=np.uint32)
        k = np.ascontiguousarray(key, dtype=np.uint32)
        out = np.zeros(4, np.uint32)
        self.lib.po_philox(u32ptr(c), u32ptr(k), u32ptr(out))
        return out

    # -- field
    def param_count(self, arch):
        return int(self.lib.po_param_count(C.byref(arch_c(arch))))

    def level_resolution(self, arch, level):
        return int(self.lib.po_level_resolution(C.byref(arch_c(arch)), level))

    def vertex_table_row(self, arch, level, x, y, z):
        return int(self.lib.po_vertex_table_row(C.byref(arch_c(arch)), level, x, y, z))

    def hash_encode(self, arch, params, xyz):
        a = arch_c(arch)
        L, F = a.hash_levels, a.features_per_level
        xyz = f32(xyz).reshape(-1, 3)
        params = f32(params)
        out = zeros(len(xyz), L * F)
        rows = np.zeros((len(xyz), L * 8), np.uint32)
        w = zeros(len(xyz), L * 8)
        for i in range(len(xyz)):
            self.lib.po_hash_encode(C.byref(a), fptr(params), fptr(xyz[i]), fptr(out[i]),
                                    u32ptr(rows[i]), fptr(w[i]))
        return out, rows, w

    def field_eval(self, arch, params, xyz, cache=False):
        a = arch_c(arch)
        xyz = f32(xyz).reshape(-1, 3)
        params = f32(params)
        n = len(xyz)
        L, F, W, H = a.hash_levels, a.features_per_level, a.hidden_width, a.hidden_layers
        sigma, rgb = zeros(n), zeros(n, 3)
        feat, pre, hid, raw = zeros(n, L * F), zeros(n, max(H * W, 1)), zeros(n, max(H * W, 1)), zeros(n, 4)
        st = 0
        for i in range(n):
            st |= self.lib.po_field_eval(C.byref(a), fptr(params), fptr(xyz[i]), fptr(sigma[i:i + 1]),
                                         fptr(rgb[i]), fptr(feat[i]), fptr(pre[i]), fptr(hid[i]),
                                         fptr(raw[i]), None, None)
        if cache:
            return sigma, rgb, dict(features=feat, pre=pre, hidden=hid, raw=raw, status=st)
        return sigma, rgb

    def field_backward(self, arch, params, xyz, d_sigma, d_rgb, grad=None):
        a = arch_c(arch)
        params = f32(params)
        xyz = f32(xyz).reshape(-1, 3)
        d_sigma = f32(d_sigma)
        d_rgb = f32(d_rgb).reshape(-1, 3)
        g = zeros(len(params)) if grad is None else f32(grad).copy()
        for i in range(len(xyz)):
            self.lib.po_field_backward(C.byref(a), fptr(params), fptr(xyz[i]), C.c_float(d_sigma[i]),
                                       fptr(d_rgb[i]), fptr(g))
        return g

    def adam_step(self, params, grads, m, v, step, lr=1e-2, b1=0.9, b2=0.999, eps=1e-8):
        p, m, v = f32(params).copy(), f32(m).copy(), f32(v).copy()
        g = f32(grads)
        s = C.c_int64(step)
        self.lib.po_adam_step(len(p), fptr(p), fptr(g), fptr(m), fptr(v), C.byref(s), lr, b1, b2, eps)
        return p, m, v, s.value

    # -- render
    def uniform_samples(self, o, d, bmin, bmax, n):
        dep, dl, pos = zeros(n), zeros(n), zeros(n, 3)
        te, tx = zeros(1), zeros(1)
        esc = self.lib.po_uniform_samples(fptr(f32(o)), fptr(f32(d)), fptr(f32(bmin)), fptr(f32(bmax)), n,
                                          fptr(dep), fptr(dl), fptr(pos), fptr(te), fptr(tx))
        return dict(escaped=bool(esc), depths=dep, deltas=dl, positions=pos, t_entry=te[0], t_exit=tx[0])

    def composite(self, sigma, rgb, deltas, depths):
        n = len(sigma)
        col, dep, tp = zeros(3), zeros(1), zeros(n)
        self.lib.po_composite(n, fptr(f32(sigma)), fptr(f32(rgb).reshape(-1)), fptr(f32(deltas)),
                              fptr(f32(depths)), fptr(col), fptr(dep), fptr(tp))
        return col, dep[0], tp

    def composite_backward(self, sigma, rgb, deltas, depths, d_color, d_depth):
        n = len(sigma)
        ds, dr = zeros(n), zeros(n, 3)
        self.lib.po_composite_backward(n, fptr(f32(sigma)), fptr(f32(rgb).reshape(-1)), fptr(f32(deltas)),
                                       fptr(f32(depths)), fptr(f32(d_color)), float(d_depth), fptr(ds), fptr(dr))
        return ds, dr

    def batch_loss(self, kind, target_rgb, target_depth, escaped, offsets, deltas, depths, sigma, rgb,
                   bg_colors, lambda_d=0.1, lambda_sigma=1e-4):
        kind = np.ascontiguousarray(kind, np.int32)
        esc = np.ascontiguousarray(escaped, np.int32)
        off = np.ascontiguousarray(offsets, np.int32)
        nr = len(kind)
        ns = int(off[-1])
        terms = np.zeros(4, np.float64)
        ds, dr = zeros(max(ns, 1)), zeros(max(ns, 1), 3)
        col, dep = zeros(nr, 3), zeros(nr)
        st = self.lib.po_batch_loss(nr, iptr(kind), fptr(f32(target_rgb).reshape(-1)), fptr(f32(target_depth)),
                                    iptr(esc), iptr(off), fptr(f32(deltas)), fptr(f32(depths)), fptr(f32(sigma)),
                                    fptr(f32(rgb).reshape(-1)), fptr(f32(bg_colors).reshape(-1)),
                                    lambda_d, lambda_sigma, dptr(terms), fptr(ds), fptr(dr), fptr(col), fptr(dep))
        return dict(status=st, terms=terms, d_sigma=ds[:ns], d_rgb=dr[:ns], color=col, depth=dep)

    def dilation_band(self, mask, value, band_px):
        m = np.ascontiguousarray(mask, np.uint8)
        out = np.zeros_like(m)
        self.lib.po_dilation_band(m.shape[1], m.shape[0], u8ptr(m), value, band_px, u8ptr(out))
        return out

    def generate_rays(self, cam, rgb, depth, mask, inst, pose, n, bg_fraction, band_px, picks=None,
                      seed=None, step=0):
        rgb, depth = f32(rgb), f32(depth)
        mask = np.ascontiguousarray(mask, np.uint8)
        out = dict(origins=zeros(n, 3), dirs=zeros(n, 3), kinds=np.zeros(n, np.int32), target_rgb=zeros(n, 3),
                   target_depth=zeros(n), pick_px=np.zeros(n, np.int32))
        cc = cam if isinstance(cam, CameraC) else cam.to_c()
        pc = pose if isinstance(pose, PoseC) else pose.to_c()
        args = (fptr(out["origins"]), fptr(out["dirs"]), iptr(out["kinds"]), fptr(out["target_rgb"]),
                fptr(out["target_depth"]), iptr(out["pick_px"]))
        if picks is not None:
            pk = np.ascontiguousarray(picks, np.uint32)
            st = self.lib.po_generate_rays(C.byref(cc), fptr(rgb), fptr(depth), u8ptr(mask), inst, C.byref(pc),
                                           n, bg_fraction, band_px, u32ptr(pk), *args, None)
        else:
            st = self.lib.po_generate_rays_philox(C.byref(cc), fptr(rgb), fptr(depth), u8ptr(mask), inst,
                                                  C.byref(pc), n, bg_fraction, band_px, seed, step, *args)
        out["status"] = st
        return out

    # -- density grid
    def trilerp(self, grid, p):
        g = f32(grid)
        return float(self.lib.po_trilerp(g.shape[0], fptr(g.reshape(-1)), fptr(f32(p))))

    def build_ray_cdf(self, grid, deltas, positions, eps):
        g = f32(grid)
        n = len(deltas)
        tp, cdf = zeros(n), zeros(n)
        esc = self.lib.po_build_ray_cdf(g.shape[0], fptr(g.reshape(-1)), n, fptr(f32(deltas)),
                                        fptr(f32(positions).reshape(-1)), eps, fptr(tp), fptr(cdf))
        return bool(esc), tp, cdf

    def sample_ray(self, grid, o, d, bmin, bmax, n_c, n_f, eps, uniforms=None, seed=0, tag=3, step=0, ray=0):
        g = f32(grid)
        dep, dl, pos = zeros(n_f), zeros(n_f), zeros(n_f, 3)
        te, tx = zeros(1), zeros(1)
        if uniforms is not None:
            esc = self.lib.po_sample_ray(g.shape[0], fptr(g.reshape(-1)), fptr(f32(o)), fptr(f32(d)),
                                         fptr(f32(bmin)), fptr(f32(bmax)), n_c, n_f, eps, fptr(f32(uniforms)),
                                         fptr(dep), fptr(dl), fptr(pos), fptr(te), fptr(tx))
        else:
            esc = self.lib.po_sample_ray_philox(g.shape[0], fptr(g.reshape(-1)), fptr(f32(o)), fptr(f32(d)),
                                                fptr(f32(bmin)), fptr(f32(bmax)), n_c, n_f, eps, seed, tag, step,
                                                ray, fptr(dep), fptr(dl), fptr(pos), fptr(te), fptr(tx))
        return dict(escaped=bool(esc), depths=dep, deltas=dl, positions=pos, t_entry=te[0], t_exit=tx[0])

    def refresh_grid(self, arch, params, R):
        out = zeros(R, R, R)
        self.lib.po_refresh_grid(C.byref(arch_c(arch)), fptr(f32(params)), R, fptr(out.reshape(-1)))
        return out

    def reptile_update(self, meta, adapted, beta):
        meta, adapted = f32(meta), f32(adapted)
        out = np.zeros_like(meta)
        self.lib.po_reptile_update(len(meta), fptr(meta), fptr(adapted), beta, fptr(out))
        return out

    # -- trainer object
    def object_create(self, arch, theta, grid, grid_res, seed, cfg, bmin, bmax):
        a = arch_c(arch)
        g = None if grid is None else f32(grid).reshape(-1)
        h = self.lib.po_object_create(C.byref(a), fptr(f32(theta)), fptr(g), grid_res, seed, C.byref(cfg),
                                      fptr(f32(bmin)), fptr(f32(bmax)))
        return OracleObject(self, h, a, grid_res)


class OracleObject:
    def __init__(self, orc: Oracle, h, arch: FieldArchC, R: int):
        self.o, self.h, self.arch, self.R = orc, h, arch, R

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.po_object_destroy(self.h)
            self.h = None

    def set_frames(self, cams, rgb, depth, mask, inst, pose):
        pc = pose if isinstance(pose, PoseC) else pose.to_c()
        return self.o.lib.po_object_set_frames(self.h, len(cams), cams_c(cams), fptr(f32(rgb)), fptr(f32(depth)),
                                               u8ptr(np.ascontiguousarray(mask, np.uint8)), inst, C.byref(pc))

    def train_step(self, n=1):
        stats = (StepStatsC * n)()
        st = self.o.lib.po_object_train_step(self.h, n, stats)
        if st:
            raise RuntimeError(f"oracle train step failed with status {st}")
        return [dict(total=s.total, color=s.color_term, depth=s.depth_term, sigma=s.sigma_term,
                     n_samples=s.n_samples, escaped=s.n_rays_escaped, frame=s.frame_index) for s in stats]

    def params(self):
        out = zeros(self.o.param_count(self.arch))
        self.o.lib.po_object_get_params(self.h, fptr(out))
        return out

    def grid(self):
        out = zeros(self.R, self.R, self.R)
        self.o.lib.po_object_get_grid(self.h, fptr(out.reshape(-1)))
        return out


# --------------------------------------------------------------------------
class Ref(_Lib):
    """The reference sources (mt19937 draws) behind oracle/ref_shim.cpp."""

    def __init__(self):
        sz = C.c_size_t
        rarch = C.POINTER(RefArch)
        rcam = C.POINTER(RefCamera)
        sigs = {
            "ref_last_error": (C.c_char_p, []),
            "ref_param_count": (sz, [rarch]),
            "ref_hash_param_count": (sz, [rarch]),
            "ref_level_resolution": (C.c_int, [rarch, C.c_int]),
            "ref_vertex_table_row": (C.c_uint32, [rarch, C.c_int, C.c_uint32, C.c_uint32, C.c_uint32]),
            "ref_init_params": (None, [rarch, C.c_uint64, f32p]),
            "ref_hash_encode": (None, [rarch, f32p, C.c_int, f32p, f32p]),
            "ref_field_eval": (C.c_int, [rarch, f32p, C.c_int, f32p, f32p, f32p, f32p, f32p, f32p, f32p]),
            "ref_field_backward": (C.c_int, [rarch, f32p, C.c_int, f32p, f32p, f32p, f32p]),
            "ref_adam_step": (C.c_int, [sz, f32p, f32p, f32p, f32p, i64p, C.c_float, C.c_float, C.c_float,
                                        C.c_float]),
            "ref_uniform_samples": (C.c_int, [f32p, f32p, f32p, f32p, C.c_int, f32p, f32p, f32p, f32p, f32p]),
            "ref_trilerp": (C.c_float, [C.c_int, f32p, f32p]),
            "ref_build_ray_cdf": (C.c_int, [C.c_int, f32p, f32p, f32p, f32p, f32p, C.c_int, C.c_float, f32p,
                                            f32p]),
            "ref_inverse_transform_sample": (C.c_int, [f32p, f32p, f32p, f32p, C.c_int, f32p, C.c_int,
                                                       C.c_uint32, f32p, f32p, f32p, f32p]),
            "ref_sample_ray": (C.c_int, [C.c_int, f32p, f32p, f32p, f32p, f32p, C.c_int, C.c_int, C.c_float,
                                         C.c_uint32, f32p, f32p, f32p, f32p, f32p]),
            "ref_composite": (None, [C.c_int, f32p, f32p, f32p, f32p, f32p, f32p, f32p]),
            "ref_composite_backward": (None, [C.c_int, f32p, f32p, f32p, f32p, f32p, C.c_float, f32p, f32p]),
            "ref_batch_loss": (C.c_int, [C.c_int, i32p, f32p, f32p, i32p, i32p, f32p, f32p, f32p, f32p,
                                         C.c_float, C.c_float, C.c_uint32, f64p, f32p, f32p, f32p]),
            "ref_dilation_band": (None, [C.c_int, C.c_int, u8p, C.c_uint8, C.c_int, u8p]),
            "ref_generate_rays": (C.c_int, [rcam, f32p, f32p, u8p, C.c_uint8, f32p, f32p, C.c_int, C.c_float,
                                            C.c_uint32, C.c_int, f32p, f32p, i32p, f32p, f32p, i32p]),
            "ref_refresh_grid": (C.c_int, [rarch, f32p, C.c_int, f32p]),
            "ref_reptile_update": (C.c_int, [sz, f32p, f32p, C.c_float, f32p]),
            "ref_meta_task_order": (C.c_int, [sz, C.c_uint64, C.c_int, C.POINTER(C.c_int64)]),
            "ref_marching_cubes": (C.c_int, [C.c_int, f32p, C.c_float, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
            "ref_mesh_get": (None, [f32p, i32p]),
            "ref_cube_case_triangles": (C.c_int, [C.c_int, i32p]),
            "ref_choose_iso": (C.c_float, [C.c_int, f32p, C.c_float]),
            "ref_save_prior": (C.c_int, [C.c_char_p, C.c_char_p, rarch, f32p, C.c_int, f32p, C.c_int64, f32p,
                                         C.c_int64, i32p, C.c_uint64, C.c_int, C.c_int, i32p, f32p]),
            "ref_prior_summary": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int]),
            "ref_iter_cost_model": (C.c_double, [rarch, C.c_int, C.c_int]),
            "ref_sample_surface": (C.c_int, [C.c_int64, f32p, C.c_int64, i32p, C.c_int, C.c_uint64, f32p]),
            "ref_transformed": (C.c_int, [C.c_int64, f32p, f32p, f32p, f32p]),
            "ref_chamfer": (C.c_int, [C.c_int64, f32p, C.c_int64, f32p, f64p]),
            "ref_load_prior": (C.c_int, [C.c_char_p, rarch, i64p, f32p, f32p, f32p, i32p]),
            "ref_bake_prior": (C.c_int, [rarch, f32p, C.c_int, C.c_float, f32p, C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int64)]),
            "ref_train_object": (C.c_int, [rarch, f32p, C.c_int, f32p, C.c_int, rcam, f32p, f32p, u8p, C.c_uint8,
                                           f32p, f32p, f32p, f32p, C.POINTER(RefTrainCfg), C.c_uint32, C.c_int,
                                           f64p, f64p]),
            "ref_trainer_create": (C.c_void_p, [rarch, f32p, C.c_int, f32p, C.c_int, rcam, f32p, f32p, u8p,
                                                C.c_uint8, f32p, f32p, f32p, f32p, C.POINTER(RefTrainCfg),
                                                C.c_uint32]),
            "ref_trainer_destroy": (None, [C.c_void_p]),
            "ref_trainer_step": (C.c_int, [C.c_void_p, C.c_int, f64p]),
            "ref_trainer_last_samples": (C.c_longlong, [C.c_void_p]),
            "ref_trainer_get_params": (None, [C.c_void_p, f32p]),
            "ref_inner_adapt": (C.c_int, [rarch, f32p, C.c_int, rcam, f32p, f32p, u8p, f32p, f32p, f32p, f32p,
                                          C.c_int, C.c_float, C.c_uint32, C.c_int, C.c_float, C.c_int, C.c_float,
                                          C.c_float, f32p, f64p]),
        }
        super().__init__(REF_SO, sigs)

    @staticmethod
    def _a(arch):
        a = arch_c(arch)
        r = RefArch()
        C.memmove(C.byref(r), C.byref(a), C.sizeof(RefArch))
        return r

    def _check(self, st):
        if st:
            raise RuntimeError(f"reference error {st}: {self.lib.ref_last_error().decode()}")

    def param_count(self, arch):
        return int(self.lib.ref_param_count(C.byref(self._a(arch))))

    def hash_param_count(self, arch):
        return int(self.lib.ref_hash_param_count(C.byref(self._a(arch))))

    def level_resolution(self, arch, level):
        return int(self.lib.ref_level_resolution(C.byref(self._a(arch)), level))

    def vertex_table_row(self, arch, level, x, y, z):
        return int(self.lib.ref_vertex_table_row(C.byref(self._a(arch)), level, x, y, z))

    def init_params(self, arch, seed):
        out = zeros(self.param_count(arch))
        self.lib.ref_init_params(C.byref(self._a(arch)), seed, fptr(out))
        return out

    def hash_encode(self, arch, params, xyz):
        a = self._a(arch)
        xyz = f32(xyz).reshape(-1, 3)
        out = zeros(len(xyz), a.hash_levels * a.features_per_level)
        self.lib.ref_hash_encode(C.byref(a), fptr(f32(params)), len(xyz), fptr(xyz), fptr(out))
        return out

    def field_eval(self, arch, params, xyz, cache=False):
        a = self._a(arch)
        xyz = f32(xyz).reshape(-1, 3)
        n = len(xyz)
        L, F, W, H = a.hash_levels, a.features_per_level, a.hidden_width, a.hidden_layers
        sigma, rgb = zeros(n), zeros(n, 3)
        feat, pre, hid, raw = zeros(n, L * F), zeros(n, H * W), zeros(n, H * W), zeros(n, 4)
        st = self.lib.ref_field_eval(C.byref(a), fptr(f32(params)), n, fptr(xyz), fptr(sigma), fptr(rgb),
                                     fptr(feat), fptr(pre), fptr(hid), fptr(raw))
        self._check(st)
        if cache:
            return sigma, rgb, dict(features=feat, pre=pre, hidden=hid, raw=raw)
        return sigma, rgb

    def field_backward(self, arch, params, xyz, d_sigma, d_rgb, grad=None):
        a = self._a(arch)
        params = f32(params)
        xyz = f32(xyz).reshape(-1, 3)
        g = zeros(len(params)) if grad is None else f32(grad).copy()
        st = self.lib.ref_field_backward(C.byref(a), fptr(params), len(xyz), fptr(xyz), fptr(f32(d_sigma)),
                                         fptr(f32(d_rgb).reshape(-1)), fptr(g))
        self._check(st)
        return g

    def adam_step(self, params, grads, m, v, step, lr=1e-2, b1=0.9, b2=0.999, eps=1e-8):
        p, m, v = f32(params).copy(), f32(m).copy(), f32(v).copy()
        s = C.c_int64(step)
        self._check(self.lib.ref_adam_step(len(p), fptr(p), fptr(f32(grads)), fptr(m), fptr(v), C.byref(s),
                                           lr, b1, b2, eps))
        return p, m, v, s.value

    def uniform_samples(self, o, d, bmin, bmax, n):
        dep, dl, pos = zeros(n), zeros(n), zeros(n, 3)
        te, tx = zeros(1), zeros(1)
        esc = self.lib.ref_uniform_samples(fptr(f32(o)), fptr(f32(d)), fptr(f32(bmin)), fptr(f32(bmax)), n,
                                           fptr(dep), fptr(dl), fptr(pos), fptr(te), fptr(tx))
        return dict(escaped=bool(esc), depths=dep, deltas=dl, positions=pos, t_entry=te[0], t_exit=tx[0])

    def trilerp(self, grid, p):
        g = f32(grid)
        return float(self.lib.ref_trilerp(g.shape[0], fptr(g.reshape(-1)), fptr(f32(p))))

    def build_ray_cdf(self, grid, o, d, bmin, bmax, n_c, eps):
        g = f32(grid)
        tp, cdf = zeros(n_c), zeros(n_c)
        st = self.lib.ref_build_ray_cdf(g.shape[0], fptr(g.reshape(-1)), fptr(f32(o)), fptr(f32(d)),
                                        fptr(f32(bmin)), fptr(f32(bmax)), n_c, eps, fptr(tp), fptr(cdf))
        return st, tp, cdf

    def inverse_transform_sample(self, o, d, bmin, bmax, n_c, cdf, n, seed):
        dep, dl, pos, u = zeros(n), zeros(n), zeros(n, 3), zeros(2 * n)
        st = self.lib.ref_inverse_transform_sample(fptr(f32(o)), fptr(f32(d)), fptr(f32(bmin)), fptr(f32(bmax)),
                                                   n_c, fptr(f32(cdf)), n, seed, fptr(dep), fptr(dl), fptr(pos),
                                                   fptr(u))
        self._check(st)
        return dict(depths=dep, deltas=dl, positions=pos, uniforms=u)

    def sample_ray(self, grid, o, d, bmin, bmax, n_c, n_f, eps, seed):
        g = f32(grid)
        dep, dl, pos = zeros(n_f), zeros(n_f), zeros(n_f, 3)
        te, tx = zeros(1), zeros(1)
        esc = self.lib.ref_sample_ray(g.shape[0], fptr(g.reshape(-1)), fptr(f32(o)), fptr(f32(d)), fptr(f32(bmin)),
                                      fptr(f32(bmax)), n_c, n_f, eps, seed, fptr(dep), fptr(dl), fptr(pos),
                                      fptr(te), fptr(tx))
        return dict(escaped=bool(esc), depths=dep, deltas=dl, positions=pos, t_entry=te[0], t_exit=tx[0])

    def composite(self, sigma, rgb, deltas, depths):
        n = len(sigma)
        col, dep, tp = zeros(3), zeros(1), zeros(n)
        self.lib.ref_composite(n, fptr(f32(sigma)), fptr(f32(rgb).reshape(-1)), fptr(f32(deltas)),
                               fptr(f32(depths)), fptr(col), fptr(dep), fptr(tp))
        return col, dep[0], tp

    def composite_backward(self, sigma, rgb, deltas, depths, d_color, d_depth):
        n = len(sigma)
        ds, dr = zeros(n), zeros(n, 3)
        self.lib.ref_composite_backward(n, fptr(f32(sigma)), fptr(f32(rgb).reshape(-1)), fptr(f32(deltas)),
                                        fptr(f32(depths)), fptr(f32(d_color)), float(d_depth), fptr(ds), fptr(dr))
        return ds, dr

    def batch_loss(self, kind, target_rgb, target_depth, escaped, offsets, deltas, depths, sigma, rgb,
                   lambda_d, lambda_sigma, seed):
        kind = np.ascontiguousarray(kind, np.int32)
        esc = np.ascontiguousarray(escaped, np.int32)
        off = np.ascontiguousarray(offsets, np.int32)
        nr, ns = len(kind), int(off[-1])
        terms = np.zeros(4, np.float64)
        ds, dr, bg = zeros(max(ns, 1)), zeros(max(ns, 1), 3), zeros(nr, 3)
        st = self.lib.ref_batch_loss(nr, iptr(kind), fptr(f32(target_rgb).reshape(-1)), fptr(f32(target_depth)),
                                     iptr(esc), iptr(off), fptr(f32(deltas)), fptr(f32(depths)), fptr(f32(sigma)),
                                     fptr(f32(rgb).reshape(-1)), lambda_d, lambda_sigma, seed, dptr(terms),
                                     fptr(ds), fptr(dr), fptr(bg))
        return dict(status=st, terms=terms, d_sigma=ds[:ns], d_rgb=dr[:ns], bg_colors=bg)

    def dilation_band(self, mask, value, band_px):
        m = np.ascontiguousarray(mask, np.uint8)
        out = np.zeros_like(m)
        self.lib.ref_dilation_band(m.shape[1], m.shape[0], u8ptr(m), value, band_px, u8ptr(out))
        return out

    def generate_rays(self, cam, rgb, depth, mask, inst, pose, n, bg_fraction, seed, band_px=8):
        rc = RefCamera()
        cc = cam if isinstance(cam, CameraC) else cam.to_c()
        C.memmove(C.byref(rc), C.byref(cc), C.sizeof(RefCamera))
        pc = pose if isinstance(pose, PoseC) else pose.to_c()
        R = np.array(list(pc.R), np.float32)
        t = np.array(list(pc.t), np.float32)
        out = dict(origins=zeros(n, 3), dirs=zeros(n, 3), kinds=np.zeros(n, np.int32), target_rgb=zeros(n, 3),
                   target_depth=zeros(n), pick_px=np.zeros(n, np.int32))
        st = self.lib.ref_generate_rays(C.byref(rc), fptr(f32(rgb)), fptr(f32(depth)),
                                        u8ptr(np.ascontiguousarray(mask, np.uint8)), inst, fptr(R), fptr(t), n,
                                        bg_fraction, seed, band_px, fptr(out["origins"]), fptr(out["dirs"]),
                                        iptr(out["kinds"]), fptr(out["target_rgb"]), fptr(out["target_depth"]),
                                        iptr(out["pick_px"]))
        self._check(st)
        return out

    def refresh_grid(self, arch, params, R):
        out = zeros(R, R, R)
        self._check(self.lib.ref_refresh_grid(C.byref(self._a(arch)), fptr(f32(params)), R, fptr(out.reshape(-1))))
        return out

    def marching_cubes(self, grid, iso):
        """marching_cubes.cpp:125-180 on a [R][R][R] (z, y, x) grid: (vertices [V,3], triangles [T,3])."""
        g = f32(grid)
        nv, nt = C.c_int64(), C.c_int64()
        self._check(self.lib.ref_marching_cubes(g.shape[0], fptr(g.reshape(-1)), iso, C.byref(nv), C.byref(nt)))
        v = zeros(nv.value, 3)
        t = np.zeros((nt.value, 3), np.int32)
        self.lib.ref_mesh_get(fptr(v), iptr(t))
        return v, t

    def cube_case_triangles(self, config):
        out = np.zeros(16 * 3, np.int32)
        n = self.lib.ref_cube_case_triangles(config, iptr(out))
        return out[:3 * n].reshape(-1, 3)

    def choose_iso(self, grid, floor_value=5.0):
        g = f32(grid)
        return float(self.lib.ref_choose_iso(g.shape[0], fptr(g.reshape(-1)), floor_value))

    # -- prior bundles (prior_bundle.cpp; bake_prior density_grid.cpp:138-143)
    def save_prior(self, path, category, arch, theta, grid, vertices, triangles, search_seed=0, population=0,
                   generations=0, genome_ints=(8, 14, 2, 32, 2, 60, 15, 0),
                   genome_floats=(1e-2, 0.1, 1.45, 0.1, 1e-4)):
        g = f32(grid)
        v = f32(vertices).reshape(-1, 3)
        t = np.ascontiguousarray(triangles, np.int32).reshape(-1, 3)
        gi = np.asarray(genome_ints, np.int32)
        gf = np.asarray(genome_floats, np.float32)
        self._check(self.lib.ref_save_prior(str(path).encode(), category.encode(), C.byref(self._a(arch)),
                                            fptr(f32(theta)), g.shape[0], fptr(g.reshape(-1)), len(v), fptr(v),
                                            len(t), iptr(t), search_seed, population, generations, iptr(gi),
                                            fptr(gf)))

    def prior_summary(self, path):
        """(status, text or error message): the reference's load_prior + prior_summary."""
        buf = C.create_string_buffer(1 << 16)
        st = self.lib.ref_prior_summary(str(path).encode(), buf, len(buf))
        return st, (buf.value.decode() if st == 0 else self.lib.ref_last_error().decode())

    def load_prior(self, path):
        a = RefArch()
        sz = np.zeros(4, np.int64)
        self._check(self.lib.ref_load_prior(str(path).encode(), C.byref(a), i64ptr(sz), None, None, None, None))
        P, R, nv, nt = (int(x) for x in sz)
        th, g, v, t = zeros(P), zeros(R, R, R), zeros(nv, 3), np.zeros((nt, 3), np.int32)
        self._check(self.lib.ref_load_prior(str(path).encode(), C.byref(a), i64ptr(sz), fptr(th),
                                            fptr(g.reshape(-1)), fptr(v), iptr(t)))
        arch = dict(hash_levels=a.hash_levels, features_per_level=a.features_per_level,
                    log2_table_size=a.log2_table_size, base_resolution=a.base_resolution,
                    per_level_scale=a.per_level_scale, hidden_width=a.hidden_width, hidden_layers=a.hidden_layers,
                    density_activation=a.density_activation)
        return arch, th, g, v, t

    # -- genome evaluation pieces (search.cpp:214-228, mesh.cpp:56-104, metrics.cpp:14-22)
    def iter_cost_model(self, arch, rays_per_iter, samples_per_ray):
        return float(self.lib.ref_iter_cost_model(C.byref(self._a(arch)), rays_per_iter, samples_per_ray))

    def sample_surface(self, vertices, triangles, n, seed):
        v = f32(vertices).reshape(-1, 3)
        t = np.ascontiguousarray(triangles, np.int32).reshape(-1, 3)
        out = zeros(n, 3)
        self._check(self.lib.ref_sample_surface(len(v), fptr(v), len(t), iptr(t), n, seed, fptr(out)))
        return out

    def transformed(self, vertices, scale, t):
        v = f32(vertices).reshape(-1, 3)
        out = np.zeros_like(v)
        self._check(self.lib.ref_transformed(len(v), fptr(v), fptr(f32(scale)), fptr(f32(t)), fptr(out)))
        return out

    def chamfer(self, a, b):
        a, b = f32(a).reshape(-1, 3), f32(b).reshape(-1, 3)
        out = np.zeros(1, np.float64)
        self._check(self.lib.ref_chamfer(len(a), fptr(a), len(b), fptr(b), dptr(out)))
        return float(out[0])

    def bake_prior(self, arch, params, R, iso):
        g = zeros(R, R, R)
        nv, nt = C.c_int64(), C.c_int64()
        self._check(self.lib.ref_bake_prior(C.byref(self._a(arch)), fptr(f32(params)), R, iso, fptr(g.reshape(-1)),
                                            C.byref(nv), C.byref(nt)))
        v = zeros(nv.value, 3)
        t = np.zeros((nt.value, 3), np.int32)
        self.lib.ref_mesh_get(fptr(v), iptr(t))
        return g, v, t

    def reptile_update(self, meta, adapted, beta):
        meta, adapted = f32(meta), f32(adapted)
        out = np.zeros_like(meta)
        self._check(self.lib.ref_reptile_update(len(meta), fptr(meta), fptr(adapted), beta, fptr(out)))
        return out

    def meta_task_order(self, n_tasks, seed, n_epochs):
        """meta_train's per-epoch task order (meta.cpp:104-110), epochs x tasks."""
        out = np.zeros(n_tasks * n_epochs, np.int64)
        self._check(self.lib.ref_meta_task_order(n_tasks, seed, n_epochs,
                                                 out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out.reshape(n_epochs, n_tasks)

    def trainer(self, arch, params, grid, grid_R, cams, rgb, depth, mask, inst, pose, bmin, bmax, cfg, seed):
        """Persistent reference train_track state (frames converted once)."""
        return RefTrainer(self, arch, params, grid, grid_R, cams, rgb, depth, mask, inst, pose, bmin, bmax, cfg, seed)

    def train_object(self, arch, params, grid, grid_R, cams, rgb, depth, mask, inst, pose, bmin, bmax, cfg,
                     seed, iters):
        """Reference train_track loop (mt19937). Returns (params, grid, losses[iters,4], seconds)."""
        a = self._a(arch)
        p = f32(params).copy()
        g = None if grid is None else f32(grid).copy().reshape(-1)
        rc = (RefCamera * len(cams))()
        for i, c in enumerate(cams):
            cc = c if isinstance(c, CameraC) else c.to_c()
            C.memmove(C.byref(rc[i]), C.byref(cc), C.sizeof(RefCamera))
        pc = pose if isinstance(pose, PoseC) else pose.to_c()
        R = np.array(list(pc.R), np.float32)
        t = np.array(list(pc.t), np.float32)
        rcfg = RefTrainCfg()
        for name, _ in RefTrainCfg._fields_:
            setattr(rcfg, name, getattr(cfg, name))
        losses = np.zeros((iters, 4), np.float64)
        secs = np.zeros(1, np.float64)
        st = self.lib.ref_train_object(C.byref(a), fptr(p), grid_R, fptr(g), len(cams), rc, fptr(f32(rgb)),
                                       fptr(f32(depth)), u8ptr(np.ascontiguousarray(mask, np.uint8)), inst,
                                       fptr(R), fptr(t), fptr(f32(bmin)), fptr(f32(bmax)), C.byref(rcfg), seed,
                                       iters, dptr(losses), dptr(secs))
        self._check(st)
        return p, (None if g is None else g.reshape(grid_R, grid_R, grid_R)), losses, float(secs[0])


class RefTrainer:
    """Handle over ref_trainer_* (oracle/ref_shim.cpp): the reference's
    train_track loop with its own mt19937, stepped from Python; ctypes
    releases the GIL, so several trainers can run on separate threads
    (the reference's one-thread-per-object parallelism, mapper.cpp:572)."""

    def __init__(self, ref, arch, params, grid, grid_R, cams, rgb, depth, mask, inst, pose, bmin, bmax, cfg, seed):
        self.ref = ref
        a = ref._a(arch)
        self.P = ref.param_count(arch)
        rc = (RefCamera * len(cams))()
        for i, c in enumerate(cams):
            cc = c if isinstance(c, CameraC) else c.to_c()
            C.memmove(C.byref(rc[i]), C.byref(cc), C.sizeof(RefCamera))
        pc = pose if isinstance(pose, PoseC) else pose.to_c()
        R = np.array(list(pc.R), np.float32)
        t = np.array(list(pc.t), np.float32)
        rcfg = RefTrainCfg()
        for name, _ in RefTrainCfg._fields_:
            setattr(rcfg, name, getattr(cfg, name))
        g = None if grid is None else f32(grid).reshape(-1)
        self.h = ref.lib.ref_trainer_create(C.byref(a), fptr(f32(params)), grid_R, fptr(g), len(cams), rc,
                                            fptr(f32(rgb)), fptr(f32(depth)), u8ptr(np.ascontiguousarray(mask, np.uint8)),
                                            inst, fptr(R), fptr(t), fptr(f32(bmin)), fptr(f32(bmax)), C.byref(rcfg), seed)
        if not self.h:
            raise RuntimeError(ref.lib.ref_last_error().decode())

    def step(self, iters=1):
        losses = np.zeros((iters, 4), np.float64)
        st = self.ref.lib.ref_trainer_step(self.h, iters, dptr(losses))
        self.ref._check(st)
        return losses

    def last_samples(self):
        return int(self.ref.lib.ref_trainer_last_samples(self.h))

    def params(self):
        out = zeros(self.P)
        self.ref.lib.ref_trainer_get_params(self.h, fptr(out))
        return out

    def close(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_trainer_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()
