"""Category priors: the PriorBundle container and bake_prior.

The prior is the input of "create object from a category prior" (SURVEY §8 O2,
mapper.cpp:133-137): architecture, meta-learned θ, a baked σ grid over the
canonical unit cube and its mesh. This module mirrors the reference's

* ``PriorBundle`` / ``PriorProvenance`` / ``Genome`` (prior_bundle.hpp:14-34,
  search.hpp:17-33),
* ``save_prior`` / ``load_prior`` / ``prior_summary`` (prior_bundle.cpp:103-220):
  magic "NOMA", u16 version, u32-length-prefixed key=value text header, then
  u64-length-prefixed little-endian sections theta / grid / mesh -- byte for
  byte, with the same validation and DataError messages,
* ``bake_prior`` (density_grid.cpp:138-143): refresh_grid at R, then
  marching_cubes (with cleanup_mesh) of that grid -- both on the device
  (prenom_extract_mesh with an explicit iso, prenom_get_mesh_grid),

and ``ObjectTrainer.from_prior`` adds the create step on top. File I/O is host
work by nature (it is the reference's too); the numbers it carries are the
device path's inputs and outputs.
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from .trainer import DataError, FieldArch, UsageError

MAGIC = b"NOMA"
SUPPORTED_VERSION = 1
CATEGORIES = ("mug", "chair", "laptop", "book", "ball")  # shapes.cpp:162-171, all_categories order
_ACT_NAMES = {_capi.ACT_EXP_CLAMPED: "exponential-clamped", _capi.ACT_SOFTPLUS: "softplus"}


@dataclass
class Genome:
    """noma::Genome (search.hpp:17-33); defaults are the reference's."""

    hash_levels: int = 8
    log2_table_size: int = 14
    features_per_level: int = 2
    hidden_width: int = 32
    hidden_layers: int = 2
    meta_steps: int = 60
    inner_iters: int = 15
    eta: float = 1e-2
    beta: float = 0.1
    per_level_scale: float = 1.45
    lambda_d: float = 0.1
    lambda_sigma: float = 1e-4
    density_activation: int = _capi.ACT_EXP_CLAMPED


@dataclass
class PriorBundle:
    """noma::PriorBundle (prior_bundle.hpp:24-32) + PriorProvenance (14-19)."""

    arch: FieldArch
    theta: np.ndarray  # [P] float32, reference parameter layout
    grid: np.ndarray  # [R,R,R] float32, x-fastest
    vertices: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.float32))
    triangles: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.int32))
    category: str = "mug"
    format_version: int = 1
    search_seed: int = 0
    population: int = 0
    generations: int = 0
    genome: Genome = field(default_factory=Genome)


# ------------------------------------------------------------ text header
def _num(x) -> str:
    """C++ ostream with precision(9), default floatfield (== printf %.9g) of a float."""
    return format(float(np.float32(x)), ".9g")


def arch_to_text(a: FieldArch) -> str:
    """field.cpp:312-324."""
    return (f"hash_levels={a.hash_levels}\nfeatures_per_level={a.features_per_level}\n"
            f"log2_table_size={a.log2_table_size}\nbase_resolution={a.base_resolution}\n"
            f"per_level_scale={_num(a.per_level_scale)}\nhidden_width={a.hidden_width}\n"
            f"hidden_layers={a.hidden_layers}\ndensity_activation={_ACT_NAMES[a.density_activation]}\n")


def _header_text(b: PriorBundle) -> str:
    """prior_bundle.cpp:41-64."""
    g = b.genome
    return (f"category={b.category}\n" + arch_to_text(b.arch) +
            f"search_seed={b.search_seed}\nsearch_population={b.population}\n"
            f"search_generations={b.generations}\ngenome_hash_levels={g.hash_levels}\n"
            f"genome_log2_table_size={g.log2_table_size}\ngenome_features_per_level={g.features_per_level}\n"
            f"genome_hidden_width={g.hidden_width}\ngenome_hidden_layers={g.hidden_layers}\n"
            f"genome_meta_steps={g.meta_steps}\ngenome_inner_iters={g.inner_iters}\n"
            f"genome_eta={_num(g.eta)}\ngenome_beta={_num(g.beta)}\n"
            f"genome_per_level_scale={_num(g.per_level_scale)}\ngenome_lambda_d={_num(g.lambda_d)}\n"
            f"genome_lambda_sigma={_num(g.lambda_sigma)}\n"
            f"genome_density_activation={_ACT_NAMES[g.density_activation]}\n")


def _config(text: str) -> dict:
    """Config::from_string (config.cpp:28-55): key=value lines, '#' comments,
    whitespace-trimmed; a line without '=' is an error."""
    out = {}
    for n, line in enumerate(text.split("\n"), 1):
        t = line.strip()
        if not t or t[0] == "#":
            continue
        if "=" not in t:
            raise DataError(f"config line {n}: expected key=value")
        k, v = t.split("=", 1)
        out[k.strip()] = v.strip()
    return out


def _get_int(cfg, key, fallback):
    v = cfg.get(key)
    if v is None:
        return fallback
    try:
        return int(v, 10)
    except ValueError:
        raise UsageError(f"config key '{key}': expected integer, got '{v}'") from None


def _get_double(cfg, key, fallback):
    v = cfg.get(key)
    if v is None:
        return fallback
    try:
        return float(v)
    except ValueError:
        raise UsageError(f"config key '{key}': expected number, got '{v}'") from None


def _activation(s: str) -> int:
    for k, name in _ACT_NAMES.items():
        if name == s:
            return k
    raise DataError(f"unknown density activation: {s}")


def arch_from_text(text: str) -> FieldArch:
    """field.cpp:326-343 (validation included)."""
    cfg = _config(text)
    d = FieldArch()
    a = FieldArch(hash_levels=_get_int(cfg, "hash_levels", d.hash_levels),
                  features_per_level=_get_int(cfg, "features_per_level", d.features_per_level),
                  log2_table_size=_get_int(cfg, "log2_table_size", d.log2_table_size),
                  base_resolution=_get_int(cfg, "base_resolution", d.base_resolution),
                  per_level_scale=float(np.float32(_get_double(cfg, "per_level_scale", d.per_level_scale))),
                  hidden_width=_get_int(cfg, "hidden_width", d.hidden_width),
                  hidden_layers=_get_int(cfg, "hidden_layers", d.hidden_layers),
                  density_activation=_activation(cfg.get("density_activation", "exponential-clamped")))
    if (a.hash_levels < 1 or a.features_per_level < 1 or a.log2_table_size < 0 or a.base_resolution < 1
            or a.per_level_scale < 1.0 or a.hidden_width < 1 or a.hidden_layers < 1):
        raise DataError("invalid architecture description")
    return a


def _parse_header(text: str, b: PriorBundle) -> None:
    """prior_bundle.cpp:66-90."""
    cfg = _config(text)
    cat = cfg.get("category", "")
    if cat not in CATEGORIES:
        raise DataError(f"unknown category: {cat}")
    b.category = cat
    b.arch = arch_from_text(text)
    b.search_seed = int(_get_double(cfg, "search_seed", 0))
    b.population = _get_int(cfg, "search_population", 0)
    b.generations = _get_int(cfg, "search_generations", 0)
    g = Genome()
    for k in ("hash_levels", "log2_table_size", "features_per_level", "hidden_width", "hidden_layers", "meta_steps",
              "inner_iters"):
        setattr(g, k, _get_int(cfg, "genome_" + k, getattr(g, k)))
    for k in ("eta", "beta", "per_level_scale", "lambda_d", "lambda_sigma"):
        setattr(g, k, float(np.float32(_get_double(cfg, "genome_" + k, getattr(g, k)))))
    g.density_activation = _activation(cfg.get("genome_density_activation", _ACT_NAMES[g.density_activation]))
    b.genome = g


# ------------------------------------------------------------ container
def save_prior(b: PriorBundle, path) -> None:
    """prior_bundle.cpp:103-139."""
    theta = np.ascontiguousarray(b.theta, np.float32).reshape(-1)
    if len(theta) != b.arch.param_count():
        raise DataError("save_prior: parameter count does not match architecture")
    grid = np.ascontiguousarray(b.grid, np.float32)
    R = grid.shape[0] if grid.ndim == 3 else round(len(grid.reshape(-1)) ** (1 / 3))
    if grid.size != R * R * R:
        raise DataError("save_prior: grid payload does not match its resolution")
    verts = np.ascontiguousarray(b.vertices, np.float32).reshape(-1, 3)
    tris = np.ascontiguousarray(b.triangles).reshape(-1, 3).astype("<u4")
    header = _header_text(b).encode()
    parts = [MAGIC, struct.pack("<H", b.format_version), struct.pack("<I", len(header)), header,
             struct.pack("<Q", theta.nbytes), theta.astype("<f4").tobytes(),
             struct.pack("<Q", 4 + grid.nbytes), struct.pack("<I", R), grid.astype("<f4").tobytes(),
             struct.pack("<Q", 16 + verts.nbytes + tris.nbytes), struct.pack("<Q", len(verts)),
             verts.astype("<f4").tobytes(), struct.pack("<Q", len(tris)), tris.tobytes()]
    try:
        with open(path, "wb") as f:
            for p in parts:
                f.write(p)
    except OSError:
        raise DataError(f"save_prior: cannot write {path}") from None


class _Reader:
    def __init__(self, data: bytes, path: str):
        self.d, self.o, self.path = data, 0, path

    def take(self, n: int, what: str) -> bytes:
        if self.o + n > len(self.d):
            raise DataError(f"prior bundle truncated in {what}")
        b = self.d[self.o:self.o + n]
        self.o += n
        return b

    def pod(self, fmt: str, what: str):
        return struct.unpack(fmt, self.take(struct.calcsize(fmt), what))[0]


def load_prior(path) -> PriorBundle:
    """prior_bundle.cpp:141-197 (same checks, same order)."""
    path = str(path)
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise DataError(f"load_prior: cannot read {path}") from None
    r = _Reader(data, path)
    if r.take(4, "magic") != MAGIC:
        raise DataError(f"{path}: not a prior bundle")
    b = PriorBundle(arch=FieldArch(), theta=np.zeros(0, np.float32), grid=np.zeros((0, 0, 0), np.float32))
    b.format_version = r.pod("<H", "version")
    if b.format_version == 0 or b.format_version > SUPPORTED_VERSION:
        raise DataError(f"{path}: unsupported prior bundle version {b.format_version}")
    hlen = r.pod("<I", "header length")
    _parse_header(r.take(hlen, "header").decode(), b)
    tlen = r.pod("<Q", "theta length")
    if tlen != b.arch.param_count() * 4:
        raise DataError(f"{path}: parameter section does not match the declared architecture")
    b.theta = np.frombuffer(r.take(tlen, "theta"), "<f4").astype(np.float32)
    glen = r.pod("<Q", "grid length")
    R = r.pod("<I", "grid resolution")
    if R < 2 or R > 4096:
        raise DataError(f"{path}: grid resolution out of range")
    if glen != 4 + R ** 3 * 4:
        raise DataError(f"{path}: grid section does not match its resolution")
    b.grid = np.frombuffer(r.take(R ** 3 * 4, "grid"), "<f4").astype(np.float32).reshape(R, R, R)
    mlen = r.pod("<Q", "mesh length")
    nv = r.pod("<Q", "vertex count")
    if mlen < 16 + nv * 12:
        raise DataError(f"{path}: mesh section shorter than its vertex payload")
    b.vertices = np.frombuffer(r.take(nv * 12, "vertices"), "<f4").astype(np.float32).reshape(nv, 3)
    nt = r.pod("<Q", "triangle count")
    if mlen != 16 + nv * 12 + nt * 12:
        raise DataError(f"{path}: mesh section length mismatch")
    tris = np.frombuffer(r.take(nt * 12, "triangles"), "<u4").reshape(nt, 3)
    if nt and int(tris.max()) >= nv:
        raise DataError(f"{path}: triangle index out of range")
    b.triangles = tris.astype(np.int32)
    if r.o != len(data):
        raise DataError(f"{path}: trailing bytes after mesh section")
    return b


def _g6(x) -> str:
    """ostream precision(6) default floatfield (%g)."""
    return format(float(np.float32(x)), "g")


def prior_summary(path) -> str:
    """prior_bundle.cpp:199-220."""
    b = load_prior(path)
    tmin = float(b.theta.min()) if len(b.theta) else 0.0
    tmax = float(b.theta.max()) if len(b.theta) else 0.0
    arch_lines = "".join(f"  {ln}\n" for ln in arch_to_text(b.arch).splitlines())
    return (f"category: {b.category}\nformat version: {b.format_version}\narchitecture:\n{arch_lines}"
            f"parameters: {len(b.theta)} (min {_g6(tmin)}, max {_g6(tmax)})\n"
            f"grid: {b.grid.shape[0]}^3, max density {_g6(b.grid.max())}\n"
            f"mesh: {len(b.vertices)} vertices, {len(b.triangles)} triangles\n"
            f"search: seed {b.search_seed}, population {b.population}, generations {b.generations}\n")


# ------------------------------------------------------------ device bake
def bake_prior(ctx, arch: FieldArch, theta, resolution: int, iso: float):
    """noma::bake_prior (density_grid.cpp:138-143) on the device: the σ lattice at
    `resolution` (refresh_grid) and its marching-cubes mesh at `iso`.
    Returns (grid [R,R,R], vertices [V,3], triangles [T,3])."""
    from . import trainer as T

    if not (isinstance(iso, float) or isinstance(iso, int)) or math.isnan(iso):
        raise UsageError("bake_prior: iso must be a number")
    obj = T.ObjectTrainer.create(ctx, arch, theta=theta)
    try:
        v, t, _ = obj.extract_mesh(resolution, iso=float(iso))
        grid = obj.get_mesh_grid()
    finally:
        obj.close()
    return grid, v, t
