"""Scene descriptions and the synthetic configurations A-E.

A scene is plain data: grid/step parameters, materials, and per-environment
particles (seeded with the library's own ``msim_seed_box``, the restatement
of seeding.hpp:13-35) plus bodies and shapes. The same Scene feeds the CUDA
path (world.GpuWorld) and the CPU checker, so both start from bit-identical
inputs.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import abi

SOFT_CLAY = (1000.0, 1e4, 0.3, 2e3)     # mpm.hpp:45
STIFF_CLAY = (1000.0, 3e5, 0.3, 1e4)    # mpm.hpp:46
FIRM_CLAY = (1000.0, 1e5, 0.3, 4e3)     # scenario.hpp:390 (write-mini)
# north_star materials without a reference implementation (parity with the
# oracle's restatement of the published algorithms): (density, E, nu, param, model)
SAND = (1600.0, 3.5e4, 0.3, 30.0, abi.MODEL_DRUCKER_PRAGER)      # param = friction angle (deg)
WATER = (1000.0, 2e4, 0.2, 0.0, abi.MODEL_FLUID)                 # K = E / (3 (1 - 2 nu))
JELLY = (1000.0, 5e4, 0.3, 0.0, abi.MODEL_FIXED_COROTATED)
V0_SOFT = 6.2e-8                        # mpm.hpp:47
V0_STIFF = 1.2e-7                       # mpm.hpp:48


@dataclass
class ShapeSpec:
    type: int
    body: int
    params: tuple = (0.0, 0.0, 0.0, 0.0)
    local_q: tuple = (1.0, 0.0, 0.0, 0.0)
    local_t: tuple = (0.0, 0.0, 0.0)
    friction: float = 0.5
    k_n: float = 1e3
    k_t: float = 10.0
    vol_dims: tuple = (0, 0, 0)
    vol_origin: tuple = (0.0, 0.0, 0.0)
    vol_voxel: float = 0.01
    vol_samples: np.ndarray | None = None

    def to_c(self) -> abi.Shape:
        s = abi.Shape()
        s.type = self.type
        s.body = self.body
        s.local_q[:] = self.local_q
        s.local_t[:] = self.local_t
        s.friction = self.friction
        s.k_n = self.k_n
        s.k_t = self.k_t
        s.params[:] = tuple(self.params) + (0.0,) * (4 - len(self.params))
        if self.type == abi.SHAPE_VOLUME:
            s.vol_dims[:] = self.vol_dims
            s.vol_origin[:] = self.vol_origin
            s.vol_voxel = self.vol_voxel
            arr = np.ascontiguousarray(self.vol_samples, dtype=np.float32)
            self._keep = arr
            s.vol_samples = arr.ctypes.data_as(C.POINTER(C.c_float))
        return s


@dataclass
class BodySpec:
    mode: int = abi.BODY_KINEMATIC
    q: tuple = (1.0, 0.0, 0.0, 0.0)
    t: tuple = (0.0, 0.0, 0.0)
    v: tuple = (0.0, 0.0, 0.0)
    w: tuple = (0.0, 0.0, 0.0)
    mass: float = 1.0
    inertia: tuple = (1e-3, 1e-3, 1e-3)
    com_offset: tuple = (0.0, 0.0, 0.0)

    def to_c(self) -> abi.Body:
        b = abi.Body()
        b.mode = self.mode
        b.q[:] = self.q
        b.t[:] = self.t
        b.v[:] = self.v
        b.w[:] = self.w
        b.mass = self.mass
        b.inertia[:] = self.inertia
        b.com_offset[:] = self.com_offset
        return b


@dataclass
class EnvSpec:
    x: np.ndarray                       # (n, 3)
    mass: np.ndarray                    # (n,)
    vol0: np.ndarray                    # (n,)
    v: np.ndarray | None = None         # (n, 3)
    F: np.ndarray | None = None         # (n, 3, 3)
    C: np.ndarray | None = None         # (n, 3, 3)
    material: np.ndarray | None = None  # (n,) int32
    bodies: list = field(default_factory=list)
    shapes: list = field(default_factory=list)

    @property
    def n(self) -> int:
        return int(self.x.shape[0])


@dataclass
class Scene:
    name: str
    h: float = 0.01
    dims: tuple = (64, 64, 64)
    origin: tuple = (0.0, 0.0, 0.0)
    boundary: tuple = (0, 0, 0, 0, 0, 0)
    gravity: tuple = (0.0, 0.0, -9.81)
    dt: float = 5e-4
    cfl_factor: float = 0.4
    max_cfl_halvings: int = 4
    lost_fraction_threshold: float = 0.01
    materials: list = field(default_factory=lambda: [SOFT_CLAY])
    envs: list = field(default_factory=list)
    coupling_mode: int = abi.COUPLING_PARTICLE
    r_c_factor: float = 0.5
    c_d: float = 10.0
    n_rigid: int = 25
    n_soft: int = 1
    rigid_gravity: tuple = (0.0, 0.0, -9.81)

    def desc(self) -> abi.SoftDesc:
        d = abi.SoftDesc()
        d.h = self.h
        d.dims[:] = self.dims
        d.origin[:] = self.origin
        d.boundary[:] = self.boundary
        d.gravity[:] = self.gravity
        d.dt = self.dt
        d.cfl_factor = self.cfl_factor
        d.max_cfl_halvings = self.max_cfl_halvings
        d.lost_fraction_threshold = self.lost_fraction_threshold
        return d

    def material_array(self):
        arr = (abi.Material * len(self.materials))()
        for i, mat in enumerate(self.materials):  # (density, E, nu, yield [, model])
            rho, E, nu, sy = mat[:4]
            arr[i].density, arr[i].youngs, arr[i].poisson, arr[i].yield_stress = rho, E, nu, sy
            arr[i].model = mat[4] if len(mat) > 4 else abi.MODEL_HENCKY_VON_MISES
        return arr

    @property
    def n_particles(self) -> int:
        return sum(e.n for e in self.envs)

    @property
    def substeps_per_env_step(self) -> int:
        return self.n_rigid * self.n_soft


# ---------------------------------------------------------------------------
# Seeding through the library (seeding.hpp:13-35 restated in csrc/msim_host.cpp).

class Rng:
    def __init__(self, seed: int):
        self._lib = abi.load()
        self._h = self._lib.msim_rng_create(seed)

    def uniform(self, lo: float, hi: float) -> float:
        return self._lib.msim_rng_uniform(self._h, lo, hi)

    def uniform_array(self, n: int, lo: float, hi: float) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self._lib.msim_rng_fill_uniform(self._h, n, lo, hi, abi.dptr(out))
        return out

    def __del__(self):
        try:
            self._lib.msim_rng_destroy(self._h)
        except Exception:
            pass


def seed_box(rng: Rng, lo, hi, density: float, particle_volume: float):
    lib = abi.load()
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    n = lib.msim_seed_box_count(abi.dptr(lo), abi.dptr(hi), particle_volume)
    x = np.zeros((n, 3))
    m = np.zeros(n)
    got = lib.msim_seed_box(rng._h, abi.dptr(lo), abi.dptr(hi), density, particle_volume, abi.dptr(x), abi.dptr(m))
    assert got == n
    return x, m


def lattice_span(n_cells: int, particle_volume: float) -> float:
    """Span giving exactly n lattice points per axis: (n + 0.5) * spacing."""
    return (n_cells + 0.5) * particle_volume ** (1.0 / 3.0)


def block_env(lo, counts, material_id: int, mat: tuple, particle_volume: float, seed: int,
              vel_seed: int | None = None, vel_amp: float = 0.1) -> EnvSpec:
    rng = Rng(seed)
    hi = [lo[a] + lattice_span(counts[a], particle_volume) for a in range(3)]
    x, m = seed_box(rng, lo, hi, mat[0], particle_volume)
    n = x.shape[0]
    v = None
    if vel_seed is not None:
        vr = Rng(vel_seed)
        v = vr.uniform_array(3 * n, -vel_amp, vel_amp).reshape(n, 3)
    return EnvSpec(x=x, mass=m, vol0=np.full(n, particle_volume), v=v,
                   material=np.full(n, material_id, dtype=np.int32))


def quat_from_axis_angle(axis, ang):
    axis = np.asarray(axis, dtype=np.float64)
    axis = axis / np.linalg.norm(axis)
    s = math.sin(0.5 * ang)
    return (math.cos(0.5 * ang), s * axis[0], s * axis[1], s * axis[2])


def soft_contact(**kw) -> dict:
    """Golden-scene contact constants (scenario.hpp:312-318)."""
    d = dict(k_n=20.0, k_t=0.1)
    d.update(kw)
    return d


def box_sdf_volume(half, voxel, pad):
    """Exact SDF of a box sampled on a voxel grid (stands in for
    bake_mesh_sdf(make_box_mesh(half)), sdf.hpp:277-309, :443-455)."""
    half = np.asarray(half, dtype=np.float64)
    lo = -half - pad
    dims = np.ceil((2 * (half + pad)) / voxel).astype(int) + 1
    zs, ys, xs = [lo[a] + voxel * np.arange(dims[a]) for a in (2, 1, 0)]
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    P = np.stack([X, Y, Z], axis=-1)
    q = np.abs(P) - half
    outside = np.linalg.norm(np.maximum(q, 0.0), axis=-1)
    inside = np.minimum(np.max(q, axis=-1), 0.0)
    samples = (outside + inside).astype(np.float32)  # (z, y, x) -> x fastest
    return tuple(int(d) for d in dims), tuple(lo), voxel, samples.reshape(-1)


# ---------------------------------------------------------------------------
# Configurations.

def config_a(material: tuple = SOFT_CLAY) -> Scene:
    """A: 8k soft clay (or another material), 64^3, one dynamic box falling onto the block."""
    s = V0_SOFT ** (1.0 / 3.0)
    lo = (0.28, 0.28, 0.05)
    env = block_env(lo, (20, 20, 20), 0, material, V0_SOFT, seed=1, vel_seed=2)
    top = lo[2] + lattice_span(20, V0_SOFT)
    cxy = lo[0] + 0.5 * lattice_span(20, V0_SOFT)
    box = BodySpec(mode=abi.BODY_DYNAMIC, t=(cxy, cxy, top + 0.002 + 0.01), v=(0.0, 0.0, -0.2),
                   mass=0.05, inertia=(8e-6, 8e-6, 8e-6))
    env.bodies = [box]
    env.shapes = [ShapeSpec(abi.SHAPE_BOX, 0, params=(0.03, 0.03, 0.01), **soft_contact())]
    del s
    return Scene(name="A", dims=(64, 64, 64), h=0.01, dt=5e-4, envs=[env], c_d=0.05, materials=[material])


def _bucket_shapes(body: int, half_w: float, half_h: float, wall: float, friction=0.2):
    sh = [ShapeSpec(abi.SHAPE_BOX, body, params=(half_w, half_w, wall), local_t=(0, 0, -half_h),
                    friction=friction, **soft_contact())]
    for sx, sy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
        if sx:
            p = (wall, half_w, half_h)
            t = (sx * (half_w + wall), 0.0, 0.0)
        else:
            p = (half_w, wall, half_h)
            t = (0.0, sy * (half_w + wall), 0.0)
        sh.append(ShapeSpec(abi.SHAPE_BOX, body, params=p, local_t=t, friction=friction, **soft_contact()))
    return sh


def config_b_env(e: int = 0, material: tuple = SOFT_CLAY) -> EnvSpec:
    """One Excavate-shaped env: 40x40x20 bed, scripted 5-box bucket scooping.
    Env e is seeded with (3 + 10 e, 4 + 10 e)."""
    lo = (0.2399, 0.2399, 0.021)
    env = block_env(lo, (40, 40, 20), 0, material, V0_SOFT, seed=3 + 10 * e, vel_seed=4 + 10 * e)
    top = lo[2] + lattice_span(20, V0_SOFT)
    bucket = BodySpec(mode=abi.BODY_SCRIPTED, t=(lo[0] + 0.04, 0.32, top + 0.02), v=(0.05, 0.0, -0.05))
    env.bodies = [bucket]
    env.shapes = _bucket_shapes(0, 0.03, 0.02, 0.004)
    return env


def config_b(material: tuple = SOFT_CLAY, n_envs: int = 1, first_env: int = 0) -> Scene:
    """B: 32k bed per env (clay parity variant by default; SAND = Drucker-Prager),
    64^3, scripted 5-box bucket scooping; n_envs batched Excavate-shaped envs."""
    envs = [config_b_env(first_env + e, material) for e in range(n_envs)]
    return Scene(name="B", dims=(64, 64, 64), h=0.01, dt=5e-4, envs=envs, c_d=0.05, materials=[material])


def config_c_env(e: int = 0, material: tuple = SOFT_CLAY) -> EnvSpec:
    """One Pour-shaped env: 40^3 column, rotating 5-box bottle + static beaker.
    Env e is seeded with (5 + 10 e, 6 + 10 e)."""
    lo = (0.24, 0.24, 0.06)
    env = block_env(lo, (40, 40, 40), 0, material, V0_SOFT, seed=5 + 10 * e, vel_seed=6 + 10 * e)
    c = lo[0] + 0.5 * lattice_span(40, V0_SOFT)
    bottle = BodySpec(mode=abi.BODY_SCRIPTED, t=(c, c, lo[2] + 0.085), w=(0.0, 0.5, 0.0))
    beaker = BodySpec(mode=abi.BODY_KINEMATIC, t=(c + 0.2, c, 0.06))
    env.bodies = [bottle, beaker]
    env.shapes = _bucket_shapes(0, 0.09, 0.085, 0.005) + _bucket_shapes(1, 0.06, 0.04, 0.005)
    return env


def config_c(material: tuple = SOFT_CLAY, n_envs: int = 1, first_env: int = 0) -> Scene:
    """C: 64k column per env (clay parity variant by default; WATER = J-only
    fluid), 128^3 h=0.005, rotating bottle + static beaker; n_envs batched
    Pour-shaped envs."""
    envs = [config_c_env(first_env + e, material) for e in range(n_envs)]
    return Scene(name="C", dims=(128, 128, 128), h=0.005, dt=5e-4, envs=envs, c_d=0.05, materials=[material])


def config_d_env(e: int) -> EnvSpec:
    """One env of D: 32x32x16 firm-clay slab, write stamp (even) or pinch fingers (odd)."""
    lat = (32, 32, 16)
    span = [lattice_span(n, V0_SOFT) for n in lat]
    lo = ((0.32 - span[0]) / 2, (0.32 - span[1]) / 2, 0.021)
    env = block_env(lo, lat, 0, FIRM_CLAY, V0_SOFT, seed=1000 + e, vel_seed=5000 + e)
    cx, cy = lo[0] + span[0] / 2, lo[1] + span[1] / 2
    top = lo[2] + span[2]
    if e % 2 == 0:
        stamp = BodySpec(mode=abi.BODY_SCRIPTED, t=(cx, cy, top + 0.008 + 0.001), v=(0.0, 0.0, -0.02))
        env.bodies = [stamp]
        env.shapes = [ShapeSpec(abi.SHAPE_BOX, 0, params=(0.03, 0.01, 0.008), friction=0.3, k_n=80.0, k_t=0.1)]
    else:
        zc = lo[2] + span[2] / 2
        off = span[0] / 2 + 0.004 + 0.001
        left = BodySpec(mode=abi.BODY_SCRIPTED, t=(cx - off, cy, zc), v=(0.01, 0.0, 0.0))
        right = BodySpec(mode=abi.BODY_SCRIPTED, t=(cx + off, cy, zc), v=(-0.01, 0.0, 0.0))
        env.bodies = [left, right]
        env.shapes = [ShapeSpec(abi.SHAPE_BOX, 0, params=(0.004, 0.012, 0.018), friction=0.5, **soft_contact()),
                      ShapeSpec(abi.SHAPE_BOX, 1, params=(0.004, 0.012, 0.018), friction=0.5, **soft_contact())]
    return env


def config_d(n_envs: int = 1024, first_env: int = 0) -> Scene:
    """D: batched Pinch/Write-shaped von Mises plasticine, 16,384 particles per env."""
    envs = [config_d_env(first_env + e) for e in range(n_envs)]
    return Scene(name="D", dims=(32, 32, 32), h=0.01, dt=2.5e-4, materials=[FIRM_CLAY], envs=envs,
                 c_d=0.05)


def config_e(clay_only: bool = True, slab=(50, 200, 100), grid: int = 256) -> Scene:
    """E: 4M particles in 4 x-slabs, 256^3 h=0.005, 8 moving colliders (3 boxes,
    2 spheres, 2 capsules, 1 SDF volume). Mixed materials (clay, sand, water,
    jelly slabs) or the clay-only variant (soft / stiff clay alternating, the
    reference's model only). `slab` / `grid` give reduced parity variants."""
    s = V0_SOFT ** (1.0 / 3.0)
    extent = grid * 0.005
    span = lattice_span(slab[1], V0_SOFT)
    lo = ((extent - span) / 2, (extent - span) / 2, 0.021)
    xs, ms, mats = [], [], []
    materials = [SOFT_CLAY, STIFF_CLAY] if clay_only else [SOFT_CLAY, SAND, WATER, JELLY]
    for k in range(4):
        slab_lo = (lo[0] + k * slab[0] * s, lo[1], lo[2])
        mid = k % 2 if clay_only else k
        mat = materials[mid]
        e = block_env(slab_lo, slab, mid, mat, V0_SOFT, seed=7 + 10 * k)
        xs.append(e.x)
        ms.append(e.mass)
        mats.append(e.material)
    x = np.concatenate(xs)
    n = x.shape[0]
    v = Rng(8).uniform_array(3 * n, -0.1, 0.1).reshape(n, 3)
    env = EnvSpec(x=x, mass=np.concatenate(ms), vol0=np.full(n, V0_SOFT), v=v,
                  material=np.concatenate(mats).astype(np.int32))
    rng = np.random.default_rng(7)
    bodies, shapes = [], []
    kinds = [abi.SHAPE_BOX] * 3 + [abi.SHAPE_SPHERE] * 2 + [abi.SHAPE_CAPSULE] * 2 + [abi.SHAPE_VOLUME]
    top = lo[2] + lattice_span(slab[2], V0_SOFT)
    for i, kind in enumerate(kinds):
        margin = 0.05 * span / lattice_span(200, V0_SOFT)  # 0.05 m at full size
        cx, cy = rng.uniform(lo[0] + margin, lo[0] + span - margin, size=2)
        q = quat_from_axis_angle(rng.normal(size=3), rng.uniform(0, math.pi))
        bodies.append(BodySpec(mode=abi.BODY_SCRIPTED, q=q, t=(cx, cy, top + 0.01),
                               v=tuple(rng.uniform(-0.05, 0.05, size=2)) + (-0.05,),
                               w=tuple(rng.uniform(-0.5, 0.5, size=3))))
        if kind == abi.SHAPE_BOX:
            shapes.append(ShapeSpec(kind, i, params=(0.04, 0.03, 0.02), **soft_contact()))
        elif kind == abi.SHAPE_SPHERE:
            shapes.append(ShapeSpec(kind, i, params=(0.04,), **soft_contact()))
        elif kind == abi.SHAPE_CAPSULE:
            shapes.append(ShapeSpec(kind, i, params=(0.04, 0.02), **soft_contact()))
        else:
            dims, org, vox, smp = box_sdf_volume((0.04, 0.04, 0.03), 0.01, 0.03)
            shapes.append(ShapeSpec(kind, i, vol_dims=dims, vol_origin=org, vol_voxel=vox, vol_samples=smp,
                                    **soft_contact()))
    env.bodies = bodies
    env.shapes = shapes
    # App. B asks for 5e-4, halved to 2.5e-4 if needed. The stiff clay's elastic wave
    # speed sqrt((lambda + 2 mu) / rho) ~ 20 m/s makes h / c = 2.5e-4 the explicit
    # stability limit at h = 0.005: it inverts at 5e-4 in the first env step and at
    # 2.5e-4 after ~10 (det F <= 0), and the reference's CFL test is velocity-only, so
    # no halving catches it. 1e-4 (elastic Courant ~0.4) is stable
    # (profiles/r02_experiments_D.txt).
    return Scene(name="E", dims=(grid, grid, grid), h=0.005, dt=1e-4, materials=materials,
                 envs=[env], c_d=0.05)


CONFIGS = {"A": config_a, "B": config_b, "C": config_c, "D": config_d, "E": config_e}
