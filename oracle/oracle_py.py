"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper of oracle/_build/liboracle.so, the double-precision CPU
restatement of the reference's soft-body path (see msim_oracle.hpp). Only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use it, as
the checker; the product path never imports this module.

``OracleWorld`` runs one environment of a ``paper_2302_04659_b200.scenes``
Scene (the reference World is single-environment). ``RefWorld`` runs the
same environment through oracle/_ref/libmsim_ref.so: the REFERENCE's own
sources compiled against the Eigen subset in oracle/ref_shim/ (see
ref_capi.cpp), with the same surface. This module never imports the product
package (it uses its own struct mirror, oracle/cabi.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from oracle import cabi as abi

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(BUILD, "liboracle.so")
REF_DIR = os.path.join(HERE, "_ref")
REF_LIB = os.path.join(REF_DIR, "libmsim_ref.so")
KAT = os.path.join(BUILD, "kat_oracle")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)
_vp = C.c_void_p

# struct pointers are passed untyped (void*): the product's and the checker's
# layout-identical ctypes mirrors are both accepted
_SIGS = {
    "oracle_create": (_vp, [_vp, _vp, C.c_int]),
    "oracle_destroy": (None, [_vp]),
    "oracle_last_error": (C.c_char_p, [_vp]),
    "oracle_set_threads": (None, [C.c_int]),
    "oracle_set_particles": (C.c_int, [_vp, C.c_int64, _dp, _dp, _dp, _dp, _dp, _dp, _ip]),
    "oracle_write_particles": (C.c_int, [_vp, C.c_int64, _dp, _dp, _dp, _dp]),
    "oracle_set_bodies": (C.c_int, [_vp, _vp, C.c_int, _vp, C.c_int]),
    "oracle_sync_bodies": (C.c_int, [_vp, _vp, C.c_int]),
    "oracle_set_coupling": (C.c_int, [_vp, _vp]),
    "oracle_set_kinematic_schedule": (C.c_int, [_vp, C.c_int, _dp, _u8p]),
    "oracle_set_stepping": (C.c_int, [_vp, C.c_int, C.c_int, _dp]),
    "oracle_set_dt": (C.c_int, [_vp, C.c_double]),
    "oracle_set_gravity": (C.c_int, [_vp, _dp]),
    "oracle_set_lost_fraction_threshold": (C.c_int, [_vp, C.c_double]),
    "oracle_init": (C.c_int, [_vp]),
    "oracle_init_buffers": (C.c_int, [_vp]),
    "oracle_env_step": (C.c_int, [_vp, _vp]),
    "oracle_soft_substep": (C.c_int, [_vp, C.c_int, C.c_int, _ip]),
    "oracle_p2g": (C.c_int, [_vp]),
    "oracle_grid_update": (C.c_int, [_vp]),
    "oracle_g2p": (C.c_int, [_vp]),
    "oracle_grid_clear": (C.c_int, [_vp]),
    "oracle_penalty_particle": (C.c_int, [_vp, _dp]),
    "oracle_penalty_grid": (C.c_int, [_vp, _dp]),
    "oracle_particle_count": (C.c_int64, [_vp]),
    "oracle_read_particles": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _u8p]),
    "oracle_read_ext_force": (C.c_int, [_vp, _dp]),
    "oracle_read_grid": (C.c_int, [_vp, _dp, _dp, _dp, _dp]),
    "oracle_write_grid_velocity": (C.c_int, [_vp, _dp]),
    "oracle_read_binning": (C.c_int, [_vp, _ip, _ip, C.c_int64, _ip, C.c_int64, _lp, _lp, C.c_int64, _lp]),
    "oracle_read_wrenches": (C.c_int, [_vp, C.c_int, _dp, _dp]),
    "oracle_read_bodies": (C.c_int, [_vp, _vp, C.c_int]),
    "oracle_lost_count": (C.c_int64, [_vp]),
    "oracle_time": (C.c_double, [_vp]),
    "oracle_mean_particle_mass": (C.c_double, [_vp]),
    "oracle_constitutive": (C.c_int, [_vp, C.c_int64, _dp, _dp, _dp]),
    "oracle_sdf": (C.c_int, [_vp, C.c_int64, _dp, _dp, _dp]),
    "oracle_state_hash": (C.c_uint64, [_vp]),
    "oracle_rng_create": (_vp, [C.c_uint64]),
    "oracle_rng_destroy": (None, [_vp]),
    "oracle_rng_uniform": (C.c_double, [_vp, C.c_double, C.c_double]),
    "oracle_seed_box": (C.c_int64, [_vp, _vp, _dp, _dp, C.c_int, C.c_double]),
    "oracle_lattice_count": (C.c_int64, [_dp, _dp, C.c_double]),
    "oracle_time_env_steps": (C.c_double, [_vp, C.c_int, _ip]),
    "oracle_read_jp": (C.c_int, [_vp, _dp]),
    "oracle_bake_grid": (C.c_int, [_dp, C.c_int64, C.c_double, C.c_double, _dp, _ip]),
    "oracle_bake_mesh_sdf": (C.c_int, [_dp, C.c_int64, C.c_double, C.c_double, C.POINTER(C.c_float), C.c_int64]),
    "oracle_make_box_mesh": (None, [_dp, _dp, _dp]),
    "oracle_metric_fill": (C.c_int, [C.c_int64, _dp, _dp, _dp, _dp, _dp, _ip]),
    "oracle_render_heightmap": (C.c_int, [C.c_int64, _dp, _dp, C.c_int, C.c_int, _dp]),
    "oracle_metric_write_iou": (C.c_int, [C.c_int, C.c_int, C.c_double, _dp, _dp, _dp, _ip]),
    "oracle_chamfer": (C.c_int, [C.c_int64, _dp, C.c_int64, _dp, _dp]),
    "oracle_metric_pinch": (C.c_int, [C.c_int64, _dp, C.c_int64, _dp, C.c_int64, _dp, _dp, _ip]),
}

# reference-harness-only entry points (ref_capi.cpp)
_REF_SIGS = {
    "ref_unsupported": (C.c_int, [_vp]),
    "ref_bench_worlds": (C.c_double, [C.POINTER(_vp), C.c_int, C.c_int, _ip]),
}

_lib = None
_ref = None


class _RefAdapter:
    """The reference harness library seen through the oracle's names."""

    def __init__(self, cdll):
        self.cdll = cdll
        for name, (res, args) in _SIGS.items():
            rname = "ref_" + name[len("oracle_"):]
            f = getattr(cdll, rname, None)
            if f is None:
                continue
            f.restype = res
            f.argtypes = args
            setattr(self, name, f)
        for name, (res, args) in _REF_SIGS.items():
            f = getattr(cdll, name)
            f.restype = res
            f.argtypes = args
            setattr(self, name, f)


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def load_ref():
    """oracle/_ref/libmsim_ref.so (built here by Makefile.ref from /root/reference)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB):
            raise FileNotFoundError(f"{REF_LIB} not built (make -C oracle -f Makefile.ref needs /root/reference)")
        _ref = _RefAdapter(C.CDLL(REF_LIB))
    return _ref


def build():
    """Compile the oracle (make -C oracle). Test infrastructure only."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = C.CDLL(LIB)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


class OracleDiverged(RuntimeError):
    pass


def _d(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(_dp)


class OracleWorld:
    """One environment of a Scene in the CPU restatement (World + SoftState)."""

    def _load(self):
        return load()

    def __init__(self, scene, env: int = 0, threads: int = 1, init: bool = True):
        self.lib = lib = self._load()
        self.scene = scene
        e = scene.envs[env]
        self.env = e
        nm = len(scene.materials)
        mats = abi.convert(scene.material_array(), abi.Material * nm)
        desc = abi.convert(scene.desc(), abi.SoftDesc)
        self.h = lib.oracle_create(C.byref(desc), mats, nm)
        self._after_create()
        lib.oracle_set_threads(threads)
        n = e.n
        self._keep = []

        def arr(a, shape, default):
            if a is None:
                a = np.broadcast_to(default, (n,) + shape)
            a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape((n,) + shape))
            self._keep.append(a)
            return a.ctypes.data_as(_dp)

        mat = np.ascontiguousarray(e.material if e.material is not None else np.zeros(n, np.int32), dtype=np.int32)
        self._keep.append(mat)
        self._check(lib.oracle_set_particles(self.h, n, arr(e.x, (3,), 0), arr(e.v, (3,), np.zeros(3)),
                                             arr(e.F, (3, 3), np.eye(3)), arr(e.C, (3, 3), np.zeros((3, 3))),
                                             arr(e.mass, (), 0), arr(e.vol0, (), 0), mat.ctypes.data_as(_ip)))
        cp = abi.Coupling()
        cp.mode, cp.r_c_factor, cp.c_d = scene.coupling_mode, scene.r_c_factor, scene.c_d
        lib.oracle_set_coupling(self.h, C.byref(cp))
        g = np.asarray(scene.rigid_gravity, dtype=np.float64)
        lib.oracle_set_stepping(self.h, scene.n_rigid, scene.n_soft, _d(g))
        if e.bodies:
            B = (abi.Body * len(e.bodies))(*[abi.convert(b.to_c(), abi.Body) for b in e.bodies])
            S = (abi.Shape * max(len(e.shapes), 1))(*[abi.convert(s.to_c(), abi.Shape) for s in e.shapes])
            self._check(lib.oracle_set_bodies(self.h, B, len(e.bodies), S, len(e.shapes)))
        if init:
            self._check(lib.oracle_init(self.h))

    def _after_create(self):
        pass

    def _check(self, rc):
        if rc == abi.MSIM_OK:
            return
        msg = self.lib.oracle_last_error(self.h).decode()
        if rc == abi.MSIM_ERR_DIVERGED:
            raise OracleDiverged(msg)
        raise ValueError(msg)

    # stepping
    def env_step(self):
        rep = abi.StepReport()
        self._check(self.lib.oracle_env_step(self.h, C.byref(rep)))
        return rep

    def set_kinematic_schedule(self, poses, mask=None):
        """poses[n_steps, n_bodies, 7] = (qw qx qy qz tx ty tz) per rigid step of the
        next env step, applied with Robot::set_kinematic_pose (rigid.hpp:142-151);
        mask selects the bodies (default: every kinematic body)."""
        p = np.ascontiguousarray(poses, dtype=np.float64)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        self._sched = (p, m)
        self._check(self.lib.oracle_set_kinematic_schedule(self.h, p.shape[0], p.ctypes.data_as(_dp),
                                                           None if m is None else m.ctypes.data_as(_u8p)))

    def soft_substep(self, n=1, hooks=True):
        cyc = C.c_int32()
        self._check(self.lib.oracle_soft_substep(self.h, n, 1 if hooks else 0, C.byref(cyc)))
        return cyc.value

    def p2g(self):
        self._check(self.lib.oracle_p2g(self.h))

    def grid_update(self):
        self._check(self.lib.oracle_grid_update(self.h))

    def g2p_advect(self):
        self._check(self.lib.oracle_g2p(self.h))

    def grid_clear(self):
        self.lib.oracle_grid_clear(self.h)

    def set_dt(self, dt):
        self.lib.oracle_set_dt(self.h, dt)

    def set_gravity(self, g):
        self.lib.oracle_set_gravity(self.h, _d(np.asarray(g, np.float64)))

    def set_lost_fraction_threshold(self, t):
        self.lib.oracle_set_lost_fraction_threshold(self.h, t)

    def penalty_particle(self):
        pen = C.c_double(0.0)
        self._check(self.lib.oracle_penalty_particle(self.h, C.byref(pen)))
        return pen.value

    # readback
    def particles(self):
        n = self.env.n
        x, v = np.zeros((n, 3)), np.zeros((n, 3))
        F, Cm = np.zeros((n, 3, 3)), np.zeros((n, 3, 3))
        lost = np.zeros(n, dtype=np.uint8)
        self.lib.oracle_read_particles(self.h, x.ctypes.data_as(_dp), v.ctypes.data_as(_dp),
                                       F.ctypes.data_as(_dp), Cm.ctypes.data_as(_dp), lost.ctypes.data_as(_u8p))
        return dict(x=x, v=v, F=F, C=Cm, lost=lost)

    def ext_force(self):
        f = np.zeros((self.env.n, 3))
        self.lib.oracle_read_ext_force(self.h, f.ctypes.data_as(_dp))
        return f

    def grid(self):
        nn = int(np.prod(self.scene.dims))
        m, p, f, v = np.zeros(nn), np.zeros((nn, 3)), np.zeros((nn, 3)), np.zeros((nn, 3))
        self.lib.oracle_read_grid(self.h, m.ctypes.data_as(_dp), p.ctypes.data_as(_dp), f.ctypes.data_as(_dp),
                                  v.ctypes.data_as(_dp))
        return dict(mass=m, momentum=p, force=f, velocity=v)

    def write_grid_velocity(self, vel):
        vel = np.ascontiguousarray(np.asarray(vel, np.float64).reshape(-1, 3))
        self.lib.oracle_write_grid_velocity(self.h, vel.ctypes.data_as(_dp))

    def binning(self):
        n = self.env.n
        d = self.scene.dims
        nbins = (d[0] - 2) * (d[1] - 2) * (d[2] - 2)
        nn = d[0] * d[1] * d[2]
        base = np.zeros((n, 3), dtype=np.int32)
        cs = np.zeros(nbins + 1, dtype=np.int32)
        cp = np.zeros(max(n, 1), dtype=np.int32)
        act = np.zeros(nn, dtype=np.int64)
        na, nact = C.c_int64(), C.c_int64()
        self._check(self.lib.oracle_read_binning(self.h, base.ctypes.data_as(_ip), cs.ctypes.data_as(_ip), cs.size,
                                                 cp.ctypes.data_as(_ip), cp.size, C.byref(na),
                                                 act.ctypes.data_as(_lp), act.size, C.byref(nact)))
        return dict(base=base, cell_start=cs, cell_particles=cp[: na.value], active_nodes=act[: nact.value])

    def wrenches(self, pending=False):
        nb = len(self.env.bodies)
        f, t = np.zeros((max(nb, 1), 3)), np.zeros((max(nb, 1), 3))
        self.lib.oracle_read_wrenches(self.h, 1 if pending else 0, f.ctypes.data_as(_dp), t.ctypes.data_as(_dp))
        return f[:nb], t[:nb]

    def bodies(self):
        nb = len(self.env.bodies)
        B = (abi.Body * max(nb, 1))()
        self.lib.oracle_read_bodies(self.h, B, nb)
        return [B[i] for i in range(nb)]

    def jp(self):
        out = np.zeros(self.env.n)
        self.lib.oracle_read_jp(self.h, out.ctypes.data_as(_dp))
        return out

    def lost_count(self):
        return int(self.lib.oracle_lost_count(self.h))

    def mean_particle_mass(self):
        return float(self.lib.oracle_mean_particle_mass(self.h))

    def time_env_steps(self, steps: int) -> float:
        err = C.c_int32(0)
        t = self.lib.oracle_time_env_steps(self.h, steps, C.byref(err))
        if err.value:
            self._check(err.value)
        return t

    def close(self):
        if getattr(self, "h", None):
            self.lib.oracle_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RefUnsupported(ValueError):
    """The scene uses something the reference does not have (a non-von-Mises model)."""


class RefWorld(OracleWorld):
    """One environment of a Scene run by the REFERENCE's own code (oracle/_ref)."""

    def _load(self):
        return load_ref()

    def _after_create(self):
        if self.lib.ref_unsupported(self.h):
            msg = self.lib.oracle_last_error(self.h).decode()
            self.lib.oracle_destroy(self.h)
            self.h = None
            raise RefUnsupported(msg)

    def state_hash(self) -> int:
        return int(self.lib.oracle_state_hash(self.h))


def constitutive(F: np.ndarray, mat=(1000.0, 1e4, 0.3, 2e3)):
    lib = load()
    m = abi.Material()
    m.density, m.youngs, m.poisson, m.yield_stress = mat[:4]
    m.model = mat[4] if len(mat) > 4 else 0
    F = np.ascontiguousarray(np.asarray(F, np.float64).reshape(-1, 3, 3))
    tau, Fp = np.zeros_like(F), np.zeros_like(F)
    rc = lib.oracle_constitutive(C.byref(m), F.shape[0], F.ctypes.data_as(_dp), tau.ctypes.data_as(_dp),
                                 Fp.ctypes.data_as(_dp))
    if rc != 0:
        raise ValueError("det(F) must be > 0")
    return tau, Fp


def run_kats() -> tuple[int, str]:
    if not os.path.exists(KAT):
        build()
    r = subprocess.run([KAT], capture_output=True, text=True)
    return r.returncode, r.stdout


# ---- task metrics and mesh baking (msim_oracle_tasks.hpp) -------------------
def _arr(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


def bake_mesh_sdf(tri, voxel, padding):
    """bake_mesh_sdf (sdf.hpp:277-310) -> (origin[3], dims[3], samples f32 x-fastest)."""
    lib = load()
    t, tp = _arr(tri)
    n = t.size // 9
    origin, dims = np.zeros(3), np.zeros(3, np.int32)
    rc = lib.oracle_bake_grid(tp, n, voxel, padding, origin.ctypes.data_as(_dp), dims.ctypes.data_as(_ip))
    if rc:
        raise ValueError("bake_mesh_sdf: invalid mesh")
    out = np.zeros(int(np.prod(dims)), np.float32)
    assert lib.oracle_bake_mesh_sdf(tp, n, voxel, padding, out.ctypes.data_as(C.POINTER(C.c_float)), out.size) == 0
    return origin, dims, out


def make_box_mesh(half, center=(0.0, 0.0, 0.0)):
    lib = load()
    h, hp = _arr(half)
    c, cp = _arr(center)
    tri = np.zeros(108)
    lib.oracle_make_box_mesh(hp, cp, tri.ctypes.data_as(_dp))
    return tri


def metric_fill(x, v, region):
    lib = load()
    xa, xp = _arr(x)
    va, vp = _arr(v)
    r, rp = _arr(region)
    f, m, s = C.c_double(), C.c_double(), C.c_int32()
    assert lib.oracle_metric_fill(len(xa), xp, vp, rp, C.byref(f), C.byref(m), C.byref(s)) == 0
    return f.value, m.value, bool(s.value)


def render_heightmap(x, region, nx, ny):
    lib = load()
    xa, xp = _arr(x)
    r, rp = _arr(region)
    out = np.zeros(nx * ny)
    assert lib.oracle_render_heightmap(len(xa), xp, rp, nx, ny, out.ctypes.data_as(_dp)) == 0
    return out


def metric_write_iou(nx, ny, threshold, a, b):
    lib = load()
    aa, ap = _arr(a)
    ba, bp = _arr(b)
    iou, s = C.c_double(), C.c_int32()
    assert lib.oracle_metric_write_iou(nx, ny, threshold, ap, bp, C.byref(iou), C.byref(s)) == 0
    return iou.value, bool(s.value)


def chamfer(a, b):
    lib = load()
    aa, ap = _arr(a)
    ba, bp = _arr(b)
    out = C.c_double()
    assert lib.oracle_chamfer(len(aa), ap, len(ba), bp, C.byref(out)) == 0
    return out.value


def metric_pinch(cur, init, tgt):
    lib = load()
    c, cp = _arr(cur)
    i, ip = _arr(init)
    t, tp = _arr(tgt)
    r, s = C.c_double(), C.c_int32()
    assert lib.oracle_metric_pinch(len(c), cp, len(i), ip, len(t), tp, C.byref(r), C.byref(s)) == 0
    return r.value, bool(s.value)
