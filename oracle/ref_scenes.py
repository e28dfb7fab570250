"""ORACLE — TEST INFRASTRUCTURE ONLY.

Configs A-D (clay parity variants) built directly inside
the reference harness (oracle/_ref/libmsim_ref.so) with the reference's own
seeder (seed_particles_box, seeding.hpp:13-35) -- for bench.py's
``--impl reference`` arm, which must not import or load the product. The
numbers below restate paper_2302_04659_b200/scenes.py; tests/test_reference_pin.py
checks every particle, body and shape of these worlds is bit-identical to the
product's scenes.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from oracle import cabi
from oracle import oracle_py

V0 = 6.2e-8                       # mpm.hpp:47
SOFT_CLAY = (1000.0, 1e4, 0.3, 2e3)
FIRM_CLAY = (1000.0, 1e5, 0.3, 4e3)
_dp = C.POINTER(C.c_double)


def lattice_span(n: int) -> float:
    return (n + 0.5) * V0 ** (1.0 / 3.0)


def _body(mode, t, v=(0.0, 0.0, 0.0), w=(0.0, 0.0, 0.0), mass=1.0, inertia=(1e-3,) * 3):
    b = cabi.Body()
    b.mode = mode
    b.q[:] = (1.0, 0.0, 0.0, 0.0)
    b.t[:] = t
    b.v[:] = v
    b.w[:] = w
    b.mass = mass
    b.inertia[:] = inertia
    return b


def _box(body, half, local_t=(0.0, 0.0, 0.0), friction=0.5, k_n=20.0, k_t=0.1):
    s = cabi.Shape()
    s.type = cabi.SHAPE_BOX
    s.body = body
    s.local_q[:] = (1.0, 0.0, 0.0, 0.0)
    s.local_t[:] = local_t
    s.friction, s.k_n, s.k_t = friction, k_n, k_t
    s.params[:] = tuple(half) + (0.0,)
    return s


def _bucket(body, half_w, half_h, wall, friction=0.2):
    sh = [_box(body, (half_w, half_w, wall), (0, 0, -half_h), friction)]
    for sx, sy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
        if sx:
            sh.append(_box(body, (wall, half_w, half_h), (sx * (half_w + wall), 0.0, 0.0), friction))
        else:
            sh.append(_box(body, (half_w, wall, half_h), (0.0, sy * (half_w + wall), 0.0), friction))
    return sh


def _spec(config: str, e: int):
    """(dims, h, dt, material, lo, lattice, seed, vel_seed, bodies, shapes)"""
    if config == "A":
        lo = (0.28, 0.28, 0.05)
        top = lo[2] + lattice_span(20)
        cxy = lo[0] + 0.5 * lattice_span(20)
        bodies = [_body(cabi.BODY_DYNAMIC, (cxy, cxy, top + 0.002 + 0.01), v=(0.0, 0.0, -0.2), mass=0.05,
                        inertia=(8e-6,) * 3)]
        return 64, 0.01, 5e-4, SOFT_CLAY, lo, (20, 20, 20), 1, 2, bodies, [_box(0, (0.03, 0.03, 0.01))]
    if config == "B":
        lo = (0.2399, 0.2399, 0.021)
        top = lo[2] + lattice_span(20)
        bodies = [_body(cabi.BODY_SCRIPTED, (lo[0] + 0.04, 0.32, top + 0.02), v=(0.05, 0.0, -0.05))]
        return 64, 0.01, 5e-4, SOFT_CLAY, lo, (40, 40, 20), 3 + 10 * e, 4 + 10 * e, bodies, _bucket(0, 0.03, 0.02, 0.004)
    if config == "C":
        lo = (0.24, 0.24, 0.06)
        c = lo[0] + 0.5 * lattice_span(40)
        bodies = [_body(cabi.BODY_SCRIPTED, (c, c, lo[2] + 0.085), w=(0.0, 0.5, 0.0)),
                  _body(cabi.BODY_KINEMATIC, (c + 0.2, c, 0.06))]
        shapes = _bucket(0, 0.09, 0.085, 0.005) + _bucket(1, 0.06, 0.04, 0.005)
        return 128, 0.005, 5e-4, SOFT_CLAY, lo, (40, 40, 40), 5 + 10 * e, 6 + 10 * e, bodies, shapes
    if config == "D":
        lat = (32, 32, 16)
        span = [lattice_span(n) for n in lat]
        lo = ((0.32 - span[0]) / 2, (0.32 - span[1]) / 2, 0.021)
        cx, cy = lo[0] + span[0] / 2, lo[1] + span[1] / 2
        top = lo[2] + span[2]
        if e % 2 == 0:
            bodies = [_body(cabi.BODY_SCRIPTED, (cx, cy, top + 0.008 + 0.001), v=(0.0, 0.0, -0.02))]
            shapes = [_box(0, (0.03, 0.01, 0.008), friction=0.3, k_n=80.0)]
        else:
            zc = lo[2] + span[2] / 2
            off = span[0] / 2 + 0.004 + 0.001
            bodies = [_body(cabi.BODY_SCRIPTED, (cx - off, cy, zc), v=(0.01, 0.0, 0.0)),
                      _body(cabi.BODY_SCRIPTED, (cx + off, cy, zc), v=(-0.01, 0.0, 0.0))]
            shapes = [_box(0, (0.004, 0.012, 0.018)), _box(1, (0.004, 0.012, 0.018))]
        return 32, 0.01, 2.5e-4, FIRM_CLAY, lo, lat, 1000 + e, 5000 + e, bodies, shapes
    raise ValueError(f"no reference-harness builder for config {config!r}")


def build_world(config: str, e: int = 0):
    """A ref_world* (reference World, initialised) for env e of config A-D."""
    lib = oracle_py.load_ref()
    dims, h, dt, mat, lo, lat, seed, vseed, bodies, shapes = _spec(config, e)
    d = cabi.SoftDesc()
    d.h = h
    d.dims[:] = (dims,) * 3
    d.gravity[:] = (0.0, 0.0, -9.81)
    d.dt = dt
    d.cfl_factor = 0.4
    d.max_cfl_halvings = 4
    d.lost_fraction_threshold = 0.01
    m = (cabi.Material * 1)()
    m[0].density, m[0].youngs, m[0].poisson, m[0].yield_stress = mat
    w = lib.oracle_create(C.byref(d), m, 1)
    lo_a = np.array(lo, dtype=np.float64)
    hi_a = np.array([lo[a] + lattice_span(lat[a]) for a in range(3)], dtype=np.float64)
    rng = lib.oracle_rng_create(seed)
    n = lib.oracle_seed_box(w, rng, lo_a.ctypes.data_as(_dp), hi_a.ctypes.data_as(_dp), 0, V0)
    lib.oracle_rng_destroy(rng)
    vr = lib.oracle_rng_create(vseed)
    v = np.array([lib.oracle_rng_uniform(vr, -0.1, 0.1) for _ in range(3 * n)], dtype=np.float64)
    lib.oracle_rng_destroy(vr)
    assert lib.oracle_write_particles(w, n, None, v.ctypes.data_as(_dp), None, None) == 0
    B = (cabi.Body * len(bodies))(*bodies)
    S = (cabi.Shape * len(shapes))(*shapes)
    assert lib.oracle_set_bodies(w, B, len(bodies), S, len(shapes)) == 0
    cp = cabi.Coupling()
    cp.mode, cp.r_c_factor, cp.c_d = cabi.COUPLING_PARTICLE, 0.5, 0.05
    lib.oracle_set_coupling(w, C.byref(cp))
    g = np.array([0.0, 0.0, -9.81])
    lib.oracle_set_stepping(w, 25, 1, g.ctypes.data_as(_dp))
    if lib.oracle_init(w) != 0:
        raise RuntimeError(lib.oracle_last_error(w).decode())
    return w
