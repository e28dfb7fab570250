"""Pinning the oracle to the REFERENCE itself.

oracle/_ref/ holds the reference's own, unchanged sources compiled against
the Eigen / GoogleTest subsets in oracle/ref_shim/ (oracle/Makefile.ref):
  * the reference's test suites (test_mpm.cpp, test_coupling.cpp, ...,
    acceptance.cpp) run here and must pass, as they did in the reference's
    own CI record (proj/test_output.txt) -- this pins the shim;
  * libmsim_ref.so drives the reference's World / soft_substep / env_step on
    the same inputs as the restatement (oracle/_build/liboracle.so), which is
    then required to agree with it to round-off.
All CPU-only (no GPU). The GPU parity tests compare the CUDA path against
both (tests/test_gpu_reference.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle_py
from oracle.oracle_py import OracleWorld, RefWorld, RefUnsupported

REF = oracle_py.REF_DIR
SUITES = ["test_geometry", "test_sdf", "test_mpm", "test_rigid", "test_control", "test_coupling", "test_scenario",
          "test_demo"]
# TEST() counts of the reference's suites (grep -c "^TEST(" proj/tests/<suite>.cpp)
SUITE_TESTS = {"test_geometry": 22, "test_sdf": 18, "test_mpm": 27, "test_rigid": 13, "test_control": 18,
               "test_coupling": 17, "test_scenario": 34, "test_demo": 17}

needs_ref = pytest.mark.skipif(not oracle_py.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_the_shim(suite):
    exe = os.path.join(REF, suite)
    if not os.path.exists(exe):
        pytest.skip(f"{suite} not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]
    ok = r.stdout.count("[       OK ]")
    assert ok == SUITE_TESTS[suite], r.stdout[-2000:]


@needs_ref
def test_reference_acceptance_criteria_pass_on_the_shim():
    exe = os.path.join(REF, "acceptance")
    if not os.path.exists(exe):
        pytest.skip("acceptance not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "ALL CRITERIA PASSED" in r.stdout
    for crit in ("grid-transfer conservation", "constitutive model", "contact coupling", "determinism"):
        assert f"PASS: {crit}" in r.stdout


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _configs():
    from paper_2302_04659_b200.scenes import config_a, config_b, config_c, config_d

    return {"A": (config_a, 0), "B": (config_b, 0), "C": (config_c, 0), "D-write": (lambda: config_d(2), 0),
            "D-pinch": (lambda: config_d(2), 1)}


@needs_ref
@pytest.mark.parametrize("cfg", ["A", "B", "C", "D-write", "D-pinch"])
def test_oracle_matches_reference_one_env_step(cfg):
    """One env step (25 substeps) of configs A-D (clay parity variants): the
    restatement equals the reference to round-off in every particle field, the
    wrenches (current and staged), the bodies and the StepReport."""
    make, env = _configs()[cfg]
    sc = make()
    o, r = OracleWorld(sc, env=env), RefWorld(sc, env=env)
    ro, rr = o.env_step(), r.env_step()
    po, pr = o.particles(), r.particles()
    assert _rel(po["x"], pr["x"]) < 1e-13
    assert _rel(po["v"], pr["v"]) < 1e-11
    assert _rel(po["F"], pr["F"]) < 1e-12
    assert _rel(po["C"], pr["C"]) < 1e-10
    assert np.array_equal(po["lost"], pr["lost"])
    for pending in (False, True):
        fo, to = o.wrenches(pending)
        fr, tr = r.wrenches(pending)
        assert np.allclose(fo, fr, rtol=1e-9, atol=1e-12) and np.allclose(to, tr, rtol=1e-9, atol=1e-12)
    for bo, br in zip(o.bodies(), r.bodies()):
        assert np.allclose(np.array(bo.t), np.array(br.t), rtol=0, atol=1e-14)
        assert np.allclose(np.array(bo.v), np.array(br.v), rtol=0, atol=1e-12)
    assert (ro.rigid_steps, ro.soft_substeps, ro.cfl_cycles, ro.lost_particles) == \
           (rr.rigid_steps, rr.soft_substeps, rr.cfl_cycles, rr.lost_particles)
    assert abs(ro.max_penetration - rr.max_penetration) <= 1e-12
    assert abs(ro.max_force_balance_error - rr.max_force_balance_error) <= 1e-12


@needs_ref
def test_oracle_binning_matches_reference_bit_exact():
    """p2g's integer work (mpm.hpp:210-280): base cells, counting-sort layout,
    active nodes -- identical between the restatement and the reference."""
    from paper_2302_04659_b200.scenes import config_b

    sc = config_b()
    o, r = OracleWorld(sc), RefWorld(sc)
    for w in (o, r):
        w.env_step()  # move the particles first
        w.grid_clear()
        w.p2g()
    bo, br = o.binning(), r.binning()
    for k in ("base", "cell_start", "cell_particles", "active_nodes"):
        assert np.array_equal(bo[k], br[k]), k


@needs_ref
def test_oracle_constitutive_matches_reference():
    """kirchhoff_stress / von_mises_return_map (mpm.hpp:152-181) on random
    trial states past yield (the ReturnMap test's distribution, test_mpm.cpp:301-328)."""
    rng = np.random.default_rng(3)
    F = np.eye(3) + 0.2 * rng.uniform(-1, 1, size=(500, 3, 3))
    F = F[np.linalg.det(F) > 0.1]
    lo, lr = oracle_py.load(), oracle_py.load_ref()
    from oracle import cabi

    m = cabi.Material(1000.0, 1e4, 0.3, 2e3, 0)
    dp = C.POINTER(C.c_double)
    out = []
    for lib in (lo, lr):
        tau, Fp = np.zeros_like(F), np.zeros_like(F)
        assert lib.oracle_constitutive(C.byref(m), F.shape[0], F.ctypes.data_as(dp), tau.ctypes.data_as(dp),
                                       Fp.ctypes.data_as(dp)) == 0
        out.append((tau, Fp))
    assert _rel(out[0][0], out[1][0]) < 1e-12
    assert _rel(out[0][1], out[1][1]) < 1e-13


@needs_ref
def test_oracle_sdf_matches_reference_all_shape_types():
    """sdf_eval / sdf_gradient (sdf.hpp:114-201), incl. the trilinear volume."""
    from oracle import cabi
    from paper_2302_04659_b200.scenes import ShapeSpec, box_sdf_volume, quat_from_axis_angle

    dims, org, vox, smp = box_sdf_volume((0.04, 0.04, 0.03), 0.01, 0.03)
    q = quat_from_axis_angle((1.0, 2.0, 0.5), 0.7)
    shapes = [ShapeSpec(0, 0, params=(0.0, 0.6, 0.8, 0.05)), ShapeSpec(1, 0, params=(0.05,), local_q=q),
              ShapeSpec(2, 0, params=(0.04, 0.03, 0.02), local_q=q, local_t=(0.01, -0.02, 0.03)),
              ShapeSpec(3, 0, params=(0.04, 0.02), local_q=q),
              ShapeSpec(4, 0, vol_dims=dims, vol_origin=org, vol_voxel=vox, vol_samples=smp, local_q=q)]
    rng = np.random.default_rng(5)
    p = rng.uniform(-0.12, 0.12, size=(2000, 3))
    dp = C.POINTER(C.c_double)
    for s in shapes:
        cs = cabi.convert(s.to_c(), cabi.Shape)
        res = []
        for lib in (oracle_py.load(), oracle_py.load_ref()):
            phi, g = np.zeros(len(p)), np.zeros_like(p)
            assert lib.oracle_sdf(C.byref(cs), len(p), p.ctypes.data_as(dp), phi.ctypes.data_as(dp),
                                  g.ctypes.data_as(dp)) == 0
            res.append((phi, g))
        assert np.allclose(res[0][0], res[1][0], rtol=0, atol=1e-15), s.type
        assert np.allclose(res[0][1], res[1][1], rtol=0, atol=1e-12), s.type


@needs_ref
@pytest.mark.parametrize("cfg,envs", [("A", [0]), ("B", [0, 1]), ("C", [0]), ("D", [0, 1, 2, 3])])
def test_reference_harness_builders_match_scenes(cfg, envs):
    """bench.py --impl reference builds its worlds in the reference harness with
    the reference's own seeder (oracle/ref_scenes.py, no product import); they
    must be the same worlds as the product's scenes (bit-identical)."""
    from oracle import ref_scenes
    from paper_2302_04659_b200 import scenes

    make = {"A": lambda n: scenes.config_a(), "B": lambda n: scenes.config_b(n_envs=n),
            "C": lambda n: scenes.config_c(n_envs=n), "D": lambda n: scenes.config_d(n)}[cfg]
    sc = make(len(envs))
    lib = oracle_py.load_ref()
    dp = C.POINTER(C.c_double)
    for e in envs:
        h = ref_scenes.build_world(cfg, e)
        n = lib.oracle_particle_count(h)
        x, v = np.zeros((n, 3)), np.zeros((n, 3))
        lib.oracle_read_particles(h, x.ctypes.data_as(dp), v.ctypes.data_as(dp), None, None, None)
        nb = len(sc.envs[e].bodies)
        B = (oracle_py.abi.Body * nb)()
        lib.oracle_read_bodies(h, B, nb)
        lib.oracle_destroy(h)
        assert np.array_equal(x, sc.envs[e].x) and np.array_equal(v, sc.envs[e].v)
        for b, spec in zip(B, sc.envs[e].bodies):
            assert tuple(b.t) == tuple(spec.t) and tuple(b.v) == tuple(spec.v) and tuple(b.w) == tuple(spec.w)
            assert b.mode == spec.mode and b.mass == spec.mass and tuple(b.inertia) == tuple(spec.inertia)
        cs = [oracle_py.abi.convert(s.to_c(), oracle_py.abi.Shape) for s in sc.envs[e].shapes]
        rs = ref_scenes._spec(cfg, e)[9]
        assert len(cs) == len(rs)
        for a, b in zip(cs, rs):
            assert bytes(a) == bytes(b)


@needs_ref
def test_reference_rejects_models_it_does_not_have():
    from paper_2302_04659_b200.scenes import SAND, config_b

    with pytest.raises(RefUnsupported):
        RefWorld(config_b(material=SAND))
