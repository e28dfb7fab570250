"""§8(f)#1: the device-resident rigid loop with a per-rigid-step kinematic
collider schedule, and msim_gpu_set_bodies isolation between envs.

The reference moves robot-driven links once per rigid step inside env_step
(coupling.hpp:252-258): Robot::set_kinematic_pose jumps each link to its new
pose and gives it the finite-difference twist (rigid.hpp:142-151). Here a
non-constant finger / stamp trajectory (accelerating, rotating) is uploaded
once per env step for all envs and must match the reference World (and the
oracle) driven by the same poses, rigid step by rigid step.
"""
import math

import numpy as np
import pytest

from gpu_helpers import rel
from oracle import oracle_py
from oracle.oracle_py import OracleWorld, RefWorld
from paper_2302_04659_b200 import GpuWorld, abi
from paper_2302_04659_b200.scenes import config_d

X_TOL, V_TOL, WRENCH_TOL = 1e-4, 1e-4, 1e-3


def _kinematic_d(n_envs=2):
    sc = config_d(n_envs=n_envs)
    for e in sc.envs:
        for b in e.bodies:
            b.mode = abi.BODY_KINEMATIC
    return sc


def schedule(sc, step, n_rigid=25):
    """Poses [n_rigid, n_total, 7] of every body for env step `step`: pinch fingers
    close with an accelerating, oscillating gap and a small yaw; the stamp
    presses down with a sinusoidal speed and tilts."""
    dt_r = sc.dt * sc.n_soft
    rows = []
    for r in range(n_rigid):
        t = (step * n_rigid + r + 1) * dt_r
        row = []
        for e in sc.envs:
            for k, b in enumerate(e.bodies):
                x0 = np.array(b.t)
                if len(e.bodies) == 2:  # pinch: fingers move toward each other
                    s = 1.0 if k == 0 else -1.0
                    d = 0.5 * 0.4 * t * t + 0.002 * math.sin(60.0 * t)
                    pos = x0 + np.array([s * d, 0.0, 0.0])
                    ang = 0.3 * t * s
                    q = (math.cos(ang / 2), 0.0, 0.0, math.sin(ang / 2))
                else:  # write stamp: presses down and tilts about x
                    pos = x0 + np.array([0.0, 0.0, -0.02 * t - 0.003 * math.sin(40.0 * t)])
                    ang = 0.5 * t
                    q = (math.cos(ang / 2), math.sin(ang / 2), 0.0, 0.0)
                row.append(list(q) + list(pos))
        rows.append(row)
    return np.array(rows, dtype=np.float64)


def _env_slice(sc, poses, e):
    off = sum(len(x.bodies) for x in sc.envs[:e])
    return np.ascontiguousarray(poses[:, off:off + len(sc.envs[e].bodies), :])


@pytest.mark.skipif(not oracle_py.ref_available(), reason="oracle/_ref not built")
def test_schedule_oracle_matches_reference_cpu():
    """CPU: the restatement's schedule handling equals the reference's own
    Robot::set_kinematic_pose path to round-off (no GPU)."""
    sc = _kinematic_d(2)
    for e in range(2):
        o, r = OracleWorld(sc, env=e), RefWorld(sc, env=e)
        for step in range(2):
            p = _env_slice(sc, schedule(sc, step), e)
            o.set_kinematic_schedule(p)
            r.set_kinematic_schedule(p)
            o.env_step()
            r.env_step()
        po, pr = o.particles(), r.particles()
        assert rel(po["x"], pr["x"]) < 1e-13 and rel(po["v"], pr["v"]) < 1e-10
        for bo, br in zip(o.bodies(), r.bodies()):
            assert np.allclose(bo.t, br.t, rtol=0, atol=1e-15) and np.allclose(bo.q, br.q, rtol=0, atol=1e-15)
            assert np.allclose(bo.v, br.v, rtol=1e-12, atol=1e-15) and np.allclose(bo.w, br.w, rtol=1e-10, atol=1e-13)
        fo, _ = o.wrenches(True)
        fr, _ = r.wrenches(True)
        assert np.allclose(fo, fr, rtol=1e-9, atol=1e-12)


def test_schedule_length_must_match_n_rigid_cpu():
    sc = _kinematic_d(2)
    o = OracleWorld(sc, env=0)
    o.set_kinematic_schedule(_env_slice(sc, schedule(sc, 0, n_rigid=5), 0))
    with pytest.raises(ValueError):
        o.env_step()


@pytest.mark.gpu
@pytest.mark.skipif(not oracle_py.ref_available(), reason="oracle/_ref not built")
def test_gpu_schedule_matches_reference_two_env_steps():
    sc = _kinematic_d(2)
    gw = GpuWorld(sc)
    refs = [RefWorld(sc, env=e) for e in range(2)]
    for step in range(2):
        poses = schedule(sc, step)
        gw.set_kinematic_schedule(poses)  # one upload for every env and rigid step
        gw.env_step()
        for e, r in enumerate(refs):
            r.set_kinematic_schedule(_env_slice(sc, poses, e))
            r.env_step()
    for e, r in enumerate(refs):
        pg, pr = gw.particles(e), r.particles()
        assert rel(pg["x"], pr["x"]) < X_TOL and rel(pg["v"], pr["v"]) < V_TOL, e
        for bg, br in zip(gw.bodies(e), r.bodies()):  # fp64 on both sides
            assert np.allclose(bg.t, br.t, rtol=0, atol=1e-15) and np.allclose(bg.q, br.q, rtol=0, atol=1e-14)
            assert np.allclose(bg.v, br.v, rtol=1e-10, atol=1e-14) and np.allclose(bg.w, br.w, rtol=1e-8, atol=1e-12)
        fg, _ = gw.wrenches(e, pending=True)
        fr, _ = r.wrenches(pending=True)
        for b in range(len(fr)):
            assert np.linalg.norm(fg[b] - fr[b]) / max(np.linalg.norm(fr[b]), 1e-6) < WRENCH_TOL, (e, b)
        assert np.linalg.norm(fr) > 0  # in contact: the trajectory matters


@pytest.mark.gpu
def test_gpu_schedule_errors():
    sc = _kinematic_d(2)
    gw = GpuWorld(sc)
    gw.set_kinematic_schedule(schedule(sc, 0, n_rigid=5))
    with pytest.raises(ValueError):
        gw.env_step()  # 5 poses for a 25-rigid-step env step
    gw.env_step()  # the rejected schedule was dropped
    sd = config_d(n_envs=1)  # scripted stamp: not selected by default ...
    gw2 = GpuWorld(sd)
    gw2.set_kinematic_schedule(schedule(sd, 0), mask=np.ones(1, np.uint8))  # ... but can be selected explicitly
    gw2.env_step()


@pytest.mark.gpu
def test_set_bodies_leaves_other_envs_untouched():
    """msim_gpu_set_bodies(env 1) must not reset or move env 0's bodies or its
    accumulating / staged wrenches (worlds are independent)."""
    from paper_2302_04659_b200.scenes import BodySpec, ShapeSpec

    sc = config_d(n_envs=3)
    gw = GpuWorld(sc)
    gw.env_step()
    before = {e: (gw.wrenches(e, False), gw.wrenches(e, True), [tuple(b.t) + tuple(b.v) for b in gw.bodies(e)])
              for e in (0, 2)}
    assert np.linalg.norm(before[0][1][0]) > 0
    newb = [BodySpec(mode=abi.BODY_SCRIPTED, t=(0.16, 0.16, 0.2), v=(0.0, 0.0, -0.01))]
    news = [ShapeSpec(abi.SHAPE_SPHERE, 0, params=(0.02,))]
    gw.set_bodies(1, newb, news)
    for e in (0, 2):
        w0, p0, b0 = before[e]
        w1, p1, b1 = gw.wrenches(e, False), gw.wrenches(e, True), [tuple(b.t) + tuple(b.v) for b in gw.bodies(e)]
        assert all(np.array_equal(a, b) for a, b in zip(w0, w1)), e
        assert all(np.array_equal(a, b) for a, b in zip(p0, p1)), e
        assert b0 == b1, e
    f1, _ = gw.wrenches(1, pending=True)
    assert np.all(f1 == 0)  # the re-configured env starts from zero wrenches
    # stepping on: envs 0 and 2 follow the same trajectory as an untouched batch
    ref = GpuWorld(sc)
    ref.env_step()
    gw.env_step()
    ref.env_step()
    for e in (0, 2):
        a, b = gw.particles(e), ref.particles(e)
        assert rel(a["x"], b["x"]) < 1e-6 and rel(a["v"], b["v"]) < 1e-5, e
