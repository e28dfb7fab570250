"""The committed golden vectors of the REFERENCE itself (tests/golden/ref_*.npz,
made by tests/golden/make_golden.py from oracle/_ref -- the reference's own
sources) pin the oracle on any machine (no /root/reference needed), and the
CUDA path on the GPU box."""
import hashlib
import os

import numpy as np
import pytest

from oracle.oracle_py import OracleWorld

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ["A", "B", "D0", "D1"]


def _case(name):
    from paper_2302_04659_b200.scenes import config_a, config_b, config_d

    return {"A": (config_a, 0), "B": (config_b, 0), "D0": (lambda: config_d(2), 0),
            "D1": (lambda: config_d(2), 1)}[name]


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_reference_golden(name):
    g = np.load(os.path.join(HERE, f"ref_{name}.npz"))
    make, env = _case(name)
    w = OracleWorld(make(), env=env)
    rep = w.env_step()
    p = w.particles()
    idx = g["idx"]
    assert _rel(p["x"][idx], g["x"]) < 1e-13 and _rel(p["v"][idx], g["v"]) < 1e-11
    assert _rel(p["F"][idx], g["F"]) < 1e-12 and _rel(p["C"][idx], g["C"]) < 1e-10
    assert int(p["lost"].sum()) == int(g["lost"])
    assert [rep.rigid_steps, rep.soft_substeps, rep.cfl_cycles, rep.lost_particles] == g["report"].tolist()
    assert abs(rep.max_penetration - g["report_f"][0]) <= 1e-12
    f, t = w.wrenches(pending=True)
    assert np.allclose(f, g["force"], rtol=1e-9, atol=1e-12) and np.allclose(t, g["torque"], rtol=1e-9, atol=1e-12)
    w.grid_clear()
    w.p2g()
    b = w.binning()
    keys = ("base", "cell_start", "cell_particles", "active_nodes")
    assert [len(b[k]) for k in keys] == g["bin_len"].tolist()
    assert [hashlib.sha256(np.ascontiguousarray(b[k]).tobytes()).hexdigest() for k in keys] == g["bin_sha"].tolist()


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_matches_reference_golden(name):
    from paper_2302_04659_b200 import GpuWorld

    g = np.load(os.path.join(HERE, f"ref_{name}.npz"))
    make, env = _case(name)
    gw = GpuWorld(make())
    gw.env_step()
    p = gw.particles(env)
    idx = g["idx"]
    assert _rel(p["x"][idx], g["x"]) < 1e-4 and _rel(p["v"][idx], g["v"]) < 1e-4
    f, _ = gw.wrenches(env, pending=True)
    for k in range(len(g["force"])):
        assert np.linalg.norm(f[k] - g["force"][k]) / max(np.linalg.norm(g["force"][k]), 1e-6) < 1e-3
