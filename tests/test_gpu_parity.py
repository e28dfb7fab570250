"""Parity of the CUDA path against the CPU oracle on identical inputs.

Bars (BASELINE.json north_star / SURVEY.md §8d):
  * integer work bit-exact: base cells, stable per-cell particle lists,
    cell_start, active node set (fp32-rounded positions fed to both, App. A.2)
  * after one env step (25 substeps): positions and velocities within
    normwise relative 1e-4, per-body coupling force within 1e-3 (floor 1e-6 N)
  * P2G conservation: grid mass 1e-6, momentum 1e-5 relative (fp32)
"""
import numpy as np
import pytest

from gpu_helpers import rel, round_f32
from oracle.oracle_py import OracleWorld
from paper_2302_04659_b200 import GpuWorld
from paper_2302_04659_b200.scenes import config_a, config_b, config_c, config_d

pytestmark = pytest.mark.gpu

X_TOL = 1e-4
V_TOL = 1e-4
WRENCH_TOL = 1e-3


def _x_err(g, r, origin=np.zeros(3)):
    return float(np.linalg.norm(g - r) / np.linalg.norm(r - origin))


def _check_step(scene, env_g=0, steps=1, gw=None, ow=None, label=""):
    gw = gw or GpuWorld(scene)
    ow = ow or OracleWorld(scene, env=env_g)
    for _ in range(steps):
        rg = gw.env_step()
        ro = ow.env_step()
    pg, po = gw.particles(env_g), ow.particles()
    ex = _x_err(pg["x"], po["x"])
    ev = rel(pg["v"], po["v"])
    assert ex < X_TOL, f"{label} x rel err {ex:.3e}"
    assert ev < V_TOL, f"{label} v rel err {ev:.3e}"
    assert np.array_equal(pg["lost"], po["lost"])
    if scene.envs[env_g].bodies:
        fg, tg = gw.wrenches(env_g, pending=True)
        fo, to = ow.wrenches(pending=True)
        for b in range(len(fo)):
            scale = max(np.linalg.norm(fo[b]), 1e-6)
            assert np.linalg.norm(fg[b] - fo[b]) / scale < WRENCH_TOL, f"{label} body {b} force {fg[b]} vs {fo[b]}"
    return gw, ow, ex, ev


def test_config_a_one_env_step_parity():
    """Config A (the CPU reference's own case): 8k clay, 64^3, dynamic box."""
    scene = config_a()
    gw, ow, ex, ev = _check_step(scene, label="A")
    bg, bo = gw.bodies(0)[0], ow.bodies()[0]
    assert np.allclose(np.array(bg.t), np.array(bo.t), atol=1e-9)
    assert abs(bg.v[2] - bo.v[2]) <= 1e-3 * abs(bo.v[2])


def test_config_a_three_env_steps_parity():
    scene = config_a()
    _check_step(scene, steps=3, label="A x3")


@pytest.mark.parametrize("cfg", [config_b, config_c])
def test_clay_variants_one_env_step(cfg):
    scene = cfg()
    _check_step(scene, label=scene.name)


def test_config_d_sampled_envs():
    """Batched D: 8 sampled envs (write + pinch) run as one batch vs the oracle per env."""
    scene = config_d(n_envs=8)
    gw = GpuWorld(scene)
    gw.env_step()
    for e in range(8):
        ow = OracleWorld(scene, env=e)
        ow.env_step()
        pg, po = gw.particles(e), ow.particles()
        assert _x_err(pg["x"], po["x"]) < X_TOL, e
        assert rel(pg["v"], po["v"]) < V_TOL, e
        fg, _ = gw.wrenches(e, pending=True)
        fo, _ = ow.wrenches(pending=True)
        for b in range(len(fo)):
            assert np.linalg.norm(fg[b] - fo[b]) / max(np.linalg.norm(fo[b]), 1e-6) < WRENCH_TOL, (e, b)


@pytest.mark.parametrize("cfg,factor", [(config_a, 2), (config_c, 1), (lambda: config_d(n_envs=4), 2)])
def test_bucket_factor_is_internal(cfg, factor):
    """Particle buckets of 1 or 2^3 node blocks (chosen from the density by
    default: A/D dense -> 1, C sparse -> 2): the other shape gives the same
    physics within the parity bars."""
    scene = cfg()
    gw = GpuWorld(scene, bucket_factor=factor)
    _check_step(scene, env_g=0, gw=gw, label=f"{scene.name} factor {factor}")  # one env step vs the oracle
    gw2 = GpuWorld(scene)  # the automatic choice
    gw2.env_step()
    for e in range(len(scene.envs)):
        a, b = gw.particles(e), gw2.particles(e)
        assert _x_err(a["x"], b["x"]) < X_TOL and rel(a["v"], b["v"]) < V_TOL


def test_integer_binning_bit_exact():
    """base, cell_start, cell_particles (index-stable), active_nodes == reference layout."""
    scene = round_f32(config_a())
    gw = GpuWorld(scene, record_binning=True)
    ow = OracleWorld(scene)
    gw.p2g()
    ow.p2g()
    bg, bo = gw.binning(0), ow.binning()
    assert np.array_equal(bg["base"], bo["base"])
    assert np.array_equal(bg["cell_start"], bo["cell_start"])
    assert np.array_equal(bg["cell_particles"], bo["cell_particles"])
    assert np.array_equal(bg["active_nodes"], bo["active_nodes"])


def test_integer_binning_with_lost_and_edges():
    """Particles outside the domain, on cell boundaries and in the boundary band."""
    from gpu_helpers import Cloud, make_scene

    rng = np.random.default_rng(5)
    c = Cloud()
    for _ in range(300):
        c.add(rng.uniform(0.0, 0.32, 3), rng.uniform(-0.1, 0.1, 3))
    for i in range(8):  # exactly on node / half-node coordinates
        c.add((0.05 + 0.01 * i, 0.105, 0.15))
    c.add((-0.01, 0.1, 0.1))
    c.add((0.5, 0.1, 0.1))
    scene = round_f32(make_scene(c))
    scene.lost_fraction_threshold = 1.0
    gw = GpuWorld(scene, record_binning=True)
    ow = OracleWorld(scene)
    gw.p2g()
    ow.p2g()
    bg, bo = gw.binning(0), ow.binning()
    for k in ("base", "cell_start", "cell_particles", "active_nodes"):
        assert np.array_equal(bg[k], bo[k]), k
    assert gw.lost_count() == ow.lost_count() > 0


def test_p2g_grid_fields_match_oracle():
    scene = round_f32(config_a())
    e = scene.envs[0]
    rng = np.random.default_rng(3)
    e.F = np.eye(3) + rng.uniform(-0.02, 0.02, (e.n, 3, 3))  # non-trivial stress (acceptance.cpp:66-69)
    e.C = rng.uniform(-0.5, 0.5, (e.n, 3, 3))
    gw = GpuWorld(scene, split_channels=True)
    ow = OracleWorld(scene)
    gw.p2g()
    ow.p2g()
    gg, go = gw.grid(0), ow.grid()
    em, ep, ef = rel(gg["mass"], go["mass"]), rel(gg["momentum"], go["momentum"]), rel(gg["force"], go["force"])
    assert em < 1e-6 and ep < 1e-5 and ef < 1e-4, (em, ep, ef)
    assert abs(gg["mass"].sum() - go["mass"].sum()) <= 1e-6 * go["mass"].sum()
