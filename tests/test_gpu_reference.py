"""The CUDA path against the REFERENCE's own code (oracle/_ref/libmsim_ref.so:
the reference sources compiled unchanged, tests/test_reference_pin.py) and the
hot path's own integer outputs against the reference's counting sort and
active nodes.

Bars (BASELINE.json north_star):
  * after one env step (25 substeps): x, v normwise relative <= 1e-4, per-body
    coupling force <= 1e-3 (floor 1e-6 N);
  * integer work bit-exact: the hot path's per-bucket particle counts equal the
    histogram of the reference's base cells, and its touched node-block list
    equals the blocks of the reference's active_nodes (mpm.hpp:251-280), with
    the reference fed the GPU's fp32 positions (App. A.2);
  * StepReport: third-law force balance (acceptance.cpp:156-193 criterion 3,
    every cycle of every substep) and max penetration against the reference's.
"""
import os

import numpy as np
import pytest

from gpu_helpers import rel
from oracle import oracle_py
from oracle.oracle_py import OracleWorld, RefWorld
from paper_2302_04659_b200 import GpuWorld
from paper_2302_04659_b200.scenes import config_a, config_b, config_c, config_d, config_e

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle_py.ref_available(), reason="oracle/_ref not built")]

X_TOL, V_TOL, WRENCH_TOL = 1e-4, 1e-4, 1e-3


def _xerr(g, r):
    return float(np.linalg.norm(g - r) / np.linalg.norm(r))


def _compare_env(gw, e, ref, rg, rr, label):
    pg, pr = gw.particles(e), ref.particles()
    ex, ev = _xerr(pg["x"], pr["x"]), rel(pg["v"], pr["v"])
    assert ex < X_TOL and ev < V_TOL, f"{label}: x {ex:.2e} v {ev:.2e}"
    assert np.array_equal(pg["lost"], pr["lost"]), label
    if ref.env.bodies:
        fg, tg = gw.wrenches(e, pending=True)
        fr, tr = ref.wrenches(pending=True)
        for b in range(len(fr)):
            assert np.linalg.norm(fg[b] - fr[b]) / max(np.linalg.norm(fr[b]), 1e-6) < WRENCH_TOL, (label, b, fg[b], fr[b])
    return ex, ev


@pytest.mark.parametrize("split", ["auto", "1"])
@pytest.mark.parametrize("name", ["A", "B", "C"])
def test_single_scene_one_env_step_matches_reference(name, split, monkeypatch):
    """split: the particle kernel's bucket split for small scenes (auto: a bucket's
    rounds over several CTAs with atomic ranks; 1: one CTA per bucket, stable ranks)."""
    if split != "auto":
        monkeypatch.setenv("MSIM_SPLIT_R", split)
    scene = {"A": config_a, "B": config_b, "C": config_c}[name]()
    gw, ref = GpuWorld(scene), RefWorld(scene)
    rg, rr = gw.env_step(), ref.env_step()
    _compare_env(gw, 0, ref, rg, rr, name)
    assert rg.cfl_cycles == rr.cfl_cycles and rg.lost_particles == rr.lost_particles
    # StepReport diagnostics (coupling.hpp:261-284): penetration to fp32 position accuracy,
    # third-law balance at the reference's own bound (acceptance.cpp:176-181: 1e-10 N)
    assert abs(rg.max_penetration - rr.max_penetration) <= 1e-6 + 1e-3 * rr.max_penetration, \
        (rg.max_penetration, rr.max_penetration)
    assert rg.max_force_balance_error <= 1e-10 and rr.max_force_balance_error <= 1e-10


def test_config_d_batch_matches_reference_per_env():
    """8 envs of D stepped as one batch; each env against its own reference World."""
    scene = config_d(n_envs=8)
    gw = GpuWorld(scene)
    gw.env_step()
    for e in range(8):
        ref = RefWorld(scene, env=e)
        rr = ref.env_step()
        _compare_env(gw, e, ref, None, rr, f"D env {e}")
        rep = gw.report(e)
        assert rep.cfl_cycles == rr.cfl_cycles
        assert abs(rep.max_penetration - rr.max_penetration) <= 1e-6 + 1e-3 * rr.max_penetration, e
        assert rep.max_force_balance_error <= 1e-10


def test_full_size_config_d_sampled_envs_match_reference():
    """The benchmark's own size: all 1024 envs of D (16.8 M particles; the
    bucket key space, the multi-tile scans and the node-block list at full
    scale) stepped as one batch, sampled envs against their own reference
    Worlds."""
    scene = config_d(n_envs=1024)
    gw = GpuWorld(scene)
    gw.env_step()
    for e in (0, 1, 511, 1022, 1023):
        ref = RefWorld(scene, env=e)
        rr = ref.env_step()
        _compare_env(gw, e, ref, None, rr, f"D/1024 env {e}")
        assert gw.report(e).cfl_cycles == rr.cfl_cycles


def test_third_law_every_substep_pinch():
    """Acceptance criterion 3 on a pinch-shaped env (two fingers squeezing a block,
    acceptance.cpp:156-193): |sum of reactions + sum of applied forces| <= 1e-10 N
    in every CFL cycle of every substep (the StepReport max over all of them),
    over several env steps with growing contact."""
    scene = config_d(n_envs=2)
    gw = GpuWorld(scene)
    ref = RefWorld(scene, env=1)
    for _ in range(4):
        gw.env_step()
        rr = ref.env_step()
        rep = gw.report(1)
        assert rep.max_force_balance_error <= 1e-10, rep.max_force_balance_error
        assert rr.max_force_balance_error <= 1e-10
    fg, _ = gw.wrenches(1, pending=True)
    assert np.linalg.norm(fg) > 0  # the fingers are in contact


def _expected_binning(b, cells, bdims, kdims, dims):
    """Bucket histogram and touched blocks implied by the reference's binning."""
    base = b["base"]
    alive = base[:, 0] >= 0
    q = base[alive] // cells
    ids = (q[:, 2] * bdims[1] + q[:, 1]) * bdims[0] + q[:, 0]
    counts = np.bincount(ids, minlength=int(np.prod(bdims))).astype(np.int32)
    an = b["active_nodes"]
    i, j, k = an % dims[0], (an // dims[0]) % dims[1], an // (dims[0] * dims[1])
    blk = np.unique((k // 2 * kdims[1] + j // 4) * kdims[0] + i // 4).astype(np.int32)
    return counts, blk


@pytest.mark.parametrize("name", ["B", "D", "C"])
def test_hot_path_bucket_counts_and_touched_blocks_bit_exact(name):
    """The hot path's OWN binning outputs (msim_gpu_read_buckets: the per-bucket
    counts k_particles produced and the node-block list of its P2G flush), not a
    rebuild, against the reference's counting sort and active nodes (and the
    oracle's), after the particles have moved for one env step."""
    scene = {"B": lambda: config_b(), "C": lambda: config_c(), "D": lambda: config_d(n_envs=4)}[name]()
    gw = GpuWorld(scene)
    gw.env_step()
    envs = range(len(scene.envs))
    xs = [gw.particles(e) for e in envs]
    gw.p2g()
    for e in envs:
        hp = gw.buckets(e)
        for W in (RefWorld, OracleWorld):
            w = W(scene, env=e)
            p = xs[e]
            w.lib.oracle_write_particles(w.h, len(p["x"]), oracle_py._d(p["x"]), oracle_py._d(p["v"]), None, None)
            w.grid_clear()
            w.p2g()
            counts, blocks = _expected_binning(w.binning(), hp["bucket_cells"], hp["bucket_dims"], hp["block_dims"],
                                               scene.dims)
            assert np.array_equal(hp["counts"], counts), (name, e, W.__name__)
            assert np.array_equal(hp["blocks"], blocks), (name, e, W.__name__, len(hp["blocks"]), len(blocks))


def test_full_size_config_e_clay_only_one_env_step():
    """config E, clay-only variant, at full size (4M particles,
    256^3, 8 moving colliders incl. an SDF volume): one env step against the
    oracle (multithreaded; the reference itself would take the same path at
    1/8 the speed, its penalty loop is serial)."""
    scene = config_e(clay_only=True)
    gw = GpuWorld(scene)
    gw.env_step()
    ow = OracleWorld(scene, threads=os.cpu_count() or 1)
    ow.env_step()
    pg, po = gw.particles(0), ow.particles()
    assert _xerr(pg["x"], po["x"]) < X_TOL
    assert rel(pg["v"], po["v"]) < V_TOL
    assert np.array_equal(pg["lost"], po["lost"])
    fg, _ = gw.wrenches(0, pending=True)
    fo, _ = ow.wrenches(pending=True)
    for b in range(len(fo)):
        assert np.linalg.norm(fg[b] - fo[b]) / max(np.linalg.norm(fo[b]), 1e-6) < WRENCH_TOL, b
    # conservation of mass on the grid is exact in the counts: every particle alive
    assert gw.lost_count() == ow.lost_count()
