"""§8(f) rows 2-3 on the device against the oracle restatement:
mesh SDF baking (sdf.hpp:277-310) bit-exact in the f32 samples, and the task
metrics (scenario.hpp:63-209) over every env's live state: fill fraction /
max speed, heightmap and write IoU bit-exact, chamfer / pinch within 1e-12
relative (summation order only)."""
import numpy as np
import pytest

from gpu_helpers import rel
from oracle import oracle_py
from paper_2302_04659_b200 import GpuWorld, bake_mesh_sdf, make_box_mesh
from paper_2302_04659_b200.scenes import V0_SOFT, Scene, block_env

pytestmark = pytest.mark.gpu


def perturbed_box(seed, half=(0.12, 0.08, 0.05)):
    """A closed but irregular mesh: the 8 box corners jittered (topology kept)."""
    rng = np.random.default_rng(seed)
    tri = make_box_mesh(half).reshape(-1, 3)
    corners = {tuple(v): v + rng.uniform(-0.02, 0.02, 3) for v in np.unique(tri, axis=0)}
    return np.array([corners[tuple(v)] for v in tri]).reshape(12, 3, 3)


def octahedron(r=0.07, c=(0.01, -0.02, 0.03)):
    v = np.array([[r, 0, 0], [-r, 0, 0], [0, r, 0], [0, -r, 0], [0, 0, r], [0, 0, -r]]) + np.asarray(c)
    faces = [(0, 2, 4), (2, 1, 4), (1, 3, 4), (3, 0, 4), (2, 0, 5), (1, 2, 5), (3, 1, 5), (0, 3, 5)]
    return np.array([[v[a], v[b], v[d]] for a, b, d in faces])


@pytest.mark.parametrize("mesh,voxel,pad", [
    ("box", 0.05, 0.15), ("box", 0.1, 0.2), ("perturbed", 0.01, 0.02), ("octa", 0.007, 0.01)])
def test_bake_mesh_sdf_bit_exact(mesh, voxel, pad):
    tri = {"box": lambda: make_box_mesh((0.5, 0.5, 0.5)), "perturbed": lambda: perturbed_box(3),
           "octa": octahedron}[mesh]()
    og, dg, sg = bake_mesh_sdf(tri, voxel, pad)
    oo, do, so = oracle_py.bake_mesh_sdf(tri, voxel, pad)
    assert np.array_equal(og, oo) and np.array_equal(dg, do)
    assert sg.dtype == np.float32 and np.array_equal(sg.view(np.uint32), so.view(np.uint32))
    assert (sg < 0).any() and (sg > 0).any()


def test_bake_errors_match_reference():
    with pytest.raises(ValueError, match="empty mesh"):
        bake_mesh_sdf(np.zeros((0, 3, 3)), 0.1, 0.1)
    with pytest.raises(ValueError, match="zero-area"):
        bake_mesh_sdf(np.array([[[0, 0, 0], [1, 0, 0], [2, 0, 0]]] * 2, float), 0.1, 0.1)


@pytest.fixture(scope="module")
def stepped():
    envs = [block_env((0.10, 0.10, 0.03), (12, 12, 8), 0, (1000.0, 1e4, 0.3, 2e3), V0_SOFT, seed=70 + e,
                      vel_seed=80 + e, vel_amp=0.05 * (e + 1)) for e in range(3)]
    envs[2].x[:5, 0] = -0.05  # a few lost particles: frozen, still counted by the metrics
    scene = Scene(name="tasks", dims=(32, 32, 32), h=0.01, dt=2e-4, envs=envs, n_rigid=3,
                  lost_fraction_threshold=1.0)
    gw = GpuWorld(scene)
    gw.env_step()
    parts = [gw.particles(e) for e in range(3)]
    return gw, parts


REGIONS = np.array([[0.0, 0.0, 0.0, 0.32, 0.32, 0.32],      # everything
                    [0.12, 0.12, 0.0, 0.16, 0.20, 0.05],    # part of the block
                    [0.10, 0.10, 0.035, 0.15, 0.15, 0.30]])


def test_metric_fill_bit_exact(stepped):
    gw, parts = stepped
    got = gw.metric_fill(REGIONS)
    for e in range(3):
        exp = oracle_py.metric_fill(parts[e]["x"], parts[e]["v"], REGIONS[e])
        assert got[e] == exp, (e, got[e], exp)
    assert 0.0 < got[1][0] < 1.0 and got[0][0] == 1.0


def test_heightmap_and_write_iou_bit_exact(stepped):
    gw, parts = stepped
    for nx, ny in ((8, 6), (31, 17)):
        maps = gw.render_heightmap(REGIONS, nx, ny)
        for e in range(3):
            exp = oracle_py.render_heightmap(parts[e]["x"], REGIONS[e], nx, ny)
            assert np.array_equal(maps[e].ravel(), exp), (nx, ny, e)
        rng = np.random.default_rng(5)
        targets = rng.uniform(0.0, 0.06, (3, ny, nx))
        iou, ok = gw.metric_write_iou(REGIONS, targets, 0.03)
        for e in range(3):
            ei, es = oracle_py.metric_write_iou(nx, ny, 0.03, maps[e].ravel(), targets[e].ravel())
            assert iou[e] == ei and ok[e] == es


def test_chamfer_and_pinch_match_oracle(stepped):
    gw, parts = stepped
    rng = np.random.default_rng(9)
    targets = [p["x"] + rng.normal(0, 0.004, p["x"].shape) for p in parts]
    initial = [p["x"][::3] + 0.01 for p in parts]
    ch = gw.chamfer(targets)
    ratio, ok = gw.metric_pinch(initial, targets)
    for e in range(3):
        exp = oracle_py.chamfer(parts[e]["x"], targets[e])
        assert abs(ch[e] - exp) <= 1e-12 * exp, (e, ch[e], exp)
        er, es = oracle_py.metric_pinch(parts[e]["x"], initial[e], targets[e])
        assert abs(ratio[e] - er) <= 1e-12 * er and ok[e] == es


def test_metric_errors_match_reference(stepped):
    gw, _ = stepped
    bad = REGIONS.copy()
    bad[1, 3] = bad[1, 0]
    with pytest.raises(ValueError, match="extents must be positive"):
        gw.metric_fill(bad)
    with pytest.raises(ValueError, match=">= 2x2"):
        gw.render_heightmap(REGIONS, 1, 4)
    with pytest.raises(ValueError, match="non-empty"):
        gw.chamfer([np.zeros((0, 3))] * 3)


def test_seed_envs_matches_host_seeder_and_steps_like_oracle():
    """§8f #4: batched reset by on-device seeding (mt19937_64 + the reference's
    jittered lattice): positions equal the host seeder's rounded to fp32, the
    rest of the state is fresh, untouched envs keep theirs, and the reset world
    then steps like the oracle fed the same state."""
    from oracle.oracle_py import OracleWorld
    from paper_2302_04659_b200.scenes import EnvSpec, Rng, lattice_span, seed_box

    counts = (10, 9, 6)
    los = [(0.10, 0.10, 0.03), (0.12, 0.08, 0.05), (0.02, 0.10, 0.03)]
    envs = [block_env(los[e], counts, 0, (1000.0, 1e4, 0.3, 2e3), V0_SOFT, seed=40 + e, vel_seed=50 + e)
            for e in range(3)]
    envs[2].x[:4, 0] = -0.05  # lost before the reset
    scene = Scene(name="reset", dims=(32, 32, 32), h=0.01, dt=2e-4, envs=envs, n_rigid=3,
                  lost_fraction_threshold=1.0)
    gw = GpuWorld(scene)
    gw.env_step()
    assert gw.lost_count(2) > 0
    before1 = gw.particles(1)
    new_lo = [(0.11, 0.12, 0.04), None, (0.15, 0.09, 0.06)]
    boxes = [list(new_lo[e]) + [new_lo[e][a] + lattice_span(counts[a], V0_SOFT) for a in range(3)] for e in (0, 2)]
    seeds = [9001, 123456789012345]
    gw.seed_envs([0, 2], seeds, boxes)
    assert gw.lost_count(2) == 0
    for r, e in enumerate((0, 2)):
        x_host, m_host = seed_box(Rng(seeds[r]), boxes[r][:3], boxes[r][3:], 1000.0, V0_SOFT)
        p = gw.particles(e)
        assert np.array_equal(p["x"], x_host.astype(np.float32).astype(np.float64)), e
        assert not p["v"].any() and not p["C"].any() and not p["lost"].any()
        assert np.array_equal(p["F"], np.broadcast_to(np.eye(3), p["F"].shape))
    after1 = gw.particles(1)
    for k in ("x", "v", "F", "C"):
        assert np.array_equal(before1[k], after1[k])
    # the reset env steps like the oracle started from the same (fp32-rounded) state
    p0 = gw.particles(0)
    env0 = EnvSpec(x=p0["x"], mass=np.full(len(p0["x"]), np.float32(1000.0 * V0_SOFT), np.float64),
                   vol0=np.full(len(p0["x"]), np.float32(V0_SOFT), np.float64),
                   material=np.zeros(len(p0["x"]), np.int32))
    ow = OracleWorld(Scene(name="reset0", dims=(32, 32, 32), h=0.01, dt=2e-4, envs=[env0], n_rigid=3,
                           lost_fraction_threshold=1.0))
    gw.env_step()
    ow.env_step()
    pg, po = gw.particles(0), ow.particles()
    assert np.linalg.norm(pg["x"] - po["x"]) / np.linalg.norm(po["x"]) < 1e-4
    assert rel(pg["v"], po["v"]) < 1e-4
