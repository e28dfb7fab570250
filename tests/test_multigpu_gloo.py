"""The multi-rank path on CPU (gloo, world_size 2): env sharding and the
per-env-step stats all-reduce, with real step reports from the CPU oracle
stepping each rank's envs (the CUDA path is the same host logic with NCCL)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2302_04659_b200.dist import StepStats, allreduce_stats, shard, weak_first_env


def test_shard_covers_batch_exactly():
    for n, w in ((1024, 1), (1024, 2), (1024, 8), (10, 3), (3, 8)):
        ranges = [shard(n, r, w) for r in range(w)]
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        assert max(hi - lo for lo, hi in ranges) - min(hi - lo for lo, hi in ranges) <= 1
    assert [weak_first_env(1024, r) for r in range(3)] == [0, 1024, 2048]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch.distributed as dist

    from oracle.oracle_py import OracleWorld
    from paper_2302_04659_b200.dist import rank_envs
    from paper_2302_04659_b200.scenes import config_d

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_total = 4
    # the rank's shard exactly as bench.py builds it: config_d(n, first_env) of rank_envs
    first, n = rank_envs(n_total, rank, world)
    scene = config_d(n_envs=n, first_env=first)
    scene.n_rigid = 2  # short step: the sharding and the reduction, not the physics, are under test
    reports, counts, hashes = [], [], {}
    for e in range(n):
        w = OracleWorld(scene, env=e)
        reports.append(w.env_step())
        counts.append(scene.envs[e].n)
        hashes[first + e] = int(w.lib.oracle_state_hash(w.h))
    local = StepStats.from_reports(reports, counts, scene.n_rigid * scene.n_soft)
    total = allreduce_stats(local)
    q.put((rank, local, total, hashes))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_stats_allreduce_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=280) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda t: t[0])
    (_, l0, t0, h0), (_, l1, t1, h1) = out
    assert t0 == t1
    # per-env results of the sharded run == a single-rank run of the whole batch
    from oracle.oracle_py import OracleWorld
    from paper_2302_04659_b200.scenes import config_d

    whole = config_d(n_envs=4)
    whole.n_rigid = 2
    single = {}
    for e in range(4):
        w = OracleWorld(whole, env=e)
        w.env_step()
        single[e] = int(w.lib.oracle_state_hash(w.h))
    assert sorted({**h0, **h1}) == [0, 1, 2, 3] and {**h0, **h1} == single
    assert t0.env_steps == 4 and t0.particle_substeps == l0.particle_substeps + l1.particle_substeps
    assert t0.cfl_cycles == l0.cfl_cycles + l1.cfl_cycles == 4 * 2
    assert t0.max_penetration == max(l0.max_penetration, l1.max_penetration)
