"""The library's multi-GPU statistics exchange on one B200 (the pool has one
GPU per box): msim_gpu_step_stats reduces the last env step's report over the
context's envs on the device and all-reduces it with NCCL (a single-rank
communicator here; the multi-rank host logic is covered with gloo on CPU)."""
import numpy as np
import pytest

from paper_2302_04659_b200 import GpuWorld
from paper_2302_04659_b200.dist import LibStats
from paper_2302_04659_b200.scenes import config_d

pytestmark = pytest.mark.gpu


def test_step_stats_match_the_report_and_allreduce():
    sc = config_d(n_envs=4)
    gw = GpuWorld(sc)
    rep = gw.env_step()
    st = LibStats(gw.lib, gw.ctx, 0, 1).step()
    assert st.particle_substeps == sc.n_particles * sc.substeps_per_env_step
    assert st.env_steps == 4
    assert st.cfl_cycles == sum(gw.report(e).cfl_cycles for e in range(4)) >= 4 * 25
    assert st.lost_particles == rep.lost_particles
    assert st.max_penetration == pytest.approx(rep.max_penetration, rel=1e-7, abs=0)
    assert st.max_force_balance_error == pytest.approx(rep.max_force_balance_error, rel=0, abs=1e-18)
