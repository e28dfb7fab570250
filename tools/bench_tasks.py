"""Time the §8(f) consumers on the device (config D state: 1024 envs x 16,384
particles) against the CPU oracle on a bounded sample, one JSON line.

  python tools/bench_tasks.py [--envs N] [--out profiles/r01_tasks.json]

Device times are CUDA-synchronous wall times of the C-ABI calls (each call
includes its host<->device copies of inputs and results), median of 5 after
one warm-up. The oracle (test infrastructure, 1 thread) is timed on 1-2 envs
and reported per env."""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle_py  # noqa: E402
from paper_2302_04659_b200 import GpuWorld, bake_mesh_sdf, make_box_mesh  # noqa: E402
from paper_2302_04659_b200.scenes import V0_SOFT, config_d, lattice_span  # noqa: E402


def timed(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=1024)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    scene = config_d(a.envs)
    gw = GpuWorld(scene)
    gw.env_step()
    n_env = gw.n_env
    res = {"workload": f"config D state, {n_env} envs x 16384 particles, after one env step", "device": {}, "cpu_oracle_per_env": {}}
    regions = np.tile([0.0, 0.0, 0.0, 0.32, 0.32, 0.08], (n_env, 1))
    res["device"]["metric_fill_s"] = timed(lambda: gw.metric_fill(regions))
    res["device"]["render_heightmap_64x64_s"] = timed(lambda: gw.render_heightmap(regions, 64, 64))
    targets = np.full((n_env, 64, 64), 0.05)
    res["device"]["metric_write_iou_64x64_s"] = timed(lambda: gw.metric_write_iou(regions, targets, 0.04))
    p0 = gw.particles(0)
    tgt = [p0["x"] + 0.003] * n_env
    res["device"]["chamfer_s"] = timed(lambda: gw.chamfer(tgt), reps=2)
    env0 = scene.envs[0]
    lo = env0.x.min(axis=0) - 0.25 * V0_SOFT ** (1 / 3)
    box = list(lo) + [lo[k] + lattice_span(c, V0_SOFT) for k, c in enumerate((32, 32, 16))]
    res["device"]["seed_envs_all_s"] = timed(lambda: gw.seed_envs(np.arange(n_env), 1000 + np.arange(n_env),
                                                                  np.tile(box, (n_env, 1))), reps=3)
    tri = make_box_mesh((0.05, 0.03, 0.02))
    res["device"]["bake_box_2mm_s"] = timed(lambda: bake_mesh_sdf(tri, 0.002, 0.01), reps=3)
    # oracle (1 thread) per env
    x, v = p0["x"], p0["v"]
    res["cpu_oracle_per_env"]["metric_fill_s"] = timed(lambda: oracle_py.metric_fill(x, v, regions[0]), reps=3)
    res["cpu_oracle_per_env"]["render_heightmap_64x64_s"] = timed(lambda: oracle_py.render_heightmap(x, regions[0], 64, 64), reps=3)
    res["cpu_oracle_per_env"]["chamfer_s"] = timed(lambda: oracle_py.chamfer(x, tgt[0]), reps=1)
    res["cpu_oracle_box_bake_2mm_s"] = timed(lambda: oracle_py.bake_mesh_sdf(tri, 0.002, 0.01), reps=1)
    for k in ("metric_fill_s", "render_heightmap_64x64_s", "chamfer_s"):
        res.setdefault("speedup_vs_oracle_all_envs", {})[k] = res["cpu_oracle_per_env"][k] * n_env / res["device"][k]
    res["speedup_vs_oracle_bake"] = res["cpu_oracle_box_bake_2mm_s"] / res["device"]["bake_box_2mm_s"]
    line = json.dumps(res)
    print(line)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
