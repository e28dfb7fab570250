"""Golden vectors from the REFERENCE itself (oracle/_ref/libmsim_ref.so: the
reference's own sources compiled unchanged against oracle/ref_shim), committed
so the oracle stays pinned where /root/reference is absent (the GPU box).

    python tests/golden/make_golden.py     # rewrites tests/golden/ref_*.npz

Each fixture: one env step (25 substeps) of a config from its seeded inputs
(paper_2302_04659_b200.scenes, clay parity variants): a particle subsample of
x, v, F, C; lost count; staged wrenches; body states; the StepReport; and the
p2g integer binning of the stepped state (sha256 of base / cell_start /
cell_particles / active_nodes, plus their sizes).
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle_py import RefWorld  # noqa: E402
from paper_2302_04659_b200.scenes import config_a, config_b, config_d  # noqa: E402

CASES = {  # name: (scene factory, env, particle stride)
    "A": (config_a, 0, 8),
    "B": (config_b, 0, 32),
    "D0": (lambda: config_d(2), 0, 16),
    "D1": (lambda: config_d(2), 1, 16),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def golden(name):
    make, env, stride = CASES[name]
    w = RefWorld(make(), env=env)
    rep = w.env_step()
    p = w.particles()
    f, t = w.wrenches(pending=True)
    bodies = np.array([list(b.q) + list(b.t) + list(b.v) + list(b.w) for b in w.bodies()]).reshape(-1, 13)
    w.grid_clear()
    w.p2g()
    b = w.binning()
    return dict(
        idx=np.arange(0, len(p["x"]), stride), x=p["x"][::stride], v=p["v"][::stride], F=p["F"][::stride],
        C=p["C"][::stride], lost=np.int64(p["lost"].sum()), force=f, torque=t, bodies=bodies,
        report=np.array([rep.rigid_steps, rep.soft_substeps, rep.cfl_cycles, rep.lost_particles]),
        report_f=np.array([rep.max_penetration, rep.max_force_balance_error]),
        bin_sha=np.array([sha(b[k]) for k in ("base", "cell_start", "cell_particles", "active_nodes")]),
        bin_len=np.array([len(b[k]) for k in ("base", "cell_start", "cell_particles", "active_nodes")]),
    )


if __name__ == "__main__":
    out = os.path.dirname(os.path.abspath(__file__))
    for name in CASES:
        np.savez_compressed(os.path.join(out, f"ref_{name}.npz"), **golden(name))
        print("wrote", f"ref_{name}.npz")
