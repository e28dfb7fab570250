"""Parity margins report (not a test): errors of the CUDA path vs the oracle
for configs A-D after k env steps. Usage: python tests/parity_report.py [steps]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from oracle.oracle_py import OracleWorld  # noqa: E402
from paper_2302_04659_b200 import GpuWorld  # noqa: E402
from paper_2302_04659_b200.scenes import config_a, config_b, config_c, config_d  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
for name, mk in (("A", config_a), ("B", config_b), ("C", config_c), ("D", lambda: config_d(4))):
    sc = mk()
    gw = GpuWorld(sc)
    ows = [OracleWorld(sc, env=e) for e in range(len(sc.envs))]
    for k in range(steps):
        t0 = time.time()
        gw.env_step()
        for o in ows:
            o.env_step()
        for e, o in enumerate(ows):
            pg, po = gw.particles(e), o.particles()
            ex = np.linalg.norm(pg["x"] - po["x"]) / np.linalg.norm(po["x"])
            ev = np.linalg.norm(pg["v"] - po["v"]) / np.linalg.norm(po["v"])
            evmax = np.max(np.linalg.norm(pg["v"] - po["v"], axis=1))
            eF = np.linalg.norm(pg["F"] - po["F"]) / np.linalg.norm(po["F"] - np.eye(3))
            fg, _ = gw.wrenches(e, pending=True)
            fo, _ = o.wrenches(pending=True)
            ew = [float(np.linalg.norm(fg[b] - fo[b]) / max(np.linalg.norm(fo[b]), 1e-6)) for b in range(len(fo))]
            print(f"{name} env{e} step{k+1}: x {ex:.2e} v {ev:.2e} (max abs {evmax:.2e}) F-I {eF:.2e} "
                  f"wrench {['%.1e' % w for w in ew]} |f| {[float('%.3g' % np.linalg.norm(f)) for f in fo]} "
                  f"lost {int(pg['lost'].sum())}/{int(po['lost'].sum())}", flush=True)
