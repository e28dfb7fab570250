"""env-steps/s of the small single-scene configs A (clay), B (sand), C (water) (launch/latency bound,
SURVEY.md §8d: reported in absolute terms, not as a roofline fraction)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2302_04659_b200 import GpuWorld  # noqa: E402
from paper_2302_04659_b200.scenes import SAND, WATER, config_a, config_b, config_c  # noqa: E402

out = {}
# BASELINE.json configs: A elastoplastic clay + box; B Drucker-Prager sand + bucket; C fluid + bottle/beaker
for name, fn in (("A", config_a), ("B", lambda: config_b(material=SAND)), ("C", lambda: config_c(material=WATER))):
    scene = fn()
    gw = GpuWorld(scene)
    for _ in range(3):
        gw.env_step()
    steps = 20
    t0 = time.perf_counter()
    for _ in range(steps):
        gw.env_step()
    dt = time.perf_counter() - t0
    n = scene.n_particles
    out[name] = {"particles": n, "env_steps_per_s": steps / dt, "ms_per_env_step": 1e3 * dt / steps,
                 "particle_substeps_per_s": n * scene.substeps_per_env_step * steps / dt,
                 "launches_per_env_step": None}
print(json.dumps(out))
