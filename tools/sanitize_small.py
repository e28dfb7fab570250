"""A tiny workload for compute-sanitizer (memcheck / racecheck / synccheck):
config A shrunk to 2 rigid steps, all kernels of the step + readbacks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_04659_b200 import GpuWorld  # noqa: E402
from paper_2302_04659_b200.scenes import config_a  # noqa: E402

scene = config_a()
scene.n_rigid = 2
gw = GpuWorld(scene)
gw.env_step()
gw.env_step()
p = gw.particles(0)
print("ok", p["x"].shape)
