"""B200-native MLS-MPM soft-body substep (the hot path of arXiv 2302.04659's
soft-body simulator), behind the C ABI in include/msim_gpu.h.

Importing the package loads libmsim_gpu.so and fails loudly if it is absent:
there is no CPU fallback.
"""
from . import abi

abi.load()

from .scenes import CONFIGS, Scene  # noqa: E402
from .world import DeviceError, GpuWorld, SimulationDiverged, bake_mesh_sdf, make_box_mesh  # noqa: E402
from .scene_json import SceneConfigError, scene_from_json  # noqa: E402

__all__ = ["abi", "CONFIGS", "Scene", "GpuWorld", "SimulationDiverged", "DeviceError", "bake_mesh_sdf", "make_box_mesh",
           "scene_from_json", "SceneConfigError"]
