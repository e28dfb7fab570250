"""ctypes mirror of include/msim_gpu.h and the loader for libmsim_gpu.so.

The shared library is built in-tree (``make -C paper_2302_04659_b200``, or
``__graft_entry__.build()``). There is no fallback: if the library is missing
or fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmsim_gpu.so")

MSIM_OK = 0
MSIM_ERR_INVALID = 2
MSIM_ERR_DIVERGED = 3
MSIM_ERR_DEVICE = 4

BOUNDARY_STICKY = 0
BOUNDARY_SLIP = 1
COUPLING_PARTICLE = 0
COUPLING_GRID = 1
SHAPE_PLANE, SHAPE_SPHERE, SHAPE_BOX, SHAPE_CAPSULE, SHAPE_VOLUME = range(5)
BODY_DYNAMIC, BODY_KINEMATIC, BODY_SCRIPTED = range(3)
# material models (MSIM_MODEL_*)
MODEL_HENCKY_VON_MISES, MODEL_FIXED_COROTATED, MODEL_DRUCKER_PRAGER, MODEL_FLUID = range(4)


class SoftDesc(C.Structure):
    _fields_ = [
        ("h", C.c_double),
        ("dims", C.c_int32 * 3),
        ("origin", C.c_double * 3),
        ("boundary", C.c_uint8 * 6),
        ("_pad", C.c_uint8 * 2),
        ("gravity", C.c_double * 3),
        ("dt", C.c_double),
        ("cfl_factor", C.c_double),
        ("max_cfl_halvings", C.c_int32),
        ("_pad2", C.c_int32),
        ("lost_fraction_threshold", C.c_double),
    ]


class Material(C.Structure):
    _fields_ = [
        ("density", C.c_double),
        ("youngs", C.c_double),
        ("poisson", C.c_double),
        ("yield_stress", C.c_double),
        ("model", C.c_int32),
        ("_pad", C.c_int32),
    ]


class Shape(C.Structure):
    _fields_ = [
        ("type", C.c_int32),
        ("body", C.c_int32),
        ("local_q", C.c_double * 4),
        ("local_t", C.c_double * 3),
        ("friction", C.c_double),
        ("k_n", C.c_double),
        ("k_t", C.c_double),
        ("params", C.c_double * 4),
        ("vol_dims", C.c_int32 * 3),
        ("_pad", C.c_int32),
        ("vol_origin", C.c_double * 3),
        ("vol_voxel", C.c_double),
        ("vol_samples", C.POINTER(C.c_float)),
    ]


class Body(C.Structure):
    _fields_ = [
        ("mode", C.c_int32),
        ("_pad", C.c_int32),
        ("q", C.c_double * 4),
        ("t", C.c_double * 3),
        ("v", C.c_double * 3),
        ("w", C.c_double * 3),
        ("mass", C.c_double),
        ("inertia", C.c_double * 3),
        ("com_offset", C.c_double * 3),
    ]


class Coupling(C.Structure):
    _fields_ = [
        ("mode", C.c_int32),
        ("_pad", C.c_int32),
        ("r_c_factor", C.c_double),
        ("c_d", C.c_double),
    ]


class StepReport(C.Structure):
    _fields_ = [
        ("rigid_steps", C.c_int32),
        ("soft_substeps", C.c_int32),
        ("cfl_cycles", C.c_int32),
        ("_pad", C.c_int32),
        ("max_penetration", C.c_double),
        ("max_force_balance_error", C.c_double),
        ("lost_particles", C.c_int64),
    ]


class Region(C.Structure):  # msim_region = RegionBox (scenario.hpp:18-30)
    _fields_ = [("min", C.c_double * 3), ("max", C.c_double * 3)]


class FillResult(C.Structure):  # msim_fill_result = FillResult (scenario.hpp:55-59)
    _fields_ = [("fraction", C.c_double), ("max_speed", C.c_double), ("success", C.c_int32), ("_pad", C.c_int32)]


# Every symbol include/msim_gpu.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "msim_gpu_create", "msim_gpu_destroy", "msim_gpu_last_error", "msim_gpu_create_error",
    "msim_gpu_version", "msim_gpu_set_particles", "msim_gpu_write_particles",
    "msim_gpu_set_bodies", "msim_gpu_set_kinematic_schedule", "msim_gpu_set_deterministic", "msim_gpu_set_coupling", "msim_gpu_sync_bodies", "msim_gpu_set_dt",
    "msim_gpu_set_rigid_gravity", "msim_gpu_set_gravity", "msim_gpu_set_lost_fraction_threshold",
    "msim_gpu_soft_substep", "msim_gpu_p2g", "msim_gpu_grid_update", "msim_gpu_g2p",
    "msim_gpu_env_step", "msim_gpu_particle_count", "msim_gpu_read_particles",
    "msim_gpu_read_grid", "msim_gpu_write_grid_velocity", "msim_gpu_set_split_channels",
    "msim_gpu_set_record_binning", "msim_gpu_read_binning", "msim_gpu_read_buckets", "msim_gpu_read_wrenches",
    "msim_gpu_read_bodies", "msim_gpu_read_report", "msim_gpu_lost_count",
    "msim_gpu_constitutive", "msim_rng_create", "msim_rng_destroy", "msim_rng_uniform",
    "msim_rng_fill_uniform", "msim_gpu_body_count", "msim_gpu_sync_all_bodies",
    "msim_gpu_read_all_wrenches", "msim_gpu_nccl_unique_id", "msim_gpu_comm_init", "msim_gpu_step_stats", "msim_gpu_stream", "msim_gpu_launches", "msim_gpu_set_kernel_timing",
    "msim_gpu_kernel_count", "msim_gpu_kernel_stats",
    "msim_seed_box_count", "msim_seed_box",
    "msim_gpu_metric_fill", "msim_gpu_render_heightmap", "msim_gpu_metric_write_iou", "msim_gpu_chamfer",
    "msim_gpu_metric_pinch", "msim_bake_grid", "msim_gpu_bake_mesh_sdf", "msim_make_box_mesh",
    "msim_gpu_seed_envs", "msim_gpu_set_bucket_factor", "msim_gpu_read_jp",
]

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)
_vp = C.c_void_p

_SIGS = {
    "msim_gpu_create": (C.c_int, [C.POINTER(SoftDesc), C.POINTER(Material), C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]),
    "msim_gpu_destroy": (None, [_vp]),
    "msim_gpu_last_error": (C.c_char_p, [_vp]),
    "msim_gpu_create_error": (C.c_char_p, []),
    "msim_gpu_version": (C.c_int, []),
    "msim_gpu_set_particles": (C.c_int, [_vp, C.c_int64, _lp, _dp, _dp, _dp, _dp, _dp, _dp, _ip]),
    "msim_gpu_write_particles": (C.c_int, [_vp, C.c_int, C.c_int64, _dp, _dp, _dp, _dp]),
    "msim_gpu_set_bodies": (C.c_int, [_vp, C.c_int, C.POINTER(Body), C.c_int, C.POINTER(Shape), C.c_int]),
    "msim_gpu_set_coupling": (C.c_int, [_vp, C.POINTER(Coupling)]),
    "msim_gpu_sync_bodies": (C.c_int, [_vp, C.c_int, C.POINTER(Body), C.c_int]),
    "msim_gpu_set_dt": (C.c_int, [_vp, C.c_double]),
    "msim_gpu_set_rigid_gravity": (C.c_int, [_vp, _dp]),
    "msim_gpu_set_gravity": (C.c_int, [_vp, _dp]),
    "msim_gpu_set_lost_fraction_threshold": (C.c_int, [_vp, C.c_double]),
    "msim_gpu_soft_substep": (C.c_int, [_vp, C.c_int, _ip]),
    "msim_gpu_p2g": (C.c_int, [_vp]),
    "msim_gpu_grid_update": (C.c_int, [_vp]),
    "msim_gpu_g2p": (C.c_int, [_vp]),
    "msim_gpu_env_step": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(StepReport)]),
    "msim_gpu_particle_count": (C.c_int64, [_vp, C.c_int]),
    "msim_gpu_read_particles": (C.c_int, [_vp, C.c_int, _dp, _dp, _dp, _dp, _u8p]),
    "msim_gpu_read_grid": (C.c_int, [_vp, C.c_int, _dp, _dp, _dp, _dp]),
    "msim_gpu_write_grid_velocity": (C.c_int, [_vp, C.c_int, _dp]),
    "msim_gpu_set_split_channels": (C.c_int, [_vp, C.c_int]),
    "msim_gpu_set_record_binning": (C.c_int, [_vp, C.c_int]),
    "msim_gpu_read_binning": (C.c_int, [_vp, C.c_int, _ip, _ip, C.c_int64, _ip, C.c_int64, _lp, _lp, C.c_int64, _lp]),
    "msim_gpu_read_buckets": (C.c_int, [_vp, C.c_int, _ip, _ip, _ip, C.c_int64, _ip, _ip, C.c_int64, _lp]),
    "msim_gpu_set_kinematic_schedule": (C.c_int, [_vp, C.c_int, _dp, _u8p]),
    "msim_gpu_nccl_unique_id": (C.c_int, [_u8p]),
    "msim_gpu_set_deterministic": (C.c_int, [_vp, C.c_int]),
    "msim_gpu_comm_init": (C.c_int, [_vp, C.c_int, C.c_int, _u8p]),
    "msim_gpu_step_stats": (C.c_int, [_vp, C.c_int, _dp, _dp]),
    "msim_gpu_read_wrenches": (C.c_int, [_vp, C.c_int, C.c_int, _dp, _dp]),
    "msim_gpu_read_bodies": (C.c_int, [_vp, C.c_int, C.POINTER(Body), C.c_int]),
    "msim_gpu_read_report": (C.c_int, [_vp, C.c_int, C.POINTER(StepReport)]),
    "msim_gpu_lost_count": (C.c_int64, [_vp, C.c_int]),
    "msim_gpu_constitutive": (C.c_int, [_vp, C.c_int, C.c_int64, _dp, _dp, _dp]),
    "msim_rng_create": (_vp, [C.c_uint64]),
    "msim_rng_destroy": (None, [_vp]),
    "msim_rng_uniform": (C.c_double, [_vp, C.c_double, C.c_double]),
    "msim_rng_fill_uniform": (None, [_vp, C.c_int64, C.c_double, C.c_double, _dp]),
    "msim_seed_box_count": (C.c_int64, [_dp, _dp, C.c_double]),
    "msim_gpu_body_count": (C.c_int, [_vp, C.c_int]),
    "msim_gpu_sync_all_bodies": (C.c_int, [_vp, C.POINTER(Body), C.c_int]),
    "msim_gpu_read_all_wrenches": (C.c_int, [_vp, C.c_int, _dp]),
    "msim_gpu_stream": (_vp, [_vp]),
    "msim_gpu_launches": (C.c_int64, [_vp]),
    "msim_gpu_set_kernel_timing": (C.c_int, [_vp, C.c_int]),
    "msim_gpu_kernel_count": (C.c_int, []),
    "msim_gpu_kernel_stats": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_char_p), _lp, _dp]),
    "msim_seed_box": (C.c_int64, [_vp, _dp, _dp, C.c_double, C.c_double, _dp, _dp]),
    "msim_gpu_metric_fill": (C.c_int, [_vp, C.POINTER(Region), C.POINTER(FillResult)]),
    "msim_gpu_render_heightmap": (C.c_int, [_vp, C.POINTER(Region), C.c_int, C.c_int, _dp]),
    "msim_gpu_metric_write_iou": (C.c_int, [_vp, C.POINTER(Region), C.c_int, C.c_int, C.c_double, _dp, _dp, _ip]),
    "msim_gpu_chamfer": (C.c_int, [_vp, _dp, _lp, _dp]),
    "msim_gpu_metric_pinch": (C.c_int, [_vp, _dp, _lp, _dp, _lp, _dp, _ip]),
    "msim_bake_grid": (C.c_int, [_dp, C.c_int64, C.c_double, C.c_double, _dp, _ip]),
    "msim_gpu_bake_mesh_sdf": (C.c_int, [C.c_int, _dp, C.c_int64, C.c_double, C.c_double, C.POINTER(C.c_float), C.c_int64]),
    "msim_make_box_mesh": (None, [_dp, _dp, _dp]),
    "msim_gpu_set_bucket_factor": (C.c_int, [_vp, C.c_int]),
    "msim_gpu_read_jp": (C.c_int, [_vp, C.c_int, _dp]),
    "msim_gpu_seed_envs": (C.c_int, [_vp, C.c_int, _ip, C.POINTER(C.c_uint64), _dp, C.c_int32, C.c_double]),
}

_lib = None


def load(path: str | None = None) -> C.CDLL:
    """Load libmsim_gpu.so (raises if it is missing: there is no fallback).
    MSIM_GPU_LIB overrides the path (profiling builds of the same sources)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("MSIM_GPU_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: build the CUDA library first (python -c 'import __graft_entry__ as g; g.build()')"
        )
    lib = C.CDLL(path)
    override = "MSIM_GPU_LIB" in os.environ  # an older profiling build may lack newer entry points
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name, None) if override else getattr(lib, name)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_ip)


def lptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_lp)


def u8ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(_u8p)
