"""ORACLE — TEST INFRASTRUCTURE ONLY.

Checker-side ctypes mirror of the POD structs in include/msim_gpu.h (the
oracle and the reference harness share the product's descriptors so both
sides are driven with the same inputs). Kept separate from the product's
``paper_2302_04659_b200.abi`` so that importing the checkers never loads the
product library; tests/test_abi.py checks the two mirrors have identical
layouts.
"""
from __future__ import annotations

import ctypes as C

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


def convert(obj, cls):
    """Re-type a layout-identical ctypes struct (or array of structs) as `cls`."""
    return cls.from_buffer_copy(obj)
