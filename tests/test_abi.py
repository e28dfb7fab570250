"""The C-ABI library loads and exports every symbol include/msim_gpu.h
declares (no device work: runs on CPU)."""
import ctypes as C
import os
import re

import numpy as np

from paper_2302_04659_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "msim_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(msim_(?:gpu|rng|seed|bake|make)_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = abi.load()
    names = header_symbols()
    assert len(names) >= 35
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(abi.EXPORTED) == names


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors have the size and field offsets the C compiler gives the header structs."""
    import subprocess

    structs = {"msim_soft_desc": abi.SoftDesc, "msim_material": abi.Material, "msim_shape": abi.Shape,
               "msim_body": abi.Body, "msim_coupling": abi.Coupling, "msim_step_report": abi.StepReport,
               "msim_region": abi.Region, "msim_fill_result": abi.FillResult}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "msim_gpu.h"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n") if l)
    for cname, py in structs.items():
        assert int(out[cname]) == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(out[f"{cname}.{f}"]) == getattr(py, f).offset, (cname, f)


def test_create_validates_like_reference_without_device():
    """Invalid material / grid are rejected before any device call
    (Material::validate mpm.hpp:35-41, MpmGrid::validate :103-106)."""
    from paper_2302_04659_b200.scenes import Scene

    lib = abi.load()
    sc = Scene(name="bad", dims=(3, 32, 32))
    ctx = C.c_void_p()
    assert lib.msim_gpu_create(C.byref(sc.desc()), sc.material_array(), 1, 1, 0, C.byref(ctx)) == abi.MSIM_ERR_INVALID
    assert b"dims" in lib.msim_gpu_create_error()
    sc = Scene(name="bad", dims=(32, 32, 32), materials=[(1000.0, 1e4, 0.5, 2e3)])
    assert lib.msim_gpu_create(C.byref(sc.desc()), sc.material_array(), 1, 1, 0, C.byref(ctx)) == abi.MSIM_ERR_INVALID
    assert b"nu" in lib.msim_gpu_create_error()


def test_seed_box_counts_match_reference_golden_scenes():
    """lattice_count (seeding.hpp:38-46) for the golden scenes."""
    lib = abi.load()
    V0 = 6.2e-8

    def count(lo, hi, v=V0):
        lo = np.array(lo, dtype=np.float64)
        hi = np.array(hi, dtype=np.float64)
        return lib.msim_seed_box_count(abi.dptr(lo), abi.dptr(hi), v)

    assert count((0.105, 0.105, 0.082), (0.155, 0.155, 0.110)) == 1008   # fill-mini
    assert count((0.10, 0.10, 0.016), (0.18, 0.16, 0.036)) == 1500       # write-mini
    assert count((0.10, 0.10, 0.06), (0.14, 0.14, 0.09)) == 700          # test_coupling block


def _oracle_box(half, center=(0.0, 0.0, 0.0)):
    from oracle import oracle_py

    lib = oracle_py.load()
    tri = np.zeros(108)
    lib.oracle_make_box_mesh(np.asarray(half, float).ctypes.data_as(C.POINTER(C.c_double)),
                             np.asarray(center, float).ctypes.data_as(C.POINTER(C.c_double)),
                             tri.ctypes.data_as(C.POINTER(C.c_double)))
    return tri


def test_bake_grid_and_box_mesh_match_reference_host_side():
    """msim_bake_grid / msim_make_box_mesh (host code of the bake API) against the
    oracle's restatement of sdf.hpp:277-296 / :443-455, and the reference's errors."""
    from oracle import oracle_py

    lib, olib = abi.load(), oracle_py.load()
    dp = C.POINTER(C.c_double)
    half, center = np.array([0.3, 0.2, 0.1]), np.array([0.05, -0.02, 0.4])
    tri = np.zeros(108)
    lib.msim_make_box_mesh(half.ctypes.data_as(dp), center.ctypes.data_as(dp), tri.ctypes.data_as(dp))
    assert np.array_equal(tri, _oracle_box(half, center))
    for voxel, pad in ((0.05, 0.15), (0.013, 0.0), (0.1, 0.2)):
        o1, o2 = np.zeros(3), np.zeros(3)
        d1, d2 = np.zeros(3, np.int32), np.zeros(3, np.int32)
        assert lib.msim_bake_grid(tri.ctypes.data_as(dp), 12, voxel, pad, o1.ctypes.data_as(dp),
                                  d1.ctypes.data_as(C.POINTER(C.c_int32))) == 0
        assert olib.oracle_bake_grid(tri.ctypes.data_as(dp), C.c_int64(12), C.c_double(voxel), C.c_double(pad),
                                     o2.ctypes.data_as(dp), d2.ctypes.data_as(C.POINTER(C.c_int32))) == 0
        assert np.array_equal(o1, o2) and np.array_equal(d1, d2)
    o, d = np.zeros(3), np.zeros(3, np.int32)
    ip = C.POINTER(C.c_int32)
    assert lib.msim_bake_grid(tri.ctypes.data_as(dp), 0, 0.1, 0.1, o.ctypes.data_as(dp), d.ctypes.data_as(ip)) == 2
    assert b"empty mesh" in lib.msim_gpu_create_error()
    assert lib.msim_bake_grid(tri.ctypes.data_as(dp), 12, 0.0, 0.1, o.ctypes.data_as(dp), d.ctypes.data_as(ip)) == 2
    assert b"voxel" in lib.msim_gpu_create_error()
    degen = np.array([0, 0, 0, 1, 0, 0, 2, 0, 0] * 2, float)
    assert lib.msim_bake_grid(degen.ctypes.data_as(dp), 2, 0.1, 0.1, o.ctypes.data_as(dp), d.ctypes.data_as(ip)) == 2
    assert b"zero-area" in lib.msim_gpu_create_error()
