"""Scene JSON loading (shell.hpp:144-320 semantics) for the batched device
world: fields, seeding identical to the reference's single mt19937_64 stream,
and the reference's error paths / warnings. CPU only (no device work)."""
import ctypes as C
import json

import numpy as np
import pytest

from paper_2302_04659_b200 import abi
from paper_2302_04659_b200.scene_json import SceneConfigError, scene_from_json

SCENE = {
    "gravity": [0.0, 0.0, -9.81],
    "grid": {"length": 0.01, "dims": [48, 48, 32], "origin": [0, 0, 0],
             "boundary": ["sticky", "sticky", "slip", "slip", "sticky", "sticky"]},
    "materials": ["soft_clay", {"density": 1000, "youngs_modulus": 1e5, "poisson_ratio": 0.3, "yield_stress": 4e3}],
    "sources": [{"box_min": [0.10, 0.10, 0.02], "box_max": [0.16, 0.14, 0.05], "material": 0},
                {"box_min": [0.20, 0.10, 0.02], "box_max": [0.24, 0.15, 0.06], "material": 1,
                 "particle_volume": 1.2e-7}],
    "bodies": [{"name": "floor", "mode": "kinematic", "pose": {"translation": [0, 0, 0.02]},
                "shapes": [{"type": "plane", "normal": [0, 0, 2], "offset": 0.0}]},
               {"name": "stamp", "mode": "dynamic", "mass": 0.05, "inertia": [1e-5, 1e-5, 1e-5],
                "pose": {"translation": [0.13, 0.12, 0.09], "rotation_wxyz": [1, 0, 0, 0]},
                "shapes": [{"type": "box", "half_extents": [0.02, 0.02, 0.01], "friction": 0.3},
                           {"type": "capsule", "half_length": 0.01, "radius": 0.005,
                            "pose": {"translation": [0, 0, 0.02]}, "k_n": 50}]}],
    "coupling": {"mode": "particle", "k_n": 20.0, "k_t": 0.1, "c_d": 0.05, "r_c_factor": 0.5},
    "stepping": {"dt_soft": 4e-4, "n_soft": 1, "n_rigid": 25, "control_hz": 100.0},
    "seed": 7,
}


def test_fields_and_defaults():
    warnings = []
    sc = scene_from_json(json.loads(json.dumps(SCENE)), warnings, n_envs=3)
    assert sc.h == 0.01 and sc.dims == (48, 48, 32) and sc.boundary == (0, 0, 1, 1, 0, 0)
    assert sc.materials[0] == (1000.0, 1e4, 0.3, 2e3) and sc.materials[1][1] == 1e5
    assert sc.dt == 4e-4 and sc.n_rigid == 25 and sc.c_d == 0.05
    assert len(sc.envs) == 3 and all(e.n == sc.envs[0].n for e in sc.envs)
    env = sc.envs[0]
    assert [b.mode for b in env.bodies] == [abi.BODY_KINEMATIC, abi.BODY_DYNAMIC]
    plane, box, cap = env.shapes
    assert plane.type == abi.SHAPE_PLANE and plane.params == (0.0, 0.0, 1.0, 0.0)  # normal normalized
    assert plane.k_n == 20.0 and plane.k_t == 0.1 and plane.friction == 0.5  # coupling defaults
    assert box.body == 1 and box.friction == 0.3 and cap.k_n == 50.0 and cap.local_t == (0.0, 0.0, 0.02)
    assert warnings == []  # inside the validated envelope (shell.hpp:120-137)


def test_seeding_is_the_reference_stream():
    """Both sources draw from ONE mt19937_64(seed) in order (shell.hpp:192-203):
    positions equal the oracle's seeding of the same boxes with one rng."""
    from oracle import oracle_py
    from paper_2302_04659_b200.scenes import Scene

    sc = scene_from_json(SCENE)
    lib = oracle_py.load()
    ref = Scene(name="s", dims=(48, 48, 32), materials=sc.materials)
    w = lib.oracle_create(C.byref(ref.desc()), ref.material_array(), len(ref.materials))
    r = lib.oracle_rng_create(7)
    dp = C.POINTER(C.c_double)
    for s in SCENE["sources"]:
        lo, hi = np.array(s["box_min"], float), np.array(s["box_max"], float)
        lib.oracle_seed_box(w, r, lo.ctypes.data_as(dp), hi.ctypes.data_as(dp), s["material"],
                            s.get("particle_volume", 6.2e-8))
    n = sc.envs[0].n
    x = np.zeros((n, 3))
    lib.oracle_read_particles(w, x.ctypes.data_as(dp), None, None, None, None)
    lib.oracle_rng_destroy(r)
    lib.oracle_destroy(w)
    assert np.array_equal(x, sc.envs[0].x)
    assert np.array_equal(np.unique(sc.envs[0].material), [0, 1])


@pytest.mark.parametrize("mutate,msg", [
    (lambda s: s.update(extra=1), "scene.extra: unknown key"),
    (lambda s: s["grid"].pop("length"), "scene.grid.length: missing required field"),
    (lambda s: s["grid"].update(dims=[1, 2]), "scene.grid.dims: expected an array of 3 integers"),
    (lambda s: s["grid"].update(boundary=["sticky"] * 5 + ["glue"]), "scene.grid.boundary[5]: unknown boundary kind"),
    (lambda s: s["materials"].__setitem__(0, "granite"), "scene.materials[0]: unknown material preset 'granite'"),
    (lambda s: s["bodies"][1]["shapes"][0].update(type="torus"), "scene.bodies[1].shapes[0].type: unknown shape type"),
    (lambda s: s["bodies"][0].update(mode="floating"), "scene.bodies[0].mode: expected 'dynamic' or 'kinematic'"),
    (lambda s: s["sources"][1].update(material=5), "scene.sources[1].material: material index out of range"),
    (lambda s: s["stepping"].update(control_hz=60.0), "scene.stepping.control_hz: inconsistent"),
    (lambda s: s.update(robot={"chain": "arm"}), "scene.robot"),
])
def test_errors_name_the_field_path(mutate, msg):
    s = json.loads(json.dumps(SCENE))
    mutate(s)
    with pytest.raises(SceneConfigError, match=msg.replace("[", r"\[").replace("]", r"\]")):
        scene_from_json(s)


def test_envelope_warnings():
    s = json.loads(json.dumps(SCENE))
    s["grid"]["length"] = 0.02
    s["stepping"].pop("control_hz")
    warnings = []
    scene_from_json(s, warnings)
    assert warnings == ["grid.length outside validated range [0.005, 0.015]"]
    s["materials"][1]["youngs_modulus"] = 5e5
    warnings = []
    scene_from_json(s, warnings)
    assert "material youngs_modulus outside validated range [1e4, 3e5]" in warnings
