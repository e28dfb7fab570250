"""Scene JSON -> batched device world, host side.

`scene_from_json` reads the reference's scene format (`scene_from_json`,
shell.hpp:144-320) into a `Scene` for `GpuWorld`, with the reference's
validation: unknown keys and missing fields are errors naming their field
path ("scene config: scene.grid.dims: expected an array of 3 integers"),
out-of-envelope parameters are warnings (shell.hpp:120-137), and the stepping
block must satisfy 1/control_hz == n_rigid * n_soft * dt_soft. Particles are
seeded exactly as the reference does: one std::mt19937_64(seed) drawn
through every source box in order (seeding.hpp:13-35, via the library's own
seeder). `n_envs > 1` replicates the scene as a batch of identical worlds.

Scope: the soft-body path. A `robot` block (kinematic chains, controllers,
gripper) belongs to the reference's control stack, which is outside this
build; it is rejected with a pointer to scripted bodies. Extension (not in
the reference): a material object may carry "model" ("von_mises",
"fixed_corotated", "drucker_prager", "fluid").
"""
from __future__ import annotations

import json
import math

import numpy as np

from . import abi
from .scenes import BodySpec, EnvSpec, Rng, Scene, ShapeSpec, seed_box

V0_DEFAULT = 6.2e-8  # kSoftClayParticleVolume (mpm.hpp:47)
SOFT_CLAY_PRESET = (1000.0, 1e4, 0.3, 2e3)  # soft_clay() (mpm.hpp:45)
_MODELS = {"von_mises": abi.MODEL_HENCKY_VON_MISES, "fixed_corotated": abi.MODEL_FIXED_COROTATED,
           "drucker_prager": abi.MODEL_DRUCKER_PRAGER, "fluid": abi.MODEL_FLUID}


class SceneConfigError(RuntimeError):
    """std::runtime_error("scene config: <path>: <what>") of shell.hpp:22-24."""


def _err(path, what):
    raise SceneConfigError(f"scene config: {path}: {what}")


def _check_keys(o, path, allowed):  # shell.hpp:26-34
    if not isinstance(o, dict):
        _err(path, "expected an object")
    for k in o:
        if k not in allowed:
            _err(f"{path}.{k}", "unknown key")


def _require(o, path, key):  # shell.hpp:36-40
    if key not in o:
        _err(f"{path}.{key}", "missing required field")
    return o[key]


def _vec3(v, path):  # shell.hpp:42-45
    if not isinstance(v, list) or len(v) != 3:
        _err(path, "expected an array of 3 numbers")
    return tuple(float(a) for a in v)


def _pose(o, path):  # shell.hpp:47-59 -> (q wxyz, t)
    _check_keys(o, path, {"translation", "rotation_wxyz"})
    t = _vec3(o["translation"], path + ".translation") if "translation" in o else (0.0, 0.0, 0.0)
    q = (1.0, 0.0, 0.0, 0.0)
    if "rotation_wxyz" in o:
        r = o["rotation_wxyz"]
        if not isinstance(r, list) or len(r) != 4:
            _err(path + ".rotation_wxyz", "expected an array of 4 numbers")
        q = tuple(float(a) for a in r)
    return q, t


def _material(m, path):  # shell.hpp:61-73 (+ the "model" extension)
    if isinstance(m, str):
        if m == "soft_clay":
            return SOFT_CLAY_PRESET
        _err(path, f"unknown material preset '{m}'")
    _check_keys(m, path, {"density", "youngs_modulus", "poisson_ratio", "yield_stress", "model"})
    mat = (float(_require(m, path, "density")), float(_require(m, path, "youngs_modulus")),
           float(_require(m, path, "poisson_ratio")), float(_require(m, path, "yield_stress")))
    if "model" in m:
        if m["model"] not in _MODELS:
            _err(path + ".model", f"unknown model '{m['model']}'")
        mat = mat + (_MODELS[m["model"]],)
    return mat


def _shape(s, path, body, k_n, k_t):  # shell.hpp:75-104
    _check_keys(s, path, {"type", "half_extents", "radius", "half_length", "normal", "offset", "pose",
                          "friction", "k_n", "k_t"})
    typ = _require(s, path, "type")
    if typ == "box":
        kind, params = abi.SHAPE_BOX, _vec3(_require(s, path, "half_extents"), path + ".half_extents")
    elif typ == "sphere":
        kind, params = abi.SHAPE_SPHERE, (float(_require(s, path, "radius")),)
    elif typ == "capsule":
        kind = abi.SHAPE_CAPSULE
        params = (float(_require(s, path, "half_length")), float(_require(s, path, "radius")))
    elif typ == "plane":
        n = _vec3(s["normal"], path + ".normal") if "normal" in s else (0.0, 0.0, 1.0)
        nn = math.sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2])  # Vec3::normalized()
        n = (n[0] / nn, n[1] / nn, n[2] / nn)
        kind, params = abi.SHAPE_PLANE, n + (float(s.get("offset", 0.0)),)
    else:
        _err(path + ".type", f"unknown shape type '{typ}'")
    q, t = _pose(s["pose"], path + ".pose") if "pose" in s else ((1.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0))
    return ShapeSpec(kind, body, params=params, local_q=q, local_t=t, friction=float(s.get("friction", 0.5)),
                     k_n=float(s.get("k_n", k_n)), k_t=float(s.get("k_t", k_t)))


def _boundary(s, path):  # shell.hpp:115-119
    if s == "sticky":
        return 0
    if s == "slip":
        return 1
    _err(path, f"unknown boundary kind '{s}'")


def _range_warnings(scene, particle_volume, warnings):  # shell.hpp:120-137
    if warnings is None:
        return
    if scene.h < 0.005 or scene.h > 0.015:
        warnings.append("grid.length outside validated range [0.005, 0.015]")
    if particle_volume > 0.0 and (particle_volume < 6.2e-8 or particle_volume > 1.2e-7):
        warnings.append("particle_volume outside validated range [6.2e-8, 1.2e-7]")
    for m in scene.materials:
        if m[0] < 300.0 or m[0] > 3000.0:
            warnings.append("material density outside validated range [300, 3000]")
        if m[1] < 1e4 or m[1] > 3e5:
            warnings.append("material youngs_modulus outside validated range [1e4, 3e5]")
        if m[2] != 0.3:
            warnings.append("material poisson_ratio outside validated value 0.3")
        if m[3] < 2e3 or m[3] > 1e4:
            warnings.append("material yield_stress outside validated range [2e3, 1e4]")


def scene_from_json(root, warnings: list | None = None, n_envs: int = 1, name: str = "json") -> Scene:
    """The reference's scene_from_json (shell.hpp:144-320) for the soft-body path.
    `root` is a dict, a JSON string or a path to a .json file."""
    if isinstance(root, str):
        root = json.loads(root) if root.lstrip().startswith("{") else json.load(open(root))
    _check_keys(root, "scene", {"gravity", "grid", "materials", "sources", "bodies", "robot", "coupling",
                                "stepping", "seed", "deterministic"})
    scene = Scene(name=name)
    if "gravity" in root:
        g = _vec3(root["gravity"], "scene.gravity")
        scene.gravity = g
        scene.rigid_gravity = g
    grid = _require(root, "scene", "grid")
    _check_keys(grid, "scene.grid", {"length", "dims", "origin", "boundary"})
    scene.h = float(_require(grid, "scene.grid", "length"))
    if "dims" in grid:
        d = grid["dims"]
        if not isinstance(d, list) or len(d) != 3:
            _err("scene.grid.dims", "expected an array of 3 integers")
        scene.dims = tuple(int(a) for a in d)
    else:
        scene.dims = (64, 64, 64)  # MpmGrid defaults (mpm.hpp:68-73)
    if "origin" in grid:
        scene.origin = _vec3(grid["origin"], "scene.grid.origin")
    if "boundary" in grid:
        b = grid["boundary"]
        if not isinstance(b, list) or len(b) != 6:
            _err("scene.grid.boundary", "expected 6 per-face kinds")
        scene.boundary = tuple(_boundary(b[i], f"scene.grid.boundary[{i}]") for i in range(6))
    mats = _require(root, "scene", "materials")
    scene.materials = [_material(m, f"scene.materials[{i}]") for i, m in enumerate(mats)]

    k_n, k_t = 1e3, 10.0
    if "coupling" in root:
        c = root["coupling"]
        _check_keys(c, "scene.coupling", {"mode", "k_n", "k_t", "c_d", "r_c_factor"})
        if "mode" in c:
            if c["mode"] == "particle":
                scene.coupling_mode = abi.COUPLING_PARTICLE
            elif c["mode"] == "grid":
                scene.coupling_mode = abi.COUPLING_GRID
            else:
                _err("scene.coupling.mode", "expected 'particle' or 'grid'")
        scene.r_c_factor = float(c.get("r_c_factor", scene.r_c_factor))
        scene.c_d = float(c.get("c_d", scene.c_d))
        k_n = float(c.get("k_n", k_n))
        k_t = float(c.get("k_t", k_t))

    rng = Rng(int(root.get("seed", 42)))
    xs, ms, vols, mids = [], [], [], []
    last_v0 = 0.0
    for i, s in enumerate(root.get("sources", [])):
        path = f"scene.sources[{i}]"
        _check_keys(s, path, {"box_min", "box_max", "material", "particle_volume"})
        lo = _vec3(_require(s, path, "box_min"), path + ".box_min")
        hi = _vec3(_require(s, path, "box_max"), path + ".box_max")
        mat = int(s.get("material", 0))
        if mat < 0 or mat >= len(scene.materials):
            _err(path + ".material", "material index out of range")
        last_v0 = float(s.get("particle_volume", V0_DEFAULT))
        x, m = seed_box(rng, lo, hi, scene.materials[mat][0], last_v0)
        xs.append(x)
        ms.append(m)
        vols.append(np.full(len(m), last_v0))
        mids.append(np.full(len(m), mat, np.int32))

    bodies, shapes = [], []
    for i, b in enumerate(root.get("bodies", [])):
        path = f"scene.bodies[{i}]"
        _check_keys(b, path, {"name", "mode", "mass", "inertia", "com_offset", "pose", "shapes"})
        mode = b.get("mode", "kinematic")
        if mode not in ("dynamic", "kinematic"):
            _err(path + ".mode", "expected 'dynamic' or 'kinematic'")
        q, t = _pose(b["pose"], path + ".pose") if "pose" in b else ((1.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0))
        bodies.append(BodySpec(mode=abi.BODY_DYNAMIC if mode == "dynamic" else abi.BODY_KINEMATIC, q=q, t=t,
                               mass=float(b.get("mass", 1.0)),
                               inertia=_vec3(b["inertia"], path + ".inertia") if "inertia" in b else (1e-3,) * 3,
                               com_offset=_vec3(b["com_offset"], path + ".com_offset") if "com_offset" in b
                               else (0.0, 0.0, 0.0)))
        for si, s in enumerate(_require(b, path, "shapes")):
            shapes.append(_shape(s, f"{path}.shapes[{si}]", i, k_n, k_t))
    if "robot" in root:
        _err("scene.robot", "robot-driven links are outside the soft-body path of this build; "
                            "drive them as scripted bodies (MSIM_BODY_SCRIPTED) or push their poses with "
                            "msim_gpu_sync_bodies")

    if "stepping" in root:
        s = root["stepping"]
        _check_keys(s, "scene.stepping", {"dt_soft", "n_soft", "n_rigid", "control_hz"})
        scene.dt = float(s.get("dt_soft", scene.dt))
        scene.n_soft = int(s.get("n_soft", scene.n_soft))
        scene.n_rigid = int(s.get("n_rigid", scene.n_rigid))
        if "control_hz" in s:
            hz = float(s["control_hz"])
            period = scene.n_rigid * scene.n_soft * scene.dt
            if abs(period - 1.0 / hz) > 1e-9 * max(1.0, period):
                _err("scene.stepping.control_hz",
                     f"inconsistent: n_rigid * n_soft * dt_soft = {period:.6f} but 1/control_hz = {1.0 / hz:.6f}")
    if scene.n_rigid < 1 or scene.n_soft < 1:
        raise ValueError("World: n_rigid and n_soft must be >= 1")  # coupling.hpp:93-94

    x = np.concatenate(xs) if xs else np.zeros((0, 3))
    env = EnvSpec(x=x, mass=np.concatenate(ms) if ms else np.zeros(0),
                  vol0=np.concatenate(vols) if vols else np.zeros(0),
                  material=np.concatenate(mids) if mids else np.zeros(0, np.int32), bodies=bodies, shapes=shapes)
    scene.envs = [env] + [EnvSpec(x=env.x.copy(), mass=env.mass, vol0=env.vol0, material=env.material,
                                  bodies=list(bodies), shapes=list(shapes)) for _ in range(n_envs - 1)]
    _range_warnings(scene, last_v0, warnings)
    return scene
