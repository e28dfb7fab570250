"""Shared fixtures for the GPU tests: small scenes built like the reference
tests' make_state / add_particle / seed_random_cloud (test_mpm.cpp:21-48)."""
from __future__ import annotations

import numpy as np

from paper_2302_04659_b200.scenes import SOFT_CLAY, STIFF_CLAY, V0_SOFT, EnvSpec, Scene


class Cloud:
    def __init__(self):
        self.x, self.v, self.m, self.mat = [], [], [], []
        self.F, self.C = [], []

    def add(self, x, v=(0, 0, 0), mass=1e-4, mat=0, F=None, C=None):
        self.x.append(np.asarray(x, dtype=np.float64))
        self.v.append(np.asarray(v, dtype=np.float64))
        self.m.append(mass)
        self.mat.append(mat)
        self.F.append(np.eye(3) if F is None else np.asarray(F, dtype=np.float64))
        self.C.append(np.zeros((3, 3)) if C is None else np.asarray(C, dtype=np.float64))

    def env(self) -> EnvSpec:
        n = len(self.x)
        return EnvSpec(x=np.array(self.x).reshape(n, 3), v=np.array(self.v).reshape(n, 3),
                       mass=np.array(self.m, dtype=np.float64), vol0=np.full(n, V0_SOFT),
                       material=np.array(self.mat, dtype=np.int32), F=np.array(self.F).reshape(n, 3, 3),
                       C=np.array(self.C).reshape(n, 3, 3))


def make_scene(cloud: Cloud | list, dims=32, h=0.01, gravity=(0, 0, 0), dt=1e-4, **kw) -> Scene:
    """make_state (test_mpm.cpp:21-30): soft + stiff clay, zero gravity, dt 1e-4."""
    envs = [c.env() for c in cloud] if isinstance(cloud, list) else [cloud.env()]
    return Scene(name="kat", dims=(dims, dims, dims), h=h, gravity=gravity, dt=dt,
                 materials=[SOFT_CLAY, STIFF_CLAY], envs=envs, **kw)


def random_cloud(n, rng, dims=32, h=0.01, lo_cells=4, hi_cells=5, vel=0.5, mass=(1e-5, 1e-3)):
    """seed_random_cloud (test_mpm.cpp:43-48)."""
    c = Cloud()
    lo, hi = lo_cells * h, (dims - hi_cells) * h
    for _ in range(n):
        c.add(rng.uniform(lo, hi, 3), rng.uniform(-vel, vel, 3), rng.uniform(*mass))
    return c


def node_pos(i, j, k, h=0.01):
    return np.array([i * h, j * h, k * h])


def node_index(i, j, k, dims=32):
    return (k * dims + j) * dims + i


def rel(a, b, floor=0.0):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), floor, 1e-300))


def round_f32(scene: Scene) -> Scene:
    """Feed both paths the fp32-rounded state (SURVEY App. A.2 integer protocol)."""
    for e in scene.envs:
        e.x = e.x.astype(np.float32).astype(np.float64)
        if e.v is not None:
            e.v = e.v.astype(np.float32).astype(np.float64)
    return scene
