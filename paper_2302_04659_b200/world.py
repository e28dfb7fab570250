"""Python mirror of the reference's soft-body API on top of the C ABI.

``GpuWorld`` is a thin, stateless-in-Python handle over one ``msim_gpu_ctx``
(include/msim_gpu.h): all state lives on the device. Method names follow the
reference (mpm.hpp / coupling.hpp): ``soft_substep``, ``p2g``,
``grid_update``, ``g2p_advect``, ``env_step``, ``sync_rigid_to_soft``.
Errors are raised as the reference's exception types: ``SimulationDiverged``
(MSIM_ERR_DIVERGED) and ``ValueError`` for std::invalid_argument.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from .scenes import Scene


class SimulationDiverged(RuntimeError):
    """mpm.hpp:18-20"""


class DeviceError(RuntimeError):
    pass


def _check(lib, ctx, rc: int):
    if rc == abi.MSIM_OK:
        return
    msg = lib.msim_gpu_last_error(ctx).decode() if ctx else lib.msim_gpu_create_error().decode()
    if rc == abi.MSIM_ERR_DIVERGED:
        raise SimulationDiverged(msg)
    if rc == abi.MSIM_ERR_INVALID:
        raise ValueError(msg)
    raise DeviceError(msg)


class GpuWorld:
    """All environments of a Scene on one device."""

    def __init__(self, scene: Scene, device: int = 0, split_channels: bool = False,
                 record_binning: bool = False, bucket_factor: int = 0, deterministic: bool = False):
        self.lib = lib = abi.load()
        self.scene = scene
        self.n_env = len(scene.envs)
        mats = scene.material_array()
        ctx = C.c_void_p()
        desc = scene.desc()
        _check(lib, None, lib.msim_gpu_create(C.byref(desc), mats, len(scene.materials), self.n_env, device,
                                              C.byref(ctx)))
        self.ctx = ctx
        if split_channels:
            self.set_split_channels(True)
        if record_binning:
            _check(lib, ctx, lib.msim_gpu_set_record_binning(ctx, 1))
        if bucket_factor:
            _check(lib, ctx, lib.msim_gpu_set_bucket_factor(ctx, bucket_factor))
        if deterministic:
            _check(lib, ctx, lib.msim_gpu_set_deterministic(ctx, 1))
        self.counts = [e.n for e in scene.envs]
        self.offsets = np.zeros(self.n_env + 1, dtype=np.int64)
        self.offsets[1:] = np.cumsum(self.counts)
        self.upload(scene)
        cp = abi.Coupling()
        cp.mode, cp.r_c_factor, cp.c_d = scene.coupling_mode, scene.r_c_factor, scene.c_d
        _check(lib, ctx, lib.msim_gpu_set_coupling(ctx, C.byref(cp)))
        g = np.asarray(scene.rigid_gravity, dtype=np.float64)
        _check(lib, ctx, lib.msim_gpu_set_rigid_gravity(ctx, abi.dptr(g)))
        for e, env in enumerate(scene.envs):
            if env.bodies:
                self.set_bodies(e, env.bodies, env.shapes)

    # ---- setup -------------------------------------------------------------
    def upload(self, scene: Scene):
        n = scene.n_particles

        def cat(attr, shape, default):
            if all(getattr(e, attr) is None for e in scene.envs):
                return None  # the C ABI defaults it (v = 0, F = I, C = 0)
            parts = []
            for e in scene.envs:
                a = getattr(e, attr)
                if a is None:
                    a = np.broadcast_to(default, (e.n,) + shape)
                parts.append(np.asarray(a, dtype=np.float64).reshape((e.n,) + shape))
            return np.ascontiguousarray(np.concatenate(parts) if parts else np.zeros((0,) + shape))

        x = cat("x", (3,), np.zeros(3))
        v = cat("v", (3,), np.zeros(3))
        F = cat("F", (3, 3), np.eye(3))
        Cm = cat("C", (3, 3), np.zeros((3, 3)))
        m = np.ascontiguousarray(np.concatenate([e.mass for e in scene.envs]).astype(np.float64))
        v0 = np.ascontiguousarray(np.concatenate([e.vol0 for e in scene.envs]).astype(np.float64))
        mat = np.ascontiguousarray(np.concatenate(
            [e.material if e.material is not None else np.zeros(e.n, np.int32) for e in scene.envs]
        ).astype(np.int32))
        _check(self.lib, self.ctx, self.lib.msim_gpu_set_particles(
            self.ctx, n, abi.lptr(self.offsets), abi.dptr(x), abi.dptr(v), abi.dptr(F), abi.dptr(Cm),
            abi.dptr(m), abi.dptr(v0), abi.iptr(mat)))

    def set_bodies(self, env: int, bodies, shapes):
        B = (abi.Body * max(len(bodies), 1))(*[b.to_c() for b in bodies])
        S = (abi.Shape * max(len(shapes), 1))(*[s.to_c() for s in shapes])
        _check(self.lib, self.ctx, self.lib.msim_gpu_set_bodies(self.ctx, env, B, len(bodies), S, len(shapes)))

    def sync_rigid_to_soft(self, env: int, bodies):
        """sync_rigid_to_soft (coupling.hpp:106-117) with new body states."""
        B = (abi.Body * max(len(bodies), 1))(*[b.to_c() for b in bodies])
        _check(self.lib, self.ctx, self.lib.msim_gpu_sync_bodies(self.ctx, env, B, len(bodies)))

    def set_dt(self, dt: float):
        _check(self.lib, self.ctx, self.lib.msim_gpu_set_dt(self.ctx, dt))

    def set_gravity(self, g):
        g = np.asarray(g, dtype=np.float64)
        _check(self.lib, self.ctx, self.lib.msim_gpu_set_gravity(self.ctx, abi.dptr(g)))

    def set_lost_fraction_threshold(self, t: float):
        _check(self.lib, self.ctx, self.lib.msim_gpu_set_lost_fraction_threshold(self.ctx, t))

    def set_split_channels(self, on: bool):
        _check(self.lib, self.ctx, self.lib.msim_gpu_set_split_channels(self.ctx, 1 if on else 0))

    def write_particles(self, env: int, x=None, v=None, F=None, Cm=None):
        n = self.counts[env]
        f = lambda a, s: None if a is None else np.ascontiguousarray(np.asarray(a, np.float64).reshape((n,) + s))
        x, v, F, Cm = f(x, (3,)), f(v, (3,)), f(F, (3, 3)), f(Cm, (3, 3))
        _check(self.lib, self.ctx, self.lib.msim_gpu_write_particles(
            self.ctx, env, n, abi.dptr(x), abi.dptr(v), abi.dptr(F), abi.dptr(Cm)))

    # ---- stepping ----------------------------------------------------------
    def set_kinematic_schedule(self, poses, mask=None):
        """poses[n_steps, n_total_bodies, 7] (qw qx qy qz tx ty tz per rigid step and
        body, all envs concatenated) for the next env_step; mask[n_total_bodies]
        selects the bodies (default: every kinematic body). See msim_gpu.h."""
        p = np.ascontiguousarray(poses, dtype=np.float64)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        _check(self.lib, self.ctx, self.lib.msim_gpu_set_kinematic_schedule(
            self.ctx, p.shape[0], abi.dptr(p), abi.u8ptr(m) if m is not None else None))

    def soft_substep(self, n: int = 1):
        cyc = np.zeros(self.n_env, dtype=np.int32)
        _check(self.lib, self.ctx, self.lib.msim_gpu_soft_substep(self.ctx, n, abi.iptr(cyc)))
        return cyc

    def p2g(self):
        _check(self.lib, self.ctx, self.lib.msim_gpu_p2g(self.ctx))

    def grid_update(self):
        _check(self.lib, self.ctx, self.lib.msim_gpu_grid_update(self.ctx))

    def g2p_advect(self):
        _check(self.lib, self.ctx, self.lib.msim_gpu_g2p(self.ctx))

    def env_step(self, n_rigid: int | None = None, n_soft: int | None = None) -> abi.StepReport:
        rep = abi.StepReport()
        nr = self.scene.n_rigid if n_rigid is None else n_rigid
        ns = self.scene.n_soft if n_soft is None else n_soft
        _check(self.lib, self.ctx, self.lib.msim_gpu_env_step(self.ctx, nr, ns, C.byref(rep)))
        return rep

    # ---- readback ----------------------------------------------------------
    def particles(self, env: int = 0):
        n = self.counts[env]
        x = np.zeros((n, 3))
        v = np.zeros((n, 3))
        F = np.zeros((n, 3, 3))
        Cm = np.zeros((n, 3, 3))
        lost = np.zeros(n, dtype=np.uint8)
        _check(self.lib, self.ctx, self.lib.msim_gpu_read_particles(
            self.ctx, env, abi.dptr(x), abi.dptr(v), abi.dptr(F), abi.dptr(Cm), abi.u8ptr(lost)))
        return dict(x=x, v=v, F=F, C=Cm, lost=lost)

    def jp(self, env: int = 0) -> np.ndarray:
        """Per-particle model scalar (fluid J, Drucker-Prager plastic strain, else 1)."""
        out = np.zeros(self.counts[env])
        _check(self.lib, self.ctx, self.lib.msim_gpu_read_jp(self.ctx, env, abi.dptr(out)))
        return out

    def grid(self, env: int = 0):
        nn = int(np.prod(self.scene.dims))
        m = np.zeros(nn)
        p = np.zeros((nn, 3))
        f = np.zeros((nn, 3))
        vel = np.zeros((nn, 3))
        _check(self.lib, self.ctx, self.lib.msim_gpu_read_grid(
            self.ctx, env, abi.dptr(m), abi.dptr(p), abi.dptr(f), abi.dptr(vel)))
        return dict(mass=m, momentum=p, force=f, velocity=vel)

    def write_grid_velocity(self, env: int, vel: np.ndarray):
        vel = np.ascontiguousarray(np.asarray(vel, dtype=np.float64).reshape(-1, 3))
        _check(self.lib, self.ctx, self.lib.msim_gpu_write_grid_velocity(self.ctx, env, abi.dptr(vel)))

    def binning(self, env: int = 0):
        n = self.counts[env]
        d = self.scene.dims
        nbins = (d[0] - 2) * (d[1] - 2) * (d[2] - 2)
        nn = d[0] * d[1] * d[2]
        base = np.zeros((n, 3), dtype=np.int32)
        cs = np.zeros(nbins + 1, dtype=np.int32)
        cp = np.zeros(max(n, 1), dtype=np.int32)
        act = np.zeros(nn, dtype=np.int64)
        n_alive = C.c_int64()
        n_act = C.c_int64()
        _check(self.lib, self.ctx, self.lib.msim_gpu_read_binning(
            self.ctx, env, abi.iptr(base), abi.iptr(cs), cs.size, abi.iptr(cp), cp.size, C.byref(n_alive),
            abi.lptr(act), act.size, C.byref(n_act)))
        return dict(base=base, cell_start=cs, cell_particles=cp[: n_alive.value], active_nodes=act[: n_act.value])

    def buckets(self, env: int = 0):
        """The hot path's own binning: bucket shape, per-bucket counts for the next
        particle launch, and the node blocks the last P2G touched (msim_gpu_read_buckets)."""
        cells, bdims, kdims = (np.zeros(3, np.int32) for _ in range(3))
        _check(self.lib, self.ctx, self.lib.msim_gpu_read_buckets(
            self.ctx, env, abi.iptr(cells), abi.iptr(bdims), None, 0, abi.iptr(kdims), None, 0, None))
        counts = np.zeros(int(np.prod(bdims)), np.int32)
        nblk = C.c_int64()
        _check(self.lib, self.ctx, self.lib.msim_gpu_read_buckets(
            self.ctx, env, None, None, abi.iptr(counts), counts.size, None, None, 0, C.byref(nblk)))
        blocks = np.zeros(max(nblk.value, 1), np.int32)
        _check(self.lib, self.ctx, self.lib.msim_gpu_read_buckets(
            self.ctx, env, None, None, None, 0, None, abi.iptr(blocks), blocks.size, C.byref(nblk)))
        return dict(bucket_cells=cells, bucket_dims=bdims, counts=counts, block_dims=kdims,
                    blocks=blocks[: nblk.value])

    def wrenches(self, env: int = 0, pending: bool = False):
        nb = len(self.scene.envs[env].bodies)
        f = np.zeros((max(nb, 1), 3))
        t = np.zeros((max(nb, 1), 3))
        _check(self.lib, self.ctx, self.lib.msim_gpu_read_wrenches(self.ctx, env, 1 if pending else 0,
                                                                    abi.dptr(f), abi.dptr(t)))
        return f[:nb], t[:nb]

    def bodies(self, env: int = 0):
        nb = len(self.scene.envs[env].bodies)
        B = (abi.Body * max(nb, 1))()
        _check(self.lib, self.ctx, self.lib.msim_gpu_read_bodies(self.ctx, env, B, nb))
        return [B[i] for i in range(nb)]

    def report(self, env: int = 0) -> abi.StepReport:
        r = abi.StepReport()
        _check(self.lib, self.ctx, self.lib.msim_gpu_read_report(self.ctx, env, C.byref(r)))
        return r

    def lost_count(self, env: int = 0) -> int:
        return int(self.lib.msim_gpu_lost_count(self.ctx, env))

    def constitutive(self, F: np.ndarray, mat: int = 0):
        """(kirchhoff_stress(F), von_mises_return_map(F)) on the device code path."""
        F = np.ascontiguousarray(np.asarray(F, dtype=np.float64).reshape(-1, 3, 3))
        n = F.shape[0]
        tau = np.zeros_like(F)
        Fp = np.zeros_like(F)
        _check(self.lib, self.ctx, self.lib.msim_gpu_constitutive(self.ctx, mat, n, abi.dptr(F), abi.dptr(tau),
                                                                  abi.dptr(Fp)))
        return tau, Fp

    def seed_envs(self, envs, seeds, boxes, material: int = 0, particle_volume: float | None = None):
        """Batched env reset on the device: seed_particles_box (seeding.hpp:13-35) with
        mt19937_64(seeds[i]) into boxes[i] = (min xyz, max xyz) for envs[i]."""
        envs = np.ascontiguousarray(np.asarray(envs, np.int32))
        seeds = np.ascontiguousarray(np.asarray(seeds, np.uint64))
        boxes = np.ascontiguousarray(np.asarray(boxes, np.float64).reshape(-1, 6))
        if particle_volume is None:
            particle_volume = float(self.scene.envs[int(envs[0])].vol0[0])
        _check(self.lib, self.ctx, self.lib.msim_gpu_seed_envs(
            self.ctx, len(envs), envs.ctypes.data_as(C.POINTER(C.c_int32)), seeds.ctypes.data_as(C.POINTER(C.c_uint64)),
            abi.dptr(boxes), material, particle_volume))

    # ---- task metrics over every env (scenario.hpp:63-209) -------------------
    def _regions(self, regions):
        regions = np.asarray(regions, dtype=np.float64).reshape(-1, 6)
        if regions.shape[0] == 1 and self.n_env > 1:
            regions = np.repeat(regions, self.n_env, axis=0)
        arr = (abi.Region * self.n_env)()
        for e in range(self.n_env):
            arr[e].min[:] = regions[e, :3]
            arr[e].max[:] = regions[e, 3:]
        return arr

    def metric_fill(self, regions):
        """metric_fill per env -> list of (fraction, max_speed, success); regions (n_env|1, 6) = min xyz, max xyz."""
        out = (abi.FillResult * self.n_env)()
        _check(self.lib, self.ctx, self.lib.msim_gpu_metric_fill(self.ctx, self._regions(regions), out))
        return [(r.fraction, r.max_speed, bool(r.success)) for r in out]

    def render_heightmap(self, regions, nx: int, ny: int):
        """render_heightmap per env -> (n_env, ny, nx) heights above each region floor."""
        maps = np.zeros((self.n_env, ny, nx))
        _check(self.lib, self.ctx, self.lib.msim_gpu_render_heightmap(self.ctx, self._regions(regions), nx, ny,
                                                                      abi.dptr(maps)))
        return maps

    def metric_write_iou(self, regions, targets, threshold: float):
        """metric_write_iou of each env's heightmap vs targets (n_env, ny, nx) -> (iou[n_env], success[n_env])."""
        t = np.ascontiguousarray(np.asarray(targets, dtype=np.float64))
        ny, nx = t.shape[-2], t.shape[-1]
        t = np.ascontiguousarray(np.broadcast_to(t, (self.n_env, ny, nx)))
        iou = np.zeros(self.n_env)
        ok = np.zeros(self.n_env, np.int32)
        _check(self.lib, self.ctx, self.lib.msim_gpu_metric_write_iou(
            self.ctx, self._regions(regions), nx, ny, threshold, abi.dptr(t), abi.dptr(iou),
            ok.ctypes.data_as(C.POINTER(C.c_int32))))
        return iou, ok.astype(bool)

    @staticmethod
    def _point_sets(sets):
        pts = np.ascontiguousarray(np.concatenate([np.asarray(p, np.float64).reshape(-1, 3) for p in sets]))
        off = np.zeros(len(sets) + 1, np.int64)
        off[1:] = np.cumsum([np.asarray(p).reshape(-1, 3).shape[0] for p in sets])
        return pts, off

    def chamfer(self, targets):
        """chamfer_distance(particles of env e, targets[e]) for every env."""
        pts, off = self._point_sets(targets)
        out = np.zeros(self.n_env)
        _check(self.lib, self.ctx, self.lib.msim_gpu_chamfer(self.ctx, abi.dptr(pts), off.ctypes.data_as(
            C.POINTER(C.c_int64)), abi.dptr(out)))
        return out

    def metric_pinch(self, initial, targets):
        """metric_pinch(current = env particles, initial[e], targets[e]) -> (ratio[n_env], success[n_env])."""
        ip, io = self._point_sets(initial)
        tp, to = self._point_sets(targets)
        ratio = np.zeros(self.n_env)
        ok = np.zeros(self.n_env, np.int32)
        lp = C.POINTER(C.c_int64)
        _check(self.lib, self.ctx, self.lib.msim_gpu_metric_pinch(
            self.ctx, abi.dptr(ip), io.ctypes.data_as(lp), abi.dptr(tp), to.ctypes.data_as(lp), abi.dptr(ratio),
            ok.ctypes.data_as(C.POINTER(C.c_int32))))
        return ratio, ok.astype(bool)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.msim_gpu_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def bake_mesh_sdf(triangles, voxel: float, padding: float, device: int = 0):
    """bake_mesh_sdf (sdf.hpp:277-310) on the GPU -> (origin[3], dims[3], samples f32 x-fastest).
    triangles: (n, 3, 3) or flat (a, b, c per triangle)."""
    lib = abi.load()
    tri = np.ascontiguousarray(np.asarray(triangles, dtype=np.float64).reshape(-1))
    n = tri.size // 9
    origin, dims = np.zeros(3), np.zeros(3, np.int32)
    ip = C.POINTER(C.c_int32)
    _check(lib, None, lib.msim_bake_grid(abi.dptr(tri), n, voxel, padding, abi.dptr(origin), dims.ctypes.data_as(ip)))
    out = np.zeros(int(np.prod(dims)), np.float32)
    _check(lib, None, lib.msim_gpu_bake_mesh_sdf(device, abi.dptr(tri), n, voxel, padding,
                                                 out.ctypes.data_as(C.POINTER(C.c_float)), out.size))
    return origin, dims, out


def make_box_mesh(half_extents, center=(0.0, 0.0, 0.0)):
    """make_box_mesh (sdf.hpp:443-455) -> (12, 3, 3) triangles."""
    lib = abi.load()
    h = np.ascontiguousarray(np.asarray(half_extents, np.float64))
    c = np.ascontiguousarray(np.asarray(center, np.float64))
    tri = np.zeros(108)
    lib.msim_make_box_mesh(abi.dptr(h), abi.dptr(c), abi.dptr(tri))
    return tri.reshape(12, 3, 3)
