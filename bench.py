#!/usr/bin/env python3
"""Benchmark of the B200 MLS-MPM substep (BASELINE.json metric:
particle-substeps/s and env-steps/s per GPU, % of HBM roofline).

Workload: config D of SURVEY.md App. B (1024 envs x 16,384 von Mises firm-clay
particles, 32^3 grid per env, 25 substeps per env step, write-stamp / pinch
colliders), synthetic seeded inputs. One "step" = one env step of all envs
(25 soft substeps through msim_gpu_env_step). Multi-GPU: one process per GPU,
each rank owns its own 1024 envs (env ids offset by rank) -> weak scaling; the
only collective is the stats all-reduce (timing max, step counters).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

BYTES_PER_PS = 268.0        # BASELINE.md / SURVEY.md §8d: algorithmic bytes per particle-substep
                            #   P2G read 112 + G2P read 56 + G2P write 100 (fp32 SoA)
# k_particles runs G2P of one cycle and P2G of the next in one pass: one launch
# is one particle-substep of every particle, so its algorithmic bytes per launch
# are 268 B x particles.
METRIC = "particle-substeps/sec and env-steps/sec per GPU, % HBM roofline, 1/2/4/8 B200"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_info():
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        model = "unknown"
    return os.cpu_count() or 1, model


# ---------------------------------------------------------------------------
# Reference arm: the CPU restatement of the reference (oracle/), all host cores,
# independent worlds on threads (the `bench --worlds K` semantics, shell.hpp:366-407).

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle.oracle_py import OracleWorld, build as build_oracle
    from paper_2302_04659_b200.scenes import config_d

    build_oracle()
    cores, model = cpu_info()
    threads = cores
    scene = config_d(n_envs=threads)
    worlds = [OracleWorld(scene, env=e, threads=1) for e in range(threads)]
    ps_per_step = sum(e.n for e in scene.envs) * scene.substeps_per_env_step

    def one_step():
        ts = [threading.Thread(target=w.env_step) for w in worlds]
        for t in ts:
            t.start()
        for t in ts:
            t.join()

    for _ in range(args.warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step()
    dt = time.perf_counter() - t0
    value = ps_per_step * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "particle-substeps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "env_steps_per_s": threads * args.steps / dt,
        "config": {"workload": "D: batched write/pinch von Mises firm clay, 16384 particles/env, 32^3 grid/env, "
                               "25 substeps/env step", "envs_per_step": threads, "particles_per_env": 16384,
                   "substeps_per_env_step": 25},
        "cpu_baseline": {"value": value, "unit": "particle-substeps/s", "cores": threads, "kind": "port",
                         "sample": f"{threads} independent config-D envs (one per thread) x {args.steps} env steps; "
                                   f"oracle/ double-precision restatement (reference unbuildable: needs Eigen3+GTest); "
                                   f"host CPU {model}"},
        "e2e": {"value": value, "unit": "particle-substeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------

def cpu_baseline_sample(scene_env_fn, substeps):
    """Oracle, 1 thread, a bounded sample (1 env of the same workload)."""
    from oracle.oracle_py import OracleWorld, build as build_oracle
    from paper_2302_04659_b200.scenes import config_d

    build_oracle()
    sc = config_d(n_envs=2)
    t_total, ps = 0.0, 0
    for e in range(2):
        w = OracleWorld(sc, env=e, threads=1)
        t_total += w.time_env_steps(1)
        ps += sc.envs[e].n * sc.substeps_per_env_step
    return ps / t_total, f"2 config-D envs (write + pinch) x 1 env step (25 substeps), {ps} particle-substeps"


def load_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per particle of the dominant kernel,
    from the committed ncu --set full capture (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        return t[kernel]["dram_bytes_per_particle"], t[kernel].get("source", "")
    except Exception:
        return None, None


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)

    from paper_2302_04659_b200 import GpuWorld, abi
    from paper_2302_04659_b200.dist import StepStats, allreduce_stats, weak_first_env
    from paper_2302_04659_b200.scenes import config_d, config_e

    lib = abi.load()
    t_setup = time.perf_counter()
    if args.config == "E":
        scene = config_e(clay_only=args.clay_only)
        n_envs = 1
        workload = (("E: 4M soft/stiff clay (clay-only variant)" if args.clay_only else
                     "E: 4M mixed clay / Drucker-Prager sand / J-only water / fixed-corotated jelly slabs")
                    + ", 256^3 grid h=0.005, 8 moving colliders (boxes, spheres, capsules, SDF volume), "
                    "25 substeps/env step, replica per GPU")
    else:
        n_envs = args.envs
        scene = config_d(n_envs=n_envs, first_env=weak_first_env(n_envs, rank))
        workload = ("D: batched write/pinch von Mises firm clay, 16384 particles/env, 32^3 grid/env, "
                    "25 substeps/env step, per-rank envs")
    gw = GpuWorld(scene, device=local)
    ctx = gw.ctx
    setup_s = time.perf_counter() - t_setup
    n_part = scene.n_particles
    S = scene.substeps_per_env_step
    stream = torch.cuda.ExternalStream(lib.msim_gpu_stream(ctx), device=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        gw.env_step()
    torch.cuda.synchronize()

    # ---- timed region: K env steps, device events on the library stream
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    l0 = lib.msim_gpu_launches(ctx)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    stats = StepStats()
    for _ in range(args.steps):
        rep = gw.env_step()
        # per-env-step statistics exchange (the only collective)
        st = StepStats(n_part * S, n_envs, rep.cfl_cycles, rep.lost_particles, rep.max_penetration,
                       rep.max_force_balance_error)
        st = allreduce_stats(st, device=torch.device("cuda", local)) if world > 1 else st
        stats.particle_substeps += st.particle_substeps
        stats.env_steps += st.env_steps
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = lib.msim_gpu_launches(ctx) - l0
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ps_total = world * n_part * S * args.steps
    value = ps_total / (ms_max / 1e3)
    env_steps = world * n_envs * args.steps / (ms_max / 1e3)

    # ---- per-kernel CUDA-event durations (instrumented pass, same stream)
    lib.msim_gpu_set_kernel_timing(ctx, 1)
    kstep = max(1, min(args.steps, 2))
    for _ in range(kstep):
        gw.env_step()
    torch.cuda.synchronize()
    kernels = {}
    for kid in range(lib.msim_gpu_kernel_count()):
        name = C.c_char_p()
        cnt = C.c_int64()
        tot = C.c_double()
        lib.msim_gpu_kernel_stats(ctx, kid, C.byref(name), C.byref(cnt), C.byref(tot))
        if cnt.value:
            kernels[name.value.decode()] = {"launches": cnt.value, "avg_ms": tot.value / cnt.value,
                                            "total_ms": tot.value}
    lib.msim_gpu_set_kernel_timing(ctx, 0)
    step_ms_instr = sum(k["total_ms"] for k in kernels.values()) / kstep
    # dominant kernel and its roofline (algorithmic bytes per launch / avg launch time)
    dom = max(kernels, key=lambda k: kernels[k]["total_ms"])
    peak, peak_src = peaks()
    # one k_particles launch = one particle-substep of every particle of the rank
    dom_bytes = BYTES_PER_PS * n_part if dom == "k_particles" else None
    achieved = dom_bytes / (kernels[dom]["avg_ms"] / 1e3) / 1e9 if dom_bytes else None
    tpp, tsrc = load_traffic(dom)
    traffic = args.traffic if args.traffic is not None else (tpp * n_part if tpp else None)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "traffic_source": tsrc, "alg_bytes_per_launch": dom_bytes, "avg_launch_ms": kernels[dom]["avg_ms"],
                "share_of_step": kernels[dom]["total_ms"] / kstep / max(step_ms_instr, 1e-9),
                "peak_source": peak_src}
    path_achieved = value / world * BYTES_PER_PS / 1e9
    roofline_path = {"bound": "hbm", "achieved": path_achieved, "peak": peak, "unit": "GB/s",
                     "frac": path_achieved / peak, "bytes_per_particle_substep": BYTES_PER_PS,
                     "note": "BASELINE.md: PS/s per GPU x 268 B / HBM peak"}

    # ---- end to end through the C ABI with host buffers: body states in, wrenches + report out
    nb = lib.msim_gpu_body_count(ctx, -1)
    bodies = (abi.Body * max(nb, 1))()
    k = 0
    for e in range(n_envs):
        for b in gw.bodies(e):
            bodies[k] = b
            k += 1
    wr = np.zeros(max(nb, 1) * 6)
    rep = abi.StepReport()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        lib.msim_gpu_sync_all_bodies(ctx, bodies, nb)
        lib.msim_gpu_env_step(ctx, scene.n_rigid, scene.n_soft, C.byref(rep))
        lib.msim_gpu_read_all_wrenches(ctx, 1, abi.dptr(wr))
    e1.record(stream)
    torch.cuda.synchronize()
    wall_e2e = time.perf_counter() - h0
    e2e_ms = max(e0.elapsed_time(e1), 1e3 * wall_e2e)
    t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = ps_total / (float(t.item()) / 1e3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, sample = cpu_baseline_sample(None, S)
        cores, model = cpu_info()
        cpu = {"value": v, "unit": "particle-substeps/s", "cores": 1, "kind": "port",
               "sample": sample + f"; oracle/ double-precision restatement, 1 thread, host {model}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "particle-substeps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded jittered lattices, seeding.hpp algorithm)",
            "env_steps_per_s": env_steps,
            "per_gpu": {"particle_substeps_per_s": value / world, "env_steps_per_s": env_steps / world},
            "config": {"workload": workload, "envs_per_gpu": n_envs,
                       "particles_per_gpu": n_part, "substeps_per_env_step": S, "dt": scene.dt,
                       "parallelism": f"env-sharded x{world} (no data-path collective)",
                       "l2": "inputs larger than L2 (particle state 2 x %.2f GB)" % (n_part * 116 / 1e9)},
            "roofline": roofline,
            "roofline_path": roofline_path,
            "kernels": kernels,
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": {"value": e2e_value, "unit": "particle-substeps/s",
                    "h2d_bytes_per_step": nb * C.sizeof(abi.Body), "d2h_bytes_per_step": nb * 48 + C.sizeof(rep)},
            "cpu_baseline": cpu,
            "setup_s": setup_s,
            "stats": {"particle_substeps": stats.particle_substeps, "env_steps": stats.env_steps},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--envs", type=int, default=1024, help="config-D envs per GPU")
    ap.add_argument("--config", choices=["D", "E"], default="D", help="workload (SURVEY.md App. B)")
    ap.add_argument("--clay-only", action="store_true", help="config E: the reference's model only")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--traffic", type=float, default=None, help="ncu dram bytes per launch of the dominant kernel")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch this command under torch.distributed.run
        import socket

        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        os.execvp(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                   f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                                   "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]])
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
