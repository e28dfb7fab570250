#!/usr/bin/env python3
"""Benchmark of the B200 MLS-MPM substep (BASELINE.json metric:
particle-substeps/s and env-steps/s per GPU, % of HBM roofline).

Workload (default): config D of SURVEY.md App. B -- 1024 envs x 16,384 von Mises
firm-clay particles, 32^3 grid per env, 25 substeps per env step, write-stamp /
pinch colliders; synthetic seeded inputs. One "step" = one env step of every env
(25 soft substeps through msim_gpu_env_step). Multi-GPU: one
process per GPU, the --envs global envs sharded contiguously over the ranks
(rank r owns [r E/G, (r+1) E/G)) -> strong scaling; --weak gives every rank its
own --envs. --config B / C run batched Excavate / Pour-shaped envs (sharded the
same way), A and E one scene per GPU (replicas). The only collective is the
per-env-step statistics all-reduce.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config A|B|C|D|E] [--envs E] [--weak] [--clay-only]

--impl reference times the reference's OWN code (oracle/_ref/libmsim_ref.so:
the reference sources compiled unchanged against oracle/ref_shim) on the box's
host cores, worlds built by the reference's seeder (oracle/ref_scenes.py); that
arm never imports or loads the product.

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
# k_particles runs G2P of one cycle and P2G of the next in one pass. One env step
# of S substeps is S + 1 launches (the first P2G-only, the last G2P-only), so the
# kernel's roofline is taken per env step: S x 268 B x particles over the
# kernel's CUDA-event time per env step.
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
# Reference arm: the reference's own code (oracle/_ref), all host cores,
# independent worlds each on its own thread (the aggregate mode of the
# reference's `bench --worlds K`, shell.hpp:366-407). No product import.

WORKLOADS = {
    "A": "A: 8k soft clay, 64^3 grid, one dynamic box, 25 substeps/env step, one scene per GPU",
    "B": "B: batched Excavate-shaped envs, 32k {mat} particles/env, 64^3 grid/env, scripted 5-box bucket, "
         "25 substeps/env step",
    "C": "C: batched Pour-shaped envs, 64k {mat} particles/env, 128^3 grid/env h=0.005, rotating bottle + "
         "static beaker, 25 substeps/env step",
    "D": "D: batched write/pinch von Mises firm clay, 16384 particles/env, 32^3 grid/env, 25 substeps/env step",
}
PARTICLES_PER_ENV = {"A": 8000, "B": 32000, "C": 64000, "D": 16384}
DEFAULT_ENVS = {"B": 128, "C": 32, "D": 1024}
# env count of the committed ncu traffic capture per config (profiles/traffic.json)
PARTICLES_N = {"D": 1024, "E": 1}


def ref_lib_or_none():
    from oracle import oracle_py

    return oracle_py.load_ref() if oracle_py.ref_available() else None


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if args.config == "E":
        print(json.dumps({"impl": "reference", "unavailable": "config E mixes materials the reference does not have "
                          "(Drucker-Prager, fluid, fixed-corotated); its reference arm runs D"}), flush=True)
        return 0
    from oracle import ref_scenes

    lib = ref_lib_or_none()
    if lib is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return 0
    cores, model = cpu_info()
    K = cores
    worlds = [ref_scenes.build_world(args.config, 0 if args.config == "A" else e) for e in range(K)]
    arr = (C.c_void_p * K)(*worlds)
    err = C.c_int32(0)
    if args.warmup:
        lib.ref_bench_worlds(arr, K, args.warmup, C.byref(err))
    sec = lib.ref_bench_worlds(arr, K, args.steps, C.byref(err))
    assert err.value == 0, "reference diverged"
    for w in worlds:
        lib.oracle_destroy(w)
    S = 25
    n_env = PARTICLES_PER_ENV[args.config]
    value = K * n_env * S * args.steps / sec
    sample = (f"{K} independent config-{args.config} worlds, one per host thread, x {args.steps} env steps "
              f"(+{args.warmup} warm-up); the reference's own sources (oracle/_ref/libmsim_ref.so, compiled "
              f"unchanged against oracle/ref_shim's Eigen subset, -O3, fp64); host CPU {model}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "particle-substeps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "env_steps_per_s": K * args.steps / sec,
        "config": {"workload": WORKLOADS[args.config].format(mat="soft clay"), "envs_per_step": K,
                   "particles_per_env": n_env, "substeps_per_env_step": S},
        "cpu_baseline": {"value": value, "unit": "particle-substeps/s", "cores": K, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "particle-substeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------

def cpu_baseline_sample(config: str):
    """The reference's own code (oracle/_ref), 1 thread, a bounded sample of the
    workload; the oracle restatement when oracle/_ref is absent."""
    from oracle import oracle_py

    cfg = config if config in ("A", "B", "C", "D") else "D"
    envs = [0, 1] if cfg == "D" else [0]
    ps = PARTICLES_PER_ENV[cfg] * 25 * len(envs)
    if oracle_py.ref_available():
        from oracle import ref_scenes

        lib = oracle_py.load_ref()
        lib.oracle_set_threads(1)
        t = 0.0
        for e in envs:
            w = ref_scenes.build_world(cfg, e)
            err = C.c_int32(0)
            t += lib.oracle_time_env_steps(w, 1, C.byref(err))
            lib.oracle_destroy(w)
        kind, what = "reference", "the reference's own sources (oracle/_ref/libmsim_ref.so)"
    else:
        from paper_2302_04659_b200.scenes import config_d

        sc = config_d(n_envs=2)
        t = sum(oracle_py.OracleWorld(sc, env=e, threads=1).time_env_steps(1) for e in envs)
        kind, what = "port", "oracle/ double-precision restatement"
    note = "" if cfg == config else f" (config {config} has no reference counterpart: D sample)"
    return ps / t, kind, (f"{len(envs)} config-{cfg} env(s) x 1 env step (25 substeps) = {ps} particle-substeps, "
                          f"{what}, 1 thread{note}")


def load_traffic(config: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per particle of one fused
    k_particles launch, from the committed `ncu --set full` capture of THIS
    config (profiles/traffic.json, tagged with the capture's git SHA), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)[config]
        return t["dram_bytes_per_particle_per_fused_launch"], t
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
    from paper_2302_04659_b200.dist import LibStats, StepStats, allreduce_stats, rank_envs
    from paper_2302_04659_b200.scenes import SAND, SOFT_CLAY, WATER, config_a, config_b, config_c, config_d, config_e

    lib = abi.load()
    t_setup = time.perf_counter()
    cfg = args.config
    scaling = "weak"
    if cfg in ("B", "C", "D"):
        lo, n_envs = rank_envs(args.envs, rank, world, weak=args.weak)
        scaling = "weak" if args.weak else "strong"
        if cfg == "D":
            scene = config_d(n_envs=n_envs, first_env=lo)
            workload = WORKLOADS["D"]
        else:
            mat = SOFT_CLAY if args.clay_only else (SAND if cfg == "B" else WATER)
            scene = (config_b if cfg == "B" else config_c)(material=mat, n_envs=n_envs, first_env=lo)
            workload = WORKLOADS[cfg].format(
                mat="soft clay" if args.clay_only else ("Drucker-Prager sand" if cfg == "B" else "J-only fluid"))
        envs_global = n_envs * world if args.weak else args.envs
    elif cfg == "A":
        scene, n_envs, workload, envs_global = config_a(), 1, WORKLOADS["A"], world
    else:
        scene = config_e(clay_only=args.clay_only)
        n_envs, envs_global = 1, world
        workload = (("E: 4M soft/stiff clay (clay-only variant)" if args.clay_only else
                     "E: 4M mixed clay / Drucker-Prager sand / J-only water / fixed-corotated jelly slabs")
                    + ", 256^3 grid h=0.005, 8 moving colliders (boxes, spheres, capsules, SDF volume), "
                    "25 substeps/env step, one scene per GPU")
    gw = GpuWorld(scene, device=local, deterministic=args.deterministic)
    ctx = gw.ctx
    setup_s = time.perf_counter() - t_setup
    n_part = scene.n_particles
    S = scene.substeps_per_env_step
    stream = torch.cuda.ExternalStream(lib.msim_gpu_stream(ctx), device=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    def barrier():
        if world > 1:
            dist.barrier()

    def tmax(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def tsum(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # the per-env-step statistics exchange: the library's device reduction + NCCL
    # all-reduce on its stream (msim_gpu_step_stats); torch's all-reduce if NCCL
    # cannot be resolved
    os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep NCCL's version banner off stdout (one JSON line)
    try:
        libstats = LibStats(lib, ctx, rank, world)
    except (RuntimeError, AttributeError) as e:
        libstats = None
        print(f"[bench] library NCCL stats unavailable ({e}); torch all-reduce", file=sys.stderr)
    for _ in range(args.warmup):
        gw.env_step()
        if libstats:
            libstats.step()
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
        if libstats:
            st = libstats.step()
        else:
            st = StepStats(n_part * S, n_envs, rep.cfl_cycles, rep.lost_particles, rep.max_penetration,
                           rep.max_force_balance_error)
            st = allreduce_stats(st, device=dev) if world > 1 else st
        stats.particle_substeps += st.particle_substeps
        stats.env_steps += st.env_steps
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = lib.msim_gpu_launches(ctx) - l0
    clocks = sampler.stop()
    ms_max = tmax(ev0.elapsed_time(ev1))
    ps_total = tsum(n_part * S * args.steps)
    value = ps_total / (ms_max / 1e3)
    env_steps = tsum(n_envs * args.steps) / (ms_max / 1e3)

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
    # dominant kernel and its roofline: algorithmic bytes of one env step (S x 268 B x
    # particles) over the kernel's CUDA-event time per env step
    dom = max(kernels, key=lambda k: kernels[k]["total_ms"])
    peak, peak_src = peaks()
    dom_ms_per_step = kernels[dom]["total_ms"] / kstep
    dom_bytes = S * BYTES_PER_PS * n_part if dom == "k_particles" else None
    achieved = dom_bytes / (dom_ms_per_step / 1e3) / 1e9 if dom_bytes else None
    tpp, tinfo = load_traffic(cfg)
    launches_per_step = kernels[dom]["launches"] / kstep
    traffic = (args.traffic if args.traffic is not None else
               (tpp * n_part * launches_per_step if tpp and world == 1 and n_envs == PARTICLES_N.get(cfg, -1) else None))
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": traffic,
                "traffic_note": ("ncu dram__bytes_read.sum + dram__bytes_write.sum of one fused launch x launches "
                                 "per env step, from " + tinfo["capture"] + " (git " + tinfo["git_sha"] + ")")
                if traffic is not None and tinfo else "no ncu capture of this exact config/size",
                "per": "env step", "alg_bytes": dom_bytes, "ms_per_env_step": dom_ms_per_step,
                "launches_per_env_step": launches_per_step, "avg_launch_ms": kernels[dom]["avg_ms"],
                "share_of_step": dom_ms_per_step / max(step_ms_instr, 1e-9), "peak_source": peak_src}
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
    e2e_value = ps_total / (tmax(max(e0.elapsed_time(e1), 1e3 * wall_e2e)) / 1e3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, kind, sample = cpu_baseline_sample(cfg)
        cores, model = cpu_info()
        cpu = {"value": v, "unit": "particle-substeps/s", "cores": 1, "kind": kind,
               "sample": sample + f"; host {model}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "particle-substeps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded jittered lattices, seeding.hpp algorithm)",
            "env_steps_per_s": env_steps,
            "per_gpu": {"particle_substeps_per_s": value / world, "env_steps_per_s": env_steps / world},
            "config": {"workload": workload + (" [deterministic mode]" if args.deterministic else ""),
                       "envs_total": envs_global, "envs_per_gpu_rank0": n_envs,
                       "particles_per_gpu_rank0": n_part, "substeps_per_env_step": S, "dt": scene.dt,
                       "parallelism": f"env-sharded x{world} ({scaling} scaling, no data-path collective)",
                       "l2": "inputs larger than L2 (particle state 2 x %.2f GB)" % (n_part * 116 / 1e9)
                       if n_part * 116 > 200e6 else "state fits L2 (small config: launch/latency bound)"},
            "roofline": roofline,
            "roofline_path": roofline_path,
            "kernels": kernels,
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": {"value": e2e_value, "unit": "particle-substeps/s",
                    "h2d_bytes_per_step": nb * C.sizeof(abi.Body), "d2h_bytes_per_step": nb * 48 + C.sizeof(rep)},
            "cpu_baseline": cpu,
            "setup_s": setup_s,
            "stats": {"particle_substeps": stats.particle_substeps, "env_steps": stats.env_steps,
                      "exchange": "msim_gpu_step_stats (device reduction + NCCL all-reduce on the library stream)"
                      if libstats else "torch.distributed all_reduce"},
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
    ap.add_argument("--envs", type=int, default=None,
                    help="B / C / D: global env count, sharded over the GPUs (default D 1024, B 128, C 32)")
    ap.add_argument("--weak", action="store_true", help="every rank owns --envs envs (weak scaling)")
    ap.add_argument("--config", choices=["A", "B", "C", "D", "E"], default="D", help="workload (SURVEY.md App. B)")
    ap.add_argument("--clay-only", action="store_true",
                    help="B / C / E: the reference's von Mises clay instead of sand / water / mixed")
    ap.add_argument("--deterministic", action="store_true",
                    help="msim_gpu_set_deterministic: bit-reproducible runs (int64 fixed-point sums)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--traffic", type=float, default=None, help="ncu dram bytes per launch of the dominant kernel")
    args = ap.parse_args()
    if args.envs is None:
        args.envs = DEFAULT_ENVS.get(args.config, 1)
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
