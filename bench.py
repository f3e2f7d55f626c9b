#!/usr/bin/env python
"""Benchmark of the B200 adaptive-BDDC hot path (one JSON line on rank 0).

A *step* is one pass of the hot path over one instance of the workload:
leaf factorization + interface Schur complements, adaptive face
eigenproblems, constraint selection, transformed preconditioner (leaf fronts +
root) and the PCG solve to 1e-8 -- i.e. the metric's "setup + solve".  The
workload defaults to BASELINE.json configs[2] (cfg3: 80^3 Poisson, 8^3
substructures, k = exp(2z), adaptive tau=5), the largest configuration that
the reference runs on one GPU (cfg5 is the 8-GPU one); `--config 1..5`
selects another.  The host-side input (mesh, assembly, globs) is built once
and uploaded before timing.  `value` is free dofs / device seconds per step,
summed over ranks; `e2e` repeats the step through the C ABI with the
host->device upload of the inputs and the device->host copy of the solution
inside the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

N > 1 (torchrun, one process per GPU) runs the sharded engine on the SAME
problem ("strong" scaling, the way BASELINE.json shards cfg5 over 8 GPUs):
substructures and face pairs partitioned over the ranks by a 3D block
partition (paper_0910_5863_b200/shard.py), NCCL send/recv for the interface
halo and the ghost Schur complements, an all-reduce of the dot-product
partials and of the root.  `--weak` grows the lattice with N along x instead
(the config's lattice per GPU, same coefficient rule); `--replicas` runs N
independent copies of the N=1 workload.

CPU legs (oracle/, the reference restated in numpy/scipy; the C++ reference
needs Eigen and cannot be built here): `cpu_baseline` times
the oracle single-threaded (the reference is serial) and `--impl reference`
times it on all host cores (face pairs in worker processes), both on a
BOUNDED SAMPLE of the workload -- the same config restricted to a smaller
substructure lattice with the same substructure size, coefficient rule,
constraints and tolerances (SAMPLE_LATTICE) -- reported in the metric's unit
(free DOF/s of the sample).  The oracle's per-dof cost grows with the
lattice (more pairs per substructure, more iterations, a larger coarse
factorization), so the sample overstates the CPU's full-size throughput.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIG_MODES = {1: ("c+e+f", 10.0, 15, False), 2: ("adaptive", 10.0, 10, False),
                3: ("adaptive", 5.0, 15, False), 4: ("adaptive", 10.0, 15, True),
                5: ("adaptive", 10.0, 15, False)}
CONFIG_NAMES = {1: "cfg1: Poisson 24^3, 3^3 subdomains, c+e+f",
                2: "cfg2: Poisson 24^3, 3^3 subdomains, 1e6 z-channels p=0.1, adaptive tau=10 max 10",
                3: "cfg3: Poisson 80^3, 8^3 subdomains, k=exp(2z), adaptive tau=5 max 15",
                4: "cfg4: elasticity 48^3, 6^3 subdomains, 20 spheres E=1e4, c+e+f + adaptive tau=10 max 15",
                5: "cfg5: elasticity 96^3, 12^3 subdomains, layered E 1/1e5, adaptive tau=10 max 15"}
METRIC = "adaptive-BDDC setup+solve throughput (free DOF/s)"
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


FP64_PEAK_TFLOPS = 35.47  # cuBLAS DGEMM 8192^3 on this pool's B200 (profiles/r01_fp64_peak.txt)
FP64_DMMA_PEAK_TFLOPS = 36.9  # mma.sync m16n8k16 f64 microbenchmark, same file


def measured_traffic(config):
    """DRAM bytes (read + write) of one leaf factorization and of one Schur +
    preconditioner apply, from the ncu capture committed under profiles/
    (tools/ncu_traffic.py); {} when this config was not captured."""
    data, name = None, None
    for name in ("r02_traffic.json", "r01_traffic.json"):  # newest capture that holds this config
        try:
            with open(os.path.join(REPO, "profiles", name)) as f:
                data = json.load(f)
        except OSError:
            continue
        if any(("cfg%d_%s" % (config, ph)) in data for ph in ("leaf", "apply")):
            break
        data = None
    if data is None:
        return {}
    out = {}
    for phase in ("leaf", "apply"):
        rec = data.get("cfg%d_%s" % (config, phase))
        if rec:
            out[phase] = rec["dram_bytes_read"] + rec["dram_bytes_write"]
            # the leaf roofline is the batched partial Cholesky alone: its own launch
            # (k_chol_dag), not the assembly, zero-fill and copies of the phase
            chol = [v for k, v in rec.get("by_kernel_bytes", {}).items() if k.endswith("k_chol_dag")]
            if phase == "leaf" and chol:
                out["leaf_phase"] = out["leaf"]
                out["leaf"] = sum(chol)
    if out:
        out["source"] = ("profiles/%s (ncu dram__bytes_{read,write}.sum: the k_chol_dag launch of one leaf "
                         "factorization; every launch of one Schur + preconditioner apply)" % name)
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        if os.environ.get("BENCH_CLOCK_MS") == "0":  # diagnostics only: no sampler
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", os.environ.get("BENCH_CLOCK_MS", "20")],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        """Median SM clock and throttle reasons over the samples taken in
        [t0, t1] (the timed region); a timed region shorter than a few sampling
        periods falls back to every loaded sample of the run (warm-up, timed and
        e2e steps), and `window` says which."""
        inside = [ln for t, ln in self.lines if t0 is None or t0 <= t <= t1]
        out = self._summarise(inside)
        out["window"] = "timed"
        if out["samples"] < 3:
            out = self._summarise([ln for _, ln in self.lines])
            out["window"] = "whole run (timed region shorter than the sampling period)"
        return out

    def _summarise(self, lines):
        sm, mx, reasons = [], 0.0, set()
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                bits = int(parts[2], 16) if parts[2].startswith("0x") else int(parts[2])
            except ValueError:
                continue
            mx = max(mx, m)
            if bits & 0x1:  # idle sample
                continue
            sm.append(s)
            for b, name in REASONS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist_mod
        backend = "nccl" if args.impl != "reference" else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist_mod.init_process_group(backend=backend)
        dist = dist_mod
    return world, rank, local, dist


def max_over_ranks(dist, value: float, device=None) -> float:
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist, device=None):
    if dist is not None:
        if device is not None:
            dist.barrier(device_ids=[device])
        else:
            dist.barrier()


# Sample lattice of the CPU legs per config (same substructure size): about
# 10-30 s of single-thread oracle work on this pool's hosts.
SAMPLE_LATTICE = {1: (3, 3, 3), 2: (3, 3, 3), 3: (3, 3, 3), 4: (2, 2, 2), 5: (2, 2, 2)}
CONFIG_GEOMETRY = {1: ((3, 3, 3), 8, 1), 2: ((3, 3, 3), 8, 1), 3: ((8, 8, 8), 10, 1), 4: ((6, 6, 6), 8, 3),
                   5: ((12, 12, 12), 8, 3)}


def free_dofs_of(lattice, epe, comps):
    """Free dofs of a structured cube with Dirichlet on x=0 (all components)."""
    nx, ny, nz = (l * epe + 1 for l in lattice)
    return (nx - 1) * ny * nz * comps


def workload_config(cfg_id, seed, world=1, sharded=False, replicas=False, weak=False):
    """The `config` object of both arms (identical dicts for the same run)."""
    lat, epe, comps = CONFIG_GEOMETRY[cfg_id]
    if sharded and weak:
        lat = (lat[0] * world, lat[1], lat[2])
    return {"workload": CONFIG_NAMES[cfg_id] + (
                " per GPU; lattice %dx%dx%d over %d GPUs" % (lat + (world,)) if sharded and weak else
                "; sharded over %d GPUs" % world if sharded else ""),
            "config": cfg_id, "seed": seed, "lattice": list(lat), "elements_per_substructure_edge": epe,
            "free_dofs": free_dofs_of(lat, epe, comps),
            "parallelism": ("sharded%d (NCCL: interface exchange, dot products, root)" % world if sharded
                            else "replicas%d" % world if world > 1 else "single GPU")}


def oracle_sample_step(cfg_id, seed, workers):
    """One oracle setup+solve on the sample lattice: (seconds, free dofs, row).
    The input (mesh, assembly, globs) is built outside the timed region, as on
    the GPU arm."""
    from oracle.experiment import baseline_config, build_pipeline
    from oracle.parallel import solve_item_parallel
    cfg = baseline_config(cfg_id, seed, subdomains=SAMPLE_LATTICE[cfg_id])
    p = build_pipeline(cfg.spec)
    t0 = time.perf_counter()
    row = solve_item_parallel(p, cfg.mode, cfg.tau, cfg.max_vectors, cfg.base_faces, workers)
    return time.perf_counter() - t0, p.dmap.free_count, row


def sample_text(cfg_id, workers, seconds=None):
    lat = SAMPLE_LATTICE[cfg_id]
    full = CONFIG_GEOMETRY[cfg_id][0]
    return ("cfg%d restricted to a %dx%dx%d substructure lattice (%d of %d substructures, same substructure "
            "size, coefficient rule, constraints and tolerances): one full oracle setup+solve "
            "(HarmonicExtension, face eigenproblems, enrichment, change of variables, preconditioner, PCG)%s, "
            "%s; DOF/s of the sample" % (
                cfg_id, lat[0], lat[1], lat[2], lat[0] * lat[1] * lat[2], full[0] * full[1] * full[2],
                " in %.1f s" % seconds if seconds is not None else "",
                "single-threaded (BLAS 1 thread, as the serial reference)" if workers <= 1 else
                "face pairs over %d worker processes, BLAS on all threads" % workers))


def cpu_baseline_single(cfg_id, seed):
    """Single-thread oracle on the sample (in-process, BLAS limited to 1 thread)."""
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):
        dt, free, row = oracle_sample_step(cfg_id, seed, 1)
    return {"value": free / dt, "unit": "DOF/s", "cores": 1, "kind": "port",
            "sample": sample_text(cfg_id, 1, dt), "sample_free_dofs": free, "sample_seconds": dt,
            "sample_iterations": row.iterations}


def reference_arm(args):
    world, rank, local, dist = dist_setup(args)
    if rank != 0:
        return 0
    cfg_id = args.config
    cores = os.cpu_count() or 1
    times = []
    row = None
    for i in range(args.warmup + args.steps):
        dt, free, row = oracle_sample_step(cfg_id, args.seed, cores)
        if i >= args.warmup:
            times.append(dt)
    sec = sum(times) / len(times)
    value = free / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong" if world > 1 and not (args.weak or args.replicas) else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded coefficient field)",
        "config": workload_config(cfg_id, args.seed, world, world > 1 and not args.replicas, args.replicas,
                                  args.weak),
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": cores, "kind": "port",
                         "sample": sample_text(cfg_id, cores), "sample_free_dofs": free},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "iterations": row.iterations, "kappa": row.kappa, "constraint_rows": row.constraint_rows,
        "omega_tilde": None if math.isnan(row.omega_tilde) else row.omega_tilde,
        "l2": "n/a (CPU)",
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--seed", type=int, default=20091030)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--apply-reps", type=int, default=10, help="operator applications timed for the rooflines")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent copies instead of sharding")
    ap.add_argument("--weak", action="store_true", help="N > 1: lattice grows with N (weak scaling)")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)

    world, rank, local, dist = dist_setup(args)
    import paper_0910_5863_b200 as pb
    lib = pb.load_library()
    if lib.bddc_b200_device_count() < 1:
        raise SystemExit("no CUDA device visible: the B200 path has no CPU fallback")
    pb._check(lib.bddc_b200_set_device(local))
    import torch
    torch.cuda.set_device(local)
    mode, tau, maxv, base_faces = CONFIG_MODES[args.config]
    sharded = world > 1 and not args.replicas
    t_in = time.perf_counter()
    if sharded:
        base = pb.BDDC(config=args.config, seed=args.seed).lattice()
        lattice = (base[0] * world, base[1], base[2]) if args.weak else base
        b = pb.BDDC(config=args.config, seed=args.seed, subdomains=lattice if args.weak else None)
        nid = [pb.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        b.shard(rank, world, backend="nccl", nccl_id=nid[0])
    else:
        b = pb.BDDC(config=args.config, seed=args.seed)
        lattice = b.lattice()
    input_seconds = time.perf_counter() - t_in
    st = b.structure()
    free = st["free_dofs"]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    def do_step(e2e=False, u=None):
        flush.zero_()
        torch.cuda.synchronize()
        return b.step(mode, tau, maxv, base_faces=base_faces, e2e=e2e, u_free=u)

    clk = ClockSampler(local).__enter__()
    t_wait = time.perf_counter()
    while not clk.lines and clk.proc is not None and time.perf_counter() - t_wait < 3.0:
        time.sleep(0.01)  # nvidia-smi start-up: sample from the first step on
    t_w = time.perf_counter()
    for _ in range(args.warmup):
        t_w = time.perf_counter()
        do_step()
    # short steps (cfg1-2: a few ms, mostly host/launch latency) keep warming
    # for about one more second of steps so the host threads and caches settle;
    # the count is agreed over the ranks (sharded steps hold collectives)
    if args.warmup == 0:  # time one step so the settle count is based on a real step
        t_w = time.perf_counter()
        do_step()
    t_last = max_over_ranks(dist, time.perf_counter() - t_w, "cuda")
    settle = min(400, int(1.0 / max(t_last, 1e-3)))
    if os.environ.get("BENCH_SETTLE"):  # profiling runs (ncu launch lists): fixed count
        settle = int(os.environ["BENCH_SETTLE"])
    for _ in range(settle):
        do_step()
    barrier(dist, local)
    torch.cuda.synchronize()
    steps = []
    t_timed0 = time.perf_counter()
    for _ in range(args.steps):
        steps.append(do_step())
    torch.cuda.synchronize()
    t_timed1 = time.perf_counter()
    barrier(dist, local)
    dev_seconds = sum(s["seconds"] for s in steps)
    dev_seconds = max_over_ranks(dist, dev_seconds, "cuda")
    sec_per_step = dev_seconds / args.steps
    jobs = 1 if sharded else world  # sharded: one problem over all ranks
    value = jobs * free / sec_per_step
    # end to end through the C ABI with host buffers
    u = torch.empty(free, dtype=torch.float64, pin_memory=True).numpy()  # page-locked result buffer
    for _ in range(max(1, args.warmup // 2)):
        do_step(True, u)
    barrier(dist, local)
    e2e_steps = [do_step(True, u) for _ in range(args.steps)]
    e2e_sec = max_over_ranks(dist, sum(s["seconds"] for s in e2e_steps), "cuda") / args.steps
    launches = max_over_ranks(dist, float(sum(s["launches"] for s in steps)), "cuda")
    clk.__exit__(None, None, None)
    if rank != 0:
        return 0
    last = steps[-1]
    # roofline of the dominant tensor kernel: the batched leaf partial Cholesky
    peaks, peak_kind = measured_peaks()
    lf_t = statistics.median(s["leaf_factor_seconds"] for s in steps)
    lf_flops = last["leaf_flops"]
    achieved = lf_flops / lf_t / 1e12
    traffic = measured_traffic(args.config) if world == 1 else {}
    roof = {"kernel": "partial_cholesky (leaf fronts: A_II eliminated, S_s formed)", "bound": "tensor",
            "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic.get("leaf"),
            "peak_source": "measured cuBLAS DGEMM (MEASURED_PEAKS.json has bf16 only)",
            "flops_per_launch": lf_flops, "seconds_per_launch": lf_t,
            "share_of_step": lf_t / sec_per_step}
    if traffic.get("leaf_phase"):
        roof["traffic_leaf_phase"] = traffic["leaf_phase"]  # with assembly, zero-fill, S copy and rhs sweep
    # second roofline: the HBM-bound PCG iteration (Schur apply + both leaf
    # sweeps + root apply), algorithmic bytes over the device-timed PCG phase
    tm = b.times()
    pcg_it = max(int(tm["pcg_iterations"]), 1)
    pcg_achieved = tm["pcg_bytes_per_iteration"] * pcg_it / max(tm["pcg"], 1e-12) / 1e9
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    roof_pcg = {"kernel": "PCG iteration (S_s GEMV + leaf sweeps + root apply)", "bound": "hbm",
                "achieved": pcg_achieved, "peak": hbm_peak, "unit": "GB/s", "frac": pcg_achieved / hbm_peak,
                "traffic": traffic.get("apply"), "bytes_per_iteration": tm["pcg_bytes_per_iteration"],
                "iterations": pcg_it,
                "peak_source": peak_kind + " (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else peak_kind}
    if traffic:
        roof["traffic_source"] = roof_pcg["traffic_source"] = traffic["source"]
    # third and fourth rooflines: the preconditioner apply alone and the Schur
    # apply alone (device-resident vectors, CUDA events on the engine stream)
    ops = b.operator_times(args.apply_reps)
    pre_achieved = ops["precond_bytes"] / ops["precond"] / 1e9
    roof_pre = {"kernel": "BDDC preconditioner apply (restrict, leaf forward sweep, primal tree, root, leaf "
                          "backward sweep, prolong, copy sum)", "bound": "hbm", "achieved": pre_achieved,
                "peak": hbm_peak, "unit": "GB/s", "frac": pre_achieved / hbm_peak,
                "bytes_per_apply": ops["precond_bytes"], "seconds_per_apply": ops["precond"],
                "stages_s": {k: ops[k] for k in ("restrict", "leaf_fwd", "tree_fwd", "root", "tree_bwd",
                                                 "leaf_bwd", "prolong", "sum_copies")},
                "leaf_sweep_bytes": ops["leaf_sweep_bytes"],
                "leaf_fwd_gbs": ops["leaf_sweep_bytes"] / max(ops["leaf_fwd"], 1e-12) / 1e9,
                "leaf_bwd_gbs": ops["leaf_sweep_bytes"] / max(ops["leaf_bwd"], 1e-12) / 1e9,
                "reps": args.apply_reps}
    sch_achieved = ops["schur_bytes"] / ops["schur"] / 1e9
    roof_schur = {"kernel": "Schur apply (dense S_s GEMV + copy sum)", "bound": "hbm", "achieved": sch_achieved,
                  "peak": hbm_peak, "unit": "GB/s", "frac": sch_achieved / hbm_peak,
                  "bytes_per_apply": ops["schur_bytes"], "seconds_per_apply": ops["schur"]}
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline_single(args.config, args.seed)
    line = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "settle_steps": settle, "ms_per_step": sec_per_step * 1e3, "higher_is_better": True,
        "scaling": "strong" if sharded and not args.weak else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded coefficient field)",
        "config": workload_config(args.config, args.seed, world, sharded, args.replicas and world > 1, args.weak),
        "l2": "flushed (256 MiB write) before every step",
        "structure": {"free_dofs": free, "subdomains": st["subdomains"], "interface_dofs": st["interface_dofs"]},
        "setup_s": statistics.median(s["setup_seconds"] for s in steps),
        "solve_s": statistics.median(s["solve_seconds"] for s in steps),
        "iterations": last["iterations"], "kappa": last["kappa"], "constraint_rows": last["constraint_rows"],
        "omega_tilde": last["omega_tilde"], "input_build_s": input_seconds,
        "phases_s": {k: v for k, v in b.times().items() if k in ("analysis", "eigen", "preconditioner", "pcg",
                                                                   "leaf_factor")},
        "roofline": roof,
        "roofline_pcg": roof_pcg,
        "roofline_precond": roof_pre,
        "roofline_schur": roof_schur,
        "cpu_baseline": cpu,
        "e2e": {"value": jobs * free / e2e_sec, "unit": "DOF/s",
                "h2d_bytes_per_step": int(e2e_steps[-1]["h2d_bytes"]),
                "d2h_bytes_per_step": int(e2e_steps[-1]["d2h_bytes"]), "ms_per_step": e2e_sec * 1e3},
        "clocks": clk.summary(t_timed0, t_timed1),
        "step_ms": [round(s["seconds"] * 1e3, 3) for s in steps],
        "e2e_step_ms": [round(s["seconds"] * 1e3, 3) for s in e2e_steps],
        "gpu_launches": int(launches),  # max over ranks
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
