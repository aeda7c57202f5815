#!/usr/bin/env python
"""Benchmark of the D3Q19 LBGK patch solver hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--precision fp64|fp32]
                    [--workload ldc256|weak384|strong768|patchy64|ldc32] [--impl product|reference]

One "step" = one LBM time step of the whole hot path (fused pull/BB/collide
sweep over every patch + the ghost exchange) on the lid-driven cavity.
Default N = 1 workload: BASELINE configs[1], LDC 256^3 fp64, one patch.
N > 1 (torchrun, one rank per GPU, NCCL): weak scaling of the same 256^3 brick
per GPU (process grid 1x1x2 / 1x2x2 / 2x2x2), ghost exchange over NCCL
overlapped with the interior sweep.  Prints ONE JSON line on rank 0.

value  = fluid lattice cell updates of all ranks / max-over-ranks device time
         (CUDA events on the library's compute stream), in MFLUPS.
e2e    = same metric through the C ABI with host buffers: set_pdfs (H2D of the
         whole state from pinned memory) + K steps + get_macroscopic (D2H).
roofline = the sweep kernel: algorithmic bytes 2*19*sizeof(real) per fluid cell
          / its average launch time, against MEASURED_PEAKS.json.
cpu_baseline = the CPU oracle (oracle/, test infrastructure) on a bounded slab
         sample of the same cavity, all host cores (rank 0, N = 1 only).
--impl reference: the oracle itself as the reference arm (rank 0 only).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import psutil  # noqa: E402

METRIC = "MFLUPS (whole job); % of B200 HBM roofline"
WORKLOADS = {
    # name: (per-GPU brick or global domain, patch, kind)
    "ldc32": ((32, 32, 32), (32, 32, 32), "fixed"),
    "ldc256": ((256, 256, 256), (256, 256, 256), "weak"),
    "weak384": ((384, 384, 384), (384, 384, 384), "weak"),
    "strong768": ((768, 768, 768), (384, 384, 384), "strong"),
    "patchy64": ((384, 384, 384), (64, 64, 64), "weak"),
}
PROC_GRID = {1: (1, 1, 1), 2: (1, 1, 2), 4: (1, 2, 2), 8: (2, 2, 2)}


def env_int(name, default):
    v = os.environ.get(name)
    return int(v) if v not in (None, "") else default


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as fh:
                for line in fh:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
            os.unlink(self.path)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        under = [v for v in sm if smax and v >= 0.5 * max(smax)] or sm
        return {"sm_mhz": statistics.median(under) if under else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons, "samples": len(rows)}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_sample(nx, ny, target_s, threads):
    """Time the CPU oracle (as it stands) on an nx x ny x Z slab of the lid-driven
    cavity (same cross-section and per-cell work), Z and steps sized to ~target_s."""
    import oracle
    from paper_1007_1388_b200 import inputs
    z, steps = 4, 1
    while True:
        n = (nx, ny, z)
        fl, wu = inputs.ldc_flags(n)
        f0 = inputs.noise_pdfs(n)
        t0 = time.perf_counter()
        oracle.run(f0, fl, wu, inputs.LDC_OMEGA, steps, nthreads=threads)
        dt = time.perf_counter() - t0
        if dt >= 0.7 * target_s or (z >= 256 and steps >= 64):
            cells = nx * ny * z
            return {"value": cells * steps / dt / 1e6, "unit": "MFLUPS", "cores": threads, "kind": "oracle",
                    "sample": f"oracle.run on a {nx}x{ny}x{z} LDC slab (lid on top), {steps} step(s), "
                              f"fp64, {threads} OpenMP threads, {dt:.2f} s"}
        scale = max(1.2, min(16.0, 1.05 * target_s / max(dt, 1e-3)))
        if z * scale <= 256:
            z = int(z * scale)
        else:  # z capped: the steps take the rest of the factor
            rest = z * scale / 256
            z = 256
            steps = max(steps + 1, int(steps * rest))


def run_reference(args):
    """Reference arm: the oracle on the same workload, each step one oracle time step
    over a bounded slab sample of it (rank 0 only)."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    import oracle
    from paper_1007_1388_b200 import inputs
    dom = WORKLOADS[args.workload][0]
    threads = cpu_cores()
    oracle.max_threads()
    # calibrate planes per step so that (K + W) steps take <= ~150 s
    budget = 150.0 / max(1, args.steps + args.warmup)
    z = 2
    while True:
        n = (dom[0], dom[1], z)
        fl, wu = inputs.ldc_flags(n)
        src = inputs.noise_pdfs(n)
        dst = np.zeros_like(src)
        t0 = time.perf_counter()
        oracle.step_slab(src, dst, fl, wu, inputs.LDC_OMEGA, 0, z, nthreads=threads)
        dt = time.perf_counter() - t0
        if dt * 2 > budget or z >= dom[2]:
            break
        z = min(dom[2], z * 2)
    for _ in range(args.warmup):
        oracle.step_slab(src, dst, fl, wu, inputs.LDC_OMEGA, 0, z, nthreads=threads)
        src, dst = dst, src
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.step_slab(src, dst, fl, wu, inputs.LDC_OMEGA, 0, z, nthreads=threads)
        src, dst = dst, src
    dt = time.perf_counter() - t0
    cells = dom[0] * dom[1] * z
    value = cells * args.steps / dt / 1e6
    sample = f"each step = one oracle time step on a {dom[0]}x{dom[1]}x{z} slab of the {args.workload} cavity"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "MFLUPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.workload, "domain": list(dom), "sample_planes": z},
            "cpu_baseline": {"value": value, "unit": "MFLUPS", "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "MFLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    emit(line)
    return 0


_JSON_OUT = None  # the process's original stdout (see __main__)


def emit(line):
    """The one JSON line -- the only thing this program writes to its stdout."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--precision", choices=("fp64", "fp32"), default="fp64")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default=None)
    ap.add_argument("--impl", choices=("product", "reference"), default="product")
    ap.add_argument("--overlap", type=int, default=1)
    ap.add_argument("--graphs", type=int, default=1)
    ap.add_argument("--layout", choices=("ab", "aa"), default="ab")
    ap.add_argument("--exchange", choices=("fused", "nccl"), default="fused",
                    help="fused: sweep stores into neighbour ghosts (NVLink peer stores across GPUs); "
                         "nccl: pack -> NCCL send/recv -> unpack")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--proc-grid", default="", help="px,py,pz (default: split z, then y, then x)")
    ap.add_argument("--repeat", type=int, default=1, help="timed regions of K steps; the median is reported")
    args = ap.parse_args()
    if args.workload is None:
        args.workload = "ldc256"
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if args.exchange == "nccl":
        os.environ["LBM_EXCHANGE"] = "nccl"
    from paper_1007_1388_b200 import inputs, lbm

    prec = lbm.LBM_FP64 if args.precision == "fp64" else lbm.LBM_FP32
    esize = 8 if prec == lbm.LBM_FP64 else 4
    brick, patch, kind = WORKLOADS[args.workload]
    pgrid = PROC_GRID.get(world, (1, 1, world))
    if args.proc_grid:  # e.g. "2,1,1": exercise the x split of the 8-GPU grid on 2 GPUs
        pgrid = tuple(int(v) for v in args.proc_grid.split(","))
        assert len(pgrid) == 3 and pgrid[0] * pgrid[1] * pgrid[2] == world, "proc grid must multiply to N"
    if kind == "weak":
        domain = tuple(brick[a] * pgrid[a] for a in range(3))
    else:
        domain = brick
    nccl_id = None
    if world > 1:
        obj = [lbm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    L = lbm.Lattice(domain, patch, inputs.LDC_OMEGA, prec, device=local, rank=rank, nranks=world,
                    proc_grid=pgrid, nccl_id=nccl_id, overlap=args.overlap, use_graphs=args.graphs,
                    layout=lbm.LBM_LAYOUT_AA if args.layout == "aa" else lbm.LBM_LAYOUT_AB)
    fl, wu = inputs.ldc_flags(domain)
    L.set_flags(fl, wu)
    del fl
    L.init_noise(inputs.NOISE_SEED)
    info0 = L.info()
    fluid_local = info0["fluid_cells_local"]
    fluid_global = info0["fluid_cells_global"]

    stream = torch.cuda.ExternalStream(L.stream(), device=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    # warm-up (also captures the CUDA graphs)
    L.step(args.warmup)
    barrier()
    # ---- timed region (device-timed, inputs resident in HBM; production path:
    # CUDA-graph step pairs, no per-phase events)
    # --repeat R (median of 3): R timed regions of exactly K steps each,
    # the median reported; default 1.
    runs_ms, runs_launches = [], []
    with ClockSampler(local) as clk:
        for _ in range(max(1, args.repeat)):
            launches0 = L.info()["kernel_launches"]
            start = torch.cuda.Event(enable_timing=True)
            end = torch.cuda.Event(enable_timing=True)
            barrier()
            start.record(stream)
            L.step_async(args.steps)
            end.record(stream)
            L.synchronize()
            barrier()
            ms = start.elapsed_time(end)
            info = L.info()
            launches = info["kernel_launches"] - launches0
            t = torch.tensor([ms], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            runs_ms.append(float(t.item()))
            runs_launches.append(launches)
    # the median region (roofline and value from the same region)
    mid = sorted(range(len(runs_ms)), key=lambda i: runs_ms[i])[(len(runs_ms) - 1) // 2]
    ms_max = runs_ms[mid]
    launches = runs_launches[mid]
    value = fluid_global * args.steps / (ms_max / 1e3) / 1e6

    # ---- per-phase breakdown: a second pass of the same K steps with library
    # CUDA events around every launch (on the stream each kernel runs on)
    L.set_timing(True)
    L.step(args.steps)
    phases = L.phase_ms()
    L.set_timing(False)

    # ---- roofline of the dominant kernel (the sweep): algorithmic bytes per launch / avg launch time
    peak, peak_src = load_peaks()
    alg_bytes = 2 * 19 * esize * fluid_local
    exchange_launches = phases["pack"][1] + phases["unpack"][1] + phases["sweep_shell"][1]
    if exchange_launches == 0:
        # the sweep and (two grids) its bounce-back list kernel, nothing else: the
        # timed region itself gives the (conservative, gap-inclusive) time per sweep
        sweep_avg_ms = ms_max / args.steps
        method = (f"timed region / K ({launches / args.steps:g} launches per step: the sweep"
                  + (" + its bounce-back list kernel" if launches > args.steps else "")
                  + "; max over ranks, median region)")
    else:
        sweep_ms = sum(phases[p][0] for p in ("sweep", "sweep_shell", "sweep_interior"))
        sweep_n = max(phases["sweep"][1], phases["sweep_interior"][1], 1)
        sweep_avg_ms = sweep_ms / sweep_n
        method = "per-launch CUDA events, second pass of K steps (shell + interior launches summed)"
    achieved = alg_bytes / (sweep_avg_ms / 1e3) / 1e9 if sweep_avg_ms > 0 else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": None,
                "kernel": "sweep_kernel", "bytes_per_launch": alg_bytes, "avg_launch_ms": sweep_avg_ms,
                "method": method, "peak_source": peak_src,
                "phase_ms_per_step": {k: (v[0] / v[1] if v[1] else 0.0) for k, v in phases.items() if v[1]}}
    prof = os.path.join(ROOT, "profiles", f"traffic_{args.workload}_{args.precision}.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            tr = json.load(fh)
        roofline["traffic"] = tr.get("dram_bytes_per_launch")
        if tr.get("gpu_time_us"):  # the ncu DRAM GB/s beside the algorithmic one
            roofline["ncu_dram_gbs"] = tr["dram_bytes_per_launch"] / (tr["gpu_time_us"] * 1e-6) / 1e9
    # against the 8 TB/s data-sheet figure
    roofline["frac_spec"] = roofline["achieved"] / 8000.0 if roofline["achieved"] else None

    # ---- end-to-end through the C ABI with host buffers
    e2e = None
    e2e_skip = None
    if not args.no_e2e:
        # pinned host state of every rank on this node must fit in host memory
        sx, sy, sz = L.owned_shape
        ncell = sx * sy * sz
        need = ncell * (19 + 4) * 8 * int(os.environ.get("LOCAL_WORLD_SIZE", world))
        avail = psutil.virtual_memory().available
        verdict = [None if need <= 0.8 * avail else
                   f"host state {need / 1e9:.1f} GB (pinned, all ranks) > 80% of available host memory "
                   f"{avail / 1e9:.1f} GB"]
        if world > 1:
            dist.broadcast_object_list(verdict, src=0)
        e2e_skip = verdict[0]
    if e2e_skip:
        e2e = {"value": None, "unit": "MFLUPS", "skipped": e2e_skip}
    elif not args.no_e2e:
        # page-locked in place (cudaHostRegister): torch's pinned allocator rounds
        # up to powers of two (68 GB of 768^3 state would pin 128 GB)
        host_f = np.empty((sz, sy, sx, 19), np.float64)
        host_rho = np.empty((sz, sy, sx), np.float64)
        host_u = np.empty((sz, sy, sx, 3), np.float64)
        cudart = torch.cuda.cudart()
        for a in (host_f, host_rho, host_u):
            a.fill(0.0)  # fault the pages in before registering
            if int(cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)) != 0:
                raise RuntimeError("cudaHostRegister failed")
        L.init_noise(inputs.NOISE_SEED)
        L.get_pdfs(host_f)  # the user's input state, in pinned host memory
        barrier()
        t0 = time.perf_counter()
        L.set_pdfs(host_f)
        t1 = time.perf_counter()
        L.step(args.steps)
        t2 = time.perf_counter()
        L.get_macroscopic(host_rho, host_u)
        barrier()
        e2e_s = time.perf_counter() - t0
        e2e_parts = {"set_pdfs_s": t1 - t0, "steps_s": t2 - t1, "get_macroscopic_s": time.perf_counter() - t2}
        tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
        e2e = {"value": fluid_global * args.steps / e2e_s / 1e6, "unit": "MFLUPS",
               "h2d_bytes_per_step": host_f.nbytes * world / args.steps,
               "d2h_bytes_per_step": (host_rho.nbytes + host_u.nbytes) * world / args.steps,
               "job": "set_pdfs(host state) + lbm_step(K) + get_macroscopic(host)", "rank0_parts": e2e_parts}
        for a in (host_f, host_rho, host_u):
            cudart.cudaHostUnregister(a.ctypes.data)
        del host_f, host_rho, host_u

    # ---- cpu baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            cpu = oracle_sample(brick[0], brick[1], args.cpu_seconds, min(cpu_cores(), oracle.max_threads()))
        except Exception as exc:  # the oracle is test infrastructure; never fail the bench on it
            cpu = {"value": None, "unit": "MFLUPS", "cores": 0, "kind": "oracle", "sample": f"failed: {exc}"}

    clocks = clk.summary()
    from paper_1007_1388_b200 import model
    est = model.b200_step_estimate(L.owned_shape, info["proc_coord"], pgrid, esize, peak,
                                   overlap=bool(args.overlap))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "MFLUPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak" if kind in ("weak", "fixed") else "strong", "vs_baseline": None,
            "dtype": "f64" if esize == 8 else "f32", "data": "synthetic",
            "config": {"workload": args.workload, "domain": list(domain), "patch": list(patch),
                       "proc_grid": list(pgrid), "parallelism": f"block-decomposition x{world}",
                       "fluid_cells": fluid_global, "mflups_per_gpu": value / world,
                       "omega": inputs.LDC_OMEGA, "lid_u": inputs.LDC_U, "init": "dyadic noise seed 1388",
                       "overlap": bool(args.overlap), "graphs": bool(args.graphs), "layout": args.layout,
                       "exchange": ("none" if not (info["halo_bytes_remote_per_step"] or
                                                   info["halo_bytes_local_per_step"]) else
                                    "fused NVLink stores" if info["exchange_fused"] else
                                    "nccl send/recv" if info["nccl_ranks"] > 0 else "same GPU only"),
                       "same_gpu_exchange": ("direct ghost stores" if info["local_direct"] else
                                             "ghost copies" if info["halo_bytes_local_per_step"] else "none"),
                       "l2": f"no flush: PDF state {2 * 19 * esize * fluid_local / 1e9:.2f} GB/GPU >> 126 MB L2",
                       "halo_bytes_remote_per_step": info["halo_bytes_remote_per_step"],
                       "row_pitch_elems": info["row_pitch_elems"], "align_bytes": info["align_bytes"],
                       "timed_regions_ms": runs_ms},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "env": environment(),
            "model": {"source": "paper_1007_1388_b200/model.py (P:577-613 re-parameterised: HBM roofline + "
                                "NVLink 770 GB/s halo)", **est},
        }
        emit(line)
    L.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def environment() -> dict:
    """GPU, driver, CUDA, NCCL and host CPU of this run (SURVEY 8(d) report record)."""
    import platform
    import torch
    env = {"gpu": torch.cuda.get_device_name(), "cuda_runtime": torch.version.cuda, "torch": torch.__version__,
           "host_cpu": platform.processor() or platform.machine(), "host_cores": len(os.sched_getaffinity(0))}
    try:
        env["nccl"] = ".".join(str(v) for v in torch.cuda.nccl.version())
    except Exception:
        env["nccl"] = None
    try:
        import pynvml
        pynvml.nvmlInit()
        env["driver"] = pynvml.nvmlSystemGetDriverVersion()
        pynvml.nvmlShutdown()
    except Exception:
        env["driver"] = None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    env["host_cpu"] = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return env


if __name__ == "__main__":
    # Libraries that print to the C stdout (NCCL's version banner at communicator
    # init) must not precede the JSON line: fd 1 goes to stderr, the line to the
    # original stdout.
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    sys.exit(main())
