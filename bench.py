"""Benchmark of the B200 range march (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--impl reference]

Workload (default cfg4): BASELINE.json configs[3] -- 64 frequencies
log-spaced 50-500 Hz, 256 x 1024 complex128 grid, dr = 1 m; one bench
"step" = one range step of Eq. (4) over all frequencies on this job's GPUs
(frequencies sharded across ranks by the reference's static block law:
strong scaling, total work fixed).  Synthetic, seeded medium.

value    = grid-point range-steps/s (F * Ntheta * Nz * K / device time, max over
           ranks), inputs resident in HBM, one march of K steps per rank
           (a march is one CUDA graph; depth factorisation and starter prologue
           included in the timed region).
e2e      = the same metric through the C-ABI host entry point pe3d_march_host
           with pinned host buffers: starter + medium H2D, K steps, final
           slab + TL stack D2H, all inside the timed region.
roofline = dominant kernel, 32 algorithmic bytes per grid point per launch
           (16 B read + 16 B write) over its mean CUDA-event
           duration in a profiled march of the same K steps, against
           MEASURED_PEAKS.json hbm_gbs.
cpu_baseline = the CPU oracle port (oracle/pe3d_oracle.py, numpy, the
           reference's algorithm) on a bounded sample, processes over host
           cores like the reference's frequency_farm.
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
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "grid-point range-steps/sec"
UNIT = "gp-steps/s"
ALG_BYTES_PER_POINT = 32          # per kernel launch: 16 B read + 16 B write
STEP_BYTES_PER_POINT = 64         # both sweeps


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=1000)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--workload", default="cfg4", choices=["cfg1", "cfg2", "cfg4", "cfg5"])
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--shard-of", type=int, default=0,
                   help="diagnostic: march only rank 0's frequency block of an N-way split on this one GPU "
                        "(value then counts only that block's points)")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def workload(name, steps):
    from paper_1711_00005_b200 import configs
    cfg = configs.build(name, n_range=max(steps, 3))
    return cfg


def peaks():
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        d = json.loads(path.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------- CPU arms

def _oracle_job(args):
    name, freq, steps = args
    sys.path.insert(0, str(ROOT))
    from oracle import pe3d_oracle as O
    from paper_1711_00005_b200 import configs
    cfg = configs.build(name, n_range=max(steps, 3), frequencies=(freq,))
    t = time.perf_counter()
    O.run_frequency(cfg, freq, n_steps=steps)
    return time.perf_counter() - t


def _warm_worker(_):
    sys.path.insert(0, str(ROOT))
    from oracle import pe3d_oracle  # noqa: F401  (imports numpy and the oracle once per worker)
    from paper_1711_00005_b200 import configs  # noqa: F401
    return os.getpid()


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_sample(name, frequencies, sample_freqs, sample_steps):
    """Time the oracle port (the reference's algorithm in numpy) on the host
    cores: one process per frequency, like the reference's frequency_farm,
    as many frequencies as there are cores (at most the workload's).  The
    worker pool is started and warmed (imports) before the timed map."""
    import multiprocessing as mp
    cfg = workload(name, 3)
    freqs = list(frequencies)
    cores = host_cores()
    n = max(1, min(len(freqs), max(sample_freqs, cores)))
    idx = np.linspace(0, len(freqs) - 1, n).round().astype(int)
    picked = [freqs[i] for i in idx]
    procs = min(len(picked), cores)
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        pool.map(_warm_worker, range(procs))
        t = time.perf_counter()
        pool.map(_oracle_job, [(name, f, sample_steps) for f in picked], chunksize=1)
        wall = time.perf_counter() - t
    g = cfg.grid
    points = len(picked) * sample_steps * g.n_azimuth * g.n_depth
    return {"value": points / wall, "unit": UNIT, "cores": procs, "kind": "port",
            "sample": f"{name}: {len(picked)} of {len(freqs)} frequencies x {sample_steps} steps, "
                      f"{g.n_azimuth}x{g.n_depth} grid, oracle/pe3d_oracle.py (numpy), "
                      f"{procs} processes on {cores} host cores (spawned and warmed before timing), "
                      f"wall {wall:.1f} s"}


CPU_SAMPLES = {"cfg1": (1, 400), "cfg2": (1, 30), "cfg4": (16, 16), "cfg5": (1, 2)}


def run_reference_arm(a, rank, world):
    if rank != 0:
        return
    cfg = workload(a.workload, 3)
    freqs = cfg.source.frequencies
    nf, ns = CPU_SAMPLES[a.workload]
    for _ in range(max(0, min(a.warmup, 1))):
        _oracle_job((a.workload, freqs[0], 1))
    vals = []
    for _ in range(max(1, min(a.steps, 2))):
        vals.append(cpu_sample(a.workload, freqs, nf, ns))
    best = vals[-1]
    v = statistics.median([x["value"] for x in vals])
    g = cfg.grid
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * len(freqs) * g.n_azimuth * g.n_depth / v,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic",
        "config": {"workload": a.workload, "frequencies": len(freqs), "n_theta": g.n_azimuth,
                   "n_depth": g.n_depth, "parallelism": f"{best['cores']} host processes"},
        "cpu_baseline": {**best, "value": v},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm

def secondary_config(name, steps, local):
    """Device-time throughput of another BASELINE config on this GPU: one
    graph of `steps` steps, inputs resident, CUDA events (as the main line)."""
    import torch
    import ctypes as C
    from paper_1711_00005_b200 import _native
    from paper_1711_00005_b200.environment import gaussian_starter, wavenumber
    from paper_1711_00005_b200.marching import _grid_params, _local_column
    from paper_1711_00005_b200.operators import StepCoefficients
    cfg = workload(name, steps)
    grid, env, source, _ = cfg
    freqs = list(source.frequencies)
    k0s = [wavenumber(f, env.c0) for f in freqs]
    coeffs = _native.make_coeffs(k0s, [StepCoefficients.for_step(k0, grid.delta_r) for k0 in k0s])
    dev = torch.device("cuda", local)
    d_local = torch.from_numpy(np.ascontiguousarray(np.stack(
        [_local_column(env, grid, grid.r_start, k0) for k0 in k0s])).view(np.float64)).to(dev)
    d_u0 = torch.from_numpy(np.ascontiguousarray(np.stack(
        [gaussian_starter(grid, source, k0).values for k0 in k0s])).view(np.float64)).to(dev)
    d_final = torch.empty_like(d_u0)
    d_cl = torch.zeros(len(freqs), dtype=torch.int64, device=dev)
    tl = torch.empty((len(freqs), 2, grid.n_azimuth, grid.n_depth), dtype=torch.float64, device=dev)
    stream = torch.cuda.Stream(device=dev)
    h = _native.handle(local)

    def march():
        g = _grid_params(grid, len(freqs), steps, steps, 0, grid.r_start)
        _native.call("pe3d_march_device", h, g, coeffs, C.c_void_p(d_local.data_ptr()), C.c_void_p(d_u0.data_ptr()),
                     C.c_void_p(d_final.data_ptr()), C.c_void_p(tl.data_ptr()), None, C.c_void_p(d_cl.data_ptr()),
                     C.c_void_p(stream.cuda_stream))
    with torch.cuda.stream(stream):
        march()
        march()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        t0.record(stream)
        march()
        t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    pts = len(freqs) * grid.n_azimuth * grid.n_depth * steps
    return {"value": pts / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
            "l2": "field L2-resident (8 MiB)", "note": "BASELINE configs[1]; HBM roofline not meaningful"}


def run_gpu_arm(a, rank, world, local):
    import torch
    import ctypes as C
    from paper_1711_00005_b200 import _native, parallel
    from paper_1711_00005_b200.environment import gaussian_starter, wavenumber
    from paper_1711_00005_b200.marching import _grid_params, _local_column
    from paper_1711_00005_b200.operators import StepCoefficients

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = workload(a.workload, max(a.steps, a.warmup))
    grid, env, source, _ = cfg
    all_freqs = list(source.frequencies)
    shard_world = a.shard_of if (a.shard_of and world == 1) else world
    mine = parallel.rank_frequencies(all_freqs, rank, shard_world)
    F, NT, NZ = len(mine), grid.n_azimuth, grid.n_depth
    k0s = [wavenumber(f, env.c0) for f in mine]
    coeffs = _native.make_coeffs(k0s, [StepCoefficients.for_step(k0, grid.delta_r) for k0 in k0s])
    local_np = np.ascontiguousarray(np.stack([_local_column(env, grid, grid.r_start, k0) for k0 in k0s]))
    u0_np = np.ascontiguousarray(np.stack([gaussian_starter(grid, source, k0).values for k0 in k0s]))
    dev = torch.device("cuda", local)
    d_local = torch.from_numpy(local_np.view(np.float64)).to(dev)
    d_u0 = torch.from_numpy(u0_np.view(np.float64)).to(dev)
    d_final = torch.empty_like(d_u0)
    d_clamped = torch.zeros(F, dtype=torch.int64, device=dev)
    stream = torch.cuda.Stream(device=dev)
    h = _native.handle(local)
    lib = _native.load_library()
    stride = max(1, a.steps)          # TL of the starter and of the last step

    S_full = 1 + a.steps // stride
    tl = torch.empty((F, S_full, NT, NZ), dtype=torch.float64, device=dev)   # one buffer: graph cache key

    def march(n_steps, flags=0):
        g = _grid_params(grid, F, n_steps, stride, 0, grid.r_start, flags)
        _native.call("pe3d_march_device", h, g, coeffs, C.c_void_p(d_local.data_ptr()),
                     C.c_void_p(d_u0.data_ptr()), C.c_void_p(d_final.data_ptr()),
                     C.c_void_p(tl.data_ptr()), None,
                     C.c_void_p(d_clamped.data_ptr()), C.c_void_p(stream.cuda_stream))

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    # warm-up (W steps) and one untimed K-step march to build the cached graph
    with torch.cuda.stream(stream):
        march(a.warmup)
        march(a.steps)
    torch.cuda.synchronize()

    # ---- timed region: exactly K steps
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        with torch.cuda.stream(stream):
            start.record(stream)
            march(a.steps)
            end.record(stream)
        torch.cuda.synchronize()
    barrier()
    n_launch = C.c_int64(0)
    lib.pe3d_last_launches(h, C.byref(n_launch))      # kernels of the timed march (graph replay included)
    ms = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    total_points = (len(all_freqs) if shard_world == world else F) * NT * NZ * a.steps
    value = total_points / (ms / 1e3)

    # ---- per-kernel timing: the same K-step march with events per launch
    with torch.cuda.stream(stream):
        march(a.steps, flags=_native.FLAG_PROFILE)
    torch.cuda.synchronize()
    kms = (C.c_double * 3)()
    kn = (C.c_int32 * 3)()
    lib.pe3d_profile_last(h, kms, kn)
    per = {name: (kms[i] / max(kn[i], 1), kn[i]) for i, name in enumerate(("depth_sweep", "azimuth_sweep", "other"))}
    dom = max(("depth_sweep", "azimuth_sweep"), key=lambda k: per[k][0])
    peak, peak_kind = peaks()
    launch_bytes = ALG_BYTES_PER_POINT * F * NT * NZ
    achieved = launch_bytes / (per[dom][0] / 1e3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / f"traffic_{a.workload}.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get(dom)

    # ---- e2e through the host ABI entry point (pinned buffers)
    e2e = None
    if not a.no_e2e:
        S = 1 + a.steps // stride
        h_local = torch.from_numpy(local_np.view(np.float64)).pin_memory()
        h_u0 = torch.from_numpy(u0_np.view(np.float64)).pin_memory()
        h_final = torch.empty_like(h_u0).pin_memory()
        h_tl = torch.empty((F, S, NT, NZ), dtype=torch.float64).pin_memory()
        h_cl = torch.zeros(F, dtype=torch.int64).pin_memory()
        g = _grid_params(grid, F, a.steps, stride, 0, grid.r_start)

        def host_march():
            _native.call("pe3d_march_host", h, g, coeffs, C.c_void_p(h_local.data_ptr()),
                         C.c_void_p(h_u0.data_ptr()), C.c_void_p(h_final.data_ptr()), C.c_void_p(h_tl.data_ptr()),
                         None, C.c_void_p(h_cl.data_ptr()))
        host_march()
        barrier()
        t0 = time.perf_counter()
        host_march()
        wall = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([wall], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            wall = float(t.item())
        h2d = (h_local.numel() + h_u0.numel()) * 8 * world
        d2h = (h_final.numel() + h_tl.numel() + h_cl.numel()) * 8 * world
        e2e = {"value": total_points / wall, "unit": UNIT, "h2d_bytes_per_step": h2d / a.steps,
               "d2h_bytes_per_step": d2h / a.steps, "wall_s": wall,
               "path": "pe3d_march_host (C ABI, pinned host buffers; starter+medium in, final slab+TL out)"}

    # BASELINE configs[1] (cfg2, L2-resident) alongside, measured the same way
    secondary = None
    if rank == 0 and world == 1 and a.workload == "cfg4" and not a.no_cpu:
        secondary = {"cfg2": secondary_config("cfg2", 400, local)}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        nf, ns = CPU_SAMPLES[a.workload]
        cpu = cpu_sample(a.workload, all_freqs, nf, ns)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": a.workload, "frequencies": len(all_freqs), "frequencies_per_gpu": F,
                       "n_theta": NT, "n_depth": NZ, "delta_r": grid.delta_r, "parallelism": f"frequency-shard x{world}",
                       **({"emulated_shard_of": shard_world} if shard_world != world else {}),
                       "l2": "inputs larger than L2 (field 256 MiB per buffer at N=1)" if a.workload in ("cfg4", "cfg5")
                       else "field L2-resident", "march": f"one graph of {a.steps} steps"},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_source": peak_kind, "traffic": traffic,
                         "alg_bytes_per_launch": launch_bytes,
                         "kernel_ms": {k: v[0] for k, v in per.items()},
                         "step_hbm_frac": STEP_BYTES_PER_POINT * value / world / 1e9 / peak},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(n_launch.value),
            "clocks": clocks.summary(),
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_slab_arm(a, rank, world, local):
    """cfg5 on N GPUs: one grid, slab-decomposed; the two transposes per step
    are peer-direct stores over NVLink fused into the sweeps (NCCL
    all-to-all when the shape does not allow it)."""
    import torch
    import torch.distributed as dist
    from paper_1711_00005_b200 import slab
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = workload(a.workload, max(a.steps, a.warmup))
    grid = cfg.grid
    f = cfg.source.frequencies[0]
    slab.distributed_slab_march(cfg, f, device=local, n_steps=a.warmup)
    dist.barrier()
    transport = "peer" if slab.peer_transport_ok(grid, world) else "nccl"
    with ClockSampler(local) as clocks:
        res = slab.distributed_slab_march(cfg, f, device=local, n_steps=a.steps, transport=transport)
    t = torch.tensor([res.step_ms], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = grid.n_azimuth * grid.n_depth * a.steps / (ms / 1e3)
    if rank == 0:
        peak, kind = peaks()
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic",
            "config": {"workload": a.workload, "frequencies": 1, "n_theta": grid.n_azimuth, "n_depth": grid.n_depth,
                       "parallelism": f"slab x{world}: depth sweep on azimuth slabs, azimuth sweep on depth slabs, "
                                      + ("transposes fused into the sweeps as NVLink peer stores (CUDA IPC)"
                                         if transport == "peer" else "2 NCCL all-to-all per step")},
            "roofline": {"bound": "hbm+nvlink", "achieved": STEP_BYTES_PER_POINT * value / world / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": STEP_BYTES_PER_POINT * value / world / 1e9 / peak,
                         "peak_source": kind, "traffic": None},
            "cpu_baseline": None, "e2e": None, "gpu_launches": None, "clocks": clocks.summary()}), flush=True)
    dist.destroy_process_group()


def main():
    a = parse()
    rank, world, local = dist_env()
    if a.impl == "reference":
        run_reference_arm(a, rank, world)
        return
    if a.workload == "cfg5" and world > 1:
        run_slab_arm(a, rank, world, local)
        return
    run_gpu_arm(a, rank, world, local)


if __name__ == "__main__":
    main()
