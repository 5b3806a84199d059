"""Benchmark of the B200 range march (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--impl reference]

Workload (default cfg4): BASELINE.json configs[3] -- 64 frequencies
log-spaced 50-500 Hz, 256 x 1024 complex128 grid, dr = 1 m, TL every 100
steps (the config's output stride); one bench "step" = one range step of
Eq. (4) over all frequencies on this job's GPUs (frequencies sharded across
ranks by the reference's static block law: strong scaling, total work
fixed).  Synthetic, seeded medium.

value    = grid-point range-steps/s (F * Ntheta * Nz * K / device time, max over
           ranks), inputs resident in HBM, one march of K steps per rank
           (one CUDA graph; depth factorisation, starter prologue and the TL
           samples the config's stride falls on are inside the timed region).
e2e      = the same metric through the C-ABI host entry point pe3d_march_host
           with pinned host buffers: starter + medium H2D, K steps, final slab
           + TL stack D2H (streamed during the march), all inside the timed region.
e2e_dropin = through the reference-facing Python API frequency_farm(config,
           frequencies) (ref parallel.py:143-185): host-side starter and medium,
           the march, results in page-locked numpy arrays.
e2e_default_stride = e2e with TL every default_output_stride(n_range) steps
           (ref marching.py:139-141; 4 for cfg4): what run_frequency records
           when a config leaves the stride unset.
roofline = both sweeps, 32 algorithmic bytes per grid point per launch
           (16 B read + 16 B write) over the median CUDA-event
           duration of the steady-state launches of a profiled march of the same
           K steps (first and last two launches of each sweep excluded; no TL,
           no final slab), against MEASURED_PEAKS.json hbm_gbs; `kernel` is the
           slower sweep.  `traffic` = ncu DRAM bytes per launch from
           profiles/traffic_<workload>.json when its hash of the sweep kernels' sources matches.
cpu_baseline / --impl reference = the UNMODIFIED reference (baseline/_ref,
           the pip install of /root/reference) through its own frequency_farm
           on the host cores, bounded sample (oracle/ref_harness.py injects the
           BASELINE medium); the numpy oracle port when the reference is absent.
"""

from __future__ import annotations

import argparse
import hashlib
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
ALG_BYTES_PER_POINT = 32          # per sweep launch: 16 B read + 16 B write
STEP_BYTES_PER_POINT = 64         # both sweeps
L2_BYTES = 126 * 2 ** 20          # B200 L2


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=1000)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--workload", default="cfg4", choices=["cfg1", "cfg2", "cfg4", "cfg5"])
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-secondary", action="store_true")
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
    return configs.build(name, n_range=max(steps, 3))


def peaks():
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        d = json.loads(path.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


SWEEP_SOURCES = ("pe3d_depth.cu", "pe3d_ring.cu", "pe3d_device.cuh", "pe3d_internal.h")


def source_hash():
    """Hash of the sweep kernels' CUDA sources (stamps traffic files: a DRAM
    traffic capture stays valid while the kernels it measured are unchanged)."""
    h = hashlib.sha256()
    csrc = ROOT / "paper_1711_00005_b200" / "csrc"
    for name in SWEEP_SOURCES:
        h.update(name.encode())
        h.update((csrc / name).read_bytes())
    return h.hexdigest()[:16]


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
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.15)
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
            time.sleep(0.15)
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

def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


CPU_SAMPLES = {"cfg1": (1, 400), "cfg2": (1, 20), "cfg4": (16, 8), "cfg5": (1, 1)}


def _sample_freqs(freqs, n):
    idx = np.linspace(0, len(freqs) - 1, min(n, len(freqs))).round().astype(int)
    return [freqs[i] for i in idx]


def reference_sample(name, frequencies, repeats=1):
    """The unmodified reference's frequency_farm (fork workers = host cores)
    over a bounded sample of the workload; the numpy oracle port when the
    reference is not installed.  Returns the cpu_baseline record."""
    nf, ns = CPU_SAMPLES[name]
    cores = host_cores()
    picked = _sample_freqs(list(frequencies), max(nf, cores) if nf > 1 else nf)
    cfg = workload(name, ns)
    g = cfg.grid
    points = len(picked) * ns * g.n_azimuth * g.n_depth
    try:
        from oracle import ref_harness as H
        pe3d = H.import_reference()
        H.install_medium(pe3d, cfg)
        rcfg = H.ref_config(pe3d, cfg, picked)
        workers = min(cores, len(picked))
        small = workload(name, 1)
        H.install_medium(pe3d, small)
        pe3d.frequency_farm(H.ref_config(pe3d, small, picked[:workers]), picked[:workers], workers=workers)
        H.install_medium(pe3d, cfg)
        walls = []
        for _ in range(max(1, repeats)):
            t = time.perf_counter()
            rep = pe3d.frequency_farm(rcfg, picked, workers=workers, schedule="static")
            walls.append(time.perf_counter() - t)
            if rep.failures:
                raise RuntimeError(f"reference farm failures: {rep.failures[:2]}")
        wall = statistics.median(walls)
        return {"value": points / wall, "unit": UNIT, "cores": workers, "kind": "reference",
                "sample": f"{name}: {len(picked)} of {len(frequencies)} frequencies x {ns} steps, "
                          f"{g.n_azimuth}x{g.n_depth} grid, reference pe3d.frequency_farm ({pe3d.__file__}) "
                          f"with {workers} fork workers on {cores} host cores, BASELINE medium injected "
                          f"(oracle/ref_harness.py), median wall {wall:.2f} s of {len(walls)}"}
    except ImportError as exc:
        return _port_sample(name, picked, ns, cores, len(frequencies), points, str(exc))


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
    from oracle import pe3d_oracle  # noqa: F401
    return os.getpid()


def _port_sample(name, picked, ns, cores, n_all, points, why):
    import multiprocessing as mp
    procs = min(len(picked), cores)
    with mp.get_context("spawn").Pool(procs) as pool:
        pool.map(_warm_worker, range(procs))
        t = time.perf_counter()
        pool.map(_oracle_job, [(name, f, ns) for f in picked], chunksize=1)
        wall = time.perf_counter() - t
    return {"value": points / wall, "unit": UNIT, "cores": procs, "kind": "port",
            "sample": f"{name}: {len(picked)} of {n_all} frequencies x {ns} steps, oracle/pe3d_oracle.py "
                      f"(numpy port; reference not installed: {why}), {procs} processes, wall {wall:.2f} s"}


def run_reference_arm(a, rank, world):
    if rank != 0:
        return
    cfg = workload(a.workload, 3)
    freqs = cfg.source.frequencies
    rec = reference_sample(a.workload, freqs, repeats=max(1, min(a.steps, 3)))
    g = cfg.grid
    v = rec["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * len(freqs) * g.n_azimuth * g.n_depth / v,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic",
        "config": {"workload": a.workload, "frequencies": len(freqs), "n_theta": g.n_azimuth,
                   "n_depth": g.n_depth, "parallelism": f"{rec['cores']} host worker processes"},
        "cpu_baseline": rec,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm

class DeviceMarch:
    """Inputs of one march resident on the device, marched through pe3d_march_device."""

    def __init__(self, cfg, freqs, local_dev, steps, stride, tl=True):
        import torch
        import ctypes as C
        from paper_1711_00005_b200 import _native
        from paper_1711_00005_b200.environment import gaussian_starter_column, wavenumber
        from paper_1711_00005_b200.marching import _local_column
        from paper_1711_00005_b200.operators import StepCoefficients
        self.C, self.native, self.torch = C, _native, torch
        self.cfg, self.freqs, self.steps, self.stride = cfg, freqs, steps, stride
        grid, env, source, _ = cfg
        self.grid = grid
        k0s = [wavenumber(f, env.c0) for f in freqs]
        self.coeffs = _native.make_coeffs(k0s, [StepCoefficients.for_step(k0, grid.delta_r) for k0 in k0s])
        self.local_np = np.ascontiguousarray(np.stack([_local_column(env, grid, grid.r_start, k0) for k0 in k0s]))
        self.cols_np = np.ascontiguousarray(np.stack([gaussian_starter_column(grid, source, k0) for k0 in k0s]))
        self.slab_shape = (len(freqs), grid.n_azimuth, grid.n_depth)
        dev = torch.device("cuda", local_dev)
        self.dev = dev
        self.d_local = torch.from_numpy(self.local_np.view(np.float64)).to(dev)
        # the Gaussian starter as one column per frequency (PE3D_FLAG_STARTER_COLUMN, as the drop-in passes it)
        self.d_u0 = torch.from_numpy(self.cols_np.view(np.float64)).to(dev)
        self.d_final = torch.empty(self.slab_shape + (2,), dtype=torch.float64, device=dev)
        self.d_clamped = torch.zeros(len(freqs), dtype=torch.int64, device=dev)
        S = 1 + steps // stride
        self.tl = torch.empty((len(freqs), S, grid.n_azimuth, grid.n_depth), dtype=torch.float64,
                              device=dev) if tl else None
        self.stream = torch.cuda.Stream(device=dev)
        self.h = _native.handle(local_dev)
        self.lib = _native.load_library()

    def march(self, n_steps, flags=0, outputs=True):
        from paper_1711_00005_b200.marching import _grid_params
        C = self.C
        g = _grid_params(self.grid, len(self.freqs), n_steps, self.stride, 0, self.grid.r_start,
                         flags | self.native.FLAG_STARTER_COLUMN)
        self.native.call("pe3d_march_device", self.h, g, self.coeffs, C.c_void_p(self.d_local.data_ptr()),
                         C.c_void_p(self.d_u0.data_ptr()),
                         C.c_void_p(self.d_final.data_ptr()) if outputs else None,
                         C.c_void_p(self.tl.data_ptr()) if (outputs and self.tl is not None) else None, None,
                         C.c_void_p(self.d_clamped.data_ptr()), C.c_void_p(self.stream.cuda_stream))

    def timed(self, n_steps):
        torch = self.torch
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(self.stream):
            t0.record(self.stream)
            self.march(n_steps)
            t1.record(self.stream)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1)

    def sweep_times(self, n_steps):
        """Steady-state CUDA-event times (ms) of both sweeps: a profiled march of
        n_steps without TL or final output, first and last two launches dropped."""
        C = self.C
        with self.torch.cuda.stream(self.stream):
            self.march(n_steps, flags=self.native.FLAG_PROFILE, outputs=False)
        self.torch.cuda.synchronize()
        def launches(cls):
            n = C.c_int32(0)
            self.lib.pe3d_profile_launches(self.h, cls, None, 0, C.byref(n))
            buf = (C.c_double * max(n.value, 1))()
            self.lib.pe3d_profile_launches(self.h, cls, buf, n.value, C.byref(n))
            return list(buf)[:n.value]

        out = {}
        for cls, name in ((0, "depth_sweep"), (1, "azimuth_sweep")):
            ms = launches(cls)
            steady = ms[2:-2] if len(ms) > 8 else ms
            out[name] = {"median_ms": statistics.median(steady), "mean_ms": statistics.fmean(steady),
                         "launches": len(steady)}
        az = launches(1)
        az = az[2:-2] if len(az) > 8 else az
        if az and max(az) > 1.25 * min(az):
            # cfg5: the steps at short range run the cluster ring kernel, the later ones the halo-form
            # split-ring kernel; a median would report only the faster majority, so report the mean
            per_step = statistics.fmean(az)
            out["azimuth_sweep"] = {"median_ms": per_step, "mean_ms": per_step, "launches": len(az),
                                    "note": "mean per step over the march: its steps run two azimuth kernels "
                                            "(cluster rings at short range, halo-form split rings after)"}
        return out


def roofline(sweeps, points_per_launch, peak, peak_kind, workload_name):
    launch_bytes = ALG_BYTES_PER_POINT * points_per_launch
    per = {}
    for name, t in sweeps.items():
        achieved = launch_bytes / (t["median_ms"] / 1e3) / 1e9
        per[name] = {"ms": t["median_ms"], "achieved": achieved, "frac": achieved / peak, "launches": t["launches"],
                     **({"note": t["note"]} if "note" in t else {})}
    dom = max(per, key=lambda k: per[k]["ms"])
    traffic, note = None, None
    tfile = ROOT / "profiles" / f"traffic_{workload_name}.json"
    if tfile.exists():
        t = json.loads(tfile.read_text())
        if t.get("source_hash") == source_hash():
            traffic = t.get(dom)
        else:
            note = f"{tfile.name} was captured from other sources ({t.get('source_hash')}); not reused"
    return {"bound": "hbm", "kernel": dom, "achieved": per[dom]["achieved"], "peak": peak, "unit": "GB/s",
            "frac": per[dom]["frac"], "peak_source": peak_kind, "traffic": traffic,
            **({"traffic_note": note} if note else {}),
            "alg_bytes_per_launch": launch_bytes, "sweeps": per,
            "timing": "median CUDA-event duration of steady-state launches (profiled march, no TL/final)"}


def l2_label(field_bytes):
    return ("inputs larger than L2" if field_bytes > L2_BYTES else "field L2-resident") + \
        f" (field {field_bytes / 2 ** 20:.0f} MiB per buffer, L2 {L2_BYTES / 2 ** 20:.0f} MiB)"


def secondary_line(name, steps, local, peak, peak_kind):
    """Another BASELINE config on this GPU: device time of one march (as the
    main line) plus both sweeps' steady-state roofline."""
    from paper_1711_00005_b200.marching import default_output_stride
    cfg = workload(name, steps)
    freqs = list(cfg.source.frequencies)
    g = cfg.grid
    m = DeviceMarch(cfg, freqs, local, steps, cfg.options.output_stride or default_output_stride(steps))
    with m.torch.cuda.stream(m.stream):
        m.march(steps)
        m.march(steps)
    m.torch.cuda.synchronize()
    ms = m.timed(steps)
    pts = len(freqs) * g.n_azimuth * g.n_depth
    field = len(freqs) * g.n_azimuth * ((g.n_depth + 7) // 8) * 8 * 16
    out = {"value": pts * steps / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
           "l2": l2_label(field)}
    sw = m.sweep_times(steps if name == "cfg5" else max(steps // 4, 12))
    out["roofline"] = roofline(sw, pts, peak, peak_kind, name)
    if field <= L2_BYTES:
        out["roofline"]["note"] = "L2-resident: the HBM fraction is not the bound"
    return out


def run_gpu_arm(a, rank, world, local):
    import torch
    import ctypes as C
    from paper_1711_00005_b200 import _native, parallel
    from paper_1711_00005_b200.marching import _grid_params, default_output_stride

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = workload(a.workload, max(a.steps, a.warmup))
    grid = cfg.grid
    all_freqs = list(cfg.source.frequencies)
    shard_world = a.shard_of if (a.shard_of and world == 1) else world
    mine = parallel.rank_frequencies(all_freqs, rank, shard_world)
    F, NT, NZ = len(mine), grid.n_azimuth, grid.n_depth
    stride = cfg.options.output_stride
    m = DeviceMarch(cfg, mine, local, a.steps, stride)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    # warm-up (W steps) and one untimed K-step march to build the cached graph
    with torch.cuda.stream(m.stream):
        m.march(a.warmup)
        m.march(a.steps)
    torch.cuda.synchronize()

    # ---- timed region: exactly K steps (inputs resident; field > L2, so no flush is needed)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        ms = m.timed(a.steps)
    barrier()
    n_launch = C.c_int64(0)
    m.lib.pe3d_last_launches(m.h, C.byref(n_launch))      # kernels of the timed march (graph replay included)
    if world > 1:
        t = torch.tensor([ms], device=m.dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    total_points = (len(all_freqs) if shard_world == world else F) * NT * NZ * a.steps
    value = total_points / (ms / 1e3)

    peak, peak_kind = peaks()
    sweeps = m.sweep_times(a.steps)
    roof = roofline(sweeps, F * NT * NZ, peak, peak_kind, a.workload)
    roof["step_hbm_frac"] = STEP_BYTES_PER_POINT * value / world / 1e9 / peak

    e2e = e2e_dropin = e2e_default = None
    if not a.no_e2e:
        e2e = host_march_e2e(m, a.steps, stride, world, total_points)
        e2e_default = host_march_e2e(m, a.steps, default_output_stride(configs_n_range(a.workload)), world,
                                     total_points)
        e2e_default["note"] = ("TL every default_output_stride(n_range) steps (ref marching.py:139-141), the "
                               "stride run_frequency uses when a config leaves it unset")
        if world == 1 and shard_world == 1:
            e2e_dropin = dropin_e2e(a.workload, a.steps, local, total_points)

    secondary = None
    if rank == 0 and world == 1 and a.workload == "cfg4" and not a.no_secondary:
        secondary = {"cfg2": secondary_line("cfg2", 400, local, peak, peak_kind),
                     "cfg5": secondary_line("cfg5", configs_n_range("cfg5"), local, peak, peak_kind)}
        secondary["cfg2"]["note"] = "BASELINE configs[1]"
        secondary["cfg5"]["note"] = ("BASELINE configs[4] on one GPU over its 1000 steps (split long columns; split rings "
                                     "where the azimuth carries only reach the segment edges, cluster sweep elsewhere)")

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = cpu_baseline_subprocess(a.workload)

    if rank == 0:
        field_bytes = F * NT * ((NZ + 7) // 8) * 8 * 16
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": a.workload, "frequencies": len(all_freqs), "frequencies_per_gpu": F,
                       "n_theta": NT, "n_depth": NZ, "delta_r": grid.delta_r,
                       "parallelism": f"frequency-shard x{world}",
                       **({"emulated_shard_of": shard_world} if shard_world != world else {}),
                       "l2": l2_label(field_bytes), "output_stride": stride,
                       "tl_samples_in_timed_region": a.steps // stride,
                       "march": f"one graph of {a.steps} steps"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_dropin": e2e_dropin,
            "e2e_default_stride": e2e_default,
            "gpu_launches": int(n_launch.value),
            "clocks": clocks.summary(),
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def cpu_baseline_subprocess(name):
    """The reference arm in a fresh interpreter (no CUDA context to fork from)."""
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, str(Path(__file__).resolve()), "--impl", "reference", "--workload", name,
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=900)
    for line in reversed(r.stdout.strip().splitlines()):
        if line.startswith("{"):
            return json.loads(line)["cpu_baseline"]
    return {"value": None, "unit": UNIT, "kind": "unavailable", "cores": 0,
            "sample": f"reference arm failed (rc {r.returncode}): {r.stderr.strip()[-300:]}"}


def configs_n_range(name):
    from paper_1711_00005_b200 import configs
    return configs.build(name).grid.n_range


def host_march_e2e(m, steps, stride, world, total_points):
    """pe3d_march_host with pinned torch buffers: H2D of starter and medium,
    the march, D2H of the final slab and the TL stack (streamed), timed by wall
    clock around the call (which synchronises)."""
    import torch
    C = m.C
    from paper_1711_00005_b200.marching import _grid_params
    F = len(m.freqs)
    S = 1 + steps // stride
    h_local = torch.from_numpy(m.local_np.view(np.float64)).pin_memory()
    # the drop-in's starter: one Gaussian column per frequency (PE3D_FLAG_STARTER_COLUMN)
    h_u0 = torch.from_numpy(m.cols_np.view(np.float64)).pin_memory()
    h_final = torch.empty(m.slab_shape + (2,), dtype=torch.float64).pin_memory()
    h_tl = torch.empty((F, S, m.grid.n_azimuth, m.grid.n_depth), dtype=torch.float64).pin_memory()
    h_cl = torch.zeros(F, dtype=torch.int64).pin_memory()
    g = _grid_params(m.grid, F, steps, stride, 0, m.grid.r_start, m.native.FLAG_STARTER_COLUMN)

    def host_march():
        m.native.call("pe3d_march_host", m.h, g, m.coeffs, C.c_void_p(h_local.data_ptr()),
                      C.c_void_p(h_u0.data_ptr()), C.c_void_p(h_final.data_ptr()), C.c_void_p(h_tl.data_ptr()),
                      None, C.c_void_p(h_cl.data_ptr()))
    host_march()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    host_march()
    wall = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([wall], device=m.dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        wall = float(t.item())
    h2d = (h_local.numel() + h_u0.numel()) * 8 * world
    d2h = (h_final.numel() + h_tl.numel() + h_cl.numel()) * 8 * world      # the result tensors
    # bytes the library actually moved (a copy-bound march sends one azimuth row of the
    # azimuth-uniform starting TL sample and replicates it on host threads)
    b_in, b_out = C.c_int64(0), C.c_int64(0)
    m.lib.pe3d_last_copy_bytes(m.h, C.byref(b_in), C.byref(b_out))
    return {"value": total_points / wall, "unit": UNIT, "h2d_bytes_per_step": b_in.value * world / steps,
            "d2h_bytes_per_step": b_out.value * world / steps, "result_bytes_per_step": d2h / steps,
            "wall_s": wall, "output_stride": stride, "tl_samples": S,
            "path": "pe3d_march_host (C ABI, pinned host buffers; starter columns + medium in, final slab + "
                    "TL stack out)"}


def dropin_e2e(name, steps, device, total_points):
    """frequency_farm(config, frequencies) -- the reference-facing Python API
    (ref parallel.py:143-185) -- on the workload cut to `steps` range steps."""
    from paper_1711_00005_b200 import configs
    from paper_1711_00005_b200.parallel import frequency_farm
    cfg = configs.build(name, n_range=steps)
    freqs = list(cfg.source.frequencies)
    rep = frequency_farm(cfg, freqs, device=device)           # warm: graph, page-locked result blocks
    del rep
    t0 = time.perf_counter()
    rep = frequency_farm(cfg, freqs, device=device)
    wall = time.perf_counter() - t0
    assert rep.ok
    r0 = rep.results[0]
    S, NT, NZ = r0.tl_field.shape
    h2d = len(freqs) * 2 * NZ * 16                      # starter column + medium column
    d2h = len(freqs) * (S * NT * NZ * 8 + NT * NZ * 16 + 8)     # the result arrays
    import ctypes as C
    from paper_1711_00005_b200 import _native
    b_in, b_out = C.c_int64(0), C.c_int64(0)
    _native.load_library().pe3d_last_copy_bytes(_native.handle(device), C.byref(b_in), C.byref(b_out))
    if b_out.value <= 0:                                # the farm marched on another handle: count the arrays
        b_in, b_out = C.c_int64(h2d), C.c_int64(d2h)
    return {"value": total_points / wall, "unit": UNIT, "h2d_bytes_per_step": b_in.value / steps,
            "d2h_bytes_per_step": b_out.value / steps, "result_bytes_per_step": d2h / steps, "wall_s": wall,
            "output_stride": r0.output_stride,
            "path": "paper_1711_00005_b200.frequency_farm(config, frequencies): host starter + medium, "
                    "one batched march, FrequencyResults in page-locked numpy arrays"}


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
