"""Timeline of one pe3d_march_host call (bench.py's e2e leg: cfg4, host buffers in pinned
memory) from CUPTI activity records via torch.profiler: per frequency group the span of its
kernels, and every copy with its size class, against the wall time of the call.

    python tools/timeline_host.py [steps]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile
    import bench
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    cfg = bench.workload("cfg4", steps)
    freqs = list(cfg.source.frequencies)
    m = bench.DeviceMarch(cfg, freqs, 0, steps, cfg.options.output_stride)
    total = len(freqs) * cfg.grid.n_azimuth * cfg.grid.n_depth * steps
    for _ in range(2):
        bench.host_march_e2e(m, steps, cfg.options.output_stride, 1, total)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = bench.host_march_e2e(m, steps, cfg.options.output_stride, 1, total)
    print(f"wall of the timed call {r['wall_s'] * 1e3:.2f} ms (under the profiler)")
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    # the last host march = the events after the last long gap
    t_end = evs[-1].time_range.end
    last = [e for e in evs if e.time_range.start > t_end - 12000.0]
    # trim to the final call: walk back from the end until a gap > 300 us
    cut = 0
    for i in range(len(last) - 1, 0, -1):
        if last[i].time_range.start - last[i - 1].time_range.end > 300.0:
            cut = i
            break
    last = last[cut:]
    t0 = last[0].time_range.start
    ker = [e for e in last if not e.name.startswith(("Memcpy", "Memset"))]
    print(f"events of the call: {len(last)}, span {last[-1].time_range.end - t0:.1f} us")
    # kernel groups: a gap of more than 40 us between kernels starts a new group
    groups, cur = [], [ker[0]]
    for e in ker[1:]:
        if e.time_range.start - max(x.time_range.end for x in cur) > 40.0:
            groups.append(cur)
            cur = [e]
        else:
            cur.append(e)
    groups.append(cur)
    for i, gk in enumerate(groups):
        print(f"  kernels {i}: +{gk[0].time_range.start - t0:8.1f} .. +{max(x.time_range.end for x in gk) - t0:8.1f} us  ({len(gk)} kernels)")
    for e in last:
        if e.name.startswith("Memcpy"):
            d = e.time_range.end - e.time_range.start
            if d > 20.0:
                print(f"  copy    +{e.time_range.start - t0:8.1f} .. +{e.time_range.end - t0:8.1f} us  {d:8.1f} us  {e.name}")


if __name__ == "__main__":
    main()
