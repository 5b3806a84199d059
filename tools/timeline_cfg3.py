"""Kernel timeline of a short cfg3 march (device medium, one cached step graph) from
CUPTI activity records via torch.profiler: the kernels of three steady-state steps with
their start offsets and durations, and totals per kernel name.

    python tools/timeline_cfg3.py [steps]
"""
import collections
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    from torch.profiler import ProfilerActivity, profile
    from paper_1711_00005_b200 import configs, march_frequencies
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    cfg = configs.build("cfg3", n_range=steps)
    for _ in range(3):
        march_frequencies(cfg, [25.0])
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        march_frequencies(cfg, [25.0])
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    ker = [e for e in evs if not e.name.startswith(("Memcpy", "Memset"))]
    t0 = ker[0].time_range.start
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for e in ker:
        d = e.time_range.end - e.time_range.start
        short = e.name.split("(")[0][:60]
        tot[short] += d
        cnt[short] += 1
    span = ker[-1].time_range.end - t0
    print(f"cfg3, {steps} steps: first to last kernel {span:.1f} us = {span / steps:.1f} us per step")
    mid = [e for e in ker if t0 + span * 0.5 <= e.time_range.start <= t0 + span * 0.5 + 150.0]
    for e in mid:
        print(f"  +{e.time_range.start - t0:9.1f} us {e.time_range.end - e.time_range.start:8.1f} us  {e.name.split('(')[0][:60]}")
    for k, v in sorted(tot.items(), key=lambda t: -t[1]):
        print(f"  {v:10.1f} us {cnt[k]:5d} x  {k}")


if __name__ == "__main__":
    main()
