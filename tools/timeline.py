"""Kernel timeline of one headline march (bench.py's DeviceMarch, cfg4, the
graph the bench times) from CUPTI activity records via torch.profiler -- no
replay, launches run as in the bench.  Prints every kernel of the last march
with its start offset and duration, and totals per kernel name.

    python tools/timeline.py [workload] [steps] [shard_of]
(shard_of N: rank 0's frequency block of an N-way split, as bench.py --shard-of)
"""
import collections
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile
    import bench
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    shard = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    cfg = bench.workload(name, steps)
    from paper_1711_00005_b200 import parallel
    freqs = parallel.rank_frequencies(list(cfg.source.frequencies), 0, shard)
    m = bench.DeviceMarch(cfg, freqs, 0, steps, cfg.options.output_stride)
    for _ in range(3):
        m.timed(steps)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ms = m.timed(steps)
    evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.name not in ("Memset", "Memcpy")]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    print(f"{name}, {len(freqs)} frequencies, {steps} steps: CUDA-event time of the march {ms * 1e3:.1f} us")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for e in evs:
        d = e.time_range.end - e.time_range.start
        short = e.name.split("(")[0][:70]
        tot[short] += d
        cnt[short] += 1
        if cnt[short] <= 3 or "prepare" in short or "factor" in short or "setup" in short:
            print(f"  +{e.time_range.start - t0:9.1f} us  {d:8.1f} us  {short}")
    print("  ... last kernels:")
    for e in evs[-5:]:
        print(f"  +{e.time_range.start - t0:9.1f} us  {e.time_range.end - e.time_range.start:8.1f} us  "
              f"{e.name.split('(')[0][:70]}")
    print(f"  last kernel ends at +{max(e.time_range.end for e in evs) - t0:.1f} us")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"  {v:9.1f} us  {cnt[k]:4d} x  {k}")


if __name__ == "__main__":
    main()
