"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, mean and total duration, share of the total.

    python tools/launch_list.py gpurun_out/launches.csv "command that was profiled" > profiles/rNN_launches_....txt
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    cmd = sys.argv[2] if len(sys.argv) > 2 else ""
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1e3)
        name = r["Kernel Name"]
        tot[name] += us
        cnt[name] += 1
    total = sum(tot.values()) or 1.0
    if cmd:
        print(f"# ncu launch list of `{cmd}`")
    print("# gpu__time_duration.sum --clock-control none; cold-cache, serialised launches: compare shares, not absolutes")
    print(f"{'kernel':60s} {'launches':>9s} {'mean us':>9s} {'total us':>10s}  share")
    for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{name[:60]:60s} {cnt[name]:9d} {t / cnt[name]:9.2f} {t:10.1f} {100 * t / total:5.1f}%")


if __name__ == "__main__":
    main()
