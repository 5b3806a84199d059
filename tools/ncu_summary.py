"""Summarise an ncu --set full report into the text kept under profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep [--traffic OUT.json KEY=regex ...]
Prints, per kernel: duration, DRAM bytes read/written and throughput, L2 hit
rate, occupancy, issue rate, IPC, registers, top stall reasons (per issued
instruction) and the dynamic instruction mix (from the SASS source page).
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys
from pathlib import Path

DETAILS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Issued Warp Per Scheduler",
           "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
           "Grid Size", "Block Size", "Cluster Size", "Dynamic Shared Memory Per Block"]
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def main():
    rep = sys.argv[1]
    out = {}
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "details", "--csv"))))
    h = rows[0]
    ik, im, iv, iu = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    kernels, first_id = [], {}
    iid = h.index("ID")
    for r in rows[1:]:
        name = r[ik].split("(")[0]
        if name not in out:
            out[name] = {}
            kernels.append(name)
            first_id[name] = int(r[iid])            # launch index in the report (instantiations share a base name)
        if r[im] in DETAILS:
            out[name][r[im]] = f"{r[iv]} {r[iu]}".strip()
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(RAW)))))
    hr = raw[0]
    for r in raw[2:]:
        name = r[hr.index("Kernel Name")].split("(")[0]
        for m in RAW:
            out[name][m] = r[hr.index(m)] + " " + raw[1][hr.index(m)]
    for name in kernels:
        src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                                              "--launch-skip", str(first_id[name]), "--launch-count", "1"))))
        hdr = src[1]
        iE0 = hdr.index("Instructions Executed")
        data = [r for r in src[2:] if len(r) == len(hdr) and r[iE0].isdigit()]   # one kernel's rows
        iE = hdr.index("Instructions Executed")
        names = [x for x in hdr if x.startswith("stall_") and "(Not" not in x]
        idx = {n: hdr.index(n) for n in names}
        tot_s = sum(int(r[idx[n]] or 0) for r in data for n in names) or 1
        stalls = sorted(((n[6:], sum(int(r[idx[n]] or 0) for r in data)) for n in names), key=lambda t: -t[1])
        mix = collections.Counter()
        for r in data:
            op = r[1].strip().split()
            if op:
                o = op[1] if op[0].startswith("@") else op[0]
                mix[o.split(".")[0]] += int(r[iE] or 0)
        tot_i = sum(mix.values()) or 1
        out[name]["stall samples (share)"] = ", ".join(f"{n} {100 * v / tot_s:.1f}%" for n, v in stalls[:8])
        out[name]["instruction mix"] = ", ".join(f"{o} {100 * v / tot_i:.1f}%" for o, v in mix.most_common(12))
    for name in kernels:
        print(name)
        for k, v in out[name].items():
            print(f"  {k:62s} {v}")
    if "--traffic" in sys.argv:
        i = sys.argv.index("--traffic")
        path, pairs = sys.argv[i + 1], sys.argv[i + 2:]
        traffic = {}
        for p in pairs:
            key, pat = p.split("=")
            for name in kernels:
                if pat in name:
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                    rd, ru = out[name]["dram__bytes_read.sum"].split()[:2]
                    wr, wu = out[name]["dram__bytes_write.sum"].split()[:2]
                    traffic[key] = float(rd) * scale[ru] + float(wr) * scale[wu]
                    dur = out[name].get("gpu__time_duration.sum", "").split()
                    if dur:
                        traffic[key + "_duration_us"] = float(dur[0])
        # stamp the capture with the hash of the CUDA sources it was built from
        # (bench.py reuses a traffic file only when the hash matches csrc/)
        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        from bench import source_hash
        traffic["source_hash"] = source_hash()
        traffic["source"] = f"ncu --set full, {Path(sys.argv[1]).name}"
        json.dump(traffic, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
