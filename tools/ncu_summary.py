"""Summarise an ncu report (details + raw pages) into a short text table."""
import csv
import subprocess
import sys

WANT = ['Duration', 'Memory Throughput', 'DRAM Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Issued Warp Per Scheduler', 'No Eligible', 'Eligible Warps Per Scheduler', 'Dynamic Shared Memory Per Block',
        'Executed Ipc Active', 'Grid Size', 'Block Size']
RAW = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
       'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
       'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'gpu__time_duration.sum']


def run(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, mi, vi, ui = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
    for r in rows[1:]:
        if r[mi] in WANT:
            print(f"{r[ki][:28]:28s} | {r[mi]:32s} = {r[vi]} {r[ui]}")
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    units = rows[1]
    for r in rows[2:]:
        name = r[h.index('Kernel Name')][:28]
        for k in RAW:
            if k in h:
                print(f"{name:28s} | {k:32s} = {r[h.index(k)]} {units[h.index(k)]}")
        stalls = []
        for i, k in enumerate(h):
            if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio'):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v > 0.1:
                    stalls.append((v, k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
        stalls.sort(reverse=True)
        print(f"{name:28s} | stalls: " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:8]))


if __name__ == '__main__':
    run(sys.argv[1])
