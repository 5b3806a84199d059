"""Dynamic instruction mix of one kernel from an ncu report's SASS source page."""
import collections
import csv
import subprocess
import sys


def mix(rep, kernel_regex, top=25):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass',
                          '-k', f'regex:{kernel_regex}'], capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(lines[1:]))
    h = rows[0]
    si, ei, wi = h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
    by_op = collections.Counter()
    stall = collections.Counter()
    total = 0
    for r in rows[1:]:
        try:
            n = int(r[ei])
        except (ValueError, IndexError):
            continue
        op = r[si].strip().split()[0] if r[si].strip() else '?'
        if op.startswith('@'):
            op = r[si].strip().split()[1]
        op = op.split('.')[0]
        by_op[op] += n
        stall[op] += int(r[wi] or 0)
        total += n
    print(f"total warp-instructions executed: {total}")
    for op, n in by_op.most_common(top):
        print(f"  {op:10s} {n:12d}  {100 * n / total:5.1f}%  stall-samples {stall[op]}")


if __name__ == '__main__':
    mix(sys.argv[1], sys.argv[2])
