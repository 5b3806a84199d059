"""Top stall-sampled SASS instructions of one kernel in an ncu report."""
import csv
import subprocess
import sys


def hot(rep, kernel_regex, top=30):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass',
                          '-k', f'regex:{kernel_regex}'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()[1:]))
    h = rows[0]
    si, wi, ei = h.index('Source'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
    items = []
    for idx, r in enumerate(rows[1:]):
        try:
            items.append((int(r[wi] or 0), idx, r[si].strip(), int(r[ei] or 0)))
        except (ValueError, IndexError):
            pass
    total = sum(x[0] for x in items)
    for w, idx, src, n in sorted(items, reverse=True)[:top]:
        print(f"{100 * w / total:5.1f}%  #{idx:5d}  exec {n:9d}  {src[:90]}")


if __name__ == '__main__':
    hot(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
