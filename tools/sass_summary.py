"""Static SASS opcode counts per kernel of libpe3d_b200.so (cuobjdump -sass):
the proof of which kernels move data with the tensor engine (UTMALDG / UTMASTG
/ UBLKCP) and which with per-thread cp.async (LDGSTS).

usage: python tools/sass_summary.py [regex] > profiles/r02_sass_kernels.txt
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

SO = Path(__file__).resolve().parents[1] / "paper_1711_00005_b200" / "libpe3d_b200.so"
OPS = ["UTMALDG", "UTMASTG", "UBLKCP", "UTMACCTL", "LDGSTS", "SYNCS", "LDG", "STG", "LDS", "STS", "SHFL", "DFMA"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out))


def main():
    pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
    sass = subprocess.run(["cuobjdump", "-sass", str(SO)], capture_output=True, text=True).stdout
    counts, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            counts[cur][m.group(2)] += 1
    names = demangle(list(counts))
    print(f"# static SASS instruction counts per kernel, cuobjdump -sass {SO.name} (sm_100a)")
    print(f"{'kernel':70s} " + " ".join(f"{o:>8s}" for o in OPS))
    for mangled, c in sorted(counts.items(), key=lambda kv: names[kv[0]]):
        n = names[mangled].replace("pe3d::", "")
        n = re.sub(r"\(.*", "", n)
        if pat and not pat.search(n):
            continue
        print(f"{n[:70]:70s} " + " ".join(f"{c[o]:8d}" for o in OPS))


if __name__ == "__main__":
    main()
