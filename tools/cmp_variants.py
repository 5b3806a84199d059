"""Compare one config's march under two environment variants of the library
(each in its own process: graph caches and kernel choices are per process).

    python tools/cmp_variants.py cfg5 3 "PE3D_RING_NO_HALF=1" ""

Prints the max |diff| of the final slab, overall and by row within the 8-row
tile and by 512-azimuth segment."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def run_one(name, steps, out):
    sys.path.insert(0, str(ROOT))
    from paper_1711_00005_b200 import configs, march_frequencies
    cfg = configs.build(name, n_range=max(steps, 3), output_stride=steps)
    r = march_frequencies(cfg, [cfg.source.frequencies[0]], n_steps=steps)[0]
    np.save(out, r.final_slab.values)


def main():
    if sys.argv[1] == "--one":
        run_one(sys.argv[2], int(sys.argv[3]), sys.argv[4])
        return
    name, steps, va, vb = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
    outs = []
    for i, v in enumerate((va, vb)):
        env = dict(os.environ)
        for kv in v.split():
            k, _, val = kv.partition("=")
            env[k] = val
        out = f"/tmp/cmp_{i}.npy"
        subprocess.run([sys.executable, __file__, "--one", name, steps, out], env=env, check=True)
        outs.append(np.load(out))
    a, b = outs
    d = np.abs(a - b)
    scale = np.abs(b).max()
    print(f"{name} {steps} steps [{va}] vs [{vb}]: max|diff| {d.max():.3e} (field max {scale:.3e}), "
          f"bitwise {a.tobytes() == b.tobytes()}")
    if d.max() > 0:
        nt, nz = d.shape
        print(" by row % 8:", [f"{d[:, r::8].max():.1e}" for r in range(8)])
        seg = 512 if nt >= 1024 else nt
        print(" by segment:", [f"{d[s * seg:(s + 1) * seg].max():.1e}" for s in range(nt // seg)])
        for thr in (1e-6, 1e-10, 1e-13):
            rows = np.where(d.max(axis=0) > thr * scale)[0]
            print(f" rows with diffs > {thr:g} of max: {len(rows)}; tiles", sorted(set((rows // 8).tolist()))[:60])
        rmax = int(np.argmax(d.max(axis=0)))
        print(f" worst row {rmax}: diff by azimuth (every 64th):", [f"{x:.1e}" for x in d[::64, rmax]])


if __name__ == "__main__":
    main()
