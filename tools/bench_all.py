"""Per-config single-GPU throughput (gp-steps/s) and per-kernel times --
a survey tool, not the driver's bench.py."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main():
    import subprocess
    for w in ("cfg1", "cfg2", "cfg4", "cfg5"):
        steps = {"cfg1": 400, "cfg2": 1000, "cfg4": 500, "cfg5": 200}[w]
        r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--workload", w, "--steps", str(steps),
                            "--no-cpu", "--no-e2e", "--no-secondary"], capture_output=True, text=True)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
            print(w, f"{d['value']:.3e} gp-steps/s", f"{d['ms_per_step'] * 1e3:.1f} us/step", {k: round(v["ms"] * 1e3, 1) for k, v in d["roofline"]["sweeps"].items()})
        except Exception:
            print(w, "FAILED", r.stderr[-500:])
    from paper_1711_00005_b200 import configs, march_frequencies
    cfg = configs.build("cfg3", n_range=200)
    march_frequencies(cfg, [25.0])          # builds (and caches) the step graph
    t = time.perf_counter()
    march_frequencies(cfg, [25.0])
    wall = time.perf_counter() - t
    g = cfg.grid
    print("cfg3", f"{g.n_azimuth * g.n_depth * 200 / wall:.3e} gp-steps/s "
                  f"(host API incl. host medium setup and copies, 200 steps, {wall * 5:.3f} ms/step)")


if __name__ == "__main__":
    main()
