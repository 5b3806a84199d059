"""cfg3 per-step time without the per-march constant (host medium setup, copies):
wall(n2 steps) - wall(n1 steps) over n2 - n1, each march after a warm-up of the same length."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1711_00005_b200 import configs, march_frequencies  # noqa: E402


def wall(n):
    cfg = configs.build("cfg3", n_range=n)
    march_frequencies(cfg, [25.0])
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        march_frequencies(cfg, [25.0])
        best = min(best, time.perf_counter() - t)
    return best


if __name__ == "__main__":
    n1, n2 = 200, 1000
    w1, w2 = wall(n1), wall(n2)
    per = (w2 - w1) / (n2 - n1)
    print(f"cfg3 {512 * 512 / per:.3e} gp-steps/s, {per * 1e6:.1f} us/step (marches of {n1} and {n2} steps: {w1 * 1e3:.1f} / {w2 * 1e3:.1f} ms)")
