import sys, time
sys.path.insert(0, '.')
from paper_1711_00005_b200 import configs, run_frequency
for name in ("cfg1", "cfg2", "cfg3"):
    cfg = configs.build(name)
    f = cfg.source.frequencies[0]
    run_frequency(cfg, f)
    best = 1e9
    for _ in range(3):
        t = time.perf_counter(); r = run_frequency(cfg, f); best = min(best, time.perf_counter() - t)
    g = cfg.grid
    print(name, f"{best*1e3:.2f} ms wall for {g.n_range} steps = {best/g.n_range*1e6:.2f} us/step, {g.n_range*g.n_azimuth*g.n_depth/best:.3e} gp-steps/s, tl {r.tl_field.shape}")
