import cProfile, pstats, sys, time
sys.path.insert(0, '.')
from paper_1711_00005_b200 import configs
from paper_1711_00005_b200.parallel import frequency_farm
cfg = configs.build("cfg4", n_range=20)
freqs = list(cfg.source.frequencies)
for _ in range(3):
    rep = frequency_farm(cfg, freqs, device=0); del rep
t=time.perf_counter(); rep = frequency_farm(cfg, freqs, device=0); print("wall", time.perf_counter()-t); del rep
pr = cProfile.Profile(); pr.enable()
rep = frequency_farm(cfg, freqs, device=0)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
