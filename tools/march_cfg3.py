import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1711_00005_b200 import configs, march_frequencies
cfg = configs.build("cfg3", n_range=int(sys.argv[1]) if len(sys.argv) > 1 else 6)
march_frequencies(cfg, [25.0])
