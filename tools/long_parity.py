"""Full-size BASELINE grids over longer marches than the golden fixtures,
against the oracle run here: prints the worst field relative L2 and |dTL|
(TL < 150 dB) over the output ranges (the contract is 1e-9 and 1e-4 dB)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import pe3d_oracle as O                            # noqa: E402
from paper_1711_00005_b200 import configs, march_frequencies    # noqa: E402

cases = [("cfg4", 500.0, 300), ("cfg4", 50.0, 300), ("cfg2", 100.0, 150), ("cfg3", 25.0, 150)]
if "--cfg5" in sys.argv:
    cases.append(("cfg5", 500.0, 12))          # the 4096 x 4096 cluster path; the oracle needs ~3 s per step
for name, freq, n in cases:
    stride = 4 if name == "cfg5" else 50
    cfg = configs.build(name, n_range=n, frequencies=(freq,), output_stride=stride) if name == "cfg4" else \
        configs.build(name, n_range=n, output_stride=stride)
    got = march_frequencies(cfg, [freq], keep_snapshots=True)[0]
    ref = O.run_frequency(cfg, freq, keep_snapshots=True)
    l2 = max(float(np.linalg.norm(got.snapshots[k] - ref.snapshots[k]) / np.linalg.norm(ref.snapshots[k]))
             for k in range(ref.tl_field.shape[0]))
    m = ref.tl_field < 150
    dtl = float(np.abs(got.tl_field - ref.tl_field)[m].max())
    print(f"{name} {freq:g} Hz, {n} steps: worst rel L2 {l2:.2e}, worst |dTL| {dtl:.2e} dB")
