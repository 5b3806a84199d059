"""Device time per step of the slab-decomposed cfg5 march with N virtual
ranks on one GPU, for the device-copy all-to-all and the peer-direct
(fused) transposes.  On one GPU the ranks' sweeps run one after another, so
this measures the transport overhead, not multi-GPU speed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_00005_b200 import configs, slab_march  # noqa: E402

cfg = configs.build("cfg5", n_range=40)
for mode in ("copy", "peer"):
    if mode == "copy":
        os.environ["PE3D_SLAB_COPY"] = "1"
    else:
        os.environ.pop("PE3D_SLAB_COPY", None)
    for n in (1, 2, 4, 8):
        slab_march(cfg, 500.0, n, n_steps=3)
        r = slab_march(cfg, 500.0, n, n_steps=40)
        print(mode, n, "ms/step", round(r.step_ms / 40, 3), flush=True)
