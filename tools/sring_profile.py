"""Per-kernel CUDA-event times of cfg5's split-ring steps: a profiled 1000-step
march (bench.py's DeviceMarch); prints the medians of the azimuth launches of
the cluster steps and of the split-ring steps (segmented sweep, carry, fix).
The split steps are the last ones (the carries reach further at short range)."""
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import ctypes as C
    import bench
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    cfg = bench.workload("cfg5", steps)
    m = bench.DeviceMarch(cfg, list(cfg.source.frequencies), 0, steps, cfg.options.output_stride)
    m.march(steps, flags=m.native.FLAG_PROFILE, outputs=False)
    m.torch.cuda.synchronize()

    def launches(cls):
        n = C.c_int32(0)
        m.lib.pe3d_profile_launches(m.h, cls, None, 0, C.byref(n))
        buf = (C.c_double * max(n.value, 1))()
        m.lib.pe3d_profile_launches(m.h, cls, buf, n.value, C.byref(n))
        return [x * 1e3 for x in list(buf)[:n.value]]

    az, ex, dep = launches(1), launches(3), launches(0)
    n_split = len(ex) // 2                                     # carry, fix per split step
    cl, sg = az[:len(az) - n_split], az[len(az) - n_split:]
    med = lambda v: round(statistics.median(v), 2) if v else None
    print(f"steps {len(az)}: cluster steps {len(cl)} (azimuth {med(cl)} us), split steps {n_split}: "
          f"segmented {med(sg)} us, carry {med(ex[0::2])} us, fix {med(ex[1::2])} us "
          f"(first {round(ex[1], 1) if ex else None}, last {round(ex[-1], 1) if ex else None}); depth {med(dep)} us")


if __name__ == "__main__":
    main()
