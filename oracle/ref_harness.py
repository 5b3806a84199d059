"""Drive the UNMODIFIED reference package ``pe3d`` on the BASELINE configs.

TEST INFRASTRUCTURE (see oracle/__init__.py): used by the fixture
generators under ``tests/golden/``, by the drop-in tests that hand the
reference's own objects to the B200 package, and by ``bench.py``'s
``--impl reference`` arm and ``cpu_baseline`` leg.  Never by the product.

Where the reference comes from, first found wins:
  1. ``$PE3D_REFERENCE_SRC`` (a directory containing the ``pe3d`` package);
  2. ``baseline/_ref`` (the pip install of /root/reference, DESIGN.md §5;
     it travels to the GPU box with the repo snapshot);
  3. ``/root/reference/pkg/src`` (this build container only).

The BASELINE media (density, fluid bottom, sponge, bathymetry, seeded
noise) are not expressible with the reference's own ``Environment``; they
are injected by rebinding ``pe3d.marching.refraction_index_grid`` (ref
marching.py:31, called at :110 and :116) to the product's shared medium
definition, with the k0 of the step being taken (the density term is
frequency dependent).  ``range_step`` is wrapped only to publish that k0
(and, for the fixture generator, to observe the result); the march, the
operators, the solves and the TL are the reference's own code.
Process pools of the reference's ``frequency_farm`` (fork) inherit the
rebinding.
"""

from __future__ import annotations

import importlib
import os
import sys
from pathlib import Path
from typing import Callable, Optional

ROOT = Path(__file__).resolve().parents[1]

_STATE = {"k0": None, "observer": None}


def reference_source() -> Optional[Path]:
    cands = []
    env = os.environ.get("PE3D_REFERENCE_SRC")
    if env:
        cands.append(Path(env))
    cands += [ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")]
    for c in cands:
        if (c / "pe3d" / "__init__.py").exists():
            return c
    return None


def import_reference():
    """The reference package ``pe3d`` (raises ImportError if none is found)."""
    src = reference_source()
    if src is None:
        raise ImportError("reference pe3d not found (PE3D_REFERENCE_SRC, baseline/_ref, /root/reference)")
    if str(src) not in sys.path:
        sys.path.insert(0, str(src))
    pe3d = importlib.import_module("pe3d")
    if not Path(pe3d.__file__).resolve().is_relative_to(src.resolve()):
        raise ImportError(f"a different pe3d is already imported: {pe3d.__file__}")
    return pe3d


def ref_grid(pe3d, g):
    return pe3d.Grid3D(g.n_range, g.n_azimuth, g.n_depth, g.delta_r, g.delta_theta, g.delta_z, g.r_start,
                       g.azimuth_topology)


def ref_env(pe3d, g, c0=1500.0):
    """A plain reference Environment (its medium is replaced by the injection)."""
    return pe3d.Environment(c0, pe3d.SoundSpeedProfile.uniform(c0), 6000.0, pe3d.Absorber(0.0, 0.0),
                            g.depth_extent)


def ref_config(pe3d, cfg, frequencies=None, output_stride=None):
    g = cfg.grid
    freqs = tuple(frequencies if frequencies is not None else cfg.source.frequencies)
    return pe3d.Config(ref_grid(pe3d, g), ref_env(pe3d, g), pe3d.SourceSpec(freqs, cfg.source.depth),
                       pe3d.RunOptions(output_stride=output_stride or cfg.options.output_stride))


def install_medium(pe3d, cfg, observer: Optional[Callable] = None):
    """Bind ``cfg``'s medium into the reference march (see the module doc).
    ``observer(old_state, new_state)`` is called after every reference step."""
    import pe3d.marching as ref_marching
    from paper_1711_00005_b200.environment import refraction_index_grid
    env, g = cfg.environment, cfg.grid
    if not hasattr(ref_marching, "_pe3d_b200_original_step"):
        ref_marching._pe3d_b200_original_step = ref_marching.range_step
    original = ref_marching._pe3d_b200_original_step
    _STATE["observer"] = observer

    def stepping(state):
        _STATE["k0"] = state.k0
        new = original(state)
        if _STATE["observer"] is not None:
            _STATE["observer"](state, new)
        return new

    ref_marching.refraction_index_grid = lambda e, gg, r: refraction_index_grid(env, g, r, _STATE["k0"])
    ref_marching.range_step = stepping
