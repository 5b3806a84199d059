"""B200-native (sm_100a) range marching for the 3-D wide-angle PE solver of
arXiv 1711.00005 -- a drop-in for the hot path of the reference package
``pe3d`` (run_frequency / range_step / frequency_farm / solve_batch).

The public names mirror ``pkg/src/pe3d/__init__.py``; compute runs in the
CUDA library ``libpe3d_b200.so`` (C ABI: ``include/pe3d_b200.h``).  There is
no CPU fallback: without the library or a GPU, compute calls raise
``NativeError``.
"""

__version__ = "0.1.0"

from .config import Config, ExecutorSpec, RunOptions
from .environment import (
    Absorber,
    Environment,
    FieldSlab,
    Grid3D,
    SoundSpeedProfile,
    SourceSpec,
    gaussian_starter,
    hankel_factor,
    refraction_index,
    refraction_index_grid,
    transmission_loss,
    transmission_loss_field,
    wavenumber,
)
from .errors import (
    ColumnTaskError, ConfigError, DomainError, InvariantError, NativeError, Pe3dError, ShapeError,
    SingularSystemError, StepError,
)
from .marching import (
    FrequencyResult, MarchState, apply_boundary, default_output_stride, march_frequencies, range_step,
    run_frequency,
)
from .medium import Bathymetry, FluidBottom, LayeredMedium, RandomPerturbation, Sponge
from .operators import StepCoefficients
from .parallel import (
    FarmFailure, FarmReport, block_ranges, distributed_frequency_farm, frequency_farm, rank_frequencies,
    static_assignment,
)
from .slab import SlabResult, distributed_slab_march, slab_march
from .tridiag import CYCLIC, OPEN, SolveBatch, TriDiagSystem, solve_batch, solve_cyclic, solve_thomas

__all__ = [name for name in dir() if not name.startswith("_")]
