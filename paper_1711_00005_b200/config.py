"""Run options and the ``Config`` bundle; ref ``pkg/src/pe3d/config.py:71-102``
and ``ExecutorSpec`` from ``pkg/src/pe3d/pool.py:19-36``.

INI ingestion (ref ``config.py:173-268``) is outside the hot-path scope
(SURVEY.md §8(f) row 4); configs are built in memory, e.g. by
:mod:`.configs`.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path
from typing import NamedTuple, Optional

from .environment import Environment, Grid3D, SourceSpec
from .errors import InvariantError

TL_FORMATS = ("csv", "binary-grid")
SCHEDULES = ("static", "dynamic")
MODES = ("run", "bench", "selftest")
PINNING_MODES = ("none", "compact")


@dataclass(frozen=True)
class ExecutorSpec:
    """Parallelism knobs of the reference.  On the GPU the intra-step
    thread count has no effect (the CUDA grid replaces the thread pool);
    ``freq_workers`` maps to the number of GPUs a farm may use."""

    intra_threads: int = 1
    freq_workers: int = 1
    pinning: str = "none"

    def __post_init__(self):
        if self.intra_threads < 1:
            raise InvariantError("intra_threads >= 1", f"got {self.intra_threads}")
        if self.freq_workers < 1:
            raise InvariantError("freq_workers >= 1", f"got {self.freq_workers}")
        if self.pinning not in PINNING_MODES:
            raise InvariantError(f"pinning in {PINNING_MODES}", f"got {self.pinning!r}")


@dataclass(frozen=True)
class RunOptions:
    mode: str = "run"
    output_dir: Path = Path("out")
    output_stride: Optional[int] = None
    tl_format: str = "csv"
    executor: ExecutorSpec = field(default_factory=ExecutorSpec)
    max_range: Optional[float] = None
    schedule: str = "static"

    def __post_init__(self):
        checks = (
            (self.mode in MODES, f"mode in {MODES}", repr(self.mode)),
            (self.output_stride is None or self.output_stride >= 1,
             "output_stride >= 1", str(self.output_stride)),
            (self.tl_format in TL_FORMATS, f"tl_format in {TL_FORMATS}", repr(self.tl_format)),
            (self.schedule in SCHEDULES, f"schedule in {SCHEDULES}", repr(self.schedule)),
            (self.max_range is None or self.max_range > 0, "max_range > 0", str(self.max_range)),
        )
        for ok, constraint, got in checks:
            if not ok:
                raise InvariantError(constraint, f"got {got}")
        object.__setattr__(self, "output_dir", Path(self.output_dir))


class Config(NamedTuple):
    grid: Grid3D
    environment: Environment
    source: SourceSpec
    options: RunOptions
