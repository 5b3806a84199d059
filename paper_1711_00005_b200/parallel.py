"""Frequency-level parallelism: the drop-in for ``frequency_farm``
(ref ``pkg/src/pe3d/parallel.py:85-185``) and its static block law
(ref ``pool.py:39-57``, ``parallel.py:85-97``).

On one GPU the frequencies of a farm are one batched device march
(frequencies are the outer batch dimension of every kernel launch).
Across GPUs (one process per GPU, ``torch.distributed``), each rank takes
the contiguous static block ``static_assignment(F, world)[rank]`` -- the
paper's MPI frequency split -- and no data-path collective is needed
(frequencies never exchange data, ref ``SPEC.md:435``); only the small
results are gathered on request.  CUDA never runs in forked workers
(SURVEY.md H7): there are no worker processes on the GPU path.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

from .errors import InvariantError
from .marching import march_frequencies


def block_ranges(n_items: int, n_blocks: int) -> list:
    """Contiguous blocks, sizes differing by at most one, larger first,
    empty blocks dropped (ref pool.py:39-57)."""
    if n_items < 0 or n_blocks < 1:
        raise InvariantError("n_items >= 0 and n_blocks >= 1")
    n_blocks = min(n_blocks, max(n_items, 1))
    base, extra = divmod(n_items, n_blocks)
    out, lo = [], 0
    for b in range(n_blocks):
        size = base + (1 if b < extra else 0)
        if size:
            out.append((lo, lo + size))
        lo += size
    return out


def static_assignment(n_jobs: int, n_workers: int) -> List[List[int]]:
    """Job indices per worker; max load ceil(n_jobs/n_workers); workers
    beyond the job count get empty lists (ref parallel.py:85-97)."""
    if n_jobs < 0 or n_workers < 1:
        raise InvariantError("n_jobs >= 0 and n_workers >= 1")
    blocks = [list(range(lo, hi)) for lo, hi in block_ranges(n_jobs, n_workers)]
    blocks += [[] for _ in range(n_workers - len(blocks))]
    return blocks


@dataclass
class FarmFailure:
    index: int
    frequency: float
    message: str


@dataclass
class FarmReport:
    """Ordered per-frequency results; failed slots hold None (ref :70-82)."""

    results: list
    failures: list

    @property
    def ok(self) -> bool:
        return not self.failures


def _march_isolating(config, jobs, device, n_steps=None):
    """March a block of (index, frequency) jobs as one batch; on a failure,
    fall back to one march per frequency so failures stay per frequency
    (ref parallel.py:126-140)."""
    freqs = [f for _, f in jobs]
    try:
        res = march_frequencies(config, freqs, device=device, n_steps=n_steps)
        return [(i, "ok", r) for (i, _), r in zip(jobs, res)]
    except Exception as exc:            # any failure of the batch (StepError, host memory, ...)
        if len(jobs) == 1:
            return [(jobs[0][0], "error", f"{type(exc).__name__}: {exc}")]
    outcomes = []
    for i, f in jobs:
        try:
            outcomes.append((i, "ok", march_frequencies(config, [f], device=device, n_steps=n_steps)[0]))
        except Exception as exc:    # collected, as the reference's farm does
            outcomes.append((i, "error", f"{type(exc).__name__}: {exc}"))
    return outcomes


def frequency_farm(config, frequencies, workers: int = 1, schedule: str = "static",
                   intra_threads: int = 1, device: int = 0) -> FarmReport:
    """Solve each frequency independently and merge in input order
    (ref parallel.py:143-185).  All frequencies of this process run as
    batched device marches on ``device``; ``workers``/``schedule``/
    ``intra_threads`` are validated and otherwise only shape the batches
    (results do not depend on them -- the reference's determinism
    contract)."""
    frequencies = list(frequencies)
    if not frequencies:
        raise InvariantError("frequencies nonempty")
    if workers < 1:
        raise InvariantError("workers >= 1")
    if schedule not in ("static", "dynamic"):
        raise InvariantError("schedule in (static, dynamic)", f"got {schedule!r}")
    if intra_threads < 1:
        raise InvariantError("intra_threads >= 1")
    jobs = list(enumerate(frequencies))
    results: list = [None] * len(frequencies)
    failures = []
    outcomes = _march_isolating(config, jobs, device)    # one outcome per job, failures included
    for index, status, payload in outcomes:
        if status == "ok":
            results[index] = payload
        else:
            failures.append(FarmFailure(index, frequencies[index], payload))
    failures.sort(key=lambda x: x.index)
    return FarmReport(results=results, failures=failures)


def rank_frequencies(frequencies, rank: int, world_size: int) -> list:
    """The contiguous static block of frequencies owned by ``rank``."""
    if not 0 <= rank < world_size:
        raise InvariantError("0 <= rank < world_size")
    block = static_assignment(len(frequencies), world_size)[rank]
    return [frequencies[i] for i in block]


def distributed_frequency_farm(config, frequencies, group=None, device: Optional[int] = None,
                               gather: bool = True) -> Optional[FarmReport]:
    """One process per GPU: this rank marches its static block on its own
    device; with ``gather`` the per-frequency results are collected on rank
    0 (object gather over the process group -- the only communication).
    Returns the full FarmReport on rank 0, this rank's partial report
    elsewhere (or when ``gather`` is False)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    frequencies = list(frequencies)
    mine = static_assignment(len(frequencies), world)[rank]
    dev = rank if device is None else device
    report = FarmReport([None] * len(frequencies), [])
    if mine:
        jobs = [(i, frequencies[i]) for i in mine]
        for index, status, payload in _march_isolating(config, jobs, dev):
            if status == "ok":
                report.results[index] = payload
            else:
                report.failures.append(FarmFailure(index, frequencies[index], payload))
    if not gather:
        return report
    parts = [None] * world if rank == 0 else None
    dist.gather_object(report, parts, dst=0, group=group)
    if rank != 0:
        return report
    merged = FarmReport([None] * len(frequencies), [])
    for part in parts:
        for i, r in enumerate(part.results):
            if r is not None:
                merged.results[i] = r
        merged.failures.extend(part.failures)
    merged.failures.sort(key=lambda x: x.index)
    return merged
