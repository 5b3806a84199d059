"""Multi-process host logic of the frequency sharding (gloo, world size 2,
CPU): each rank marches its static block (ref parallel.py:85-97), results
are gathered on rank 0 in input order, per-frequency failures are
collected, and no data-path collective is involved."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, queue, fail_freq):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1711_00005_b200 import parallel
    from paper_1711_00005_b200.errors import StepError

    marched = []

    def fake_march(config, freqs, device=0, n_steps=None):
        for f in freqs:
            if f == fail_freq:
                raise StepError(1, "depth", 0, "injected")
        marched.extend(freqs)
        return [("result", f, rank) for f in freqs]

    parallel.march_frequencies = fake_march
    freqs = [50.0 + 10 * i for i in range(7)]
    report = parallel.distributed_frequency_farm(config=None, frequencies=freqs, device=0)
    queue.put((rank, marched, None if rank else (report.results, [(x.index, x.frequency) for x in report.failures])))
    dist.destroy_process_group()


@pytest.mark.parametrize("fail_freq", [None, 80.0])
def test_gloo_two_ranks_static_blocks(fail_freq):
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, queue, fail_freq)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        rank, marched, merged = queue.get(timeout=120)
        out[rank] = (marched, merged)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    freqs = [50.0 + 10 * i for i in range(7)]
    # static law: rank 0 owns indices 0..3, rank 1 owns 4..6
    if fail_freq is None:
        assert out[0][0] == freqs[:4] and out[1][0] == freqs[4:]
    results, failures = out[0][1]
    for i, f in enumerate(freqs):
        if f == fail_freq:
            assert results[i] is None
        else:
            assert results[i][1] == f and results[i][2] == (0 if i < 4 else 1)
    assert failures == ([] if fail_freq is None else [(freqs.index(fail_freq), fail_freq)])
