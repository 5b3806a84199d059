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


def _slab_worker(rank, world, port, queue, transport):
    import ctypes as C
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1711_00005_b200 import configs, slab
    seen = {}

    def fake_call(name, handle, g, *args):
        if name == "pe3d_slab_p2p_export":          # (nranks, rank, out): a blob naming the rank
            nranks, rnk, out = args
            C.memmove(out, bytes([rnk + 1]) * slab._native.SLAB_IPC_BYTES, slab._native.SLAB_IPC_BYTES)
            seen["exported"] = (nranks, rnk)
            return
        coeffs, nranks, rnk, blob = args[:4]
        seen.update(name=name, nranks=nranks, rank=rnk, blob=bytes(blob), n_depth=g.n_depth)

    slab.new_nccl_id = lambda: bytes(range(128))
    slab._native.call = fake_call
    slab._native.handle = lambda device=0: None
    cfg = configs.build("cfg5", n_range=3)
    res = slab.distributed_slab_march(cfg, 500.0, device=0, n_steps=2, transport=transport)
    queue.put((rank, seen, res.final.shape, res.tl_field.shape))
    dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_gloo_slab_march_handshake_and_slabs(transport):
    """Host protocol of the distributed slab march on 2 gloo ranks: NCCL
    transport -- rank 0's unique id reaches every rank; peer transport --
    every rank exports its IPC blob and marches with all blobs in rank order."""
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, 2, port, queue, transport)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((lambda t: (t[0], t[1:]))(queue.get(timeout=180)) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    nb = 192
    for rank in (0, 1):
        seen, final_shape, tl_shape = out[rank]
        assert seen["nranks"] == 2 and seen["rank"] == rank
        if transport == "nccl":
            assert seen["name"] == "pe3d_march_slab"
            assert seen["blob"] == bytes(range(128))        # rank 0's NCCL id reached every rank
        else:
            assert seen["name"] == "pe3d_march_slab_p2p" and seen["exported"] == (2, rank)
            assert seen["blob"][:2 * nb] == bytes([1]) * nb + bytes([2]) * nb   # all blobs, rank order
        assert final_shape == (4096, 2048)                 # this rank's depth slab
        assert tl_shape == (1, 4096, 2048)                 # stride 100: starter sample only


def test_slab_shape_rules():
    import math
    from paper_1711_00005_b200.environment import Grid3D
    from paper_1711_00005_b200.errors import InvariantError
    from paper_1711_00005_b200.slab import check_slab_shape, depth_slab
    import numpy as np
    g = Grid3D(3, 64, 256, 1.0, 2 * math.pi / 64, 1.0, 1.0)
    check_slab_shape(g, 4)
    with pytest.raises(InvariantError):
        check_slab_shape(g, 3)
    v = np.arange(64 * 256).reshape(64, 256)
    parts = [depth_slab(v, 4, r) for r in range(4)]
    assert np.array_equal(np.concatenate(parts, axis=1), v)


def _farm_worker(rank, world, port, queue):
    import numpy as np
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1711_00005_b200 import configs, parallel
    cfg = configs.build("cfg4", n_range=6, frequencies=tuple(50.0 + 40.0 * i for i in range(5)), output_stride=3)
    report = parallel.distributed_frequency_farm(cfg, list(cfg.source.frequencies), device=0)
    if rank == 0:
        queue.put((rank, [(r.frequency, np.asarray(r.tl_field).copy(), np.asarray(r.final_slab.values).copy(),
                           r.clamped_samples) for r in report.results], len(report.failures)))
    else:
        queue.put((rank, None, len(report.failures)))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_two_processes_real_frequency_farm():
    """Two real processes (gloo, world size 2) run distributed_frequency_farm
    with the CUDA kernels -- both on device 0 here, each marching its static
    block independently (ref parallel.py:85-97, 143-185; no kernel of one
    process waits for the other's) -- and rank 0's gathered report is bitwise
    the single-process batched march."""
    import numpy as np
    from paper_1711_00005_b200 import configs, march_frequencies
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_farm_worker, args=(r, 2, port, queue)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((t[0], t[1:]) for t in (queue.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    gathered, n_fail = out[0]
    assert n_fail == 0 and out[1][1] == 0
    cfg = configs.build("cfg4", n_range=6, frequencies=tuple(50.0 + 40.0 * i for i in range(5)), output_stride=3)
    ref = march_frequencies(cfg, list(cfg.source.frequencies))
    assert [g[0] for g in gathered] == [r.frequency for r in ref]
    for (f, tl, fin, cl), r in zip(gathered, ref):
        assert tl.tobytes() == np.asarray(r.tl_field).tobytes()
        assert fin.tobytes() == r.final_slab.values.tobytes()
        assert cl == r.clamped_samples
