"""Multi-rank host logic on CPU (gloo, world size 2): slice sharding, coil-sharded
normal operator (partial sums + all-reduce), gather.  The per-rank operators are
oracle (numpy) operators, so this checks the partition arithmetic the GPU path uses."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sketch_oracle as O
from paper_2305_06482_b200.parallel_recon import CoilShard, gather_slices, readout_phases, shard_range, sharded_normal


def test_shard_range_partitions():
    for n in (0, 1, 7, 64, 256, 257):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_readout_phases_give_centered_idft():
    rng = np.random.default_rng(0)
    for n in (8, 16, 256, 10):
        k = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        pre, post = readout_phases(n)
        got = post * (np.fft.ifft(k * pre) * n)
        ref = O.centered_dft(k, 1, inverse=True)
        assert np.allclose(got, ref, atol=1e-12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(1)
        dims = (16, 12)
        pts = np.argwhere(rng.random(dims) < 0.4) - np.array([8, 6])
        kern = O.CartesianKernel(dims, pts)
        C = 5
        maps = rng.standard_normal((C, 192)) + 1j * rng.standard_normal((C, 192))
        x = rng.standard_normal(192) + 1j * rng.standard_normal(192)
        shard = CoilShard(rank, world)
        lo, hi = shard.coils(C)

        def partial(v):
            return torch.from_numpy(O.Sense(maps[lo:hi], kern).normal(v.numpy()))

        got = sharded_normal(partial, torch.from_numpy(x), shard).numpy()
        ref = O.Sense(maps, kern).normal(x)
        err_normal = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        # slice sharding + gather
        nslice = 7
        a, b = shard_range(nslice, rank, world)
        local = torch.arange(a, b, dtype=torch.float64).reshape(-1, 1) * torch.ones(1, 3, dtype=torch.float64)
        full = gather_slices(local, nslice, rank, world)
        ok_gather = True if rank != 0 else bool(torch.equal(full[:, 0], torch.arange(nslice, dtype=torch.float64)))
        q.put((rank, err_normal, ok_gather))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_coil_sharded_normal_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, ok in res:
        assert err < 1e-12, (rank, err)
        assert ok
