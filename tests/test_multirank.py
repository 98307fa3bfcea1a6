"""World-size-2 gloo tests (CPU) of the multi-GPU host logic used by bench.py."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_17785_b200 import dist as sdist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from synth import get_params, key_randomness, lwe_randomness
        P = get_params("TOY")
        # keys replicated: identical draws on every rank
        k = key_randomness(P, 7)["lwe_key"]
        kt = torch.from_numpy(k.astype(np.int64))
        gathered = [torch.zeros_like(kt) for _ in range(world)]
        dist.all_gather(gathered, kt)
        keys_equal = all(torch.equal(gathered[0], g) for g in gathered)
        # inputs sharded: per-rank seeds give distinct ciphertext masks
        m = lwe_randomness(P, 4, sdist.input_seed(7, rank))["mask"]
        mt = torch.from_numpy(m.view(np.int64).copy())
        gm = [torch.zeros_like(mt) for _ in range(world)]
        dist.all_gather(gm, mt)
        inputs_distinct = not torch.equal(gm[0], gm[1])
        # max-over-ranks timing and whole-job throughput
        t = 1.0 + rank  # rank 1 is the slow one
        tmax = sdist.max_over_ranks(t)
        fails = sdist.sum_over_ranks(rank)
        thr = sdist.aggregate_throughput(world, 100, 3, tmax)
        q.put((rank, keys_equal, inputs_distinct, tmax, fails, thr))
    finally:
        dist.destroy_process_group()


def test_two_rank_weak_scaling_logic():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, keys_equal, inputs_distinct, tmax, fails, thr in res:
        assert keys_equal and inputs_distinct
        assert tmax == 2.0  # the slowest rank's time
        assert fails == 1
        assert thr == 2 * 100 * 3 / 2.0


def test_shard_bounds_cover_exactly():
    for total in [0, 1, 7, 131072]:
        for world in [1, 2, 3, 8]:
            spans = [sdist.shard_bounds(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def _worker_moduli(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        base = [5, 7, 9, 11, 13, 16]
        idx, mods = sdist.shard_moduli(base, world, rank)
        # stand-in for this rank's Matmul^RNS channels: residue "ciphertexts" tagged by modulus
        local = torch.stack([torch.full((2, 3, 4), m, dtype=torch.int64) for m in mods])
        full = sdist.gather_channels(local, len(base), world, rank)
        q.put((rank, idx, [int(full[i, 0, 0, 0]) for i in range(len(base))]))
    finally:
        dist.destroy_process_group()


def test_two_rank_modulus_sharding():
    """Config-3 sharding by modulus: the ranks' channels partition
    the base and the all-gather returns every channel in modulus order."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_moduli, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(res[0][1] + res[1][1]) == list(range(6))
    for _, _, order in res:
        assert order == [5, 7, 9, 11, 13, 16]


def _worker_rows(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        k, a, c = 6, 5, 3
        lo, hi = sdist.shard_rows(a, world, rank)
        # stand-in for this rank's Matmul^RNS output rows: values tagged (modulus index, row, col)
        local = torch.tensor([[[100 * mi + 10 * row + col for col in range(c)] for row in range(lo, hi)]
                              for mi in range(k)], dtype=torch.int64).reshape(k, hi - lo, c, 1)
        full = sdist.gather_rows(local, a, world, rank)
        q.put((rank, (lo, hi), full.reshape(k, a, c).tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_output_row_sharding():
    """Config-3 sharding by output tile: the ranks' row blocks
    partition the 5 output rows (uneven split), and the all-gather returns the
    full [k][a][c] output, rows in order, on every rank."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_rows, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == (0, 3) and res[1][1] == (3, 5)
    want = [[[100 * mi + 10 * row + col for col in range(3)] for row in range(5)] for mi in range(6)]
    for _, _, full in res:
        assert full == want
    # 16 rows over 8 ranks (configs[3] on 8 GPUs): 2 rows each
    assert [sdist.shard_rows(16, 8, r)[1] - sdist.shard_rows(16, 8, r)[0] for r in range(8)] == [2] * 8
