"""Multi-GPU host logic: weak-scaling shards of independent ciphertexts.

PBS ciphertexts are independent: each rank bootstraps its
own batch with keys generated locally from the same key seed (replicated), so
the data path has no collective. The only collectives are the barrier around
the timed region and the max-over-ranks reduction of elapsed time.
"""
import torch
import torch.distributed as dist


def input_seed(seed: int, rank: int) -> int:
    """Per-rank seed for ciphertext inputs (keys use `seed` on every rank)."""
    return seed + 1000 * rank


def shard_bounds(total: int, world: int, rank: int):
    """Contiguous shard [lo, hi) of `total` independent ciphertexts for `rank`
    (strong-scaling helper; bench.py uses weak scaling, one full batch per rank)."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def max_over_ranks(x: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: int, device=None) -> int:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return int(x)
    t = torch.tensor([int(x)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())


def aggregate_throughput(world: int, batch_per_rank: int, steps: int, max_seconds: float) -> float:
    """Whole-job PBS/s: units all ranks processed / the slowest rank's time."""
    return world * batch_per_rank * steps / max_seconds


# ---------------------------------------------------- gadget-layer sharding
# Matmul^RNS (config 3) shards by modulus -- the k residue
# channels are independent -- with the keys replicated on every rank; the only
# collective is one all-gather of the residue ciphertexts at the end.
def shard_moduli(moduli, world: int, rank: int):
    """Round-robin modulus channels of this rank: (indices, moduli)."""
    idx = list(range(rank, len(moduli), world))
    return idx, [moduli[i] for i in idx]


def gather_channels(local: torch.Tensor, k: int, world: int, rank: int) -> torch.Tensor:
    """local [k_rank][...] residue ciphertexts of this rank's channels ->
    [k][...] on every rank, channels back in modulus order (all_gather of
    equal-sized, zero-padded slabs)."""
    per = (k + world - 1) // world
    slab = torch.zeros((per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    slab[: local.shape[0]] = local
    if world == 1:
        return slab[:k].clone()
    parts = [torch.empty_like(slab) for _ in range(world)]
    dist.all_gather(parts, slab)
    out = torch.empty((k,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    for r in range(world):
        idx = list(range(r, k, world))
        out[idx] = parts[r][: len(idx)]
    return out


# Output-tile sharding of Matmul^RNS (SURVEY.md §8(e) "or by output tile"):
# rank r computes the rows [lo, hi) of X W for every modulus. Every row costs
# the same number of PBS, so any world size up to the row count is balanced
# (modulus sharding caps at k ranks and is unbalanced: m in {9, 11, 13} cost
# 4 PBS per product, {5, 7} 2). One all-gather returns the full output.
def shard_rows(a: int, world: int, rank: int):
    """Rows [lo, hi) of the a-row output owned by `rank`."""
    return shard_bounds(a, world, rank)


def gather_rows(local: torch.Tensor, a: int, world: int, rank: int) -> torch.Tensor:
    """local [k][rows of this rank][c][...] -> [k][a][c][...] on every rank
    (all_gather of equal-sized, zero-padded slabs, rows back in order)."""
    per = (a + world - 1) // world
    shape = (local.shape[0], per) + tuple(local.shape[2:])
    slab = torch.zeros(shape, dtype=local.dtype, device=local.device)
    slab[:, : local.shape[1]] = local
    if world == 1:
        return slab[:, :a].clone()
    parts = [torch.empty_like(slab) for _ in range(world)]
    dist.all_gather(parts, slab)
    out = torch.empty((local.shape[0], a) + tuple(local.shape[2:]), dtype=local.dtype, device=local.device)
    for r in range(world):
        lo, hi = shard_rows(a, world, r)
        out[:, lo:hi] = parts[r][:, : hi - lo]
    return out
