"""Series-sharded data parallelism: the host-side contract.

Rank r of W owns dataset rows [floor(r*N/W), floor((r+1)*N/W)) — contiguous blocks in
dataset order, so the partition is bit-exact and documented.  Every rank draws the SAME
global shuffled window order from the trainer RNG (make_batches, trainer.hpp:82-102) and
keeps, for each global batch, the windows whose row it owns, in batch order.  Losses and
shared-network gradients are scaled by the GLOBAL mask count M (autodiff.hpp:614), so the
per-rank partial sums add up to the full-batch values; one all-reduce over
[shared grads | per-series squared norm | loss sum] per step then gives every rank the
identical clip scale (trainer.hpp:603-615) and Adam update for the replicated network,
while per-series parameters and their Adam state never leave their owner.

The C++ engine implements exactly this (csrc/engine.cu: esrnn_trainer_create row0/N,
append_step filtering, K3 partials, ncclAllReduce, k_finalize); this module is the
reference used by the multi-process tests and by bench.py.
"""
from __future__ import annotations


def shard_range(rank: int, world: int, n: int) -> tuple[int, int]:
    """Rows [begin, end) owned by `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("rank out of range")
    return (rank * n) // world, ((rank + 1) * n) // world


def local_windows(rows, anchors, rank: int, world: int, n: int):
    """Indices (into the global batch) of the windows `rank` owns, in batch order."""
    b, e = shard_range(rank, world, n)
    return [i for i, r in enumerate(rows) if b <= r < e]


def slots_first_appearance(rows) -> list:
    """Slot order of a (local) batch: series rows in first-appearance order (trainer.hpp:494-501)."""
    seen, out = set(), []
    for r in rows:
        if r not in seen:
            seen.add(r)
            out.append(r)
    return out


LOCAL_PARTIALS_ID = bytes([0xEE]) * 128
"""esrnn_dist.nccl_unique_id value that runs a shard's data path without the collective,
so a test can sum the per-rank partials itself (one GPU, several ranks)."""
