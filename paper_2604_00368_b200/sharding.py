"""Multi-GPU partitioning of the data plane: every intent is independent
and every slice writes an absolute destination range, so ranks shard units with no
data-path collective. One process per GPU; torch.distributed is only plumbing (rendezvous,
IPC-handle exchange, barrier, max-over-ranks timing)."""
from __future__ import annotations

from typing import List, Tuple


def kv_shard(n_blocks: int, rank: int, world: int) -> Tuple[int, int]:
    """[first, last) of the KV blocks rank owns (config 3 is per GPU / PCIe root: weak
    scaling gives every rank the full per-GPU batch; this helper splits a shared one)."""
    base, extra = divmod(n_blocks, world)
    first = rank * base + min(rank, extra)
    return first, first + base + (1 if rank < extra else 0)


def flow_peer(rank: int, world: int) -> int:
    """Elephant-flow permutation i -> (i+1) mod N (config 2 at N GPUs: disjoint flows)."""
    return (rank + 1) % world


def broadcast_tree(world: int, root: int = 0) -> List[Tuple[int, int]]:
    """Pipelined relay chain for the weight broadcast (config 4): root -> r1 -> r2 ...,
    each receiver forwards what it received, so every link carries the payload once."""
    order = [root] + [r for r in range(world) if r != root]
    return [(order[i], order[i + 1]) for i in range(len(order) - 1)]
