"""Round-boundary sharding protocol of the multi-GPU runner (runner.cpp).

Pure host logic, shared by the C++ runner (which implements it over NCCL) and
the CPU tests (which run it over gloo):
  * sampled slot si (ascending client id) trains on rank si % world;
  * the flat canonical parameter vector is cut into `world` contiguous shards
    of `shard` elements (padded to a multiple of 4 for 128-bit access);
  * every surviving slot's model is scattered shard-wise to the shard owners
    in ascending slot order, so each owner sees its shard of every model in
    the reference's canonical aggregation order (aggregator.cpp:177);
  * owners apply the anchored mean -> pseudo-gradient -> outer step on their
    shard; an all-gather rebuilds theta_{t+1} everywhere.
"""
from __future__ import annotations

from typing import List, Tuple


def owned_slots(k: int, rank: int, world: int) -> List[int]:
    return [si for si in range(k) if si % world == rank]


def shard_layout(n_params: int, world: int) -> Tuple[int, int]:
    """(shard length, padded total) -- runner.cpp: shard = ceil(P/G) up to 4."""
    shard = ((n_params + world - 1) // world + 3) // 4 * 4
    return shard, shard * world


def shard_range(rank: int, n_params: int, world: int) -> Tuple[int, int]:
    shard, _ = shard_layout(n_params, world)
    lo = min(rank * shard, n_params)
    return lo, min(lo + shard, n_params)


def exchange_order(survivors: List[int], world: int) -> List[Tuple[int, int]]:
    """(slot, owner rank) in the order every rank posts its send/recv pairs."""
    return [(si, si % world) for si in survivors]


def wire_bytes_per_gpu(n_params: int, world: int, elem_bytes: int = 4) -> float:
    """Reduce-scatter + all-gather volume per GPU: 2 (G-1)/G * P * b."""
    return 2.0 * (world - 1) / world * n_params * elem_bytes
