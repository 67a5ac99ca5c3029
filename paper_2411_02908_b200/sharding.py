"""Round-boundary sharding protocol of the multi-GPU runner, through the
product's own host logic (`photon_shard_len`, `photon_slot_owner`,
`photon_boundary_peer` in libphoton.so -- the functions runner.cpp and
central.cpp call; no GPU needed), for the CPU tests that run the protocol
over gloo:
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

from . import _capi as A


def owned_slots(k: int, rank: int, world: int) -> List[int]:
    return [si for si in range(k) if A.lib().photon_slot_owner(si, world) == rank]


def shard_layout(n_params: int, world: int) -> Tuple[int, int]:
    """(shard length, padded total)."""
    shard = int(A.lib().photon_shard_len(n_params, world))
    return shard, shard * world


def shard_range(rank: int, n_params: int, world: int) -> Tuple[int, int]:
    shard, _ = shard_layout(n_params, world)
    lo = min(rank * shard, n_params)
    return lo, min(lo + shard, n_params)


def exchange_order(survivors: List[int], world: int) -> List[Tuple[int, int]]:
    """(slot, owner rank) in the order every rank posts its send/recv pairs."""
    return [(si, A.lib().photon_slot_owner(si, world)) for si in survivors]


def peer_boundary(n_params: int, k: int, n_survivors: int, world: int) -> bool:
    """Whether the round takes the NVLink peer-memory kernel (else NCCL)."""
    return bool(A.lib().photon_boundary_peer(n_params, k, n_survivors, world))


def wire_bytes_per_gpu(n_params: int, world: int, elem_bytes: int = 4) -> float:
    """Reduce-scatter + all-gather volume per GPU: 2 (G-1)/G * P * b."""
    return 2.0 * (world - 1) / world * n_params * elem_bytes
