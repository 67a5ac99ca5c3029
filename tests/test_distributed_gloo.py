"""The multi-GPU round boundary, run on CPU with world_size = 2 over gloo.

Each rank owns slots si % world == rank, scatters shards of its client models in
ascending slot order (the send/recv order of runner.cpp), applies the fused
anchored-mean -> pseudo-gradient -> outer step on its shard in f64, and
all-gathers theta_{t+1}.  The result must be bit-identical to the
single-process reference aggregation (oracle: param_vector.cpp:127-152 +
optim.cpp:124-159) for every world size -- the property that lets the GPU
runner's output not depend on the GPU count (test_aggregator.cpp:138-159)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fused_update(models, theta, vel, kind, eta, mu, nesterov):
    """Element-wise restatement of optim.cu's aggregate_kernel (f64)."""
    anchor = models[0]
    corr = np.zeros_like(anchor)
    for m in models[1:]:
        corr = corr + (m - anchor)
    mean = np.where(corr != 0.0, anchor + corr / float(len(models)), anchor)
    if kind == 0:
        return mean, vel
    delta = theta + (-1.0) * mean
    vel = mu * vel + delta
    if eta == 1.0 and mu == 0.0:
        return mean, vel
    direction = mu * vel + delta if nesterov else vel
    return theta - eta * direction, vel


def _worker(rank, world, port, P, K, dropped, server, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2411_02908_b200.sharding import exchange_order, owned_slots, shard_layout

    rng = np.random.default_rng(0)
    theta = rng.normal(size=P) * 0.02
    vel0 = rng.normal(size=P) * 1e-3
    models = [theta + rng.normal(size=P) * 1e-3 for _ in range(K)]  # identical on all ranks
    shard, ppad = shard_layout(P, world)
    pad = lambda a: np.concatenate([a, np.zeros(ppad - P)])  # noqa: E731
    mine = owned_slots(K, rank, world)
    survivors = [si for si in range(K) if si not in dropped]
    # scatter: every survivor's model shard-wise to the owners, ascending slot order
    recv = []
    for si, owner in exchange_order(survivors, world):
        parts = [torch.zeros(shard, dtype=torch.float64) for _ in range(world)]
        if owner == rank:
            assert si in mine
            full = torch.from_numpy(pad(models[si]))
            send = list(full.split(shard))
        else:
            send = [torch.zeros(shard, dtype=torch.float64) for _ in range(world)]
        # the owner's shard q goes to rank q (gloo: scatter from the owner)
        dist.scatter(parts[rank], send if owner == rank else None, src=owner)
        recv.append(parts[rank].numpy().copy())
    lo = rank * shard
    th_s = pad(theta)[lo:lo + shard]
    v_s = pad(vel0)[lo:lo + shard]
    new_s, v_s = fused_update(recv, th_s, v_s, *server)
    gathered = [torch.zeros(shard, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(new_s))
    vg = [torch.zeros(shard, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(vg, torch.from_numpy(v_s))
    if rank == 0:
        out_q.put((torch.cat(gathered).numpy()[:P], torch.cat(vg).numpy()[:P]))
    dist.destroy_process_group()


@pytest.mark.parametrize("server", [(0, 1.0, 0.0, 0), (1, 0.1, 0.9, 1), (1, 0.5, 0.3, 0)])
@pytest.mark.parametrize("P,K,dropped", [(10007, 4, ()), (4099, 3, (1,)), (64, 2, ())])
def test_sharded_round_boundary_world2(oracle, server, P, K, dropped):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, P, K, dropped, server, q))
             for r in range(world)]
    for p in procs:
        p.start()
    theta_new, vel_new = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference aggregation through the oracle
    from oracle import ServerCfg

    rng = np.random.default_rng(0)
    theta = rng.normal(size=P) * 0.02
    vel = rng.normal(size=P) * 1e-3
    models = [theta + rng.normal(size=P) * 1e-3 for _ in range(K)]
    surv = [models[i] for i in range(K) if i not in dropped]
    mean = oracle.mean(surv)
    delta = oracle.sub(theta, mean)
    want = oracle.server_step(ServerCfg(*server), theta, delta, mean, vel)
    assert theta_new.tobytes() == want.tobytes()
    if server[0] == 1:
        assert vel_new.tobytes() == vel.tobytes()


def test_slot_ownership_and_volume():
    from paper_2411_02908_b200.sharding import (owned_slots, shard_layout, shard_range,
                                                wire_bytes_per_gpu)

    for K, world in ((8, 8), (16, 8), (3, 2), (5, 4)):
        owned = sorted(s for r in range(world) for s in owned_slots(K, r, world))
        assert owned == list(range(K))
    shard, ppad = shard_layout(164044480, 8)
    assert shard % 4 == 0 and ppad >= 164044480 and ppad - 164044480 < 32
    covered = sum(hi - lo for lo, hi in (shard_range(r, 1001, 3) for r in range(3)))
    assert covered == 1001
    assert wire_bytes_per_gpu(164044480, 8) == pytest.approx(2 * 7 / 8 * 164044480 * 4)


def test_peer_boundary_decision(monkeypatch):
    """The NVLink peer-memory boundary vs the NCCL path (runner.cpp, host.hpp
    peer_round_ok): decided from quantities every rank shares, so a rank that
    holds more local models than the peer kernel takes sends every rank down
    the NCCL path together (K = 33 on 2 GPUs, 17 dropouts)."""
    from paper_2411_02908_b200.sharding import peer_boundary

    P = 164044480
    assert peer_boundary(P, 8, 8, 8)
    assert peer_boundary(P, 2, 2, 2)
    assert not peer_boundary(P, 33, 16, 2)   # busiest rank holds 17 > 16 models
    assert not peer_boundary(P, 20, 17, 4)   # 17 survivors > 16
    assert not peer_boundary(6865216704, 4, 4, 4)  # 27.5 GB replicas: NCCL path
    assert not peer_boundary(P, 1, 1, 1)     # one GPU: no boundary exchange
    monkeypatch.setenv("PHOTON_BOUNDARY", "nccl")
    assert not peer_boundary(P, 8, 8, 8)
    monkeypatch.setenv("PHOTON_BOUNDARY", "p2p")
    assert peer_boundary(6865216704, 4, 4, 4)


def _decision_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2411_02908_b200.sharding import owned_slots, peer_boundary

    rng = np.random.default_rng(rank)  # each rank draws its own dropout pattern ...
    cases = [(k, n) for k in (2, 16, 33, 40) for n in range(1, k + 1, 3)]
    mine = torch.tensor([int(peer_boundary(164044480, k, n, world)) for k, n in cases])
    local = torch.tensor([len(owned_slots(k, rank, world)) for k, _ in cases])
    del rng  # ... but the decision only reads shared quantities
    allm = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allm, mine)
    alll = [torch.zeros_like(local) for _ in range(world)]
    dist.all_gather(alll, local)
    if rank == 0:
        out_q.put(([a.tolist() for a in allm], [a.tolist() for a in alll], cases))
    dist.destroy_process_group()


def test_peer_boundary_decision_agrees_across_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_decision_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    decisions, local_counts, cases = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert decisions[0] == decisions[1]
    for (k, n), d, l0, l1 in zip(cases, decisions[0], local_counts[0], local_counts[1]):
        # the peer path only when the busiest rank's models fit its tables
        assert d == int(n <= 16 and max(l0, l1) <= 16), (k, n)
