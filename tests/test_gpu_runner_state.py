"""SURVEY 8(f) rows 1-2 on the device runner: per-round evaluation on the
held-out set (aggregator.cpp:207-212, model.cpp:176-192) and PHCK resume
(harness.cpp:802-905, acceptance c10).

Bars: the eval cadence fires exactly when the reference's does; eval_ppl equals
the oracle's perplexity of the runner's own theta_{t+1} (f32 mode, rel 1e-5);
a run interrupted after 2 rounds, saved and resumed by a fresh runner ends
bit-identical (theta, velocity, cursors) to an uninterrupted run; the written
checkpoint.phck is readable by the reference reader when oracle/_ref exists."""
import math

import numpy as np
import pytest

from oracle import ModelCfg, load_reference

pytestmark = pytest.mark.gpu

HETERO4 = (1, 32, 2, 4, 64, 16)


def _setup(F, oracle, rounds, server=(1, 0.1, 0.9, True), precision="f32"):
    mc = ModelCfg(*HETERO4)
    theta0 = oracle.init_params(mc, 1)
    corpus = oracle.generate_corpus("web", 200000, 7, 64)
    plan = F.partition_iid(corpus, 3, 16, 7)
    local = F.LocalTrainConfig(model=F.ModelConfig(*HETERO4), local_steps=8, batch_size=4,
                               schedule=F.LrSchedule(2e-3, 16, 160, 0.1))
    fed = F.FederationConfig(3, 2, rounds, F.Topology.kParameterServer, 42)
    srv = F.ServerOptConfig(*server)
    es = F.EvalSet(["web"], 24, 7, F.ModelConfig(*HETERO4), 8)
    return mc, theta0, plan, local, fed, srv, es


def test_eval_cadence_and_value(F, oracle):
    mc, theta0, plan, local, fed, srv, es = _setup(F, oracle, rounds=5)
    runner = F.FederationRunner(fed, local, srv, plan, theta0, precision="f32", eval_set=es,
                                eval_every=2)
    bs = es.batches()
    inp = np.concatenate([b.inputs for b in bs])
    tgt = np.concatenate([b.targets for b in bs])
    sizes = [b.batch_size for b in bs]
    init = runner.evaluate()
    assert abs(init - oracle.eval_perplexity(mc, theta0, inp, tgt, sizes, 16)) <= 1e-5 * init
    fired = []
    for r in range(5):
        rec = runner.run_round()
        if math.isnan(rec.eval_ppl):
            continue
        fired.append(r)
        want = oracle.eval_perplexity(mc, runner.theta(), inp, tgt, sizes, 16)
        assert abs(rec.eval_ppl - want) <= 1e-5 * want
    # round % every == every - 1, plus the final round (aggregator.cpp:207-212)
    assert fired == [1, 3, 4]


@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_save_resume_bitwise(F, oracle, tmp_path, precision):
    mc, theta0, plan, local, fed, srv, es = _setup(F, oracle, rounds=4)
    full = F.FederationRunner(fed, local, srv, plan, theta0, precision=precision)
    for _ in range(4):
        full.run_round()
    part = F.FederationRunner(fed, local, srv, plan, theta0, precision=precision)
    part.run_round()
    part.run_round()
    d = str(tmp_path)
    part.save(d)
    del part
    fresh = F.FederationRunner(fed, local, srv, plan, oracle.init_params(mc, 99),
                               precision=precision)
    fresh.resume(d)
    assert fresh.next_round() == 2
    while not fresh.done():
        fresh.run_round()
    assert fresh.theta().tobytes() == full.theta().tobytes()
    assert fresh.velocity().tobytes() == full.velocity().tobytes()
    for c in range(3):
        assert fresh.client_cursor(c) == full.client_cursor(c)
    ref = load_reference()
    if ref is not None:
        th, rd = ref.read_checkpoint(mc, d + "/checkpoint.phck")
        assert rd == 2 and np.all(np.isfinite(th))


def test_resume_errors(F, oracle, tmp_path):
    mc, theta0, plan, local, fed, srv, es = _setup(F, oracle, rounds=3)
    runner = F.FederationRunner(fed, local, srv, plan, theta0)
    with pytest.raises(F.IoError):
        runner.resume(str(tmp_path))  # nothing to resume
    runner.run_round()
    runner.save(str(tmp_path))
    import os
    os.remove(str(tmp_path / "velocity.phck"))
    with pytest.raises(F.IntegrityError):
        F.FederationRunner(fed, local, srv, plan, theta0).resume(str(tmp_path))
    other = F.FederationConfig(4, 2, 3, F.Topology.kParameterServer, 42)
    plan4 = F.partition_iid(oracle.generate_corpus("web", 200000, 7, 64), 4, 16, 7)
    runner.save(str(tmp_path))
    with pytest.raises(F.IntegrityError):  # population changed
        F.FederationRunner(other, local, srv, plan4, theta0).resume(str(tmp_path))


def test_token_pipeline_prefetch(F, oracle):
    """round t+1's batches are staged while round t trains, so
    only round 0 (and a round after restore) stages on the critical path; the
    token streams are unchanged (the oracle comparisons of test_gpu_parity.py
    run multi-round on prefetched batches)."""
    mc, theta0, plan, local, fed, srv, es = _setup(F, oracle, rounds=4)
    runner = F.FederationRunner(fed, local, srv, plan, theta0)
    recs = [runner.run_round() for _ in range(2)]
    assert recs[0].host_ms > 0 and recs[1].host_ms == 0
    runner.restore(runner.theta(), runner.velocity(), 2,
                   [runner.client_cursor(c) for c in range(3)])
    assert runner.run_round().host_ms > 0  # the restore dropped the prefetch
    assert runner.run_round().host_ms == 0


@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_topology_invariance(F, oracle, precision):
    # acceptance c6 (acceptance_main.cpp:390-463): the topology only changes the
    # reference's cost model, so theta, velocity and cursors after the rounds
    # are bit-identical for parameter-server, all-reduce and ring all-reduce
    mc, theta0, plan, local, _, srv, _ = _setup(F, oracle, 3, precision=precision)
    out = []
    for topo in (F.Topology.kParameterServer, F.Topology.kAllReduce, F.Topology.kRingAllReduce):
        r = F.FederationRunner(F.FederationConfig(3, 2, 3, topo, 42), local, srv, plan, theta0,
                               precision=precision)
        losses = [r.run_round().mean_client_loss for _ in range(3)]
        out.append((losses, r.theta().tobytes(), r.velocity().tobytes(),
                    [r.client_cursor(c) for c in range(3)]))
    for o in out[1:]:
        assert o == out[0]
