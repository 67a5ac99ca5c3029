"""Perplexity trajectory of the small config on the device runner:
the reference's acceptance c7 run (acceptance_main.cpp:467-534: 16 clients,
L2 d32 H2 e4 V64 S32, tau 64, B 4, DiLoCo outer Nesterov eta 0.1 mu 0.9, ring
topology, 5 rounds, held-out perplexity after every round).

Bars: f32 mode follows the oracle's per-round perplexities within 2e-3
relative; bf16 mode (fp32 accumulate, fp32 master) stays within 3 % of them
and ends within 2 % of the fixture the reference authors recorded
(2.9094513044307808, acceptance_main.cpp:472-473)."""
import numpy as np
import pytest

from oracle import ModelCfg, ServerCfg, TrainCfg

pytestmark = pytest.mark.gpu

C7_MODEL = (2, 32, 2, 4, 64, 32)
C7_FIXTURE = 2.9094513044307808


def _oracle_trajectory(oracle):
    cfg = ModelCfg(*C7_MODEL)
    t = TrainCfg(eta_max=3e-3, warmup_steps=32, decay_steps=256, alpha=0.05, local_steps=64,
                 batch_size=4)
    s = ServerCfg(1, 0.1, 0.9, 1)
    theta = oracle.init_params(cfg, 1)
    vel = np.zeros_like(theta)
    plan = oracle.plan_iid(oracle.generate_corpus("web", 200000, 7, 64), 16, 32, 7)
    cursors = np.zeros(16, np.uint64)
    bl = 33
    c = oracle.generate_corpus("web", 64 * bl, oracle.mix_seed(7, 0x4576616C), 64)
    inp = np.concatenate([c[q * bl:q * bl + 32] for q in range(64)]).astype(np.int32)
    tgt = np.concatenate([c[q * bl + 1:q * bl + 33] for q in range(64)]).astype(np.int32)
    traj = []
    for r in range(5):
        oracle.run_round(cfg, t, s, plan, 16, 16, 42, r, theta, vel, cursors, ring=True)
        traj.append(oracle.eval_perplexity(cfg, theta, inp, tgt, [8] * 8, 32))
    return theta, traj


@pytest.fixture(scope="module")
def c7_oracle(oracle):
    theta0 = oracle.init_params(ModelCfg(*C7_MODEL), 1)
    theta, traj = _oracle_trajectory(oracle)
    assert abs(traj[-1] - C7_FIXTURE) <= 1e-9 * C7_FIXTURE  # the oracle is pinned first
    return theta0, traj


@pytest.mark.parametrize("precision,tol", [("f32", 2e-3), ("bf16", 3e-2)])
def test_c7_perplexity_trajectory(F, oracle, c7_oracle, precision, tol):
    theta0, traj = c7_oracle
    model = F.ModelConfig(*C7_MODEL)
    plan = F.partition_iid(oracle.generate_corpus("web", 200000, 7, 64), 16, 32, 7)
    local = F.LocalTrainConfig(model=model, local_steps=64, batch_size=4,
                               schedule=F.LrSchedule(3e-3, 32, 256, 0.05))
    fed = F.FederationConfig(16, 16, 5, F.Topology.kRingAllReduce, 42)
    es = F.EvalSet(["web"], 64, 7, model, 8)
    runner = F.FederationRunner(fed, local, F.ServerOptConfig(1, 0.1, 0.9, True), plan, theta0,
                                precision=precision, eval_set=es, eval_every=1)
    got = [runner.run_round().eval_ppl for _ in range(5)]
    for r, (g, w) in enumerate(zip(got, traj)):
        assert abs(g - w) <= tol * w, (precision, r, g, w)
    if precision == "bf16":
        assert abs(got[-1] - C7_FIXTURE) <= 0.02 * C7_FIXTURE
