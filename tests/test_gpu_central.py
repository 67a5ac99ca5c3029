"""Device centralized / DDP baseline (run_centralized, baselines.cpp:25-127)
vs the oracle composition pinned to the reference (tests/test_central.py).

Bars: f32 mode -- per-step mean loss rel <= 1e-5, parameters max-abs <= 2e-4
after 6 steps (AdamW with an optimizer reset, and SGD); cursors exact.
Acceptance c3 at device scale: one worker with opt_reset_interval = tau is the
K = 1 federation (FedAvg of one model is the model), bit for bit, in f32 and
bf16.  Config / divergence errors map to the reference's exception types."""
import numpy as np
import pytest

from central_case import oracle_centralized
from oracle import ModelCfg, TrainCfg

pytestmark = pytest.mark.gpu

HETERO4 = (1, 32, 2, 4, 64, 16)


def _cfg(F, opt=0, n_workers=2, steps=6, reset=3, gb=4):
    return F.CentralizedConfig(model=F.ModelConfig(*HETERO4),
                               schedule=F.LrSchedule(2e-3, 2, 16, 0.1), opt=opt,
                               sgd_clip_norm=1.0, n_workers=n_workers, global_batch=gb,
                               total_steps=steps, opt_reset_interval=reset)


@pytest.mark.parametrize("opt,reset", [(0, 3), (1, 0)])
def test_central_vs_oracle_f32(F, oracle, opt, reset):
    mc = ModelCfg(*HETERO4)
    theta0 = oracle.init_params(mc, 1)
    corpus = oracle.generate_corpus("web", 20000, 7, 64)
    t = TrainCfg(eta_max=2e-3, warmup_steps=2, decay_steps=16, alpha=0.1, opt=opt,
                 sgd_clip_norm=1.0, batch_size=4)
    th_o, loss_o, cur_o = oracle_centralized(oracle, mc, t, corpus, 2, 6, reset, 42, 7, theta0)
    plan = F.partition_iid(corpus, 2, 16, 7)
    res = F.run_centralized(_cfg(F, opt=opt, reset=reset), plan, 42, theta0, precision="f32")
    for s, lo in zip(res.steps, loss_o):
        assert abs(s.loss - lo) / lo <= 1e-5
        assert s.tokens == 4 * 16
    assert np.max(np.abs(res.theta - th_o)) <= 2e-4
    assert res.cursors == cur_o and res.sync_events == 6


@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_c3_central_is_k1_federation(F, oracle, precision):
    """acceptance_main.cpp c3 on the device: centralized(n=1, reset=tau) == K=1 FedAvg."""
    mc = ModelCfg(*HETERO4)
    theta0 = oracle.init_params(mc, 2)
    corpus = oracle.generate_corpus("web", 20000, 7, 64)
    plan = F.partition_iid(corpus, 1, 16, 7)
    tau, rounds = 4, 2
    cen = F.run_centralized(_cfg(F, n_workers=1, steps=tau * rounds, reset=tau, gb=4), plan, 42,
                            theta0, precision=precision)
    local = F.LocalTrainConfig(model=F.ModelConfig(*HETERO4),
                               schedule=F.LrSchedule(2e-3, 2, 16, 0.1), local_steps=tau,
                               batch_size=4)
    fed = F.FederationRunner(F.FederationConfig(1, 1, rounds, F.Topology.kParameterServer, 42),
                             local, F.ServerOptConfig(), plan, theta0, precision=precision)
    for _ in range(rounds):
        fed.run_round()
    assert cen.theta.tobytes() == fed.theta().tobytes()
    assert cen.cursors == [fed.client_cursor(0)]


def test_central_errors(F, oracle):
    mc = ModelCfg(*HETERO4)
    theta0 = oracle.init_params(mc, 1)
    plan = F.partition_iid(oracle.generate_corpus("web", 20000, 7, 64), 2, 16, 7)
    with pytest.raises(F.ConfigError):  # global batch must divide by n_workers
        F.CentralizedTrainer(_cfg(F, n_workers=2, gb=3), plan, 42, theta0)
    with pytest.raises(F.ConfigError):  # plan too small
        F.CentralizedTrainer(_cfg(F, n_workers=4, gb=4), plan, 42, theta0)
    bad = theta0.copy()
    bad[-1] = np.nan  # head.b: every row's logits
    tr = F.CentralizedTrainer(_cfg(F), plan, 42, bad)
    with pytest.raises(F.DivergenceError) as ei:
        tr.step()
    assert ei.value.step == 0
    tr = F.CentralizedTrainer(_cfg(F, steps=1), plan, 42, theta0)
    tr.step()
    with pytest.raises(F.UsageError):
        tr.step()
