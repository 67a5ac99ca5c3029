"""GPU parity: the CUDA path through the C ABI vs the CPU oracle.

Tolerances (stated, per precision mode; the oracle is the reference's f64 math):
  f64 aggregation / optimizer entry points: bit-exact.
  f32 mode (fp32 storage, fp32 SIMT contractions): loss rel <= 1e-5, gradient
      rel-L2 <= 1e-4; local round (AdamW) loss rel <= 1e-4, weights max-abs <= 2e-4.
  bf16 mode (bf16 operands, fp32 accumulate): loss rel <= 2e-2, gradient
      rel-L2 <= 6e-2.
"""
import numpy as np
import pytest

from oracle import ModelCfg, ServerCfg, TrainCfg

pytestmark = pytest.mark.gpu

TINY = (1, 8, 2, 4, 16, 4)
HETERO4 = (1, 32, 2, 4, 64, 16)   # configs/hetero4.cfg:15-21 (BASELINE config #1)
DEFAULT = (2, 64, 2, 4, 64, 32)   # ModelConfig{} model.h:12-18
DILOCO = (2, 32, 2, 4, 64, 32)    # configs/diloco.cfg, acceptance c7
WIDE128 = (1, 128, 2, 4, 96, 32)  # d = 128 * NV: register-resident LayerNorm kernels
WIDE256 = (1, 256, 4, 4, 96, 160)  # dh = 64: tcgen05 attention, ragged S
WIDE1024 = (1, 1024, 16, 4, 96, 32)  # d = 512 * 2: row-split LayerNorm kernels
WIDE2048 = (1, 2048, 16, 4, 96, 16)  # d = 512 * 4, dh = 128 (the 1.3B widths)


def _mc(F, t):
    return F.ModelConfig(*t)


def _batch(oracle, cfg_t, B, seed=7, client=0, tokens=20000, shards=2):
    V, S = cfg_t[4], cfg_t[5]
    corpus = oracle.generate_corpus("web", tokens, seed, V)
    plan = oracle.plan_iid(corpus, shards, S, seed)
    inp, tgt, _ = oracle.stream_next(plan, client, B, oracle.stream_seed(42, client), 0)
    return inp, tgt


def _rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("cfg_t,B", [(TINY, 2), (HETERO4, 4), (DEFAULT, 4), (WIDE128, 2),
                                     (WIDE256, 2), (WIDE1024, 2), (WIDE2048, 2)])
def test_forward_backward_f32(F, oracle, cfg_t, B):
    mc = ModelCfg(*cfg_t)
    params = oracle.init_params(mc, 3)
    inp, tgt = _batch(oracle, cfg_t, B)
    l_ref, g_ref = oracle.forward_backward(mc, params, inp, tgt, B, cfg_t[5])
    model = F.TransformerModel(_mc(F, cfg_t), precision="f32", max_batch=B)
    loss, g = model.forward_loss(params, F.Batch(inp, tgt, B, cfg_t[5]))
    assert abs(loss - l_ref) / abs(l_ref) <= 1e-5
    assert _rel_l2(g, g_ref) <= 1e-4
    # every canonical entry individually (no entry silently dropped)
    for name, off, shape in model.layout():
        n = int(np.prod(shape))
        gr = g_ref[off:off + n]
        if np.linalg.norm(gr) > 1e-8:
            assert _rel_l2(g[off:off + n], gr) <= 5e-4, name


@pytest.mark.parametrize("cfg_t,B", [(HETERO4, 4), (DEFAULT, 4), (WIDE128, 2), (WIDE256, 2),
                                     (WIDE1024, 2), (WIDE2048, 2)])
def test_forward_backward_bf16(F, oracle, cfg_t, B):
    mc = ModelCfg(*cfg_t)
    params = oracle.init_params(mc, 3)
    inp, tgt = _batch(oracle, cfg_t, B)
    l_ref, g_ref = oracle.forward_backward(mc, params, inp, tgt, B, cfg_t[5])
    model = F.TransformerModel(_mc(F, cfg_t), precision="bf16", max_batch=B)
    loss, g = model.forward_loss(params, F.Batch(inp, tgt, B, cfg_t[5]))
    assert abs(loss - l_ref) / abs(l_ref) <= 2e-2
    assert _rel_l2(g, g_ref) <= 6e-2


def test_forward_only_and_eval_perplexity(F, oracle):
    cfg_t = HETERO4
    mc = ModelCfg(*cfg_t)
    params = oracle.init_params(mc, 1)
    corpus = oracle.generate_corpus("web", 20000, 11, 64)
    plan = oracle.plan_iid(corpus, 1, 16, 3)
    batches, ins, tgs = [], [], []
    cur = 0
    for bs in (4, 4, 3):
        i, t, cur = oracle.stream_next(plan, 0, bs, 5, cur)
        batches.append(F.Batch(i, t, bs, 16))
        ins.append(i)
        tgs.append(t)
    ppl_ref = oracle.eval_perplexity(mc, params, np.concatenate(ins), np.concatenate(tgs),
                                     [4, 4, 3], 16)
    model = F.TransformerModel(_mc(F, cfg_t), precision="f32", max_batch=4)
    ppl = model.eval_perplexity(params, batches)
    assert abs(ppl - ppl_ref) / ppl_ref <= 1e-5
    # init perplexity band of the reference's unit test (test_model.cpp:173-187)
    assert 40.0 < ppl < 90.0


def test_f64_aggregation_bit_exact(F, oracle):
    rng = np.random.default_rng(0)
    n = 10007
    for k in (1, 2, 3, 5, 8):
        models = [rng.normal(size=n) * 0.02 for _ in range(k)]
        theta = rng.normal(size=n) * 0.02
        assert np.array_equal(F.ParamVector.mean(models), oracle.mean(models))
        assert np.array_equal(F.ParamVector.sub(theta, models[0]), oracle.sub(theta, models[0]))
        for kind, eta, mu, nest in ((0, 1.0, 0.0, 0), (1, 0.1, 0.9, 1), (1, 0.7, 0.5, 0),
                                    (1, 1.0, 0.0, 0)):
            scfg = ServerCfg(kind, eta, mu, nest)
            v0 = rng.normal(size=n) * 1e-3
            v_ref = v0.copy()
            v_gpu = v0.copy()
            mean = oracle.mean(models)
            delta = oracle.sub(theta, mean)
            out_ref = oracle.server_step(scfg, theta, delta, mean, v_ref)
            st = F.ServerOptState(F.ServerOptConfig(kind, eta, mu, bool(nest)), v_gpu)
            out = F.server_step(st, theta, delta, mean)
            assert np.array_equal(out, out_ref)
            assert np.array_equal(st.velocity, v_ref)
            # fused kernel == mean -> sub -> server_step
            v2 = v0.copy()
            st2 = F.ServerOptState(F.ServerOptConfig(kind, eta, mu, bool(nest)), v2)
            fused = F.aggregate(models, theta, st2)
            assert np.array_equal(fused, out_ref)
            assert np.array_equal(st2.velocity, v_ref)


def test_f64_mean_invariants(F):
    # test_param_vector.cpp:75-101: mean of equals is bitwise, -0.0 kept, midpoints exact
    pv = np.array([0.1, 1.0 / 3.0, -7.3e-11, -0.0, 0.30000000000000004, 1e300])
    for k in (1, 2, 3, 5, 7):
        m = F.ParamVector.mean([pv] * k)
        assert m.tobytes() == pv.tobytes()
    a = np.array([1.0, -4.0, 8.0])
    b = np.array([3.0, -2.0, 16.0])
    assert list(F.ParamVector.mean([a, b])) == [2.0, -3.0, 12.0]
    with pytest.raises(F.UsageError):
        F.ParamVector.mean([])


def test_f64_server_traces(F):
    # test_optim.cpp:148-186 Nesterov / heavy-ball traces, :188-207 FedAvg bit identity
    for nest, want in ((True, [-0.19, -0.461, -0.8049000000000001]),
                       (False, [-0.1, -0.29000000000000004, -0.561])):
        st = F.ServerOptState.init(F.ServerOptConfig(1, 0.1, 0.9, nest), np.zeros(1))
        theta = np.zeros(1)
        for r in range(3):
            mean = theta - 1.0
            theta = F.server_step(st, theta, np.ones(1), mean)
            assert theta[0] == pytest.approx(want[r], rel=1e-12)
    theta = np.array([0.3])
    mean = np.array([1.0 / 3.0])
    delta = F.ParamVector.sub(theta, mean)
    for cfg in (F.ServerOptConfig(), F.ServerOptConfig(1, 1.0, 0.0, False)):
        out = F.server_step(F.ServerOptState.init(cfg, theta), theta, delta, mean)
        assert out.tobytes() == mean.tobytes()
    with pytest.raises(F.ConfigError):
        F.ServerOptConfig(0, 0.5, 0.0).validate()


def test_f64_adamw_sgd_bit_exact(F, oracle):
    rng = np.random.default_rng(1)
    n = 4099
    t = TrainCfg()
    p0 = rng.normal(size=n) * 0.02
    for clip in (1.0, 0.0, 1e-3):
        t.clip_norm = clip
        p_ref, m_ref, v_ref = p0.copy(), np.zeros(n), np.zeros(n)
        st = F.AdamWState.fresh(F.AdamWConfig(clip_norm=clip), p0)
        p = p0.copy()
        sc = 0
        for step in range(5):
            g = rng.normal(size=n) * 0.1
            sc = oracle.adamw_step(p_ref, g, m_ref, v_ref, sc, t, 1e-3 * (step + 1))
            F.adamw_step(p, g, st, 1e-3 * (step + 1))
            assert p.tobytes() == p_ref.tobytes()
            assert st.m.tobytes() == m_ref.tobytes() and st.v.tobytes() == v_ref.tobytes()
        assert st.step_count == sc == 5
    # KAT test_optim.cpp:75-87
    th = np.zeros(1)
    st = F.AdamWState.fresh(F.AdamWConfig(), th)
    F.adamw_step(th, np.ones(1), st, 0.1)
    assert th[0] == pytest.approx(-0.09999999900000002, rel=1e-14)
    assert st.m[0] == pytest.approx(0.1, rel=1e-14) and st.v[0] == pytest.approx(0.05, rel=1e-14)
    with pytest.raises(F.NumericError):
        F.adamw_step(np.zeros(2), np.array([np.inf, 0.0]), F.AdamWState.fresh(F.AdamWConfig(),
                                                                              np.zeros(2)), 0.1)
    # SGD (test_optim.cpp:136-146)
    th = np.ones(1)
    F.sgd_step(th, np.array([2.0]), 0.25)
    assert th[0] == 0.5
    th = np.ones(1)
    F.sgd_step(th, np.array([2.0]), 0.25, 0.5)
    assert th[0] == 0.875
    g = rng.normal(size=n)
    a, b = p0.copy(), p0.copy()
    oracle.sgd_step(a, g, 0.01, 0.5)
    F.sgd_step(b, g, 0.01, 0.5)
    assert a.tobytes() == b.tobytes()


def _hetero4_train(F, tau=16, opt=0):
    return F.LocalTrainConfig(
        model=F.ModelConfig(*HETERO4), schedule=F.LrSchedule(2e-3, 16, 160, 0.1), opt=opt,
        local_steps=tau, batch_size=4)


def test_local_round_f32(F, oracle):
    cfg_t = HETERO4
    mc = ModelCfg(*cfg_t)
    theta0 = oracle.init_params(mc, 1)
    corpus = oracle.generate_corpus("web", 50000, 7, 64)
    oplan = oracle.plan_iid(corpus, 2, 16, 7)
    t = TrainCfg(eta_max=2e-3, warmup_steps=16, decay_steps=160, alpha=0.1, local_steps=16,
                 batch_size=4)
    th_ref, loss_ref, cur_ref = oracle.local_round(mc, t, theta0, oplan, 1, 42, 0, 1, 16)
    plan = F.partition_iid(corpus, 2, 16, 7)
    stream = F.BatchStream(plan, 1, 4, 16, F.stream_seed(42, 1))
    res = F.run_local_round(theta0, stream, _hetero4_train(F), 1, 1, 16)
    losses = np.array([s.loss for s in res.steps])
    assert res.cursor == cur_ref == 64
    assert all(s.tokens == 64 for s in res.steps)
    assert np.max(np.abs(losses - loss_ref) / loss_ref) <= 1e-4
    assert np.max(np.abs(res.theta - th_ref)) <= 2e-4
    # SGD keeps the update linear in the grads: tighter (acceptance_main.cpp:254-255)
    t.opt = 1
    th_ref, loss_ref, _ = oracle.local_round(mc, t, theta0, oplan, 1, 42, 0, 1, 16)
    stream = F.BatchStream(plan, 1, 4, 16, F.stream_seed(42, 1))
    res = F.run_local_round(theta0, stream, _hetero4_train(F, opt=1), 1, 1, 16)
    assert np.max(np.abs(res.theta - th_ref)) <= 1e-6


def test_local_round_divergence(F, oracle):
    mc = ModelCfg(*HETERO4)
    theta0 = oracle.init_params(mc, 1)
    theta0[-1] = np.nan  # head.b[V-1]: every row's softmax sees it
    corpus = oracle.generate_corpus("web", 50000, 7, 64)
    plan = F.partition_iid(corpus, 2, 16, 7)
    stream = F.BatchStream(plan, 0, 4, 16, F.stream_seed(42, 0))
    with pytest.raises(F.DivergenceError) as ei:
        F.run_local_round(theta0, stream, _hetero4_train(F, tau=4), 3, 0, 48)
    assert (ei.value.round, ei.value.client, ei.value.step) == (3, 0, 0)


def _runner_case(F, oracle, server, rounds=4, K=2, P=2, precision="f32", tau=16):
    mc = ModelCfg(*HETERO4)
    theta0 = oracle.init_params(mc, 1)
    corpus = oracle.generate_corpus("web", 200000, 7, 64)
    oplan = oracle.plan_iid(corpus, P, 16, 7)
    t = TrainCfg(eta_max=2e-3, warmup_steps=16, decay_steps=160, alpha=0.1, local_steps=tau,
                 batch_size=4)
    th_ref, vel_ref = theta0.copy(), np.zeros_like(theta0)
    cursors = np.zeros(P, np.uint64)
    ref_losses = []
    for r in range(rounds):
        _, cl = oracle.run_round(mc, t, ServerCfg(*server), oplan, P, K, 42, r, th_ref, vel_ref,
                                 cursors)
        ref_losses.append(cl.mean())
    plan = F.partition_iid(corpus, P, 16, 7)
    runner = F.FederationRunner(F.FederationConfig(P, K, rounds, F.Topology.kRingAllReduce, 42),
                                _hetero4_train(F, tau), F.ServerOptConfig(*server[:3],
                                                                          bool(server[3])),
                                plan, theta0, precision=precision)
    recs = [runner.run_round() for _ in range(rounds)]
    return runner, recs, th_ref, vel_ref, ref_losses, cursors


@pytest.mark.parametrize("server", [(0, 1.0, 0.0, 0), (1, 0.1, 0.9, 1)])
def test_runner_vs_oracle_f32(F, oracle, server):
    runner, recs, th_ref, vel_ref, ref_losses, cursors = _runner_case(F, oracle, server)
    th = runner.theta()
    assert np.max(np.abs(th - th_ref)) <= 5e-4
    for rec, lr in zip(recs, ref_losses):
        assert abs(rec.mean_client_loss - lr) / lr <= 2e-4
    for c in range(2):
        assert runner.client_cursor(c) == int(cursors[c])
    if server[0] == 1:
        assert np.max(np.abs(runner.velocity() - vel_ref)) <= 5e-4
    assert runner.done()
    with pytest.raises(F.UsageError):
        runner.run_round()


def test_runner_bf16_tracks_oracle(F, oracle):
    runner, recs, th_ref, _, ref_losses, _ = _runner_case(F, oracle, (1, 0.1, 0.9, 1),
                                                          precision="bf16")
    for rec, lr in zip(recs, ref_losses):
        assert abs(rec.mean_client_loss - lr) / lr <= 3e-2


def test_runner_zero_lr_fixed_point(F, oracle):
    # test_aggregator.cpp:118-136 (tau = 1, lr(0) = 0): theta is a fixed point,
    # bitwise at the device's fp32 resolution.
    mc = ModelCfg(*TINY)
    theta0 = oracle.init_params(mc, 17)
    corpus = oracle.generate_corpus("web", 4000, 5, 16)
    plan = F.partition_iid(corpus, 3, 4, 3)
    local = F.LocalTrainConfig(model=F.ModelConfig(*TINY), local_steps=1, batch_size=2)
    runner = F.FederationRunner(F.FederationConfig(3, 3, 1, F.Topology.kParameterServer, 5), local,
                                F.ServerOptConfig(), plan, theta0)
    runner.run_round()
    assert runner.theta().tobytes() == theta0.astype(np.float32).astype(np.float64).tobytes()


def test_runner_dropouts(F, oracle):
    mc = ModelCfg(*TINY)
    theta0 = oracle.init_params(mc, 37)
    corpus = oracle.generate_corpus("web", 4000, 5, 16)
    plan = F.partition_iid(corpus, 2, 4, 3)
    local = F.LocalTrainConfig(model=F.ModelConfig(*TINY), local_steps=2, batch_size=2)
    fed = F.FederationConfig(2, 2, 1, F.Topology.kParameterServer, 13)
    runner = F.FederationRunner(fed, local, F.ServerOptConfig(), plan, theta0, dropouts=[(0, 0)])
    rec = runner.run_round()
    survivor = F.run_local_round(theta0, F.BatchStream(plan, 1, 2, 4, F.stream_seed(13, 1)),
                                 local, 0, 1, 0)
    assert np.array_equal(runner.theta(), survivor.theta.astype(np.float32).astype(np.float64))
    assert rec.min_client_loss == rec.max_client_loss
    assert runner.client_cursor(0) == 4 and runner.client_cursor(1) == 4
    ring = F.FederationRunner(F.FederationConfig(2, 2, 1, F.Topology.kRingAllReduce, 13), local,
                              F.ServerOptConfig(), plan, theta0, dropouts=[(0, 1)])
    with pytest.raises(F.RoundFailureError):
        ring.run_round()
    allgone = F.FederationRunner(fed, local, F.ServerOptConfig(), plan, theta0,
                                 dropouts=[(0, 0), (0, 1)])
    with pytest.raises(F.RoundFailureError):
        allgone.run_round()


def test_runner_guards(F, oracle):
    mc = ModelCfg(*TINY)
    theta0 = oracle.init_params(mc, 1)
    corpus = oracle.generate_corpus("web", 4000, 5, 16)
    plan = F.partition_iid(corpus, 2, 4, 3)
    local = F.LocalTrainConfig(model=F.ModelConfig(*TINY), local_steps=1, batch_size=2)
    with pytest.raises(F.ConfigError):
        F.FederationRunner(F.FederationConfig(4, 2, 1), local, F.ServerOptConfig(), plan, theta0)
    with pytest.raises(F.ConfigError):
        F.FederationRunner(F.FederationConfig(2, 3, 1), local, F.ServerOptConfig(), plan, theta0)


@pytest.mark.parametrize("opt", [0, 1])
def test_local_round_post_process_clip(F, oracle, opt):
    """post_process clip-update-norm (client.cpp:96-110): the round update
    theta_k - theta_t is rescaled to the threshold when its norm exceeds it.
    Tolerances as test_local_round_f32 (AdamW 2e-4, SGD 1e-6 max-abs)."""
    mc = ModelCfg(*HETERO4)
    theta0 = oracle.init_params(mc, 1)
    corpus = oracle.generate_corpus("web", 50000, 7, 64)
    oplan = oracle.plan_iid(corpus, 2, 16, 7)
    plan = F.partition_iid(corpus, 2, 16, 7)
    tol = 2e-4 if opt == 0 else 1e-6
    # the unclipped update norm decides which thresholds clip
    t = TrainCfg(eta_max=2e-3, warmup_steps=16, decay_steps=160, alpha=0.1, local_steps=16,
                 batch_size=4, opt=opt)
    th_free, _, _ = oracle.local_round(mc, t, theta0, oplan, 1, 42, 0, 1, 16)
    norm = float(np.linalg.norm(th_free - theta0))
    assert norm > 0
    for thr in (0.25 * norm, 0.9 * norm, 4.0 * norm):
        t.post_kind, t.post_threshold = 1, thr
        th_ref, loss_ref, _ = oracle.local_round(mc, t, theta0, oplan, 1, 42, 0, 1, 16)
        local = _hetero4_train(F, opt=opt)
        local.post = F.PostProcessPolicy(1, thr)
        stream = F.BatchStream(plan, 1, 4, 16, F.stream_seed(42, 1))
        res = F.run_local_round(theta0, stream, local, 1, 1, 16)
        assert np.max(np.abs(res.theta - th_ref)) <= tol, thr
        got = float(np.linalg.norm(res.theta - theta0))
        if thr < norm:  # clipped: the update norm is the threshold
            assert abs(got - thr) / thr <= 1e-3
        else:           # identity branch
            assert abs(got - norm) / norm <= 1e-3
    local = _hetero4_train(F, opt=opt)
    local.post = F.PostProcessPolicy(1, 0.0)
    with pytest.raises(F.ConfigError):
        F.run_local_round(theta0, F.BatchStream(plan, 1, 4, 16, F.stream_seed(42, 1)), local,
                          1, 1, 16)


def test_runner_post_process_clip(F, oracle):
    """The clip post-process inside FederationRunner rounds (aggregator.cpp:114 ->
    client.cpp:156): 3 rounds of DiLoCo, theta and velocity vs the oracle."""
    mc = ModelCfg(*HETERO4)
    theta0 = oracle.init_params(mc, 1)
    corpus = oracle.generate_corpus("web", 200000, 7, 64)
    oplan = oracle.plan_iid(corpus, 2, 16, 7)
    t = TrainCfg(eta_max=2e-3, warmup_steps=16, decay_steps=160, alpha=0.1, local_steps=16,
                 batch_size=4, post_kind=1, post_threshold=0.05)
    server = ServerCfg(1, 0.1, 0.9, 1)
    th_ref, vel_ref = theta0.copy(), np.zeros_like(theta0)
    cursors = np.zeros(2, np.uint64)
    for r in range(3):
        oracle.run_round(mc, t, server, oplan, 2, 2, 42, r, th_ref, vel_ref, cursors)
    local = _hetero4_train(F)
    local.post = F.PostProcessPolicy(1, 0.05)
    runner = F.FederationRunner(F.FederationConfig(2, 2, 3, F.Topology.kRingAllReduce, 42),
                                local, F.ServerOptConfig(1, 0.1, 0.9, True),
                                F.partition_iid(corpus, 2, 16, 7), theta0)
    for _ in range(3):
        runner.run_round()
    assert np.max(np.abs(runner.theta() - th_ref)) <= 5e-4
    assert np.max(np.abs(runner.velocity() - vel_ref)) <= 5e-4


def test_f64_mean_more_models_than_smem_table(F, oracle):
    # ParamVector::mean has no model-count limit (param_vector.cpp:127-152): past
    # the 256-entry shared-memory pointer table the kernel reads the global table
    rng = np.random.default_rng(7)
    n = 1001
    models = [rng.normal(size=n) * 0.02 for _ in range(300)]
    assert np.array_equal(F.ParamVector.mean(models), oracle.mean(models))
    theta = rng.normal(size=n) * 0.02
    mean = oracle.mean(models)
    v_ref = np.zeros(n)
    out_ref = oracle.server_step(ServerCfg(1, 0.1, 0.9, 1), theta, oracle.sub(theta, mean), mean,
                                 v_ref)
    st = F.ServerOptState(F.ServerOptConfig(1, 0.1, 0.9, True), np.zeros(n))
    assert np.array_equal(F.aggregate(models, theta, st), out_ref)
    assert np.array_equal(st.velocity, v_ref)


@pytest.mark.parametrize("precision,cfg_t,B,mb", [("f32", HETERO4, 5, 2), ("f32", DEFAULT, 4, 1),
                                                  ("bf16", WIDE256, 4, 1), ("bf16", HETERO4, 6, 4)])
def test_micro_batched_step_matches_whole_batch(F, oracle, precision, cfg_t, B, mb):
    """A batch above the context's activation capacity runs as accumulated
    micro-batches (GEMM Accum epilogues, accumulating column reductions and
    embedding scatter, one loss scale 1/#targets): same loss and gradient as
    the whole batch (client.cpp:135-154) -- f32 within the oracle tolerances,
    and micro vs whole within fp32 summation-order noise."""
    mc = ModelCfg(*cfg_t)
    params = oracle.init_params(mc, 3)
    inp, tgt = _batch(oracle, cfg_t, B)
    whole = F.TransformerModel(_mc(F, cfg_t), precision=precision, max_batch=B)
    micro = F.TransformerModel(_mc(F, cfg_t), precision=precision, micro_batch=mb)
    batch = F.Batch(inp, tgt, B, cfg_t[5])
    lw, gw = whole.forward_loss(params, batch)
    lm, gm = micro.forward_loss(params, batch)
    assert abs(lm - lw) / abs(lw) <= (1e-6 if precision == "f32" else 2e-3)
    assert _rel_l2(gm, gw) <= (1e-5 if precision == "f32" else 2e-2)
    if precision == "f32":
        l_ref, g_ref = oracle.forward_backward(mc, params, inp, tgt, B, cfg_t[5])
        assert abs(lm - l_ref) / abs(l_ref) <= 1e-5
        for name, off, shape in micro.layout():
            n = int(np.prod(shape))
            gr = g_ref[off:off + n]
            if np.linalg.norm(gr) > 1e-8:
                assert _rel_l2(gm[off:off + n], gr) <= 5e-4, name
        # forward-only / eval through micro-batches
        assert abs(micro.forward_loss(params, batch, build_grad=False)[0] - l_ref) / l_ref <= 1e-5


def test_micro_batched_runner_vs_oracle(F, oracle):
    """FederationRunner with micro_batch=1 (B=4): 3 DiLoCo rounds vs the oracle,
    tolerances of test_runner_vs_oracle_f32."""
    server = (1, 0.1, 0.9, 1)
    mc = ModelCfg(*HETERO4)
    theta0 = oracle.init_params(mc, 1)
    corpus = oracle.generate_corpus("web", 200000, 7, 64)
    oplan = oracle.plan_iid(corpus, 2, 16, 7)
    t = TrainCfg(eta_max=2e-3, warmup_steps=16, decay_steps=160, alpha=0.1, local_steps=16,
                 batch_size=4)
    th_ref, vel_ref = theta0.copy(), np.zeros_like(theta0)
    cursors = np.zeros(2, np.uint64)
    for r in range(3):
        oracle.run_round(mc, t, ServerCfg(*server), oplan, 2, 2, 42, r, th_ref, vel_ref, cursors)
    runner = F.FederationRunner(F.FederationConfig(2, 2, 3, F.Topology.kRingAllReduce, 42),
                                _hetero4_train(F), F.ServerOptConfig(1, 0.1, 0.9, True),
                                F.partition_iid(corpus, 2, 16, 7), theta0, micro_batch=1)
    for _ in range(3):
        runner.run_round()
    assert np.max(np.abs(runner.theta() - th_ref)) <= 5e-4
    assert np.max(np.abs(runner.velocity() - vel_ref)) <= 5e-4


@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_launch_count_graph_replay_matches_eager(F, oracle, precision):
    # photon_launch_count (bench.py's gpu_launches) counts every launch site and,
    # for a CUDA-graph replay of a local round, the graph's kernel nodes: the
    # first round runs eager, the second is captured and replayed, later ones
    # replay -- every round must add the same number of kernels
    from paper_2411_02908_b200 import _capi as A

    cfg_t = WIDE256
    mc = ModelCfg(*cfg_t)
    theta0 = oracle.init_params(mc, 3)
    corpus = oracle.generate_corpus("web", 60000, 5, cfg_t[4])
    plan = F.partition_iid(corpus, 2, cfg_t[5], 3)
    local = F.LocalTrainConfig(model=F.ModelConfig(*cfg_t), local_steps=3, batch_size=2)
    runner = F.FederationRunner(F.FederationConfig(2, 2, 4, F.Topology.kRingAllReduce, 5), local,
                                F.ServerOptConfig(1, 0.1, 0.9, True), plan, theta0,
                                precision=precision)
    counts = []
    for _ in range(4):
        n0 = A.lib().photon_launch_count()
        runner.run_round()
        counts.append(A.lib().photon_launch_count() - n0)
    assert counts[0] > 0
    assert counts == [counts[0]] * 4, counts
