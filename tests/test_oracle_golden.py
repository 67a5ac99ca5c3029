"""Pin the oracle (C restatement of the reference path) before trusting it.

Three anchors, all bit-exact unless a tolerance is stated:
  1. known-answer values from the reference's own unit tests
     (/root/reference/proj/tests/unit/*.cpp, cited per test);
  2. tests/golden/fixtures.json, outputs of the reference compiled from its
     own sources (tests/golden/make_golden.py);
  3. the live reference (oracle/_ref) when it was built here;
plus the acceptance-c7 perplexity fixture recorded by the reference authors
(acceptance_main.cpp:472-473), reproduced through the oracle.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import ModelCfg, ServerCfg, TrainCfg

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fixtures.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fx(s):
    return float.fromhex(s)


# ---- 1. reference unit-test known answers ---------------------------------------------
def test_mix64_kats(oracle):  # test_rng.cpp:10-16
    assert oracle.mix64(0) == 0xE220A8397B1DCDAF
    assert oracle.mix64(1) == 0x910A2DEC89025CC1
    assert oracle.mix64(42) == 0xBDD732262FEB6E95
    assert oracle.mix64(0xDEADBEEF) == 0x4ADFB90F68C9EB9B
    assert oracle.mix_seed(7, 1, 2) == oracle.mix_seed(oracle.mix_seed(7, 1), 2)
    assert oracle.mix_seed(7, 1, 2, 3) == oracle.mix_seed(oracle.mix_seed(7, 1, 2), 3)


def test_rng_moments_and_ranges(oracle):  # test_rng.cpp:21-45
    _, u, _ = oracle.rng_draws(123, 10000)
    assert (u >= 0).all() and (u < 1).all()
    _, _, g = oracle.rng_draws(99, 100000)
    assert abs(g.mean()) < 0.02 and abs(g.var() - 1) < 0.03


def test_lr_schedule_kats(oracle):  # test_optim.cpp:45-73
    t = TrainCfg(eta_max=1e-2, warmup_steps=10, decay_steps=100, alpha=0.1)
    assert oracle.lr_at(t, 0) == 0.0
    assert oracle.lr_at(t, 5) == pytest.approx(5e-3, rel=1e-14)
    assert oracle.lr_at(t, 10) == pytest.approx(1e-2, rel=1e-14)
    assert oracle.lr_at(t, 60) == pytest.approx(5.5e-3, rel=1e-12)
    assert oracle.lr_at(t, 110) == pytest.approx(1e-3, rel=1e-12)
    assert oracle.lr_at(t, 100000) == pytest.approx(1e-3, rel=1e-12)
    for s in range(1, 11):
        assert oracle.lr_at(t, s) > oracle.lr_at(t, s - 1)
    for s in range(11, 111):
        assert oracle.lr_at(t, s) <= oracle.lr_at(t, s - 1)


def test_optimizer_kats(oracle):  # test_optim.cpp:75-186
    th, m, v = np.zeros(1), np.zeros(1), np.zeros(1)
    sc = oracle.adamw_step(th, np.ones(1), m, v, 0, TrainCfg(), 0.1)
    assert sc == 1
    assert th[0] == pytest.approx(-0.09999999900000002, rel=1e-14)
    assert m[0] == pytest.approx(0.1, rel=1e-14) and v[0] == pytest.approx(0.05, rel=1e-14)
    th = np.array([2.0])
    oracle.adamw_step(th, np.zeros(1), np.zeros(1), np.zeros(1), 0,
                      TrainCfg(weight_decay=0.5, clip_norm=0.0), 0.1)
    assert th[0] == pytest.approx(2.0 * (1.0 - 0.1 * 0.5), rel=1e-14)
    th = np.ones(1)
    oracle.sgd_step(th, np.array([2.0]), 0.25)
    assert th[0] == 0.5
    th = np.ones(1)
    oracle.sgd_step(th, np.array([2.0]), 0.25, 0.5)
    assert th[0] == 0.875
    for nest, want in ((1, [-0.19, -0.461, -0.8049000000000001]),
                       (0, [-0.1, -0.29000000000000004, -0.561])):
        theta, vel = np.zeros(1), np.zeros(1)
        for r in range(3):
            theta = oracle.server_step(ServerCfg(1, 0.1, 0.9, nest), theta, np.ones(1),
                                       theta - 1.0, vel)
            assert theta[0] == pytest.approx(want[r], rel=1e-12)
    theta, mean = np.array([0.3]), np.array([1.0 / 3.0])
    delta = oracle.sub(theta, mean)
    for s in (ServerCfg(), ServerCfg(1, 1.0, 0.0, 0)):
        assert oracle.server_step(s, theta, delta, mean, np.zeros(1)).tobytes() == mean.tobytes()


def test_mean_kats(oracle):  # test_param_vector.cpp:75-101
    pv = np.array([0.1, 1.0 / 3.0, -7.3e-11, -0.0, 0.30000000000000004, 1e300])
    for k in (1, 2, 3, 5, 7):
        assert oracle.mean([pv] * k).tobytes() == pv.tobytes()
    assert list(oracle.mean([np.array([1.0, -4.0, 8.0]), np.array([3.0, -2.0, 16.0])])) == \
        [2.0, -3.0, 12.0]


def test_param_counts(oracle):  # test_model.cpp:62-75 + SURVEY 8d shapes
    assert oracle.param_count(ModelCfg()) == 110400
    assert oracle.param_count(ModelCfg(1, 8, 2, 4, 16, 4)) == 1192
    assert oracle.param_count(ModelCfg(12, 768, 12, 4, 50368, 2048)) == 164044480
    assert oracle.param_count(ModelCfg(24, 2048, 16, 4, 50368, 2048)) == 1419154624
    assert oracle.param_count(ModelCfg(32, 4096, 32, 4, 50368, 2048)) == 6865216704
    assert oracle.param_count(ModelCfg()) * 8 / 2**20 == 0.84228515625


def test_init_stats(oracle):  # test_model.cpp:84-110
    cfg = ModelCfg()
    p = oracle.init_params(cfg, 42)
    lay = {n: (o, s) for n, o, s in oracle.layout(cfg)}
    for n, (o, s) in lay.items():
        v = p[o:o + int(np.prod(s))]
        if n.endswith(".gain"):
            assert (v == 1.0).all()
        elif len(s) == 1:
            assert (v == 0.0).all()
    std = lambda n: p[lay[n][0]:lay[n][0] + int(np.prod(lay[n][1]))].std()  # noqa: E731
    assert abs(std("token_embedding") - 0.02) < 0.002
    assert abs(std("block0.attn.wo") - 0.01) < 0.001
    assert abs(std("block1.mlp.w2") - 0.01) < 0.001


def test_iid_partition_kat(oracle):  # test_data.cpp:83-121: 111 blocks -> 28/28/28/27
    plan = oracle.plan_iid(oracle.generate_corpus("web", 1000, 5), 4, 8, 77)
    sizes = [plan.client_blocks(k) for k in range(4)]
    assert sum(sizes) == 111 and max(sizes) - min(sizes) <= 1
    offs = [o for k in range(4) for _, o in plan.blocks(k)]
    assert len(set(offs)) == 111 and all(o % 9 == 0 and o + 9 <= 1000 for o in offs)
    with pytest.raises(Exception):
        oracle.plan_iid(oracle.generate_corpus("web", 20, 5), 4, 8, 1)


def test_by_source_partition_kat(oracle):  # test_data.cpp:124-149
    plan = oracle.plan_by_source([oracle.generate_corpus("academic", 105, 1),
                                  oracle.generate_corpus("web", 100, 2)], 2, 9)
    for k in range(4):
        blocks = plan.blocks(k)
        assert len(blocks) == 5
        assert blocks == [(k // 2, (k % 2) * 50 + 10 * i) for i in range(5)]


def test_stream_kats(oracle):  # test_data.cpp:157-215
    plan = oracle.plan_iid(oracle.generate_corpus("web", 720, 21), 1, 8, 21)
    seed = oracle.stream_seed(9, 0)
    inp, tgt, cur = oracle.stream_next(plan, 0, 2, seed, 0)
    assert cur == 2 and (inp >= 0).all() and (inp < 64).all()
    for r in range(2):
        assert (tgt[r * 8:r * 8 + 7] == inp[r * 8 + 1:r * 8 + 8]).all()
    # cursor rebuild continues the sequence
    c, seq = 0, []
    for _ in range(8):
        i, t, c = oracle.stream_next(plan, 0, 2, seed, c)
        seq.append(i)
    c = 10
    for k in range(3):
        i, _, c = oracle.stream_next(plan, 0, 2, seed, c)
        assert (i == seq[5 + k]).all()


def test_sampling_kats(oracle):  # test_aggregator.cpp:66-91
    s1 = oracle.sample_clients(16, 4, 42, 3)
    assert s1 == sorted(s1) and len(set(s1)) == 4
    assert oracle.sample_clients(16, 4, 42, 4) != s1
    assert oracle.sample_clients(4, 4, 7, 0) == [0, 1, 2, 3]
    counts = np.zeros(16)
    for r in range(10000):
        for i in oracle.sample_clients(16, 4, 9, r):
            counts[i] += 1
    assert (counts > 2370).all() and (counts < 2630).all()


# ---- 2. golden fixtures produced by the reference -----------------------------------------
def test_golden_rng(oracle):
    for x, h in GOLD["rng"]["mix64"].items():
        assert oracle.mix64(int(x)) == int(h, 16)
    _, _, g = oracle.rng_draws(99, 9)
    assert [v.hex() for v in g] == GOLD["rng"]["normals_seed99"]


def test_golden_data(oracle):
    d = GOLD["data"]
    for style in ("academic", "web", "reference", "prose"):
        c = oracle.generate_corpus(style, 5000, 7, 64)
        assert sha(c) == d[f"corpus_{style}_5000_7_64"]["sha256"]
    assert sha(oracle.generate_corpus("web", 50000, 7, 50368)) == \
        d["corpus_web_50000_7_50368"]["sha256"]
    plan = oracle.plan_iid(oracle.generate_corpus("web", 20000, 7, 64), 4, 16, 7)
    for client in (0, 1, 3):
        ins, tgs, cur = [], [], 0
        for _ in range(20):
            i, t, cur = oracle.stream_next(plan, client, 4, oracle.stream_seed(42, client), cur)
            ins.append(i)
            tgs.append(t)
        g = d[f"stream_iid_web20000_c{client}_b4_x20"]
        assert sha(np.concatenate(ins)) == g["inputs_sha256"]
        assert sha(np.concatenate(tgs)) == g["targets_sha256"] and cur == g["cursor"]
    corp = [oracle.generate_corpus(s, 3000, 7, 64)
            for s in ("academic", "web", "reference", "prose")]
    plan = oracle.plan_by_source(corp, 2, 16)
    ins, tgs, cur = [], [], 7
    for _ in range(30):
        i, t, cur = oracle.stream_next(plan, 5, 3, oracle.stream_seed(9, 5), cur)
        ins.append(i)
        tgs.append(t)
    g = d["stream_by_source_c5_b3_from7_x30"]
    assert sha(np.concatenate(ins)) == g["inputs_sha256"] and cur == g["cursor"]


def test_golden_sampling_and_lr(oracle):
    for key, want in GOLD["sample_clients"].items():
        p, k, s, r = (int(x) for x in key.split("_"))
        assert oracle.sample_clients(p, k, s, r) == want
    t = TrainCfg(eta_max=1e-2, warmup_steps=10, decay_steps=100, alpha=0.1)
    for s, h in GOLD["lr_at"].items():
        assert oracle.lr_at(t, int(s)).hex() == h


@pytest.mark.parametrize("name,cfg", [("default", ModelCfg()),
                                      ("tiny", ModelCfg(1, 8, 2, 4, 16, 4)),
                                      ("hetero4", ModelCfg(1, 32, 2, 4, 64, 16))])
def test_golden_model(oracle, name, cfg):
    g = GOLD["model"]
    p = oracle.init_params(cfg, 1)
    assert sha(p) == g[f"init_{name}_seed1"]["sha256"]
    plan = oracle.plan_iid(oracle.generate_corpus("web", 20000, 7, cfg.vocab_size), 2,
                           cfg.seq_len, 7)
    inp, tgt, _ = oracle.stream_next(plan, 0, 4, oracle.stream_seed(42, 0), 0)
    loss, grads = oracle.forward_backward(cfg, p, inp, tgt, 4, cfg.seq_len)
    assert loss.hex() == g[f"fwdbwd_{name}"]["loss"]
    assert sha(grads) == g[f"fwdbwd_{name}"]["grads_sha256"]


def test_golden_local_round_and_rounds(oracle):
    cfg = ModelCfg(1, 32, 2, 4, 64, 16)
    t = TrainCfg(eta_max=2e-3, warmup_steps=16, decay_steps=160, alpha=0.1, local_steps=16,
                 batch_size=4)
    th0 = oracle.init_params(cfg, 1)
    plan = oracle.plan_iid(oracle.generate_corpus("web", 50000, 7, 64), 2, 16, 7)
    th, losses, cur = oracle.local_round(cfg, t, th0, plan, 1, 42, 0, 1, 16)
    g = GOLD["local_round_hetero4_c1_r1"]
    assert sha(th) == g["theta_sha256"] and cur == g["cursor"]
    assert [x.hex() for x in losses] == g["losses"]
    plan = oracle.plan_iid(oracle.generate_corpus("web", 200000, 7, 64), 2, 16, 7)
    for name, s in (("fedavg", ServerCfg()), ("diloco", ServerCfg(1, 0.1, 0.9, 1))):
        theta, vel = th0.copy(), np.zeros_like(th0)
        cursors = np.zeros(2, np.uint64)
        rl = []
        for r in range(4):
            _, cl = oracle.run_round(cfg, t, s, plan, 2, 2, 42, r, theta, vel, cursors)
            rl.append(cl.mean())
        g = GOLD["rounds_hetero4_P2K2_tau16_4rounds"][name]
        assert sha(theta) == g["theta_sha256"] and sha(vel) == g["velocity_sha256"]
        assert [x.hex() for x in rl] == g["round_losses"]
    # SURVEY 8c recorded values (same runs)
    assert float.fromhex(GOLD["rounds_hetero4_P2K2_tau16_4rounds"]["fedavg"]["round_losses"][-1]) \
        == 1.6591960376792079
    assert float.fromhex(GOLD["rounds_hetero4_P2K2_tau16_4rounds"]["diloco"]["round_losses"][-1]) \
        == 2.8408618129986269


# ---- 3. live reference (when built here) -------------------------------------------------
def test_live_reference_round_trip(oracle, reference):
    cfg = ModelCfg(2, 32, 2, 4, 64, 32)
    t = TrainCfg(eta_max=3e-3, warmup_steps=8, decay_steps=64, alpha=0.05, local_steps=6,
                 batch_size=3, opt=0)
    th0 = reference.init_params(cfg, 5)
    assert np.array_equal(th0, oracle.init_params(cfg, 5))
    th_r, vel_r, rl_r, _ = reference.run_rounds(cfg, t, ServerCfg(1, 0.7, 0.5, 0), 0, "prose",
                                                30000, 3, 5, 3, 3, 11, 0, 2, th0)
    plan = oracle.plan_iid(oracle.generate_corpus("prose", 30000, 3, 64), 5, 32, 3)
    theta, vel, cursors = th0.copy(), np.zeros_like(th0), np.zeros(5, np.uint64)
    for r in range(3):
        _, cl = oracle.run_round(cfg, t, ServerCfg(1, 0.7, 0.5, 0), plan, 5, 3, 11, r, theta,
                                 vel, cursors)
        assert cl.mean().hex() == rl_r[r].hex()
    assert theta.tobytes() == th_r.tobytes() and vel.tobytes() == vel_r.tobytes()


# ---- acceptance c7: 16-client DiLoCo perplexity fixture -------------------------------------
def _c7_eval_batches(oracle, V, S, n_seq=64, bsz=8):
    # harness.cpp:440-472: held-out slice from mix_seed(data_seed, "Eval")
    bl = S + 1
    c = oracle.generate_corpus("web", n_seq * bl, oracle.mix_seed(7, 0x4576616C), V)
    inp = np.concatenate([c[s * bl:s * bl + S] for s in range(n_seq)]).astype(np.int32)
    tgt = np.concatenate([c[s * bl + 1:s * bl + S + 1] for s in range(n_seq)]).astype(np.int32)
    return inp, tgt, [bsz] * (n_seq // bsz)


def test_acceptance_c7_fixture(oracle):
    """acceptance_main.cpp:467-534: fed final ppl 2.9094513044307808 (rel 1e-9)."""
    cfg = ModelCfg(2, 32, 2, 4, 64, 32)
    t = TrainCfg(eta_max=3e-3, warmup_steps=32, decay_steps=256, alpha=0.05, local_steps=64,
                 batch_size=4)
    s = ServerCfg(1, 0.1, 0.9, 1)
    theta = oracle.init_params(cfg, 1)
    vel = np.zeros_like(theta)
    plan = oracle.plan_iid(oracle.generate_corpus("web", 200000, 7, 64), 16, 32, 7)
    cursors = np.zeros(16, np.uint64)
    inp, tgt, bs = _c7_eval_batches(oracle, 64, 32)
    ppl = None
    for r in range(5):
        oracle.run_round(cfg, t, s, plan, 16, 16, 42, r, theta, vel, cursors, ring=True)
        ppl = oracle.eval_perplexity(cfg, theta, inp, tgt, bs, 32)
    assert abs(ppl - 2.9094513044307808) <= 1e-9 * 2.9094513044307808
