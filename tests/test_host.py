"""Host-side determinism layer of libphoton.so (no GPU needed) vs the oracle:
bit-exact client sampling, corpora, shard plans, batch streams and cursors,
LR schedule, canonical layout and parameter init; reference error behaviour."""
import numpy as np
import pytest

from oracle import ModelCfg, TrainCfg


def test_mix64_and_seeds(F, oracle):
    for x in (0, 1, 42, 0xDEADBEEF, 2**63 + 5):
        assert F.mix64(x) == oracle.mix64(x)
    for s, c in ((42, 0), (42, 7), (9, 123)):
        assert F.stream_seed(s, c) == oracle.stream_seed(s, c)


@pytest.mark.parametrize("p,k,seed", [(16, 4, 42), (8, 8, 42), (1000, 8, 1), (3, 1, 0)])
def test_sample_clients(F, oracle, p, k, seed):
    for r in range(20):
        assert F.sample_clients(p, k, seed, r) == oracle.sample_clients(p, k, seed, r)


def test_sample_clients_errors(F):
    with pytest.raises(F.ConfigError):
        F.sample_clients(4, 5, 7, 0)
    with pytest.raises(F.ConfigError):
        F.sample_clients(4, 0, 7, 0)


def test_lr_schedule(F, oracle):
    for sch in ((1e-2, 10, 100, 0.1), (6e-4, 64, 1024, 0.1), (3e-3, 0, 5, 0.0)):
        t = TrainCfg(eta_max=sch[0], warmup_steps=sch[1], decay_steps=sch[2], alpha=sch[3])
        s = F.LrSchedule(*sch)
        for step in list(range(0, 130)) + [5000]:
            assert F.lr_at(s, step) == oracle.lr_at(t, step)
    with pytest.raises(F.ConfigError):
        F.lr_at(F.LrSchedule(0.0, 1, 1, 0.1), 0)
    with pytest.raises(F.ConfigError):
        F.lr_at(F.LrSchedule(1.0, 1, 0, 0.1), 0)
    with pytest.raises(F.ConfigError):
        F.lr_at(F.LrSchedule(1.0, 1, 1, 1.5), 0)


@pytest.mark.parametrize("style", ["academic", "web", "reference", "prose"])
@pytest.mark.parametrize("vocab", [16, 64, 50368])
def test_generate_corpus(F, oracle, style, vocab):
    a = F.generate_corpus(style, 7777, 7, vocab)
    assert np.array_equal(a, oracle.generate_corpus(style, 7777, 7, vocab))
    band = vocab // 4
    assert a.min() // band == a.max() // band  # never leaves its quarter (test_data.cpp:37)


def test_generate_corpus_errors(F):
    with pytest.raises(F.ConfigError):
        F.generate_corpus("gibberish", 100, 1)
    with pytest.raises(F.ConfigError):
        F.generate_corpus("web", 100, 1, 6)
    with pytest.raises(F.ConfigError):
        F.generate_corpus("web", 0, 1)


@pytest.mark.parametrize("tokens,shards,S,seed", [(1000, 4, 8, 77), (20000, 3, 16, 7),
                                                  (4000, 8, 4, 3)])
def test_iid_plan_and_streams(F, oracle, tokens, shards, S, seed):
    corpus = oracle.generate_corpus("web", tokens, 5, 64)
    plan = F.partition_iid(corpus, shards, S, seed)
    oplan = oracle.plan_iid(corpus, shards, S, seed)
    assert plan.n_clients() == shards
    for c in range(shards):
        assert plan.client_blocks(c) == oplan.client_blocks(c)
        # several epochs worth of batches, with an odd batch size (epoch straddles)
        s = F.BatchStream(plan, c, 3, S, F.stream_seed(42, c))
        cur = 0
        for _ in range(2 * max(1, oplan.client_blocks(c)) // 3 + 3):
            b = s.next()
            i, t, cur = oracle.stream_next(oplan, c, 3, oracle.stream_seed(42, c), cur)
            assert np.array_equal(b.inputs, i) and np.array_equal(b.targets, t)
            assert s.cursor() == cur


def test_by_source_plan(F, oracle):
    corp = [oracle.generate_corpus(s, 3000, 7, 64) for s in ("academic", "web", "reference",
                                                              "prose")]
    plan = F.partition_by_source(corp, 2, 16)
    oplan = oracle.plan_by_source(corp, 2, 16)
    assert plan.n_clients() == 8
    for c in range(8):
        s = F.BatchStream(plan, c, 5, 16, 99, cursor=11)
        cur = 11
        for _ in range(6):
            b = s.next()
            i, t, cur = oracle.stream_next(oplan, c, 5, 99, cur)
            assert np.array_equal(b.inputs, i)
    with pytest.raises(F.ConfigError):
        F.partition_by_source([oracle.generate_corpus("academic", 15, 1), corp[1]], 2, 9)


def test_stream_guards(F, oracle):
    plan = F.partition_iid(oracle.generate_corpus("web", 1000, 5, 64), 2, 8, 1)
    with pytest.raises(F.ConfigError):
        F.BatchStream(plan, 0, 0, 8, 1)
    with pytest.raises(F.UsageError):
        F.BatchStream(plan, 0, 2, 9, 1)
    with pytest.raises(F.LookupError):
        F.BatchStream(plan, 5, 2, 8, 1)
    with pytest.raises(F.ConfigError):
        F.partition_iid(oracle.generate_corpus("web", 20, 5, 64), 4, 8, 1)


@pytest.mark.parametrize("cfg", [(1, 8, 2, 4, 16, 4), (2, 64, 2, 4, 64, 32), (1, 32, 2, 4, 64, 16),
                                 (3, 48, 4, 2, 72, 12)])
def test_layout_and_init(F, oracle, cfg):
    m = F.ModelConfig(*cfg)
    oc = ModelCfg(*cfg)
    assert m.param_count() == oracle.param_count(oc)
    assert F.TransformerModel(m).layout() == oracle.layout(oc)
    for seed in (1, 3, 42):
        assert np.array_equal(F.TransformerModel(m).init_params(seed), oracle.init_params(oc, seed))


def test_photon_shapes(F):
    assert F.ModelConfig(12, 768, 12, 4, 50368, 2048).param_count() == 164044480
    assert F.ModelConfig(24, 2048, 16, 4, 50368, 2048).param_count() == 1419154624
    assert F.ModelConfig(32, 4096, 32, 4, 50368, 2048).param_count() == 6865216704
    assert F.ModelConfig().payload_mib() == 0.84228515625
    with pytest.raises(F.ConfigError):
        F.ModelConfig(2, 64, 3, 4, 64, 32).validate()


def test_server_cfg_validation(F):
    with pytest.raises(F.ConfigError):
        F.ServerOptConfig(0, 0.5, 0.0).validate()
    with pytest.raises(F.ConfigError):
        F.ServerOptConfig(0, 1.0, 0.3).validate()
    with pytest.raises(F.ConfigError):
        F.ServerOptConfig(1, 0.1, 1.0).validate()
    F.diloco_server_opt().validate()
