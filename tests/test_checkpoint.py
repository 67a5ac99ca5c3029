"""PHCK snapshots (checkpoint.h:17-45, checkpoint.cpp:69-167) and the held-out
evaluation set (harness.cpp:440-472): host code of the C ABI, no GPU needed.

Bars: CRC-64/XZ known answer; our writer is byte-identical to the reference's
(oracle/_ref, built from /root/reference) for the same (params, round); each
reader reads the other's file bit-exactly; integrity / layout failures raise
the reference's exception types; the eval set equals the batches of the c7
fixture builder (pinned by acceptance c7's perplexity, test_oracle_golden.py)."""
import os

import numpy as np
import pytest

from oracle import ModelCfg, load_reference

F = pytest.importorskip("paper_2411_02908_b200.fedsim")

SMALL = (2, 32, 2, 4, 64, 32)


def _model(t):
    return F.ModelConfig(*t)


def test_crc64_xz_known_answer():
    assert F.crc64(b"123456789") == 0x995DC9BBDF1939FA  # CRC-64/XZ check value
    assert F.crc64(b"") == 0


def test_roundtrip(tmp_path, oracle):
    params = oracle.init_params(ModelCfg(*SMALL), 5)
    path = str(tmp_path / "c.phck")
    F.write_checkpoint(path, _model(SMALL), params, 7)
    back, rd = F.read_checkpoint(path, _model(SMALL))
    assert rd == 7 and back.tobytes() == params.tobytes()
    assert not os.path.exists(path + ".tmp")


def test_byte_identical_to_reference_writer(tmp_path, oracle):
    ref = load_reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    params = oracle.init_params(ModelCfg(*SMALL), 3)
    params[5] = -0.0  # signed zero survives
    ours, theirs = str(tmp_path / "ours.phck"), str(tmp_path / "ref.phck")
    F.write_checkpoint(ours, _model(SMALL), params, 12)
    ref.write_checkpoint(ModelCfg(*SMALL), params, 12, theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    back, rd = ref.read_checkpoint(ModelCfg(*SMALL), ours)
    assert rd == 12 and back.tobytes() == params.tobytes()
    back2, rd2 = F.read_checkpoint(theirs, _model(SMALL))
    assert rd2 == 12 and back2.tobytes() == params.tobytes()


def test_integrity_errors(tmp_path, oracle):
    params = oracle.init_params(ModelCfg(*SMALL), 1)
    path = str(tmp_path / "c.phck")
    F.write_checkpoint(path, _model(SMALL), params, 1)
    raw = bytearray(open(path, "rb").read())
    bad = str(tmp_path / "bad.phck")
    flipped = bytearray(raw)
    flipped[-3] ^= 0x10  # payload bit flip -> checksum mismatch
    open(bad, "wb").write(bytes(flipped))
    with pytest.raises(F.IntegrityError):
        F.read_checkpoint(bad, _model(SMALL))
    open(bad, "wb").write(bytes(raw[:-8]))  # truncated
    with pytest.raises(F.IntegrityError):
        F.read_checkpoint(bad, _model(SMALL))
    open(bad, "wb").write(b"NOPE" + bytes(raw[4:]))
    with pytest.raises(F.IntegrityError):
        F.read_checkpoint(bad, _model(SMALL))
    with pytest.raises(F.IoError):
        F.read_checkpoint(str(tmp_path / "missing.phck"), _model(SMALL))
    with pytest.raises(F.ShapeError):  # another model's layout
        F.read_checkpoint(path, _model((1, 32, 2, 4, 64, 32)))


def _c7_builder(oracle, V, S, n_seq, bsz, style="web", data_seed=7):
    # the test-side builder pinned by acceptance c7 (test_oracle_golden.py)
    bl = S + 1
    c = oracle.generate_corpus(style, n_seq * bl, oracle.mix_seed(data_seed, 0x4576616C), V)
    inp = np.concatenate([c[s * bl:s * bl + S] for s in range(n_seq)]).astype(np.int32)
    tgt = np.concatenate([c[s * bl + 1:s * bl + S + 1] for s in range(n_seq)]).astype(np.int32)
    return inp, tgt


def test_eval_set_matches_c7_builder(oracle):
    es = F.EvalSet(["web"], 64, 7, _model((2, 32, 2, 4, 64, 32)), 8)
    batches = es.batches()
    assert [b.batch_size for b in batches] == [8] * 8
    inp, tgt = _c7_builder(oracle, 64, 32, 64, 8)
    assert np.array_equal(np.concatenate([b.inputs for b in batches]), inp)
    assert np.array_equal(np.concatenate([b.targets for b in batches]), tgt)


def test_eval_set_multi_style_and_short_batch(oracle):
    # by-source specs evaluate every style: eval_sequences / n_styles each, the
    # batch counter runs across styles and the last batch may be short
    model = _model((1, 32, 2, 4, 64, 16))
    es = F.EvalSet(["academic", "prose"], 10, 9, model, 4)
    batches = es.batches()
    assert [b.batch_size for b in batches] == [4, 4, 2]
    parts = [_c7_builder(oracle, 64, 16, 5, 4, style=s, data_seed=9) for s in ("academic", "prose")]
    assert np.array_equal(np.concatenate([b.inputs for b in batches]),
                          np.concatenate([p[0] for p in parts]))
    assert np.array_equal(np.concatenate([b.targets for b in batches]),
                          np.concatenate([p[1] for p in parts]))


def test_eval_set_initial_ppl_matches_reference_harness(tmp_path, oracle):
    """run_experiment's initial_ppl = eval_fn(theta0) over build_eval_batches."""
    ref = load_reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from oracle import ServerCfg, TrainCfg
    cfg = ModelCfg(1, 32, 2, 4, 64, 16)
    t = TrainCfg(eta_max=2e-3, warmup_steps=4, decay_steps=32, alpha=0.1, local_steps=2,
                 batch_size=2)
    init_ppl, _ = ref.run_experiment_fed(cfg, t, ServerCfg(0, 1.0, 0.0, 0), 20000, 2, 1, 42, 1, 7,
                                         24, 8, str(tmp_path))
    es = F.EvalSet(["web"], 24, 7, _model((1, 32, 2, 4, 64, 16)), 8)
    bs = es.batches()
    ppl = oracle.eval_perplexity(cfg, oracle.init_params(cfg, 1),
                                 np.concatenate([b.inputs for b in bs]),
                                 np.concatenate([b.targets for b in bs]),
                                 [b.batch_size for b in bs], 16)
    assert ppl == init_ppl
    # and the reference run directory's checkpoint reads back through our reader
    theta, rd = F.read_checkpoint(str(tmp_path / "checkpoint.phck"), _model((1, 32, 2, 4, 64, 16)))
    assert rd == 1 and np.all(np.isfinite(theta))
