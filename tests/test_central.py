"""Centralized / DDP baseline: the test-side oracle
composition of run_centralized equals the reference's own run_centralized
(oracle/_ref) bit for bit in f64 -- it is then the checker for the device
trainer (tests/test_gpu_central.py)."""
import numpy as np
import pytest

from oracle import ModelCfg, TrainCfg, load_reference
from central_case import oracle_centralized

CFG = ModelCfg(1, 32, 2, 4, 64, 16)


@pytest.mark.parametrize("opt,reset", [(0, 3), (1, 0)])
def test_oracle_composition_matches_reference(oracle, opt, reset):
    ref = load_reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    t = TrainCfg(eta_max=2e-3, warmup_steps=2, decay_steps=16, alpha=0.1, opt=opt,
                 sgd_clip_norm=1.0, batch_size=4)
    theta0 = oracle.init_params(CFG, 1)
    corpus = oracle.generate_corpus("web", 20000, 7, 64)
    th_o, loss_o, cur_o = oracle_centralized(oracle, CFG, t, corpus, 2, 5, reset, 42, 7, theta0)
    th_r, loss_r, cur_r = ref.run_centralized(CFG, t, "web", 20000, 7, 2, 5, reset, 42, theta0)
    assert th_o.tobytes() == th_r.tobytes()
    assert loss_o.tobytes() == loss_r.tobytes()
    assert list(cur_o) == [int(x) for x in cur_r] == [10, 10]
