"""Parity at the 125M ARCHITECTURE (L12 d768 H12 e4 V50368) against the
reference itself: tests/golden/arch125m_b2_s256.npz was produced by the
unmodified reference (oracle/_ref, tests/golden/make_golden_125m.py) at B=2,
S=256 (M = 512 rows: more than 2 x 148, so the cross-entropy kernels refill;
V = 50,368 is the headline vocabulary; d = 768 runs the register-resident
LayerNorm kernels, dh = 64 the tcgen05 attention; the bf16-only fused bias
gradients -- b1 from the GeluBwd epilogue, bq/bk/bv from the attention
backward's stores, head.b from the cross-entropy pass -- are checked entry
by entry).

Stated tolerances (per canonical entry; "rel" = ||got - ref|| / ||ref|| over
the entry's stored values -- every value of 1-D entries, 1,024 fixed samples of
matrices -- and "norm" = | ||got|| / ||ref|| - 1 | over the whole entry).
Measured on B200 (worst entry) in brackets:

                      f32 mode (fp32 SIMT)       bf16 mode (tcgen05, fp32 accumulate)
  loss                rel 1e-6   [5e-9]          rel 2e-4   [1.4e-5]
  gradient            rel 1e-4   [7e-6]          rel 4e-2   [2.0e-2, attn.wq/wk]
                      norm 1e-5  [1e-6]          norm 5e-3  [1.4e-3]
  attn.bk (mathematically 0: softmax is shift-invariant per query row; the
  reference holds rounding noise): ||g|| <= 1e-5 x ||g_total||  [<= 1.5e-6]
  local round, tau = 2, clipped SGD, per-entry update
                      rel 1e-2   [3.3e-3]        rel 8e-2   [4.7e-2]
      (f32: the fp32 master's ulp at theta ~ 1 (LN gains, 1.2e-7) against
      per-element updates ~ 2e-5 -- storage quantization, not arithmetic)
  local round, tau = 2, AdamW: update norm
                      1e-4       [8e-6]          1e-2       [2.7e-3]
      sign agreement of the sampled update values
                      >= 99.9 %  [100 %]         >= 97 %    [98.4 %]
      (m_hat / sqrt(v_hat) is +-1 at the first steps, so a gradient entry near 0
      may flip -- the reference's own caveat, acceptance_main.cpp:254-255)
  both step losses of each round: as "loss"
"""
import json
import os

import numpy as np
import pytest

from oracle import ModelCfg

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURE = os.path.join(HERE, "golden", "arch125m_b2_s256.npz")
CFG_T = (12, 768, 12, 4, 50368, 256)
B = 2

TOL = {
    "f32": dict(loss=1e-6, g_rel=1e-4, g_norm=1e-5, sgd_rel=1e-2, adamw_norm=1e-4,
                adamw_sign=0.999),
    "bf16": dict(loss=2e-4, g_rel=4e-2, g_norm=5e-3, sgd_rel=8e-2, adamw_norm=1e-2,
                 adamw_sign=0.97),
}
ZERO_ENTRIES = (".attn.bk",)


@pytest.fixture(scope="module")
def fx():
    return np.load(FIXTURE)


@pytest.fixture(scope="module")
def theta0(oracle):
    # init_params(1): the oracle's restatement is pinned bit-exact to the reference
    return oracle.init_params(ModelCfg(*CFG_T), 1)


def _report(name, rows):
    out = os.environ.get("PHOTON_PARITY_REPORT")
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, f"{name}.json"), "w") as f:
            json.dump(rows, f, indent=1)


def _layout(F):
    return F.TransformerModel(F.ModelConfig(*CFG_T), precision="f32", max_batch=1).layout()


@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_headline_forward_backward_per_entry(F, fx, theta0, precision):
    tol = TOL[precision]
    model = F.TransformerModel(F.ModelConfig(*CFG_T), precision=precision, max_batch=B)
    loss, g = model.forward_loss(theta0, F.Batch(fx["inputs"], fx["targets"], B, CFG_T[5]))
    l_ref = float(fx["loss"])
    rows = [{"entry": "loss", "got": loss, "ref": l_ref, "rel": abs(loss - l_ref) / l_ref}]
    g_total = float(np.sqrt(sum(float(fx[f"g_norm/{n}"]) ** 2 for n in fx["names"])))
    fails = []
    for name, off, shape in model.layout():
        n = int(np.prod(shape))
        ge = g[off:off + n]
        ref_norm = float(fx[f"g_norm/{name}"])
        got_norm = float(np.linalg.norm(ge))
        if name.endswith(ZERO_ENTRIES):
            r = {"entry": name, "got_norm": got_norm, "ref_norm": ref_norm,
                 "frac_of_total": got_norm / g_total}
            rows.append(r)
            if not got_norm <= 1e-5 * g_total:
                fails.append(r)
            continue
        idx, ref = fx[f"g_idx/{name}"], fx[f"g_val/{name}"].astype(np.float64)
        rel = float(np.linalg.norm(ge[idx] - ref) / np.linalg.norm(ref))
        nrm = abs(got_norm / ref_norm - 1.0)
        r = {"entry": name, "rel": rel, "norm": nrm, "ref_norm": ref_norm}
        rows.append(r)
        if not (rel <= tol["g_rel"] and nrm <= tol["g_norm"]):
            fails.append(r)
    _report(f"headline_grads_{precision}", rows)
    assert rows[0]["rel"] <= tol["loss"], rows[0]
    assert not fails, fails[:8]


def _local_round(F, theta0, precision, opt):
    # tests/golden/make_golden_125m.py: client 1, round 3, step_base 200, tau 2
    corpus = F.generate_corpus("web", 20000, 7, CFG_T[4])
    plan = F.partition_iid(corpus, 2, CFG_T[5], 7)
    if opt == "adamw":
        sched = F.LrSchedule(6e-4, 64, 1024, 0.1)
        local = F.LocalTrainConfig(model=F.ModelConfig(*CFG_T), schedule=sched, local_steps=2,
                                   batch_size=B)
    else:
        sched = F.LrSchedule(0.5, 64, 1024, 0.1)
        local = F.LocalTrainConfig(model=F.ModelConfig(*CFG_T), schedule=sched, opt=1,
                                   sgd_clip_norm=1.0, local_steps=2, batch_size=B)
    stream = F.BatchStream(plan, 1, B, CFG_T[5], F.stream_seed(42, 1))
    return F.run_local_round(theta0, stream, local, 3, 1, 200, precision=precision)


@pytest.mark.parametrize("precision", ["f32", "bf16"])
@pytest.mark.parametrize("opt", ["sgd", "adamw"])
def test_headline_local_round_per_entry(F, fx, theta0, precision, opt):
    tol = TOL[precision]
    res = _local_round(F, theta0, precision, opt)
    cur_ref = int(fx["cursors"][0 if opt == "adamw" else 1])
    assert res.cursor == cur_ref
    losses = np.array([s.loss for s in res.steps])
    ref_losses = fx[f"{opt}_losses"]
    lrel = float(np.max(np.abs(losses - ref_losses) / ref_losses))
    upd = res.theta - theta0
    rows = [{"entry": "losses", "got": losses.tolist(), "ref": ref_losses.tolist(), "rel": lrel}]
    fails = []
    for name, off, shape in _layout(F):
        n = int(np.prod(shape))
        ue = upd[off:off + n]
        ref_norm = float(fx[f"u_norm_{opt}/{name}"])
        idx, ref = fx[f"u_idx/{name}"], fx[f"u_val_{opt}/{name}"].astype(np.float64)
        got = ue[idx]
        nrm = abs(float(np.linalg.norm(ue)) / ref_norm - 1.0) if ref_norm > 0 else 0.0
        r = {"entry": name, "ref_norm": ref_norm, "norm": nrm}
        if name.endswith(ZERO_ENTRIES):
            continue  # the update is a function of rounding noise only
        if opt == "sgd":
            r["rel"] = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
            ok = r["rel"] <= tol["sgd_rel"]
        else:
            live = np.abs(ref) > 0
            r["sign"] = float(np.mean(np.sign(got[live]) == np.sign(ref[live]))) if live.any() \
                else 1.0
            ok = r["sign"] >= tol["adamw_sign"] and nrm <= tol["adamw_norm"]
        rows.append(r)
        if not ok:
            fails.append(r)
    _report(f"headline_round_{opt}_{precision}", rows)
    assert lrel <= tol["loss"], rows[0]
    assert not fails, fails[:8]
