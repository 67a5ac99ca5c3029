"""Golden fixture at the 125M ARCHITECTURE (L12 d768 H12 e4 V50368), reduced B and S.

Runs the unmodified reference (oracle/_ref/libfedsim_ref.so, compiled by
oracle/Makefile from /root/reference/proj/core/src) once and stores what the
GPU parity tests compare against (tests/test_gpu_headline.py):

  * forward_loss + backward + collect_grads (model.cpp:98-174) on one B=2, S=256
    batch of client 0 (M = 512 rows > 2 x 148, so the persistent cross-entropy
    kernel's refill path runs; V = 50,368 is the headline vocabulary):
    the loss, every canonical entry's gradient L2 norm, every 1-D entry
    (gains, biases incl. head.b) in full, 1,024 fixed samples of every matrix;
  * run_local_round (client.cpp:125-158) with tau = 2 for client 1, once with
    AdamW (the headline optimizer) and once with clipped SGD (update linear in
    the gradients, acceptance_main.cpp:254-255): both step losses, every
    entry's update L2 norm ||theta_out - theta_0|| and 256 samples of the update.

Sample values are stored as float32 (the tests' tolerances are >= 1e-5 relative),
the loss and norms as float64.  About 10 minutes on 3 host cores (the three
reference calls run in parallel processes).

    python tests/golden/make_golden_125m.py
"""
import multiprocessing as mp
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ModelCfg, TrainCfg, build, load_oracle, load_reference  # noqa: E402

CFG = ModelCfg(12, 768, 12, 4, 50368, 256)
B = 2
TOKENS = 20000      # corpus "web", data_seed 7: 77 blocks of S+1, IID over 2 shards
SHARDS = 2
SEED = 42           # stream_seed(42, client)
MODEL_SEED = 1
STEP_BASE = 200     # past warmup: lr_at is on the cosine branch
ADAMW = TrainCfg(eta_max=6e-4, warmup_steps=64, decay_steps=1024, alpha=0.1, local_steps=2,
                 batch_size=B)
SGD = TrainCfg(eta_max=0.5, warmup_steps=64, decay_steps=1024, alpha=0.1, opt=1,
               sgd_clip_norm=1.0, local_steps=2, batch_size=B)
OUT = os.path.join(HERE, "arch125m_b2_s256.npz")


def _fwdbwd(_):
    ref = load_reference()
    theta0 = ref.init_params(CFG, MODEL_SEED)
    inp, tgt, _ = ref.stream(0, "web", TOKENS, 7, CFG.vocab_size, SHARDS, CFG.seq_len, 0, B,
                             SEED, 0, 1)
    loss, g = ref.forward_backward(CFG, theta0, inp, tgt, B, CFG.seq_len)
    return loss, g, inp, tgt


def _round(t):
    ref = load_reference()
    theta0 = ref.init_params(CFG, MODEL_SEED)
    th, losses, cur = ref.local_round(CFG, t, 0, "web", TOKENS, 7, SHARDS, 1, SEED, 0, 3,
                                      STEP_BASE, theta0)
    return th - theta0, losses, cur


def main():
    build()
    assert load_reference() is not None, "reference not built (needs /root/reference)"
    layout = load_oracle().layout(CFG)
    with mp.get_context("fork").Pool(3) as pool:
        fb = pool.apply_async(_fwdbwd, (0,))
        ra = pool.apply_async(_round, (ADAMW,))
        rs = pool.apply_async(_round, (SGD,))
        loss, g, inp, tgt = fb.get()
        upd_a, loss_a, cur_a = ra.get()
        upd_s, loss_s, cur_s = rs.get()

    rng = np.random.default_rng(2024)
    out = {"loss": np.float64(loss), "inputs": inp, "targets": tgt,
           "adamw_losses": loss_a, "sgd_losses": loss_s,
           "cursors": np.array([cur_a, cur_s], np.uint64)}
    names = []
    for name, off, shape in layout:
        n = int(np.prod(shape))
        names.append(name)
        gs = g[off:off + n]
        out[f"g_norm/{name}"] = np.float64(np.linalg.norm(gs))
        if len(shape) == 1:
            gidx = np.arange(n, dtype=np.int64)
        else:
            gidx = np.sort(rng.choice(n, 1024, replace=False)).astype(np.int64)
        out[f"g_idx/{name}"] = gidx
        out[f"g_val/{name}"] = gs[gidx].astype(np.float32)
        uidx = np.sort(rng.choice(n, min(n, 256), replace=False)).astype(np.int64)
        out[f"u_idx/{name}"] = uidx
        for tag, upd in (("adamw", upd_a), ("sgd", upd_s)):
            us = upd[off:off + n]
            out[f"u_norm_{tag}/{name}"] = np.float64(np.linalg.norm(us))
            out[f"u_val_{tag}/{name}"] = us[uidx].astype(np.float32)
    out["names"] = np.array(names)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, f"loss {loss!r} adamw {list(loss_a)} sgd {list(loss_s)} "
          f"cursors {cur_a} {cur_s}")


if __name__ == "__main__":
    main()
