"""Shared oracle composition of run_centralized (baselines.cpp:25-127) for the
centralized-baseline tests: per-worker streams (shard w, stream_seed(seed, w)),
per-worker forward/backward, ascending-worker anchored mean of the gradients,
one AdamW / SGD update, optimizer reset every `reset` steps."""
import numpy as np


def oracle_centralized(oracle, mc, t, corpus, n_workers, steps, reset, seed, data_seed, theta0):
    S = mc.seq_len
    plan = oracle.plan_iid(corpus, n_workers, S, data_seed)
    pw = t.batch_size // n_workers
    theta = np.array(theta0, np.float64)
    m, v = np.zeros_like(theta), np.zeros_like(theta)
    sc = 0
    cursors = [0] * n_workers
    losses = []
    for step in range(steps):
        if reset and step % reset == 0:
            m[:] = 0.0
            v[:] = 0.0
            sc = 0
        grads, ls = [], []
        for w in range(n_workers):
            inp, tgt, cursors[w] = oracle.stream_next(plan, w, pw, oracle.stream_seed(seed, w),
                                                      cursors[w])
            loss, g = oracle.forward_backward(mc, theta, inp, tgt, pw, S)
            ls.append(loss)
            grads.append(g)
        acc = 0.0
        for x in ls:
            acc += x
        losses.append(acc / n_workers)
        g = oracle.mean(grads)
        lr = oracle.lr_at(t, step)
        if t.opt == 0:
            sc = oracle.adamw_step(theta, g, m, v, sc, t, lr)
        else:
            oracle.sgd_step(theta, g, lr, t.sgd_clip_norm)
    return theta, np.array(losses), cursors
