"""ctypes bindings for the oracle libraries (test infrastructure only)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfedsim_ref.so")

STYLES = ["academic", "web", "reference", "prose"]  # data.cpp:24-29


def build(quiet: bool = True) -> None:
    """Run oracle/Makefile (restatement always; reference when its sources exist)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


@dataclass
class ModelCfg:  # ModelConfig model.h:12-25 (defaults kept)
    n_blocks: int = 2
    d_model: int = 64
    n_heads: int = 2
    expansion_ratio: int = 4
    vocab_size: int = 64
    seq_len: int = 32

    def as_array(self):
        return (C.c_uint64 * 6)(self.n_blocks, self.d_model, self.n_heads,
                                self.expansion_ratio, self.vocab_size, self.seq_len)

    def param_count(self) -> int:  # model.cpp:21-26
        d, e = self.d_model, self.expansion_ratio
        per_block = (4 + 2 * e) * d * d + (9 + e) * d
        return (self.vocab_size * d + self.seq_len * d + self.n_blocks * per_block + 2 * d
                + d * self.vocab_size + self.vocab_size)


@dataclass
class TrainCfg:  # LrSchedule + AdamWConfig + LocalTrainConfig (optim.h, client.h)
    eta_max: float = 6e-4
    warmup_steps: int = 64
    decay_steps: int = 1024
    alpha: float = 0.1
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.01
    clip_norm: float = 1.0
    opt: int = 0  # 0 AdamW, 1 SGD
    sgd_clip_norm: float = 0.0
    local_steps: int = 64
    batch_size: int = 8
    post_kind: int = 0
    post_threshold: float = 0.0

    def as_doubles(self):
        return (C.c_double * 15)(self.eta_max, self.warmup_steps, self.decay_steps, self.alpha,
                                 self.beta1, self.beta2, self.eps, self.weight_decay,
                                 self.clip_norm, self.opt, self.sgd_clip_norm,
                                 self.local_steps, self.batch_size, self.post_kind,
                                 self.post_threshold)


@dataclass
class ServerCfg:  # ServerOptConfig optim.h:54-63
    kind: int = 0  # 0 FedAvg, 1 FedMomentum
    eta: float = 1.0
    momentum: float = 0.0
    nesterov: int = 0

    def as_doubles(self):
        return (C.c_double * 4)(self.kind, self.eta, self.momentum, self.nesterov)


class _OrcModel(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("n_blocks", "d_model", "n_heads", "expansion_ratio", "vocab_size", "seq_len")]


class _OrcTrain(C.Structure):
    _fields_ = [("eta_max", C.c_double), ("warmup_steps", C.c_uint64),
                ("decay_steps", C.c_uint64), ("alpha", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("weight_decay", C.c_double),
                ("clip_norm", C.c_double), ("opt", C.c_int32), ("sgd_clip_norm", C.c_double),
                ("local_steps", C.c_uint64), ("batch_size", C.c_uint64),
                ("post_kind", C.c_int32), ("post_threshold", C.c_double)]


class _OrcServer(C.Structure):
    _fields_ = [("kind", C.c_int32), ("eta", C.c_double), ("momentum", C.c_double),
                ("nesterov", C.c_int32)]


def _m(cfg: ModelCfg) -> _OrcModel:
    return _OrcModel(cfg.n_blocks, cfg.d_model, cfg.n_heads, cfg.expansion_ratio,
                     cfg.vocab_size, cfg.seq_len)


def _t(t: TrainCfg) -> _OrcTrain:
    return _OrcTrain(t.eta_max, t.warmup_steps, t.decay_steps, t.alpha, t.beta1, t.beta2,
                     t.eps, t.weight_decay, t.clip_norm, t.opt, t.sgd_clip_norm,
                     t.local_steps, t.batch_size, t.post_kind, t.post_threshold)


def _s(s: ServerCfg) -> _OrcServer:
    return _OrcServer(s.kind, s.eta, s.momentum, s.nesterov)


def _p(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: oracle error code {code}")
        self.code = code


def _check(rc: int, where: str) -> None:
    if rc != 0:
        raise OracleError(rc, where)


class Plan:
    """Owning handle for an orc_plan (data.cpp ShardPlan restatement)."""

    def __init__(self, lib, ptr, seq_len: int):
        self._lib, self.ptr, self.seq_len = lib, ptr, seq_len

    def __del__(self):
        if self.ptr:
            self._lib.orc_plan_free(self.ptr)
            self.ptr = None

    @property
    def n_clients(self) -> int:
        return int(self._lib.orc_plan_n_clients(self.ptr))

    def client_blocks(self, client: int) -> int:
        return int(self._lib.orc_plan_client_blocks(self.ptr, client))

    def blocks(self, client: int):
        src, off = C.c_uint32(), C.c_uint64()
        out = []
        for b in range(self.client_blocks(client)):
            self._lib.orc_plan_block(self.ptr, client, b, C.byref(src), C.byref(off))
            out.append((src.value, off.value))
        return out


class Oracle:
    """The C restatement (fedsim_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.lib = L
        u64, i32, dbl = C.c_uint64, C.c_int32, C.c_double
        P = C.POINTER
        L.orc_mix64.restype = u64
        L.orc_mix64.argtypes = [u64]
        L.orc_param_count.restype = u64
        L.orc_layout_size.restype = u64
        L.orc_stream_seed.restype = u64
        L.orc_stream_seed.argtypes = [u64, u64]
        L.orc_global_norm.restype = dbl
        L.orc_global_norm.argtypes = [P(dbl), u64]
        L.orc_plan_iid.restype = C.c_void_p
        L.orc_plan_iid.argtypes = [P(C.c_uint16), u64, u64, u64, u64, P(C.c_int)]
        L.orc_plan_by_source.restype = C.c_void_p
        L.orc_plan_by_source.argtypes = [P(P(C.c_uint16)), P(u64), u64, u64, u64, P(C.c_int)]
        L.orc_plan_free.argtypes = [C.c_void_p]
        L.orc_plan_n_clients.restype = u64
        L.orc_plan_n_clients.argtypes = [C.c_void_p]
        L.orc_plan_client_blocks.restype = u64
        L.orc_plan_client_blocks.argtypes = [C.c_void_p, u64]
        L.orc_plan_block.argtypes = [C.c_void_p, u64, u64, P(C.c_uint32), P(u64)]
        L.orc_stream_next.argtypes = [C.c_void_p, u64, u64, u64, u64, P(u64), P(i32), P(i32)]
        L.orc_local_round.argtypes = [P(_OrcModel), P(_OrcTrain), P(dbl), C.c_void_p, u64, u64,
                                      P(u64), u64, u64, P(dbl), P(dbl), P(u64)]
        L.orc_run_round.argtypes = [P(_OrcModel), P(_OrcTrain), P(_OrcServer), C.c_void_p, u64,
                                    u64, u64, u64, P(dbl), P(dbl), P(u64), P(u64), u64, i32,
                                    P(u64), P(dbl)]
        L.orc_sample_clients.argtypes = [u64, u64, u64, u64, P(u64)]
        L.orc_generate_corpus.argtypes = [i32, u64, u64, C.c_uint32, P(C.c_uint16)]
        L.orc_rng_draws.argtypes = [u64, u64, P(u64), P(dbl), P(dbl)]
        L.orc_mix_seed.restype = u64
        L.orc_mix_seed.argtypes = [u64, u64]
        L.orc_mix_seed2.restype = u64
        L.orc_mix_seed2.argtypes = [u64, u64, u64]
        L.orc_mix_seed3.restype = u64
        L.orc_mix_seed3.argtypes = [u64, u64, u64, u64]

    # --- rng ---------------------------------------------------------------
    def mix64(self, x: int) -> int:
        return int(self.lib.orc_mix64(x))

    def mix_seed(self, seed, *args) -> int:
        f = {1: self.lib.orc_mix_seed, 2: self.lib.orc_mix_seed2, 3: self.lib.orc_mix_seed3}
        return int(f[len(args)](seed, *args))

    def rng_draws(self, seed: int, n: int):
        u = np.zeros(n, np.uint64)
        f = np.zeros(n)
        g = np.zeros(n)
        self.lib.orc_rng_draws(seed, n, _p(u, C.c_uint64), _p(f, C.c_double), _p(g, C.c_double))
        return u, f, g

    # --- model -------------------------------------------------------------
    def param_count(self, cfg: ModelCfg) -> int:
        m = _m(cfg)
        return int(self.lib.orc_param_count(C.byref(m)))

    def layout(self, cfg: ModelCfg):
        m = _m(cfg)
        n = int(self.lib.orc_layout_size(C.byref(m)))
        out = []
        off, r, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        name = C.create_string_buffer(64)
        for i in range(n):
            self.lib.orc_layout_entry(C.byref(m), C.c_uint64(i), C.byref(off), C.byref(r),
                                      C.byref(c), name, 64)
            shape = (r.value, c.value) if c.value else (r.value,)
            out.append((name.value.decode(), off.value, shape))
        return out

    def init_params(self, cfg: ModelCfg, seed: int) -> np.ndarray:
        out = np.zeros(cfg.param_count())
        m = _m(cfg)
        _check(self.lib.orc_init_params(C.byref(m), C.c_uint64(seed), _p(out, C.c_double)),
               "init_params")
        return out

    def forward_backward(self, cfg: ModelCfg, params, inputs, targets, batch: int, seq: int,
                         grads: bool = True):
        m = _m(cfg)
        params = np.ascontiguousarray(params, np.float64)
        inputs = np.ascontiguousarray(inputs, np.int32)
        targets = np.ascontiguousarray(targets, np.int32)
        loss = C.c_double()
        g = np.zeros(cfg.param_count()) if grads else None
        _check(self.lib.orc_forward_backward(
            C.byref(m), _p(params, C.c_double), _p(inputs, C.c_int32), _p(targets, C.c_int32),
            C.c_uint64(batch), C.c_uint64(seq), C.byref(loss),
            _p(g, C.c_double) if grads else None), "forward_backward")
        return loss.value, g

    def eval_perplexity(self, cfg: ModelCfg, params, inputs, targets, batch_sizes, seq: int):
        m = _m(cfg)
        params = np.ascontiguousarray(params, np.float64)
        inputs = np.ascontiguousarray(inputs, np.int32)
        targets = np.ascontiguousarray(targets, np.int32)
        bs = np.ascontiguousarray(batch_sizes, np.uint64)
        out = C.c_double()
        _check(self.lib.orc_eval_perplexity(
            C.byref(m), _p(params, C.c_double), _p(inputs, C.c_int32), _p(targets, C.c_int32),
            C.c_uint64(len(bs)), _p(bs, C.c_uint64), C.c_uint64(seq), C.byref(out)),
            "eval_perplexity")
        return out.value

    # --- data --------------------------------------------------------------
    def generate_corpus(self, style: str, length: int, seed: int, vocab: int = 64):
        out = np.zeros(length, np.uint16)
        _check(self.lib.orc_generate_corpus(STYLES.index(style), length, seed, vocab,
                                            _p(out, C.c_uint16)), "generate_corpus")
        return out

    def plan_iid(self, tokens: np.ndarray, n_shards: int, seq_len: int, seed: int) -> Plan:
        tokens = np.ascontiguousarray(tokens, np.uint16)
        err = C.c_int()
        ptr = self.lib.orc_plan_iid(_p(tokens, C.c_uint16), len(tokens), n_shards, seq_len, seed,
                                    C.byref(err))
        _check(err.value, "plan_iid")
        return Plan(self.lib, ptr, seq_len)

    def plan_by_source(self, corpora, clients_per_source: int, seq_len: int) -> Plan:
        arrs = [np.ascontiguousarray(c, np.uint16) for c in corpora]
        ptrs = (C.POINTER(C.c_uint16) * len(arrs))(*[_p(a, C.c_uint16) for a in arrs])
        lens = (C.c_uint64 * len(arrs))(*[len(a) for a in arrs])
        err = C.c_int()
        ptr = self.lib.orc_plan_by_source(ptrs, lens, len(arrs), clients_per_source, seq_len,
                                          C.byref(err))
        _check(err.value, "plan_by_source")
        return Plan(self.lib, ptr, seq_len)

    def stream_seed(self, seed: int, client: int) -> int:
        return int(self.lib.orc_stream_seed(seed, client))

    def stream_next(self, plan: Plan, client: int, batch: int, seed: int, cursor: int):
        S = plan.seq_len
        inp = np.zeros(batch * S, np.int32)
        tgt = np.zeros(batch * S, np.int32)
        cur = C.c_uint64(cursor)
        _check(self.lib.orc_stream_next(plan.ptr, client, batch, S, seed, C.byref(cur),
                                        _p(inp, C.c_int32), _p(tgt, C.c_int32)), "stream_next")
        return inp, tgt, cur.value

    # --- optim / aggregation -----------------------------------------------
    def sample_clients(self, population: int, k: int, seed: int, round_: int):
        out = np.zeros(k, np.uint64)
        _check(self.lib.orc_sample_clients(population, k, seed, round_, _p(out, C.c_uint64)),
               "sample_clients")
        return [int(x) for x in out]

    def lr_at(self, t: TrainCfg, step: int) -> float:
        tt = _t(t)
        out = C.c_double()
        _check(self.lib.orc_lr_at(C.byref(tt), C.c_uint64(step), C.byref(out)), "lr_at")
        return out.value

    def global_norm(self, x) -> float:
        x = np.ascontiguousarray(x, np.float64)
        return float(self.lib.orc_global_norm(_p(x, C.c_double), len(x)))

    def adamw_step(self, p, g, m, v, step_count: int, t: TrainCfg, lr: float) -> int:
        sc = C.c_uint64(step_count)
        tt = _t(t)
        _check(self.lib.orc_adamw_step(_p(p, C.c_double), _p(g, C.c_double), _p(m, C.c_double),
                                       _p(v, C.c_double), C.c_uint64(len(p)), C.byref(sc),
                                       C.byref(tt), C.c_double(lr)), "adamw_step")
        return sc.value

    def sgd_step(self, p, g, lr: float, clip_norm: float = 0.0) -> None:
        _check(self.lib.orc_sgd_step(_p(p, C.c_double), _p(g, C.c_double), C.c_uint64(len(p)),
                                     C.c_double(lr), C.c_double(clip_norm)), "sgd_step")

    def mean(self, vs) -> np.ndarray:
        arrs = [np.ascontiguousarray(v, np.float64) for v in vs]
        ptrs = (C.POINTER(C.c_double) * len(arrs))(*[_p(a, C.c_double) for a in arrs])
        n = len(arrs[0]) if arrs else 0
        out = np.zeros(n)
        _check(self.lib.orc_mean(ptrs, C.c_uint64(len(arrs)), C.c_uint64(n),
                                 _p(out, C.c_double)), "mean")
        return out

    def sub(self, a, b) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.zeros_like(a)
        self.lib.orc_sub(_p(a, C.c_double), _p(b, C.c_double), C.c_uint64(len(a)),
                         _p(out, C.c_double))
        return out

    def server_step(self, s: ServerCfg, theta, delta, mean, velocity) -> np.ndarray:
        ss = _s(s)
        out = np.zeros(len(theta))
        theta, delta, mean = (np.ascontiguousarray(x, np.float64) for x in (theta, delta, mean))
        _check(self.lib.orc_server_step(C.byref(ss), _p(theta, C.c_double),
                                        _p(delta, C.c_double), _p(mean, C.c_double),
                                        _p(velocity, C.c_double), C.c_uint64(len(theta)),
                                        _p(out, C.c_double)), "server_step")
        return out

    # --- client / round ------------------------------------------------------
    def local_round(self, cfg: ModelCfg, t: TrainCfg, theta, plan: Plan, client: int,
                    seed: int, cursor: int, round_: int, step_base: int):
        m, tt = _m(cfg), _t(t)
        theta = np.ascontiguousarray(theta, np.float64)
        out = np.zeros_like(theta)
        losses = np.zeros(max(t.local_steps, 1))
        cur = C.c_uint64(cursor)
        es = C.c_uint64()
        _check(self.lib.orc_local_round(C.byref(m), C.byref(tt), _p(theta, C.c_double),
                                        plan.ptr, C.c_uint64(client),
                                        C.c_uint64(self.stream_seed(seed, client)),
                                        C.byref(cur), C.c_uint64(round_), C.c_uint64(step_base),
                                        _p(out, C.c_double), _p(losses, C.c_double),
                                        C.byref(es)), "local_round")
        return out, losses[: t.local_steps], cur.value

    def run_round(self, cfg: ModelCfg, t: TrainCfg, s: ServerCfg, plan: Plan, population: int,
                  k: int, seed: int, round_: int, theta, velocity, cursors, dropped=(),
                  ring: bool = False):
        m, tt, ss = _m(cfg), _t(t), _s(s)
        dr = np.ascontiguousarray(list(dropped) or [0], np.uint64)
        sampled = np.zeros(k, np.uint64)
        losses = np.zeros(k)
        _check(self.lib.orc_run_round(C.byref(m), C.byref(tt), C.byref(ss), plan.ptr,
                                      population, k, seed, round_, _p(theta, C.c_double),
                                      _p(velocity, C.c_double), _p(cursors, C.c_uint64),
                                      _p(dr, C.c_uint64), len(dropped), int(ring),
                                      _p(sampled, C.c_uint64), _p(losses, C.c_double)),
               "run_round")
        return [int(x) for x in sampled], losses


class Reference:
    """The unmodified reference compiled from /root/reference (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.lib = L
        L.ref_mix64.restype = C.c_uint64
        L.ref_mix64.argtypes = [C.c_uint64]
        L.ref_param_count.restype = C.c_uint64

    def mix64(self, x: int) -> int:
        return int(self.lib.ref_mix64(x))

    def rng_normals(self, seed: int, n: int):
        out = np.zeros(n)
        self.lib.ref_rng_normals(C.c_uint64(seed), C.c_uint64(n), _p(out, C.c_double))
        return out

    def init_params(self, cfg: ModelCfg, seed: int):
        out = np.zeros(cfg.param_count())
        _check(self.lib.ref_init_params(cfg.as_array(), C.c_uint64(seed), _p(out, C.c_double)),
               "ref_init_params")
        return out

    def generate_corpus(self, style: str, length: int, seed: int, vocab: int = 64):
        out = np.zeros(length, np.uint16)
        _check(self.lib.ref_generate_corpus(C.c_int32(STYLES.index(style)), C.c_uint64(length),
                                            C.c_uint64(seed), C.c_uint32(vocab),
                                            _p(out, C.c_uint16)), "ref_generate_corpus")
        return out

    def sample_clients(self, population, k, seed, round_):
        out = np.zeros(k, np.uint64)
        _check(self.lib.ref_sample_clients(C.c_uint64(population), C.c_uint64(k),
                                           C.c_uint64(seed), C.c_uint64(round_),
                                           _p(out, C.c_uint64)), "ref_sample_clients")
        return [int(x) for x in out]

    def lr_at(self, t: TrainCfg, step: int) -> float:
        s = (C.c_double * 4)(t.eta_max, t.warmup_steps, t.decay_steps, t.alpha)
        out = C.c_double()
        _check(self.lib.ref_lr_at(s, C.c_uint64(step), C.byref(out)), "ref_lr_at")
        return out.value

    def stream(self, policy: int, style: str, tokens: int, data_seed: int, vocab: int,
               shards: int, seq_len: int, client: int, batch: int, seed: int, cursor: int,
               n_steps: int):
        inp = np.zeros(n_steps * batch * seq_len, np.int32)
        tgt = np.zeros_like(inp)
        cur = C.c_uint64()
        _check(self.lib.ref_stream(C.c_int32(policy), C.c_int32(STYLES.index(style)),
                                   C.c_uint64(tokens), C.c_uint64(data_seed), C.c_uint32(vocab),
                                   C.c_uint64(shards), C.c_uint64(seq_len), C.c_uint64(client),
                                   C.c_uint64(batch), C.c_uint64(seed), C.c_uint64(cursor),
                                   C.c_uint64(n_steps), _p(inp, C.c_int32),
                                   _p(tgt, C.c_int32), C.byref(cur)), "ref_stream")
        return inp, tgt, cur.value

    def forward_backward(self, cfg: ModelCfg, params, inputs, targets, batch, seq,
                         grads: bool = True):
        params = np.ascontiguousarray(params, np.float64)
        inputs = np.ascontiguousarray(inputs, np.int32)
        targets = np.ascontiguousarray(targets, np.int32)
        loss = C.c_double()
        g = np.zeros(cfg.param_count()) if grads else None
        _check(self.lib.ref_forward_backward(cfg.as_array(), _p(params, C.c_double),
                                             _p(inputs, C.c_int32), _p(targets, C.c_int32),
                                             C.c_uint64(batch), C.c_uint64(seq), C.byref(loss),
                                             _p(g, C.c_double) if grads else None),
               "ref_forward_backward")
        return loss.value, g

    def adamw_step(self, p, g, m, v, step_count, t: TrainCfg, lr):
        sc = C.c_uint64(step_count)
        _check(self.lib.ref_adamw_step(_p(p, C.c_double), _p(g, C.c_double),
                                       _p(m, C.c_double), _p(v, C.c_double),
                                       C.c_uint64(len(p)), C.byref(sc), t.as_doubles(),
                                       C.c_double(lr)), "ref_adamw_step")
        return sc.value

    def mean(self, vs):
        arrs = [np.ascontiguousarray(v, np.float64) for v in vs]
        ptrs = (C.POINTER(C.c_double) * len(arrs))(*[_p(a, C.c_double) for a in arrs])
        out = np.zeros(len(arrs[0]))
        _check(self.lib.ref_mean(ptrs, C.c_uint64(len(arrs)), C.c_uint64(len(out)),
                                 _p(out, C.c_double)), "ref_mean")
        return out

    def server_step(self, s: ServerCfg, theta, delta, mean, velocity):
        out = np.zeros(len(theta))
        theta, delta, mean = (np.ascontiguousarray(x, np.float64) for x in (theta, delta, mean))
        _check(self.lib.ref_server_step(s.as_doubles(), _p(theta, C.c_double),
                                        _p(delta, C.c_double), _p(mean, C.c_double),
                                        _p(velocity, C.c_double), C.c_uint64(len(theta)),
                                        _p(out, C.c_double)), "ref_server_step")
        return out

    def local_round(self, cfg: ModelCfg, t: TrainCfg, policy, style, tokens, data_seed,
                    shards, client, seed, cursor, round_, step_base, theta):
        theta = np.ascontiguousarray(theta, np.float64)
        out = np.zeros_like(theta)
        losses = np.zeros(max(t.local_steps, 1))
        cur = C.c_uint64()
        _check(self.lib.ref_local_round(cfg.as_array(), t.as_doubles(), C.c_int32(policy),
                                        C.c_int32(STYLES.index(style)), C.c_uint64(tokens),
                                        C.c_uint64(data_seed), C.c_uint64(shards),
                                        C.c_uint64(client), C.c_uint64(seed),
                                        C.c_uint64(cursor), C.c_uint64(round_),
                                        C.c_uint64(step_base), _p(theta, C.c_double),
                                        _p(out, C.c_double), _p(losses, C.c_double),
                                        C.byref(cur)), "ref_local_round")
        return out, losses[: t.local_steps], cur.value

    def run_rounds(self, cfg: ModelCfg, t: TrainCfg, s: ServerCfg, policy, style, tokens,
                   data_seed, population, k, rounds, seed, topology, n_threads, theta0):
        theta0 = np.ascontiguousarray(theta0, np.float64)
        out = np.zeros_like(theta0)
        vel = np.zeros_like(theta0)
        losses = np.zeros(rounds)
        secs = np.zeros(rounds)
        _check(self.lib.ref_run_rounds(cfg.as_array(), t.as_doubles(), s.as_doubles(),
                                       C.c_int32(policy), C.c_int32(STYLES.index(style)),
                                       C.c_uint64(tokens), C.c_uint64(data_seed),
                                       C.c_uint64(population), C.c_uint64(k),
                                       C.c_uint64(rounds), C.c_uint64(seed),
                                       C.c_int32(topology), C.c_uint64(n_threads),
                                       _p(theta0, C.c_double), _p(out, C.c_double),
                                       _p(vel, C.c_double), _p(losses, C.c_double),
                                       _p(secs, C.c_double)), "ref_run_rounds")
        return out, vel, losses, secs

    def train_sample(self, cfg: ModelCfg, t: TrainCfg, batch: int, seq: int, steps: int,
                     threads: int):
        """(wall seconds, last loss) of `threads` reference clients x `steps` steps."""
        secs, loss = C.c_double(), C.c_double()
        _check(self.lib.ref_train_sample(cfg.as_array(), t.as_doubles(), C.c_uint64(batch),
                                         C.c_uint64(seq), C.c_uint64(steps),
                                         C.c_uint64(threads), C.byref(secs), C.byref(loss)),
               "ref_train_sample")
        return secs.value, loss.value

    def run_experiment_fed(self, cfg: ModelCfg, t: TrainCfg, s: ServerCfg, corpus_tokens,
                           population, rounds, seed, model_seed, data_seed, eval_sequences,
                           eval_batch, out_dir: str):
        ppl = np.zeros(2)
        _check(self.lib.ref_run_experiment_fed(cfg.as_array(), t.as_doubles(), s.as_doubles(),
                                               C.c_uint64(corpus_tokens),
                                               C.c_uint64(population), C.c_uint64(rounds),
                                               C.c_uint64(seed), C.c_uint64(model_seed),
                                               C.c_uint64(data_seed),
                                               C.c_uint64(eval_sequences),
                                               C.c_uint64(eval_batch),
                                               out_dir.encode(), _p(ppl, C.c_double)),
               "ref_run_experiment_fed")
        return float(ppl[0]), float(ppl[1])


    def run_centralized(self, cfg: ModelCfg, t: TrainCfg, style, tokens, data_seed, n_workers,
                        total_steps, reset, seed, theta0):
        """baselines.cpp:25-127 (t.batch_size is the global batch)."""
        theta0 = np.ascontiguousarray(theta0, np.float64)
        out = np.zeros_like(theta0)
        losses = np.zeros(total_steps)
        cursors = np.zeros(n_workers, np.uint64)
        _check(self.lib.ref_run_centralized(cfg.as_array(), t.as_doubles(),
                                            C.c_int32(STYLES.index(style)), C.c_uint64(tokens),
                                            C.c_uint64(data_seed), C.c_uint64(n_workers),
                                            C.c_uint64(total_steps), C.c_uint64(reset),
                                            C.c_uint64(seed), _p(theta0, C.c_double),
                                            _p(out, C.c_double), _p(losses, C.c_double),
                                            _p(cursors, C.c_uint64)), "ref_run_centralized")
        return out, losses, cursors

    def write_checkpoint(self, cfg: ModelCfg, params, round_: int, path: str) -> None:
        _check(self.lib.ref_write_checkpoint(cfg.as_array(), _p(np.ascontiguousarray(params,
                                             np.float64), C.c_double), C.c_uint64(round_),
                                             path.encode()), "ref_write_checkpoint")

    def read_checkpoint(self, cfg: ModelCfg, path: str):
        out = np.zeros(cfg.param_count())
        rd = C.c_uint64()
        _check(self.lib.ref_read_checkpoint(path.encode(), _p(out, C.c_double),
                                            C.c_uint64(len(out)), C.byref(rd)),
               "ref_read_checkpoint")
        return out, int(rd.value)


_ORACLE = None
_REF = None


def load_oracle() -> Oracle:
    global _ORACLE
    if _ORACLE is None:
        _ORACLE = Oracle()
    return _ORACLE


def load_reference():
    """The compiled reference, or None when oracle/_ref was never built."""
    global _REF
    if _REF is None and os.path.exists(REF_SO):
        _REF = Reference()
    return _REF
