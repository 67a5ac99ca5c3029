"""Reference-facing host API of the B200 Photon round.

Mirrors the names, argument meaning and error behaviour of the reference
library `fedsim::core` (/root/reference/proj/core/include/fedsim/*.h) for the
federated-round path, so the parity tests read like the reference's own unit
tests.  Every call goes through the C ABI of libphoton.so (include/photon.h);
parameters cross the boundary as flat f64 numpy arrays in canonical order
(ParamVector::flatten, param_vector.cpp:154-159).  There is no CPU fallback.
"""
from __future__ import annotations

import builtins
import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi as A

# ---------------------------------------------------------------------------
# errors (fedsim/errors.h:9-72)
# ---------------------------------------------------------------------------


class FedsimError(RuntimeError):
    pass


class ConfigError(FedsimError):
    pass


class CapacityError(ConfigError):
    pass


class ShapeError(FedsimError):
    pass


class IndexError(FedsimError, builtins.IndexError):  # noqa: A001 - reference name
    pass


class UsageError(FedsimError):
    pass


class LookupError(FedsimError, builtins.LookupError):  # noqa: A001 - reference name
    pass


class NumericError(FedsimError):
    pass


class DivergenceError(NumericError):
    def __init__(self, what: str, round: int, client: int, step: int):  # noqa: A002
        super().__init__(what)
        self.round, self.client, self.step = round, client, step


class IoError(FedsimError):
    pass


class IntegrityError(IoError):
    pass


class RoundFailureError(FedsimError):
    pass


class ParseError(FedsimError):
    pass


class DeviceError(FedsimError):
    """CUDA / NCCL failure (no reference equivalent)."""


_CODE = {1: ConfigError, 2: CapacityError, 3: ShapeError, 4: IndexError, 5: UsageError,
         6: LookupError, 7: NumericError, 9: IoError, 10: IntegrityError, 11: RoundFailureError,
         12: ParseError, 20: DeviceError, 21: DeviceError}


def _raise(rc: int, err: A.photon_err):
    if rc == 0:
        return
    msg = err.msg.decode(errors="replace")
    if rc == 8:
        raise DivergenceError(msg, int(err.round), int(err.client), int(err.step))
    raise _CODE.get(rc, FedsimError)(msg)


def _call(fn, *args):
    err = A.photon_err()
    rc = fn(*args, C.byref(err))
    _raise(rc, err)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


# ---------------------------------------------------------------------------
# configs (model.h, optim.h, client.h, aggregator.h)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class ModelConfig:
    n_blocks: int = 2
    d_model: int = 64
    n_heads: int = 2
    expansion_ratio: int = 4
    vocab_size: int = 64
    seq_len: int = 32

    def c(self) -> A.photon_model_cfg:
        return A.photon_model_cfg(self.n_blocks, self.d_model, self.n_heads,
                                  self.expansion_ratio, self.vocab_size, self.seq_len)

    def validate(self) -> None:  # model.cpp:10-19
        if self.n_blocks == 0 or self.d_model == 0 or self.n_heads == 0 or \
                self.d_model % self.n_heads or self.expansion_ratio == 0 or \
                self.vocab_size < 2 or self.seq_len == 0:
            raise ConfigError("model: invalid configuration")

    def param_count(self) -> int:
        return int(A.lib().photon_param_count(C.byref(self.c())))

    def payload_mib(self) -> float:
        return self.param_count() * 8.0 / (1024.0 * 1024.0)


@dataclass
class LrSchedule:
    eta_max: float = 6e-4
    warmup_steps: int = 64
    decay_steps: int = 1024
    alpha: float = 0.1

    def c(self):
        return A.photon_lr_schedule(self.eta_max, self.warmup_steps, self.decay_steps, self.alpha)


@dataclass
class AdamWConfig:
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.01
    clip_norm: float = 1.0

    def c(self):
        return A.photon_adamw_cfg(self.beta1, self.beta2, self.eps, self.weight_decay,
                                  self.clip_norm)


class ClientOptKind:
    kAdamW = 0
    kSgd = 1


@dataclass
class PostProcessPolicy:
    kind: int = 0  # 0 identity, 1 clip update norm
    threshold: float = 0.0


@dataclass
class LocalTrainConfig:
    model: ModelConfig = field(default_factory=ModelConfig)
    adamw: AdamWConfig = field(default_factory=AdamWConfig)
    schedule: LrSchedule = field(default_factory=LrSchedule)
    opt: int = ClientOptKind.kAdamW
    sgd_clip_norm: float = 0.0
    local_steps: int = 64
    batch_size: int = 8
    throughput_bps: float = 2.0
    post: PostProcessPolicy = field(default_factory=PostProcessPolicy)

    def c(self):
        return A.photon_train_cfg(self.model.c(), self.adamw.c(), self.schedule.c(), self.opt,
                                  self.sgd_clip_norm, self.local_steps, self.batch_size,
                                  self.throughput_bps, self.post.kind, self.post.threshold)


class ServerOptKind:
    FedAvg = 0
    FedMomentum = 1


@dataclass
class ServerOptConfig:
    kind: int = ServerOptKind.FedAvg
    eta: float = 1.0
    momentum: float = 0.0
    nesterov: bool = False

    def c(self):
        return A.photon_server_cfg(self.kind, self.eta, self.momentum, int(self.nesterov))

    def validate(self) -> None:  # optim.cpp:105-113
        if not self.eta > 0.0:
            raise ConfigError("server opt: eta must be > 0")
        if self.momentum < 0.0 or self.momentum >= 1.0:
            raise ConfigError("server opt: momentum must be in [0,1)")
        if self.kind == ServerOptKind.FedAvg and (self.eta != 1.0 or self.momentum != 0.0):
            raise ConfigError("server opt: fedavg is eta=1, momentum=0 by definition")


def diloco_server_opt(momentum: float = 0.9) -> ServerOptConfig:  # baselines.cpp:129-136
    return ServerOptConfig(ServerOptKind.FedMomentum, 0.1, momentum, True)


@dataclass
class CentralizedConfig:
    """baselines.h:19-35."""
    model: ModelConfig = field(default_factory=ModelConfig)
    adamw: AdamWConfig = field(default_factory=AdamWConfig)
    schedule: LrSchedule = field(default_factory=LrSchedule)
    opt: int = ClientOptKind.kAdamW
    sgd_clip_norm: float = 0.0
    n_workers: int = 1
    global_batch: int = 8
    total_steps: int = 1
    opt_reset_interval: int = 0
    throughput_bps: float = 2.0

    def c(self):
        return A.photon_central_cfg(self.model.c(), self.adamw.c(), self.schedule.c(), self.opt,
                                    self.sgd_clip_norm, self.n_workers, self.global_batch,
                                    self.total_steps, self.opt_reset_interval,
                                    self.throughput_bps)


class Topology:
    kParameterServer = 0
    kAllReduce = 1
    kRingAllReduce = 2


@dataclass
class FederationConfig:
    population: int = 1
    clients_per_round: int = 1
    rounds: int = 1
    topology: int = Topology.kRingAllReduce
    seed: int = 0

    def c(self):
        return A.photon_fed_cfg(self.population, self.clients_per_round, self.rounds,
                                self.topology, self.seed)


@dataclass
class StepMetric:
    loss: float
    tokens: int
    sim_seconds: float


@dataclass
class ClientResult:
    theta: np.ndarray
    steps: List[StepMetric]
    cursor: int

    def mean_loss(self) -> float:  # client.cpp:112-117
        return sum(s.loss for s in self.steps) / len(self.steps) if self.steps else 0.0

    def tokens_consumed(self) -> int:
        return sum(s.tokens for s in self.steps)


@dataclass
class RoundRecord:
    round: int
    sampled_ids: List[int]
    mean_client_loss: float
    min_client_loss: float
    max_client_loss: float
    local_ms: float
    aggregate_ms: float
    round_ms: float
    tokens: int
    host_ms: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    eval_ppl: float = float("nan")  # RoundRecord::eval_ppl (NaN when the cadence skips)
    boundary_ms: float = 0.0  # device time of the boundary's exchange + update alone


# ---------------------------------------------------------------------------
# determinism primitives (rng.h, data.cpp, aggregator.cpp:25-41, optim.cpp:16-27)
# ---------------------------------------------------------------------------


def mix64(x: int) -> int:
    return int(A.lib().photon_mix64(x))


def stream_seed(global_seed: int, client: int) -> int:
    return int(A.lib().photon_stream_seed(global_seed, client))


def sample_clients(population: int, k: int, seed: int, round: int) -> List[int]:  # noqa: A002
    out = (C.c_uint64 * max(k, 1))()
    _call(A.lib().photon_sample_clients, population, k, seed, round, out)
    return [int(x) for x in out[:k]]


def lr_at(schedule: LrSchedule, step: int) -> float:
    out = C.c_double()
    s = schedule.c()
    _call(A.lib().photon_lr_at, C.byref(s), step, C.byref(out))
    return out.value


STYLES = ("academic", "web", "reference", "prose")


def known_styles() -> List[str]:
    return list(STYLES)


def generate_corpus(style: str, length: int, seed: int, vocab_size: int = 64) -> np.ndarray:
    out = np.zeros(length, np.uint16)
    _call(A.lib().photon_generate_corpus, style.encode(), length, seed, vocab_size,
          out.ctypes.data_as(C.POINTER(C.c_uint16)))
    return out


class ShardPlan:
    """Immutable assignment of disjoint (seq_len+1)-token blocks to clients."""

    def __init__(self, handle: int, seq_len: int):
        self._h = C.c_void_p(handle)
        self._seq_len = seq_len

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            A.lib().photon_plan_free(self._h)
            self._h = C.c_void_p()

    def n_clients(self) -> int:
        return int(A.lib().photon_plan_n_clients(self._h))

    def seq_len(self) -> int:
        return self._seq_len

    def block_len(self) -> int:
        return self._seq_len + 1

    def client_blocks(self, client: int) -> int:
        if client >= self.n_clients():
            raise LookupError(f"unknown client id {client}")
        return int(A.lib().photon_plan_client_blocks(self._h, client))

    def client_tokens(self, client: int) -> int:
        return self.client_blocks(client) * self.block_len()


def partition_iid(corpus: np.ndarray, n_shards: int, seq_len: int, seed: int) -> ShardPlan:
    toks = np.ascontiguousarray(corpus, np.uint16)
    h = C.c_void_p()
    _call(A.lib().photon_plan_iid, toks.ctypes.data_as(C.POINTER(C.c_uint16)), len(toks),
          n_shards, seq_len, seed, C.byref(h))
    return ShardPlan(h.value, seq_len)


def partition_by_source(corpora: Sequence[np.ndarray], clients_per_source: int,
                        seq_len: int) -> ShardPlan:
    arrs = [np.ascontiguousarray(c, np.uint16) for c in corpora]
    ptrs = (C.POINTER(C.c_uint16) * len(arrs))(
        *[a.ctypes.data_as(C.POINTER(C.c_uint16)) for a in arrs])
    lens = (C.c_uint64 * len(arrs))(*[len(a) for a in arrs])
    h = C.c_void_p()
    _call(A.lib().photon_plan_by_source, ptrs, lens, len(arrs), clients_per_source, seq_len,
          C.byref(h))
    return ShardPlan(h.value, seq_len)


@dataclass
class Batch:
    inputs: np.ndarray   # int32 [batch_size * seq_len]
    targets: np.ndarray  # int32, shifted by one
    batch_size: int
    seq_len: int

    def tokens(self) -> int:
        return len(self.inputs)


class BatchStream:
    """data.h:85-106: deterministic, resumable batch iterator over a client shard."""

    def __init__(self, plan: ShardPlan, client: int, batch_size: int, seq_len: int, seed: int,
                 cursor: int = 0):
        if batch_size == 0:
            raise ConfigError("stream: batch_size must be >= 1")
        if seq_len != plan.seq_len():
            raise UsageError("stream: seq_len does not match the plan's block size")
        plan.client_blocks(client)  # validates the id
        self.plan, self.client, self.batch_size, self.seq_len = plan, client, batch_size, seq_len
        self.seed = seed
        self._cursor = cursor

    def cursor(self) -> int:
        return self._cursor

    def next(self) -> Batch:
        n = self.batch_size * self.seq_len
        inp = np.zeros(n, np.int32)
        tgt = np.zeros(n, np.int32)
        cur = C.c_uint64(self._cursor)
        _call(A.lib().photon_stream_next, self.plan._h, self.client, self.batch_size, self.seed,
              C.byref(cur), inp.ctypes.data_as(C.POINTER(C.c_int32)),
              tgt.ctypes.data_as(C.POINTER(C.c_int32)))
        self._cursor = cur.value
        return Batch(inp, tgt, self.batch_size, self.seq_len)

    def take(self, steps: int) -> Tuple[np.ndarray, np.ndarray]:
        """tau consecutive batches as [tau, B*S] inputs / targets."""
        bs = [self.next() for _ in range(steps)]
        return (np.stack([b.inputs for b in bs]) if bs else np.zeros((0, 0), np.int32),
                np.stack([b.targets for b in bs]) if bs else np.zeros((0, 0), np.int32))


# ---------------------------------------------------------------------------
# device contexts
# ---------------------------------------------------------------------------

PRECISIONS = {"f32": 0, "bf16": 1}


class Context:
    """One GPU's engine (photon_ctx) for a model at a precision."""

    def __init__(self, model: ModelConfig, device: int = 0, precision: str = "f32",
                 max_batch: int = 8):
        self.model, self.device, self.precision, self.max_batch = model, device, precision, \
            max_batch
        h = C.c_void_p()
        m = model.c()
        _call(A.lib().photon_ctx_create, device, C.byref(m), PRECISIONS[precision], max_batch,
              C.byref(h))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            A.lib().photon_ctx_destroy(self._h)
            self._h = C.c_void_p()

    @property
    def handle(self):
        return self._h

    def last_ms(self) -> float:
        return float(A.lib().photon_ctx_last_ms(self._h))


_CTX: Dict[tuple, Context] = {}
_UTIL_MODEL = ModelConfig(1, 8, 2, 4, 16, 4)


def context(model: ModelConfig, device: int = 0, precision: str = "f32",
            max_batch: int = 8) -> Context:
    key = (model, device, precision, max_batch)
    if key not in _CTX:
        _CTX[key] = Context(model, device, precision, max_batch)
    return _CTX[key]


def _util_ctx(device: int = 0) -> Context:
    return context(_UTIL_MODEL, device, "f32", 1)


# ---------------------------------------------------------------------------
# model (model.h:45-72)
# ---------------------------------------------------------------------------


class TransformerModel:
    def __init__(self, cfg: ModelConfig, device: int = 0, precision: str = "f32",
                 max_batch: int = 8, micro_batch: Optional[int] = None):
        """micro_batch: activation capacity in rows -- larger batches run as
        accumulated micro-batches; None: sized for the batch (>= max_batch)."""
        cfg.validate()
        self.cfg, self.device, self.precision, self.max_batch = cfg, device, precision, max_batch
        self.micro_batch = micro_batch

    def config(self) -> ModelConfig:
        return self.cfg

    def layout(self) -> List[Tuple[str, int, Tuple[int, ...]]]:
        m = self.cfg.c()
        n = int(A.lib().photon_layout_size(C.byref(m)))
        off, r, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        name = C.create_string_buffer(64)
        out = []
        for i in range(n):
            A.lib().photon_layout_entry(C.byref(m), i, C.byref(off), C.byref(r), C.byref(c),
                                        name, 64)
            out.append((name.value.decode(), off.value,
                        (r.value, c.value) if c.value else (r.value,)))
        return out

    def init_params(self, seed: int) -> np.ndarray:
        out = np.zeros(self.cfg.param_count())
        m = self.cfg.c()
        _call(A.lib().photon_init_params, C.byref(m), seed, _dp(out))
        return out

    def _ctx(self, batch: int) -> Context:
        cap = self.micro_batch or max(self.max_batch, batch)
        return context(self.cfg, self.device, self.precision, cap)

    def forward_loss(self, params: np.ndarray, batch: Batch, build_grad: bool = True):
        """(loss, grads-or-None): forward_loss + backward + collect_grads."""
        p = _f64(params)
        if len(p) != self.cfg.param_count():
            raise ShapeError("forward: params do not match model layout")
        inp, tgt = _i32(batch.inputs), _i32(batch.targets)
        if len(inp) != batch.batch_size * batch.seq_len or len(tgt) != len(inp):
            raise ShapeError("forward: inconsistent batch")
        loss = C.c_double()
        g = np.zeros_like(p) if build_grad else None
        ctx = self._ctx(batch.batch_size)
        _call(A.lib().photon_forward_backward, ctx.handle, _dp(p),
              inp.ctypes.data_as(C.POINTER(C.c_int32)), tgt.ctypes.data_as(C.POINTER(C.c_int32)),
              batch.batch_size, batch.seq_len, C.byref(loss), _dp(g) if build_grad else None)
        return loss.value, g

    def eval_perplexity(self, params: np.ndarray, batches: Sequence[Batch]) -> float:
        if not batches:
            raise UsageError("eval_perplexity: no batches")
        p = _f64(params)
        inp = _i32(np.concatenate([b.inputs for b in batches]))
        tgt = _i32(np.concatenate([b.targets for b in batches]))
        bs = np.array([b.batch_size for b in batches], np.uint64)
        out = C.c_double()
        ctx = self._ctx(int(bs.max()))
        _call(A.lib().photon_eval_perplexity, ctx.handle, _dp(p),
              inp.ctypes.data_as(C.POINTER(C.c_int32)), tgt.ctypes.data_as(C.POINTER(C.c_int32)),
              len(batches), bs.ctypes.data_as(C.POINTER(C.c_uint64)), batches[0].seq_len,
              C.byref(out))
        return out.value


# ---------------------------------------------------------------------------
# ParamVector reductions + optimizers, f64 on the device (bit-exact)
# ---------------------------------------------------------------------------


class ParamVector:
    """Canonical-order f64 vectors; static reductions mirror param_vector.h:50-54."""

    @staticmethod
    def mean(vs: Sequence[np.ndarray], device: int = 0) -> np.ndarray:
        if len(vs) == 0:
            raise UsageError("mean of zero param vectors")
        arrs = [_f64(v) for v in vs]
        n = len(arrs[0])
        if any(len(a) != n for a in arrs):
            raise ShapeError("param vectors are not combinable (names/shapes differ)")
        ptrs = (C.POINTER(C.c_double) * len(arrs))(*[_dp(a) for a in arrs])
        out = np.zeros(n)
        _call(A.lib().photon_mean, _util_ctx(device).handle, ptrs, len(arrs), n, _dp(out))
        return out

    @staticmethod
    def sub(a: np.ndarray, b: np.ndarray, device: int = 0) -> np.ndarray:
        a, b = _f64(a), _f64(b)
        if len(a) != len(b):
            raise ShapeError("param vectors are not combinable (names/shapes differ)")
        out = np.zeros_like(a)
        _call(A.lib().photon_sub, _util_ctx(device).handle, _dp(a), _dp(b), len(a), _dp(out))
        return out

    @staticmethod
    def global_norm(x: np.ndarray) -> float:
        return float(np.sqrt(np.sum(np.square(_f64(x)))))


def compute_pseudo_gradient(theta: np.ndarray, models: Sequence[np.ndarray],
                            device: int = 0) -> np.ndarray:  # aggregator.cpp:43-48
    if len(models) == 0:
        raise UsageError("pseudo-gradient of zero client models")
    return ParamVector.sub(theta, ParamVector.mean(models, device), device)


@dataclass
class ServerOptState:
    cfg: ServerOptConfig
    velocity: np.ndarray

    @staticmethod
    def init(cfg: ServerOptConfig, like: np.ndarray) -> "ServerOptState":
        cfg.validate()
        return ServerOptState(cfg, np.zeros(len(like)))


def server_step(state: ServerOptState, theta: np.ndarray, delta: np.ndarray,
                client_mean: np.ndarray, device: int = 0) -> np.ndarray:
    """optim.cpp:124-159; state.velocity is updated in place."""
    theta, delta, client_mean = _f64(theta), _f64(delta), _f64(client_mean)
    if not (len(theta) == len(delta) == len(client_mean) == len(state.velocity)):
        raise ShapeError("param vectors are not combinable (names/shapes differ)")
    out = np.zeros_like(theta)
    s = state.cfg.c()
    vel = state.velocity
    if not vel.flags.c_contiguous or vel.dtype != np.float64:
        state.velocity = vel = _f64(vel).copy()
    _call(A.lib().photon_server_step, _util_ctx(device).handle, C.byref(s), _dp(theta),
          _dp(delta), _dp(client_mean), _dp(vel), len(theta), _dp(out))
    return out


def aggregate(models: Sequence[np.ndarray], theta: np.ndarray, state: ServerOptState,
              device: int = 0) -> np.ndarray:
    """Fused mean -> pseudo-gradient -> outer step (aggregator.cpp:177-179)."""
    arrs = [_f64(v) for v in models]
    if not arrs:
        raise UsageError("mean of zero param vectors")
    theta = _f64(theta)
    ptrs = (C.POINTER(C.c_double) * len(arrs))(*[_dp(a) for a in arrs])
    out = np.zeros_like(theta)
    s = state.cfg.c()
    _call(A.lib().photon_aggregate, _util_ctx(device).handle, ptrs, len(arrs), len(theta),
          _dp(theta), _dp(state.velocity), C.byref(s), _dp(out))
    return out


@dataclass
class AdamWState:
    cfg: AdamWConfig
    m: np.ndarray
    v: np.ndarray
    step_count: int = 0

    @staticmethod
    def fresh(cfg: AdamWConfig, like: np.ndarray) -> "AdamWState":
        return AdamWState(cfg, np.zeros(len(like)), np.zeros(len(like)), 0)


def adamw_step(params: np.ndarray, grads: np.ndarray, state: AdamWState, lr: float,
               device: int = 0) -> None:
    """optim.cpp:61-90, in place on params / state (f64, bit-exact)."""
    g = _f64(grads)
    if len(params) != len(g):
        raise ShapeError("param vectors are not combinable (names/shapes differ)")
    sc = C.c_uint64(state.step_count)
    a = state.cfg.c()
    _call(A.lib().photon_adamw_step, _util_ctx(device).handle, _dp(params), _dp(g),
          _dp(state.m), _dp(state.v), len(params), C.byref(sc), C.byref(a), lr)
    state.step_count = sc.value


def sgd_step(params: np.ndarray, grads: np.ndarray, lr: float, clip_norm: float = 0.0,
             device: int = 0) -> None:
    g = _f64(grads)
    _call(A.lib().photon_sgd_step, _util_ctx(device).handle, _dp(params), _dp(g), len(params),
          lr, clip_norm)


# ---------------------------------------------------------------------------
# client update (client.h:97-99)
# ---------------------------------------------------------------------------


def run_local_round(theta_t: np.ndarray, stream: BatchStream, cfg: LocalTrainConfig,
                    round: int, client_id: int, step_base: int, device: int = 0,  # noqa: A002
                    precision: str = "f32", micro_batch: Optional[int] = None) -> ClientResult:
    theta = _f64(theta_t)
    if len(theta) != cfg.model.param_count():
        raise ShapeError("forward: params do not match model layout")
    tau = cfg.local_steps
    start = stream.cursor()
    inp, tgt = stream.take(tau)
    out = np.zeros_like(theta)
    metrics = (A.photon_step_metric * max(tau, 1))()
    ctx = context(cfg.model, device, precision, micro_batch or cfg.batch_size)
    t = cfg.c()
    try:
        _call(A.lib().photon_client_round, ctx.handle, C.byref(t), _dp(theta),
              _i32(inp).ctypes.data_as(C.POINTER(C.c_int32)),
              _i32(tgt).ctypes.data_as(C.POINTER(C.c_int32)), round, client_id, step_base,
              _dp(out), metrics)
    except Exception:
        stream._cursor = start + tau * cfg.batch_size
        raise
    steps = [StepMetric(metrics[i].loss, int(metrics[i].tokens), metrics[i].sim_seconds)
             for i in range(tau)]
    return ClientResult(out, steps, stream.cursor())


# ---------------------------------------------------------------------------
# federated runner (aggregator.h:70-102)
# ---------------------------------------------------------------------------


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _call(A.lib().photon_nccl_unique_id, buf)
    return bytes(buf)


class FederationRunner:
    """Device-resident outer loop.  With world > 1 (one process per GPU), each
    rank trains the sampled slots with slot % world == rank and the round
    boundary is a sharded NCCL exchange; results do not depend on world."""

    def __init__(self, fed: FederationConfig, local: LocalTrainConfig, server: ServerOptConfig,
                 plan: ShardPlan, theta0: np.ndarray, device: int = 0, precision: str = "f32",
                 rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 dropouts: Sequence[Tuple[int, int]] = (), eval_set: "Optional[EvalSet]" = None,
                 eval_every: int = 0, micro_batch: Optional[int] = None):
        """micro_batch: activation capacity in rows; a local batch (or eval
        batch) above it runs as accumulated micro-batches of that many rows
        (same loss and gradient as the whole batch).  None: the whole batch."""
        self.fed, self.local, self.server, self.plan = fed, local, server, plan
        if micro_batch:
            max_batch = micro_batch
        else:  # the context's activations hold the whole batch and the largest eval batch
            max_batch = max([local.batch_size] + ([eval_set.max_batch()] if eval_set else []))
        self.ctx = context(local.model, device, precision, max_batch)
        theta0 = _f64(theta0)
        self._P = len(theta0)
        h = C.c_void_p()
        f, t, s = fed.c(), local.c(), server.c()
        idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id else None
        _call(A.lib().photon_runner_create, self.ctx.handle, C.byref(f), C.byref(t), C.byref(s),
              plan._h, _dp(theta0), rank, world, idbuf, C.byref(h))
        self._h = h
        for r, c in dropouts:
            A.lib().photon_runner_add_dropout(h, r, c)
        self._eval_set = eval_set  # keeps the host set alive alongside the runner
        if eval_set is not None:
            _call(A.lib().photon_runner_set_eval, h, eval_set._h, eval_every)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            A.lib().photon_runner_destroy(self._h)
            self._h = C.c_void_p()

    def run_round(self) -> RoundRecord:
        rec = A.photon_round_record()
        _call(A.lib().photon_runner_run_round, self._h, C.byref(rec))
        k = int(rec.n_sampled)
        return RoundRecord(int(rec.round), [int(x) for x in rec.sampled_ids[:min(k, 64)]],
                           rec.mean_client_loss, rec.min_client_loss, rec.max_client_loss,
                           rec.local_ms, rec.aggregate_ms, rec.round_ms, int(rec.tokens),
                           rec.host_ms, int(rec.h2d_bytes), int(rec.d2h_bytes), rec.eval_ppl,
                           rec.boundary_ms)

    def done(self) -> bool:
        return self.next_round() >= self.fed.rounds

    def next_round(self) -> int:
        return int(A.lib().photon_runner_next_round(self._h))

    def theta(self) -> np.ndarray:
        out = np.zeros(self._P)
        _call(A.lib().photon_runner_theta, self._h, _dp(out))
        return out

    def velocity(self) -> np.ndarray:
        out = np.zeros(self._P)
        _call(A.lib().photon_runner_velocity, self._h, _dp(out))
        return out

    def client_cursor(self, client: int) -> int:
        if client >= self.fed.population:
            raise LookupError("unknown client id")
        return int(A.lib().photon_runner_cursor(self._h, client))

    def restore(self, theta: np.ndarray, velocity: np.ndarray, next_round: int,
                cursors: Sequence[int]) -> None:
        cur = np.ascontiguousarray(cursors, np.uint64)
        _call(A.lib().photon_runner_restore, self._h, _dp(_f64(theta)), _dp(_f64(velocity)),
              next_round, cur.ctypes.data_as(C.POINTER(C.c_uint64)), len(cur))

    def evaluate(self) -> float:
        """eval_fn(theta) (harness.cpp:797-799) on the runner's eval set."""
        ppl = C.c_double()
        _call(A.lib().photon_runner_eval, self._h, C.byref(ppl))
        return ppl.value

    def save(self, directory: str) -> None:
        """checkpoint.phck + velocity.phck + state.json (harness.cpp:802-905)."""
        _call(A.lib().photon_runner_save, self._h, os.fsencode(directory))

    def resume(self, directory: str) -> None:
        _call(A.lib().photon_runner_resume, self._h, os.fsencode(directory))


@dataclass
class CentralizedResult:
    """baselines.h:37-42."""
    theta: np.ndarray
    steps: List[StepMetric]
    sync_events: int
    cursors: List[int]


class CentralizedTrainer:
    """Device-resident run_centralized (baselines.cpp:25-127): worker w on rank
    w % world, one ascending-order gradient all-reduce and one shared update per
    step; results do not depend on world."""

    def __init__(self, cfg: CentralizedConfig, plan: ShardPlan, seed: int, theta0: np.ndarray,
                 device: int = 0, precision: str = "f32", rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None, micro_batch: Optional[int] = None):
        self.cfg, self.plan = cfg, plan
        per_worker = cfg.global_batch // max(cfg.n_workers, 1)
        self.ctx = context(cfg.model, device, precision, micro_batch or max(per_worker, 1))
        theta0 = _f64(theta0)
        self._P = len(theta0)
        h = C.c_void_p()
        c = cfg.c()
        idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id else None
        _call(A.lib().photon_central_create, self.ctx.handle, C.byref(c), plan._h, seed,
              _dp(theta0), rank, world, idbuf, C.byref(h))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            A.lib().photon_central_destroy(self._h)
            self._h = C.c_void_p()

    def step(self) -> StepMetric:
        m = A.photon_step_metric()
        _call(A.lib().photon_central_step, self._h, C.byref(m))
        return StepMetric(m.loss, int(m.tokens), m.sim_seconds)

    def next_step(self) -> int:
        return int(A.lib().photon_central_next_step(self._h))

    def cursor(self, worker: int) -> int:
        return int(A.lib().photon_central_cursor(self._h, worker))

    def theta(self) -> np.ndarray:
        out = np.zeros(self._P)
        _call(A.lib().photon_central_theta, self._h, _dp(out))
        return out


def run_centralized(cfg: CentralizedConfig, plan: ShardPlan, seed: int, theta0: np.ndarray,
                    n_threads: int = 1, observer=None, **kw) -> CentralizedResult:
    """baselines.h:47-51 (n_threads is accepted for signature parity)."""
    tr = CentralizedTrainer(cfg, plan, seed, theta0, **kw)
    steps = []
    for t in range(cfg.total_steps):
        steps.append(tr.step())
        if observer is not None:
            observer(t, tr.theta())
    return CentralizedResult(tr.theta(), steps, cfg.total_steps if cfg.n_workers > 1 else 0,
                             [tr.cursor(w) for w in range(cfg.n_workers)])


class EvalSet:
    """build_eval_batches (harness.cpp:440-472): held-out batches from
    mix_seed(data_seed, "Eval"); host memory, uploaded once by the runner."""

    def __init__(self, styles: Sequence[str], eval_sequences: int, data_seed: int,
                 model: ModelConfig, eval_batch: int):
        arr = (C.c_char_p * len(styles))(*[s.encode() for s in styles])
        h = C.c_void_p()
        _call(A.lib().photon_eval_set_create, arr, len(styles), eval_sequences, data_seed,
              model.vocab_size, model.seq_len, eval_batch, C.byref(h))
        self._h, self.seq_len = h, model.seq_len

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            A.lib().photon_eval_set_destroy(self._h)
            self._h = C.c_void_p()

    def __len__(self) -> int:
        return int(A.lib().photon_eval_set_batches(self._h))

    def max_batch(self) -> int:
        return max((b.batch_size for b in self.batches()), default=0)

    def batches(self) -> List["Batch"]:
        out = []
        for i in range(len(self)):
            pi, pt, b = C.POINTER(C.c_int32)(), C.POINTER(C.c_int32)(), C.c_uint64()
            _call(A.lib().photon_eval_set_batch, self._h, i, C.byref(pi), C.byref(pt), C.byref(b))
            n = int(b.value) * self.seq_len
            out.append(Batch(np.ctypeslib.as_array(pi, (n,)).copy(),
                             np.ctypeslib.as_array(pt, (n,)).copy(), int(b.value), self.seq_len))
        return out


def crc64(data: bytes) -> int:
    """CRC-64/XZ (checkpoint.h:14-16)."""
    buf = C.create_string_buffer(bytes(data), len(data))
    return int(A.lib().photon_crc64(buf, len(data)))


def write_checkpoint(path: str, model: ModelConfig, params: np.ndarray, round: int) -> None:  # noqa: A002
    """PHCK writer (checkpoint.h:27-41), byte-identical to the reference's."""
    m = model.c()
    _call(A.lib().photon_checkpoint_write, os.fsencode(path), C.byref(m), _dp(_f64(params)), round)


def read_checkpoint(path: str, model: ModelConfig) -> Tuple[np.ndarray, int]:
    """PHCK reader (checkpoint.h:42): (params, round); IntegrityError / ShapeError."""
    m = model.c()
    out = np.zeros(model.param_count())
    rd = C.c_uint64()
    _call(A.lib().photon_checkpoint_read, os.fsencode(path), C.byref(m), _dp(out), C.byref(rd))
    return out, int(rd.value)
