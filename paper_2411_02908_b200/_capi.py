"""ctypes declarations of include/photon.h (the C ABI of libphoton.so).

Loading fails loudly: there is no CPU fallback for any entry point.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PHOTON_LIB") or os.path.join(_HERE, "libphoton.so")

u64, i32, dbl, u8 = C.c_uint64, C.c_int32, C.c_double, C.c_uint8
P = C.POINTER


class photon_err(C.Structure):
    _fields_ = [("code", i32), ("round", u64), ("client", u64), ("step", u64),
                ("msg", C.c_char * 256)]


class photon_model_cfg(C.Structure):
    _fields_ = [(n, u64) for n in
                ("n_blocks", "d_model", "n_heads", "expansion_ratio", "vocab_size", "seq_len")]


class photon_lr_schedule(C.Structure):
    _fields_ = [("eta_max", dbl), ("warmup_steps", u64), ("decay_steps", u64), ("alpha", dbl)]


class photon_adamw_cfg(C.Structure):
    _fields_ = [("beta1", dbl), ("beta2", dbl), ("eps", dbl), ("weight_decay", dbl),
                ("clip_norm", dbl)]


class photon_train_cfg(C.Structure):
    _fields_ = [("model", photon_model_cfg), ("adamw", photon_adamw_cfg),
                ("schedule", photon_lr_schedule), ("opt", i32), ("sgd_clip_norm", dbl),
                ("local_steps", u64), ("batch_size", u64), ("throughput_bps", dbl),
                ("post_kind", i32), ("post_threshold", dbl)]


class photon_server_cfg(C.Structure):
    _fields_ = [("kind", i32), ("eta", dbl), ("momentum", dbl), ("nesterov", i32)]


class photon_fed_cfg(C.Structure):
    _fields_ = [("population", u64), ("clients_per_round", u64), ("rounds", u64),
                ("topology", i32), ("seed", u64)]


class photon_step_metric(C.Structure):
    _fields_ = [("loss", dbl), ("tokens", u64), ("sim_seconds", dbl)]


class photon_central_cfg(C.Structure):
    _fields_ = [("model", photon_model_cfg), ("adamw", photon_adamw_cfg),
                ("schedule", photon_lr_schedule), ("opt", i32), ("sgd_clip_norm", dbl),
                ("n_workers", u64), ("global_batch", u64), ("total_steps", u64),
                ("opt_reset_interval", u64), ("throughput_bps", dbl)]


class photon_round_record(C.Structure):
    _fields_ = [("round", u64), ("n_sampled", u64), ("sampled_ids", u64 * 64),
                ("mean_client_loss", dbl), ("min_client_loss", dbl), ("max_client_loss", dbl),
                ("local_ms", dbl), ("aggregate_ms", dbl), ("round_ms", dbl), ("tokens", u64),
                ("host_ms", dbl), ("h2d_bytes", u64), ("d2h_bytes", u64), ("eval_ppl", dbl),
                ("boundary_ms", dbl)]


_SIGS = {
    "photon_abi_version": (i32, []),
    "photon_status_name": (C.c_char_p, [i32]),
    "photon_mix64": (u64, [u64]),
    "photon_stream_seed": (u64, [u64, u64]),
    "photon_sample_clients": (i32, [u64, u64, u64, u64, P(u64), P(photon_err)]),
    "photon_lr_at": (i32, [P(photon_lr_schedule), u64, P(dbl), P(photon_err)]),
    "photon_param_count": (u64, [P(photon_model_cfg)]),
    "photon_layout_size": (u64, [P(photon_model_cfg)]),
    "photon_layout_entry": (i32, [P(photon_model_cfg), u64, P(u64), P(u64), P(u64), C.c_char_p,
                                  C.c_int]),
    "photon_init_params": (i32, [P(photon_model_cfg), u64, P(dbl), P(photon_err)]),
    "photon_generate_corpus": (i32, [C.c_char_p, u64, u64, C.c_uint32, P(C.c_uint16),
                                     P(photon_err)]),
    "photon_plan_iid": (i32, [P(C.c_uint16), u64, u64, u64, u64, P(C.c_void_p), P(photon_err)]),
    "photon_plan_by_source": (i32, [P(P(C.c_uint16)), P(u64), u64, u64, u64, P(C.c_void_p),
                                    P(photon_err)]),
    "photon_plan_free": (None, [C.c_void_p]),
    "photon_plan_n_clients": (u64, [C.c_void_p]),
    "photon_plan_client_blocks": (u64, [C.c_void_p, u64]),
    "photon_stream_next": (i32, [C.c_void_p, u64, u64, u64, P(u64), P(i32), P(i32),
                                 P(photon_err)]),
    "photon_ctx_create": (i32, [C.c_int, P(photon_model_cfg), C.c_int, u64, P(C.c_void_p),
                                P(photon_err)]),
    "photon_ctx_destroy": (None, [C.c_void_p]),
    "photon_ctx_last_ms": (dbl, [C.c_void_p]),
    "photon_forward_backward": (i32, [C.c_void_p, P(dbl), P(i32), P(i32), u64, u64, P(dbl),
                                      P(dbl), P(photon_err)]),
    "photon_eval_perplexity": (i32, [C.c_void_p, P(dbl), P(i32), P(i32), u64, P(u64), u64,
                                     P(dbl), P(photon_err)]),
    "photon_client_round": (i32, [C.c_void_p, P(photon_train_cfg), P(dbl), P(i32), P(i32), u64,
                                  u64, u64, P(dbl), P(photon_step_metric), P(photon_err)]),
    "photon_mean": (i32, [C.c_void_p, P(P(dbl)), u64, u64, P(dbl), P(photon_err)]),
    "photon_sub": (i32, [C.c_void_p, P(dbl), P(dbl), u64, P(dbl), P(photon_err)]),
    "photon_server_step": (i32, [C.c_void_p, P(photon_server_cfg), P(dbl), P(dbl), P(dbl),
                                 P(dbl), u64, P(dbl), P(photon_err)]),
    "photon_aggregate": (i32, [C.c_void_p, P(P(dbl)), u64, u64, P(dbl), P(dbl),
                               P(photon_server_cfg), P(dbl), P(photon_err)]),
    "photon_adamw_step": (i32, [C.c_void_p, P(dbl), P(dbl), P(dbl), P(dbl), u64, P(u64),
                                P(photon_adamw_cfg), dbl, P(photon_err)]),
    "photon_sgd_step": (i32, [C.c_void_p, P(dbl), P(dbl), u64, dbl, dbl, P(photon_err)]),
    "photon_aggregate_device_f32": (i32, [C.c_void_p, P(C.c_void_p), u64, u64, C.c_void_p,
                                          C.c_void_p, P(photon_server_cfg), P(dbl),
                                          P(photon_err)]),
    "photon_plan_from_blocks": (i32, [P(C.c_void_p), P(u64), u64, u64, P(u64), u64,
                                      P(C.c_uint32), P(u64), P(C.c_void_p), P(photon_err)]),
    "photon_shard_len": (u64, [u64, C.c_int]),
    "photon_slot_owner": (C.c_int, [u64, C.c_int]),
    "photon_boundary_peer": (C.c_int, [u64, u64, u64, C.c_int]),
    "photon_debug_gemm": (i32, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int64,
                                C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p,
                                C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_int, P(dbl), P(photon_err)]),
    "photon_debug_colsum": (i32, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, P(dbl),
                                  P(photon_err)]),
    "photon_debug_ce": (i32, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_float,
                              C.c_void_p, C.c_int, C.c_void_p, P(dbl), P(photon_err)]),
    "photon_debug_layernorm": (i32, [C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 13 +
                               [P(dbl), P(photon_err)]),
    "photon_debug_attention": (i32, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     P(dbl), P(photon_err)]),
    "photon_ctx_set_timing": (i32, [C.c_void_p, C.c_int]),
    "photon_ctx_kernel_times": (i32, [C.c_void_p, P(dbl)]),
    "photon_launch_count": (C.c_uint64, []),
    "photon_nccl_unique_id": (i32, [P(u8), P(photon_err)]),
    "photon_runner_create": (i32, [C.c_void_p, P(photon_fed_cfg), P(photon_train_cfg),
                                   P(photon_server_cfg), C.c_void_p, P(dbl), C.c_int, C.c_int,
                                   P(u8), P(C.c_void_p), P(photon_err)]),
    "photon_runner_destroy": (None, [C.c_void_p]),
    "photon_runner_add_dropout": (i32, [C.c_void_p, u64, u64]),
    "photon_runner_run_round": (i32, [C.c_void_p, P(photon_round_record), P(photon_err)]),
    "photon_runner_next_round": (u64, [C.c_void_p]),
    "photon_runner_theta": (i32, [C.c_void_p, P(dbl), P(photon_err)]),
    "photon_runner_velocity": (i32, [C.c_void_p, P(dbl), P(photon_err)]),
    "photon_runner_cursor": (u64, [C.c_void_p, u64]),
    "photon_runner_restore": (i32, [C.c_void_p, P(dbl), P(dbl), u64, P(u64), u64,
                                    P(photon_err)]),
    "photon_debug_boundary": (i32, [C.c_int, u64, C.c_int, C.c_int, P(u8), P(photon_server_cfg),
                                    C.c_int, P(dbl), P(photon_err)]),
    "photon_central_create": (i32, [C.c_void_p, P(photon_central_cfg), C.c_void_p, u64, P(dbl),
                                    C.c_int, C.c_int, P(u8), P(C.c_void_p), P(photon_err)]),
    "photon_central_destroy": (None, [C.c_void_p]),
    "photon_central_step": (i32, [C.c_void_p, P(photon_step_metric), P(photon_err)]),
    "photon_central_next_step": (u64, [C.c_void_p]),
    "photon_central_cursor": (u64, [C.c_void_p, u64]),
    "photon_central_theta": (i32, [C.c_void_p, P(dbl), P(photon_err)]),
    "photon_eval_set_create": (i32, [P(C.c_char_p), u64, u64, u64, u64, u64, u64,
                                     P(C.c_void_p), P(photon_err)]),
    "photon_eval_set_destroy": (None, [C.c_void_p]),
    "photon_eval_set_batches": (u64, [C.c_void_p]),
    "photon_eval_set_batch": (i32, [C.c_void_p, u64, P(P(i32)), P(P(i32)), P(u64),
                                    P(photon_err)]),
    "photon_runner_set_eval": (i32, [C.c_void_p, C.c_void_p, u64, P(photon_err)]),
    "photon_runner_eval": (i32, [C.c_void_p, P(dbl), P(photon_err)]),
    "photon_crc64": (u64, [C.c_void_p, u64]),
    "photon_checkpoint_write": (i32, [C.c_char_p, P(photon_model_cfg), P(dbl), u64,
                                      P(photon_err)]),
    "photon_checkpoint_read": (i32, [C.c_char_p, P(photon_model_cfg), P(dbl), P(u64),
                                     P(photon_err)]),
    "photon_runner_save": (i32, [C.c_void_p, C.c_char_p, P(photon_err)]),
    "photon_runner_resume": (i32, [C.c_void_p, C.c_char_p, P(photon_err)]),
}

EXPORTED = sorted(_SIGS)

_lib = None


def lib():
    """The loaded libphoton.so.  Raises if it was never built: no fallback."""
    global _lib
    if _lib is None:
        # NCCL is bound at runtime (nccl_api.hpp): point it at torch's bundled
        # copy so a later `import torch` finds the same libnccl.so.2 loaded.
        if "PHOTON_NCCL_LIB" not in os.environ:
            import glob
            import sysconfig

            for sp in {sysconfig.get_paths()["purelib"], sysconfig.get_paths()["platlib"]}:
                hits = glob.glob(os.path.join(sp, "nvidia", "nccl", "lib", "libnccl.so.2"))
                if hits:
                    os.environ["PHOTON_NCCL_LIB"] = hits[0]
                    break
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -m paper_2411_02908_b200.build` "
                "(the CUDA extension is required; there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.photon_abi_version() != 2:
            raise ImportError("libphoton.so ABI version mismatch")
        _lib = L
    return _lib
