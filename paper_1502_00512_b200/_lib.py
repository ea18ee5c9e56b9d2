"""ctypes binding of libdesklm_cuda.so (include/desklm_cuda.h).

The library is built in-tree (``make -C paper_1502_00512_b200``).  There is no
fallback: if the .so is missing or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdesklm_cuda.so")
# tuning experiments (scripts/build_variant.sh) may point at another build
LIB_PATH = os.environ.get("DL_LIB_PATH", LIB_PATH)

# Every symbol include/desklm_cuda.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "dl_last_error", "dl_version", "dl_create", "dl_destroy", "dl_set_params",
    "dl_get_params", "dl_set_opt", "dl_get_opt", "dl_window", "dl_get_grads", "dl_set_grads",
    "dl_rmsprop", "dl_train_window", "dl_score", "dl_sharded_perplexity", "dl_rnn_perplexity",
    "dl_trainer_init", "dl_trainer_run", "dl_trainer_get_state",
    "dl_trainer_set_state", "dl_comm_unique_id", "dl_comm_init",
    "dl_launch_count", "dl_set_profiling", "dl_kernel_ms", "dl_test_gemm", "dl_cuda_stream",
    "dl_test_embed", "dl_rank_cursors", "dl_init_uniform", "dl_local_group_create",
    "dl_local_group_destroy", "dl_comm_init_local", "dl_set_vocab_shard",
    "dl_ln_z_samples", "dl_score_candidates", "dl_set_loss_mode", "dl_set_noise", "dl_set_noise_dist", "dl_set_rng_state", "dl_get_rng_state",
    "dl_rng_seed_state", "dl_bn_create", "dl_bn_destroy", "dl_bn_last_error",
    "dl_bn_set_params", "dl_bn_get_params", "dl_bn_set_opt", "dl_bn_get_opt", "dl_bn_window",
    "dl_bn_get_grads", "dl_bn_rmsprop", "dl_bn_train_window", "dl_bn_sharded_perplexity",
    "dl_bn_launch_count", "dl_bn_cuda_stream", "dl_bn_set_loss_mode", "dl_bn_set_noise",
    "dl_bn_set_rng_state", "dl_bn_get_rng_state", "dl_bn_set_params_quantized", "dl_bn_score",
    "dl_bn_set_noise_dist", "dl_bn_trainer_init", "dl_bn_trainer_run",
    "dl_bn_trainer_get_state", "dl_bn_trainer_set_state",
)

DL_OK, DL_EINVAL, DL_EDATA, DL_EDEVICE = 0, 1, 2, 3
DL_FP32, DL_BF16, DL_TF32X3 = 0, 1, 2

_lib = None


class DataError(RuntimeError):
    """Mirrors desklm::DataError (util.hpp:34-37)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL failure inside libdesklm_cuda."""


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `make -C {_HERE}` (or __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    vp, i64, u64 = C.c_void_p, C.c_int64, C.c_uint64
    P = C.POINTER
    sig = {
        "dl_last_error": (C.c_char_p, [vp]),
        "dl_version": (C.c_char_p, []),
        "dl_create": (C.c_int, [P(vp), C.c_int, i64, i64, C.c_int, C.c_int]),
        "dl_destroy": (C.c_int, [vp]),
        "dl_set_params": (C.c_int, [vp, vp, vp, vp]),
        "dl_get_params": (C.c_int, [vp, vp, vp, vp]),
        "dl_set_opt": (C.c_int, [vp, vp, vp, vp, C.c_double, C.c_double]),
        "dl_get_opt": (C.c_int, [vp, vp, vp, vp]),
        "dl_window": (C.c_int, [vp, i64, i64, vp, vp, vp, vp, vp, C.c_double, C.c_float,
                                C.c_int, P(C.c_double), P(C.c_uint64)]),
        "dl_get_grads": (C.c_int, [vp, vp, vp, vp]),
        "dl_set_grads": (C.c_int, [vp, i64, vp, vp, vp, vp]),
        "dl_rmsprop": (C.c_int, [vp, C.c_double, P(C.c_int)]),
        "dl_train_window": (C.c_int, [vp, i64, i64, vp, vp, vp, vp, vp, C.c_double, C.c_float,
                                      C.c_double, P(C.c_double), P(C.c_uint64), P(C.c_int)]),
        "dl_score": (C.c_int, [vp, i64, i64, vp, vp, vp, vp, vp, P(C.c_double),
                               P(C.c_uint64)]),
        "dl_sharded_perplexity": (C.c_int, [vp, vp, i64, C.c_int, C.c_uint32,
                                            P(C.c_double), P(C.c_uint64), P(C.c_double)]),
        "dl_rnn_perplexity": (C.c_int, [vp, vp, i64, C.c_uint32, P(C.c_double),
                                        P(C.c_uint64), P(C.c_double)]),
        "dl_ln_z_samples": (C.c_int, [vp, vp, i64, i64, vp, P(C.c_int64)]),
        "dl_score_candidates": (C.c_int, [vp, vp, i64, i64, vp, vp]),
        "dl_trainer_init": (C.c_int, [vp, vp, i64, C.c_int, C.c_int, C.c_int, C.c_double,
                                      C.c_uint32]),
        "dl_trainer_run": (C.c_int, [vp, i64, i64, C.c_double, P(C.c_double),
                                     P(C.c_uint64)]),
        "dl_trainer_get_state": (C.c_int, [vp, vp, vp]),
        "dl_trainer_set_state": (C.c_int, [vp, vp, vp]),
        "dl_comm_unique_id": (C.c_int, [vp]),
        "dl_comm_init": (C.c_int, [vp, vp, C.c_int, C.c_int]),
        "dl_test_gemm": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp,
                                   vp, C.c_int, vp]),
        "dl_test_embed": (C.c_int, [vp, C.c_int, i64, i64, vp, vp, C.c_float, vp]),
        "dl_rank_cursors": (C.c_int, [i64, C.c_int, C.c_int, C.c_int, C.c_int, vp]),
        "dl_init_uniform": (C.c_int, [i64, i64, u64, C.c_double, vp, vp, vp]),
        "dl_local_group_create": (C.c_int, [C.c_int, P(vp)]),
        "dl_local_group_destroy": (C.c_int, [vp]),
        "dl_comm_init_local": (C.c_int, [vp, vp, C.c_int]),
        "dl_set_vocab_shard": (C.c_int, [vp, C.c_int]),
        "dl_set_loss_mode": (C.c_int, [vp, C.c_int]),
        "dl_set_noise": (C.c_int, [vp, vp, i64, C.c_int, C.c_double]),
        "dl_set_noise_dist": (C.c_int, [vp, vp, i64, C.c_int]),
        "dl_set_rng_state": (C.c_int, [vp, vp]),
        "dl_get_rng_state": (C.c_int, [vp, vp]),
        "dl_rng_seed_state": (C.c_int, [u64, vp]),
        "dl_bn_create": (C.c_int, [P(vp), C.c_int, i64, i64, i64, C.c_int, C.c_int]),
        "dl_bn_destroy": (C.c_int, [vp]),
        "dl_bn_last_error": (C.c_char_p, [vp]),
        "dl_bn_set_params": (C.c_int, [vp, vp, vp, vp, vp]),
        "dl_bn_get_params": (C.c_int, [vp, vp, vp, vp, vp]),
        "dl_bn_set_opt": (C.c_int, [vp, vp, vp, vp, vp, C.c_double, C.c_double]),
        "dl_bn_get_opt": (C.c_int, [vp, vp, vp, vp, vp]),
        "dl_bn_window": (C.c_int, [vp, i64, i64, vp, vp, vp, vp, vp, C.c_double, C.c_float,
                                   C.c_int, P(C.c_double), P(C.c_uint64)]),
        "dl_bn_get_grads": (C.c_int, [vp, vp, vp, vp, vp]),
        "dl_bn_rmsprop": (C.c_int, [vp, C.c_double, P(C.c_int)]),
        "dl_bn_train_window": (C.c_int, [vp, i64, i64, vp, vp, vp, vp, vp, C.c_double,
                                         C.c_float, C.c_double, P(C.c_double), P(C.c_uint64),
                                         P(C.c_int)]),
        "dl_bn_sharded_perplexity": (C.c_int, [vp, vp, i64, C.c_int, C.c_uint32,
                                               P(C.c_double), P(C.c_uint64), P(C.c_double)]),
        "dl_bn_set_loss_mode": (C.c_int, [vp, C.c_int]),
        "dl_bn_set_params_quantized": (C.c_int, [vp, vp]),
        "dl_bn_set_noise": (C.c_int, [vp, vp, i64, C.c_int, C.c_double]),
        "dl_bn_set_noise_dist": (C.c_int, [vp, vp, i64, C.c_int]),
        "dl_bn_score": (C.c_int, [vp, i64, i64, vp, vp, vp, vp, vp, P(C.c_double), P(u64)]),
        "dl_bn_trainer_init": (C.c_int, [vp, vp, i64, C.c_int, C.c_int, C.c_int, C.c_double,
                                         C.c_uint32]),
        "dl_bn_trainer_run": (C.c_int, [vp, i64, i64, C.c_double, P(C.c_double), P(u64),
                                        P(u64)]),
        "dl_bn_trainer_get_state": (C.c_int, [vp, vp, vp]),
        "dl_bn_trainer_set_state": (C.c_int, [vp, vp, vp]),
        "dl_bn_set_rng_state": (C.c_int, [vp, vp]),
        "dl_bn_get_rng_state": (C.c_int, [vp, vp]),
        "dl_bn_launch_count": (u64, [vp]),
        "dl_bn_cuda_stream": (vp, [vp]),
        "dl_launch_count": (u64, [vp]),
        "dl_cuda_stream": (vp, [vp]),
        "dl_set_profiling": (C.c_int, [vp, C.c_int]),
        "dl_kernel_ms": (C.c_double, [vp, C.c_char_p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(rc: int, ctx=None):
    if rc == DL_OK:
        return
    lib = load()
    msg = (lib.dl_last_error(ctx) or b"").decode()
    if rc == DL_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == DL_EDATA:
        raise DataError(msg)
    raise DeviceError(msg)
