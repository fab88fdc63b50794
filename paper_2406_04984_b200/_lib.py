"""ctypes binding of the C ABI in include/meft_cuda.h (libmeft_cuda.so, built in-tree).

Loading fails loudly when the library is missing: there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MEFT_LIB: an alternative build of the same library (developer A/B variants, e.g. tools/ab_variants.sh)
LIB_PATH = os.environ.get("MEFT_LIB") or os.path.join(HERE, "libmeft_cuda.so")

P = C.c_void_p
I64 = C.c_int64
I32P = C.POINTER(C.c_int32)
D = C.c_double
INT = C.c_int

class BaseFfn(C.Structure):
    """meft_base_ffn (include/meft_cuda.h): frozen base FFN, bf16 device w_in [d x n], w_out [n x d]."""
    _fields_ = [("w_in", P), ("w_out", P), ("n", I64), ("act", INT)]


class PeerOut(C.Structure):
    """meft_peer_out (include/meft_cuda.h)."""
    _fields_ = [("world", INT), ("rank", INT), ("rows", I64), ("out_recv", P * 8), ("grad_h_recv", P * 8)]


class CkptHeader(C.Structure):
    _fields_ = [("layers", I64), ("dim", I64), ("pairs", I64), ("experts", I64), ("step", I64),
                ("train_router", INT)]


# meft_host_comm (include/meft_cuda.h): host-exchange communicator callbacks
HC_ALL_GATHER = C.CFUNCTYPE(INT, P, P, C.c_size_t, P)
HC_ALL_TO_ALL_V = C.CFUNCTYPE(INT, P, P, C.POINTER(C.c_size_t), P, C.POINTER(C.c_size_t))


class HostComm(C.Structure):
    _fields_ = [("user", P), ("all_gather", HC_ALL_GATHER), ("all_to_all_v", HC_ALL_TO_ALL_V)]


# meft_ckpt_source / meft_ckpt_sink (include/meft_cuda.h)
CKPT_SOURCE = C.CFUNCTYPE(INT, P, I64, INT, P, I64)
CKPT_SINK = C.CFUNCTYPE(INT, P, C.POINTER(CkptHeader), I64, INT, P, I64)

# name -> (restype, argtypes)
_SIGS = {
    "meft_version": (C.c_char_p, []),
    "meft_ctx_create": (INT, [INT, P, C.POINTER(P)]),
    "meft_ctx_destroy": (None, [P]),
    "meft_ctx_stream": (P, [P]),
    "meft_last_error": (C.c_char_p, [P]),
    "meft_last_error_index": (I64, [P]),
    "meft_synchronize": (INT, [P]),
    "meft_kernel_launches": (I64, []),
    "meft_route_select": (INT, [P, P, P, I64, I64, I64, I64, P]),
    "meft_row_stats": (INT, [P, P, I64, I64, P, P]),
    "meft_store_key_stats": (INT, [P, P, I64, P, P]),
    "meft_score_candidates": (INT, [P, P, I64, P, P, I64, P]),
    "meft_exact_scores": (INT, [P, P, I64, P, I64, P, P, I64, P]),
    "meft_topk_classify": (INT, [P, P, P, I64, I64, I64, I64, I64, P, P, P, P, P, P]),
    "meft_topk_finalize": (INT, [P, P, P, P, P, P, I64, I64, I64, P, P]),
    "meft_layer_ffn_local": (INT, [P, P, I64, P, P, I64, P, I64, D, D, D, D, P, P, P, P, P, P]),
    "meft_peer_reduce": (INT, [P, P, INT, I64, I64, P]),
    "meft_ipc_handle": (INT, [P, P, P]),
    "meft_ipc_open": (INT, [P, P, C.POINTER(P)]),
    "meft_ipc_close": (INT, [P, P]),
    "meft_ctx_set_timing": (INT, [P, INT]),
    "meft_ctx_set_selection": (INT, [P, INT]),
    "meft_ctx_set_gather": (INT, [P, INT]),
    "meft_ctx_set_adam": (INT, [P, INT]),
    "meft_ctx_set_check_finite": (INT, [P, INT]),
    "meft_ctx_set_host_sync": (INT, [P, INT]),
    "meft_graph_begin": (INT, [P]),
    "meft_graph_end": (INT, [P, C.POINTER(P)]),
    "meft_graph_launch": (INT, [P, P]),
    "meft_graph_destroy": (None, [P]),
    "meft_set_gemm_sm_reserve": (INT, [INT]),
    "meft_ctx_read_timing": (INT, [P, P, P]),
    "meft_device_alloc": (INT, [P, C.c_size_t, C.POINTER(P)]),
    "meft_device_free": (INT, [P, P]),
    "meft_host_alloc": (INT, [P, C.c_size_t, C.POINTER(P)]),
    "meft_host_free": (INT, [P, P]),
    "meft_copy_to_device": (INT, [P, P, P, C.c_size_t]),
    "meft_copy_to_host": (INT, [P, P, P, C.c_size_t]),
    "meft_memset": (INT, [P, P, INT, C.c_size_t]),
    "meft_convert": (INT, [P, P, INT, P, INT, I64]),
    "meft_selection_shape": (INT, [I64, I64, I64, I64, C.POINTER(I64), C.POINTER(I64), C.POINTER(INT)]),
    "meft_route_scores": (INT, [P, INT, P, P, I64, I64, I64, P]),
    "meft_select_experts": (INT, [P, P, I64, I64, I64, P]),
    "meft_ke_select": (INT, [P, INT, P, P, P, I64, I64, I64, I64, I64, I64, P, P, P, P]),
    "meft_topk_select": (INT, [P, INT, P, P, I64, I64, I64, I64, P, P, P]),
    "meft_gather_adapter": (INT, [P, INT, P, P, I64, I64, P, I64, P, P]),
    "meft_ffn_forward": (INT, [P, INT, P, P, P, I64, I64, I64, I64, P, P, INT]),
    "meft_ffn_backward": (INT, [P, INT, P, P, P, P, P, I64, I64, I64, I64, P, P, P, P, INT]),
    "meft_base_ffn_forward": (INT, [P, P, P, P, I64, I64, I64, INT, P, P]),
    "meft_base_ffn_backward": (INT, [P, P, P, P, P, I64, I64, I64, INT, P]),
    "meft_matmul_f64": (INT, [P, P, P, I64, I64, I64, P]),
    # expert-sharded selection bookkeeping (csrc/shard_plan.cu)
    "meft_shard_dispatch": (INT, [P, P, I64, I64, I64, INT, P, I64, P, P, P, P, C.POINTER(I64)]),
    "meft_shard_unpermute_rows": (INT, [P, P, P, I64, I64, P]),
    "meft_shard_requests": (INT, [P, P, P, P, P, I64, I64, I64, I64, I64, INT, C.POINTER(I64), P, P, P,
                                  C.POINTER(I64), C.POINTER(I64)]),
    "meft_shard_scatter_f64": (INT, [P, P, P, I64, P]),
    "meft_gather_rows": (INT, [P, P, I64, P, I64, P]),
    # toy trunk (model.cpp:50-218), fp64 device buffers
    "meft_embed_f64": (INT, [P, P, I64, P, I64, I64, P, I64, I64, P]),
    "meft_attention_forward_f64": (INT, [P, P, P, P, P, P, P, I64, I64, I64, P, P, P, P, P]),
    "meft_attention_backward_f64": (INT, [P, P, P, P, P, P, I64, I64, I64, P, P, P, P, P, P]),
    "meft_lm_loss_f64": (INT, [P, P, I64, I64, P, I64, P, P, D, C.POINTER(D), P]),
    "meft_argmax_logits_f64": (INT, [P, P, I64, I64, P, C.POINTER(I64)]),
    "meft_transpose_f64": (INT, [P, P, P, I64, I64]),
    "meft_activation_f64": (INT, [P, INT, P, P, I64]),
    "meft_adam_rows_f64": (INT, [P, P, P, P, P, P, P, P, I64, I64, D, D, D, D]),
    "meft_rows_add": (INT, [P, INT, P, I64, P, I64, P, P]),
    "meft_store_create": (INT, [P, I64, I64, I64, I64, INT, C.POINTER(P)]),
    "meft_store_enable_router": (INT, [P, P]),
    "meft_store_expert_histogram": (INT, [P, P, I64, P, INT]),
    "meft_store_train_router": (INT, [P, C.POINTER(INT)]),
    "meft_store_save": (INT, [P, P, C.c_char_p, I64, C.c_char_p]),
    "meft_store_load": (INT, [P, C.c_char_p, INT, C.POINTER(P), C.POINTER(CkptHeader), C.c_char_p, C.c_size_t]),
    "meft_ckpt_save": (INT, [C.c_char_p, C.POINTER(CkptHeader), C.c_char_p, CKPT_SOURCE, P]),
    "meft_ckpt_load": (INT, [C.c_char_p, C.POINTER(CkptHeader), C.c_char_p, C.c_size_t, CKPT_SINK, P]),
    "meft_store_destroy": (None, [P]),
    "meft_store_info": (INT, [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64), C.POINTER(I64), C.POINTER(INT)]),
    "meft_store_init_reference": (INT, [P, P, C.c_uint64]),
    "meft_reference_uniform": (INT, [C.c_uint64, C.c_uint64, I64, D, D, INT, P]),
    "meft_store_upload_host": (INT, [P, P, I64, INT, P, I64, I64]),
    "meft_store_download_host": (INT, [P, P, I64, INT, P, I64, I64]),
    "meft_store_tensor": (INT, [P, I64, INT, C.POINTER(P), C.POINTER(INT), C.POINTER(I64), C.POINTER(I64)]),
    "meft_fetch": (INT, [P, P, I64, P, I64, P, P]),
    "meft_scatter_grads": (INT, [P, P, I64, P, I64, P, P, INT]),
    "meft_sparse_adam_update": (INT, [P, P, I64, D, D, D, D]),
    "meft_layer_step": (INT, [P, P, I64, P, P, I64, I64, I64, D, D, D, D, P, P, P, P, P]),
    "meft_layer_step_base": (INT, [P, P, I64, P, P, I64, I64, I64, D, D, D, D, P, P, P, P, P, P]),
    "meft_layer_step_host": (INT, [P, P, I64, P, P, I64, I64, I64, D, D, D, D, P, P, P]),
    # the expert-sharded step behind the C ABI (csrc/sharded_step.cu)
    "meft_nccl_unique_id": (INT, [P]),
    "meft_ctx_comm_init": (INT, [P, P, INT, INT]),
    "meft_ctx_set_comm": (INT, [P, P, INT, INT]),
    "meft_ctx_set_host_comm": (INT, [P, C.POINTER(HostComm), INT, INT]),
    "meft_ctx_clear_comm": (INT, [P]),
    "meft_layer_step_sharded": (INT, [P, P, I64, P, P, P, I64, I64, I64, D, D, D, D, P, P, P, P]),
    "meft_ctx_sharded_paths": (INT, [P, P, P]),
}

F64, F32, BF16 = 0, 1, 2
STORE_F64, STORE_MIXED, STORE_COMPACT = 0, 1, 2

TENSORS = {"w_a": 0, "w_b": 1, "w_g": 2, "m_a": 3, "v_a": 4, "m_b": 5, "v_b": 6, "stage_a": 7, "stage_b": 8,
           "pair_step": 9, "staged": 10, "w_a_compute": 11, "w_b_compute": 12, "w_g_compute": 13, "m_g": 14,
           "v_g": 15, "router_step": 16}
TENSOR_NAMES = {v: k for k, v in TENSORS.items()}



class StepInfo(C.Structure):
    _fields_ = [("union_size", I64), ("take", I64), ("kk_eff", I64), ("warned", INT), ("gpu_launches", INT),
                ("rescored", INT), ("fallbacks", INT), ("meter_h2d", I64), ("meter_d2h", I64),
                ("meter_hidden", I64), ("beta_paper", D), ("dedup_ratio", D), ("activated_fraction", D),
                ("router_flops", I64), ("expert_scoring_flops", I64)]


class MeftError(RuntimeError):
    """Error raised from a meft_status != MEFT_OK; `kind` mirrors the reference exception type."""

    KINDS = {1: "ShapeError", 2: "invalid_argument", 3: "out_of_range", 4: "logic_error", 5: "non-finite",
             6: "cuda", 7: "nccl", 8: "oom", 9: "CheckpointHeaderError", 10: "CheckpointShapeError",
             11: "CheckpointTruncatedError", 12: "io"}

    def __init__(self, code: int, msg: str, index: int = -1):
        super().__init__(f"{self.KINDS.get(code, code)}: {msg}")
        self.code = code
        self.kind = self.KINDS.get(code, str(code))
        self.index = index


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("MEFT_LIB") and not hasattr(L, name):
                continue  # an older A/B build (MEFT_LIB) may predate some entry points
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(status: int, ctx=None):
    if status != 0:
        L = lib()
        raise MeftError(status, L.meft_last_error(ctx).decode(errors="replace"), int(L.meft_last_error_index(ctx)))
