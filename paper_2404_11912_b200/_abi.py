"""ctypes binding of the C ABI in `include/hs_abi.h` (libhs_b200.so).

This is the drop-in boundary: every compute call of the package goes through
these entry points.  There is no CPU fallback -- importing the package on a
machine without the built library raises, and calling into it without a CUDA
device raises.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import CapacityError, ContractError, FiniteError, ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhs_b200.so")

HS_OK = 0
HS_ERR_SHAPE = -1
HS_ERR_CONTRACT = -2
HS_ERR_CAPACITY = -3
HS_ERR_FINITE = -4
HS_ERR_VALUE = -5
HS_ERR_CUDA = -10

HS_KV_LINEAR = 0
HS_KV_SLOTTED = 1
HS_APPEND_POS = 0
HS_APPEND_LINEAR = 1
HS_APPEND_RING = 2

vp = C.c_void_p
i32 = C.c_int
i64 = C.c_longlong
f32 = C.c_float
f64 = C.c_double
sz = C.c_size_t


class HsModel(C.Structure):
    _fields_ = [("n_layers", i32), ("n_heads", i32), ("n_kv_heads", i32), ("head_dim", i32),
                ("d_ff", i32), ("vocab_size", i32), ("max_seq", i32), ("d_model", i32),
                ("ld_d", i32), ("ld_ff", i32), ("norm_eps", f32),
                ("emb", vp), ("head", vp), ("final_norm", vp), ("attn_norm", vp), ("mlp_norm", vp),
                ("wqkv", vp), ("wo", vp), ("wgu", vp), ("wdown", vp), ("rope_cos", vp), ("rope_sin", vp),
                ("blocked", i32)]


class HsCache(C.Structure):
    _fields_ = [("kind", i32), ("n_layers", i32), ("n_kv_heads", i32), ("head_dim", i32), ("cap", i32),
                ("k", vp), ("v", vp), ("pos", vp)]


class HsStep(C.Structure):
    _fields_ = [("pos0", i32), ("append_mode", i32), ("append_base", i32), ("n_sink", i32), ("ring", i32),
                ("n_view", i32), ("window", i32), ("win_lo", i32), ("split", i32), ("pos_base", i32),
                ("own_hi", i32), ("dyn", vp)]


class HsShard(C.Structure):
    _fields_ = [("comm", vp), ("rank", i32), ("world", i32)]


_P = C.POINTER
_SIGS = {
    "hs_last_error": (C.c_char_p, []),
    "hs_abi_version": (i32, []),
    "hs_device_sm_count": (i32, [i32]),
    "hs_launch_count": (C.c_ulonglong, []),
    "hs_note_launches": (None, [C.c_ulonglong]),
    "hs_stream_sync": (i32, [vp]),
    "hs_forward_workspace_bytes": (sz, [_P(HsModel), i32, i32, i32, i32]),
    "hs_forward_workspace_clean_bytes": (sz, [_P(HsModel)]),
    "hs_gemv_tc_workspace_bytes": (sz, [i32, i32]),
    "hs_gemv_tc": (i32, [vp, i32, vp, i32, i32, i32, vp, i32, vp, i32, vp, sz, vp]),
    "hs_split_rows": (i32, [vp, i32, i32, i32, i32, vp, f32, vp, vp]),
    "hs_forward": (i32, [_P(HsModel), _P(HsCache), _P(HsStep), _P(HsShard), vp, i32, vp, vp, vp, sz, vp]),
    "hs_forward_tp_workspace_bytes": (sz, [_P(HsModel), i32, i32, i32, i32, i32]),
    "hs_forward_tp": (i32, [_P(HsModel), _P(HsCache), _P(HsStep), _P(HsShard), _P(HsShard), vp, i32, vp, vp, vp, sz,
                            vp]),
    "hs_forward_attn_probs": (i32, [_P(HsModel), _P(HsCache), _P(HsStep), vp, i32, vp, vp, vp, vp, vp, sz, vp]),
    "hs_forward_probe": (i32, [_P(HsModel), _P(HsCache), _P(HsStep), vp, i32, vp, vp, vp, vp, sz, vp]),
    "hs_forward_topk_workspace_bytes": (sz, [_P(HsModel), i32, i32]),
    "hs_forward_topk": (i32, [_P(HsModel), _P(HsCache), _P(HsStep), i32, vp, vp, vp, vp, sz, vp]),
    "hs_prefill_workspace_bytes": (sz, [_P(HsModel), i32, i32, i32]),
    "hs_prefill": (i32, [_P(HsModel), _P(HsCache), _P(HsStep), vp, i32, vp, vp, vp, sz, vp]),
    "hs_prefill_sharded_workspace_bytes": (sz, [_P(HsModel), i32, i32, i32, i32]),
    "hs_prefill_sharded": (i32, [_P(HsModel), _P(HsCache), _P(HsStep), _P(HsShard), vp, i32, vp, vp, vp, sz, vp]),
    "hs_embed": (i32, [vp, i32, i32, vp, i32, vp, vp]),
    "hs_rope_append": (i32, [_P(HsModel), _P(HsCache), _P(HsStep), i32, vp, i32, vp, vp, vp]),
    "hs_kv_write": (i32, [_P(HsCache), i32, vp, vp, i32, vp, vp, vp]),
    "hs_attention_workspace_bytes": (sz, [i32, i32, i32, i32, i32]),
    "hs_attention": (i32, [_P(HsCache), i32, _P(HsStep), i32, vp, i32, vp, vp, sz, vp]),
    "hs_attention_partial": (i32, [_P(HsCache), i32, _P(HsStep), i32, vp, i32, vp, vp, sz, vp]),
    "hs_prefill_attention": (i32, [_P(HsCache), i32, _P(HsStep), i32, vp, i32, vp, vp, vp]),
    "hs_chunk_score": (i32, [vp, i32, i64, i64, i64, i32, i32, i32, i32, i32, vp, i32, vp, vp]),
    "hs_chunk_select_workspace_bytes": (sz, [i32, i32]),
    "hs_chunk_select": (i32, [vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, sz, vp]),
    "hs_retrieval_gather": (i32, [_P(HsCache), _P(HsCache), vp, i32, i32, i32, i32, i32, i32, vp]),
    "hs_retrieval_commit": (i32, [_P(HsCache), vp, i32, i32, i32, i32, i32, vp]),
    "hs_cache_copy": (i32, [_P(HsCache), _P(HsCache), i32, vp]),
    "hs_probs": (i32, [vp, i32, i32, f64, vp, vp]),
    "hs_sample": (i32, [vp, i32, vp, vp, vp, vp]),
    "hs_draft_sample": (i32, [vp, i32, f64, vp, vp, vp, vp, vp]),
    "hs_draft_step": (i32, [vp, i32, f64, vp, vp, vp, vp, vp, i32, i32, vp, i32, vp]),
    "hs_graph_step": (i32, [vp, i32, i32, i32, vp, vp, i32, vp]),
    "hs_upload_i32": (i32, [vp, vp, i32, vp]),
    "hs_weights_block": (i32, [vp, vp, i32, i32, i32, vp]),
    "hs_verify_chain": (i32, [vp, i32, vp, vp, i32, vp, vp, vp, vp]),
    "hs_verify_token": (i32, [i32, vp, vp, vp, vp, vp, vp]),
    "hs_correct_token": (i32, [vp, vp, i32, vp, vp, vp, vp]),
    "hs_shard_merge": (i32, [vp, i32, i32, i32, vp, vp]),
    "hs_profile_attention": (i32, [i32, i32]),
    "hs_profile_attention_read": (i32, [_P(f64), _P(i64), _P(i32)]),
    "hs_comm_id_bytes": (sz, []),
    "hs_comm_unique_id": (i32, [vp]),
    "hs_comm_init": (i32, [_P(vp), vp, i32, i32]),
    "hs_comm_destroy": (i32, [vp]),
    "hs_all_gather": (i32, [vp, vp, vp, sz, vp]),
    "hs_all_reduce_sum": (i32, [vp, vp, sz, i32, vp]),
    "hs_all_gather_v": (i32, [vp, i32, i32, vp, vp, vp, vp]),
    "hs_comm_check": (i32, [vp]),
    "hs_comm_abort": (i32, [vp]),
    "hs_gemm3_tc": (i32, [vp, vp, vp, i32, i32, vp, i32, i32, vp, i32, i32, vp]),
    "hs_loopback_create": (i32, [i32, vp]),
    "hs_loopback_destroy": (i32, [vp]),
    "hs_retrieval_exchange_workspace_bytes": (sz, [_P(HsCache)]),
    "hs_retrieval_exchange": (i32, [_P(HsShard), _P(HsCache), vp, vp, sz, vp]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a library with "
            "`python -m paper_2404_11912_b200.build` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.hs_abi_version() != 2:
        raise ImportError("libhs_b200.so ABI version mismatch")
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc == HS_OK:
        return
    msg = lib.hs_last_error().decode(errors="replace")
    if rc == HS_ERR_SHAPE:
        raise ShapeError(msg)
    if rc == HS_ERR_CONTRACT:
        raise ContractError(msg)
    if rc == HS_ERR_CAPACITY:
        raise CapacityError(msg)
    if rc == HS_ERR_FINITE:
        raise FiniteError(msg)
    if rc == HS_ERR_VALUE:
        raise ValueError(msg)
    raise RuntimeError(f"libhs_b200 error {rc}: {msg}")


def status_error(code: int, what: str):
    """Exception for a status reported by a kernel through device memory."""
    if code == HS_ERR_CONTRACT:
        return ContractError(what)
    return RuntimeError(f"{what} (status {code})")
