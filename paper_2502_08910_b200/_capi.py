"""ctypes binding of the C ABI declared in include/hipprune_b200.h.

This module only loads ``_lib/libhipprune_b200.so`` (built for sm_100a by
``paper_2502_08910_b200.build``) and mirrors its structs. There is no fallback:
if the library or a CUDA device is missing, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "_lib" / ("libhipprune_b200_trace.so" if os.environ.get("HP_TRACE") in ("1", "cuts")
                           else "libhipprune_b200.so")
if os.environ.get("HP_LIB"):  # dev: an alternative build of the kernel library (A/B timing)
    LIB_PATH = Path(os.environ["HP_LIB"])

HP_OK = 0
HP_F32, HP_BF16 = 0, 1
HP_ROPE_CHUNK_INDEXED, HP_ROPE_RELATIVE, HP_ROPE_STREAMING = 0, 1, 2
STAGE_VARIANTS = {0: "classic", 1: "lookahead", 2: "wide", 3: "allrows"}  # hp_stage_variant
PRUNE_VARIANTS = {0: "cuda_core", 1: "tensor_core"}  # hp_prune_variant
BSA_VARIANTS = {0: "ticket", 1: "cluster"}  # hp_bsa_variant


class ContractViolation(RuntimeError):
    """hipprune::ContractViolation (reference errors.hpp:8-10)."""


class LogicError(RuntimeError):
    """std::logic_error."""


class PartialCommitError(RuntimeError):
    """hipprune::PartialCommitError (reference kv_store.hpp:41-45)."""


_EXC = {1: ContractViolation, 2: ValueError, 3: IndexError, 4: LogicError, 5: RuntimeError,
        6: PartialCommitError}


class KvView(C.Structure):
    _fields_ = [("k_pool", C.c_void_p), ("v_pool", C.c_void_p), ("k_host", C.c_void_p),
                ("v_host", C.c_void_p), ("page_table", C.c_void_p), ("touched", C.c_void_p),
                ("num_pages", C.c_int32), ("page_size", C.c_int32), ("n_kv", C.c_int32),
                ("d", C.c_int32), ("dtype", C.c_int32), ("t_kv", C.c_int32),
                ("row_bits", C.c_void_p), ("row_bits_stride", C.c_int64)]


class RopeCtx(C.Structure):
    _fields_ = [("cos_tab", C.c_void_p), ("sin_tab", C.c_void_p), ("rope_max", C.c_int64),
                ("extension", C.c_int32), ("early_cutoff", C.c_int32),
                ("early_policy", C.c_int32), ("late_policy", C.c_int32), ("layer", C.c_int32),
                ("pad_", C.c_int32)]


class StageArgs(C.Structure):
    _fields_ = [("query_block", C.c_int32), ("chunk_size", C.c_int32), ("keep", C.c_int32),
                ("n_masks", C.c_int32), ("heads_per_mask", C.c_int32), ("n_q_heads", C.c_int32),
                ("n_blocks", C.c_int32), ("q_rows", C.c_int32), ("q", C.c_void_p),
                ("query_offset", C.c_int64), ("stream_tokens", C.c_int32),
                ("max_chunks", C.c_int32), ("in_list", C.c_void_p), ("in_start", C.c_void_p),
                ("in_count", C.c_void_p), ("in_stride", C.c_int64), ("out_list", C.c_void_p),
                ("out_count", C.c_void_p), ("out_stride", C.c_int64), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("keys", KvView), ("rope", RopeCtx),
                ("keys_exact", C.c_void_p), ("path_out", C.c_void_p), ("descend_always", C.c_int32),
                ("pad2_", C.c_int32)]


class BsaArgs(C.Structure):
    _fields_ = [("n_q_heads", C.c_int32), ("heads_per_mask", C.c_int32), ("n_rows", C.c_int32),
                ("q", C.c_void_p), ("query_offset", C.c_int64), ("sel_list", C.c_void_p),
                ("sel_count", C.c_void_p), ("sel_stride", C.c_int64), ("max_sel", C.c_int32),
                ("out", C.c_void_p), ("part_m", C.c_void_p), ("part_l", C.c_void_p),
                ("part_o", C.c_void_p), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("kv", KvView), ("rope", RopeCtx)]


class ListRef(C.Structure):
    _fields_ = [("depth", C.c_int32), ("pad_", C.c_int32), ("sel", C.c_void_p * 4),
                ("sel_stride", C.c_int32 * 4), ("lc", C.c_int32 * 4), ("base_list", C.c_void_p),
                ("base_stride", C.c_int64), ("range_start", C.c_int64)]


class DecodeStageArgs(C.Structure):
    _fields_ = [("chunk_size", C.c_int32), ("keep", C.c_int32), ("n_masks", C.c_int32),
                ("heads_per_mask", C.c_int32), ("n_q_heads", C.c_int32),
                ("stream_tokens", C.c_int32), ("q", C.c_void_p), ("query_position", C.c_int64),
                ("in_", ListRef), ("in_count", C.c_void_p), ("in_count_const", C.c_int64),
                ("max_chunks", C.c_int32), ("sel_stride", C.c_int32), ("sel_out", C.c_void_p),
                ("out_count", C.c_void_p), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("keys", KvView), ("rope", RopeCtx),
                ("keys_exact", C.c_void_p), ("list_out", C.c_void_p),
                ("list_out_stride", C.c_int64), ("scores_out", C.c_void_p)]


class DecodeBsaArgs(C.Structure):
    _fields_ = [("n_q_heads", C.c_int32), ("heads_per_mask", C.c_int32),
                ("sink_tokens", C.c_int32), ("stream_tokens", C.c_int32), ("q", C.c_void_p),
                ("query_position", C.c_int64), ("mask", ListRef), ("mask_count", C.c_void_p),
                ("max_mask", C.c_int32), ("out", C.c_void_p), ("part_m", C.c_void_p),
                ("part_l", C.c_void_p), ("part_o", C.c_void_p), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("kv", KvView), ("rope", RopeCtx),
                ("mask_stable", C.c_int32)]


class DecodeLayerArgs(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("chunk_size", C.c_int32 * 4), ("keep", C.c_int32 * 4),
                ("refresh", C.c_int32 * 4), ("n_masks", C.c_int32), ("heads_per_mask", C.c_int32),
                ("n_q_heads", C.c_int32), ("sink_tokens", C.c_int32), ("stream_tokens", C.c_int32),
                ("pad_", C.c_int32), ("q", C.c_void_p), ("query_position", C.c_int64),
                ("sel", C.c_void_p * 4), ("sel_stride", C.c_int32 * 4), ("count", C.c_void_p * 4),
                ("cache", C.c_void_p * 4), ("cache_stride", C.c_int64 * 4), ("out", C.c_void_p),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t), ("kv", KvView),
                ("keys_exact", C.c_void_p)]


class BsaPrefillArgs(C.Structure):
    _fields_ = [("n_q_heads", C.c_int32), ("heads_per_mask", C.c_int32), ("n_rows", C.c_int32),
                ("block_size", C.c_int32), ("q", C.c_void_p), ("query_offset", C.c_int64),
                ("mask_list", C.c_void_p), ("mask_count", C.c_void_p), ("mask_stride", C.c_int64),
                ("n_mask_blocks", C.c_int32), ("max_mask", C.c_int32), ("sink_tokens", C.c_int32),
                ("stream_tokens", C.c_int32), ("out", C.c_void_p), ("kv", KvView)]


class PageCache(C.Structure):
    _fields_ = [("k_slots", C.c_void_p), ("v_slots", C.c_void_p), ("k_host", C.c_void_p),
                ("v_host", C.c_void_p), ("page_table", C.c_void_p), ("slot_page", C.c_void_p),
                ("slot_stamp", C.c_void_p), ("touched", C.c_void_p), ("num_pages", C.c_int32),
                ("num_slots", C.c_int32), ("page_size", C.c_int32), ("n_kv", C.c_int32),
                ("d", C.c_int32), ("dtype", C.c_int32)]


_lib = None

# every symbol include/hipprune_b200.h declares
EXPORTS = ["hp_last_error", "hp_version", "hp_device_available", "hp_build_rope_table",
           "hp_stage_workspace_bytes", "hp_prune_stage", "hp_prune_stage_variant", "hp_remap_blocks",
           "hp_selected_indices", "hp_bsa_workspace_bytes", "hp_bsa", "hp_lse_merge",
           "hp_decode_stage_workspace_bytes", "hp_decode_stage", "hp_decode_bsa_workspace_bytes",
           "hp_decode_bsa", "hp_decode_stage_variant", "hp_decode_bsa_variant",
           "hp_decode_layer_workspace_bytes", "hp_decode_layer_supported", "hp_decode_layer", "hp_decode_materialize", "hp_decode_append",
           "hp_cache_workspace_bytes", "hp_cache_commit", "hp_select_topk", "hp_select_topk_sharded",
           "hp_bsa_prefill_smem_bytes", "hp_bsa_prefill"]


def lib():
    """Load the CUDA C-ABI library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"hipprune_b200 CUDA library not built: {LIB_PATH} "
                           "(run python -c 'import __graft_entry__ as g; g.build()')")
    L = C.CDLL(str(LIB_PATH))
    L.hp_last_error.restype = C.c_char_p
    L.hp_version.restype = C.c_int
    L.hp_device_available.restype = C.c_int
    L.hp_build_rope_table.restype = C.c_int
    L.hp_build_rope_table.argtypes = [C.c_int64, C.c_int32, C.c_float, C.c_void_p, C.c_void_p]
    L.hp_stage_workspace_bytes.restype = C.c_size_t
    L.hp_stage_workspace_bytes.argtypes = [C.c_int32] * 4
    L.hp_prune_stage.restype = C.c_int
    L.hp_prune_stage.argtypes = [C.POINTER(StageArgs), C.c_void_p]
    L.hp_prune_stage_variant.restype = C.c_int
    L.hp_prune_stage_variant.argtypes = [C.POINTER(StageArgs), C.POINTER(C.c_int32)]
    L.hp_remap_blocks.restype = C.c_int
    L.hp_remap_blocks.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                  C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                                  C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    L.hp_selected_indices.restype = C.c_int
    L.hp_selected_indices.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_void_p,
                                      C.c_void_p, C.c_int64, C.c_void_p]
    L.hp_bsa_workspace_bytes.restype = C.c_size_t
    L.hp_bsa_workspace_bytes.argtypes = [C.c_int32] * 4
    L.hp_bsa.restype = C.c_int
    L.hp_bsa.argtypes = [C.POINTER(BsaArgs), C.c_void_p]
    L.hp_decode_stage_workspace_bytes.restype = C.c_size_t
    L.hp_decode_stage_workspace_bytes.argtypes = [C.c_int32, C.c_int32]
    L.hp_decode_stage.restype = C.c_int
    L.hp_decode_stage.argtypes = [C.POINTER(DecodeStageArgs), C.c_void_p]
    L.hp_decode_bsa_workspace_bytes.restype = C.c_size_t
    L.hp_decode_bsa_workspace_bytes.argtypes = [C.c_int32, C.c_int32]
    L.hp_decode_bsa.restype = C.c_int
    L.hp_decode_bsa.argtypes = [C.POINTER(DecodeBsaArgs), C.c_void_p]
    L.hp_decode_stage_variant.restype = C.c_int
    L.hp_decode_stage_variant.argtypes = [C.POINTER(DecodeStageArgs), C.POINTER(C.c_int32)]
    L.hp_decode_bsa_variant.restype = C.c_int
    L.hp_decode_bsa_variant.argtypes = [C.POINTER(DecodeBsaArgs), C.POINTER(C.c_int32)]
    L.hp_decode_layer_workspace_bytes.restype = C.c_size_t
    L.hp_decode_layer_workspace_bytes.argtypes = [C.c_int32, C.c_int32]
    L.hp_decode_layer_supported.restype = C.c_int
    L.hp_decode_layer_supported.argtypes = [C.POINTER(DecodeLayerArgs)]
    L.hp_decode_layer.restype = C.c_int
    L.hp_decode_layer.argtypes = [C.POINTER(DecodeLayerArgs), C.c_void_p]
    L.hp_decode_materialize.restype = C.c_int
    L.hp_decode_materialize.argtypes = [C.POINTER(ListRef), C.POINTER(C.c_void_p),
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.c_int32,
                                        C.c_int32, C.c_int32, C.c_void_p]
    L.hp_decode_append.restype = C.c_int
    L.hp_decode_append.argtypes = [C.POINTER(KvView), C.c_void_p, C.c_void_p, C.c_int64,
                                   C.c_void_p, C.c_void_p]
    L.hp_bsa_prefill_smem_bytes.restype = C.c_size_t
    L.hp_bsa_prefill_smem_bytes.argtypes = [C.c_int32]
    L.hp_bsa_prefill.restype = C.c_int
    L.hp_bsa_prefill.argtypes = [C.POINTER(BsaPrefillArgs), C.c_void_p]
    L.hp_select_topk.restype = C.c_int
    L.hp_select_topk.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64, C.c_int32,
                                 C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
    L.hp_select_topk_sharded.restype = C.c_int
    L.hp_select_topk_sharded.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                         C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.hp_cache_workspace_bytes.restype = C.c_size_t
    L.hp_cache_workspace_bytes.argtypes = [C.c_int32, C.c_int32]
    L.hp_cache_commit.restype = C.c_int
    L.hp_cache_commit.argtypes = [C.POINTER(PageCache), C.c_uint32, C.c_void_p, C.c_void_p,
                                  C.c_size_t, C.c_void_p]
    L.hp_lse_merge.restype = C.c_int
    L.hp_lse_merge.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                               C.c_int32, C.c_void_p, C.c_void_p]
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != HP_OK:
        msg = lib().hp_last_error().decode(errors="replace")
        raise _EXC.get(rc, RuntimeError)(msg)


def exported_symbols() -> list[str]:
    L = lib()
    return [s for s in EXPORTS if hasattr(L, s)]
