"""ctypes mirror of include/fsvd_b200.h (the C-ABI boundary).

The product library is ``paper_2508_01506_b200/lib/libfsvd_b200.so`` (built in
tree by ``__graft_entry__.build()``).  Loading fails loudly when it is
missing: there is no Python or CPU fallback for any compute entry point.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FSVD_LIB") or os.path.join(_HERE, "lib", "libfsvd_b200.so")

# fsvd_status (errors.hpp:11-21 ErrorKind, offset by one) -----------------
OK, ERR_SHAPE, ERR_RANK, ERR_CONFIG, ERR_BUDGET, ERR_ACCOUNTING = 0, 1, 2, 3, 4, 5
ERR_FORMAT, ERR_NUMERIC, ERR_INFEASIBLE, ERR_IO, ERR_CUDA = 6, 7, 8, 9, 10
STATUS_NAMES = {
    0: "OK", 1: "ShapeError", 2: "RankError", 3: "ConfigError", 4: "BudgetError",
    5: "AccountingError", 6: "FormatError", 7: "NumericError", 8: "InfeasibleError",
    9: "IoError", 10: "CudaError",
}

F32, BF16 = 0, 1
ACT_GELU_ERF, ACT_GELU_TANH, ACT_RELU, ACT_IDENTITY = 0, 1, 2, 3
MODE_DENSE, MODE_NAIVE_LOWRANK, MODE_FLASH_V1, MODE_FLASH_V2 = 0, 1, 2, 3
MODE_NAMES = {"dense": 0, "naive_lowrank": 1, "flash_v1": 2, "flash_v2": 3}
KERNEL_ATTENTION, KERNEL_FFN_V1, KERNEL_FFN_V2 = 0, 1, 2
(FORMULA_DENSE_ATTN, FORMULA_FLASH_ATTN_DENSE_QKV, FORMULA_FLASH_SVD_ATTN,
 FORMULA_GROUPED_ATTN, FORMULA_FFN_DENSE, FORMULA_FFN_NAIVE_LOWRANK, FORMULA_FFN_V1,
 FORMULA_FFN_V2) = range(8)
TRANSIENT, PERSISTENT, EXCLUDED = 0, 1, 2

_fp = C.POINTER(C.c_float)
_sz = C.c_size_t


class TilePlan(C.Structure):
    _fields_ = [("bm", _sz), ("br", _sz), ("bdf", _sz), ("sram_budget_bytes", _sz)]

    @classmethod
    def default(cls):  # memtier.hpp:152-157
        return cls(16, 16, 64, 131072)


class Geometry(C.Structure):
    _fields_ = [("batch", _sz), ("seq_len", _sz), ("d_model", _sz), ("d_ff", _sz),
                ("heads", _sz), ("groups", _sz), ("rank", _sz), ("layers", _sz)]


class LinearDesc(C.Structure):
    _fields_ = [("in_dim", _sz), ("rank", _sz), ("out_dim", _sz),
                ("u", _fp), ("v", _fp), ("bias", _fp)]


class FactorJob(C.Structure):
    _fields_ = [("a", _fp), ("m", _sz), ("n", _sz), ("rank", _sz), ("u", _fp), ("v", _fp)]


class DenseLayer(C.Structure):
    _fields_ = [("d_model", _sz), ("d_ff", _sz)] + [
        (n, _fp) for n in ("wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo", "w_in", "b_in",
                           "w_out", "b_out")]


class FactorBuffers(C.Structure):
    _fields_ = [(n, _fp) for n in ("attn_u", "attn_v", "attn_b", "out_u", "out_v", "out_b",
                                   "up_u", "up_v", "up_b", "down_u", "down_v", "down_b")]


class AttnDesc(C.Structure):
    _fields_ = [("d_model", _sz), ("groups", _sz), ("rank", _sz),
                ("u", _fp), ("v", _fp), ("bias", _fp)]


class FfnDesc(C.Structure):
    _fields_ = [("up", LinearDesc), ("down", LinearDesc), ("activation", C.c_int)]


class LayerDesc(C.Structure):
    _fields_ = [("heads", _sz), ("attn", AttnDesc), ("out_proj", LinearDesc), ("ffn", FfnDesc),
                ("ln1_gamma", _fp), ("ln1_beta", _fp), ("ln1_eps", C.c_float),
                ("ln2_gamma", _fp), ("ln2_beta", _fp), ("ln2_eps", C.c_float),
                ("dense", C.POINTER(DenseLayer))]


def fptr(arr):
    """float* of a C-contiguous float32 numpy array (caller keeps it alive)."""
    import numpy as np
    assert arr.dtype == np.float32 and arr.flags["C_CONTIGUOUS"], "need contiguous float32"
    return arr.ctypes.data_as(_fp)


class FsvdError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.kind = STATUS_NAMES.get(status, str(status))


_lib = None


def _declare(lib):
    vp, st = C.c_void_p, C.c_int
    P = C.POINTER
    sigs = {
        "fsvd_abi_version": (C.c_int, []),
        "fsvd_last_error": (C.c_char_p, []),
        "fsvd_device_available": (C.c_int, []),
        "fsvd_meter_create": (st, [P(vp)]),
        "fsvd_meter_destroy": (None, [vp]),
        "fsvd_meter_alloc": (st, [vp, C.c_char_p, C.c_int, _sz, P(C.c_uint64)]),
        "fsvd_meter_free": (st, [vp, C.c_uint64]),
        "fsvd_meter_pin": (st, [vp, C.c_char_p, _sz]),
        "fsvd_meter_region_begin": (st, [vp, C.c_char_p, P(_sz)]),
        "fsvd_meter_region_end": (st, [vp, C.c_char_p, _sz]),
        "fsvd_meter_current_transient": (_sz, [vp]),
        "fsvd_meter_peak_transient": (_sz, [vp]),
        "fsvd_meter_persistent": (_sz, [vp]),
        "fsvd_meter_current_excluded": (_sz, [vp]),
        "fsvd_meter_reset_peak": (None, [vp]),
        "fsvd_meter_assert_clean": (st, [vp]),
        "fsvd_meter_event_count": (_sz, [vp]),
        "fsvd_meter_event": (st, [vp, _sz, P(C.c_int), P(C.c_int), P(_sz), P(C.c_uint64),
                                  C.c_char_p, _sz]),
        "fsvd_meter_device_peak_bytes": (_sz, [vp]),
        "fsvd_meter_device_persistent_bytes": (_sz, [vp]),
        "fsvd_validate_tile_plan": (st, [P(TilePlan), C.c_int, P(Geometry), P(_sz)]),
        "fsvd_expected_bytes": (st, [C.c_int, P(Geometry), P(_sz)]),
        "fsvd_flops_exact": (st, [P(Geometry), C.c_int, P(C.c_uint64)]),
        "fsvd_io_bytes": (st, [P(Geometry), C.c_int, P(C.c_uint64), P(C.c_uint64)]),
        "fsvd_flash_layer_peak_transient_bytes": (_sz, [P(Geometry)]),
        "fsvd_flash_layer_persistent_bytes": (_sz, [P(Geometry)]),
        "fsvd_flash_layer_bound_bytes": (_sz, [P(Geometry)]),
        "fsvd_layer_pack_create": (st, [P(LayerDesc), C.c_int, C.c_int, P(vp)]),
        "fsvd_layer_pack_destroy": (None, [vp]),
        "fsvd_layer_pack_device_bytes": (_sz, [vp]),
        "fsvd_layer_pack_uses_tensor_cores": (C.c_int, [vp]),
        "fsvd_layer_pack_row_pitch": (_sz, [vp]),
        "fsvd_pack_cache_stats": (st, [P(_sz), P(_sz), P(C.c_uint64), P(C.c_uint64)]),
        "fsvd_pack_cache_clear": (st, []),
        "fsvd_workspace_bytes": (st, [P(vp), _sz, _sz, _sz, C.c_int, P(_sz)]),
        "fsvd_workspace_bytes_ln": (st, [P(vp), _sz, _sz, _sz, C.c_int, C.c_int, P(_sz)]),
        "fsvd_attention_fwd": (st, [vp, _sz, _sz, vp, vp, vp, _sz, vp]),
        "fsvd_outproj_fwd": (st, [vp, _sz, _sz, vp, vp, vp, _sz, vp]),
        "fsvd_ffn_fwd": (st, [vp, C.c_int, _sz, _sz, vp, vp, vp, _sz, vp]),
        "fsvd_ffn_block_workspace_bytes": (st, [vp, C.c_int, _sz, _sz, C.POINTER(_sz)]),
        "fsvd_ffn_block_fwd": (st, [vp, C.c_int, _sz, _sz, vp, vp, vp, _sz, vp]),
        "fsvd_layer_fwd": (st, [vp, C.c_int, C.c_int, _sz, _sz, vp, vp, vp, _sz, vp]),
        "fsvd_model_fwd": (st, [P(vp), _sz, C.c_int, C.c_int, _sz, _sz, vp, vp, vp, _sz, vp]),
        "fsvd_model_file_probe": (st, [C.c_char_p, P(_sz), P(Geometry)]),
        "fsvd_model_load": (st, [C.c_char_p, C.c_int, C.c_int, P(vp), _sz, P(_sz)]),
        "fsvd_last_error_offset": (_sz, []),
        "fsvd_factor_rank_r": (st, [_fp, _sz, _sz, _sz, _fp, _fp]),
        "fsvd_factor_rank_r_batch": (st, [P(FactorJob), _sz]),
        "fsvd_factorize_attention": (st, [_fp] * 6 + [_sz, _sz, _sz, _fp, _fp, _fp]),
        "fsvd_factorize_layers": (st, [P(DenseLayer), _sz, _sz, P(_sz), P(_sz), P(_sz),
                                       P(FactorBuffers)]),
        "fsvd_last_factor_sweeps": (C.c_int, []),
        "fsvd_decoder_kv_cache_bytes": (st, [P(Geometry), P(_sz)]),
        "fsvd_decoder_prefill_bytes": (st, [P(Geometry), P(_sz)]),
        "fsvd_decoder_decode_step_bytes": (st, [P(Geometry), _sz, P(_sz)]),
        "fsvd_kv_cache_bytes": (st, [vp, _sz, _sz, P(_sz)]),
        "fsvd_decoder_workspace_bytes": (st, [P(vp), _sz, _sz, _sz, C.c_int, P(_sz)]),
        "fsvd_decoder_prefill": (st, [P(vp), _sz, C.c_int, _sz, _sz, vp, vp, P(vp), _sz, vp, _sz,
                                      vp]),
        "fsvd_decoder_step": (st, [P(vp), _sz, C.c_int, _sz, _sz, vp, vp, P(vp), _sz, vp, _sz,
                                   vp]),
        "fsvd_decoder_graph_create": (st, [P(vp), _sz, C.c_int, _sz, vp, vp, P(vp), _sz, vp, _sz,
                                           P(vp)]),
        "fsvd_decoder_graph_step": (st, [vp, _sz, vp]),
        "fsvd_decoder_graph_destroy": (None, [vp]),
        "fsvd_stream_workspace_bytes": (st, [P(vp), _sz, _sz, _sz, C.c_int, P(_sz)]),
        "fsvd_model_fwd_stream": (st, [P(vp), _sz, C.c_int, C.c_int, _sz, _sz, _sz, P(vp), P(vp),
                                       vp, _sz, vp]),
        "fsvd_flash_svd_attention": (st, [_fp, _sz, _sz, _sz, P(AttnDesc), _sz, P(TilePlan),
                                          C.c_int, vp, C.c_char_p, _fp, _sz, _sz, _sz]),
        "fsvd_lowrank_output_projection": (st, [_fp, _sz, _sz, _sz, P(LinearDesc), C.c_int, vp,
                                                C.c_char_p, _fp, _sz, _sz, _sz]),
        "fsvd_ffn": (st, [C.c_int, _fp, _sz, _sz, _sz, P(FfnDesc), P(TilePlan), C.c_int, vp,
                          C.c_char_p, _fp, _sz, _sz, _sz]),
        "fsvd_run_layer": (st, [_fp, _sz, _sz, _sz, P(LayerDesc), C.c_int, P(TilePlan), C.c_int,
                                C.c_char_p, C.c_int, vp, _fp]),
        "fsvd_run_model": (st, [_fp, _sz, _sz, _sz, P(LayerDesc), _sz, C.c_int, P(TilePlan),
                                C.c_int, C.c_char_p, C.c_int, vp, _fp]),
        "fsvd_kernel_launch_count": (C.c_uint64, []),
        "fsvd_kernel_name": (C.c_char_p, [C.c_int]),
        "fsvd_test_gemm": (st, [vp, _sz, vp, _sz, vp, _sz, _sz, _sz, _sz, vp, C.c_int, C.c_int,
                                vp]),
        "fsvd_test_gemm_ln": (st, [vp, _sz, vp, _sz, vp, vp, vp, vp, C.c_float, vp, _sz, _sz,
                                   _sz, vp]),
        "fsvd_test_resid_layernorm": (st, [vp, vp, vp, vp, C.c_float, vp, _sz, _sz, vp]),
        "fsvd_test_attention": (st, [vp, _sz, _sz, _sz, _sz, _sz, _sz, _sz, _sz, _sz, vp, _sz, vp]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return sorted(sigs)


EXPORTED = None


def lib():
    """Load the in-tree C-ABI library; raise loudly if it was not built."""
    global _lib, EXPORTED
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() -- there is no fallback")
        _lib = C.CDLL(LIB_PATH, mode=C.RTLD_LOCAL)
        EXPORTED = _declare(_lib)
    return _lib


def check(status: int):
    if status != OK:
        msg = lib().fsvd_last_error().decode(errors="replace")
        raise FsvdError(status, msg)
