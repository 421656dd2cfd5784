"""ctypes binding of include/vortex_b200.h (libvortex_b200.so, built in-tree for sm_100a).

There is no fallback: if the library is missing or the device is not an sm_100
part, the calls raise.  The binding mirrors the C-ABI one-to-one; the friendlier
classes live in index.py / component.py.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libvortex_b200.so"

VX_OK = 0
STATUS = {0: "VX_OK", 1: "VX_ERR_INVALID", 2: "VX_ERR_CUDA", 3: "VX_ERR_OOM", 4: "VX_ERR_NCCL",
          5: "VX_ERR_STATE", 6: "VX_ERR_UNSUPPORTED"}
VX_SCAN_AUTO, VX_SCAN_F32, VX_SCAN_TC = 0, 1, 2
VX_OPT_SCAN, VX_OPT_GRID, VX_OPT_GRAPHS, VX_OPT_MAXSIM = 1, 2, 3, 4
VX_MAXSIM_AUTO, VX_MAXSIM_CC, VX_MAXSIM_TC, VX_MAXSIM_TC_BF16Q = 0, 1, 2, 3
VX_OPT_COARSE, VX_OPT_SCAN_TILE, VX_OPT_SCAN_PAIRS, VX_OPT_KPRIME, VX_OPT_SCAN_SEED = 5, 6, 7, 8, 9
VX_OPT_I8_SCALE = 10
VX_OPT_STAGE_EVENTS = 11
VX_COARSE_AUTO, VX_COARSE_TF32, VX_COARSE_BF16, VX_COARSE_I8 = 0, 1, 2, 3
VX_FLAG_NO_BF16_SHADOW = 1
VX_FLAG_NO_I8_SHADOW = 2
VX_FLAG_TOKENS_F32 = 4
VX_PREPARE_SEARCH, VX_PREPARE_RESCORE = 1, 2


class VxError(RuntimeError):
    """Raised for any non-VX_OK status (message from vx_last_error)."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class IndexDesc(C.Structure):
    _fields_ = [("n_docs", C.c_int64), ("dim", C.c_int32), ("device", C.c_int32),
                ("n_shards", C.c_int32), ("shard", C.c_int32), ("tok_per_doc", C.c_int32),
                ("tok_dim", C.c_int32), ("tok_blocks", C.c_int64), ("max_batch", C.c_int32),
                ("max_k", C.c_int32), ("max_qtok", C.c_int32), ("flags", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("kernel_launches", C.c_uint64), ("batches", C.c_uint64), ("queries", C.c_uint64),
                ("graph_replays", C.c_uint64), ("cert_fallbacks", C.c_uint64),
                ("last_scan_ms", C.c_float), ("last_step_ms", C.c_float),
                ("scan_ms_total", C.c_double), ("step_ms_total", C.c_double),
                ("timed_batches", C.c_uint64), ("phase_ms", C.c_float * 4),
                ("cert_level2", C.c_uint64), ("host_staged_bytes", C.c_uint64),
                ("kt_launches", C.c_uint64 * 4), ("kt_ms", C.c_double * 4), ("kt_sm_mhz", C.c_double * 4),
                ("phase_detail_ms", C.c_float * 6), ("kt_rerank_launches", C.c_uint64),
                ("kt_rerank_ms", C.c_double), ("kt_last_us", C.c_double * 10),
                ("kt_origin_ns", C.c_uint64)]


P = C.c_void_p
I32, I64, U64 = C.c_int32, C.c_int64, C.c_uint64
FP, LP, HP = C.POINTER(C.c_float), C.POINTER(C.c_int64), C.POINTER(C.c_uint16)

# name -> (argtypes)
SIGNATURES = {
    "vx_abi_version": [],
    "vx_last_error": [],
    "vx_index_create": [C.POINTER(IndexDesc), C.POINTER(P)],
    "vx_index_destroy": [P],
    "vx_index_shard_range": [P, C.POINTER(I64), C.POINTER(I64)],
    "vx_set_option": [P, I32, I64],
    "vx_get_option": [P, I32, C.POINTER(I64)],
    "vx_get_stats": [P, C.POINTER(Stats)],
    "vx_reset_stats": [P],
    "vx_index_synth": [P, U64],
    "vx_index_synth_dist": [P, U64, I32],
    "vx_index_upload": [P, FP, I64, I64],
    "vx_index_download": [P, FP, I64, I64],
    "vx_tokens_synth": [P, U64],
    "vx_tokens_download": [P, HP, I64, I64],
    "vx_tokens_upload": [P, HP, I64, I64],
    "vx_tokens_upload_f32": [P, FP, I64, I64],
    "vx_tokens_download_f32": [P, FP, I64, I64],
    "vx_search": [P, FP, I32, I32, LP, FP],
    "vx_search_rows": [P, C.POINTER(FP), I32, I32, LP, FP],
    "vx_search_rescore_rows": [P, C.POINTER(FP), C.POINTER(FP), I32, I32, I32, LP, FP, FP],
    "vx_maxsim": [P, FP, I32, I32, LP, I32, FP],
    "vx_search_rescore": [P, FP, FP, I32, I32, I32, LP, FP, FP],
    "vx_search_dev": [P, P, I32, I32, P, P, P],
    "vx_maxsim_dev": [P, P, I32, I32, P, I32, P, P],
    "vx_search_rescore_dev": [P, P, P, I32, I32, I32, P, P, P, P],
    "vx_sync": [P],
    "vx_prepare": [P, I32, I32, I32, I32],
    "vx_batcher_simulate": [C.POINTER(U64), I64, I32, C.POINTER(I32), C.POINTER(C.c_double), I32,
                            LP, C.POINTER(U64), C.POINTER(U64), C.POINTER(I64)],
    "vx_batcher_simulate_replicas": [C.POINTER(U64), I64, I32, I32, C.POINTER(I32),
                                     C.POINTER(C.c_double), I32, U64, C.POINTER(I32),
                                     C.POINTER(U64), C.POINTER(U64), C.POINTER(I64)],
    "vx_arrival_times": [C.c_double, I64, U64, U64, I32, C.POINTER(U64)],
    "vx_serve_trace": [P, C.POINTER(U64), I64, I32, FP, FP, I32, I32, LP,
                       C.POINTER(C.c_double), LP, C.POINTER(I64)],
    "vx_serve_trace_replicas": [C.POINTER(P), I32, C.POINTER(U64), I64, I32, FP, FP, I32, I32, U64,
                                C.POINTER(I32), C.POINTER(U64), C.POINTER(U64), C.POINTER(U64),
                                C.POINTER(U64), C.POINTER(U64), LP, C.POINTER(C.c_double), LP, LP],
    "vx_comm_unique_id": [C.POINTER(C.c_uint8)],
    "vx_comm_init": [P, C.POINTER(C.c_uint8), I32, I32],
    "vx_shard_serve": [P],
    "vx_shard_stop": [P],
}

_lib = None


def load(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load libvortex_b200.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"{p} is missing: build it with `python -m paper_2511_02062_b200.build` "
                          "(the retrieval stage has no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, argt in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argt
        fn.restype = C.c_int32
    lib.vx_last_error.restype = C.c_char_p
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != VX_OK:
        raise VxError(status, load().vx_last_error().decode(errors="replace"))
