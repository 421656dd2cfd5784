"""ctypes binding of the CPU oracle (oracle/libvx_oracle.so).  TEST INFRASTRUCTURE ONLY:
imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg — never by the product package.  See vx_oracle.h for what it restates.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libvx_oracle.so"
F64, F32 = 0, 1
_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE), "libvx_oracle.so"], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        fp, dp, lp, hp = (C.POINTER(C.c_float), C.POINTER(C.c_double), C.POINTER(C.c_int64),
                          C.POINTER(C.c_uint16))
        i32, i64, u64 = C.c_int32, C.c_int64, C.c_uint64
        L.vxo_threads.restype = C.c_int
        L.vxo_synth_rows.argtypes = [u64, i64, i64, i32, fp]
        L.vxo_synth_rows.restype = None
        L.vxo_synth_tokens.argtypes = [u64, i64, i64, i32, i32, hp]
        L.vxo_synth_tokens.restype = None
        L.vxo_dot.argtypes = [fp, fp, i32, i32]
        L.vxo_dot.restype = C.c_double
        L.vxo_flat_topk.argtypes = [fp, i64, i32, i64, fp, i32, i32, i32, i32, lp, dp]
        L.vxo_maxsim.argtypes = [fp, i32, i32, i32, lp, i32, hp, i64, i32, i32, i32, dp]
        L.vxo_search_rescore.argtypes = [fp, i64, i32, fp, fp, i32, i32, i32, i32, hp, i64, i32, i32,
                                         i32, lp, dp, dp]
        L.vxo_percentile.argtypes = [dp, i64, C.c_double]
        L.vxo_percentile.restype = C.c_double
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def threads() -> int:
    return lib().vxo_threads()


def synth_rows(seed: int, row0: int, n: int, dim: int) -> np.ndarray:
    out = np.empty((n, dim), np.float32)
    lib().vxo_synth_rows(seed, row0, n, dim, _p(out, C.c_float))
    return out


def synth_tokens(seed: int, blk0: int, nblk: int, ntok: int, dim: int) -> np.ndarray:
    out = np.empty((nblk, ntok, dim), np.uint16)
    lib().vxo_synth_tokens(seed, blk0, nblk, ntok, dim, _p(out, C.c_uint16))
    return out


def flat_topk(X, Q, k, mode=F64, id_base=0, threads=0):
    X = np.ascontiguousarray(X, np.float32)
    Q = np.ascontiguousarray(Q, np.float32)
    B = Q.shape[0]
    ids = np.empty((B, k), np.int64)
    sc = np.empty((B, k), np.float64)
    rc = lib().vxo_flat_topk(_p(X, C.c_float), X.shape[0], X.shape[1], id_base, _p(Q, C.c_float),
                             B, k, mode, threads, _p(ids, C.c_int64), _p(sc, C.c_double))
    assert rc == 0
    return ids, sc


def maxsim(qtok, cand, table, mode=F64, threads=0):
    qtok = np.ascontiguousarray(qtok, np.float32)
    cand = np.ascontiguousarray(cand, np.int64)
    table = np.ascontiguousarray(table, np.uint16)
    B, nq, d = qtok.shape
    out = np.empty(cand.shape, np.float64)
    rc = lib().vxo_maxsim(_p(qtok, C.c_float), B, nq, d, _p(cand, C.c_int64), cand.shape[1],
                          _p(table, C.c_uint16), table.shape[0], table.shape[1], mode, threads,
                          _p(out, C.c_double))
    assert rc == 0
    return out


def search_rescore(X, Q, qtok, table, k, mode=F64, threads=0):
    X = np.ascontiguousarray(X, np.float32)
    Q = np.ascontiguousarray(Q, np.float32)
    qtok = np.ascontiguousarray(qtok, np.float32)
    table = np.ascontiguousarray(table, np.uint16)
    B, nq, d = qtok.shape
    ids = np.empty((B, k), np.int64)
    ip = np.empty((B, k), np.float64)
    ms = np.empty((B, k), np.float64)
    rc = lib().vxo_search_rescore(_p(X, C.c_float), X.shape[0], X.shape[1], _p(Q, C.c_float),
                                  _p(qtok, C.c_float), B, nq, d, k, _p(table, C.c_uint16),
                                  table.shape[0], table.shape[1], mode, threads,
                                  _p(ids, C.c_int64), _p(ip, C.c_double), _p(ms, C.c_double))
    assert rc == 0
    return ids, ip, ms


def percentile(v, p: float) -> float:
    a = np.array(v, np.float64)
    return lib().vxo_percentile(_p(a, C.c_double), a.shape[0], p)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, np.uint32) << 16).view(np.float32)
