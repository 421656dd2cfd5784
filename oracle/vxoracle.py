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
F64, F32, F64_Q32 = 0, 1, 2
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
        L.vxo_synth_rows_dist.argtypes = [u64, i64, i64, i32, i32, fp]
        L.vxo_synth_rows_dist.restype = None
        L.vxo_synth_tokens.argtypes = [u64, i64, i64, i32, i32, hp]
        L.vxo_synth_tokens.restype = None
        L.vxo_synth_token_blocks.argtypes = [u64, lp, i64, i32, i32, hp]
        L.vxo_synth_token_blocks.restype = None
        L.vxo_dot.argtypes = [fp, fp, i32, i32]
        L.vxo_dot.restype = C.c_double
        L.vxo_flat_topk.argtypes = [fp, i64, i32, i64, fp, i32, i32, i32, i32, lp, dp]
        L.vxo_maxsim.argtypes = [fp, i32, i32, i32, lp, i32, hp, i64, i32, i32, i32, dp]
        L.vxo_maxsim_f32tab.argtypes = [fp, i32, i32, i32, lp, i32, fp, i64, i32, i32, i32, dp]
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


def synth_rows(seed: int, row0: int, n: int, dim: int, dist: int = 0) -> np.ndarray:
    out = np.empty((n, dim), np.float32)
    lib().vxo_synth_rows_dist(seed, row0, n, dim, dist, _p(out, C.c_float))
    return out


def synth_tokens(seed: int, blk0: int, nblk: int, ntok: int, dim: int) -> np.ndarray:
    out = np.empty((nblk, ntok, dim), np.uint16)
    lib().vxo_synth_tokens(seed, blk0, nblk, ntok, dim, _p(out, C.c_uint16))
    return out


def synth_token_blocks(seed: int, blks, ntok: int, dim: int) -> np.ndarray:
    blks = np.ascontiguousarray(blks, np.int64)
    out = np.empty((blks.shape[0], ntok, dim), np.uint16)
    lib().vxo_synth_token_blocks(seed, _p(blks, C.c_int64), blks.shape[0], ntok, dim,
                                 _p(out, C.c_uint16))
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
    """table: uint16 bf16 bits [T][Nd][d] (the bf16 store) or float32 (the fp32 store,
    vx_oracle.c vxo_maxsim_f32tab)."""
    qtok = np.ascontiguousarray(qtok, np.float32)
    cand = np.ascontiguousarray(cand, np.int64)
    B, nq, d = qtok.shape
    out = np.empty(cand.shape, np.float64)
    if np.asarray(table).dtype == np.float32:
        table = np.ascontiguousarray(table, np.float32)
        rc = lib().vxo_maxsim_f32tab(_p(qtok, C.c_float), B, nq, d, _p(cand, C.c_int64),
                                     cand.shape[1], _p(table, C.c_float), table.shape[0],
                                     table.shape[1], mode, threads, _p(out, C.c_double))
        assert rc == 0
        return out
    table = np.ascontiguousarray(table, np.uint16)
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


# ---- full-size helpers: the headline index (10M x 768 = 30.7 GB) never exists on the host;
# rows are generated chunk by chunk and the per-chunk lists merged, so the oracle checks the
# benched configuration itself.

def merge_topk(ids_a, sc_a, ids_b, sc_b, k):
    """Top-k of the union of two per-query lists, ordered (score desc, id asc); -1 ids pad."""
    ids = np.concatenate([ids_a, ids_b], axis=1)
    sc = np.concatenate([sc_a, sc_b], axis=1)
    sc = np.where(ids < 0, -np.inf, sc)
    idk = np.where(ids < 0, np.iinfo(np.int64).max, ids)
    out_i = np.empty((ids.shape[0], k), np.int64)
    out_s = np.empty((ids.shape[0], k), np.float64)
    for b in range(ids.shape[0]):
        o = np.lexsort((idk[b], -sc[b]))[:k]
        out_i[b], out_s[b] = ids[b][o], sc[b][o]
    out_i[~np.isfinite(out_s)] = -1
    return out_i, out_s


def flat_topk_synth(seed, n_docs, dim, Q, k, mode=F32, row0=0, chunk=1 << 20, threads=0, dist=0):
    """Exact top-k of Q over the synthetic rows [row0, row0 + n_docs) (vx_synth.h, seed),
    generated in chunks.  Returns (ids, scores, scan_seconds): scan_seconds times only the
    top-k passes (row generation is input preparation, untimed)."""
    import time
    Q = np.ascontiguousarray(Q, np.float32)
    B = Q.shape[0]
    ids = np.full((B, k), -1, np.int64)
    sc = np.full((B, k), -np.inf)
    t_scan = 0.0
    for r0 in range(row0, row0 + n_docs, chunk):
        n = min(chunk, row0 + n_docs - r0)
        X = synth_rows(seed, r0, n, dim, dist)
        t0 = time.perf_counter()
        ci, cs = flat_topk(X, Q, k, mode=mode, id_base=r0, threads=threads)
        t_scan += time.perf_counter() - t0
        ids, sc = merge_topk(ids, sc, ci, cs, k)
        del X
    return ids, sc, t_scan


def maxsim_synth(qtok, cand, seed, T, ntok, dim, mode=F64, threads=0):
    """MaxSim of qtok [B][nq][d] against cand [B][C] over the synthetic token table (seed,
    T blocks), generating only the blocks the candidates use (doc id -> block id mod T)."""
    cand = np.asarray(cand, np.int64)
    blk = np.where(cand >= 0, cand % T, 0)
    uniq, inv = np.unique(blk, return_inverse=True)
    table = synth_token_blocks(seed, uniq, ntok, dim)
    local = np.where(cand >= 0, inv.reshape(cand.shape), -1).astype(np.int64)
    # ids index the compact table directly (local < len(uniq) = its T)
    return maxsim(qtok, local, table, mode=mode, threads=threads)


def order_by_maxsim(ids, ms):
    """The fused stage's output order: MaxSim desc, id asc (-1 / -inf last)."""
    out_i, out_m = np.empty_like(ids), np.empty_like(ms)
    for b in range(ids.shape[0]):
        idk = np.where(ids[b] < 0, np.iinfo(np.int64).max, ids[b])
        o = np.lexsort((idk, -np.where(ids[b] < 0, -np.inf, ms[b])))
        out_i[b], out_m[b] = ids[b][o], ms[b][o]
    return out_i, out_m
