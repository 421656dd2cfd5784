"""Host-side handle of one index shard on one B200 (wraps the vx_* C-ABI).

This is the Python face of the search-stage operator; the reference's operator
contract (batch in, top-k ids/scores out, output i <-> input i;
proj/include/vortex/runtime.hpp:179, :656-672) is implemented by component.py on
top of it, and by include/vortex_b200_component.hpp for C++ hosts.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import FP, HP, LP, IndexDesc, Stats, check


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


class Index:
    """One shard (rows [row0, row0+n_local)) of an N x D fp32 inner-product index,
    plus an optional bf16 late-interaction token store (doc id -> block id mod T)."""

    def __init__(self, n_docs: int, dim: int, *, device: int = 0, n_shards: int = 1, shard: int = 0,
                 tok_per_doc: int = 0, tok_dim: int = 128, tok_blocks: int = 1,
                 max_batch: int = 64, max_k: int = 128, max_qtok: int = 32, flags: int = 0):
        self.lib = _lib.load()
        d = IndexDesc(n_docs=n_docs, dim=dim, device=device, n_shards=n_shards, shard=shard,
                      tok_per_doc=tok_per_doc, tok_dim=tok_dim if tok_per_doc else 0,
                      tok_blocks=tok_blocks if tok_per_doc else 0, max_batch=max_batch,
                      max_k=max_k, max_qtok=max_qtok if tok_per_doc else 0, flags=flags)
        self.desc = d
        self._h = C.c_void_p()
        check(self.lib.vx_index_create(C.byref(d), C.byref(self._h)))
        r0, nl = C.c_int64(), C.c_int64()
        check(self.lib.vx_index_shard_range(self._h, C.byref(r0), C.byref(nl)))
        self.row0, self.n_local = r0.value, nl.value
        self.n_docs, self.dim = n_docs, dim
        self.tok_per_doc, self.tok_dim, self.tok_blocks = tok_per_doc, tok_dim, tok_blocks
        self.max_batch, self.max_k, self.max_qtok = max_batch, max_k, max_qtok

    # -- lifecycle ------------------------------------------------------------------
    def close(self) -> None:
        if self._h:
            check(self.lib.vx_index_destroy(self._h))
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    # -- options / stats --------------------------------------------------------------
    def set_option(self, option: int, value: int) -> None:
        check(self.lib.vx_set_option(self._h, option, value))

    def get_option(self, option: int) -> int:
        v = C.c_int64()
        check(self.lib.vx_get_option(self._h, option, C.byref(v)))
        return v.value

    def coarse_auto(self) -> str:
        """The coarse format the tensor-core scan will use: "bf16", "tf32" or "i8"."""
        return {_lib.VX_COARSE_BF16: "bf16", _lib.VX_COARSE_TF32: "tf32",
                _lib.VX_COARSE_I8: "i8"}[self.get_option(_lib.VX_OPT_COARSE)]

    def stats(self) -> dict:
        s = Stats()
        check(self.lib.vx_get_stats(self._h, C.byref(s)))
        out = {f: getattr(s, f) for f, _ in Stats._fields_}
        out["phase_ms"] = list(s.phase_ms)
        for f in ("kt_launches", "kt_ms", "kt_sm_mhz", "phase_detail_ms", "kt_last_us"):
            out[f] = list(getattr(s, f))
        return out

    def reset_stats(self) -> None:
        check(self.lib.vx_reset_stats(self._h))

    # -- data ---------------------------------------------------------------------------
    def synth(self, seed: int = 42, dist: int = 0) -> None:
        """Device fill with the vx_synth.h generator; dist 1 = anisotropic rows."""
        check(self.lib.vx_index_synth_dist(self._h, seed, dist))

    def upload(self, rows: np.ndarray, row0: int | None = None) -> None:
        rows = _f32(rows)
        r0 = self.row0 if row0 is None else row0
        check(self.lib.vx_index_upload(self._h, rows.ctypes.data_as(FP), r0, rows.shape[0]))

    def download(self, row0: int, n: int) -> np.ndarray:
        out = np.empty((n, self.dim), np.float32)
        check(self.lib.vx_index_download(self._h, out.ctypes.data_as(FP), row0, n))
        return out

    @property
    def tokens_f32(self) -> bool:
        """The token store is fp32 (VX_FLAG_TOKENS_F32), else bf16."""
        return bool(self.desc.flags & _lib.VX_FLAG_TOKENS_F32)

    def tokens_download(self, blk0: int, n: int) -> np.ndarray:
        """Token blocks [n][Nd][d]: uint16 bf16 bits (bf16 store) or float32 (fp32 store)."""
        if self.tokens_f32:
            out = np.empty((n, self.tok_per_doc, self.tok_dim), np.float32)
            check(self.lib.vx_tokens_download_f32(self._h, out.ctypes.data_as(FP), blk0, n))
            return out
        out = np.empty((n, self.tok_per_doc, self.tok_dim), np.uint16)
        check(self.lib.vx_tokens_download(self._h, out.ctypes.data_as(HP), blk0, n))
        return out

    def tokens_synth(self, seed: int = 45) -> None:
        check(self.lib.vx_tokens_synth(self._h, seed))

    def tokens_upload(self, tokens: np.ndarray, blk0: int = 0) -> None:
        """bf16 store: uint16 bf16 bits; fp32 store (VX_FLAG_TOKENS_F32): float32 values."""
        if self.tokens_f32:
            t = np.ascontiguousarray(tokens, dtype=np.float32)
            check(self.lib.vx_tokens_upload_f32(self._h, t.ctypes.data_as(FP), blk0, t.shape[0]))
            return
        t = np.ascontiguousarray(tokens, dtype=np.uint16)
        check(self.lib.vx_tokens_upload(self._h, t.ctypes.data_as(HP), blk0, t.shape[0]))

    # -- host-buffer operators ------------------------------------------------------------
    def search(self, q: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
        q = _f32(q)
        B = q.shape[0]
        ids = np.empty((B, k), np.int64)
        sc = np.empty((B, k), np.float32)
        check(self.lib.vx_search(self._h, q.ctypes.data_as(FP), B, k, ids.ctypes.data_as(LP),
                                 sc.ctypes.data_as(FP)))
        return ids, sc

    def maxsim(self, qtok: np.ndarray, cand: np.ndarray) -> np.ndarray:
        qtok = _f32(qtok)
        cand = np.ascontiguousarray(cand, dtype=np.int64)
        B, nq, _ = qtok.shape
        C_ = cand.shape[1]
        out = np.empty((B, C_), np.float32)
        check(self.lib.vx_maxsim(self._h, qtok.ctypes.data_as(FP), B, nq, cand.ctypes.data_as(LP),
                                 C_, out.ctypes.data_as(FP)))
        return out

    def search_rescore(self, q: np.ndarray, qtok: np.ndarray, k: int):
        q, qtok = _f32(q), _f32(qtok)
        B = q.shape[0]
        nq = qtok.shape[1]
        ids = np.empty((B, k), np.int64)
        ip = np.empty((B, k), np.float32)
        ms = np.empty((B, k), np.float32)
        check(self.lib.vx_search_rescore(self._h, q.ctypes.data_as(FP), qtok.ctypes.data_as(FP), B,
                                         nq, k, ids.ctypes.data_as(LP), ip.ctypes.data_as(FP),
                                         ms.ctypes.data_as(FP)))
        return ids, ip, ms

    def search_rescore_rows(self, q_rows, tok_rows, k: int):
        """Row-gather variant: per-query arrays (e.g. views into payload buffers); the library
        copies each once into its pinned staging (vx_search_rescore_rows)."""
        qs = [_f32(r) for r in q_rows]
        ts = [_f32(t) for t in tok_rows]
        B, nq = len(qs), ts[0].shape[0]
        qp = (FP * B)(*[r.ctypes.data_as(FP) for r in qs])
        tp = (FP * B)(*[t.ctypes.data_as(FP) for t in ts])
        ids = np.empty((B, k), np.int64)
        ip = np.empty((B, k), np.float32)
        ms = np.empty((B, k), np.float32)
        check(self.lib.vx_search_rescore_rows(self._h, qp, tp, B, nq, k, ids.ctypes.data_as(LP),
                                              ip.ctypes.data_as(FP), ms.ctypes.data_as(FP)))
        return ids, ip, ms

    def search_rows(self, q_rows, k: int) -> tuple[np.ndarray, np.ndarray]:
        qs = [_f32(r) for r in q_rows]
        B = len(qs)
        qp = (FP * B)(*[r.ctypes.data_as(FP) for r in qs])
        ids = np.empty((B, k), np.int64)
        sc = np.empty((B, k), np.float32)
        check(self.lib.vx_search_rows(self._h, qp, B, k, ids.ctypes.data_as(LP), sc.ctypes.data_as(FP)))
        return ids, sc

    # -- device-pointer operators (torch tensors resident in HBM) ------------------------------
    def search_dev(self, q, ids, scores, k: int, stream: int | None = None) -> None:
        check(self.lib.vx_search_dev(self._h, C.c_void_p(q.data_ptr()), q.shape[0], k,
                                     C.c_void_p(ids.data_ptr()), C.c_void_p(scores.data_ptr()),
                                     C.c_void_p(stream or 0)))

    def search_rescore_dev(self, q, qtok, ids, ip, ms, k: int, stream: int | None = None) -> None:
        check(self.lib.vx_search_rescore_dev(self._h, C.c_void_p(q.data_ptr()),
                                             C.c_void_p(qtok.data_ptr()), q.shape[0], qtok.shape[1],
                                             k, C.c_void_p(ids.data_ptr()), C.c_void_p(ip.data_ptr()),
                                             C.c_void_p(ms.data_ptr()), C.c_void_p(stream or 0)))

    def maxsim_dev(self, qtok, cand, out, stream: int | None = None) -> None:
        check(self.lib.vx_maxsim_dev(self._h, C.c_void_p(qtok.data_ptr()), qtok.shape[0],
                                     qtok.shape[1], C.c_void_p(cand.data_ptr()), cand.shape[1],
                                     C.c_void_p(out.data_ptr()), C.c_void_p(stream or 0)))

    def sync(self) -> None:
        check(self.lib.vx_sync(self._h))

    def prepare(self, k: int, b_max: int | None = None, nq: int = 0) -> None:
        """Model load: capture the stage graph of every batch size 1..b_max (nq > 0: the
        fused search+rescore stage, else search) before serving."""
        op = _lib.VX_PREPARE_RESCORE if nq else _lib.VX_PREPARE_SEARCH
        check(self.lib.vx_prepare(self._h, op, k, nq, b_max or self.max_batch))

    # -- multi-GPU -----------------------------------------------------------------------------
    @staticmethod
    def comm_unique_id() -> bytes:
        lib = _lib.load()
        buf = (C.c_uint8 * 128)()
        check(lib.vx_comm_unique_id(buf))
        return bytes(buf)

    def comm_init(self, uid: bytes, nranks: int, rank: int) -> None:
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        check(self.lib.vx_comm_init(self._h, buf, nranks, rank))

    def shard_serve(self) -> None:
        check(self.lib.vx_shard_serve(self._h))

    def shard_stop(self) -> None:
        check(self.lib.vx_shard_stop(self._h))
