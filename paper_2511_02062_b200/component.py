"""The search-stage operator in the reference's plugin shape.

Reference contract (proj/include/vortex/runtime.hpp):
  * ``using ComponentFn = std::function<std::vector<Payload>(const std::vector<Payload>&)>``  (:179)
  * registered per model id with ``Runtime::register_component`` — a duplicate id is
    ``errc::already_registered`` (:202-211); the search stage is ``modelD``
    (proj/assets/pipeline.json:7);
  * called by ``Runtime::complete_batch`` with the FIFO batch the opportunistic batcher
    formed (:617-672); output ``i`` must correspond to input ``i`` and there must be at
    least as many outputs as inputs (:663-666).
  * errors are ``vortex::error(errc, msg)`` (proj/include/vortex/common.hpp:70-80).

``SearchComponent`` is that callable: a list of query payloads (bytes) in, a list of
result payloads out, one fused GPU call per batch.  ``Registry`` mirrors
``register_component`` for Python hosts; the C++ twin is include/vortex_b200_component.hpp.

Wire format (little endian; identical in the C++ adapter):
  query  : b"VXQ1" u16 version=1 u16 dtype=0(f32) u32 dim u32 nq u32 tok_dim u32 0
           f32[dim] f32[nq*tok_dim]
  result : b"VXR1" u16 version=1 u16 flags(bit0: maxsim valid) u32 k u32 0
           k x { i64 id, f32 ip_score, f32 maxsim_score }   (ordered as the stage ranks them)
"""
from __future__ import annotations

import struct
from typing import Callable, Sequence

import numpy as np

QUERY_MAGIC = b"VXQ1"
RESULT_MAGIC = b"VXR1"
_QHDR = struct.Struct("<4sHHIIII")
_RHDR = struct.Struct("<4sHHII")
RESULT_DTYPE = np.dtype([("id", "<i8"), ("ip", "<f4"), ("ms", "<f4")])


class VortexError(RuntimeError):
    """Python mirror of vortex::error — ``code`` is the reference errc name."""

    def __init__(self, code: str, what: str):
        super().__init__(f"{code}: {what}")
        self.code = code


def encode_query(q: np.ndarray, qtok: np.ndarray | None = None) -> bytes:
    q = np.ascontiguousarray(q, dtype="<f4").reshape(-1)
    if qtok is None:
        nq, td, tb = 0, 0, b""
    else:
        qtok = np.ascontiguousarray(qtok, dtype="<f4")
        nq, td = qtok.shape
        tb = qtok.tobytes()
    return _QHDR.pack(QUERY_MAGIC, 1, 0, q.shape[0], nq, td, 0) + q.tobytes() + tb


def decode_query(p: bytes) -> tuple[np.ndarray, np.ndarray | None]:
    if len(p) < _QHDR.size:
        raise VortexError("BadConfig", f"query payload of {len(p)} bytes")
    magic, ver, dtype, dim, nq, td, _ = _QHDR.unpack_from(p)
    if magic != QUERY_MAGIC or ver != 1 or dtype != 0:
        raise VortexError("BadConfig", "query payload header")
    need = _QHDR.size + 4 * (dim + nq * td)
    if len(p) != need:
        raise VortexError("BadConfig", f"query payload {len(p)} bytes, header says {need}")
    q = np.frombuffer(p, "<f4", dim, _QHDR.size)
    qtok = np.frombuffer(p, "<f4", nq * td, _QHDR.size + 4 * dim).reshape(nq, td) if nq else None
    return q, qtok


def encode_result(ids: np.ndarray, ip: np.ndarray, ms: np.ndarray | None) -> bytes:
    k = ids.shape[0]
    rec = np.empty(k, RESULT_DTYPE)
    rec["id"], rec["ip"] = ids, ip
    rec["ms"] = ms if ms is not None else np.float32("nan")
    return _RHDR.pack(RESULT_MAGIC, 1, 1 if ms is not None else 0, k, 0) + rec.tobytes()


def decode_result(p: bytes) -> np.ndarray:
    magic, ver, flags, k, _ = _RHDR.unpack_from(p)
    if magic != RESULT_MAGIC or ver != 1 or len(p) != _RHDR.size + 16 * k:
        raise VortexError("BadConfig", "result payload")
    return np.frombuffer(p, RESULT_DTYPE, k, _RHDR.size)


class SearchComponent:
    """ComponentFn for the retrieval stage: IP top-k over the index, MaxSim
    re-scoring of those k when the queries carry tokens."""

    def __init__(self, index, k: int):
        self.index = index
        self.k = k

    def __call__(self, inputs: Sequence[bytes]) -> list[bytes]:
        if len(inputs) == 0:
            return []
        if len(inputs) > self.index.max_batch:
            raise VortexError("BadConfig", f"batch {len(inputs)} > max_batch {self.index.max_batch}")
        dec = [decode_query(p) for p in inputs]
        dims = {q.shape[0] for q, _ in dec}
        if dims != {self.index.dim}:
            raise VortexError("BadConfig", f"query dims {sorted(dims)} != index dim {self.index.dim}")
        with_tok = {t is not None for _, t in dec}
        if len(with_tok) != 1:
            raise VortexError("BadConfig", "mixed batches (with and without query tokens)")
        Q = np.stack([q for q, _ in dec])
        if with_tok.pop():
            shapes = {t.shape for _, t in dec}
            if len(shapes) != 1:
                raise VortexError("BadConfig", f"ragged query-token shapes {sorted(shapes)}")
            T = np.stack([t for _, t in dec])
            ids, ip, ms = self.index.search_rescore(Q, T, self.k)
            return [encode_result(ids[i], ip[i], ms[i]) for i in range(len(inputs))]
        ids, ip = self.index.search(Q, self.k)
        return [encode_result(ids[i], ip[i], None) for i in range(len(inputs))]


class Registry:
    """``Runtime::register_component`` semantics (runtime.hpp:202-211): one function per
    model id, duplicates rejected, the id is returned as the handler id; unregistered
    stages behave as identity (runtime.hpp:660)."""

    def __init__(self):
        self._fns: dict[str, Callable[[Sequence[bytes]], list[bytes]]] = {}

    def register_component(self, model_id: str, fn) -> str:
        if model_id in self._fns:
            raise VortexError("AlreadyRegistered", model_id)
        self._fns[model_id] = fn
        return model_id

    def invoke(self, model_id: str, inputs: Sequence[bytes]) -> list[bytes]:
        fn = self._fns.get(model_id)
        out = list(inputs) if fn is None else fn(inputs)
        if len(out) < len(inputs):
            raise VortexError("BadConfig", f"{model_id} returned {len(out)} outputs for {len(inputs)} inputs")
        return out
