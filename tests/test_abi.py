"""C-ABI library loads and exports every symbol include/vortex_b200.h declares; host logic
(payload codec, registry) behaves like the reference's operator contract.  CPU only: no
compute call is made (there is no GPU here, and the library must refuse rather than fall
back)."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols() -> set[str]:
    text = (ROOT / "include" / "vortex_b200.h").read_text()
    return set(re.findall(r"\b(vx_[a-z0-9_]+)\s*\(", text))


def test_exports_every_declared_symbol(vxlib):
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in sorted(syms):
        assert hasattr(vxlib, s), s
    from paper_2511_02062_b200._lib import SIGNATURES
    assert syms == set(SIGNATURES), syms ^ set(SIGNATURES)


def test_abi_version(vxlib):
    assert vxlib.vx_abi_version() == 1


def test_no_cpu_fallback_without_gpu(vxlib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2511_02062_b200 import Index, VxError
    with pytest.raises(VxError) as ei:
        Index(1000, 64)
    assert "VX_ERR_CUDA" in str(ei.value)


def test_invalid_desc_rejected(vxlib):
    from paper_2511_02062_b200._lib import IndexDesc
    h = C.c_void_p()
    bad = IndexDesc(n_docs=10, dim=33, device=0, n_shards=1, shard=0, max_batch=1, max_k=1)
    assert vxlib.vx_index_create(C.byref(bad), C.byref(h)) == 1  # VX_ERR_INVALID
    assert b"dim" in vxlib.vx_last_error()
    bad = IndexDesc(n_docs=10, dim=32, device=0, n_shards=2, shard=2, max_batch=1, max_k=1)
    assert vxlib.vx_index_create(C.byref(bad), C.byref(h)) == 1
    bad = IndexDesc(n_docs=10, dim=32, device=0, n_shards=1, shard=0, max_batch=1, max_k=300)
    assert vxlib.vx_index_create(C.byref(bad), C.byref(h)) == 1


def test_query_payload_roundtrip():
    from paper_2511_02062_b200 import decode_query, encode_query
    q = np.arange(768, dtype=np.float32)
    t = np.ones((32, 128), np.float32)
    q2, t2 = decode_query(encode_query(q, t))
    assert np.array_equal(q, q2) and np.array_equal(t, t2)
    q3, t3 = decode_query(encode_query(q))
    assert np.array_equal(q, q3) and t3 is None


def test_payload_errors_are_bad_config():
    from paper_2511_02062_b200 import VortexError, decode_query, encode_query
    p = encode_query(np.zeros(64, np.float32))
    for bad in (p[:10], p[:-4], b"XXXX" + p[4:]):
        with pytest.raises(VortexError) as ei:
            decode_query(bad)
        assert ei.value.code == "BadConfig"


def test_result_payload_roundtrip():
    from paper_2511_02062_b200 import decode_result, encode_result
    ids = np.array([5, 3, -1], np.int64)
    ip = np.array([0.5, 0.25, -np.inf], np.float32)
    ms = np.array([9.0, 8.0, -np.inf], np.float32)
    r = decode_result(encode_result(ids, ip, ms))
    assert r["id"].tolist() == [5, 3, -1] and r["ms"][0] == 9.0


def test_registry_semantics():
    # runtime.hpp:202-211 duplicate -> AlreadyRegistered; :660 identity when unregistered;
    # test_runtime.cpp:352-365 output i <-> input i.
    from paper_2511_02062_b200 import Registry, VortexError
    reg = Registry()
    assert reg.register_component("modelD", lambda xs: [x + b"!" for x in xs]) == "modelD"
    with pytest.raises(VortexError) as ei:
        reg.register_component("modelD", lambda xs: xs)
    assert ei.value.code == "AlreadyRegistered"
    assert reg.invoke("modelD", [b"hey", b"yo"]) == [b"hey!", b"yo!"]
    assert reg.invoke("modelA", [b"x"]) == [b"x"]
    reg.register_component("short", lambda xs: xs[:-1])
    with pytest.raises(VortexError):
        reg.invoke("short", [b"a", b"b"])
