"""Generates the committed golden fixtures that pin the CPU oracle.

The reference (/root/reference) contains no retrieval arithmetic, so
these fixtures are computed independently of the C oracle:
  * the synthetic generator of include/vx_synth.h re-implemented in numpy uint64 arithmetic;
  * fp64 inner products with numpy (X.astype(f64) @ Q.astype(f64).T) and the (score desc,
    id asc) order via np.lexsort;
  * ColBERT MaxSim sum_i max_j <q_i, d_j> in fp64 over bf16-rounded inputs;
  * hand-computed known-answer cases with exact ties.
Run:  python tests/golden/make_golden.py     (writes tests/golden/*.npz)
"""
from __future__ import annotations

from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def synth_int(seed: int, rows: np.ndarray, dim: int) -> np.ndarray:
    rows = np.asarray(rows, np.uint64)[:, None]
    cols = np.arange(dim, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15) + rows)
        h = splitmix64(h ^ (cols * np.uint64(0xD1B54A32D192ED03)))
    m = np.uint64(0xFFFF)
    s = ((h & m) + ((h >> np.uint64(16)) & m) + ((h >> np.uint64(32)) & m) + (h >> np.uint64(48)))
    return s.astype(np.int64) - 131070


def synth_rows(seed: int, row0: int, n: int, dim: int) -> np.ndarray:
    v = synth_int(seed, np.arange(row0, row0 + n), dim)
    ss = (v * v).sum(axis=1)
    nrm = np.sqrt(ss.astype(np.float64))
    return (v.astype(np.float64) / nrm[:, None]).astype(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))
    return (u >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, np.uint32) << 16).view(np.float32)


def topk_f64(X: np.ndarray, Q: np.ndarray, k: int):
    S = Q.astype(np.float64) @ X.astype(np.float64).T  # [B][N]
    ids = np.empty((Q.shape[0], k), np.int64)
    sc = np.empty((Q.shape[0], k), np.float64)
    for b in range(Q.shape[0]):
        order = np.lexsort((np.arange(X.shape[0]), -S[b]))[:k]
        ids[b], sc[b] = order, S[b, order]
    return ids, sc


def maxsim_f64(qtok_f32: np.ndarray, cand: np.ndarray, table_bits: np.ndarray) -> np.ndarray:
    qb = bf16_bits_to_f32(f32_to_bf16_bits(qtok_f32)).astype(np.float64)
    T = table_bits.shape[0]
    out = np.empty(cand.shape, np.float64)
    for b in range(cand.shape[0]):
        for c in range(cand.shape[1]):
            d = cand[b, c]
            if d < 0:
                out[b, c] = -np.inf
                continue
            D = bf16_bits_to_f32(table_bits[d % T]).astype(np.float64)
            out[b, c] = (qb[b] @ D.T).max(axis=1).sum()
    return out


def main() -> None:
    rng = np.random.default_rng(2511)
    # 1. generator known answers (first rows of the bench seeds)
    gen = {f"rows_s{s}_d{d}": synth_rows(s, r0, 4, d) for s, r0, d in
           [(42, 0, 768), (43, 0, 768), (42, 9_999_996, 1024), (45, 123456, 128)]}
    np.savez_compressed(HERE / "synth.npz", **gen)

    # 2. flat IP top-k on generator data (fp64 truth)
    for name, (N, D, B, k) in {"ip_small": (1000, 64, 5, 7), "ip_768": (3000, 768, 4, 10),
                               "ip_k100": (2500, 128, 3, 100)}.items():
        X = synth_rows(42, 0, N, D)
        Q = synth_rows(43, 0, B, D)
        ids, sc = topk_f64(X, Q, k)
        np.savez_compressed(HERE / f"{name}.npz", N=N, D=D, B=B, k=k, ids=ids, scores=sc)

    # 3. hand-computed ties: score desc then id asc
    X = np.array([[1, 0], [0, 1], [1, 0], [0.5, 0.5], [-1, 0], [1, 0]], np.float32)
    Q = np.array([[1, 0], [0, 1]], np.float32)
    # q0 scores: [1,0,1,.5,-1,1] -> ids 0,2,5 (ties by id), then 3
    # q1 scores: [0,1,0,.5,0,0]  -> ids 1,3, then 0,2,4,5 tie at 0 -> 0
    np.savez_compressed(HERE / "kat_ties.npz", X=X, Q=Q, k=4,
                        ids=np.array([[0, 2, 5, 3], [1, 3, 0, 2]], np.int64),
                        scores=np.array([[1, 1, 1, .5], [1, .5, 0, 0]], np.float64))

    # 4. MaxSim on a small token table (bf16), candidates with a skip (-1) and wraparound ids
    T, Nd, d, B, nq, Cc = 7, 16, 64, 3, 4, 5
    table = np.stack([f32_to_bf16_bits(synth_rows(45, b * Nd, Nd, d)) for b in range(T)])
    qtok = synth_rows(44, 0, B * nq, d).reshape(B, nq, d)
    cand = rng.integers(0, 50, size=(B, Cc)).astype(np.int64)
    cand[1, 2] = -1
    ms = maxsim_f64(qtok, cand, table)
    np.savez_compressed(HERE / "maxsim_small.npz", table=table, qtok=qtok, cand=cand, ms=ms)
    print("wrote", sorted(p.name for p in HERE.glob("*.npz")))


if __name__ == "__main__":
    main()
