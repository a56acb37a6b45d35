"""DLRM embedding-bag driver (BASELINE configs[1] and [4]; new workload — the reference's
ancestor is the synthetic gather of bench/sweeps.py:1-9, which "stands in for embedding lookups").

* 26 Criteo-shaped tables (Kaggle cardinalities scaled to a byte budget), dim 128, fp32 rows,
  8 rows per 4 KiB page, laid out contiguously in the emulated device's page store.
* Indices: bounded Zipf(alpha) ranks per table, optionally scattered over rows by a bijective
  multiplicative hash (hashed categorical ids), deterministic per (seed, batch).
* Table-wise sharding over G ranks, balanced by bytes (largest first); pooled outputs of a
  rank's tables are [B, T_g, D], i.e. already in the peer-major layout all_to_all_single
  splits along B.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# Criteo Kaggle categorical cardinalities (26 sparse features)
CRITEO_KAGGLE = (1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683, 8351593, 3194,
                 27, 14992, 5461306, 10, 5652, 2173, 4, 7046547, 18, 15, 286181, 105, 142572)


def table_rows(total_bytes: int, dim: int = 128, tables: int = 26) -> np.ndarray:
    """Row counts with the Criteo skew, scaled so the tables total ~total_bytes."""
    base = np.array([CRITEO_KAGGLE[i % len(CRITEO_KAGGLE)] for i in range(tables)], dtype=np.float64)
    scale = total_bytes / (base.sum() * dim * 4)
    return np.maximum(1, np.floor(base * scale)).astype(np.int64)


def layout(rows: np.ndarray, dim: int, dev: int = 0, first_page: int = 0):
    """Contiguous page ranges per table: returns (key0[T] uint64, total_pages)."""
    rpp = 4096 // (4 * dim)
    pages = (rows + rpp - 1) // rpp
    start = first_page + np.concatenate([[0], np.cumsum(pages)[:-1]])
    key0 = (np.uint64(dev) << np.uint64(36)) | start.astype(np.uint64)
    return key0, int(first_page + pages.sum())


def _scatter_mult(n: int) -> int:
    m = 2654435761 % n if n > 1 else 1
    while math.gcd(m, n) != 1:
        m += 1
    return m


def zipf_rows(rng: np.random.Generator, n: int, size, alpha: float, scatter: bool) -> np.ndarray:
    """Bounded Zipf over ranks 1..n (inverse-CDF of the continuous approximation), mapped to rows."""
    u = rng.random(size)
    if abs(alpha - 1.0) < 1e-9:
        r = np.exp(u * np.log(n + 1.0))
    else:
        a1 = 1.0 - alpha
        r = (1.0 + u * ((n + 1.0) ** a1 - 1.0)) ** (1.0 / a1)
    rank = np.clip(np.floor(r).astype(np.int64) - 1, 0, n - 1)
    if not scatter or n == 1:
        return rank
    return (rank * _scatter_mult(n) + 12345) % n


def make_batch(seed: int, step: int, rows: np.ndarray, B: int, L: int, alpha: float, scatter: bool,
               tables=None) -> np.ndarray:
    """int64 [B, len(tables), L]; table t's indices depend only on (seed, step, t), so every rank
    generates exactly its own tables' slice of the global batch."""
    tables = range(len(rows)) if tables is None else tables
    return np.stack([zipf_rows(np.random.default_rng([seed, step, int(t)]), int(rows[t]), (B, L), alpha, scatter)
                     for t in tables], axis=1)


def shard_tables(rows: np.ndarray, G: int):
    """Table-wise assignment balanced by bytes (largest first onto the lightest rank)."""
    load = [0] * G
    owner = np.zeros(len(rows), dtype=np.int64)
    for t in np.argsort(-rows, kind="stable"):
        g = int(np.argmin(load))
        owner[t] = g
        load[g] += int(rows[t])
    return [np.nonzero(owner == g)[0] for g in range(G)], owner


@dataclass
class DlrmShard:
    """One rank's share: its tables, their rows and page keys in the rank's own store."""
    tables: np.ndarray
    rows: np.ndarray
    key0: np.ndarray
    pages: int


def build_shard(all_rows: np.ndarray, tables: np.ndarray, dim: int) -> DlrmShard:
    rows = all_rows[tables]
    key0, pages = layout(rows, dim)
    return DlrmShard(tables=tables, rows=rows, key0=key0, pages=pages)
