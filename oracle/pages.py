"""Synthetic page contents and the raw block-image format (oracle; test infrastructure only).

Page model: reference ``BlockStore`` (ssd_model.py:61-101) — fixed 4 KiB blocks, unwritten
blocks read as zeros, raw image offset = blk * block_size, little-endian, short tail zero-padded.
Synthetic fill: u64 word k of block b on device d is splitmix64(seed ^ d<<56 ^ b<<9 ^ k); the GPU
fill kernel (agile_b200.cu fill_store_kernel) computes the same function.
"""

from __future__ import annotations

import numpy as np

BLOCK = 4096
_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def page_words(seed: int, dev: int, blks) -> np.ndarray:
    """uint64 [len(blks), 512] synthetic contents of the given blocks."""
    b = np.asarray(blks, dtype=np.uint64).reshape(-1, 1)
    k = np.arange(512, dtype=np.uint64).reshape(1, -1)
    x = np.uint64(seed) ^ (np.uint64(dev) << np.uint64(56)) ^ (b << np.uint64(9)) ^ k
    return splitmix64(x)


def page_bytes(seed: int, dev: int, blks) -> np.ndarray:
    return page_words(seed, dev, blks).view(np.uint8).reshape(-1, BLOCK)


def page_floats(seed: int, dev: int, blks) -> np.ndarray:
    """float32 [n, 1024]: each 32-bit half h of a page word maps to (h >> 8) * 2^-23 - 1
    (exact in fp32; the DLRM tables are built from these pages)."""
    u = page_words(seed, dev, blks).view(np.uint32)
    return ((u >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)).astype(np.float32)


def row_floats(seed: int, table: int, rows, D: int) -> np.ndarray:
    """float32 [len(rows), D]: embedding rows keyed by (table, global row) — u64 word k of row r
    is splitmix64(seed ^ table<<56 ^ r<<8 ^ k), each 32-bit half h stored as (h >> 8) * 2^-23 - 1
    (agile_b200.cu fill_rows_kernel).  A row-wise shard of a table holds these same values."""
    r = np.asarray(rows, dtype=np.uint64).reshape(-1, 1)
    k = np.arange(D // 2, dtype=np.uint64).reshape(1, -1)
    x = np.uint64(seed) ^ (np.uint64(table) << np.uint64(56)) ^ (r << np.uint64(8)) ^ k
    u = splitmix64(x).view(np.uint32).reshape(len(r), D)
    return ((u >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)).astype(np.float32)


def load_image(path, num_blocks: int) -> np.ndarray:
    """BlockStore.load_image (ssd_model.py:84-95): blocks past the file are zero."""
    out = np.zeros((num_blocks, BLOCK), dtype=np.uint8)
    data = np.fromfile(path, dtype=np.uint8)[: num_blocks * BLOCK]
    out.reshape(-1)[: len(data)] = data
    return out


def save_image(path, blocks: dict, block_size: int = BLOCK) -> None:
    """BlockStore.save_image (ssd_model.py:97-101): top = max written block + 1."""
    top = max(blocks, default=-1) + 1
    with open(path, "wb") as fh:
        for b in range(top):
            fh.write(blocks.get(b, bytes(block_size)))
