"""On-disk and dataset formats of the page store.

The store file is the reference's raw block image (``BlockStore.save_image`` / ``load_image``,
ssd_model.py:84-101): block b occupies bytes [b * 4096, (b + 1) * 4096), little-endian, a short
tail is zero-padded.  ``AgileSystem.load_image(dev, path)`` / ``agile_store_attach`` map such a
file into the GPU-visible host store.  The packers below lay workload data out in it:

* embedding tables (DLRM): table t's rows packed ``4096 // (4 * dim)`` per page, tables in
  contiguous page ranges in table order — the layout ``bench.dlrm.layout`` and the embedding-bag
  kernel (K5) address (key of a row = table first page + row // rows_per_page);
* CSR graphs (BFS / SpMV): ``col_idx`` (int32) paged 1,024 entries per page from page 0, then the
  optional ``vals`` (fp32) from the next page — the layout of K6/K7 (``col_key0``, ``val_key0``);
  ``row_ptr`` stays in HBM and is stored beside the image.

Each packer returns a manifest (JSON-serialisable) with what a later run needs to address the
data; ``write_image`` writes the image plus ``<path>.json``.
"""

from __future__ import annotations

import json
import os

import numpy as np

BLOCK = 4096
ENTRIES_PER_PAGE = BLOCK // 4


def rows_per_page(dim: int) -> int:
    if dim <= 0 or (BLOCK // 4) % dim:
        raise ValueError("dim must divide 1024 (whole rows per 4 KiB page)")
    return BLOCK // (4 * dim)


def pack_embedding_tables(tables, first_page: int = 0):
    """tables: list of fp32 arrays [rows_t, dim] -> (pages uint8 [n, 4096], manifest)."""
    tables = [np.ascontiguousarray(t, dtype=np.float32) for t in tables]
    if not tables:
        raise ValueError("no tables")
    dim = tables[0].shape[1]
    if any(t.ndim != 2 or t.shape[1] != dim for t in tables):
        raise ValueError("every table must be [rows, dim] with the same dim")
    rpp = rows_per_page(dim)
    npages = [(t.shape[0] + rpp - 1) // rpp for t in tables]
    start = first_page + np.concatenate([[0], np.cumsum(npages)[:-1]]).astype(np.int64)
    total = int(sum(npages))
    pages = np.zeros((total, BLOCK), dtype=np.uint8)
    flat = pages.view(np.float32).reshape(total * rpp, dim)
    for t, s in zip(tables, start):
        r0 = (int(s) - first_page) * rpp
        flat[r0:r0 + t.shape[0]] = t
    manifest = {"kind": "embedding_tables", "dim": int(dim), "rows_per_page": rpp, "first_page": first_page,
                "pages": total, "tables": [{"rows": int(t.shape[0]), "first_page": int(s)}
                                           for t, s in zip(tables, start)]}
    return pages, manifest


def table_keys(manifest, dev: int = 0) -> np.ndarray:
    """Per-table page key (dev << 36 | first page) for ``AgileSystem.embbag``."""
    return np.array([(dev << 36) | t["first_page"] for t in manifest["tables"]], dtype=np.uint64)


def pack_csr(row_ptr, col_idx, vals=None, first_page: int = 0):
    """CSR -> (pages uint8 [n, 4096], manifest); col_idx int32 paged from first_page, vals fp32
    (optional) from the page after the last col page.  row_ptr is kept in the manifest's sidecar
    (it lives in HBM at run time)."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
    E = col_idx.size
    if row_ptr.ndim != 1 or row_ptr[0] != 0 or row_ptr[-1] != E or np.any(np.diff(row_ptr) < 0):
        raise ValueError("row_ptr must be non-decreasing from 0 to len(col_idx)")
    if E and (col_idx.min() < 0 or col_idx.max() >= row_ptr.size - 1):
        raise ValueError("col_idx entries must be vertex ids in [0, V)")
    cp = (E + ENTRIES_PER_PAGE - 1) // ENTRIES_PER_PAGE
    vp = 0 if vals is None else cp
    pages = np.zeros((cp + vp, BLOCK), dtype=np.uint8)
    pages[:cp].reshape(-1).view(np.int32)[:E] = col_idx
    if vals is not None:
        vals = np.ascontiguousarray(vals, dtype=np.float32)
        if vals.size != E:
            raise ValueError("vals must have one weight per edge")
        pages[cp:].reshape(-1).view(np.float32)[:E] = vals
    manifest = {"kind": "csr", "vertices": int(row_ptr.size - 1), "edges": int(E), "first_page": first_page,
                "col_key0": first_page, "val_key0": None if vals is None else first_page + cp,
                "pages": int(cp + vp)}
    return pages, manifest


def write_image(path, pages: np.ndarray, manifest: dict, row_ptr=None) -> None:
    """Raw block image (ssd_model.py:97-101 layout) + ``<path>.json`` manifest (+ ``<path>.rowptr.npy``)."""
    pages = np.ascontiguousarray(pages, dtype=np.uint8).reshape(-1, BLOCK)
    first = int(manifest.get("first_page", 0))
    with open(path, "wb") as fh:
        if first:
            fh.write(bytes(first * BLOCK))
        fh.write(pages.tobytes())
    with open(str(path) + ".json", "w") as fh:
        json.dump(manifest, fh)
    if row_ptr is not None:
        np.save(str(path) + ".rowptr.npy", np.ascontiguousarray(row_ptr, dtype=np.int64))


def read_image(path, num_blocks: int | None = None) -> np.ndarray:
    """Blocks of a raw image; a short tail (and blocks past the end) read as zeros
    (BlockStore.load_image, ssd_model.py:84-95)."""
    size = os.path.getsize(path)
    n = num_blocks if num_blocks is not None else (size + BLOCK - 1) // BLOCK
    out = np.zeros((n, BLOCK), dtype=np.uint8)
    raw = np.fromfile(path, dtype=np.uint8, count=min(size, n * BLOCK))
    out.reshape(-1)[:raw.size] = raw
    return out


def read_manifest(path) -> dict:
    with open(str(path) + ".json") as fh:
        return json.load(fh)
