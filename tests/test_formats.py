"""Store file and dataset formats: the raw block image of the reference
(BlockStore.save_image / load_image, ssd_model.py:84-101) and the page packers for embedding
tables and CSR graphs.  CPU tests pin the byte layout; the GPU tests run the kernels over packed
images loaded through AgileSystem.load_image."""

import json
import os

import numpy as np
import pytest

from oracle.pages import load_image as oracle_load_image
from paper_2504_19365_b200 import formats
from paper_2504_19365_b200.bench.dlrm import layout

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def test_read_image_matches_reference_blockstore_image():
    img = os.path.join(HERE, "golden", "store.img")   # written by the reference's BlockStore.save_image
    n = GOLD["image"]["num_blocks"]
    assert np.array_equal(formats.read_image(img, n), oracle_load_image(img, n))


def test_embedding_pack_layout_and_bytes(tmp_path):
    rng = np.random.default_rng(0)
    tables = [rng.standard_normal((r, 64)).astype(np.float32) for r in (100, 3, 17, 1000)]
    pages, man = formats.pack_embedding_tables(tables)
    key0, total = layout(np.array([t.shape[0] for t in tables]), 64)
    assert man["pages"] == total == pages.shape[0]
    assert np.array_equal(formats.table_keys(man), key0)
    rpp = man["rows_per_page"]
    for t, meta in zip(tables, man["tables"]):
        for r in (0, t.shape[0] - 1, t.shape[0] // 2):
            p, slot = meta["first_page"] + r // rpp, r % rpp
            row = pages[p].view(np.float32)[slot * 64:(slot + 1) * 64]
            assert np.array_equal(row, t[r])
    path = tmp_path / "emb.img"
    formats.write_image(path, pages, man)
    assert np.array_equal(formats.read_image(path), pages)
    assert formats.read_manifest(path) == man


def test_csr_pack_and_first_page_offset(tmp_path):
    rng = np.random.default_rng(1)
    V = 50
    deg = rng.integers(0, 60, size=V)
    row_ptr = np.concatenate([[0], np.cumsum(deg)])
    col = rng.integers(0, V, size=row_ptr[-1]).astype(np.int32)
    vals = rng.random(row_ptr[-1]).astype(np.float32)
    pages, man = formats.pack_csr(row_ptr, col, vals, first_page=3)
    cp = (col.size + 1023) // 1024
    assert man["col_key0"] == 3 and man["val_key0"] == 3 + cp and man["pages"] == 2 * cp
    assert np.array_equal(pages[:cp].reshape(-1).view(np.int32)[:col.size], col)
    assert np.array_equal(pages[cp:].reshape(-1).view(np.float32)[:col.size], vals)
    path = tmp_path / "g.img"
    formats.write_image(path, pages, man, row_ptr=row_ptr)
    img = formats.read_image(path)
    assert not img[:3].any() and np.array_equal(img[3:], pages)
    assert np.array_equal(np.load(str(path) + ".rowptr.npy"), row_ptr)
    with pytest.raises(ValueError):
        formats.pack_csr(row_ptr, np.full_like(col, V))


@pytest.mark.gpu
def test_gpu_embbag_over_packed_image(gpu_system, tmp_path):
    import torch
    rng = np.random.default_rng(2)
    tables = [rng.standard_normal((r, 128)).astype(np.float32) for r in (900, 40, 2500)]
    pages, man = formats.pack_embedding_tables(tables)
    path = tmp_path / "emb.img"
    formats.write_image(path, pages, man)
    s = gpu_system(cache_lines=128, ways=16, blocks=man["pages"], pairs=4, engine_warps=4, warps=2)
    s.load_image(0, path)
    B, L = 40, 20
    idx = np.stack([rng.integers(0, t.shape[0], size=(B, L)) for t in tables], axis=1).astype(np.int64)
    dev = torch.device("cuda", 0)
    out = torch.zeros((B, len(tables), 128), dtype=torch.float32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    s.embbag(torch.from_numpy(idx).to(dev), torch.from_numpy(formats.table_keys(man).view(np.int64)).to(dev),
             torch.tensor([t.shape[0] for t in tables], dtype=torch.int64, device=dev), out, cnt)
    s.sync(torch.cuda.current_stream(dev).cuda_stream)
    ref = np.stack([np.stack([tables[t][idx[b, t]].sum(axis=0, dtype=np.float32) for t in range(len(tables))])
                    for b in range(B)])
    assert np.max(np.abs(out.cpu().numpy() - ref) / np.maximum(np.abs(ref), 1.0)) < 1e-5
