"""GPU: torch.ops.agile.embedding_bag (paper_2504_19365_b200/ops.py, a torch.library custom op over
K5) against the row-keyed oracle, fixed pooling and variable-length bags."""

import numpy as np
import pytest
import torch

from oracle.embbag import embbag_offsets_reference, embbag_rows_reference
from paper_2504_19365_b200 import ops  # noqa: F401  (registers torch.ops.agile.embedding_bag)
from paper_2504_19365_b200.bench.dlrm import fill_rank_store, plan_shards

pytestmark = pytest.mark.gpu
SEED, D = 5, 128
DEV = torch.device("cuda", 0)


def _system(gpu_system, rows):
    plan = plan_shards(np.asarray(rows, dtype=np.int64), 1, D)
    descs, _, pages = plan.rank_layout(0)
    s = gpu_system(cache_lines=512, ways=32, blocks=max(pages, 64), pairs=8, sq_depth=256, cq_depth=256,
                   engine_warps=8, warps=4)
    fill_rank_store(s, plan, 0, SEED)
    k0 = torch.from_numpy(descs["key0"].view(np.int64).copy()).to(DEV)
    return s, k0, torch.tensor(rows, dtype=torch.int64, device=DEV)


def test_op_fixed_pooling(gpu_system):
    rows = [5000, 300, 9000]
    s, k0, rt = _system(gpu_system, rows)
    rng = np.random.default_rng(2)
    idx = np.stack([rng.integers(0, r, size=(40, 20)) for r in rows], axis=1).astype(np.int64)
    out = torch.ops.agile.embedding_bag(s.handle.value, torch.from_numpy(idx).to(DEV), None, k0, rt, D)
    s.sync()
    assert np.array_equal(out.cpu().numpy(), embbag_rows_reference(SEED, idx, D))


def test_op_variable_length_bags(gpu_system):
    rows = [4000, 70, 800]
    s, k0, rt = _system(gpu_system, rows)
    rng = np.random.default_rng(3)
    B, T = 17, 3
    lens = rng.integers(0, 70, size=B * T)
    lens[:2] = [0, 33]
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    flat = np.array([rng.integers(0, rows[i % T]) for i in range(B * T) for _ in range(lens[i])], dtype=np.int64)
    out = torch.ops.agile.embedding_bag(s.handle.value, torch.from_numpy(flat).to(DEV), torch.from_numpy(offs).to(DEV),
                                        k0, rt, D, 1)
    s.sync()
    assert np.array_equal(out.cpu().numpy(), embbag_offsets_reference(SEED, flat, offs, T, D))
