"""GPU parity of the DLRM embedding-bag (K5) against the oracle: fp64 accumulation rounded once,
bit-exact (north_star allows 1e-5 relative; the synthetic rows make the sum exact, so 0 ulp is
required here)."""

import numpy as np
import pytest
import torch

from oracle.embbag import embbag_reference

pytestmark = pytest.mark.gpu


def _run(s, seed, T, rows, B, L, D, pd, rng, zipf=None):
    rpp = 4096 // (4 * D)
    pages = [(r + rpp - 1) // rpp for r in rows]
    k0 = np.concatenate([[0], np.cumsum(pages)[:-1]]).astype(np.uint64)
    if zipf:
        idx = np.stack([(rng.zipf(zipf, size=(B, L)) - 1) % rows[t] for t in range(T)], axis=1).astype(np.int64)
    else:
        idx = np.stack([rng.integers(0, rows[t], size=(B, L)) for t in range(T)], axis=1).astype(np.int64)
    dev = torch.device("cuda", 0)
    out = torch.full((B, T, D), float("nan"), dtype=torch.float32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    s.embbag(torch.from_numpy(idx).to(dev), torch.from_numpy(k0.view(np.int64)).to(dev),
             torch.tensor(rows, dtype=torch.int64, device=dev), out, cnt, prefetch_distance=pd)
    s.sync(torch.cuda.current_stream(dev).cuda_stream)
    ref = embbag_reference(seed, 0, k0, idx, D)
    o = out.cpu().numpy()
    assert np.array_equal(o, ref), "pooled vectors differ from the oracle"
    return float(np.max(np.abs(o - ref))), cnt.cpu().numpy()


@pytest.mark.parametrize("pd", [0, 1, 2])
@pytest.mark.parametrize("lines,ways", [(4096, 32), (512, 16), (256, 8)])
def test_embbag_matches_oracle(gpu_system, pd, lines, ways):
    s = gpu_system(cache_lines=lines, ways=ways, blocks=1 << 14, pairs=8, sq_depth=256, cq_depth=256,
                   engine_warps=8, warps=4)
    s.fill_store(0, seed=21, kind="f32")
    rng = np.random.default_rng(lines + pd)
    rows = [5000, 700, 12000, 64, 3000]
    err, cnt = _run(s, 21, len(rows), rows, 64, 20, 128, pd, rng)
    assert err < 1e-5
    assert cnt[0] == 64 * len(rows) * 20


def test_embbag_zipf_warm_cache_hits(gpu_system):
    s = gpu_system(cache_lines=1 << 16, ways=32, blocks=1 << 16, pairs=16, engine_warps=8, warps=4)
    s.fill_store(0, seed=3, kind="f32")
    rng = np.random.default_rng(9)
    rows = [100000] * 4
    err1, c1 = _run(s, 3, 4, rows, 256, 20, 128, 1, rng, zipf=1.05)
    err2, c2 = _run(s, 3, 4, rows, 256, 20, 128, 1, np.random.default_rng(9), zipf=1.05)
    assert err1 < 1e-5 and err2 < 1e-5
    assert c2[1] == 0          # same batch again: everything is resident
    assert c1[1] > 0


@pytest.mark.parametrize("D,L", [(64, 20), (32, 7), (128, 1), (128, 32)])
def test_embbag_shapes(gpu_system, D, L):
    s = gpu_system(cache_lines=1024, ways=16, blocks=1 << 13, pairs=4, engine_warps=4)
    s.fill_store(0, seed=8, kind="f32")
    err, _ = _run(s, 8, 3, [3000, 50, 999], 33, L, D, 1, np.random.default_rng(D + L))
    assert err < 1e-5


@pytest.mark.parametrize("pinned", [False, True])
def test_embbag_host_entry_matches_device_entry(gpu_system, pinned):
    # pageable output: staged + downloaded; pinned output: the kernel stores into it directly
    s = gpu_system(cache_lines=1024, ways=16, blocks=1 << 13, pairs=4, engine_warps=4)
    s.fill_store(0, seed=4, kind="f32")
    rng = np.random.default_rng(1)
    rows = np.array([4000, 4000], dtype=np.int64)
    idx = rng.integers(0, 4000, size=(16, 2, 20)).astype(np.int64)
    k0 = np.array([0, 500], dtype=np.uint64)
    o = torch.full((16, 2, 128), float("nan")).pin_memory().numpy() if pinned else None
    out, cnt = s.embbag_host(idx, k0, rows, 128, prefetch_distance=1, out=o)
    ref = embbag_reference(4, 0, k0, idx, 128)
    assert np.max(np.abs(out - ref) / np.maximum(np.abs(ref), 1)) < 1e-5
    assert int(cnt[0]) == 16 * 2 * 20


@pytest.mark.parametrize("user_ctas,pd", [(1, 0), (2, 3), (5, 0)])
def test_embbag_bounded_grid(gpu_system, user_ctas, pd):
    """A gather bounded to a few user CTAs (the async DLRM pipeline's side-stream launch) gives
    the same sums; tiny cache so bags see evictions while they are read."""
    s = gpu_system(cache_lines=128, ways=8, blocks=1 << 13, pairs=4, engine_warps=4, warps=2)
    s.fill_store(0, seed=12, kind="f32")
    rng = np.random.default_rng(user_ctas * 10 + pd)
    rows = [4000, 900, 2500]
    idx = np.stack([rng.integers(0, r, size=(96, 20)) for r in rows], axis=1).astype(np.int64)
    rpp = 8
    k0 = np.concatenate([[0], np.cumsum([(r + rpp - 1) // rpp for r in rows])[:-1]]).astype(np.uint64)
    dev = torch.device("cuda", 0)
    out = torch.full((96, 3, 128), float("nan"), dtype=torch.float32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    s.embbag(torch.from_numpy(idx).to(dev), torch.from_numpy(k0.view(np.int64)).to(dev),
             torch.tensor(rows, dtype=torch.int64, device=dev), out, cnt, prefetch_distance=pd,
             user_ctas=user_ctas)
    s.sync(torch.cuda.current_stream(dev).cuda_stream)
    ref = embbag_reference(12, 0, k0, idx, 128)
    o = out.cpu().numpy()
    assert np.max(np.abs(o - ref) / np.maximum(np.abs(ref), 1.0)) < 1e-5
    assert int(cnt.cpu()[0]) == 96 * 3 * 20


@pytest.mark.parametrize("user_ctas", [1, 3])
def test_embbag_prefetch_then_gather_all_hits(gpu_system, user_ctas):
    """Batch-level prefetch (AgileApi.prefetch, gpu_api.py:139-162) pulls every page of the batch
    into the cache; the gather that follows takes no miss path and matches the oracle."""
    s = gpu_system(cache_lines=4096, ways=32, blocks=1 << 13, pairs=8, engine_warps=8, warps=2)
    s.fill_store(0, seed=17, kind="f32")
    rng = np.random.default_rng(5 + user_ctas)
    rows = [6000, 1500, 800]
    idx = np.stack([rng.integers(0, r, size=(100, 20)) for r in rows], axis=1).astype(np.int64)
    k0 = np.concatenate([[0], np.cumsum([(r + 7) // 8 for r in rows])[:-1]]).astype(np.uint64)
    dev = torch.device("cuda", 0)
    di = torch.from_numpy(idx).to(dev)
    dk = torch.from_numpy(k0.view(np.int64)).to(dev)
    dr = torch.tensor(rows, dtype=torch.int64, device=dev)
    pc = torch.zeros(2, dtype=torch.int64, device=dev)
    s.embbag_prefetch(di, dk, dr, 128, pc, user_ctas=user_ctas)
    out = torch.full((100, 3, 128), float("nan"), dtype=torch.float32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    s.embbag(di, dk, dr, out, cnt, prefetch_distance=0)
    s.sync(torch.cuda.current_stream(dev).cuda_stream)
    assert int(pc.cpu()[0]) == 100 * 3 * 20
    assert int(cnt.cpu()[1]) == 0
    ref = embbag_reference(17, 0, k0, idx, 128)
    assert np.max(np.abs(out.cpu().numpy() - ref) / np.maximum(np.abs(ref), 1.0)) < 1e-5


def test_fused_launch_mode_matches(gpu_system, monkeypatch):
    """AGILE_LAUNCH=fused (one grid, roles by arrival ticket: the profiling mode) computes the same
    embedding-bag sums as the default split launch."""
    monkeypatch.setenv("AGILE_LAUNCH", "fused")
    s = gpu_system(cache_lines=512, ways=16, blocks=1 << 13, pairs=4, engine_warps=8, warps=2)
    s.fill_store(0, seed=23, kind="f32")
    err, cnt = _run(s, 23, 3, [3000, 700, 1200], 48, 20, 128, 0, np.random.default_rng(3))
    assert err < 1e-5
    assert cnt[0] == 48 * 3 * 20 and cnt[1] > 0


@pytest.mark.parametrize("pinned", [False, True])
def test_embbag_host_async_slots_match(gpu_system, pinned):
    """The pipelined host entry (two staging slots) gives the same sums as the one-call entry, with
    pageable output (device staging + download) and pinned output (the kernel stores into it)."""
    s = gpu_system(cache_lines=1024, ways=16, blocks=1 << 13, pairs=4, engine_warps=4)
    s.fill_store(0, seed=6, kind="f32")
    rng = np.random.default_rng(11)
    rows = np.array([4000, 2000], dtype=np.int64)
    k0 = np.array([0, 500], dtype=np.uint64)
    batches = [np.stack([rng.integers(0, r, size=(24, 20)) for r in rows], axis=1).astype(np.int64) for _ in range(5)]
    if pinned:
        outs = [torch.empty((24, 2, 128), dtype=torch.float32).pin_memory().numpy() for _ in range(2)]
    else:
        outs = [np.empty((24, 2, 128), dtype=np.float32) for _ in range(2)]
    cnts = [np.zeros(2, dtype=np.uint64) for _ in range(2)]
    got = []
    for k, b in enumerate(batches):
        slot = k % 2
        if k >= 2:
            s.embbag_host_wait(slot)
            got.append(outs[slot].copy())
        s.embbag_host_submit(b, k0, rows, 128, outs[slot], cnts[slot], slot)
    for k in (len(batches) - 2, len(batches) - 1):
        s.embbag_host_wait(k % 2)
        got.append(outs[k % 2].copy())
    for b, o in zip(batches, got):
        ref = embbag_reference(6, 0, k0, b, 128)
        assert np.max(np.abs(o - ref) / np.maximum(np.abs(ref), 1)) < 1e-5
    assert int(cnts[0][0] + cnts[1][0]) == 5 * 24 * 2 * 20


def test_side_infra_size_for_bounded_runs():
    """engine.side_warps / service.side_warps: bounded runs use a smaller infra grid (different
    queue ownership strides) interleaved with full runs on the same context; sums and counters
    stay exact."""
    from paper_2504_19365_b200 import AgileSystem
    from conftest import small_config
    cfg = small_config(cache_lines=256, ways=16, blocks=1 << 13, pairs=16, engine_warps=16, warps=8)
    cfg.engine.side_warps, cfg.service.side_warps = 4, 2
    with AgileSystem(cfg, device=0) as s2:
        s2.fill_store(0, seed=31, kind="f32")
        rng = np.random.default_rng(4)
        rows = [3000, 1200]
        k0 = np.array([0, 375], dtype=np.uint64)
        dev = torch.device("cuda", 0)
        for user_ctas in (2, 0, 3, 0):
            idx = np.stack([rng.integers(0, r, size=(64, 20)) for r in rows], axis=1).astype(np.int64)
            out = torch.full((64, 2, 128), float("nan"), dtype=torch.float32, device=dev)
            cnt = torch.zeros(2, dtype=torch.int64, device=dev)
            s2.embbag(torch.from_numpy(idx).to(dev), torch.from_numpy(k0.view(np.int64)).to(dev),
                      torch.tensor(rows, dtype=torch.int64, device=dev), out, cnt, prefetch_distance=0,
                      user_ctas=user_ctas)
            s2.sync(torch.cuda.current_stream(dev).cuda_stream)
            ref = embbag_reference(31, 0, k0, idx, 128)
            assert np.max(np.abs(out.cpu().numpy() - ref) / np.maximum(np.abs(ref), 1.0)) < 1e-5
            assert int(cnt.cpu()[0]) == 64 * 2 * 20
