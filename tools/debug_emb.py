import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np, torch
from conftest import small_config
from paper_2504_19365_b200 import AgileSystem
from oracle.embbag import embbag_reference
lines, ways, pd = [int(x) for x in sys.argv[1:4]]
s = AgileSystem(small_config(cache_lines=lines, ways=ways, blocks=1 << 14, pairs=8, engine_warps=8, warps=4), device=0)
s.fill_store(0, seed=21, kind="f32")
rng = np.random.default_rng(1)
rows = [5000, 700, 12000, 64, 3000]
T = len(rows); B = int(sys.argv[4]) if len(sys.argv) > 4 else 64; L = 20; D = 128
k0 = np.concatenate([[0], np.cumsum([(r + 7) // 8 for r in rows])[:-1]]).astype(np.uint64)
idx = np.stack([rng.integers(0, rows[t], size=(B, L)) for t in range(T)], axis=1).astype(np.int64)
dev = torch.device("cuda", 0)
out = torch.full((B, T, D), float("nan"), device=dev)
cnt = torch.zeros(2, dtype=torch.int64, device=dev)
s.embbag(torch.from_numpy(idx).to(dev), torch.from_numpy(k0.view(np.int64)).to(dev), torch.tensor(rows, device=dev), out, cnt, prefetch_distance=pd)
s.sync(torch.cuda.current_stream(dev).cuda_stream)
o = out.cpu().numpy(); ref = embbag_reference(21, 0, k0, idx, D)
bad = ~np.isclose(o, ref, rtol=1e-5, atol=1e-5)
print("nan bags", np.isnan(o).any(axis=2).sum(), "bad elems", bad.sum(), "counters", cnt.cpu().numpy(), s.stats())
bb = np.argwhere(bad.any(axis=2))[:10]
print("bad bags (b,t)", bb.tolist())
