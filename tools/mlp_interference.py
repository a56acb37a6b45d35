"""Which part of a side-stream AGILE run slows the DLRM MLPs beside it? (GPU-box tool)

MLP graph alone vs beside: (a) bounded all-hit gathers (HBM reads only, no link traffic),
(b) bounded batch prefetches of fresh batches (link + page fills), (c) a bounded gather whose
users spin on a stalled... (idle infra: a launch with no user work)."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_2504_19365_b200.bench.dlrm import gpu_zipf_batch, DlrmModel, mlp_graph_ms
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
from pipe_probe import make, B, T, L, D

dev = torch.device("cuda", 0)
os.environ.setdefault("SIDE", "")
s, rows_np, key0, rows = make(16, 64, 128, 48)
gen = torch.Generator(device=dev).manual_seed(1)
out = torch.zeros((B, T, D), dtype=torch.float32, device=dev)
cnt = torch.zeros(2, dtype=torch.int64, device=dev)
for _ in range(80):
    s.embbag(gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev), key0, rows, out, cnt, prefetch_distance=0)
s.sync(torch.cuda.current_stream(dev).cuda_stream)
model = DlrmModel(dev, D, T)
dense = torch.randn(B, 13, device=dev, dtype=torch.bfloat16)
CARVE = int(os.environ.get("CARVE", "32"))
g = model.capture(dense, out, 40, sm_carveout=CARVE)
main = torch.cuda.current_stream(dev)
side = torch.cuda.Stream(dev, priority=-1)


def mlp_beside(side_fn, n=4):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(side):
        side_fn()
    a.record(main)
    for _ in range(n):
        g.replay()
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


hitbat = gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev)
s.embbag(hitbat, key0, rows, out, cnt, prefetch_distance=0)
res = {"alone": mlp_beside(lambda: None)}
res["beside_hit_gathers_16ctas"] = mlp_beside(lambda: [s.embbag(hitbat, key0, rows, out, cnt, prefetch_distance=0,
                                                                  user_ctas=16, stream=side.cuda_stream) for _ in range(60)])
fresh = [gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev) for _ in range(8)]
res["beside_prefetch_16ctas"] = mlp_beside(lambda: [s.embbag_prefetch(x, key0, rows, D, cnt, 16, stream=side.cuda_stream)
                                                    for x in fresh])
res["alone_again"] = mlp_beside(lambda: None)
# the host link loaded by the copy engines only (no SM work beside the MLPs): pinned H2D copies
pin = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
dst = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
res["beside_h2d_copies"] = mlp_beside(lambda: [dst.copy_(pin, non_blocking=True) for _ in range(12)])
res["carveout"] = CARVE
res["side"] = os.environ.get("SIDE")
# a side launch of idle CTAs only (the infra grid of a run with one user CTA that has no work)
empty = torch.zeros((1, T, L), dtype=torch.int64, device=dev)
res["beside_1user_empty_runs"] = mlp_beside(lambda: [s.embbag(empty, key0, rows, out[:1], cnt, prefetch_distance=0,
                                                             user_ctas=1, stream=side.cuda_stream) for _ in range(400)])
print(json.dumps(res))
s.close()
