"""Profiling probe: fwd + bwd on one synthetic sequence (development aid)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200.attention import attn_backward, attn_forward, build_tiles  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=32768)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=32)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--single", action="store_true")
ap.add_argument("--doc", type=int, default=0, help="uniform documents of this length")
ap.add_argument("--v3-min-rows", type=int, default=-1, help="backward kernel selection threshold")
ap.add_argument("--pairs", type=int, default=-1, help="v3 backward as 2-CTA clusters (1/0)")
a = ap.parse_args()
from paper_2503_17924_b200.attention import set_bwd_pairs, set_bwd_v3_min_rows  # noqa: E402
set_bwd_v3_min_rows(a.v3_min_rows)
set_bwd_pairs(a.pairs)
lengths = [d.length for d in wl.generate_synthetic_stream(wl.SyntheticSpec(a.T, a.T), 0, a.batch + 1)[a.batch]]
if a.single:
    lengths = [a.T]
if a.doc:
    lengths = [a.doc] * (a.T // a.doc)
plan = wl.build_shard_plan([lengths], 1, "per_document")
g, pos, ro = plan.rank_local(0, 0)
tiles = build_tiles(ro, pos, lengths)
dev = torch.device("cuda")
q = torch.randn(a.T, a.hq, a.d, device=dev, dtype=torch.bfloat16)
k = torch.randn(a.T, a.hkv, a.d, device=dev, dtype=torch.bfloat16)
v = torch.randn_like(k)
do = torch.randn_like(q)
pairs = sum(x * (x + 1) // 2 for x in lengths)
fs, bs = [], []
for it in range(a.iters):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    o, lse = attn_forward(q, k, v, tiles)
    e[1].record()
    dq, dk, dv = attn_backward(q, k, v, o, lse, do, tiles)
    e[2].record()
    torch.cuda.synchronize()
    fs.append(e[0].elapsed_time(e[1]))
    bs.append(e[1].elapsed_time(e[2]))
f, b = sorted(fs)[len(fs) // 2], sorted(bs)[len(bs) // 2]
print(f"docs={len(lengths)} maxdoc={max(lengths)} median of {a.iters}: fwd {f:.3f} ms "
      f"{4*a.d*a.hq*pairs/f/1e9:.0f} TF/s | bwd {b:.3f} ms {10*a.d*a.hq*pairs/b/1e9:.0f} TF/s "
      f"(min {min(bs):.3f} max {max(bs):.3f})")
