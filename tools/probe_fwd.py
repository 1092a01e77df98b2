"""Quick forward-throughput probe (development aid; bench.py is the contract)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import argparse
import math

import torch

import paper_2503_17924_b200 as wl
from paper_2503_17924_b200.attention import attn_forward, build_tiles


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=32768)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=32)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--cp", type=int, default=1)
    ap.add_argument("--batches", type=int, default=8)
    ap.add_argument("--single", action="store_true", help="one document of length T")
    args = ap.parse_args()
    dev = torch.device("cuda")
    spec = wl.SyntheticSpec(args.T, args.T)
    stream = wl.generate_synthetic_stream(spec, 0, args.batches)
    if args.single:
        stream = [[wl.Document(0, args.T)]]
    for bi, docs in enumerate(stream):
        lengths = [d.length for d in docs]
        plan = wl.build_shard_plan([lengths], args.cp, "per_document")
        gidx, pos, ro = plan.rank_local(0, 0)
        tl = pos.numel()
        q = torch.randn(tl, args.hq, args.d, device=dev, dtype=torch.bfloat16)
        k = torch.randn(args.T, args.hkv, args.d, device=dev, dtype=torch.bfloat16)
        v = torch.randn_like(k)
        tiles = build_tiles(ro, pos, lengths)
        pairs = int(plan.rank_pairs[0, 0])
        for _ in range(3):
            attn_forward(q, k, v, tiles)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10
        e0.record()
        for _ in range(n):
            attn_forward(q, k, v, tiles)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        flops = 4.0 * args.d * args.hq * pairs
        print(f"batch {bi}: docs={len(lengths)} maxdoc={max(lengths)} tiles={int(tiles.n_tiles.item())} "
              f"fwd {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
