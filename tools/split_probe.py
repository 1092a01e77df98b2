"""Cost of running the attention in G head-group launches (the CP exchange's
head-group pipeline) instead of one launch, on one GPU with no exchange:
interleaved repetitions of fwd+bwd over the same rank workload.

    python tools/split_probe.py [--cp 4] [--seq 0] [--groups 1 2 4 8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200.attention import (attn_backward, attn_forward, bwd_workspace,  # noqa: E402
                                             build_tiles, head_groups)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--window", type=int, default=131072)
    ap.add_argument("--cp", type=int, default=4)
    ap.add_argument("--seq", type=int, nargs="+", default=[0, 2, 3])
    ap.add_argument("--groups", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--reps", type=int, default=4)
    a = ap.parse_args()
    dev = torch.device("cuda")
    spec = wl.SyntheticSpec(context_window=a.window, tokens_per_global_batch=a.window)
    stream = wl.generate_synthetic_stream(spec, 0, max(a.seq) + 1)
    hq = hkv = 32
    d = 128
    for si in a.seq:
        lengths = [x.length for x in stream[si]]
        plan = wl.build_shard_plan([lengths], a.cp, "measured")
        g, pos, ro = plan.rank_local(0, 0)
        tiles = build_tiles(ro, pos, lengths)
        T, tl = sum(lengths), g.numel()
        q = torch.randn(tl, hq, d, device=dev, dtype=torch.bfloat16)
        do = torch.randn_like(q)
        k = torch.randn(T, hkv, d, device=dev, dtype=torch.bfloat16)
        v = torch.randn_like(k)
        dk = torch.empty((T, hkv, d), dtype=torch.float32, device=dev)
        dv = torch.empty_like(dk)

        def run(G):
            grps = head_groups(hkv, G)
            o = lse = None
            for grp in grps:
                o, lse = attn_forward(q, k, v, tiles, kv_heads=grp, out=None if o is None else (o, lse))
            dq, ws = torch.empty_like(q), bwd_workspace(q, k, tiles)
            for grp in grps:
                attn_backward(q, k, v, o, lse, do, tiles, dk_out=dk, dv_out=dv, covered_only=True,
                              kv_heads=grp, dq_out=dq, ws=ws)

        res = {G: [] for G in a.groups}
        for G in a.groups:
            run(G)
        for _ in range(a.reps):
            for G in a.groups:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run(G)
                e1.record()
                e1.synchronize()
                res[G].append(e0.elapsed_time(e1))
        best = {G: min(v_) for G, v_ in res.items()}
        print(json.dumps({"seq": si, "docs": len(lengths), "cp": a.cp, "rank": 0,
                          "ms": {G: round(x, 3) for G, x in best.items()},
                          "split_cost": {G: round(best[G] / best[a.groups[0]] - 1, 4)
                                         for G in a.groups}}), flush=True)


if __name__ == "__main__":
    main()
