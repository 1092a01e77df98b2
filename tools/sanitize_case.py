"""Small cases of every device entry point, for compute-sanitizer runs
(tools/sanitize.sh): shard plan (reference + measured policies), tile lists,
forward, both backward kernels (D = 128 v2 / v3, D = 64), bf16 partials,
the one-GPU CP exchange (covered and full push / pull) and QKV RoPE."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200.attention import (attn_backward, attn_forward, build_tiles,  # noqa: E402
                                             qkv_rope, set_bwd_v3_min_rows)
from paper_2503_17924_b200.cp import LocalPeersExchange, shard_for_rank  # noqa: E402


def main():
    dev = torch.device("cuda")
    torch.manual_seed(0)
    cp = 2
    lengths = [300, 17, 1, 200, 130]
    plan = wl.build_shard_plan([lengths, [512, 128]], cp, "adaptive")
    wl.build_shard_plan([lengths, [512, 128]], cp, "measured")
    T = sum(lengths)
    for d, hq, hkv in ((128, 4, 2), (64, 4, 4)):
        q = torch.randn(T, hq, d, device=dev, dtype=torch.bfloat16)
        k = torch.randn(T, hkv, d, device=dev, dtype=torch.bfloat16)
        v = torch.randn_like(k)
        for w in range(cp):
            g, pos, ro = plan.rank_local(0, w)
            ql = q[g.long()].contiguous()
            tiles = build_tiles(ro, pos, lengths)
            o, lse = attn_forward(ql, k, v, tiles)
            for v3 in ((0, 1 << 30) if d == 128 else (1 << 30,)):
                prev = set_bwd_v3_min_rows(v3)
                attn_backward(ql, k, v, o, lse, ql, tiles)
                dkb = torch.empty(T, hkv, d, device=dev, dtype=torch.bfloat16)
                attn_backward(ql, k, v, o, lse, ql, tiles, dk_out=dkb, dv_out=torch.empty_like(dkb))
                set_bwd_v3_min_rows(prev)
        torch.cuda.synchronize()
    # one-GPU CP exchange
    hq, hkv, d = 4, 2, 128
    sh = [shard_for_rank(plan, 0, r) for r in range(cp)]
    for covered in (True, False):
        ex = LocalPeersExchange.create(cp, T, hkv, d, dev)
        for e in ex:
            e.push_covered = e.pull_covered = covered
        q = torch.randn(T, hq, d, device=dev, dtype=torch.bfloat16)
        k = torch.randn(T, hkv, d, device=dev, dtype=torch.bfloat16)
        v = torch.randn_like(k)
        full = [ex[r].gather(k[sh[r].gather_local.long()].contiguous(),
                             v[sh[r].gather_local.long()].contiguous(), sh[r], 0) for r in range(cp)]
        parts = []
        for r in range(cp):
            ql = q[sh[r].gather_local.long()].contiguous()
            o, lse = attn_forward(ql, full[r][0], full[r][1], sh[r].tiles)
            dko, dvo = ex[r].dkv_out(sh[r], 0, torch.cuda.current_stream())
            parts.append(attn_backward(ql, full[r][0], full[r][1], o, lse, ql, sh[r].tiles,
                                       dk_out=dko, dv_out=dvo))
        for r in range(cp):
            ex[r].scatter(parts[r][1], parts[r][2], sh[r], 0)
    y = torch.randn(T // cp, (hq + 2 * hkv) * d, device=dev, dtype=torch.bfloat16)
    qkv_rope(y, sh[0].tiles.positions, hq, hkv, d)
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
