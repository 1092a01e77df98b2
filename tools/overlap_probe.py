"""Exposed CP exchange of ONE micro-batch (the verdict's intra-micro-batch
overlap metric), under torchrun on N GPUs:

    torchrun --nproc-per-node 4 tools/overlap_probe.py [--window 131072] [--seq 0]

Per rank, with CUDA events (max over ranks):
  attn   : forward + backward kernels alone on pre-gathered K/V (no exchange)
  step_G : cp_doc_attention forward + backward through the symmetric exchange
           with G head groups (per-peer arrival flags), G in --groups
  nccl   : cp_doc_attention through NCCL all-gather / reduce-scatter
exposed = (step - attn) / step.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200.attention import (attn_backward, attn_forward, bwd_workspace, set_bwd_reserve_sms,  # noqa: E402
                                             head_groups)
from paper_2503_17924_b200.cp import SymmExchange, cp_doc_attention, shard_for_rank  # noqa: E402


def timed_interleaved(fns, reps):
    """min over `reps` rounds of each fn's time, the fns alternating inside a
    round (GPU clocks drift by several % over a run under the power cap, so
    back-to-back blocks of one fn would bias the comparison); max over ranks."""
    for fn in fns.values():
        fn()
    best = {k: float("inf") for k in fns}
    for _ in range(reps):
        for k, fn in fns.items():
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            best[k] = min(best[k], a.elapsed_time(b))
    out = {}
    for k, v in best.items():
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[k] = float(t)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--window", type=int, default=131072)
    ap.add_argument("--seq", type=int, default=0)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=32)
    ap.add_argument("--groups", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--reserve", type=int, nargs="+", default=[0],
                    help="SMs the persistent backward leaves to the exchange (set_bwd_reserve_sms)")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    spec = wl.SyntheticSpec(context_window=a.window, tokens_per_global_batch=a.window)
    lengths = [d.length for d in wl.generate_synthetic_stream(spec, 0, a.seq + 1)[a.seq]]
    d = 128
    plan = wl.build_shard_plan([lengths], world, "measured",
                               model=wl.TileModel.for_shape(a.hq, a.hkv, d))
    sh = shard_for_rank(plan, 0, rank)
    T, tl = sum(lengths), sum(lengths) // world
    g = torch.Generator(device=dev).manual_seed(rank)
    mk = lambda h: torch.randn((tl, h, d), generator=g, device=dev, dtype=torch.bfloat16)
    q, k, v, do = mk(a.hq), mk(a.hkv), mk(a.hkv), mk(a.hq)
    kf = torch.randn((T, a.hkv, d), generator=g, device=dev, dtype=torch.bfloat16)
    vf = torch.randn_like(kf)

    def attn_only():
        o, lse = attn_forward(q, kf, vf, sh.tiles)
        attn_backward(q, kf, vf, o, lse, do, sh.tiles, covered_only=True)

    res = {"world": world, "window": a.window, "seq": a.seq, "docs": len(lengths),
           "strategy": sh.strategy.value, "heads": [a.hq, a.hkv]}
    fns = {"attn": attn_only}
    exchanges = []
    for G in a.groups:
        grps = head_groups(a.hkv, G)

        def attn_groups(grps=grps):
            # the same kernels split into G head-group launches, no exchange
            o = lse = None
            for grp in grps:
                o, lse = attn_forward(q, kf, vf, sh.tiles, kv_heads=grp,
                                      out=None if o is None else (o, lse))
            dq, ws = torch.empty_like(q), bwd_workspace(q, kf, sh.tiles)
            dk = torch.empty((T, a.hkv, d), dtype=torch.float32, device=dev)
            dv = torch.empty_like(dk)
            for grp in grps:
                attn_backward(q, kf, vf, o, lse, do, sh.tiles, dk_out=dk, dv_out=dv,
                              covered_only=True, kv_heads=grp, dq_out=dq, ws=ws)

        ex = SymmExchange(dist.group.WORLD, T, a.hkv, d, dev, groups=G)
        exchanges.append(ex)

        def step(ex=ex, r=0):
            prev = set_bwd_reserve_sms(r)
            qq, kk, vv = (x.detach().requires_grad_(True) for x in (q, k, v))
            o = cp_doc_attention(qq, kk, vv, sh, exchange=ex)
            o.backward(do)
            set_bwd_reserve_sms(prev)

        fns[f"attn_g{G}"] = attn_groups
        for r in a.reserve:
            fns[f"step_g{G}" + (f"_r{r}" if r else "")] = (lambda ex=ex, r=r: step(ex, r))

    def nccl_step():
        qq, kk, vv = (x.detach().requires_grad_(True) for x in (q, k, v))
        o = cp_doc_attention(qq, kk, vv, sh)
        o.backward(do)

    fns["nccl"] = nccl_step
    ms = timed_interleaved(fns, a.reps)
    res["ms"] = {k: round(v, 3) for k, v in ms.items()}
    for G in a.groups:
        for r in a.reserve:
            if r:
                res[f"exposed_g{G}_r{r}"] = round(1 - ms["attn"] / ms[f"step_g{G}_r{r}"], 4)
        if f"step_g{G}" not in ms:
            continue
        res[f"exposed_g{G}"] = round(1 - ms["attn"] / ms[f"step_g{G}"], 4)
        res[f"exposed_vs_split_g{G}"] = round(1 - ms[f"attn_g{G}"] / ms[f"step_g{G}"], 4)
    res["exposed_nccl"] = round(1 - ms["attn"] / ms["nccl"], 4)
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
