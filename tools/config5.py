"""BASELINE config 5: 64 micro-batches packed by the W(d) packer with outlier
delay queues, padded for CP=8, per-seq / per-doc selection by the measured
tile model (one batched GPU launch; the reference CostProfile's choices are
reported beside it), then CP=8 attention fwd+bwd for a sample of the packed
micro-batches, each rank replayed on this GPU (exact per-rank kernel time,
the backward as the CP pipeline runs it: covered dK/dV partial rows only).

    python tools/config5.py --iters 2 --sample 6 --out r.json
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_17924_b200 as wl
from paper_2503_17924_b200.attention import attn_backward, attn_forward, build_tiles


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--sample", type=int, default=6)
    ap.add_argument("--cp", type=int, default=8)
    ap.add_argument("--policy", default="measured", choices=["measured", "adaptive"])
    ap.add_argument("--bwd-persistent", type=int, default=-1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from paper_2503_17924_b200.attention import set_bwd_persistent
    if a.bwd_persistent >= 0:
        set_bwd_persistent(a.bwd_persistent)
    dev = torch.device("cuda")
    prof = wl.CostProfile()
    spec = wl.SyntheticSpec(context_window=131072, tokens_per_global_batch=64 * 131072)
    stream = wl.generate_synthetic_stream(spec, seed=0, n_batches=a.iters)
    packer = wl.HeuristicPacker(wl.OutlierQueueSet((32768, 98304)), 64, 163840, prof)
    filler = wl._FillerIds()
    hq, hkv, d = 32, 32, 128
    rows = []
    for it, batch in enumerate(stream):
        t0 = time.perf_counter()
        plan_h = packer.feed(batch, it)
        pack_ms = (time.perf_counter() - t0) * 1e3
        mbs = [wl.pad_for_cp(mb, a.cp, filler, it) for mb in plan_h.microbatches if mb.docs]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        model = wl.TileModel.for_shape(hq, hkv, d)
        plan = wl.build_shard_plan(mbs, a.cp, a.policy, prof,    # ONE launch, 64 micro-batches
                                   model=model if a.policy == "measured" else None)
        e1.record()
        torch.cuda.synchronize()
        plan_ms = e0.elapsed_time(e1)
        choices = [plan.strategy(b).value for b in range(plan.n_mb)]
        ref = wl.build_shard_plan(mbs, a.cp, "adaptive", prof, with_tokens=False)
        ref_choices = [ref.strategy(b).value for b in range(plan.n_mb)]
        rec = {"iteration": it, "docs": len(batch), "microbatches": plan.n_mb, "pack_ms": round(pack_ms, 2),
               "plan_ms_gpu": round(plan_ms, 3), "policy": a.policy,
               "per_document_chosen": choices.count("per_document"),
               "reference_profile_per_document": ref_choices.count("per_document"),
               "imbalance_degree_attention": round(wl.imbalance_degree_attention(plan_h.microbatches), 4),
               "carried": len(plan_h.carried_over), "sample": []}
        # heaviest micro-batches first
        order = sorted(range(plan.n_mb), key=lambda b: -sum(x * (x + 1) // 2 for x in plan.lengths[b]))
        for b in order[:a.sample]:
            lengths = plan.lengths[b]
            T = sum(lengths)
            q_full = torch.randn(T, hq, d, device=dev, dtype=torch.bfloat16)
            k = torch.randn(T, hkv, d, device=dev, dtype=torch.bfloat16)
            v = torch.randn_like(k)
            times = []
            for r in range(a.cp):
                g, pos, ro = plan.rank_local(b, r)
                q = q_full[g.long()]
                tiles = build_tiles(ro, pos, lengths)
                o, lse = attn_forward(q, k, v, tiles)
                attn_backward(q, k, v, o, lse, q, tiles, covered_only=True)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                o, lse = attn_forward(q, k, v, tiles)
                attn_backward(q, k, v, o, lse, q, tiles, covered_only=True)
                e.record()
                e.synchronize()
                times.append(s.elapsed_time(e))
            pairs = sum(x * (x + 1) // 2 for x in lengths)
            mx = max(times)
            rec["sample"].append({"mb": b, "tokens": T, "docs": len(lengths), "strategy": choices[b],
                                  "imbalance": round(mx / (sum(times) / len(times)), 4),
                                  "tflops_per_gpu": round(14 * d * hq * pairs / a.cp / (mx / 1e3) / 1e12, 1)})
            del q_full, k, v
        print(json.dumps(rec), flush=True)
        rows.append(rec)
    if a.out:
        json.dump(rows, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
