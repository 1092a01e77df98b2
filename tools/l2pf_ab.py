"""A/B of persistent 128-query backward switches, interleaved on the same
inputs: uniform documents of several lengths and the bench's 8 synthetic 32K
sequences (CP=1).  --knob l2pf: L2 prefetch of the next unit
(`set_bwd_l2_prefetch` 0 vs 1).  (Knobs "defer" and "qfirst" timed two
removed unit-boundary variants: profiles/r02_bwd3_unit_boundary_trace.txt.)  (--knob red timed a hybrid dQ drain, RED.v4
for --value of the 4 rounds, since removed: profiles/r02_ab_bwd3_hybrid_drain.txt.)

    python tools/l2pf_ab.py [--knob l2pf|red] [--value 2] [--hq 32 --hkv 32] [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200.attention import (attn_backward, attn_forward, build_tiles,  # noqa: E402
                                             set_bwd_l2_prefetch)


def case(lengths, hq, hkv, d=128):
    plan = wl.build_shard_plan([lengths], 1, "per_document")
    _, pos, ro = plan.rank_local(0, 0)
    tiles = build_tiles(ro, pos, lengths)
    T = sum(lengths)
    dev = torch.device("cuda")
    q = torch.randn(T, hq, d, device=dev, dtype=torch.bfloat16)
    k = torch.randn(T, hkv, d, device=dev, dtype=torch.bfloat16)
    v = torch.randn_like(k)
    do = torch.randn_like(q)
    o, lse = attn_forward(q, k, v, tiles)
    pairs = sum(x * (x + 1) // 2 for x in lengths)
    return (lambda: attn_backward(q, k, v, o, lse, do, tiles)), 10 * d * hq * pairs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--knob", default="l2pf", choices=["l2pf"])
    ap.add_argument("--docs", type=int, nargs="*", default=[256, 512, 1024, 2048, 4096, 32768])
    a = ap.parse_args()
    setter = set_bwd_l2_prefetch
    val = {0: 0, 1: 1}
    T = 32768
    cases = {f"doc{n}": [n] * (T // n) for n in a.docs}
    for i, b in enumerate(wl.generate_synthetic_stream(wl.SyntheticSpec(T, T), 0, 8)):
        cases[f"bench_seq{i}"] = [x.length for x in b]
    out = {}
    for name, lengths in cases.items():
        fn, flops = case(lengths, a.hq, a.hkv)
        t = {0: [], 1: []}
        for _ in range(a.reps):
            for on in (0, 1):
                setter(val[on])
                fn()
                e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                e[0].record()
                fn()
                e[1].record()
                e[1].synchronize()
                t[on].append(e[0].elapsed_time(e[1]))
        setter(-1)
        m = {k: sorted(v)[len(v) // 2] for k, v in t.items()}
        out[name] = {"off_ms": round(m[0], 4), "on_ms": round(m[1], 4),
                     "off_tflops": round(flops / m[0] / 1e9, 1),
                     "on_tflops": round(flops / m[1] / 1e9, 1), "gain": round(m[0] / m[1] - 1, 4)}
        print(name, json.dumps(out[name]), flush=True)
    tot = {k: sum(v[k] for n, v in out.items() if n.startswith("bench")) for k in ("off_ms", "on_ms")}
    print("bench_total", json.dumps({**tot, "gain": round(tot["off_ms"] / tot["on_ms"] - 1, 4)}))


if __name__ == "__main__":
    main()
