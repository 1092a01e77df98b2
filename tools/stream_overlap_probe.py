"""Does running consecutive micro-batches on two streams fill the kernels'
tails?  The bench's 8 synthetic 32K sequences (7B shape, CP=1): fwd + bwd of
every sequence serially on one stream vs alternating two streams, whole-step
time with CUDA events, interleaved repetitions.

    python tools/stream_overlap_probe.py [--hq 32 --hkv 32] [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200.attention import attn_backward, attn_forward, build_tiles  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    T, d = 32768, 128
    dev = torch.device("cuda")
    seqs = [[x.length for x in b] for b in wl.generate_synthetic_stream(wl.SyntheticSpec(T, T), 0, 8)]
    cases = []
    for ls in seqs:
        plan = wl.build_shard_plan([ls], 1, "per_document")
        _, pos, ro = plan.rank_local(0, 0)
        tiles = build_tiles(ro, pos, ls)
        mk = lambda h: torch.randn(T, h, d, device=dev, dtype=torch.bfloat16)
        cases.append((tiles, mk(a.hq), mk(a.hkv), mk(a.hkv), mk(a.hq)))
    flops = sum(14.0 * d * a.hq * sum(x * (x + 1) // 2 for x in ls) for ls in seqs)
    streams = [torch.cuda.current_stream(), torch.cuda.Stream()]

    def one(c):
        tiles, q, k, v, do = c
        o, lse = attn_forward(q, k, v, tiles)
        attn_backward(q, k, v, o, lse, do, tiles)

    def serial():
        for c in cases:
            one(c)

    def two_streams():
        main_s = streams[0]
        done = torch.cuda.Event()
        done.record(main_s)
        streams[1].wait_event(done)
        for i, c in enumerate(cases):
            with torch.cuda.stream(streams[i % 2]):
                one(c)
        fin = torch.cuda.Event()
        fin.record(streams[1])
        main_s.wait_event(fin)

    fns = {"serial": serial, "two_streams": two_streams}
    for f in fns.values():
        f()
    torch.cuda.synchronize()
    t = {k: [] for k in fns}
    for _ in range(a.reps):
        for k, f in fns.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            e1.synchronize()
            t[k].append(e0.elapsed_time(e1))
    m = {k: sorted(v)[len(v) // 2] for k, v in t.items()}
    print(json.dumps({"hq": a.hq, "hkv": a.hkv, "ms": m,
                      "tflops": {k: round(flops / v / 1e9, 1) for k, v in m.items()},
                      "gain": round(m["serial"] / m["two_streams"] - 1, 4)}))


if __name__ == "__main__":
    main()
