"""Development aid: compute cost of running the bench step's attention in
KV-head groups (CPStepPipeline.run(io_groups=G), inputs resident) against
whole micro-batches, CP = 1, 32K synthetic sequences."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200.cp import CPStepPipeline, build_cp_shards  # noqa: E402

hq, hkv = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (32, 32)
T, d = 32768, 128
lengths = [[x.length for x in s] for s in wl.generate_synthetic_stream(wl.SyntheticSpec(T, T), 0, 8)]
dev = torch.device("cuda")
ins = [tuple(torch.randn((T, h, d), device=dev, dtype=torch.bfloat16) for h in (hq, hkv, hkv, hq))
       for _ in range(8)]
pipe = CPStepPipeline()
shards = build_cp_shards(lengths, 1, 0, "adaptive")
for G in (None, 1, 2, 4, 8, None, 4):
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        pipe.run(shards, ins, keep_outputs=False, io_groups=G)
        b.record()
        b.synchronize()
    print(f"hq {hq} hkv {hkv} io_groups {G}: {a.elapsed_time(b):.1f} ms", flush=True)
