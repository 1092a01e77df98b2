"""A/B the bench step at CP=1: direct kernel loop vs CPStepPipeline (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_17924_b200 as wl
from paper_2503_17924_b200.attention import attn_backward, attn_forward
from paper_2503_17924_b200.cp import CPStepPipeline, build_cp_shards

spec = wl.SyntheticSpec(32768, 32768)
lengths = [[d.length for d in b] for b in wl.generate_synthetic_stream(spec, 0, 8)]
dev = torch.device("cuda")
ins = [tuple(torch.randn(32768, 32, 128, device=dev, dtype=torch.bfloat16) for _ in range(4)) for _ in range(8)]
pipe = CPStepPipeline()

def direct():
    shards = build_cp_shards(lengths, 1, 0, "adaptive")
    for b, sh in enumerate(shards):
        q, k, v, do = ins[b]
        o, lse = attn_forward(q, k, v, sh.tiles)
        attn_backward(q, k, v, o, lse, do, sh.tiles)

def piped():
    shards = build_cp_shards(lengths, 1, 0, "adaptive")
    pipe.run(shards, ins)

def shards_only():
    build_cp_shards(lengths, 1, 0, "adaptive")

for name, fn in (("shards_only", shards_only), ("direct", direct), ("piped", piped), ("direct", direct)):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record()
    for _ in range(3): fn()
    b.record(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"{name:12s} gpu {a.elapsed_time(b)/3:8.2f} ms/step  cpu-enqueue {(t1-t0)/3*1e3:8.2f} ms/step  wall {(t2-t0)/3*1e3:8.2f}")
