"""GPU-event timeline of one bench step (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_17924_b200 as wl
from paper_2503_17924_b200.cp import CPStepPipeline, build_cp_shards

spec = wl.SyntheticSpec(32768, 32768)
lengths = [[d.length for d in b] for b in wl.generate_synthetic_stream(spec, 0, 8)]
dev = torch.device("cuda")
gen = torch.Generator(device=dev)
ins = []
for b in range(8):
    gen.manual_seed(1000 + 64 * b)
    ins.append(tuple(torch.randn((32768, 32, 128), generator=gen, device=dev, dtype=torch.bfloat16) for _ in range(4)))
pipe = CPStepPipeline()
E = lambda: torch.cuda.Event(enable_timing=True)
for it in range(5):
    marks = [("start", E())]; marks[0][1].record()
    shards = build_cp_shards(lengths, 1, 0, "adaptive")
    m = E(); m.record(); marks.append(("plan+tiles", m))
    def on_k(b, sh, fn):
        a, z = E(), E(); a.record(); r = fn(); z.record(); marks.append((f"k{b}_start", a)); marks.append((f"k{b}_end", z)); return r
    pipe.run(shards, ins, on_kernels=on_k)
    m = E(); m.record(); marks.append(("end", m))
    torch.cuda.synchronize()
    t0 = marks[0][1]
    if it >= 3:
        print(" ".join(f"{n}={t0.elapsed_time(e):.1f}" for n, e in marks))
