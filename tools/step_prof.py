"""cProfile of the bench step's host side (dev aid)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_17924_b200 as wl
from paper_2503_17924_b200.cp import CPStepPipeline, build_cp_shards

spec = wl.SyntheticSpec(32768, 32768)
lengths = [[d.length for d in b] for b in wl.generate_synthetic_stream(spec, 0, 8)]
dev = torch.device("cuda")
ins = [tuple(torch.randn(32768, 32, 128, device=dev, dtype=torch.bfloat16) for _ in range(4)) for _ in range(8)]
pipe = CPStepPipeline()
def step():
    shards = build_cp_shards(lengths, 1, 0, "adaptive")
    pipe.run(shards, ins)
for _ in range(2): step()
torch.cuda.synchronize()
t0 = time.perf_counter()
pr = cProfile.Profile(); pr.enable()
for _ in range(3): step()
pr.disable()
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"enqueue {(t1-t0)/3*1e3:.1f} ms/step, wall {(t2-t0)/3*1e3:.1f} ms/step")
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
