"""Development aid: timeline of one host-streamed step at CP = N (128K
sequences, 7B shape) under torchrun, against the same step with inputs
resident: per micro-batch on rank 0, when its H2D copies end, its kernels
run (device-resident and host-streamed) and its D2H copies end.

    python -m torch.distributed.run --nproc-per-node 4 tools/e2e_timeline_mp.py [groups]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200 import hoststream  # noqa: E402
from paper_2503_17924_b200.cp import CPStepPipeline, SymmExchange, build_cp_shards  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
dev = torch.device("cuda", torch.cuda.current_device())
dist.init_process_group("nccl", device_id=dev)
G = sys.argv[1] if len(sys.argv) > 1 else "auto"
G = None if G == "mb" else G if G == "auto" else int(G)
hq, hkv, d, T = 32, 32, 128, 131072
cp, tl = world, T // world
lengths = [[x.length for x in s] for s in wl.generate_synthetic_stream(wl.SyntheticSpec(T, T), 0, 8)]
model = wl.TileModel.for_shape(hq, hkv, d)
shapes_in, shapes_out = (hq, hkv, hkv, hq), (hq, hq, hkv, hkv)
host_in = tuple(torch.randn((tl, h, d), dtype=torch.bfloat16).pin_memory() for h in shapes_in)
host_out = tuple(torch.empty((tl, h, d), dtype=torch.bfloat16, pin_memory=True) for h in shapes_out)
dev_in = [tuple(torch.randn((tl, h, d), dtype=torch.bfloat16, device=dev) for h in shapes_in)
          for _ in range(8)]
pipe = CPStepPipeline(exchange=SymmExchange(dist.group.WORLD, T, hkv, d, dev))
step = hoststream.HostStreamedStep(pipe, groups=G)
marks = []
orig = hoststream._copy_cols


def traced(dst, src, h0, nh, stream):
    orig(dst, src, h0, nh, stream)
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    marks.append(("h2d" if stream is step.h2d else "d2h", e))


def kern(b, sh, fn):
    a = torch.cuda.Event(enable_timing=True)
    a.record()
    r = fn()
    z = torch.cuda.Event(enable_timing=True)
    z.record()
    marks.append((f"k{b}", (a, z)))
    return r


hoststream._copy_cols = traced


def timed(fn):
    dist.barrier()
    torch.cuda.synchronize()
    marks.clear()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    fn()
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record()
    t1.synchronize()
    return t0, t1


shards = build_cp_shards(lengths, cp, rank, "measured", model=model)
for it in range(3):
    r0, r1 = timed(lambda: pipe.run(shards, dev_in, on_kernels=kern, keep_outputs=False))
res_marks = list(marks)
for it in range(3):
    t0, t1 = timed(lambda: step.run(shards, [host_in] * 8, dev_in, [host_out] * 8, on_kernels=kern))
if rank == 0:
    print(f"world {world} groups {step.last_groups}: resident step {r0.elapsed_time(r1):.1f} ms, "
          f"host-streamed step {t0.elapsed_time(t1):.1f} ms")
    h = [(t0.elapsed_time(e)) for k, e in marks if k == "h2d"]
    dd = [(t0.elapsed_time(e)) for k, e in marks if k == "d2h"]
    per_h, per_d = len(h) // 8, len(dd) // 8
    for b in range(8):
        ks = [v for k, v in marks if k == f"k{b}"][0]
        kr = [v for k, v in res_marks if k == f"k{b}"][0]
        print(f"mb{b}: h2d {min(h[b*per_h:(b+1)*per_h]):7.1f}-{max(h[b*per_h:(b+1)*per_h]):7.1f} | "
              f"kernels {t0.elapsed_time(ks[0]):7.1f}-{t0.elapsed_time(ks[1]):7.1f} "
              f"({ks[0].elapsed_time(ks[1]):6.1f} ms; resident {kr[0].elapsed_time(kr[1]):6.1f}) | "
              f"d2h {min(dd[b*per_d:(b+1)*per_d]):7.1f}-{max(dd[b*per_d:(b+1)*per_d]):7.1f}", flush=True)
dist.destroy_process_group()
