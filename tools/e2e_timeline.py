"""Development aid: timeline of one host-streamed bench step (CP = 1, 32K,
7B shape): when each micro-batch's H2D copies end, its kernels run and its
D2H copies end, from CUDA events on the three streams."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200 import hoststream  # noqa: E402
from paper_2503_17924_b200.cp import CPStepPipeline, build_cp_shards  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 4
hq, hkv = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (32, 32)
T, d = 32768, 128
lengths = [[x.length for x in s] for s in wl.generate_synthetic_stream(wl.SyntheticSpec(T, T), 0, 8)]
dev = torch.device("cuda")
shapes_in, shapes_out = (hq, hkv, hkv, hq), (hq, hq, hkv, hkv)
host_in = tuple(torch.randn((T, h, d), dtype=torch.bfloat16).pin_memory() for h in shapes_in)
host_out = tuple(torch.empty((T, h, d), dtype=torch.bfloat16, pin_memory=True) for h in shapes_out)
dev_in = [tuple(torch.empty((T, h, d), dtype=torch.bfloat16, device=dev) for h in shapes_in)
          for _ in range(8)]
step = hoststream.HostStreamedStep(CPStepPipeline(), groups=G)
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
shards = build_cp_shards(lengths, 1, 0, "adaptive")
for it in range(3):
    marks.clear()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    step.run(shards, [host_in] * 8, dev_in, [host_out] * 8, on_kernels=kern)
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record()
    t1.synchronize()
print(f"hq {hq} hkv {hkv} groups {G}: step {t0.elapsed_time(t1):.1f} ms")
h = [t0.elapsed_time(e) for k, e in marks if k == "h2d"]
dd = [t0.elapsed_time(e) for k, e in marks if k == "d2h"]
print(f"h2d: {len(h)} copies, last ends {max(h):.1f} ms; d2h: {len(dd)} copies, first ends "
      f"{min(dd):.1f}, last ends {max(dd):.1f}")
per = 4 * G
for b in range(8):
    ks = [v for k, v in marks if k == f"k{b}"][0]
    hb = h[b * per:(b + 1) * per]
    db = dd[b * per:(b + 1) * per]
    print(f"mb{b}: h2d {min(hb):7.1f}-{max(hb):7.1f} | kernels {t0.elapsed_time(ks[0]):7.1f}-"
          f"{t0.elapsed_time(ks[1]):7.1f} | d2h {min(db):7.1f}-{max(db):7.1f}")
