"""Development aid: the PCIe floor of the bench's e2e step: the same
per-KV-head-group H2D (q, k, v, dO) and D2H (o, dq, dk, dv) copies of 8
micro-batches as hoststream.HostStreamedStep, both directions at once, no
attention (each D2H waits for the matching H2D, nothing else)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_17924_b200.attention import head_groups  # noqa: E402
from paper_2503_17924_b200.hoststream import _copy_cols  # noqa: E402

T, hq, hkv, d, n = 32768, int(sys.argv[1]) if len(sys.argv) > 1 else 32, int(sys.argv[2]) if len(sys.argv) > 2 else 32, 128, 8
dev = torch.device("cuda")
shapes = (hq, hkv, hkv, hq)
host_in = [torch.empty((T, h, d), dtype=torch.bfloat16, pin_memory=True) for h in shapes]
host_out = [torch.empty((T, h, d), dtype=torch.bfloat16, pin_memory=True) for h in (hq, hq, hkv, hkv)]
dev_in = [[torch.empty((T, h, d), dtype=torch.bfloat16, device=dev) for h in shapes] for _ in range(n)]
h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
rg = hq // hkv
for G in (1, 4, 8):
    groups = head_groups(hkv, G)
    for rep in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h2d.wait_stream(torch.cuda.current_stream())
        d2h.wait_stream(torch.cuda.current_stream())
        for m in range(n):
            evs = []
            for (g0, ng) in groups:
                for i, (dst, src) in enumerate(zip(dev_in[m], host_in)):
                    r = rg if i in (0, 3) else 1
                    _copy_cols(dst, src, g0 * r, ng * r, h2d)
                e = torch.cuda.Event()
                e.record(h2d)
                evs.append(e)
            for gi, (g0, ng) in enumerate(groups):
                d2h.wait_event(evs[gi])
                for i, (dst, src) in enumerate(zip(host_out, (dev_in[m][0], dev_in[m][3], dev_in[m][1], dev_in[m][2]))):
                    r = rg if i in (0, 1) else 1
                    _copy_cols(dst, src, g0 * r, ng * r, d2h)
        torch.cuda.current_stream().wait_stream(d2h)
        torch.cuda.current_stream().wait_stream(h2d)
        b.record()
        b.synchronize()
        if rep:
            print(f"hq {hq} hkv {hkv} groups {G}: {a.elapsed_time(b):.1f} ms per step "
                  f"({2 * n * sum(shapes) * T * d * 2 / 1e9:.2f} GB both ways)", flush=True)
