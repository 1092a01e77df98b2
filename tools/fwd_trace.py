"""Development aid: per-KV-step timeline of the forward kernel's first CTA
(the heaviest tile pair of head 0).  Needs a -DWLB_TRACE library (see
tools/bwd_trace.py).  Events: 0/1 MMA saw p_full X/Y (step j), 8 MMA saw
v_full(j); 2/5 softmax X/Y s_full ok, 3/6 S in registers, 4/7 P stored."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200 import _native  # noqa: E402
from paper_2503_17924_b200.attention import attn_forward, build_tiles  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
plan = wl.build_shard_plan([[T]], 1, "per_document")
g, pos, ro = plan.rank_local(0, 0)
tiles = build_tiles(ro, pos, [T])
dev = torch.device("cuda")
q = torch.randn(T, 32, 128, device=dev, dtype=torch.bfloat16)
k = torch.randn_like(q)
v = torch.randn_like(q)
for _ in range(3):
    attn_forward(q, k, v, tiles)
torch.cuda.synchronize()
buf = np.zeros((12, 256), dtype=np.int64)
lib = _native.lib()
lib.wlb_debug_fwd_trace.argtypes = [ctypes.c_void_p]
assert lib.wlb_debug_fwd_trace(buf.ctypes.data) == 0
t = buf.astype(np.float64)
t0 = t[2, 0]
print("   j  mmaPX  mmaPY  mmaV |  X sfull  X regs  X done |  Y sfull  Y regs  Y done | step")
for j in range(1, 30):
    print(f"{j:4d} {t[0,j]-t0:7.0f} {t[1,j]-t0:7.0f} {t[8,j]-t0:7.0f} | {t[2,j]-t0:7.0f} {t[3,j]-t0:7.0f} "
          f"{t[4,j]-t0:7.0f} | {t[5,j]-t0:7.0f} {t[6,j]-t0:7.0f} {t[7,j]-t0:7.0f} | {t[2,j]-t[2,j-1]:6.0f}")
j = np.arange(20, 200)
print(f"steady cycles per KV step: {np.mean(t[2, j + 1] - t[2, j]):.0f}  (tensor ideal 2048)")
print(f"X: sfull->regs {np.mean(t[3, j] - t[2, j]):.0f}, regs->done {np.mean(t[4, j] - t[3, j]):.0f}, "
      f"done->next sfull {np.mean(t[2, j + 1] - t[4, j]):.0f}")
print(f"Y: sfull->regs {np.mean(t[6, j] - t[5, j]):.0f}, regs->done {np.mean(t[7, j] - t[6, j]):.0f}, "
      f"done->next sfull {np.mean(t[5, j + 1] - t[7, j]):.0f}")
print(f"X detail: regs->max {np.mean(t[9, j] - t[3, j]):.0f}, max->exp loop done {np.mean(t[10, j] - t[9, j]):.0f}, "
      f"->st_wait done {np.mean(t[11, j] - t[10, j]):.0f}, ->arrive {np.mean(t[4, j] - t[11, j]):.0f}")
print(f"MMA: X done -> MMA sees p_full X {np.mean(t[0, j] - t[4, j]):.0f}; "
      f"Y done -> sees {np.mean(t[1, j] - t[7, j]):.0f}")
