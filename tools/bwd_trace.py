"""Development aid: per-iteration timeline of the backward kernel's first CTA.

Run with a library built with -DWLB_TRACE:
    WLB_NVCC_EXTRA=-DWLB_TRACE WLB_LIB_OUT=build_var/libT.so python -m paper_2503_17924_b200.build
    WLB_LIB_PATH=build_var/libT.so python tools/bwd_trace.py [--doc 32768]
Events (clock64, SM cycles): 0 MMA q_full ok, 1 MMA s_free ok (dP issue),
2 MMA p_full(j) ok (dQ/dV/dK issue), 3 compute s_full ok, 4 compute S/dP in
registers, 5 compute P/dS stored (p_full arrive), 6 drain mma2_done ok,
7 drain dQ^T loaded (s_free arrive).
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200 import _native  # noqa: E402
from paper_2503_17924_b200.attention import attn_backward, attn_forward, build_tiles  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--doc", type=int, default=32768)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=32)
ap.add_argument("--ndocs", type=int, default=1, help="documents of --doc rows each")
ap.add_argument("--show", type=int, default=40)
a = ap.parse_args()
lengths = [a.doc] * a.ndocs
plan = wl.build_shard_plan([lengths], 1, "per_document")
g, pos, ro = plan.rank_local(0, 0)
tiles = build_tiles(ro, pos, lengths)
dev = torch.device("cuda")
T, d = a.doc * a.ndocs, 128
q = torch.randn(T, a.hq, d, device=dev, dtype=torch.bfloat16)
k = torch.randn(T, a.hkv, d, device=dev, dtype=torch.bfloat16)
v = torch.randn_like(k)
do = torch.randn_like(q)
o, lse = attn_forward(q, k, v, tiles)
for _ in range(3):
    attn_backward(q, k, v, o, lse, do, tiles)
torch.cuda.synchronize()
buf = np.zeros((2, 8, 128), dtype=np.int64)
lib = _native.lib()
lib.wlb_debug_bwd_trace.argtypes = [ctypes.c_void_p]
assert lib.wlb_debug_bwd_trace(buf.ctypes.data) == 0
t = buf[0].astype(np.float64)
t0 = t[0, 0]
names = ["mma_q", "mma_sfree", "mma_pfull", "cmp_sfull", "cmp_regs", "cmp_done", "drn_mma2", "drn_ld"]
print("iter " + " ".join(f"{n:>9s}" for n in names) + "   per-iter(mma_q delta)")
for i in range(2, min(a.show, 128)):
    row = " ".join(f"{t[e, i] - t0:9.0f}" for e in range(8))
    print(f"{i:4d} {row}   {t[0, i] - t[0, i - 1]:7.0f}")
it = np.arange(10, 100)
if a.ndocs > 1:
    sys.exit(0)
per = np.diff(t[0, 10:101]).mean()
print(f"steady-state cycles per q-tile (MMA warp): {per:.0f}")
print("mean waits (cycles), iters 10..99:")
print("  compute: s_full(i) wait end -> regs            ", np.mean(t[4, it] - t[3, it]).round())
print("  compute: regs -> p_full arrive                  ", np.mean(t[5, it] - t[4, it]).round())
print("  compute: p_full(i) -> s_full(i+1) ok            ", np.mean(t[3, it + 1] - t[5, it]).round())
print("  MMA: p_full(i) arrive -> MMA sees it           ", np.mean(t[2, it + 1] - t[5, it]).round())
print("  MMA: q_full(i) ok -> s_free ok (dP issue)       ", np.mean(t[1, it] - t[0, it]).round())
print("  MMA: s_free ok -> p_full(i-1) ok                ", np.mean(t[2, it - 1 + 1] - t[1, it]).round())
print("  MMA: p_full(j) ok -> next q_full ok             ", np.mean(t[0, it + 1] - t[2, it]).round())
print("  drain: mma2_done(j) ok -> ld done               ", np.mean(t[7, it] - t[6, it]).round())
print("  drain: p_full(j) MMA-issue -> mma2_done(j) ok   ", np.mean(t[6, it] - t[2, it]).round())
