"""Development aid: per-tile timeline of the v3 backward kernel's first CTA
(indexed by the CTA's global tile counter, so a persistent CTA's units follow
each other; --units summarises the S-issue interval across unit boundaries
against the interval inside units).

    WLB_NVCC_EXTRA=-DWLB_TRACE WLB_LIB_OUT=var/libT.so python -m paper_2503_17924_b200.build
    WLB_LIB_PATH=var/libT.so python tools/bwd3_trace.py [--doc 32768]
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
ap.add_argument("--units", action="store_true")
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
buf = np.zeros((2, 16, 128), dtype=np.int64)
lib = _native.lib()
lib.wlb_debug_bwd3_trace.argtypes = [ctypes.c_void_p]
assert lib.wlb_debug_bwd3_trace(buf.ctypes.data) == 0
t2 = buf.astype(np.float64)
t = t2[0]
if a.units:
    s_issue = t[0]
    n_tr = int((s_issue > 0).sum())
    # unit-start markers left by earlier launches (dynamic scheduling differs)
    # are dropped: a real start's fetch (14) lies within this launch's trace
    starts = sorted(int(x) for x in np.nonzero(t[4][:n_tr])[0]
                    if x == 0 or t[14][x] >= s_issue[0])
    dt = np.diff(s_issue[:n_tr])
    inside = [dt[i - 1] for i in range(1, n_tr) if i not in starts]
    across = [dt[i - 1] for i in starts if i > 0]
    print(f"doc {a.doc} x {a.ndocs}: {len(starts)} unit starts in the first {n_tr} tiles; "
          f"tiles per unit {n_tr / max(1, len(starts)):.1f}")
    print(f"S-issue interval inside units: median {np.median(inside):.0f} mean {np.mean(inside):.0f} cycles")
    print(f"S-issue interval across unit boundaries: median {np.median(across):.0f} "
          f"mean {np.mean(across):.0f} cycles")
    extra = (np.sum(across) - len(across) * np.median(inside)) / max(1.0, np.sum(dt))
    print(f"boundary excess share of the traced time: {extra:.3f}")
    # per boundary (unit starting at tile I): cycles from the previous tile's S
    # issue to the unit fetch (14), to its K / V landing (15) and to its S (0);
    # the previous tile's dS done (c_ds1, 11) and dQ drained (d_sfree, 13)
    print("boundary   fetch  kv_free   kv_land   S_issue  prev_ds1  epi_end  P0_done  (cycles after the previous S)")
    for I in starts[1:]:
        b = s_issue[I - 1]
        print(f"{I:8d} {t[14][I] - b:8.0f} {t[12][I] - b:8.0f} {t[15][I] - b:9.0f} {s_issue[I] - b:9.0f} "
              f"{t[11][I - 1] - b:9.0f} {t[13][I] - b:8.0f} {t[7][I] - b:8.0f}")
    sys.exit(0)
names = ["m_qfull", "m_sfree", "m_p0", "m_p1", "d_pfree", "m_ds1", "c_sfull", "c_p0", "c_p1",
         "c_dpfull", "c_ds0", "c_ds1", "d_dqfull", "d_sfree", "d_rx0", "d_rx3"]
n = len(names)
print("iter " + " ".join(f"{x:>8s}" for x in names) + "  per-tile")
for i in range(10, 20):
    row = " ".join(f"{t[e, i] - t[0, i]:8.0f}" for e in range(n))
    print(f"{i:4d} {row}  {t[0, i + 1] - t[0, i]:7.0f}")
it = np.arange(10, 100)
print(f"steady-state cycles per 128-query tile: {np.diff(t[0, 10:101]).mean():.0f}")
print("mean offsets from m_qfull(i) (S issue), iters 10..99:")
for e in range(1, n):
    print(f"  {names[e]:9s} {np.mean(t[e, it] - t[0, it]):8.0f}")
print(f"  next S    {np.mean(t[0, it + 1] - t[0, it]):8.0f}")

if t2[1].any():
    t1 = t2[1]
    print("CTA 1 (same zero: CTA 0's m_qfull(i)):")
    for e in range(1, n):
        print(f"  {names[e]:9s} {np.mean(t1[e, it] - t[0, it]):8.0f}")
    print(f"  m_qfull   {np.mean(t1[0, it] - t[0, it]):8.0f}")
