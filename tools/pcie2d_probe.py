"""Development aid: pinned-host <-> device bandwidth of head-group slices
(cudaMemcpy2DAsync, rows of `width` bytes at a [T][H][D] pitch) against
contiguous copies, alone and with both directions at once."""
import time

import torch
from cuda.bindings import runtime as rt

T, H, D = 32768, 32, 128
pitch = H * D * 2
dev = torch.device("cuda")
h_in = torch.empty((T, H, D), dtype=torch.bfloat16, pin_memory=True)
h_out = torch.empty((T, H, D), dtype=torch.bfloat16, pin_memory=True)
d_in = torch.empty((T, H, D), dtype=torch.bfloat16, device=dev)
d_out = torch.randn((T, H, D), dtype=torch.bfloat16, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost


def copy(dst, src, groups, kind, stream):
    w = pitch // groups
    for g in range(groups):
        err, = rt.cudaMemcpy2DAsync(dst.data_ptr() + g * w, pitch, src.data_ptr() + g * w, pitch,
                                    w, T, kind, stream.cuda_stream)
        assert err == rt.cudaError_t.cudaSuccess, err


def run(groups, h2d, d2h, reps=4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            copy(d_in, h_in, groups, H2D, s1)
        if d2h:
            copy(h_out, d_out, groups, D2H, s2)
    torch.cuda.synchronize()
    return reps * T * pitch / (time.perf_counter() - t) / 1e9


run(1, True, True, 1)
for g in (1, 2, 4, 8, 16):
    print(f"groups {g:2d} (rows of {pitch // g} B): H2D {run(g, True, False):.1f} GB/s | "
          f"D2H {run(g, False, True):.1f} | both at once, each {run(g, True, True):.1f}", flush=True)
