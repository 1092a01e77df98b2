"""A step's CP attention streamed from and to pinned host memory.

The end-to-end form of `CPStepPipeline.run`: every micro-batch's q, k, v and
dO arrive from pinned host buffers and O, dQ, dK, dV go back, with the PCIe
copies pipelined against the attention at KV-head-group granularity.  A
micro-batch's group g starts its forward as soon as the q / k / v columns of
g have landed (not the whole micro-batch), and the O / dQ / dK / dV columns
of g leave as soon as they are complete, so the copy engines see one
continuous stream in each direction and only one head group's transfer (not
one micro-batch's) is exposed at the start and the end of the step.

Head-group columns of a [T, H, D] tensor are strided (H*D elements per
row), so each copy is one `cudaMemcpy2DAsync` of T rows of G*D elements: on
B200 these run at the contiguous-copy rate down to 512-byte rows
(`tools/pcie2d_probe.py`).  Copies use the CUDA runtime through cuda-python
(`cuda.bindings.runtime`) on torch's streams; this is data movement only, the
attention is the library's sm_100a kernels.
"""

from __future__ import annotations

import torch

from .cp import CPStepPipeline

try:
    from cuda.bindings import runtime as _rt
except ImportError:   # pragma: no cover - the image ships cuda-python
    _rt = None


# Rates used only to order micro-batches (not reported): attention fwd+bwd
# TFLOP/s of a B200 rank and the per-direction pinned-host copy rate of one
# GPU with both directions busy (tools/pcie2d_probe.py: 47-50 GB/s).
_ATTN_FLOPS_EST = 950e12
_PCIE_EST = 48e9


def _estimates(shards, hq: int, hkv: int, d: int):
    """Per micro-batch (input copy seconds, attention seconds) estimates."""
    row_bytes = (2 * hq + 2 * hkv) * d * 2
    out = []
    for sh in shards:
        ls = sh.plan.lengths[sh.index]
        attn = 14.0 * d * hq * sum(x * (x + 1) // 2 for x in ls) / sh.cp / _ATTN_FLOPS_EST
        out.append((sum(ls) / sh.cp * row_bytes / _PCIE_EST, attn))
    return out


def johnson_order(shards, hq: int, hkv: int, d: int):
    """Johnson's rule for the two-stage flow copy-in -> attention: micro-
    batches whose attention outlasts their copies first (by increasing copy
    time), then the rest by decreasing attention time, so a PCIe-bound step
    does not end on a long attention after its last input byte.  Uses only
    document lengths, so every CP rank gets the same order."""
    jobs = [(i, c, a) for i, (c, a) in enumerate(_estimates(shards, hq, hkv, d))]
    first = sorted((j for j in jobs if j[1] < j[2]), key=lambda j: j[1])
    rest = sorted((j for j in jobs if j[1] >= j[2]), key=lambda j: -j[2])
    return [j[0] for j in first + rest]


def _copy_cols(dst, src, h0: int, nh: int, stream) -> None:
    """dst[:, h0:h0+nh] = src[:, h0:h0+nh] (or the whole of a [T, nh, D]
    side) for [T, H, D] tensors, host <-> device, on `stream`."""
    if nh == dst.shape[1] and nh == src.shape[1]:   # whole tensors: torch's async copy
        with torch.cuda.stream(stream):
            dst.copy_(src, non_blocking=True)
        return
    if _rt is None:
        raise RuntimeError("cuda-python (cuda.bindings) is required for host streaming")
    T = dst.shape[0]
    es = dst.element_size()
    w = nh * dst.shape[2] * es

    def side(t):
        full = t.shape[1] != nh
        return t.data_ptr() + (h0 * t.shape[2] * es if full else 0), t.shape[1] * t.shape[2] * es

    dp, dpitch = side(dst)
    sp, spitch = side(src)
    err, = _rt.cudaMemcpy2DAsync(dp, dpitch, sp, spitch, w, T,
                                 _rt.cudaMemcpyKind.cudaMemcpyDefault, stream.cuda_stream)
    if err != _rt.cudaError_t.cudaSuccess:
        raise RuntimeError(f"cudaMemcpy2DAsync failed: {err}")


class HostStreamedStep:
    """Run a step's micro-batches from pinned host inputs to pinned host
    outputs through `pipe` (a `CPStepPipeline`), head group by head group.

    run(shards, host_in, dev_in, host_out):
      host_in[b]  = (q, k, v, do) pinned host bf16 [T/cp, H, D] (local rows)
      dev_in[b]   = device bf16 buffers of the same shapes (overwritten)
      host_out[b] = (o, dq, dk, dv) pinned host bf16 [T/cp, H, D]
    Entries may repeat the same tensors (e.g. one host buffer for every
    micro-batch).  groups: "auto" (4 KV-head groups where the pipeline can
    run them, else whole micro-batches), an int, or None (whole micro-batches).
    order: "given" (default), "johnson" (`johnson_order`) or "auto"
    (Johnson where the estimated copies outlast the attention).
    The outputs are complete on the current stream when run returns
    (stream-ordered; no host sync).  The step's input copies start after the
    work already on the current stream (the previous step)."""

    def __init__(self, pipe: CPStepPipeline, groups="auto", order: str = "given"):
        if not (groups in ("auto", None) or (isinstance(groups, int) and groups >= 1)):
            raise ValueError("groups must be 'auto', None or a positive int")
        if order not in ("auto", "given", "johnson"):
            raise ValueError("order must be 'auto', 'given' or 'johnson'")
        self.pipe = pipe
        self.groups = groups
        self.order = order
        self.last_groups = None
        self.last_order = None
        self.h2d = torch.cuda.Stream()
        self.d2h = torch.cuda.Stream()

    def run(self, shards, host_in, dev_in, host_out, scale=None, on_kernels=None):
        cur = torch.cuda.current_stream()
        n = len(shards)
        hkv = dev_in[0][1].shape[1]
        hq = dev_in[0][0].shape[1]
        for b in range(n):
            want = [t.shape for t in dev_in[b]]
            want = (want[0], want[0], want[1], want[1])
            if ([t.shape for t in host_in[b]] != [t.shape for t in dev_in[b]]
                    or [t.shape for t in host_out[b]] != list(want)):
                raise ValueError(f"micro-batch {b}: host_in must match dev_in (q, k, v, do) and "
                                 "host_out be (o, dq, dk, dv) shaped like (q, q, k, k)")
            if not all(t.is_pinned() for t in host_in[b] + host_out[b]):
                raise ValueError(f"micro-batch {b}: host buffers must be pinned")
        order = self.order
        if order == "auto":
            # Johnson's rule only where the estimated copies outlast the
            # attention.  Measured (same box, e2e): 7B N=1 +1.2 %, but 70B GQA
            # N=1 -11 % and N=2 -13 %: the flow has a third stage (copy-out)
            # that the rule ignores, so "given" is the default
            est = _estimates(shards, hq, hkv, dev_in[0][0].shape[2])
            order = "johnson" if sum(c for c, _ in est) >= sum(a for _, a in est) else "given"
        self.last_order = order
        if order == "johnson":
            perm = johnson_order(shards, hq, hkv, dev_in[0][0].shape[2])
            shards, host_in, dev_in, host_out = ([x[i] for i in perm]
                                                 for x in (shards, host_in, dev_in, host_out))
        groups = self.groups
        if groups == "auto":
            # 4 head groups wherever the pipeline runs them (same box, e2e
            # TFLOP/s: N=1 424 vs 400 per micro-batch, N=2 1927 vs 1862, N=4
            # 3072 vs 2952); whole micro-batches with the NCCL / fused exchange
            groups = 4
            if any(sh.cp > 1 for sh in shards) and not (self.pipe.flagged and
                                                        not self.pipe.exchange.fused_sync):
                groups = None
        self.last_groups = groups
        self.h2d.wait_stream(cur)            # the previous step is done with the inputs
        if groups is None:
            self._run_mb(shards, host_in, dev_in, host_out, scale, on_kernels)
            cur.wait_stream(self.d2h)
            return
        g_of = [self.pipe.io_head_groups(hkv, groups, sh.cp) for sh in shards]
        ready, bwd_ready = [], []
        for b in range(n):
            q_h, k_h, v_h, do_h = host_in[b]
            q_d, k_d, v_d, do_d = dev_in[b]
            rg = hq // hkv
            ev_f, ev_b = [], []
            for (g0, ng) in g_of[b]:         # k, v, q of each group (the forward needs them)
                _copy_cols(k_d, k_h, g0, ng, self.h2d)
                _copy_cols(v_d, v_h, g0, ng, self.h2d)
                _copy_cols(q_d, q_h, g0 * rg, ng * rg, self.h2d)
                e = torch.cuda.Event()
                e.record(self.h2d)
                ev_f.append(e)
            for (g0, ng) in g_of[b]:         # dO behind them (only the backward needs it)
                _copy_cols(do_d, do_h, g0 * rg, ng * rg, self.h2d)
                e = torch.cuda.Event()
                e.record(self.h2d)
                ev_b.append(e)
            ready.append(ev_f)
            bwd_ready.append(ev_b)

        def on_group_forward(b, gi, o, ev):
            g0, ng = g_of[b][gi]
            rg = o.shape[1] // hkv
            self.d2h.wait_event(ev)
            _copy_cols(host_out[b][0], o, g0 * rg, ng * rg, self.d2h)
            o.record_stream(self.d2h)

        def on_group_outputs(b, gi, outs, ev):
            g0, ng = g_of[b][gi]
            o, dq, dk, dv = outs
            rg = dq.shape[1] // hkv
            self.d2h.wait_event(ev)
            with torch.cuda.stream(self.d2h):
                _copy_cols(host_out[b][1], dq, g0 * rg, ng * rg, self.d2h)
                for src, dst in ((dk, host_out[b][2]), (dv, host_out[b][3])):
                    if src.dtype != dst.dtype:       # (the pipeline stores the host dtype)
                        src = src[:, g0:g0 + ng].to(dst.dtype)
                        _copy_cols(dst, src, g0, ng, self.d2h)
                    else:
                        _copy_cols(dst, src, g0, ng, self.d2h)
                    src.record_stream(self.d2h)
                for t in (dq, dk, dv):
                    t.record_stream(self.d2h)

        self.pipe.run(shards, dev_in, scale=scale, ready=ready, bwd_ready=bwd_ready,
                      on_kernels=on_kernels, keep_outputs=False, io_groups=groups,
                      on_group_forward=on_group_forward, on_group_outputs=on_group_outputs,
                      dkv_dtype=host_out[0][2].dtype)
        cur.wait_stream(self.d2h)

    def _run_mb(self, shards, host_in, dev_in, host_out, scale, on_kernels):
        """Whole-micro-batch granularity: k, v, q then dO of each micro-batch
        in one copy each; O leaves after the forward, dQ / dK / dV after the
        backward (and the exchange pull)."""
        ready, bwd_ready = [], []
        for b in range(len(shards)):
            q_h, k_h, v_h, do_h = host_in[b]
            q_d, k_d, v_d, do_d = dev_in[b]
            for dst, src in ((k_d, k_h), (v_d, v_h), (q_d, q_h)):
                _copy_cols(dst, src, 0, dst.shape[1], self.h2d)
            e = torch.cuda.Event()
            e.record(self.h2d)
            ready.append(e)
            _copy_cols(do_d, do_h, 0, do_d.shape[1], self.h2d)
            e = torch.cuda.Event()
            e.record(self.h2d)
            bwd_ready.append(e)

        def on_forward(b, o, ev):
            self.d2h.wait_event(ev)
            _copy_cols(host_out[b][0], o, 0, o.shape[1], self.d2h)
            o.record_stream(self.d2h)

        def on_outputs(b, outs, ev):
            self.d2h.wait_event(ev)
            with torch.cuda.stream(self.d2h):
                for src, dst in zip(outs[1:], host_out[b][1:]):
                    if src.dtype != dst.dtype:       # (NCCL exchange: fp32 sums)
                        src = src.to(dst.dtype)
                    _copy_cols(dst, src, 0, dst.shape[1], self.d2h)
                    src.record_stream(self.d2h)

        self.pipe.run(shards, dev_in, scale=scale, ready=ready, bwd_ready=bwd_ready,
                      on_kernels=on_kernels, keep_outputs=False, on_forward=on_forward,
                      on_outputs=on_outputs, dkv_dtype=host_out[0][2].dtype)
