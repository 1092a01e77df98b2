"""CPStepPipeline (exchange overlapped with compute) == direct kernel calls."""

import pytest
import torch

import paper_2503_17924_b200 as wl
from paper_2503_17924_b200.attention import attn_backward, attn_forward
from paper_2503_17924_b200.cp import CPStepPipeline, build_cp_shards

pytestmark = pytest.mark.gpu


def test_pipeline_matches_direct_cp1():
    lengths = [[300, 17, 1, 640, 129, 2, 959], [2048], [1000, 1048]]
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(3)
    ins = []
    for ls in lengths:
        T = sum(ls)
        mk = lambda h: torch.randn((T, h, 64), generator=g, device=dev, dtype=torch.bfloat16)
        ins.append((mk(4), mk(2), mk(2), mk(4)))
    shards = build_cp_shards(lengths, 1, 0, "adaptive")
    outs = CPStepPipeline().run(shards, ins)
    torch.cuda.synchronize()
    for (q, k, v, do), sh, (o, dq, dk, dv) in zip(ins, shards, outs):
        o2, lse = attn_forward(q, k, v, sh.tiles)
        dq2, dk2, dv2 = attn_backward(q, k, v, o2, lse, do, sh.tiles)
        assert torch.equal(o, o2)                              # deterministic forward
        assert (dq.float() - dq2.float()).abs().max() < 1e-2   # dQ uses fp32 atomics
        assert torch.allclose(dk, dk2, atol=1e-4) and torch.allclose(dv, dv2, atol=1e-4)


def test_pipeline_host_buffers_hooks():
    """The e2e path: inputs arrive by H2D copies on another stream (`ready`
    events), outputs leave through `on_outputs` (D2H on a third stream) with
    keep_outputs=False; results equal the direct kernels."""
    lengths = [[300, 17, 1, 640, 129, 2, 959], [2048], [1000, 1048]]
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(5)
    host = []
    for ls in lengths:
        T = sum(ls)
        mk = lambda h: torch.randn((T, h, 128), generator=g).to(torch.bfloat16).pin_memory()
        host.append((mk(4), mk(2), mk(2), mk(4)))
    dev_in = [tuple(torch.empty_like(t, device=dev) for t in hs) for hs in host]
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    ready = []
    with torch.cuda.stream(h2d):
        for dst, src in zip(dev_in, host):
            for a, b in zip(dst, src):
                a.copy_(b, non_blocking=True)
            e = torch.cuda.Event()
            e.record(h2d)
            ready.append(e)
    got = [None] * len(lengths)

    def on_outputs(b, outs, fin):
        d2h.wait_event(fin)
        with torch.cuda.stream(d2h):
            got[b] = tuple(t.to("cpu", non_blocking=True) for t in outs)
            for t in outs:
                t.record_stream(d2h)

    shards = build_cp_shards(lengths, 1, 0, "adaptive")
    CPStepPipeline().run(shards, dev_in, ready=ready, on_outputs=on_outputs, keep_outputs=False)
    torch.cuda.synchronize()
    for b, ((q, k, v, do), sh) in enumerate(zip(dev_in, shards)):
        o2, lse = attn_forward(q, k, v, sh.tiles)
        dq2, dk2, dv2 = attn_backward(q, k, v, o2, lse, do, sh.tiles)
        o, dq, dk, dv = got[b]
        assert torch.equal(o, o2.cpu())
        assert (dq.float() - dq2.float().cpu()).abs().max() < 1e-2
        assert torch.allclose(dk, dk2.cpu(), atol=1e-4) and torch.allclose(dv, dv2.cpu(), atol=1e-4)


@pytest.mark.parametrize("hq,hkv,groups", [(8, 8, 4), (8, 4, 2), (16, 4, 4), (8, 8, 3), (8, 4, None),
                                            (8, 8, "auto")])
def test_host_streamed_step_cp1(hq, hkv, groups):
    """hoststream.HostStreamedStep: per-KV-head-group H2D (2-D copies of the
    group's columns), the attention gated group by group, per-group D2H of
    O / dQ / dK / dV into pinned host buffers.  Host results equal the direct
    kernels (O and dK / dV bit for bit after the bf16 rounding, dQ within the
    fp32-atomics noise).  groups=None: whole micro-batches (one copy per
    tensor, the CP = 1 backward storing bf16 dK / dV); "auto" picks one."""
    from paper_2503_17924_b200.hoststream import HostStreamedStep
    lengths = [[300, 17, 1, 640, 129, 2, 959], [2048], [1000, 1048, 6]]
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(11)
    host_in, host_out, dev_in = [], [], []
    for ls in lengths:
        T = sum(ls)
        mk = lambda h: torch.randn((T, h, 128), generator=g).to(torch.bfloat16).pin_memory()
        host_in.append((mk(hq), mk(hkv), mk(hkv), mk(hq)))
        host_out.append(tuple(torch.full((T, h, 128), float("nan"), dtype=torch.bfloat16).pin_memory()
                              for h in (hq, hq, hkv, hkv)))
        dev_in.append(tuple(torch.empty_like(t, device=dev) for t in host_in[-1]))
    shards = build_cp_shards(lengths, 1, 0, "adaptive")
    step = HostStreamedStep(CPStepPipeline(), groups=groups)
    for _ in range(2):                                   # buffers reused across steps
        step.run(shards, host_in, dev_in, host_out)
    torch.cuda.synchronize()
    for hi, ho, sh in zip(host_in, host_out, shards):
        q, k, v, do = (t.to(dev) for t in hi)
        o2, lse = attn_forward(q, k, v, sh.tiles)
        dq2, dk2, dv2 = attn_backward(q, k, v, o2, lse, do, sh.tiles)
        o, dq, dk, dv = (t.to(dev) for t in ho)
        assert torch.equal(o, o2)
        assert (dq.float() - dq2.float()).abs().max() < 1e-2
        assert torch.equal(dk, dk2.to(torch.bfloat16)) and torch.equal(dv, dv2.to(torch.bfloat16))
