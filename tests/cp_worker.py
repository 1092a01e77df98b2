"""torchrun worker: CP document-masked attention fwd+bwd across ranks (NCCL) vs
the unsharded fp32 oracle.  Launched by tests/test_cp_multi.py (or by hand):

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/cp_worker.py
"""

import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200.cp import (CPStepPipeline, NcclExchange, SymmExchange,  # noqa: E402
                                      cp_doc_attention, shard_for_rank)
from oracle import attention_oracle as ao  # noqa: E402
from oracle import shard_oracle as so  # noqa: E402


def check(name, got, ref, atol=2e-2, rtol=1e-2):
    """Elementwise |got - ref| <= atol + rtol*|ref| (see tests/test_gpu_attention.py)."""
    got, ref = got.float().cpu(), ref.float()
    err = (got - ref).abs()
    ok = bool((err <= atol + rtol * ref.abs()).all())
    return ok, f"{name}: max abs err {err.max().item():.3e} (ref max {ref.abs().max().item():.2f})"


def pipeline_cases(rank, world, dev):
    failures = []
    for policy in ("adaptive", "per_sequence"):
        failures += _pipeline_cases(rank, world, dev, policy)
    return failures


def _pipeline_cases(rank, world, dev, policy):
    """CPStepPipeline over 3 micro-batches (slot reuse in the symmetric
    exchange) with both exchanges: each vs the oracle, and symm == NCCL.  The
    symmetric push / pull that skip ranks' uncovered rows (default) must equal
    the ones that move every row bit for bit (o, dK, dV; dQ sums by atomics)."""
    failures = []
    hq, hkv, d = 4, 2, 128
    mbs = [so.pad_lengths_for_cp(x, world) for x in
           ([900, 3, 129, 1000, 1], [2048], [300, 300, 1000, 17, 512, 33])]
    plan = wl.build_shard_plan(mbs, world, policy)
    shards = [shard_for_rank(plan, b, rank) for b in range(len(mbs))]
    g = torch.Generator().manual_seed(11)
    full, inputs = [], []
    for b, lengths in enumerate(mbs):
        T = sum(lengths)
        t = [torch.randn(T, h, d, generator=g).bfloat16() for h in (hq, hkv, hkv, hq)]
        full.append(t)
        idx = shards[b].gather_local.long().cpu()
        inputs.append(tuple(x[idx].to(dev) for x in t))
    t_max = max(sum(x) for x in mbs)
    res = {}
    symm_all = SymmExchange(dist.group.WORLD, t_max, hkv, d, dev)
    symm_all.pull_covered = symm_all.push_covered = False
    for name, ex in (("nccl", NcclExchange()),
                     ("symm", SymmExchange(dist.group.WORLD, t_max, hkv, d, dev)),
                     ("symm-all", symm_all)):
        pipe = CPStepPipeline(exchange=ex)
        for _ in range(2):                      # second pass reuses both slots again
            outs = pipe.run(shards, inputs)
        torch.cuda.synchronize()
        res[name] = [[t.float().cpu() for t in o] for o in outs]
    # the same step streamed from / to pinned host memory by KV-head group
    # (hoststream.HostStreamedStep over the symmetric exchange)
    from paper_2503_17924_b200.hoststream import HostStreamedStep
    host_in = [tuple(t.cpu().pin_memory() for t in x) for x in inputs]
    host_out = [tuple(torch.full(t.shape, float("nan"), dtype=torch.bfloat16).pin_memory()
                      for t in (x[0], x[0], x[1], x[1])) for x in inputs]
    dev_in = [tuple(torch.empty_like(t) for t in x) for x in inputs]
    hs = HostStreamedStep(CPStepPipeline(exchange=SymmExchange(dist.group.WORLD, t_max, hkv, d,
                                                               dev)))
    for _ in range(2):
        hs.run(shards, host_in, dev_in, host_out)
    torch.cuda.synchronize()
    for b in range(len(mbs)):
        for tn, a, c in zip(("o", "dq", "dk", "dv"), host_out[b], res["symm"][b]):
            c = c.bfloat16()
            same = torch.equal(a, c) if tn != "dq" else \
                (a.float() - c.float()).abs().max().item() <= 1e-2 * max(1.0, c.abs().max().item())
            if not same:
                failures.append(f"[rank {rank} {policy} mb{b}] host-streamed != pipeline {tn}: "
                                f"{(a.float() - c.float()).abs().max().item():.3e}")
    for b, lengths in enumerate(mbs):
        q, k, v, do = full[b]
        idx = shards[b].gather_local.long().cpu()
        segs = [(p, 0, x) for p, x in enumerate(lengths)]
        ro, _, rdq, rdk, rdv = ao.segment_attention_fwd_bwd(q, k, v, do, lengths, segs)
        for name in res:
            for tn, got, ref in zip(("o", "dq", "dk", "dv"), res[name][b],
                                    (ro[idx], rdq[idx], rdk[idx], rdv[idx])):
                ok, msg = check(tn, got, ref)
                tag = f"[rank {rank} pipeline {policy} {name} mb{b}] {msg}"
                print(tag, flush=True)
                if not ok:
                    failures.append(tag)
        for tn, a, c in zip(("o", "dq", "dk", "dv"), res["nccl"][b], res["symm"][b]):
            # same kernels; o and dq are rank-local (dq only differs by the order
            # of its fp32 atomic reductions), dK/dV partials are summed in fp32 by
            # NCCL and by the symmetric pull (fp32 partials by default; bf16
            # with WLB_XCHG_DKV=bf16): they agree to fp32 summation order
            err = (a - c).abs().max().item()
            tol = (1e-3 if tn in ("o", "dq") else 8e-3) * max(1.0, a.abs().max().item())
            if err > tol:
                failures.append(f"[rank {rank} {policy} mb{b}] symm vs nccl {tn}: {err:.3e}")
        for tn, a, c in (("o", res["symm"][b][0], res["symm-all"][b][0]),
                         ("dk", res["symm"][b][2], res["symm-all"][b][2]),
                         ("dv", res["symm"][b][3], res["symm-all"][b][3])):
            if not torch.equal(a, c):
                failures.append(f"[rank {rank} {policy} mb{b}] covered push/pull != full {tn}: "
                                f"{(a - c).abs().max().item():.3e}")
    return failures


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    failures = []
    cases = [([700, 3, 129, 2000, 1, 257, 64], "per_document", 4, 2, 128),
             ([700, 3, 129, 2000, 1, 257, 64], "per_sequence", 4, 4, 64),
             ([1500, 500], "adaptive", 8, 2, 128)]
    for lengths, policy, hq, hkv, d in cases:
        lengths = so.pad_lengths_for_cp(lengths, world)
        T = sum(lengths)
        g = torch.Generator().manual_seed(7)
        q = torch.randn(T, hq, d, generator=g).bfloat16()
        k = torch.randn(T, hkv, d, generator=g).bfloat16()
        v = torch.randn(T, hkv, d, generator=g).bfloat16()
        do = torch.randn(T, hq, d, generator=g).bfloat16()
        plan = wl.build_shard_plan([lengths], world, policy)
        shard = shard_for_rank(plan, 0, rank)
        idx = shard.gather_local.long().cpu()
        full = [(p, 0, x) for p, x in enumerate(lengths)]
        ro, _, rdq, rdk, rdv = ao.segment_attention_fwd_bwd(q, k, v, do, lengths, full)
        symm = SymmExchange(dist.group.WORLD, sum(lengths), hkv, d, dev)
        for xname, xch in (("nccl", None), ("symm-groups", symm)):
            for rep in range(3):            # slots reused (epochs advance)
                ql = q[idx].to(dev).requires_grad_(True)
                kl = k[idx].to(dev).requires_grad_(True)
                vl = v[idx].to(dev).requires_grad_(True)
                o = cp_doc_attention(ql, kl, vl, shard, exchange=xch)
                o.backward(do[idx].to(dev))
                torch.cuda.synchronize()
                for name, got, ref in (("o", o, ro[idx]), ("dq", ql.grad, rdq[idx]),
                                       ("dk", kl.grad, rdk[idx]), ("dv", vl.grad, rdv[idx])):
                    ok, msg = check(name, got, ref)
                    tag = (f"[rank {rank} {xname} {policy} {shard.strategy.value} hq={hq} "
                           f"hkv={hkv} d={d} rep {rep}] {msg}")
                    if rep == 0:
                        print(tag, flush=True)
                    if not ok:
                        failures.append(tag)
    failures += pipeline_cases(rank, world, dev)
    dist.barrier()
    dist.destroy_process_group()
    if failures:
        print("FAIL", failures, flush=True)
        sys.exit(1)
    print(f"rank {rank}: CP OK", flush=True)


if __name__ == "__main__":
    main()
