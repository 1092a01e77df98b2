"""torch-CPU fp32 restatement of document-prefix causal attention.  TEST ORACLE ONLY.

The reference never computes attention; it prices a query range [s, e) of a
document as attending that document's causal prefix [0, e)
(`/root/reference/pkg/src/balsim/sharding.py:19-21`, `SPEC.md:301,328`) under a
block-diagonal causal mask (`workload.py:3-4`).  This module states exactly
that computation in fp32 so the sm_100a kernels can be checked against it:

    O[i] = softmax( Q[i] . K[doc_start : doc_start + pos_i + 1]^T * scale ) V[...]
    LSE[i] = logsumexp of the same scaled scores (natural log)

GQA: query head h reads kv head h // (Hq // Hkv).
"""

from __future__ import annotations

import math

import torch


def _expand_kv(x: torch.Tensor, hq: int) -> torch.Tensor:
    hkv = x.shape[1]
    return x if hkv == hq else x.repeat_interleave(hq // hkv, dim=1)


def segment_attention(q, k_full, v_full, doc_lengths, worker_ranges, scale=None):
    """Forward for one CP worker.

    q:            [Tl, Hq, D] local queries, rows in the worker's canonical order
    k_full/v_full:[T, Hkv, D] full keys/values in document (global) order
    worker_ranges: [(pos, start, end), ...] canonical ranges of this worker
    Returns (out [Tl, Hq, D] fp32, lse [Hq, Tl] fp32).
    """
    q = q.float()
    k_full = k_full.float()
    v_full = v_full.float()
    hq, d = q.shape[1], q.shape[2]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    starts = [0]
    for x in doc_lengths:
        starts.append(starts[-1] + int(x))
    outs, lses = [], []
    row = 0
    for p, s, e in worker_ranges:
        n = e - s
        qs = q[row:row + n].transpose(0, 1)                       # [H, n, D]
        ks = _expand_kv(k_full[starts[p]:starts[p] + e], hq).transpose(0, 1)
        vs = _expand_kv(v_full[starts[p]:starts[p] + e], hq).transpose(0, 1)
        scores = torch.matmul(qs, ks.transpose(1, 2)) * scale       # [H, n, e]
        allowed = torch.arange(e)[None, :] <= (torch.arange(n) + s)[:, None]
        scores = scores.masked_fill(~allowed, float("-inf"))
        lse = torch.logsumexp(scores, dim=-1)                      # [H, n]
        probs = torch.exp(scores - lse[..., None])
        outs.append(torch.matmul(probs, vs).transpose(0, 1))       # [n, H, D]
        lses.append(lse)
        row += n
    if not outs:
        return q.new_zeros(q.shape), q.new_zeros((hq, 0))
    return torch.cat(outs, 0), torch.cat(lses, 1)


def segment_attention_fwd_bwd(q, k_full, v_full, do, doc_lengths, worker_ranges,
                              scale=None):
    """Forward + autograd backward of `segment_attention` in fp32.

    Returns (out, lse, dq [Tl,Hq,D], dk_full [T,Hkv,D], dv_full [T,Hkv,D]);
    dk/dv are this worker's partial contributions over the full sequence.
    """
    q = q.detach().float().requires_grad_(True)
    k = k_full.detach().float().requires_grad_(True)
    v = v_full.detach().float().requires_grad_(True)
    out, lse = segment_attention(q, k, v, doc_lengths, worker_ranges, scale)
    out.backward(do.float())
    return out.detach(), lse.detach(), q.grad, k.grad, v.grad


def doc_causal_attention(q, k, v, doc_lengths, scale=None):
    """Unsharded reference: per-document causal attention over full tensors.
    Equal to `segment_attention` with the single worker owning everything."""
    ranges = [(p, 0, int(x)) for p, x in enumerate(doc_lengths)]
    return segment_attention(q, k, v, doc_lengths, ranges, scale)


def segment_attention_fwd_bwd_blocked(q, k_full, v_full, do, doc_lengths, worker_ranges,
                                      scale=None, block=256):
    """Same math as `segment_attention_fwd_bwd`, restated with an explicit
    (non-autograd) backward over query blocks of `block` rows, so config-scale
    segments (32K-128K keys, 32-64 heads) fit in memory.  Runs on whatever
    device the inputs live on (fp32 on a GPU for the config-scale tests; TF32
    is switched off for the duration).  TEST ORACLE ONLY.

    Per query block of a range (p, [s, e)) with rows [a, b) of the worker:
        S  = Q K[0:kb]^T * scale     (kb = last row's position + 1; mask pos >= key)
        P  = exp(S - lse),  O = P V,  lse = logsumexp(S)
        dP = dO V^T,  Delta = rowsum(dO * O),  dS = P * (dP - Delta)
        dQ = dS K * scale,  dK[0:kb] += dS^T Q * scale,  dV[0:kb] += P^T dO
    GQA: the group's query heads are stacked so one batched matmul per KV
    head serves them (query head h reads KV head h // (Hq // Hkv)).
    Returns (out [Tl,Hq,D], lse [Hq,Tl], dq [Tl,Hq,D], dk [T,Hkv,D], dv [T,Hkv,D]), fp32.
    """
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        return _blocked(q, k_full, v_full, do, doc_lengths, worker_ranges, scale, block)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32


def _blocked(q, k_full, v_full, do, doc_lengths, worker_ranges, scale, block):
    tl, hq, d = q.shape
    T, hkv = k_full.shape[0], k_full.shape[1]
    g = hq // hkv
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    dev = q.device
    out = torch.zeros((tl, hq, d), dtype=torch.float32, device=dev)
    lse_all = torch.zeros((hq, tl), dtype=torch.float32, device=dev)
    dq = torch.zeros((tl, hq, d), dtype=torch.float32, device=dev)
    dk = torch.zeros((T, hkv, d), dtype=torch.float32, device=dev)
    dv = torch.zeros((T, hkv, d), dtype=torch.float32, device=dev)
    starts = [0]
    for x in doc_lengths:
        starts.append(starts[-1] + int(x))
    row = 0
    for p, s, e in worker_ranges:
        for a in range(s, e, block):
            b = min(a + block, e)
            n, kb = b - a, b                      # keys [0, b) of document p
            r0 = row + (a - s)
            k0 = starts[p]
            # [Hkv, g*n, D]: query heads of one KV head stacked (head-major)
            qb = q[r0:r0 + n].float().view(n, hkv, g, d).permute(1, 2, 0, 3).reshape(hkv, g * n, d)
            dob = do[r0:r0 + n].float().view(n, hkv, g, d).permute(1, 2, 0, 3).reshape(hkv, g * n, d)
            kk = k_full[k0:k0 + kb].float().transpose(0, 1)          # [Hkv, kb, D]
            vv = v_full[k0:k0 + kb].float().transpose(0, 1)
            sc = torch.matmul(qb, kk.transpose(1, 2)) * scale          # [Hkv, g*n, kb]
            pos = torch.arange(a, b, device=dev).repeat(g)             # query positions
            allowed = torch.arange(kb, device=dev)[None, :] <= pos[:, None]
            sc = sc.masked_fill(~allowed[None], float("-inf"))
            lse = torch.logsumexp(sc, dim=-1)                          # [Hkv, g*n]
            pr = torch.exp(sc - lse[..., None])
            del sc
            o = torch.matmul(pr, vv)                                   # [Hkv, g*n, D]
            dp = torch.matmul(dob, vv.transpose(1, 2))
            delta = (dob * o).sum(-1, keepdim=True)
            ds = pr * (dp - delta)
            del dp
            dqb = torch.matmul(ds, kk) * scale
            dk[k0:k0 + kb] += (torch.matmul(ds.transpose(1, 2), qb) * scale).transpose(0, 1)
            dv[k0:k0 + kb] += torch.matmul(pr.transpose(1, 2), dob).transpose(0, 1)
            del ds, pr
            unstack = lambda x: x.reshape(hkv, g, n, d).permute(2, 0, 1, 3).reshape(n, hq, d)
            out[r0:r0 + n] = unstack(o)
            dq[r0:r0 + n] = unstack(dqb)
            lse_all[:, r0:r0 + n] = lse.reshape(hkv, g, n).reshape(hq, n)
        row += e - s
    return out, lse_all, dq, dk, dv
