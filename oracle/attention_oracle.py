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
