"""Document-prefix causal attention on sm_100a (forward + backward).

Host-side orchestration of the tcgen05 kernels in `csrc/attn_fwd.cu` and
`csrc/attn_bwd.cu`.  The computation is the one the reference prices but
never runs (`sharding.py:19-21`): a query row at in-document position t of
document p attends keys [doc_start_p, doc_start_p + t + 1) of the
document-ordered K/V.  All tensors are THD ([tokens, heads, dim]) bf16.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _native

BLOCK_M = 128


@dataclass
class AttnTiles:
    """Query-tile work list of one rank (device)."""

    tiles: torch.Tensor       # [4*max_tiles, 4] int32: 2 rows per tile pair, then scratch
    n_tiles: torch.Tensor     # [1] int32 (number of tile pairs)
    max_tiles: int
    positions: torch.Tensor   # [Tl] int32
    rowset_off: torch.Tensor  # [n_docs+1] int32
    doc_start: torch.Tensor   # [n_docs+1] int32
    n_docs: int
    T: int                    # full (global) token count of the micro-batch


def build_tiles(rowset_off: torch.Tensor, positions: torch.Tensor, doc_lengths,
                block_m: int = BLOCK_M) -> AttnTiles:
    """Cut one rank's (rank, document) row-sets into query tiles on the GPU."""
    _native.require_device()
    dev = positions.device
    n_docs = len(doc_lengths)
    starts = [0]
    for x in doc_lengths:
        starts.append(starts[-1] + int(x))
    doc_start = _native.to_device(starts, torch.int32, dev)
    tl = positions.numel()
    max_tiles = tl // (2 * block_m) + n_docs + 1
    tiles = torch.empty((4 * max_tiles, 4), dtype=torch.int32, device=dev)
    n_tiles = torch.empty(1, dtype=torch.int32, device=dev)
    p = _native.ptr
    _native.check(_native.lib().wlb_attn_tiles(
        n_docs, p(rowset_off), p(positions), p(doc_start), block_m, max_tiles, p(tiles),
        p(n_tiles), _native.stream_ptr()), "wlb_attn_tiles")
    return AttnTiles(tiles, n_tiles, max_tiles, positions, rowset_off, doc_start, n_docs,
                     starts[-1])


def _check_inputs(q, k, v):
    for name, t in (("q", q), ("k", k), ("v", v)):
        if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous() or t.dim() != 3:
            raise ValueError(f"{name} must be a contiguous CUDA bf16 [tokens, heads, dim] tensor")
    if q.shape[2] != k.shape[2] or k.shape != v.shape or q.shape[1] % k.shape[1]:
        raise ValueError("shape mismatch between q, k, v")


def attn_forward(q, k, v, tiles: AttnTiles, scale: float | None = None, kv_heads=None,
                 out=None, sync=None):
    """O [Tl,Hq,D] bf16 and LSE [Hq,Tl] fp32 for one rank's local queries.

    kv_heads=(begin, count): only those KV heads and their query heads, into
    `out` = (o, lse) from an earlier call (the CP head-group pipeline).
    sync (`_native.WlbCpSync`): all heads in one launch, each CTA waiting on
    the device for its head group's K/V arrival flags."""
    _check_inputs(q, k, v)
    tl, hq, d = q.shape
    hkv = k.shape[1]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    if out is None:
        o = torch.empty_like(q)
        lse = torch.empty((hq, tl), dtype=torch.float32, device=q.device)
    else:
        o, lse = out
    p = _native.ptr
    if sync is not None:
        _native.check(_native.lib().wlb_attn_fwd_sync(
            p(q), p(k), p(v), p(o), p(lse), p(tiles.tiles), p(tiles.n_tiles), tiles.max_tiles,
            p(tiles.positions), tl, k.shape[0], hq, hkv, d, scale, sync, _native.stream_ptr()),
            "wlb_attn_fwd_sync")
        return o, lse
    if kv_heads is None:
        _native.check(_native.lib().wlb_attn_fwd(
            p(q), p(k), p(v), p(o), p(lse), p(tiles.tiles), p(tiles.n_tiles), tiles.max_tiles,
            p(tiles.positions), tl, k.shape[0], hq, hkv, d, scale, _native.stream_ptr()),
            "wlb_attn_fwd")
        return o, lse
    _native.check(_native.lib().wlb_attn_fwd_heads(
        p(q), p(k), p(v), p(o), p(lse), p(tiles.tiles), p(tiles.n_tiles), tiles.max_tiles,
        p(tiles.positions), tl, k.shape[0], hq, hkv, d, scale, kv_heads[0], kv_heads[1],
        _native.stream_ptr()), "wlb_attn_fwd_heads")
    return o, lse


def bwd_workspace(q, k, tiles: AttnTiles):
    """Backward workspace for one rank's micro-batch (shareable by the calls of
    a head-group sequence)."""
    tl, hq, d = q.shape
    return torch.empty(_native.lib().wlb_attn_bwd_workspace(tl, k.shape[0], hq, k.shape[1], d,
                                                            tiles.n_docs),
                       dtype=torch.uint8, device=q.device)


def attn_backward(q, k, v, o, lse, do, tiles: AttnTiles, scale: float | None = None,
                  dk_out=None, dv_out=None, covered_only: bool = False, kv_heads=None,
                  dq_out=None, ws=None, sync=None):
    """dQ [Tl,Hq,D] bf16 and fp32 dK/dV partials over the full sequence
    (written into dk_out / dv_out when given, e.g. symmetric exchange buffers;
    bf16 dk_out / dv_out take bf16 partials).  covered_only: rows no KV tile
    of this rank covers are left unwritten instead of zeroed (for the covered
    CP pull, which never reads them).  kv_heads=(begin, count): only those KV
    heads (dK/dV columns) and their query heads (dQ), into dq_out / dk_out /
    dv_out with workspace `ws` shared across the head groups.  sync
    (`_native.WlbCpSync`): all heads in one launch, publishing each head
    group's completion to every peer's DKV arrival flags from the device."""
    _check_inputs(q, k, v)
    tl, hq, d = q.shape
    T, hkv = k.shape[0], k.shape[1]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    do = do.contiguous()
    dq = torch.empty_like(q) if dq_out is None else dq_out
    dk = torch.empty((T, hkv, d), dtype=torch.float32, device=q.device) if dk_out is None else dk_out
    dv = torch.empty((T, hkv, d), dtype=torch.float32, device=q.device) if dv_out is None else dv_out
    if dk.dtype != dv.dtype or dk.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("dk_out / dv_out must both be fp32 or both bf16")
    flags = _native.WLB_BWD_DKV_BF16 if dk.dtype == torch.bfloat16 else 0
    if covered_only:
        flags |= _native.WLB_BWD_COVERED_ONLY
    lib = _native.lib()
    ws = bwd_workspace(q, k, tiles) if ws is None else ws
    p = _native.ptr
    args = (p(q), p(k), p(v), p(o), p(do), p(lse), p(dq), p(dk), p(dv), p(tiles.rowset_off),
            p(tiles.doc_start), tiles.n_docs, p(tiles.positions), tl, T, hq, hkv, d, scale,
            p(ws), flags)
    if sync is not None:
        _native.check(lib.wlb_attn_bwd_sync(*args, sync, _native.stream_ptr()),
                      "wlb_attn_bwd_sync")
    elif kv_heads is None:
        _native.check(lib.wlb_attn_bwd_ex(*args, _native.stream_ptr()), "wlb_attn_bwd_ex")
    else:
        _native.check(lib.wlb_attn_bwd_heads(*args, kv_heads[0], kv_heads[1],
                                             _native.stream_ptr()), "wlb_attn_bwd_heads")
    return dq, dk, dv


def head_groups(hkv: int, groups: int):
    """Split KV heads [0, hkv) into `groups` contiguous (begin, count) ranges."""
    groups = max(1, min(groups, hkv))
    base, extra = divmod(hkv, groups)
    out, b = [], 0
    for i in range(groups):
        c = base + (1 if i < extra else 0)
        out.append((b, c))
        b += c
    return out


def qkv_rope(y, positions, hq: int, hkv: int, d: int, base: float = 10000.0):
    """Split a fused QKV projection y [Tl, (hq + 2*hkv)*d] bf16 into THD q, k, v
    with rotary embeddings at the builder's in-document positions [Tl]."""
    if y.dtype != torch.bfloat16 or not y.is_cuda or not y.is_contiguous():
        raise ValueError("y must be a contiguous CUDA bf16 tensor")
    tl = y.shape[0]
    if y.numel() != tl * (hq + 2 * hkv) * d or positions.numel() != tl:
        raise ValueError("y / positions do not match Tl x (hq + 2*hkv) x d")
    q = torch.empty((tl, hq, d), dtype=torch.bfloat16, device=y.device)
    k = torch.empty((tl, hkv, d), dtype=torch.bfloat16, device=y.device)
    v = torch.empty_like(k)
    p = _native.ptr
    _native.check(_native.lib().wlb_qkv_rope(p(y), p(q), p(k), p(v), p(positions), tl, hq, hkv,
                                             d, float(base), _native.stream_ptr()),
                  "wlb_qkv_rope")
    return q, k, v


def set_bwd_v3_min_rows(rows: int) -> int:
    """Backward kernel choice for D = 128: the 128-query-tile kernel runs when a
    rank's local rows >= rows * n_docs (default 1, i.e. always for D = 128; negative restores it).
    Returns the previous threshold."""
    return int(_native.lib().wlb_attn_bwd_select(int(rows)))


def set_bwd_persistent(on: int) -> int:
    """64-query backward as a persistent kernel (1) or one CTA per work unit
    (0); negative = default.  Returns the previous setting."""
    return int(_native.lib().wlb_attn_bwd_persistent(int(on)))


def set_bwd_reserve_sms(n: int) -> int:
    """SMs the persistent backward kernels leave free for the CP exchange's
    kernels on the communication stream (0 = none, the default; negative
    restores it).  Returns the previous value."""
    return int(_native.lib().wlb_attn_bwd_reserve_sms(int(n)))


def set_bwd_l2_prefetch(on: int) -> int:
    """Persistent 128-query backward: L2 prefetch of the next unit's K / V and
    first Q / dO tile (1 on, 0 off, negative = default).  Returns the previous
    setting."""
    return int(_native.lib().wlb_attn_bwd_l2_prefetch(int(on)))


def set_bwd_pairs(on: int) -> int:
    """v3 backward as 2-CTA clusters sharing dQ (1 on, 0 off, negative =
    default).  Returns the previous setting."""
    return int(_native.lib().wlb_attn_bwd_pairs(int(on)))


class DocPrefixAttention(torch.autograd.Function):
    """Single-rank (CP=1 or pre-gathered KV) autograd wrapper."""

    @staticmethod
    def forward(ctx, q, k, v, tiles: AttnTiles, scale):
        o, lse = attn_forward(q, k, v, tiles, scale)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.tiles, ctx.scale = tiles, scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        dq, dk, dv = attn_backward(q, k, v, o, lse, do, ctx.tiles, ctx.scale)
        return dq, dk.to(k.dtype), dv.to(v.dtype), None, None


def doc_prefix_attention(q, k, v, tiles: AttnTiles, scale: float | None = None):
    return DocPrefixAttention.apply(q, k, v, tiles, scale)
