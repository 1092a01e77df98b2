"""Context-parallel document-masked attention across ranks (one process per GPU).

The paper's CP exchange (`PAPER.md:102,425`; absent from the reference, which
folds it into W_l, `SPEC.md:335`): each rank owns T/cp tokens chosen by the
shard builder (per-sequence or per-document, selected per micro-batch).

  forward : all-gather local K,V (bf16, NCCL over NVLink)  -> rank-contiguous
            buffer -> scatter rows to document order (wlb_rows_scatter) ->
            doc-prefix attention for the local queries.
  backward: attention backward -> full-length fp32 dK/dV partials -> gather
            rows to rank-contiguous order (wlb_rows_gather) -> NCCL
            reduce-scatter (sum) -> local dK/dV.

`gather_index` of the micro-batch (ranks concatenated) is exactly the
all-gather output order, so one index serves both permutations.
"""

from __future__ import annotations

import ctypes
import os

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native
from .attention import (AttnTiles, attn_backward, attn_forward, build_tiles, bwd_workspace,
                        head_groups, qkv_rope)
from .sharding import ShardPlan, build_shard_plan
from .workload import CostProfile


@dataclass
class CPShard:
    """Everything one rank needs for one micro-batch."""

    plan: ShardPlan
    index: int             # micro-batch index inside the plan
    rank: int
    cp: int
    tiles: AttnTiles
    gather_all: torch.Tensor   # [T] int32: all ranks' local rows -> global token
    gather_local: torch.Tensor  # [T/cp] int32

    @property
    def pairs(self) -> int:
        """Causal pairs of this rank (FLOP basis); reading it syncs with the GPU."""
        return int(self.plan.host("rank_pairs")[self.index, self.rank])

    @property
    def strategy(self):
        return self.plan.strategy(self.index)


def project_qkv(x, w_qkv, shard: CPShard, hq: int, hkv: int, d: int, base: float = 10000.0,
                gather: bool = False, gather_in_gemm: bool = False):
    """The step before the path: this rank's q, k, v (THD bf16) from hidden
    states and the fused QKV weight w_qkv [hidden, (hq + 2*hkv)*d] (x @ W),
    with rotary embeddings at each row's in-document position
    (`shard.tiles.positions`), ready for `cp_doc_attention` / `CPStepPipeline`.

    x: this rank's local hidden states [T/cp, hidden] in local order, or with
    gather=True the micro-batch's hidden states [T, hidden] in global order,
    whose rows `shard.gather_local` are this rank's.  D = 128: one tcgen05
    kernel (`wlb_qkv_proj_rope`: projection and RoPE fused); other D: a
    library GEMM then `wlb_qkv_rope`.

    With gather=True the rank's rows are first packed by one `wlb_rows_gather`
    pass (T/cp x hidden bf16).  The kernel can instead gather them itself with
    TMA gather4 (`gather_in_gemm=True`), but it then re-gathers every row once
    per 256-column output tile (48 times at the Llama-7B shape) and measured
    2.5x slower than pack + tiled loads (profiles/r02_proj_bench.jsonl)."""
    tl = shard.gather_local.numel()
    if gather and not gather_in_gemm:
        if x.dtype != torch.bfloat16 or not x.is_cuda or not x.is_contiguous() or x.dim() != 2:
            raise ValueError("x must be a contiguous 2-D CUDA bf16 tensor")
        packed = torch.empty((tl, x.shape[1]), dtype=x.dtype, device=x.device)
        _rows("wlb_rows_gather", x, packed, shard.gather_local)
        x, gather = packed, False
    if d == 128:
        for name, t in (("x", x), ("w_qkv", w_qkv)):
            if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous() or t.dim() != 2:
                raise ValueError(f"{name} must be a contiguous 2-D CUDA bf16 tensor")
        if w_qkv.shape != (x.shape[1], (hq + 2 * hkv) * d):
            raise ValueError("w_qkv must be [hidden, (hq + 2*hkv)*d]")
        q = torch.empty((tl, hq, d), dtype=torch.bfloat16, device=x.device)
        k = torch.empty((tl, hkv, d), dtype=torch.bfloat16, device=x.device)
        v = torch.empty_like(k)
        p = _native.ptr
        _native.check(_native.lib().wlb_qkv_proj_rope(
            p(x), x.shape[0], p(shard.gather_local) if gather else None, p(w_qkv), p(q), p(k),
            p(v), p(shard.tiles.positions), tl, x.shape[1], hq, hkv, d, float(base),
            _native.stream_ptr()), "wlb_qkv_proj_rope")
        return q, k, v
    x_local = x[shard.gather_local.long()] if gather else x
    y = torch.matmul(x_local, w_qkv)
    return qkv_rope(y, shard.tiles.positions, hq, hkv, d, base)


def shard_for_rank(plan: ShardPlan, index: int, rank: int) -> CPShard:
    lengths = plan.lengths[index]
    g, pos, ro = plan.rank_local(index, rank)
    T = sum(lengths)
    lo = plan.tok_off[index]
    tiles = build_tiles(ro, pos, lengths)
    return CPShard(plan=plan, index=index, rank=rank, cp=plan.cp, tiles=tiles,
                   gather_all=plan.gather_index[lo:lo + T], gather_local=g)


def build_cp_shards(microbatches, cp: int, rank: int, policy: str = "adaptive",
                    profile: CostProfile | None = None, model=None) -> list[CPShard]:
    """Shard + select every micro-batch of a step in one GPU launch, then cut
    this rank's attention tiles.  policy "measured" selects with the B200 tile
    model `model` (`tilemodel.TileModel`)."""
    plan = build_shard_plan(microbatches, cp, policy, profile, model=model)
    return [shard_for_rank(plan, b, rank) for b in range(plan.n_mb)]


def _rows(fn, src, dst, index):
    row_bytes = src[0].numel() * src.element_size()
    _native.check(getattr(_native.lib(), fn)(src.data_ptr(), dst.data_ptr(), index.data_ptr(),
                                             index.numel(), row_bytes, _native.stream_ptr()), fn)


def gather_kv(k_local, v_local, shard: CPShard, group=None):
    """All-gather local K/V and return them in document order [T, Hkv, D]."""
    if shard.cp == 1:
        return k_local, v_local
    T = shard.gather_all.numel()
    kv = torch.stack((k_local, v_local))                       # [2, Tl, Hkv, D]
    gathered = torch.empty((shard.cp,) + tuple(kv.shape), dtype=kv.dtype, device=kv.device)
    dist.all_gather_into_tensor(gathered, kv, group=group)
    outs = []
    for i in range(2):
        src = gathered[:, i].reshape(T, *k_local.shape[1:])
        dst = torch.empty_like(src)
        _rows("wlb_rows_scatter", src.contiguous(), dst, shard.gather_all)
        outs.append(dst)
    return outs[0], outs[1]


def scatter_dkv(dk_full, dv_full, shard: CPShard, group=None):
    """Sum full-length fp32 dK/dV partials over ranks; return this rank's rows."""
    if shard.cp == 1:
        return dk_full, dv_full
    T = dk_full.shape[0]
    tl = T // shard.cp
    both = torch.empty((shard.cp, 2, tl) + tuple(dk_full.shape[1:]), dtype=dk_full.dtype,
                       device=dk_full.device)
    for i, full in enumerate((dk_full, dv_full)):
        perm = torch.empty_like(full)
        _rows("wlb_rows_gather", full, perm, shard.gather_all)
        both[:, i] = perm.view(shard.cp, tl, *full.shape[1:])
    out = torch.empty((2, tl) + tuple(dk_full.shape[1:]), dtype=dk_full.dtype, device=dk_full.device)
    dist.reduce_scatter_tensor(out, both, group=group)
    return out[0], out[1]


class CPDocAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, shard: CPShard, group, scale, exchange):
        ctx.shard, ctx.group, ctx.scale, ctx.exchange = shard, group, scale, exchange
        if isinstance(exchange, SymmExchange) and shard.cp > 1:
            # push K/V head group by head group on a side stream; the attention
            # of each group starts once every peer's rows of it have landed
            cur = torch.cuda.current_stream()
            b = exchange.begin_microbatch()
            side = exchange.side_stream()
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                k_full, v_full = exchange.gather(k, v, shard, b)
            if exchange.fused_sync:
                o, lse = attn_forward(q, k_full, v_full, shard.tiles, scale,
                                      sync=exchange.fwd_sync(b))
            else:
                o = lse = None
                for gi, grp in enumerate(exchange.groups):
                    exchange.wait_kv(b, gi)
                    o, lse = attn_forward(q, k_full, v_full, shard.tiles, scale, kv_heads=grp,
                                          out=None if o is None else (o, lse))
            for t in (k, v, k_full, v_full):
                t.record_stream(side)
            ctx.b = b
        else:
            k_full, v_full = gather_kv(k, v, shard, group)
            o, lse = attn_forward(q, k_full, v_full, shard.tiles, scale)
        ctx.save_for_backward(q, k_full, v_full, o, lse)
        return o

    @staticmethod
    def backward(ctx, do):
        q, k_full, v_full, o, lse = ctx.saved_tensors
        shard, ex = ctx.shard, ctx.exchange
        if isinstance(ex, SymmExchange) and shard.cp > 1:
            cur = torch.cuda.current_stream()
            b = ctx.b
            dk_out, dv_out = ex.dkv_out(shard, b, cur)
            cov = ex.pull_covered and shard.tiles.n_docs > 0
            dq, ws = torch.empty_like(q), bwd_workspace(q, k_full, shard.tiles)
            do = do.contiguous()
            if ex.fused_sync:
                attn_backward(q, k_full, v_full, o, lse, do, shard.tiles, ctx.scale, dk_out,
                              dv_out, covered_only=cov, dq_out=dq, ws=ws, sync=ex.bwd_sync(b))
            else:
                for gi, grp in enumerate(ex.groups):
                    attn_backward(q, k_full, v_full, o, lse, do, shard.tiles, ctx.scale, dk_out,
                                  dv_out, covered_only=cov, kv_heads=grp, dq_out=dq, ws=ws)
                    ex.signal_dkv(b, gi)
            # each group's pull starts once every peer's partials of it are in
            side = ex.side_stream()
            with torch.cuda.stream(side):
                dk, dv = ex.scatter(dk_out, dv_out, shard, b)
            cur.wait_stream(side)
            ex.end_microbatch(b)
            return dq, dk.to(torch.bfloat16), dv.to(torch.bfloat16), None, None, None, None
        dq, dk_full, dv_full = attn_backward(q, k_full, v_full, o, lse, do, shard.tiles,
                                             ctx.scale)
        dk, dv = scatter_dkv(dk_full, dv_full, shard, ctx.group)
        return dq, dk.to(torch.bfloat16), dv.to(torch.bfloat16), None, None, None, None


def cp_doc_attention(q, k, v, shard: CPShard, group=None, scale=None, exchange=None):
    """Document-masked causal attention of this rank's local tokens.

    q [T/cp, Hq, D], k/v [T/cp, Hkv, D] bf16 in the rank's local order
    (`shard.gather_local`); returns O [T/cp, Hq, D] bf16.  Differentiable.

    exchange=None: NCCL all-gather / reduce-scatter (no overlap).  A
    `SymmExchange`: the one-sided head-group exchange with per-peer arrival
    flags, overlapped with the attention of the groups already landed (at
    most `exchange.slots` micro-batches between a forward and its backward).
    """
    return CPDocAttention.apply(q, k, v, shard, group, scale, exchange)


class NcclExchange:
    """CP exchange through NCCL collectives (all-gather / reduce-scatter) plus
    the row-permutation kernels."""

    depth = 1            # collectives on one communicator stay on one stream

    def __init__(self, group=None):
        self.group = group

    def gather(self, k, v, shard, b):
        return gather_kv(k, v, shard, self.group)

    def dkv_out(self, shard, b, cur):
        return None, None

    def scatter(self, dkf, dvf, shard, b):
        return scatter_dkv(dkf, dvf, shard, self.group)


MAX_GROUPS = 8          # head groups per micro-batch in the flag layout
_KV, _DKV, _KV_FREE, _DKV_FREE = 0, 1, 2, 3   # flag kinds
_KINDS = 4


class SymmExchange:
    """CP exchange as ONE-SIDED NVLink traffic on symmetric memory.

    Every rank owns `slots` slots (micro-batch b uses slot b % slots) of a
    document-ordered K/V buffer and of fp32 dK/dV partial buffers
    (WLB_XCHG_DKV=bf16: bf16 partials, summed in fp32 by the pull), mapped
    into every peer, plus a small flag buffer.  With more than 2 slots the
    pipeline pushes K/V slots-1 micro-batches ahead on a stream of its own
    (3 slots measured slower at N=4: 3748-3758 vs 3785-3791 TFLOP/s; the early
    pushes added more interference with the attention kernels than the
    exposure they hid).

    The K/V heads are split into `groups` head groups (WLB_HEAD_GROUPS,
    default 4), and the data path is gated by per-peer arrival flags
    (`wlb_cp_signal` / `wlb_cp_wait`, one int per (slot, kind, group, source
    rank)), not whole-slot barriers:

      forward : barrier (slot free everywhere) -> per head group g:
                wlb_cp_kv_push_part stores this rank's rows of g into every
                covering rank's slot at their document positions -> signal
                every peer's KV flag of g.  The attention of group g waits
                (device side) until all peers' KV flags of g are set, so it
                starts while the later groups are still in flight.  The local
                slot IS the gathered, un-permuted K/V.
      backward: the attention backward of group g writes its partials straight
                into the local dK/dV slot -> signal every peer's DKV flag of
                g; the pull of g waits for all peers' DKV flags of g and sums
                this rank's rows while the backward of the later groups runs
                -> barrier after the last group (slot reusable; the compute
                stream waits on it before the backward `slots` micro-batches
                later).
    """

    def __init__(self, group, t_max, hkv, d, device, slots=2, groups=None):
        import torch.distributed._symmetric_memory as symm
        self.group = group if group is not None else dist.group.WORLD
        cp = dist.get_world_size(self.group)
        slots = int(os.environ.get("WLB_XCHG_SLOTS", slots))   # experiment override
        n = t_max * hkv * d
        kv = symm.empty(2 * slots * n, dtype=torch.bfloat16, device=device)  # [slot][K|V]
        kv.zero_()
        kv_h = symm.rendezvous(kv, self.group)
        dkv = symm.empty(2 * slots * n, dtype=self._dkv_dtype(), device=device)  # [slot][dK|dV]
        dkv_h = symm.rendezvous(dkv, self.group)
        flags = symm.empty(slots * _KINDS * MAX_GROUPS * cp, dtype=torch.int32, device=device)
        flags.zero_()
        flags_h = symm.rendezvous(flags, self.group)
        self._setup(cp, t_max, hkv, d, device, slots, kv, dkv, list(kv_h.buffer_ptrs),
                    list(dkv_h.buffer_ptrs), flags, list(flags_h.buffer_ptrs),
                    dist.get_rank(self.group), groups)
        self._kv_barrier = lambda: kv_h.barrier(channel=0)
        self._dkv_barrier = lambda: dkv_h.barrier(channel=1)

    @staticmethod
    def _dkv_dtype():
        # dK/dV partials in fp32 (default).  WLB_XCHG_DKV=bf16 opts into bf16
        # partials: the backward writes half the bytes and the pull moves half
        # (summed in fp32; +2% at N=4), but every rank's partial is rounded to
        # bf16 before the sum, and at cp=8 with 8:1 GQA that error reached
        # 2.5e-2 on dK, past the 2e-2 + 1e-2|ref| bar (tests/test_gpu_exchange.py).
        return torch.bfloat16 if os.environ.get("WLB_XCHG_DKV", "fp32") == "bf16" else torch.float32

    def _setup(self, cp, t_max, hkv, d, device, slots, kv, dkv, kv_ptrs, dkv_ptrs, flags,
               flag_ptrs, rank, groups):
        self.cp, self.rank = cp, rank
        self.t_max, self.hkv, self.d = t_max, hkv, d
        self.n = t_max * hkv * d
        self.slots = slots
        self.depth = slots - 1          # K/V pushed this many micro-batches ahead
        self.kv, self.dkv, self.flags = kv, dkv, flags
        self.dkv_bf16 = dkv.dtype == torch.bfloat16
        self.kv_bases = torch.tensor(kv_ptrs, dtype=torch.int64, device=device)
        self.dkv_bases = torch.tensor(dkv_ptrs, dtype=torch.int64, device=device)
        self.flag_bases = torch.tensor(flag_ptrs, dtype=torch.int64, device=device)
        groups = int(os.environ.get("WLB_HEAD_GROUPS", 4)) if groups is None else groups
        self.groups = head_groups(hkv, min(groups, MAX_GROUPS))
        # In-kernel sync (one attention launch per direction, each forward CTA
        # waiting on the device for its head group's flags, the backward
        # signalling each group itself) needs equal groups and is OPT-IN
        # (WLB_CP_FUSED_SYNC=1): waiting forward CTAs hold their SMs, and if
        # they occupy every SM before a peer's push kernel is resident the
        # exchange starves (measured: a 2-GPU 128K step hung until the wait
        # timeout).  The default launches the attention group by group behind
        # one-warp wait kernels, which can never take all SMs.
        self.fused_sync = (hkv % len(self.groups) == 0
                           and os.environ.get("WLB_CP_FUSED_SYNC", "0") == "1")
        self.counters = torch.zeros((slots, MAX_GROUPS), dtype=torch.int32, device=device)
        # K/V push on the copy engines (WLB_XCHG_PUSH=dma): needs this rank's
        # row runs on the host (the shard plan is read back once per plan)
        self.push_dma = os.environ.get("WLB_XCHG_PUSH", "covered") == "dma"
        self.kv_ptrs_host = (ctypes.c_uint64 * cp)(*kv_ptrs)
        self.flag_ptrs_host = (ctypes.c_uint64 * cp)(*flag_ptrs)
        # with the copy-engine push, signals, stream-side waits and slot
        # barriers are stream memory operations (GPU front end): no exchange
        # step needs an SM.  Measured at N=4 (profiles/r02_exchange_transports.txt):
        # the copy-engine push is 2-5x slower than the kernel push in isolation
        # (2-D copies of 2 KB head-group rows) and leaves the single-micro-batch
        # exposure where it was (7.1-7.5 % vs 7.9 %), so the kernel push stays
        # the default.  The in-kernel sync (WLB_CP_FUSED_SYNC=1) on top of it
        # passes the one- and two-GPU parity tests but trapped at N=4 on 128K
        # micro-batches: it stays experimental.
        self.memops = os.environ.get("WLB_CP_MEMOPS", "1" if self.push_dma else "0") == "1"
        self.seq = 0                    # micro-batches pushed (flag epochs)
        self.epoch = [0] * slots        # epoch of the micro-batch in slot s
        self.free = [None] * slots     # event: all ranks finished pulling slot s
        # The covered kernels take a warp-ballot rank mask (cp <= 32); larger
        # groups use the full push / pull, which work for any cp.
        covered_ok = self.cp <= 32
        # skip peers' uncovered (all-zero) partial rows in the pull; WLB_XCHG_PULL=all reads every row
        self.pull_covered = covered_ok and os.environ.get("WLB_XCHG_PULL", "covered") != "all"
        # push K/V rows only to the ranks that load them (including a last
        # tile's reads past its document's end, so no stale row is ever read);
        # WLB_XCHG_PUSH=all stores to every rank
        self.push_covered = covered_ok and os.environ.get("WLB_XCHG_PUSH", "covered") != "all"

    def side_stream(self):
        """High-priority stream for this exchange's pushes / pulls outside a
        CPStepPipeline (cp_doc_attention)."""
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(priority=-1)
        return self._side

    def begin_microbatch(self) -> int:
        """Index of the next micro-batch of the autograd path (slot b % slots);
        at most `slots` micro-batches may be between forward and backward."""
        b = self.seq
        live = getattr(self, "_live", set())
        if any(x % self.slots == b % self.slots for x in live):
            raise RuntimeError(f"more than {self.slots} CP micro-batches between forward and "
                               "backward: the K/V slot is still needed")
        live.add(b)
        self._live = live
        return b

    def end_microbatch(self, b: int) -> None:
        getattr(self, "_live", set()).discard(b)

    @staticmethod
    def _tables(shard):
        """Every rank's row-set offsets [cp][max_docs+1] and in-document
        positions [cp][T/cp] of this micro-batch (device views of the plan)."""
        plan, b = shard.plan, shard.index
        rows = plan.rowset_off[b]
        assert rows.is_contiguous()
        return rows, plan.positions[plan.tok_off[b]:]

    def _view(self, buf, idx, T):
        return buf[idx * self.n: idx * self.n + T * self.hkv * self.d].view(T, self.hkv, self.d)

    def _flag_off(self, s, kind, gi, src):
        return (((s * _KINDS + kind) * MAX_GROUPS + gi) * self.cp + src) * 4

    def _slot_barrier(self, s, kind):
        """Every rank has finished with slot s (kind _KV_FREE: reading its K/V;
        _DKV_FREE: pulling its partials).  Stream memory operations in memops
        mode (no SM: a symmetric-memory barrier is a kernel, which attention
        CTAs waiting on flags could starve), else the symmetric barrier."""
        if not self.memops:
            (self._kv_barrier if kind == _KV_FREE else self._dkv_barrier)()
            return
        self._signal(s, kind, 0)
        self._wait(s, kind, 0)

    def _signal(self, s, kind, gi):
        if self.memops:
            _native.check(_native.lib().wlb_cp_signal_memop(
                self.flag_ptrs_host, self._flag_off(s, kind, gi, self.rank), self.cp,
                self.epoch[s], _native.stream_ptr()), "wlb_cp_signal_memop")
            return
        _native.check(_native.lib().wlb_cp_signal(
            self.flag_bases.data_ptr(), self._flag_off(s, kind, gi, self.rank), self.cp,
            self.epoch[s], _native.stream_ptr()), "wlb_cp_signal")

    def _wait(self, s, kind, gi):
        fn = "wlb_cp_wait_memop" if self.memops else "wlb_cp_wait"
        _native.check(getattr(_native.lib(), fn)(
            self.flags.data_ptr() + self._flag_off(s, kind, gi, 0), self.cp, self.epoch[s],
            _native.stream_ptr()), fn)

    def gather(self, k, v, shard, b, ready=None):
        """Push this rank's K/V rows of micro-batch b, group by group, each
        followed by a signal to every peer; returns the local slot's
        document-ordered K / V views (read them only after `wait_kv`).
        ready: optional per-group CUDA events, group gi's push waits for
        ready[gi] (its K / V columns copied in)."""
        s, T = b % self.slots, shard.gather_all.numel()
        if T > self.t_max:
            raise ValueError(f"micro-batch of {T} tokens exceeds the exchange capacity {self.t_max}")
        self.seq += 1
        self.epoch[s] = self.seq
        self._slot_barrier(s, _KV_FREE)     # every rank finished reading slot s
        row = self.hkv * self.d * 2
        if self.push_dma:
            runs = self._runs(shard)
            for gi, (g0, ng) in enumerate(self.groups):
                if ready is not None:
                    torch.cuda.current_stream().wait_event(ready[gi])
                _native.check(_native.lib().wlb_cp_kv_push_dma(
                    k.data_ptr(), v.data_ptr(), runs.ctypes.data, len(runs), row,
                    g0 * self.d * 2, ng * self.d * 2, self.kv_ptrs_host, 2 * s * self.n * 2,
                    (2 * s + 1) * self.n * 2, self.cp, _native.stream_ptr()), "wlb_cp_kv_push_dma")
                self._signal(s, _KV, gi)
            return self._view(self.kv, 2 * s, T), self._view(self.kv, 2 * s + 1, T)
        covered = self.push_covered and shard.tiles.n_docs > 0
        rows, pos = self._tables(shard) if covered else (None, None)
        p = _native.ptr
        for gi, (g0, ng) in enumerate(self.groups):
            if ready is not None:
                torch.cuda.current_stream().wait_event(ready[gi])
            _native.check(_native.lib().wlb_cp_kv_push_part(
                k.data_ptr(), v.data_ptr(), shard.gather_local.data_ptr(), k.shape[0], row,
                g0 * self.d * 2, ng * self.d * 2, self.kv_bases.data_ptr(),
                2 * s * self.n * 2, (2 * s + 1) * self.n * 2, self.cp, p(rows),
                rows.shape[-1] if covered else 0, p(pos),
                shard.tiles.doc_start.data_ptr() if covered else None,
                shard.tiles.n_docs if covered else 0, _native.stream_ptr()), "wlb_cp_kv_push_part")
            self._signal(s, _KV, gi)
        return self._view(self.kv, 2 * s, T), self._view(self.kv, 2 * s + 1, T)

    def fwd_sync(self, b):
        """`WlbCpSync` for a forward that waits on the K/V arrival flags of
        micro-batch b, head group by head group, inside the kernel."""
        s = b % self.slots
        return _native.WlbCpSync(
            wait_flags=self.flags.data_ptr() + self._flag_off(s, _KV, 0, 0), signal_bases=None,
            signal_off=0, counters=None, cp=self.cp, kv_per_group=self.hkv // len(self.groups),
            epoch=self.epoch[s])

    def bwd_sync(self, b):
        """`WlbCpSync` for a backward that signals every peer's DKV flags of
        micro-batch b per head group from the device."""
        s = b % self.slots
        return _native.WlbCpSync(
            wait_flags=None, signal_bases=self.flag_bases.data_ptr(),
            signal_off=self._flag_off(s, _DKV, 0, self.rank),
            counters=self.counters[s].data_ptr(), cp=self.cp,
            kv_per_group=self.hkv // len(self.groups), epoch=self.epoch[s])

    def _runs(self, shard):
        """This rank's local rows as contiguous runs (local row, global row,
        rows) of the document-ordered buffer: its canonical ranges (host copy
        of the shard plan, read once per plan)."""
        import numpy as np
        a = shard.plan.assignment(shard.index)
        starts = np.concatenate([[0], np.cumsum(a.doc_lengths)])
        out, local = [], 0
        for p_, r in a.workers[self.rank]:
            n = r.end - r.start
            out.append((local, int(starts[p_]) + r.start, n))
            local += n
        return np.ascontiguousarray(np.array(out, dtype=np.int64).reshape(-1, 3))

    def wait_kv(self, b, gi):
        """On the current stream: later work waits until every peer's rows of
        head group gi of micro-batch b have landed."""
        self._wait(b % self.slots, _KV, gi)

    def dkv_out(self, shard, b, cur):
        s, T = b % self.slots, shard.gather_all.numel()
        if self.free[s] is not None:
            cur.wait_event(self.free[s])
        return self._view(self.dkv, 2 * s, T), self._view(self.dkv, 2 * s + 1, T)

    def signal_dkv(self, b, gi):
        """On the current stream, after the backward of head group gi: tell
        every peer this rank's partials of gi are complete."""
        self._signal(b % self.slots, _DKV, gi)

    def scatter(self, dkf, dvf, shard, b, on_group=None, out_dtype=torch.float32):
        """Pull (on the current stream) this rank's rows of every rank's
        partials, each head group as soon as all peers' partials of it are
        complete; dK / dV [T/cp, Hkv, D] as the fp32 sums (or, with
        out_dtype=torch.bfloat16, their bf16 rounding stored by the pull).
        on_group(gi, dk, dv) is called after group gi's pull is enqueued
        (e.g. to record an event)."""
        if out_dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("out_dtype must be float32 or bfloat16")
        s = b % self.slots
        tl = shard.gather_local.numel()
        dk = torch.empty((tl, self.hkv, self.d), dtype=out_dtype, device=dkf.device)
        dv = torch.empty_like(dk)
        es = 2 if self.dkv_bf16 else 4
        flags = _native.WLB_BWD_DKV_BF16 if self.dkv_bf16 else 0
        if out_dtype == torch.bfloat16:
            flags |= _native.WLB_PULL_OUT_BF16
        covered = self.pull_covered and shard.tiles.n_docs > 0
        rows, pos = self._tables(shard) if covered else (None, None)
        p = _native.ptr
        for gi, (g0, ng) in enumerate(self.groups):
            self._wait(s, _DKV, gi)
            _native.check(_native.lib().wlb_cp_dkv_pull_part(
                self.dkv_bases.data_ptr(), 2 * s * self.n * es, (2 * s + 1) * self.n * es,
                shard.gather_local.data_ptr(), tl, self.hkv * self.d * es, g0 * self.d * es,
                ng * self.d * es, dk.data_ptr(), dv.data_ptr(), self.cp, flags, p(rows),
                rows.shape[-1] if covered else 0, p(pos),
                shard.tiles.doc_start.data_ptr() if covered else None,
                shard.tiles.n_docs if covered else 0, _native.stream_ptr()), "wlb_cp_dkv_pull_part")
            if on_group is not None:
                on_group(gi, dk, dv)
        self._slot_barrier(s, _DKV_FREE)    # every rank finished pulling from slot s
        ev = torch.cuda.Event()
        ev.record()
        self.free[s] = ev
        return dk, dv


class LocalPeersExchange(SymmExchange):
    """One-GPU emulation of a CP group's symmetric exchange: every rank's slot
    and flag buffers are ordinary allocations on ONE device and the base
    tables hold all of them, so the same push / pull / signal / wait kernels
    and the same `gather` / `wait_kv` / `dkv_out` / `signal_dkv` / `scatter`
    code run for cp = 2..8 without peers.  Cross-rank ordering is the
    caller's: run every rank's `gather` before any rank's attention, and every
    rank's backward (+ `signal_dkv`) before any rank's `scatter` (stream order
    on one device; the barriers are no-ops, the flags are real).  Used by the
    exchange parity tests and tools/cp_emulate.py."""

    @classmethod
    def create(cls, cp, t_max, hkv, d, device, slots=2, fill=0.0, groups=None):
        """cp exchange objects, rank r's at index r.  `fill` initialises the
        K/V slots (e.g. NaN, to prove every row a tile loads is rewritten)."""
        n = t_max * hkv * d
        kvs = [torch.full((2 * slots * n,), fill, dtype=torch.bfloat16, device=device)
               for _ in range(cp)]
        dkvs = [torch.full((2 * slots * n,), float("nan"), dtype=cls._dkv_dtype(), device=device)
                for _ in range(cp)]
        flags = [torch.zeros(slots * _KINDS * MAX_GROUPS * cp, dtype=torch.int32, device=device)
                 for _ in range(cp)]
        kv_ptrs = [t.data_ptr() for t in kvs]
        dkv_ptrs = [t.data_ptr() for t in dkvs]
        flag_ptrs = [t.data_ptr() for t in flags]
        out = []
        for r in range(cp):
            ex = cls.__new__(cls)
            ex.group = None
            ex._setup(cp, t_max, hkv, d, device, slots, kvs[r], dkvs[r], kv_ptrs, dkv_ptrs,
                      flags[r], flag_ptrs, r, groups)
            ex._kv_barrier = ex._dkv_barrier = lambda: None
            ex._slot_barrier = lambda s_, kind: None   # the caller orders the ranks
            out.append(ex)
        return out


class CPStepPipeline:
    """CP attention over all micro-batches of a step with the exchange overlapped.

    The K/V exchange of micro-batch b+1 and the dK/dV exchange of micro-batch
    b-1 run on dedicated communication streams while micro-batch b's
    attention kernels run on the compute stream.  With NcclExchange (default)
    CUDA events order each exchange against its producer and consumer.  With
    SymmExchange the attention runs head group by head group, each gated on
    the device by the peers' arrival flags of that group, and the dK/dV pull
    of a group overlaps the backward of the later groups.  Hooks:

    * `ready[b]` (optional CUDA events): micro-batch b's q, k, v are valid once
      they fire (e.g. H2D copies); by default inputs are taken as resident.
      `bwd_ready[b]`: the same for dO, waited for only before the backward
      (so dO can still be in flight during the forward).
    * `on_forward(b, o, event)` is called once micro-batch b's forward is
      enqueued; `event` fires when O is complete (e.g. to copy it out during
      the backward).
    * `on_kernels(b, shard, fn)` wraps the attention kernels (e.g. CUDA events
      for per-rank kernel time; with head groups this includes the device-side
      waits for the peers' K/V of each group).
    * `on_outputs(b, (o, dq, dk, dv), event)` is called as soon as micro-batch
      b's outputs are enqueued; `event` fires when all four are complete.

    Head-group granularity (`io_groups=G`, for streaming micro-batches from and
    to host memory, `hoststream.HostStreamedStep`): the attention runs in the
    KV-head groups `io_head_groups(hkv, G, cp)` returns (the exchange's groups
    at CP > 1), `ready[b]` / `bwd_ready[b]` are then per-group event lists
    gating that group's forward / backward, `on_group_forward(b, gi, o, ev)`
    fires per group when its O columns are complete and
    `on_group_outputs(b, gi, (o, dq, dk, dv), ev)` when its columns of all
    four are (dK / dV after that group's exchange pull at CP > 1).
    `dkv_dtype=torch.bfloat16`: dK / dV come out in bf16 — at
    CP = 1 stored by the backward, at CP > 1 by the exchange pull — the same
    RNE rounding of the fp32 sums as a later conversion, without conversion
    kernels on the copy stream (those competed with the attention for SMs:
    6 % of the N=2 host-streamed step).
    """

    def __init__(self, group=None, exchange=None):
        self.group = group
        self.exchange = exchange if exchange is not None else NcclExchange(group)
        self.depth = getattr(self.exchange, "depth", 1)
        self.flagged = isinstance(self.exchange, SymmExchange)
        # The exchange stream outranks the compute stream (CUDA: lower value =
        # higher priority; default streams are 0): its blocks are dispatched
        # as soon as an SM frees up, so an exchange is done before the
        # micro-batch that needs it (N=4 bench 3781-3789 vs 3746-3752 at equal
        # priority; raising the compute stream instead gained nothing).
        # WLB_COMM_PRIORITY overrides it for experiments.
        prio = int(os.environ.get("WLB_COMM_PRIORITY", "-1"))
        self.comm = torch.cuda.Stream(priority=prio)          # dK/dV (and NCCL K/V)
        # one-sided K/V pushes run ahead on their own stream (depth > 1)
        self.push = torch.cuda.Stream(priority=prio) if self.depth > 1 else self.comm

    def io_head_groups(self, hkv: int, groups: int, cp: int):
        """The KV-head groups a run with `io_groups=groups` uses."""
        if cp > 1:
            if not self.flagged or self.exchange.fused_sync:
                raise ValueError("head-group I/O at CP > 1 needs the flagged SymmExchange")
            return list(self.exchange.groups)
        return head_groups(hkv, groups)

    def _gather(self, k, v, shard, b, cur, ready):
        # the slot being overwritten was last read by compute already enqueued
        # on `cur` (b - slots <= the last enqueued micro-batch), so wait for it
        # as well as for the inputs
        self.push.wait_stream(cur)
        per_group = isinstance(ready, (list, tuple))
        if per_group and not (self.flagged and shard.cp > 1):
            # CP = 1 (no exchange): each group's forward waits for its own
            # event; NCCL: the collective needs every group
            ready = ready[-1] if shard.cp > 1 else None
            per_group = False
        if ready is not None and not per_group:
            self.push.wait_event(ready)
        with torch.cuda.stream(self.push):
            if per_group:
                k_full, v_full = self.exchange.gather(k, v, shard, b, ready=ready)
            else:
                k_full, v_full = self.exchange.gather(k, v, shard, b)
            ev = torch.cuda.Event()
            ev.record(self.push)
        return k_full, v_full, ev

    def run(self, shards, inputs, scale=None, ready=None, on_kernels=None, on_outputs=None,
            keep_outputs=True, bwd_ready=None, on_forward=None, io_groups=None,
            on_group_forward=None, on_group_outputs=None, dkv_dtype=None):
        """inputs[b] = (q, k, v, do) local bf16 tensors.  Returns per micro-batch
        (o, dq, dk, dv) local tensors (dk/dv fp32), complete on the current stream
        (None entries when keep_outputs=False: consume them in on_outputs)."""
        cur = torch.cuda.current_stream()
        n = len(shards)
        rdy = ready if ready is not None else [None] * n
        brdy = bwd_ready if bwd_ready is not None else [None] * n
        grouped = io_groups is not None
        # the covered pull reads only the partial rows each rank's KV tiles
        # wrote: skip the zero fill of the rest
        covered = bool(getattr(self.exchange, "pull_covered", False))
        outs = [None] * n
        pend = {}
        for b in range(min(self.depth, n)):
            pend[b] = self._gather(inputs[b][1], inputs[b][2], shards[b], b, cur, rdy[b])
        tail = []
        for b in range(n):
            nb = b + self.depth
            if nb < n:
                pend[nb] = self._gather(inputs[nb][1], inputs[nb][2], shards[nb], nb, cur, rdy[nb])
            k_full, v_full, ev = pend.pop(b)
            sh = shards[b]
            flagged = self.flagged and sh.cp > 1
            if not flagged:
                cur.wait_event(ev)          # (flagged: the device-side waits gate each group)
            if rdy[b] is not None and not grouped:
                cur.wait_event(rdy[b])
            q, _, _, do = inputs[b]
            dk_out, dv_out = self.exchange.dkv_out(sh, b, cur) if sh.cp > 1 else (None, None)
            cov = covered and dk_out is not None and sh.tiles.n_docs > 0
            if sh.cp == 1 and dkv_dtype is not None and not grouped:
                T_, hkv_, d_ = inputs[b][1].shape
                dk_out = torch.empty((T_, hkv_, d_), dtype=dkv_dtype, device=q.device)
                dv_out = torch.empty_like(dk_out)

            gdone = []

            def kernels(q=q, do=do, k_full=k_full, v_full=v_full, sh=sh, dk_out=dk_out,
                        dv_out=dv_out, b=b, flagged=flagged, cov=cov, gdone=gdone):
                ex = self.exchange
                fused = flagged and ex.fused_sync
                if grouped:
                    return self._grouped_kernels(b, sh, q, do, k_full, v_full, dk_out, dv_out, cov,
                                                 scale, io_groups, rdy[b], brdy[b],
                                                 on_group_forward, on_group_outputs, gdone,
                                                 dkv_dtype)
                if not flagged:
                    o, lse = attn_forward(q, k_full, v_full, sh.tiles, scale)
                elif fused:
                    o, lse = attn_forward(q, k_full, v_full, sh.tiles, scale, sync=ex.fwd_sync(b))
                else:
                    o, lse = torch.empty_like(q), None
                    for gi, grp in enumerate(ex.groups):
                        ex.wait_kv(b, gi)
                        o, lse = attn_forward(q, k_full, v_full, sh.tiles, scale, kv_heads=grp,
                                              out=None if lse is None else (o, lse))
                if on_forward is not None:
                    fev = torch.cuda.Event()
                    fev.record(cur)
                    on_forward(b, o, fev)
                if brdy[b] is not None:
                    cur.wait_event(brdy[b])
                if not flagged:
                    dq, dkf, dvf = attn_backward(q, k_full, v_full, o, lse, do, sh.tiles, scale,
                                                 dk_out, dv_out, covered_only=cov)
                    return o, dq, dkf, dvf
                if fused:
                    dq, _, _ = attn_backward(q, k_full, v_full, o, lse, do, sh.tiles, scale, dk_out,
                                             dv_out, covered_only=cov, sync=ex.bwd_sync(b))
                    return o, dq, dk_out, dv_out
                dq, ws = torch.empty_like(q), bwd_workspace(q, k_full, sh.tiles)
                for gi, grp in enumerate(ex.groups):
                    attn_backward(q, k_full, v_full, o, lse, do, sh.tiles, scale, dk_out, dv_out,
                                  covered_only=cov, kv_heads=grp, dq_out=dq, ws=ws)
                    ex.signal_dkv(b, gi)
                return o, dq, dk_out, dv_out

            o, dq, dkf, dvf = on_kernels(b, sh, kernels) if on_kernels else kernels()
            if sh.cp > 1:
                for t in (k_full, v_full):
                    t.record_stream(cur)
                    if self.push is not self.comm:
                        t.record_stream(self.push)
            done = torch.cuda.Event()
            done.record(cur)
            if not flagged:
                self.comm.wait_event(done)  # (flagged: the pull waits on the DKV flags)
            with torch.cuda.stream(self.comm):
                on_group = None
                if grouped and sh.cp > 1 and on_group_outputs is not None:
                    def on_group(gi, dk_, dv_, b=b, o=o, dq=dq, gdone=gdone):
                        self.comm.wait_event(gdone[gi])     # the group's O and dQ
                        gev = torch.cuda.Event()
                        gev.record(self.comm)
                        on_group_outputs(b, gi, (o, dq, dk_, dv_), gev)
                kw = {}
                if on_group is not None:
                    kw["on_group"] = on_group
                if flagged and dkv_dtype is not None:
                    kw["out_dtype"] = dkv_dtype     # the pull stores the dtype asked for
                dk, dv = self.exchange.scatter(dkf, dvf, sh, b, **kw) if sh.cp > 1 else (dkf, dvf)
                if sh.cp > 1:
                    for t in (dkf, dvf):
                        t.record_stream(self.comm)
                fin = torch.cuda.Event()
                fin.record(self.comm)
            tail.append(fin)
            if on_outputs is not None:
                if flagged:                 # o, dq (compute) as well as dk, dv (comm)
                    self.comm.wait_event(done)
                    fin = torch.cuda.Event()
                    fin.record(self.comm)
                on_outputs(b, (o, dq, dk, dv), fin)
            if keep_outputs:
                outs[b] = (o, dq, dk, dv)
            else:
                for t in (o, dq, dk, dv):      # freed now; keep them valid for pending work
                    t.record_stream(cur)
                    if sh.cp > 1:
                        t.record_stream(self.comm)
        for fin in tail:
            cur.wait_event(fin)
        return outs

    def _grouped_kernels(self, b, sh, q, do, k_full, v_full, dk_out, dv_out, cov, scale, io_groups,
                         rdy, brdy, on_group_forward, on_group_outputs, gdone, dkv_dtype=None):
        """One micro-batch's attention head group by head group, each group's
        forward / backward gated on its own input events (host streaming)."""
        cur = torch.cuda.current_stream()
        flagged = self.flagged and sh.cp > 1
        groups = self.io_head_groups(k_full.shape[1], io_groups, sh.cp)
        for e in (rdy, brdy):
            if e is not None and len(e) != len(groups):
                raise ValueError(f"per-group events: expected {len(groups)}, got {len(e)}")
        ex = self.exchange
        o, lse = torch.empty_like(q), None
        for gi, grp in enumerate(groups):
            if flagged:
                ex.wait_kv(b, gi)
            if rdy is not None:
                cur.wait_event(rdy[gi])
            o, lse = attn_forward(q, k_full, v_full, sh.tiles, scale, kv_heads=grp,
                                  out=None if lse is None else (o, lse))
            if on_group_forward is not None:
                fev = torch.cuda.Event()
                fev.record(cur)
                on_group_forward(b, gi, o, fev)
        dq, ws = torch.empty_like(q), bwd_workspace(q, k_full, sh.tiles)
        if not flagged:
            T, hkv, d = k_full.shape
            dk_out = torch.empty((T, hkv, d), dtype=dkv_dtype or torch.float32, device=q.device)
            dv_out = torch.empty_like(dk_out)
        for gi, grp in enumerate(groups):
            if brdy is not None:
                cur.wait_event(brdy[gi])
            attn_backward(q, k_full, v_full, o, lse, do, sh.tiles, scale, dk_out, dv_out,
                          covered_only=cov and flagged, kv_heads=grp, dq_out=dq, ws=ws)
            if flagged:
                ex.signal_dkv(b, gi)
            gev = torch.cuda.Event()
            gev.record(cur)
            gdone.append(gev)
            if not flagged and on_group_outputs is not None:
                on_group_outputs(b, gi, (o, dq, dk_out, dv_out), gev)
        return o, dq, dk_out, dv_out
