"""Context-parallel sharding, balsim-compatible API on the GPU shard builder.

Drop-in for `/root/reference/pkg/src/balsim/sharding.py:36-200`: the same
names, signatures, canonical-range output (`ShardAssignment`), exceptions
(`ValueError` for cp < 1, non-divisible lengths, unknown policies) and
selection rule (per-sequence when its modelled group latency is <= the
per-document one).  The difference is where the work runs: every function
here launches `wlb_shard_plan` / `wlb_kernel_latency_sum`
(`csrc/shard_plan.cu`) on the current CUDA device -- there is no CPU fallback.

`build_shard_plan` is the batched, device-resident form used by the attention
path: it builds (and, under the adaptive policy, selects) the shards of many
micro-batches in one launch and keeps gather indices, in-document positions
and per-(rank, document) row-set offsets on the GPU.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import torch

from . import _native
from .tilemodel import FEATURES, TileModel
from .workload import CostProfile, MicroBatch, TokenRange

_DEFAULT_PROFILE = CostProfile()


class ShardStrategy(str, enum.Enum):
    """`sharding.py:36-41`."""

    PER_SEQUENCE = "per_sequence"
    PER_DOCUMENT = "per_document"

    def __str__(self) -> str:
        return self.value


_STRATS = (ShardStrategy.PER_SEQUENCE, ShardStrategy.PER_DOCUMENT)
_POLICY_CODE = {"per_sequence": 0, "per_document": 1, "adaptive": 2, "measured": 3}


@dataclass
class ShardAssignment:
    """Per-worker canonical ranges of one micro-batch (`sharding.py:44-60`)."""

    strategy: ShardStrategy
    cp: int
    doc_ids: list[int]
    doc_lengths: list[int]
    workers: list[list[tuple[int, TokenRange]]] = field(default_factory=list)

    def worker_token_count(self, worker: int) -> int:
        return sum(len(r) for _, r in self.workers[worker])


def _check_divisible(total: int, cp: int) -> None:
    """`sharding.py:77-83`."""
    if cp < 1:
        raise ValueError("cp must be >= 1")
    if total % (2 * cp) != 0:
        raise ValueError(f"micro-batch length {total} not divisible by 2*cp = {2 * cp}; "
                         "pad with a filler document first")


@dataclass
class ShardPlan:
    """Device-resident output of one batched `wlb_shard_plan` launch."""

    cp: int
    lengths: list[list[int]]          # host copy of the inputs
    doc_ids: list[list[int]]
    tok_off: list[int]                # token offset of each micro-batch
    choice: torch.Tensor              # [n_mb] int32
    rank_latency: torch.Tensor        # [n_mb, 2, cp] float64
    rank_pairs: torch.Tensor          # [n_mb, cp] int64
    seg_count: torch.Tensor           # [n_mb, 2, cp] int32
    segs: torch.Tensor                # [n_mb, 2, cp, max_segs, 3] int32
    rowset_off: torch.Tensor          # [n_mb, cp, max_docs+1] int32
    gather_index: torch.Tensor | None  # [sum T] int32
    positions: torch.Tensor | None     # [sum T] int32
    # measured-latency model path only: the model and the per-(strategy,
    # rank) work-list features it priced, [n_mb, 2, cp, 8] int64 (FEATURES)
    model: TileModel | None = None
    features: torch.Tensor | None = None
    _host: dict = field(default_factory=dict)

    @property
    def n_mb(self) -> int:
        return len(self.lengths)

    def host(self, name: str):
        if name not in self._host:
            self._host[name] = getattr(self, name).cpu()
        return self._host[name]

    def strategy(self, b: int) -> ShardStrategy:
        return _STRATS[int(self.host("choice")[b])]

    def assignment(self, b: int, strategy: ShardStrategy | None = None) -> ShardAssignment:
        strategy = self.strategy(b) if strategy is None else strategy
        s = _STRATS.index(strategy)
        counts = self.host("seg_count")[b, s].tolist()
        segs = self.host("segs")[b, s]
        workers = []
        for w in range(self.cp):
            rows = segs[w, :counts[w]].tolist()
            workers.append([(p, TokenRange(a, e)) for p, a, e in rows])
        return ShardAssignment(strategy=strategy, cp=self.cp, doc_ids=list(self.doc_ids[b]),
                               doc_lengths=list(self.lengths[b]), workers=workers)

    def group_latency(self, b: int, strategy: ShardStrategy) -> float:
        return float(self.host("rank_latency")[b, _STRATS.index(strategy)].max())

    def rank_local(self, b: int, rank: int):
        """(gather_index, positions, rowset_off[n_docs+1]) device views for one rank."""
        T = sum(self.lengths[b])
        n = T // self.cp
        lo = self.tok_off[b] + rank * n
        nd = len(self.lengths[b])
        return (self.gather_index[lo:lo + n], self.positions[lo:lo + n],
                self.rowset_off[b, rank, :nd + 1])


def build_shard_plan(microbatches, cp: int, policy: str = "adaptive",
                     profile: CostProfile | None = None, with_tokens: bool = True,
                     device=None, model: TileModel | None = None) -> ShardPlan:
    """Shard (and select) many micro-batches in one GPU launch.

    `microbatches`: MicroBatch objects or plain length lists.  Raises
    ValueError exactly where the reference would (`sharding.py:77-83,200`).

    policy "adaptive" selects with the reference CostProfile (bit-exact with
    balsim); "measured" selects with the B200 tile model (`tilemodel.py`,
    `model` or the shipped calibration for the default 32 x 128 shape) and
    also fills `features`.  Passing `model` with "per_sequence" /
    "per_document" prices both strategies with it without selecting.
    """
    if policy not in _POLICY_CODE:
        raise ValueError(f"unknown sharding policy {policy!r}")
    profile = _DEFAULT_PROFILE if profile is None else profile
    lengths, ids = [], []
    for mb in microbatches:
        if isinstance(mb, MicroBatch):
            lengths.append(mb.lengths())
            ids.append([d.id for d in mb.docs])
        else:
            lengths.append([int(x) for x in mb])
            ids.append(list(range(len(lengths[-1]))))
    for ls in lengths:
        _check_divisible(sum(ls), cp)
    _native.require_device()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    n_mb = len(lengths)
    max_docs = max(1, max(len(x) for x in lengths))
    max_segs = 4 * max_docs + 2
    doc_off, tok_off = [0], [0]
    for ls in lengths:
        doc_off.append(doc_off[-1] + len(ls))
        tok_off.append(tok_off[-1] + sum(ls))
    i32 = dict(dtype=torch.int32, device=dev)
    flat = [x for ls in lengths for x in ls] or [0]
    up = _native.to_device        # no host sync: the step can be enqueued ahead
    d_doc_off = up(doc_off, torch.int32, dev)
    d_len = up(flat, torch.int64, dev)
    d_tok = up(tok_off, torch.int64, dev)
    cq, cv = profile.curve_arrays()
    d_cq = up(cq, torch.int64, dev)
    d_cv = up(cv, torch.float64, dev)
    choice = torch.empty(n_mb, **i32)
    lat = torch.empty((n_mb, 2, cp), dtype=torch.float64, device=dev)
    pairs = torch.empty((n_mb, cp), dtype=torch.int64, device=dev)
    seg_count = torch.empty((n_mb, 2, cp), **i32)
    segs = torch.empty((n_mb, 2, cp, max_segs, 3), **i32)
    rowset = torch.empty((n_mb, cp, max_docs + 1), **i32)
    gidx = torch.empty(tok_off[-1], **i32) if with_tokens else None
    pos = torch.empty(tok_off[-1], **i32) if with_tokens else None
    p = _native.ptr
    if policy == "measured" or model is not None:
        if policy == "adaptive":
            raise ValueError("a tile model prices the 'measured' policy, not 'adaptive'")
        model = TileModel.for_shape(32, 32, 128) if model is None else model
        d_model = up(model.array(), torch.float64, dev)
        feats = torch.empty((n_mb, 2, cp, len(FEATURES)), dtype=torch.int64, device=dev)
        _native.check(_native.lib().wlb_shard_plan_measured(
            n_mb, p(d_doc_off), p(d_len), p(d_tok), cp, _POLICY_CODE[policy], p(d_model),
            max_segs, max_docs, p(choice), p(lat), p(pairs), p(seg_count), p(segs), p(rowset),
            p(gidx), p(pos), p(feats), _native.stream_ptr()), "wlb_shard_plan_measured")
        return ShardPlan(cp=cp, lengths=lengths, doc_ids=ids, tok_off=tok_off[:-1],
                         choice=choice, rank_latency=lat, rank_pairs=pairs, seg_count=seg_count,
                         segs=segs, rowset_off=rowset, gather_index=gidx, positions=pos,
                         model=model, features=feats)
    _native.check(_native.lib().wlb_shard_plan(
        n_mb, p(d_doc_off), p(d_len), p(d_tok), cp, _POLICY_CODE[policy], profile.tile_size,
        p(d_cq), p(d_cv), len(cq), profile.op_scale, max_segs, max_docs, p(choice), p(lat),
        p(pairs), p(seg_count), p(segs), p(rowset), p(gidx), p(pos), _native.stream_ptr()),
        "wlb_shard_plan")
    return ShardPlan(cp=cp, lengths=lengths, doc_ids=ids, tok_off=tok_off[:-1], choice=choice,
                     rank_latency=lat, rank_pairs=pairs, seg_count=seg_count, segs=segs,
                     rowset_off=rowset, gather_index=gidx, positions=pos)


def per_sequence_shard(mb: MicroBatch, cp: int) -> ShardAssignment:
    """`sharding.py:86-110` on the GPU builder."""
    plan = build_shard_plan([mb], cp, "per_sequence", with_tokens=False)
    return plan.assignment(0, ShardStrategy.PER_SEQUENCE)


def per_document_shard(mb: MicroBatch, cp: int) -> ShardAssignment:
    """`sharding.py:113-141` on the GPU builder."""
    plan = build_shard_plan([mb], cp, "per_document", with_tokens=False)
    return plan.assignment(0, ShardStrategy.PER_DOCUMENT)


def worker_attention_latency(assignment: ShardAssignment, worker: int,
                             profile: CostProfile) -> float:
    """Tile-padded model latency of one worker's ranges (`sharding.py:151-161`),
    summed on the GPU in canonical order (bit-identical to the reference)."""
    ranges = assignment.workers[worker]
    if not ranges:
        return 0.0
    _native.require_device()
    dev = torch.device("cuda", torch.cuda.current_device())
    q = torch.tensor([r.end - r.start for _, r in ranges], dtype=torch.int64, device=dev)
    kv = torch.tensor([r.end for _, r in ranges], dtype=torch.int64, device=dev)
    cq, cv = profile.curve_arrays()
    d_cq = torch.tensor(cq, dtype=torch.int64, device=dev)
    d_cv = torch.tensor(cv, dtype=torch.float64, device=dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    p = _native.ptr
    _native.check(_native.lib().wlb_kernel_latency_sum(
        p(q), p(kv), len(ranges), profile.tile_size, p(d_cq), p(d_cv), len(cq), profile.op_scale,
        p(out), _native.stream_ptr()), "wlb_kernel_latency_sum")
    return float(out.item())


def group_attention_latency(assignment: ShardAssignment, profile: CostProfile) -> float:
    """Slowest worker (`sharding.py:164-168`)."""
    return max(worker_attention_latency(assignment, w, profile) for w in range(assignment.cp))


def strategy_latencies(mb: MicroBatch, cp: int, profile: CostProfile) -> dict:
    """Group latency of both strategies (`sharding.py:171-179`), one GPU launch."""
    plan = build_shard_plan([mb], cp, "adaptive", profile, with_tokens=False)
    return {s: plan.group_latency(0, s) for s in _STRATS}


def adaptive_select(mb: MicroBatch, cp: int, profile: CostProfile) -> ShardAssignment:
    """Cheaper strategy, ties -> per-sequence (`sharding.py:182-188`).  Both
    strategies are built and priced once, on the GPU, and the winner is
    returned directly (the reference builds it a second time)."""
    plan = build_shard_plan([mb], cp, "adaptive", profile, with_tokens=False)
    return plan.assignment(0)


def shard(mb: MicroBatch, cp: int, policy: str, profile: CostProfile) -> ShardAssignment:
    """Policy dispatch (`sharding.py:191-200`)."""
    if policy == "adaptive":
        return adaptive_select(mb, cp, profile)
    if policy == ShardStrategy.PER_SEQUENCE.value:
        return per_sequence_shard(mb, cp)
    if policy == ShardStrategy.PER_DOCUMENT.value:
        return per_document_shard(mb, cp)
    raise ValueError(f"unknown sharding policy {policy!r}")
