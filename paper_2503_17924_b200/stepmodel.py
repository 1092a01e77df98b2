"""Measured CP attention latency into the reference's pipeline step model.

SURVEY.md §8(f) row 4.  The reference prices a micro-batch's pipeline stage
from the MODELLED CP-group attention latency
(`/root/reference/pkg/src/balsim/pipeline.py:28-86,150-154`,
`harness.py:340-390`):

    forward  = (group_attention_latency + linear(T/cp)) / pp
    backward = backward_ratio * forward
    step     = sum(f_i + b_i) + (pp - 1) * max(f_i + b_i)      (1F1B critical path)

This module keeps those types and formulas (`StageLatency`, `StepReport`,
`stage_latency_for_assignment`, `pp_critical_path`, `dp_step_latency`) and
adds the measured variant: the attention term is the slowest CP rank's
CUDA-event time of this repo's forward / backward kernels, so the reference's
offline pipeline analysis can run on real B200 numbers:

    forward  = (max_r t_fwd_r + linear(T/cp)) / pp
    backward = (max_r t_bwd_r + backward_ratio * linear(T/cp)) / pp

(the linear ops are outside this path and stay modelled).  The event-driven
1F1B simulator (`pipeline.py:89-147`) is the reference's PP simulator and is
out of scope; `event_makespan` is left None.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .attention import attn_backward, attn_forward
from .packing import imbalance_degree_attention, imbalance_degree_latency
from .sharding import ShardAssignment, group_attention_latency, shard
from .workload import (CostProfile, Document, MicroBatch, ParallelismConfig, attention_workload,
                       linear_workload_latency)


@dataclass(frozen=True)
class StageLatency:
    """Per-stage forward and backward time of one micro-batch (`pipeline.py:28-37`)."""

    forward: float
    backward: float

    @property
    def round_trip(self) -> float:
        return self.forward + self.backward


@dataclass
class StepReport:
    """One training iteration (`pipeline.py:40-57`, same fields)."""

    iteration: int
    microbatch_tokens: list[int]
    microbatch_attention_pairs: list[int]
    forward: list[float]
    backward: list[float]
    strategy_choices: list[str]
    imbalance_attention: float
    imbalance_latency: float
    replica_paths: list[float]
    dp_step_latency: float
    pack_seconds: float
    carried_over_docs: int
    queue_depths: list[int]
    event_makespan: float | None = None


def stage_latency_for_assignment(assignment: ShardAssignment, config: ParallelismConfig,
                                 profile: CostProfile) -> StageLatency:
    """Modelled stage cost of a chosen assignment (`pipeline.py:60-66`)."""
    attn = group_attention_latency(assignment, profile)
    tokens_per_worker = sum(assignment.doc_lengths) // assignment.cp
    forward = (attn + linear_workload_latency(tokens_per_worker, profile)) / config.pp
    return StageLatency(forward, profile.backward_ratio * forward)


def microbatch_stage_latency(mb: MicroBatch, config: ParallelismConfig, profile: CostProfile,
                             policy: str = "adaptive") -> StageLatency:
    """`pipeline.py:69-75`: shard under `policy`, then price the stage."""
    return stage_latency_for_assignment(shard(mb, config.cp, policy, profile), config, profile)


def measured_stage_latency(attn_fwd_s: float, attn_bwd_s: float, tokens_per_worker: int,
                           config: ParallelismConfig, profile: CostProfile) -> StageLatency:
    """Stage cost with the attention term MEASURED (seconds, max over CP ranks)."""
    lin = linear_workload_latency(tokens_per_worker, profile)
    return StageLatency((attn_fwd_s + lin) / config.pp,
                        (attn_bwd_s + profile.backward_ratio * lin) / config.pp)


def pp_critical_path(stages: list[StageLatency], pp: int) -> float:
    """Analytic 1F1B step latency (`pipeline.py:78-86`)."""
    if pp < 1:
        raise ValueError("pp must be >= 1")
    if not stages:
        return 0.0
    trips = [s.round_trip for s in stages]
    return sum(trips) + (pp - 1) * max(trips)


def dp_step_latency(replica_paths: list[float]) -> float:
    """Slowest data-parallel replica (`pipeline.py:150-154`)."""
    if not replica_paths:
        raise ValueError("at least one replica is required")
    return max(replica_paths)


def measure_attention_latency(shards, inputs, exchange=None, scale=None, reps: int = 3,
                              group=None):
    """Per micro-batch (fwd_s, bwd_s) of this rank's attention kernels (median
    of `reps` CUDA-event timings on the launching stream, after one warm-up),
    reduced to the max over the CP group when torch.distributed is up.

    `shards[b]` are CPShard objects of this rank, `inputs[b] = (q, k, v, do)`
    local tensors; `exchange` (cp.NcclExchange / cp.SymmExchange) gathers the
    full K/V first -- the exchange itself is not timed.
    """
    from .cp import NcclExchange
    if exchange is None:
        exchange = NcclExchange(group)
    fwd, bwd = [], []
    for b, (sh, (q, k, v, do)) in enumerate(zip(shards, inputs)):
        kf, vf = exchange.gather(k, v, sh, b) if sh.cp > 1 else (k, v)
        samples = []
        for _ in range(reps + 1):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
            o, lse = attn_forward(q, kf, vf, sh.tiles, scale)
            ev[1].record()
            attn_backward(q, kf, vf, o, lse, do, sh.tiles, scale)
            ev[2].record()
            samples.append(ev)
        torch.cuda.synchronize()
        f = sorted(e[0].elapsed_time(e[1]) for e in samples[1:])[reps // 2]
        g = sorted(e[1].elapsed_time(e[2]) for e in samples[1:])[reps // 2]
        fwd.append(f / 1e3)
        bwd.append(g / 1e3)
    if dist.is_available() and dist.is_initialized() and shards and shards[0].cp > 1:
        t = torch.tensor([fwd, bwd], dtype=torch.float64, device=torch.device("cuda"))
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        fwd, bwd = t[0].tolist(), t[1].tolist()
    return fwd, bwd


def measured_step_report(iteration: int, microbatches, strategies, attn_fwd_s, attn_bwd_s,
                         config: ParallelismConfig, profile: CostProfile,
                         pack_seconds: float = 0.0, carried_over_docs: int = 0,
                         queue_depths=None) -> StepReport:
    """`harness.report_for` (`harness.py:340-390`) for one replica with the
    attention term of every stage measured on the GPU."""
    stages, tokens, pairs = [], [], []
    for mb, f, b in zip(microbatches, attn_fwd_s, attn_bwd_s):
        lengths = mb.lengths() if isinstance(mb, MicroBatch) else list(mb)
        total = sum(lengths)
        tokens.append(total)
        pairs.append(attention_workload(lengths))
        stages.append(measured_stage_latency(f, b, total // config.cp, config, profile))
    mbs = [mb if isinstance(mb, MicroBatch) else
           MicroBatch([Document(i, int(x)) for i, x in enumerate(mb)]) for mb in microbatches]
    path = pp_critical_path(stages, config.pp)
    return StepReport(
        iteration=iteration, microbatch_tokens=tokens, microbatch_attention_pairs=pairs,
        forward=[s.forward for s in stages], backward=[s.backward for s in stages],
        strategy_choices=[str(s) for s in strategies],
        imbalance_attention=imbalance_degree_attention(mbs),
        imbalance_latency=imbalance_degree_latency(mbs, max(len(mbs), 1), profile),
        replica_paths=[path], dp_step_latency=dp_step_latency([path]),
        pack_seconds=pack_seconds, carried_over_docs=carried_over_docs,
        queue_depths=list(queue_depths or []), event_makespan=None)
