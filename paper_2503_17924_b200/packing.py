"""Workload-aware variable-length packer with outlier delay queues (host side).

The north star keeps this on the host with unchanged output.  Mirrors
`/root/reference/pkg/src/balsim/packing.py:28-92,342-425,428-449`
(`PackingPlan`, `OutlierQueueSet`, `HeuristicPacker`, `heuristic_var_len_pack`,
`imbalance_degree_attention`); the placement kernel `heuristic_fill`
(`_compiled.pyx:50-86`) runs natively in libwlbcp.so (`wlb_heuristic_fill`,
plain C++ on the CPU, bit-identical fp64 expression order).
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ConfigError
from .workload import CostProfile, Document, MicroBatch, attention_workload, latency_of_lengths


@dataclass
class PackingPlan:
    """One iteration's packing result (`packing.py:28-41`)."""

    iteration: int
    microbatches: list[MicroBatch]
    carried_over: list[Document] = field(default_factory=list)
    delayed_tokens: dict[int, int] = field(default_factory=dict)


class OutlierQueueSet:
    """FIFO delay queues bucketed by ascending length thresholds (`packing.py:44-92`)."""

    def __init__(self, thresholds):
        thresholds = [int(t) for t in thresholds]
        if not thresholds:
            raise ConfigError("at least one queue threshold is required")
        if min(thresholds) < 1 or sorted(set(thresholds)) != thresholds:
            raise ConfigError("queue thresholds must be positive and increasing")
        self.thresholds = tuple(thresholds)
        self.queues: list[deque[Document]] = [deque() for _ in thresholds]

    def is_outlier(self, doc: Document) -> bool:
        return doc.length >= self.thresholds[0]

    def push(self, doc: Document) -> None:
        if not self.is_outlier(doc):
            raise ValueError("document below the first outlier threshold")
        bucket = sum(1 for t in self.thresholds if doc.length >= t) - 1
        self.queues[bucket].append(doc)

    def pop_ready(self, n: int) -> list[Document]:
        out: list[Document] = []
        for q in self.queues:
            if len(q) >= n:
                out.extend(q.popleft() for _ in range(n))
        return out

    def drain(self) -> list[Document]:
        out = [d for q in self.queues for d in q]
        for q in self.queues:
            q.clear()
        return out

    def depths(self) -> list[int]:
        return [len(q) for q in self.queues]

    def __len__(self) -> int:
        return sum(len(q) for q in self.queues)


def heuristic_fill(lengths, n_mb: int, l_max: int, attn_coeff: float,
                   linear_coeff: float) -> np.ndarray:
    """Native min-W placement of descending-length documents; -1 = unplaced."""
    arr = np.ascontiguousarray(lengths, dtype=np.int64)
    out = np.empty(len(arr), dtype=np.int32)
    _native.check(_native.lib().wlb_heuristic_fill(
        arr.ctypes.data, len(arr), int(n_mb), int(l_max), float(attn_coeff),
        float(linear_coeff), out.ctypes.data), "wlb_heuristic_fill")
    return out


class HeuristicPacker:
    """Streaming packer, Algorithm 1 of the paper (`packing.py:342-411`)."""

    def __init__(self, queues: OutlierQueueSet, n_microbatches: int, l_max: int,
                 profile: CostProfile):
        if n_microbatches < 1:
            raise ConfigError("n_microbatches must be >= 1")
        if l_max < queues.thresholds[0]:
            raise ConfigError("l_max below the first outlier threshold")
        self.queues = queues
        self.n = n_microbatches
        self.l_max = l_max
        self.profile = profile
        self._carried: list[Document] = []

    def _pack(self, pending: list[Document], iteration: int) -> PackingPlan:
        order = sorted(range(len(pending)), key=lambda i: (-pending[i].length, i))
        lengths = np.array([pending[i].length for i in order], dtype=np.int64)
        if len(lengths) and lengths[0] > self.l_max:
            raise ConfigError(f"document of length {int(lengths[0])} can never fit "
                              f"l_max {self.l_max}")
        bins = heuristic_fill(lengths, self.n, self.l_max, self.profile.attn_coeff,
                              self.profile.linear_coeff)
        mbs = [MicroBatch() for _ in range(self.n)]
        carried: list[Document] = []
        delays: dict[int, int] = {}
        for i, b in zip(order, bins.tolist()):
            doc = pending[i]
            if b < 0:
                carried.append(doc)
                continue
            mbs[b].docs.append(doc)
            delays[doc.id] = max(0, iteration - doc.arrival_batch)
        self._carried = carried
        return PackingPlan(iteration, mbs, carried_over=list(carried), delayed_tokens=delays)

    def feed(self, docs, iteration: int) -> PackingPlan:
        pending, self._carried = self._carried, []
        for doc in docs:
            if self.queues.is_outlier(doc):
                self.queues.push(doc)
            else:
                pending.append(doc)
        pending.extend(self.queues.pop_ready(self.n))
        return self._pack(pending, iteration)

    def flush(self, iteration: int) -> list[PackingPlan]:
        plans: list[PackingPlan] = []
        pending = self._carried + self.queues.drain()
        self._carried = []
        while pending:
            plans.append(self._pack(pending, iteration))
            iteration += 1
            pending, self._carried = self._carried, []
        return plans


def heuristic_var_len_pack(loader, queues: OutlierQueueSet, n: int, l_max: int,
                           profile: CostProfile):
    """Generator of per-iteration plans, then a flush (`packing.py:414-425`)."""
    packer = HeuristicPacker(queues, n, l_max, profile)
    iteration = -1
    for iteration, batch in enumerate(loader):
        yield packer.feed(batch, iteration)
    yield from packer.flush(iteration + 1)


def imbalance_degree_attention(microbatches) -> float:
    """max / mean of per-micro-batch causal pair counts (`packing.py:428-435`)."""
    works = [attention_workload(mb.lengths()) for mb in microbatches]
    total = sum(works)
    if not works or total == 0:
        return 1.0
    return max(works) * len(works) / total


def imbalance_degree_latency(microbatches, pp_size: int, profile: CostProfile) -> float:
    """max latency * pp_size / total latency (`packing.py:437-449`)."""
    lats = [latency_of_lengths(mb.lengths(), profile) for mb in microbatches]
    total = sum(lats)
    if not lats or total == 0:
        return 1.0
    return max(lats) * pp_size / total
