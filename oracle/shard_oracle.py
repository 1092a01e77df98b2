"""Pure-Python restatement of the reference CP sharding path.  TEST ORACLE ONLY.

Every function cites the reference code it restates.  Outputs use plain
tuples so the oracle shares no types with the product package:

    assignment = [ [(pos, start, end), ...]  for each worker ]   (canonical)

The restatement deliberately follows the reference's *procedure* (raw span
lists, sort, merge), not the closed form used by the GPU builder, so the
two are independent derivations of the same answer.
"""

from __future__ import annotations

SEQ, DOC = 0, 1


def check_divisible(total: int, cp: int) -> None:
    """`sharding.py:77-83`: cp >= 1 and total % (2*cp) == 0 else ValueError."""
    if cp < 1:
        raise ValueError("cp must be >= 1")
    if total % (2 * cp):
        raise ValueError(f"length {total} not divisible by 2*cp")


def canonical(raw):
    """`sharding.py:63-74`: sort (pos, start, end); merge same-pos touching spans."""
    out = []
    for pos, s, e in sorted(raw):
        if out and out[-1][0] == pos and out[-1][2] == s:
            out[-1] = (pos, out[-1][1], e)
        else:
            out.append((pos, s, e))
    return out


def per_sequence(lengths, cp):
    """`sharding.py:86-110`: 2*cp global chunks, worker w takes w and 2cp-1-w."""
    lengths = [int(x) for x in lengths]
    total = sum(lengths)
    check_divisible(total, cp)
    c = total // (2 * cp)
    bounds = [0]
    for x in lengths:
        bounds.append(bounds[-1] + x)
    workers = []
    for w in range(cp):
        raw = []
        if c:
            for chunk in (w, 2 * cp - 1 - w):
                lo, hi = chunk * c, (chunk + 1) * c
                for p in range(len(lengths)):
                    a, b = bounds[p], bounds[p + 1]
                    if b > lo and a < hi:
                        raw.append((p, max(lo, a) - a, min(hi, b) - a))
        workers.append(canonical(raw))
    return workers


def per_document(lengths, cp):
    """`sharding.py:113-141`: per-doc 2*cp chunks + tail tokens dealt round-robin
    with a cursor that runs across documents."""
    lengths = [int(x) for x in lengths]
    check_divisible(sum(lengths), cp)
    raws = [[] for _ in range(cp)]
    cursor = 0
    for p, length in enumerate(lengths):
        d = length // (2 * cp)
        if d:
            for w in range(cp):
                raws[w].append((p, w * d, (w + 1) * d))
                raws[w].append((p, (2 * cp - 1 - w) * d, (2 * cp - w) * d))
        ts = 2 * cp * d
        for k in range(length - ts):
            raws[(cursor + k) % cp].append((p, ts + k, ts + k + 1))
        cursor += length - ts
    return [canonical(r) for r in raws]


def shard(lengths, cp, strategy):
    return per_sequence(lengths, cp) if strategy == SEQ else per_document(lengths, cp)


def kernel_latency_sum(q_lens, kv_lens, tile, curve_q, curve_v, op_scale):
    """`_kernels/_pure.py:41-66`; same expression order -> same float."""
    total = 0.0
    n = len(curve_q)
    for q, kv in zip(q_lens, kv_lens):
        q, kv = int(q), int(kv)
        if q == 0:
            continue
        j = n - 1
        while j > 0 and curve_q[j] > q:
            j -= 1
        padded = ((q + tile - 1) // tile) * tile
        total += op_scale * float(padded * kv) / curve_v[j]
    return total


def worker_latency(worker_ranges, tile, curve_q, curve_v, op_scale):
    """`sharding.py:151-161`: q = end - start, kv = end (doc-prefix KV)."""
    if not worker_ranges:
        return 0.0
    return kernel_latency_sum([e - s for _, s, e in worker_ranges],
                              [e for _, _, e in worker_ranges],
                              tile, curve_q, curve_v, op_scale)


def strategy_latencies(lengths, cp, tile, curve_q, curve_v, op_scale):
    """`sharding.py:164-179`: group latency = max over workers, both strategies."""
    out = {}
    for strat in (SEQ, DOC):
        a = shard(lengths, cp, strat)
        out[strat] = max(worker_latency(a[w], tile, curve_q, curve_v, op_scale)
                         for w in range(cp))
    return out


def adaptive(lengths, cp, tile, curve_q, curve_v, op_scale):
    """`sharding.py:182-188`: per-seq if lat_seq <= lat_doc (ties -> per-seq)."""
    lats = strategy_latencies(lengths, cp, tile, curve_q, curve_v, op_scale)
    return SEQ if lats[SEQ] <= lats[DOC] else DOC


def range_pairs(s, e):
    """`_kernels/_pure.py:25-38`."""
    return (e * (e + 1) - s * (s + 1)) // 2


def worker_pairs(worker_ranges):
    return sum(range_pairs(s, e) for _, s, e in worker_ranges)


def pad_lengths_for_cp(lengths, cp):
    """`harness.py:291-298` on raw lengths: append 2cp - T mod 2cp if nonzero."""
    lengths = [int(x) for x in lengths]
    r = sum(lengths) % (2 * cp)
    return lengths + ([2 * cp - r] if r else [])


def local_layout(lengths, worker_ranges):
    """Local token order of one worker (the concatenation of its canonical
    ranges) as (global token index, in-document position) lists.  This is the
    layout the GPU builder's gather_index / positions must reproduce."""
    starts = [0]
    for x in lengths:
        starts.append(starts[-1] + int(x))
    gidx, pos = [], []
    for p, s, e in worker_ranges:
        for t in range(s, e):
            gidx.append(starts[p] + t)
            pos.append(t)
    return gidx, pos
