"""Generate golden vectors by importing the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are committed here
as small gzip'd JSON fixtures.  Floats are stored with float.hex() so parity
checks are exact.  Everything is seeded; rerunning reproduces byte-identical
files.
"""

from __future__ import annotations

import gzip
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    sys.dont_write_bytecode = True
    os.environ.setdefault("BALSIM_PURE_KERNELS", "1")   # read-only mount: pure backend
    sys.path.insert(0, REF_SRC)
    import balsim  # noqa: F401
    return balsim


def _dump(name, obj):
    path = os.path.join(HERE, name)
    raw = json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()
    with open(path, "wb") as fh:
        # mtime=0 keeps the gzip header deterministic
        with gzip.GzipFile(fileobj=fh, mode="wb", mtime=0) as gz:
            gz.write(raw)
    print(f"wrote {path} ({len(raw)} bytes raw)")


def _workers(a):
    return [[[p, r.start, r.end] for p, r in w] for w in a.workers]


def _case(b, lengths, cp, profile):
    from balsim.sharding import (adaptive_select, per_document_shard,
                                 per_sequence_shard, worker_attention_latency)
    mb = b.MicroBatch([b.Document(i, int(x)) for i, x in enumerate(lengths)])
    seq = per_sequence_shard(mb, cp)
    doc = per_document_shard(mb, cp)
    lat_seq = [worker_attention_latency(seq, w, profile) for w in range(cp)]
    lat_doc = [worker_attention_latency(doc, w, profile) for w in range(cp)]
    chosen = adaptive_select(mb, cp, profile)
    return {
        "lengths": [int(x) for x in lengths], "cp": cp,
        "per_sequence": _workers(seq), "per_document": _workers(doc),
        "lat_seq": [x.hex() for x in lat_seq], "lat_doc": [x.hex() for x in lat_doc],
        "adaptive": chosen.strategy.value,
    }


def sharding_random(b):
    rng = np.random.default_rng(20240817)
    prof = b.CostProfile()
    cases = []
    for i in range(480):
        cp = int(rng.choice([1, 2, 4, 8]))
        if i % 3 == 0:      # short documents: exercises tails and empty chunks
            k = int(rng.integers(1, 41))
            lengths = [int(x) for x in rng.integers(1, 24, size=k)]
        else:               # reference-test style (test_sharding.py:59-66)
            k = int(rng.integers(1, 9))
            lengths = [int(x) for x in rng.integers(1, 4096, size=k)]
        pad = -sum(lengths) % (2 * cp)
        if pad:
            lengths.append(pad)
        cases.append(_case(b, lengths, cp, prof))
    # hand examples from the reference tests (test_sharding.py:69-145)
    for lengths, cp in (([16], 2), ([5, 7], 1), ([24, 8], 2), ([10, 6], 2),
                        ([32], 4), ([1, 1, 1, 1], 2), ([256], 1),
                        ([128 * 1024], 4), ([128] * 64, 4),
                        ([96 * 1024] + [1024] * 32, 4)):
        cases.append(_case(b, lengths, cp, prof))
    _dump("sharding_random.json.gz", {"cases": cases})


def synthetic_streams(b):
    out = {}
    cases = []
    prof = b.CostProfile()
    for window in (8192, 32768, 131072):
        spec = b.SyntheticSpec(context_window=window, tokens_per_global_batch=window)
        batches = b.generate_synthetic_stream(spec, seed=0, n_batches=8)
        out[str(window)] = [[[d.id, d.length, d.arrival_batch] for d in bt] for bt in batches]
        for bt in batches:
            for cp in (1, 2, 4, 8):
                cases.append(_case(b, [d.length for d in bt], cp, prof))
    # a second seed and a multi-window global batch for the generator check
    spec = b.SyntheticSpec(context_window=32768, tokens_per_global_batch=4 * 32768)
    out["32768x4_seed7"] = [[[d.id, d.length, d.arrival_batch] for d in bt]
                            for bt in b.generate_synthetic_stream(spec, seed=7, n_batches=3)]
    _dump("synthetic_streams.json.gz", {"streams": out})
    _dump("sharding_synthetic.json.gz", {"cases": cases})


def kernels(b):
    from balsim._kernels import _pure
    rng = np.random.default_rng(7)
    kl = []
    for _ in range(200):
        n = int(rng.integers(0, 40))
        q = rng.integers(0, 5000, size=n).astype(np.int64)
        q[rng.random(n) < 0.1] = 0
        kv = q + rng.integers(1, 200000, size=n)
        tile = int(rng.choice([1, 64, 128, 256]))
        cq = np.array([0, 256], dtype=np.int64) if rng.random() < 0.5 else \
            np.array([0, 100, 1000, 4000], dtype=np.int64)
        cv = np.sort(rng.uniform(1e10, 1e12, size=len(cq)))
        op = float(rng.uniform(1.0, 200.0))
        res = _pure.kernel_latency_sum(q, kv, tile, cq, cv, op)
        kl.append({"q": q.tolist(), "kv": kv.tolist(), "tile": tile, "cq": cq.tolist(),
                   "cv": [x.hex() for x in cv.tolist()], "op": op.hex(), "out": res.hex()})
    hf = []
    for _ in range(120):
        n = int(rng.integers(1, 64))
        lengths = np.sort(rng.integers(1, 50000, size=n))[::-1].astype(np.int64)
        n_mb = int(rng.integers(1, 9))
        l_max = int(lengths.sum() // n_mb) + int(lengths[0]) - int(rng.integers(0, 2) * lengths[0] // 2)
        l_max = max(l_max, int(lengths[0]))
        out = _pure.heuristic_fill(lengths, n_mb, l_max, 2e-10, 2e-6)
        hf.append({"lengths": lengths.tolist(), "n_mb": n_mb, "l_max": l_max,
                   "out": out.tolist()})
    hf.append({"lengths": [10, 10, 10], "n_mb": 2, "l_max": 10, "out": [0, 1, -1]})
    pc = []
    for _ in range(50):
        lengths = rng.integers(0, 200000, size=int(rng.integers(0, 50))).tolist()
        pc.append({"lengths": lengths, "out": int(_pure.sum_pair_counts(lengths))})
    rp = []
    for _ in range(50):
        n = int(rng.integers(0, 40))
        s = rng.integers(0, 100000, size=n)
        e = s + rng.integers(0, 10000, size=n)
        rp.append({"s": s.tolist(), "e": e.tolist(), "out": int(_pure.range_pair_sum(s, e))})
    _dump("kernels.json.gz", {"kernel_latency_sum": kl, "heuristic_fill": hf,
                              "sum_pair_counts": pc, "range_pair_sum": rp})


def packer_config5(b):
    """BASELINE config 5: 64 micro-batches per iteration from the W(d) packer
    with outlier queues (harness defaults, harness.py:115-126), padded for cp=8,
    adaptive selection per micro-batch."""
    from balsim.harness import _FillerIds, pad_for_cp
    prof = b.CostProfile()
    spec = b.SyntheticSpec(context_window=131072, tokens_per_global_batch=64 * 131072)
    stream = b.generate_synthetic_stream(spec, seed=0, n_batches=2)
    packer = b.HeuristicPacker(b.OutlierQueueSet((32768, 98304)), 64, 163840, prof)
    filler = _FillerIds()
    iters = []
    for it, batch in enumerate(stream):
        plan = packer.feed(batch, it)
        mbs = []
        for mb in plan.microbatches:
            padded = pad_for_cp(mb, 8, filler, it)
            choice = b.adaptive_select(padded, 8, prof).strategy.value if padded.docs else None
            mbs.append({"ids": [d.id for d in padded.docs],
                        "lengths": [d.length for d in padded.docs],
                        "arrivals": [d.arrival_batch for d in padded.docs],
                        "choice": choice})
        iters.append({"microbatches": mbs,
                      "carried": [d.id for d in plan.carried_over],
                      "delayed": sorted([int(k), int(v)] for k, v in plan.delayed_tokens.items()),
                      "depths": packer.queues.depths()})
    _dump("packer_config5.json.gz", {"iterations": iters})


def records(b):
    """Wire formats written by the reference itself (records.py:60-116)."""
    from balsim import records as rec
    from balsim.sharding import per_document_shard, per_sequence_shard
    spec = b.SyntheticSpec(context_window=8192, tokens_per_global_batch=4 * 8192)
    stream = b.generate_synthetic_stream(spec, seed=3, n_batches=3)
    packer = b.HeuristicPacker(b.OutlierQueueSet((2048, 6144)), 4, 10240, b.CostProfile())
    plans = [packer.feed(batch, it) for it, batch in enumerate(stream)] + packer.flush(3)
    rec.write_plans(plans, os.path.join(HERE, "records_plans.jsonl"))
    assigns = []
    for lengths, cp in (([700, 3, 129, 2000, 1, 257, 6], 4), ([16], 2), ([10, 6], 2),
                        ([5000, 3000, 120, 7, 1], 8)):
        mb = b.MicroBatch([b.Document(100 + i, x) for i, x in enumerate(lengths)])
        assigns += [per_sequence_shard(mb, cp), per_document_shard(mb, cp)]
    rec.write_assignments(assigns, os.path.join(HERE, "records_shards.jsonl"))
    print("wrote records_plans.jsonl, records_shards.jsonl")


def pipeline_model(b):
    """Stage pricing and the 1F1B critical path (pipeline.py:60-86, packing.py:437-449)."""
    from balsim.pipeline import StageLatency, pp_critical_path, stage_latency_for_assignment
    from balsim.packing import imbalance_degree_latency
    from balsim.sharding import shard
    rng = np.random.default_rng(99)
    prof = b.CostProfile()
    cases = []
    for i in range(40):
        cp = int(rng.choice([1, 2, 4, 8]))
        pp = int(rng.choice([1, 2, 4]))
        k = int(rng.integers(1, 12))
        lengths = [int(x) for x in rng.integers(1, 6000, size=k)]
        pad = -sum(lengths) % (2 * cp)
        if pad:
            lengths.append(pad)
        mb = b.MicroBatch([b.Document(j, x) for j, x in enumerate(lengths)])
        par = b.ParallelismConfig(context_window=65536, cp=cp, pp=pp)
        policy = ["per_sequence", "per_document", "adaptive"][i % 3]
        st = stage_latency_for_assignment(shard(mb, cp, policy, prof), par, prof)
        cases.append({"lengths": lengths, "cp": cp, "pp": pp, "policy": policy,
                      "forward": st.forward.hex(), "backward": st.backward.hex()})
    paths = []
    for _ in range(30):
        n = int(rng.integers(0, 10))
        pp = int(rng.integers(1, 6))
        stages = [StageLatency(float(f), float(f) * 2) for f in rng.uniform(0.01, 1.0, size=n)]
        paths.append({"stages": [[s.forward.hex(), s.backward.hex()] for s in stages], "pp": pp,
                      "out": pp_critical_path(stages, pp).hex()})
    imb = []
    for _ in range(20):
        mbs = [b.MicroBatch([b.Document(j, int(x)) for j, x in
                             enumerate(rng.integers(1, 9000, size=int(rng.integers(1, 8))))])
               for _ in range(int(rng.integers(1, 9)))]
        imb.append({"mbs": [m.lengths() for m in mbs],
                    "out": imbalance_degree_latency(mbs, len(mbs), prof).hex()})
    _dump("pipeline_model.json.gz", {"stages": cases, "paths": paths, "imbalance_latency": imb})


def main():
    b = _import_reference()
    sharding_random(b)
    synthetic_streams(b)
    kernels(b)
    packer_config5(b)
    records(b)
    pipeline_model(b)


if __name__ == "__main__":
    main()
