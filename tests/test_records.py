"""Wire formats byte-identical to the reference's (records.py)."""

import os

import pytest

import paper_2503_17924_b200 as wl
from paper_2503_17924_b200 import records as rec
from conftest import GOLDEN
from oracle import shard_oracle as so

CASES = (([700, 3, 129, 2000, 1, 257, 6], 4), ([16], 2), ([10, 6], 2), ([5000, 3000, 120, 7, 1], 8))


def _read(path):
    with open(path, "rb") as fh:
        return fh.read()


def test_plans_bytes_match_reference(tmp_path):
    spec = wl.SyntheticSpec(context_window=8192, tokens_per_global_batch=4 * 8192)
    stream = wl.generate_synthetic_stream(spec, seed=3, n_batches=3)
    packer = wl.HeuristicPacker(wl.OutlierQueueSet((2048, 6144)), 4, 10240, wl.CostProfile())
    plans = [packer.feed(batch, it) for it, batch in enumerate(stream)] + packer.flush(3)
    out = tmp_path / "plans.jsonl"
    rec.write_plans(plans, out)
    assert _read(out) == _read(os.path.join(GOLDEN, "records_plans.jsonl"))
    back = rec.read_plans(out)
    assert [[mb.lengths() for mb in p.microbatches] for p in back] == \
        [[mb.lengths() for mb in p.microbatches] for p in plans]


def _oracle_assignments():
    out = []
    for lengths, cp in CASES:
        for strat, name in ((so.SEQ, "per_sequence"), (so.DOC, "per_document")):
            workers = [[(p, wl.TokenRange(s, e)) for p, s, e in w] for w in so.shard(lengths, cp, strat)]
            out.append(wl.ShardAssignment(wl.ShardStrategy(name), cp,
                                          [100 + i for i in range(len(lengths))], list(lengths),
                                          workers))
    return out


def test_shards_bytes_match_reference(tmp_path):
    out = tmp_path / "shards.jsonl"
    rec.write_assignments(_oracle_assignments(), out)
    assert _read(out) == _read(os.path.join(GOLDEN, "records_shards.jsonl"))
    back = rec.read_assignments(out)
    assert [a.workers for a in back] == [a.workers for a in _oracle_assignments()]


def test_bad_files_rejected(tmp_path):
    p = tmp_path / "x.jsonl"
    p.write_text('{"type":"header","schema":"balsim.plans.v1"}\n')
    with pytest.raises(wl.IngestError):
        rec.read_assignments(p)
    p.write_text("not json\n")
    with pytest.raises(wl.IngestError):
        rec.read_plans(p)


def test_trace_round_trip(tmp_path):
    docs = [wl.Document(3, 100, 0), wl.Document(9, 20000, 2)]
    p = tmp_path / "t.txt"
    rec.write_trace(docs, p)
    assert rec.ingest_trace(p) == docs
    assert rec.ingest_trace(p, context_window=8192)[1].length == 8192


@pytest.mark.gpu
def test_gpu_built_shards_bytes_match_reference(tmp_path):
    assigns = []
    for lengths, cp in CASES:
        mb = wl.MicroBatch([wl.Document(100 + i, x) for i, x in enumerate(lengths)])
        assigns += [wl.per_sequence_shard(mb, cp), wl.per_document_shard(mb, cp)]
    out = tmp_path / "shards.jsonl"
    rec.write_assignments(assigns, out)
    assert _read(out) == _read(os.path.join(GOLDEN, "records_shards.jsonl"))
