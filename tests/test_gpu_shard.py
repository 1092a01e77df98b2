"""GPU shard builder + selector: bit-exact against the reference's outputs."""

import pytest
import torch

from conftest import load_golden, to_workers
import paper_2503_17924_b200 as wl
from oracle import shard_oracle as so

pytestmark = pytest.mark.gpu

PROFILE = wl.CostProfile()


def _mb(lengths):
    return wl.MicroBatch([wl.Document(i, x) for i, x in enumerate(lengths)])


@pytest.mark.parametrize("name", ["sharding_random.json.gz", "sharding_synthetic.json.gz"])
def test_batched_plan_bit_exact(name):
    """All golden cases, grouped by cp, each group in ONE batched launch."""
    cases = load_golden(name)["cases"]
    for cp in (1, 2, 4, 8):
        group = [c for c in cases if c["cp"] == cp]
        if not group:
            continue
        plan = wl.build_shard_plan([c["lengths"] for c in group], cp, "adaptive", PROFILE)
        lat = plan.rank_latency.cpu()
        for b, c in enumerate(group):
            assert to_workers(plan.assignment(b, wl.ShardStrategy.PER_SEQUENCE)) == c["per_sequence"]
            assert to_workers(plan.assignment(b, wl.ShardStrategy.PER_DOCUMENT)) == c["per_document"]
            assert [x.hex() for x in lat[b, 0].tolist()] == c["lat_seq"]
            assert [x.hex() for x in lat[b, 1].tolist()] == c["lat_doc"]
            assert plan.strategy(b).value == c["adaptive"]


def test_token_layout_and_pairs_match_oracle():
    cases = load_golden("sharding_random.json.gz")["cases"][:120]
    for cp in (1, 2, 4, 8):
        group = [c for c in cases if c["cp"] == cp]
        for policy in ("per_sequence", "per_document"):
            plan = wl.build_shard_plan([c["lengths"] for c in group], cp, policy)
            pairs = plan.rank_pairs.cpu()
            for b, c in enumerate(group):
                a = so.shard(c["lengths"], cp, so.SEQ if policy == "per_sequence" else so.DOC)
                for w in range(cp):
                    g, p, ro = plan.rank_local(b, w)
                    eg, ep = so.local_layout(c["lengths"], a[w])
                    assert g.tolist() == eg and p.tolist() == ep
                    assert int(pairs[b, w]) == so.worker_pairs(a[w])
                    # row-set offsets: tokens of each doc on this rank, in doc order
                    counts = [0] * len(c["lengths"])
                    for pos, s, e in a[w]:
                        counts[pos] += e - s
                    exp = [0]
                    for x in counts:
                        exp.append(exp[-1] + x)
                    assert ro.tolist() == exp


def test_reference_api_hand_examples():
    """test_sharding.py:69-145,152-216 of the reference, through the drop-in API."""
    a = wl.per_sequence_shard(_mb([16]), 2)
    assert a.workers[0] == [(0, wl.TokenRange(0, 4)), (0, wl.TokenRange(12, 16))]
    assert a.workers[1] == [(0, wl.TokenRange(4, 12))]
    a = wl.per_document_shard(_mb([10, 6]), 2)
    assert a.workers[0] == [(0, wl.TokenRange(0, 2)), (0, wl.TokenRange(6, 9)),
                            (1, wl.TokenRange(0, 1)), (1, wl.TokenRange(3, 5))]
    assert a.workers[1] == [(0, wl.TokenRange(2, 6)), (0, wl.TokenRange(9, 10)),
                            (1, wl.TokenRange(1, 3)), (1, wl.TokenRange(5, 6))]
    assert wl.per_document_shard(_mb([1, 1, 1, 1]), 2).worker_token_count(0) == 2
    with pytest.raises(ValueError):
        wl.per_sequence_shard(_mb([10]), 2)
    with pytest.raises(ValueError):
        wl.per_document_shard(_mb([8]), 0)
    a = wl.per_sequence_shard(_mb([16]), 2)
    assert wl.worker_attention_latency(a, 1, PROFILE) == wl.attention_kernel_latency(8, 12, PROFILE)
    a.workers[1] = []
    assert wl.worker_attention_latency(a, 1, PROFILE) == 0.0
    assert wl.adaptive_select(_mb([128 * 1024]), 4, PROFILE).strategy is wl.ShardStrategy.PER_SEQUENCE
    assert wl.adaptive_select(_mb([128] * 64), 4, PROFILE).strategy is wl.ShardStrategy.PER_SEQUENCE
    assert wl.adaptive_select(_mb([96 * 1024] + [1024] * 32), 4, PROFILE).strategy \
        is wl.ShardStrategy.PER_DOCUMENT
    assert wl.shard(_mb([32]), 2, "per_document", PROFILE).strategy is wl.ShardStrategy.PER_DOCUMENT
    with pytest.raises(ValueError):
        wl.shard(_mb([32]), 2, "bogus", PROFILE)


def test_worker_latency_bit_exact_random(rng):
    for _ in range(50):
        cp = int(rng.choice([2, 4, 8]))
        k = int(rng.integers(1, 30))
        lengths = [int(x) for x in rng.integers(1, 9000, size=k)]
        lengths = so.pad_lengths_for_cp(lengths, cp)
        a = wl.per_document_shard(_mb(lengths), cp)
        ref = so.per_document(lengths, cp)
        for w in range(cp):
            got = wl.worker_attention_latency(a, w, PROFILE)
            assert got == so.worker_latency(ref[w], 128, [0, 256], [3.5e11, 7e11], 70.0)
        lats = wl.strategy_latencies(_mb(lengths), cp, PROFILE)
        exp = so.strategy_latencies(lengths, cp, 128, [0, 256], [3.5e11, 7e11], 70.0)
        assert lats[wl.ShardStrategy.PER_SEQUENCE] == exp[so.SEQ]
        assert lats[wl.ShardStrategy.PER_DOCUMENT] == exp[so.DOC]


def test_config5_selection_matches_reference():
    """64 packed micro-batches per step, padded for cp=8, one batched launch."""
    g = load_golden("packer_config5.json.gz")["iterations"]
    for it in g:
        mbs = [m for m in it["microbatches"] if m["lengths"]]
        plan = wl.build_shard_plan([m["lengths"] for m in mbs], 8, "adaptive", PROFILE)
        assert [plan.strategy(b).value for b in range(len(mbs))] == [m["choice"] for m in mbs]


def test_attention_tiles_cover_rows_once():
    from paper_2503_17924_b200.attention import build_tiles
    lengths = so.pad_lengths_for_cp([700, 3, 129, 2000, 1, 257], 4)
    plan = wl.build_shard_plan([lengths], 4, "per_document")
    for w in range(4):
        g, pos, ro = plan.rank_local(0, w)
        t = build_tiles(ro, pos, lengths)
        n = int(t.n_tiles.item())
        items = t.tiles[:2 * n].cpu().view(n, 8).tolist()
        seen = torch.zeros(pos.numel(), dtype=torch.int32)
        ext = []
        for rx, nx, kvb, kvx, ry, ny, kvy, _ in items:
            assert 1 <= nx <= 128 and 0 <= ny <= 128
            seen[rx:rx + nx] += 1
            assert kvx - kvb == pos[rx + nx - 1].item() + 1
            if ny:
                assert ry + ny == rx                      # Y is the tile just before X
                seen[ry:ry + ny] += 1
                assert kvy - kvb == pos[ry + ny - 1].item() + 1 and kvy <= kvx
            ext.append((kvx - kvb + 127) // 128)
        assert bool((seen == 1).all())
        assert ext == sorted(ext, reverse=True)   # longest first


def _work_list_features(plan, b, rank):
    """The 8 tile-model features of one rank, recomputed from the work lists
    the kernels run: wlb_attn_tiles items (forward) and the backward's KV-tile
    rule (128-key tiles below a row-set's last position; rows with position
    >= k0), from the rank's positions / row-set offsets."""
    from paper_2503_17924_b200.attention import build_tiles
    lengths = plan.lengths[b]
    g, pos, ro = plan.rank_local(b, rank)
    t = build_tiles(ro, pos, lengths)
    n = int(t.n_tiles.item())
    items = t.tiles[:2 * n].cpu().view(n, 8).tolist()
    f_steps = f_max = 0
    for rx, nx, kvb, kvx, ry, ny, kvy, _ in items:
        s = (kvx - kvb + 127) // 128 + ((kvy - kvb + 127) // 128 if ny else 0)
        f_steps += s
        f_max = max(f_max, s)
    pos, ro = pos.cpu().tolist(), ro.cpu().tolist()
    b_items = q64 = q128 = m64 = m128 = 0
    for p in range(len(lengths)):
        rows = pos[ro[p]:ro[p + 1]]
        if not rows:
            continue
        for tk in range((rows[-1] + 128) // 128):
            cnt = sum(1 for x in rows if x >= 128 * tk)
            b_items += 1
            q64 += (cnt + 63) // 64
            q128 += (cnt + 127) // 128
            m64, m128 = max(m64, (cnt + 63) // 64), max(m128, (cnt + 127) // 128)
    return [n, f_steps, f_max, b_items, q64, q128, m64, m128]


@pytest.mark.parametrize("cp", [1, 2, 4, 8])
def test_tile_model_features_match_kernel_work_lists(cp):
    """The measured-latency selector prices exactly the work the attention
    kernels run: its per-(strategy, rank) features equal counts taken from
    the kernels' own tile lists, for both strategies."""
    mbs = [so.pad_lengths_for_cp(x, cp) for x in
           ([700, 3, 129, 2000, 1, 257], [4096], [300] * 9 + [17, 5000], [1] * 40 + [64])]
    model = wl.TileModel()
    for s, strat in enumerate(("per_sequence", "per_document")):
        plan = wl.build_shard_plan(mbs, cp, strat, model=model)
        feats = plan.features.cpu()
        for b in range(len(mbs)):
            for r in range(cp):
                assert feats[b, s, r].tolist() == _work_list_features(plan, b, r), (strat, b, r)


@pytest.mark.parametrize("shape", [None, "tail", (32, 32), (64, 8)])
def test_measured_policy_selects_by_predicted_latency(shape):
    """policy="measured": per-sequence iff its slowest rank's predicted time is
    <= per-document's (ties -> per-sequence, the reference's rule); the
    prediction equals TileModel.predict on the returned features (defaults,
    and the shipped B200 calibrations, whose two backward kernels have their
    own per-item costs)."""
    cp = 4
    mbs = [so.pad_lengths_for_cp(x, cp) for x in
           ([30000, 100, 2000], [512] * 32, [8192], [100] * 40 + [20000])]
    if shape is None:
        model = wl.TileModel()
    elif shape == "tail":           # list-scheduling tail weights on both directions
        model = wl.TileModel(fwd_tail=0.4, bwd_tail=0.9)
    else:
        model = wl.TileModel.for_shape(*shape, 128)
    plan = wl.build_shard_plan(mbs, cp, "measured", model=model)
    lat, feats = plan.rank_latency.cpu(), plan.features.cpu()
    for b, ls in enumerate(mbs):
        tl = sum(ls) // cp
        for s in range(2):
            for r in range(cp):
                pred = model.predict(feats[b, s, r].tolist(), tl, len(ls))
                assert abs(lat[b, s, r].item() - pred) <= 1e-12 * max(1.0, pred)
        g = lat[b].max(dim=1).values
        exp = "per_sequence" if g[0] <= g[1] else "per_document"
        assert plan.strategy(b).value == exp
    # the chosen strategy's token layout is the one built
    a = plan.assignment(0)
    ref = so.shard(mbs[0], cp, so.SEQ if a.strategy == wl.ShardStrategy.PER_SEQUENCE else so.DOC)
    assert to_workers(a) == [[list(x) for x in w] for w in ref]
