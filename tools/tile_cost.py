"""Tile-level cost features of a CP rank, mirroring the kernels' work lists.

fwd: back-aligned 128-row query tiles per (rank, doc) row-set, paired from the
     end -> n_pairs items, sum over tiles of ceil((last_pos + 1) / 128) KV steps
bwd: 128-key KV tiles up to the row-set's largest position -> n_kv items,
     sum over them of ceil(rows with pos >= k0 / 64) query iterations
"""
import math


def rank_features(ranges):
    """ranges: canonical [(doc, s, e), ...] of one rank."""
    by_doc = {}
    for p, s, e in ranges:
        by_doc.setdefault(p, []).append((s, e))
    f_pairs = f_steps = b_items = b_iters = 0
    for segs in by_doc.values():
        segs.sort()
        n = sum(e - s for s, e in segs)
        # position of local row index r (0-based)
        def pos_of(r):
            for s, e in segs:
                if r < e - s:
                    return s + r
                r -= e - s
            raise IndexError
        nt = (n + 127) // 128
        f_pairs += (nt + 1) // 2
        for m in range(nt):                      # tile m from the end
            last = n - 1 - 128 * m
            f_steps += (pos_of(last) + 1 + 127) // 128
        maxpos = segs[-1][1] - 1
        for t in range((maxpos + 128) // 128):
            k0 = 128 * t
            c = sum(max(0, e - max(s, k0)) for s, e in segs)
            b_items += 1
            b_iters += (c + 63) // 64
    return f_pairs, f_steps, b_items, b_iters
