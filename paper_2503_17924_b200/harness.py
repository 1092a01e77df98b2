"""CP alignment padding, the one harness piece on the hot path.

Mirrors `/root/reference/pkg/src/balsim/harness.py:279-298`: a micro-batch whose
length is not a multiple of 2*cp gets ONE filler document of length
2cp - (T mod 2cp), with running negative ids starting at -1,000,000, so the
shard builder's inputs are identical to the reference's.
"""

from __future__ import annotations

from .workload import Document, MicroBatch


class _FillerIds:
    """Running negative ids for alignment filler, unique per experiment."""

    def __init__(self, start: int = -1_000_000):
        self.next_id = start

    def take(self) -> int:
        nid, self.next_id = self.next_id, self.next_id - 1
        return nid


FillerIds = _FillerIds


def pad_for_cp(mb: MicroBatch, cp: int, filler: _FillerIds, arrival: int) -> MicroBatch:
    """Return `mb` unchanged if divisible by 2*cp, else a copy with one filler doc."""
    short = mb.total_length % (2 * cp)
    if short == 0:
        return mb
    return MicroBatch(mb.docs + [Document(filler.take(), 2 * cp - short, arrival)])
