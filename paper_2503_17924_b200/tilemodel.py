"""Measured-latency model of the B200 attention kernels for the CP selector.

North-star item 4: per-sequence vs per-document sharding is selected by
MEASURED kernel latency (`/root/reference/PAPER.md:425-429`: the paper
profiles the attention kernel and picks the strategy with the lower
predicted latency).  The reference encodes its prediction as a
`balsim.profile.v1` CostProfile that charges every canonical range a dense
q x kv rectangle (`workload.py:239-255`, `sharding.py:151-188`); that form
cannot see this repo's causal tile skipping, back-aligned query tiles or
tile pairing, so no calibration of it ranks the strategies reliably.

`TileModel` instead prices the work lists the kernels will actually run.
The GPU planner (`wlb_shard_plan_measured`, `csrc/shard_plan.cu`) counts,
per (strategy, rank):

* forward: query-tile pairs (items) and 128 x 128 (query tile, KV tile)
  steps; the largest item;
* backward: 128-key KV tiles (items) and their 64-query (v2) / 128-query
  (v3) steps; the largest item;

and predicts, per direction, from the even-spread time S = (item and step
costs summed) / SMs and the largest item M,

    t_dir = max(S, M) + g_dir * min(S, M)
    t     = t_fwd + t_bwd + c0

max(S, M) is the ideal makespan; the tail term g * min(S, M) is the part of
the largest item that list scheduling cannot hide behind the others (Graham's
bound S + M is g = 1).  Without it the model under-priced per-sequence ranks
of few, long KV tiles by 1.3-1.7x (GQA 32K at cp 2-4).  The per-unit costs of
the backward kernel the library picks for that rank, the two tail weights and
c0 are fitted to kernel times measured on B200 (`calibrate.fit_tile_model`).  The selector keeps the
reference's rule: per-sequence when its slowest rank is predicted no slower.
The reference `CostProfile` path stays available, bit-exact, for parity.
"""

from __future__ import annotations

import json
import os
from dataclasses import asdict, dataclass

from .errors import ConfigError

SCHEMA = "wlbcp.tilemodel.v1"
DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")
FEATURES = ("fwd_items", "fwd_steps", "fwd_max", "bwd_items", "bwd_q64", "bwd_q128",
            "bwd_max64", "bwd_max128")


@dataclass(frozen=True)
class TileModel:
    hq: int = 32
    hkv: int = 32
    d: int = 128
    sms: int = 148
    fwd_item_s: float = 3.0e-6
    fwd_step_s: float = 0.95e-6
    bwd_item_s: float = 4.0e-6
    bwd_step64_s: float = 1.5e-6
    bwd_step128_s: float = 2.75e-6
    v3_min_rows: int = 1
    const_s: float = 3.0e-5
    source: str = "defaults (pre-calibration estimates from the kernel traces)"
    # per-item cost of the 128-query backward (bwd_item_s is the 64-query
    # kernel's; its persistent unit queue makes an item much cheaper); None:
    # same as bwd_item_s (models calibrated before the split)
    bwd_item128_s: float | None = None
    # list-scheduling tail weights (0: the pre-tail model, max(S, M) only)
    fwd_tail: float = 0.0
    bwd_tail: float = 0.0

    def __post_init__(self):
        if self.hq <= 0 or self.hkv <= 0 or self.hq % self.hkv:
            raise ConfigError("hq must be a positive multiple of hkv")
        costs = (self.fwd_item_s, self.fwd_step_s, self.bwd_item_s, self.bwd_step64_s,
                 self.bwd_step128_s, self.const_s, self.item128, self.fwd_tail, self.bwd_tail)
        if min(costs) < 0 or self.sms < 1:
            raise ConfigError("tile-model costs must be >= 0 and sms >= 1")

    @property
    def item128(self) -> float:
        return self.bwd_item_s if self.bwd_item128_s is None else self.bwd_item128_s

    def array(self) -> list[float]:
        """The WLB_TILE_MODEL_LEN doubles `wlb_shard_plan_measured` reads."""
        return [float(self.sms), float(self.hq), float(self.hkv), self.fwd_item_s,
                self.fwd_step_s, self.bwd_item_s, self.bwd_step64_s, self.bwd_step128_s,
                float(self.v3_min_rows), self.const_s, 1.0 if self.d == 128 else 0.0,
                self.item128, self.fwd_tail, self.bwd_tail]

    def predict(self, f, tl: int, n_docs: int) -> float:
        """Host restatement of the kernel's prediction for one feature row
        (dict or sequence in FEATURES order); used by calibration reports."""
        if not isinstance(f, dict):
            f = dict(zip(FEATURES, f))
        v3 = self.d == 128 and tl >= self.v3_min_rows * max(1, n_docs)
        bq, bm = (f["bwd_q128"], f["bwd_max128"]) if v3 else (f["bwd_q64"], f["bwd_max64"])
        bs = self.bwd_step128_s if v3 else self.bwd_step64_s
        bi = self.item128 if v3 else self.bwd_item_s
        sf = (self.fwd_item_s * f["fwd_items"] + self.fwd_step_s * f["fwd_steps"]) * self.hq / self.sms
        mf = self.fwd_item_s + self.fwd_step_s * f["fwd_max"]
        sb = (bi * f["bwd_items"] * self.hkv + bs * bq * self.hq) / self.sms
        mb = bi + bs * bm * self.hq / self.hkv
        tf = max(sf, mf) + self.fwd_tail * min(sf, mf)
        tb = max(sb, mb) + self.bwd_tail * min(sb, mb)
        return tf + tb + self.const_s

    def to_dict(self) -> dict:
        return {"schema": SCHEMA, **asdict(self)}

    @classmethod
    def from_dict(cls, data: dict) -> "TileModel":
        if data.get("schema") != SCHEMA:
            raise ConfigError(f"not a {SCHEMA} document")
        fields = {k: v for k, v in data.items() if k != "schema"}
        return cls(**fields)

    def to_file(self, path: str) -> None:
        with open(path, "w") as fh:
            json.dump(self.to_dict(), fh, indent=1)

    @classmethod
    def from_file(cls, path: str) -> "TileModel":
        with open(path) as fh:
            return cls.from_dict(json.load(fh))

    @classmethod
    def for_shape(cls, hq: int, hkv: int, d: int) -> "TileModel":
        """The B200-calibrated model shipped for this head shape
        (`data/b200_tiles_h{hq}_kv{hkv}_d{d}.json`), else the nearest shipped
        calibration re-labelled for this shape, else the defaults."""
        path = os.path.join(DATA, f"b200_tiles_h{hq}_kv{hkv}_d{d}.json")
        if os.path.exists(path):
            return cls.from_file(path)
        for name in sorted(os.listdir(DATA)) if os.path.isdir(DATA) else []:
            if name.startswith("b200_tiles_") and name.endswith(f"_d{d}.json"):
                m = cls.from_file(os.path.join(DATA, name)).to_dict()
                m.update(hq=hq, hkv=hkv, source=f"{name} (calibrated for another head count)")
                return cls.from_dict(m)
        return cls(hq=hq, hkv=hkv, d=d)
