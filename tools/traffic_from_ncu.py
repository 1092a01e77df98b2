"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch) of
`bench.py --steps 1 --warmup 1`: per-kernel shares of the timed step, and the
DRAM traffic per attention fwd+bwd launch pair written to profiles/traffic.json
(read by bench.py for `roofline.traffic`).  Dev aid; the per-launch times are
cold-cache and serialised, so shares (not absolutes) are what compare.

    python tools/traffic_from_ncu.py gpurun_out/launches.csv llama7b-attn-32k-cp1 > profiles/..txt
"""
import collections
import csv
import json
import os
import sys

path, workload = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
launch = collections.OrderedDict()
for r in rows[1:]:
    lid = int(r[ix["ID"]])
    d = launch.setdefault(lid, {"name": r[ix["Kernel Name"]]})
    d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
ids = list(launch)
# the second shard-plan launch starts the timed step (warm-up step first)
plan = [i for i in ids if "shard_plan_kernel" in launch[i]["name"]]
step = [i for i in ids if i >= plan[-1]] if len(plan) >= 2 else ids


def short(n):
    n = n.replace("void ", "")
    return n.split("(")[0][:60]


agg = collections.OrderedDict()
for i in step:
    d = launch[i]
    a = agg.setdefault(short(d["name"]), [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
unit_t = "ns" if tot > 1e6 else "?"
print(f"# ncu launch list of one timed bench step ({workload}): {len(step)} launches")
print(f"# {'kernel':60s} {'n':>4s} {'time share':>10s} {'DRAM GB':>9s}")
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k:60s} {n:4d} {t / tot:10.1%} {b / 1e9:9.3f}")
fb = [a for k, a in agg.items() if "attn_fwd_kernel" in k or "attn_bwd" in k and "kernel" in k]
pairs = max(1, sum(a[0] for k, a in agg.items() if "attn_fwd_kernel" in k))
traffic = sum(a[2] for k, a in agg.items() if k.startswith(("wlb::attn_fwd_kernel", "wlb::attn_bwd_kernel", "wlb::attn_bwd3_kernel")))
per_pair = traffic / pairs
print(f"# attention fwd+bwd DRAM traffic per launch pair: {per_pair / 1e9:.3f} GB over {pairs} pairs")
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
data = json.load(open(out)) if os.path.exists(out) else {}
data[workload] = {"attn_fwd+bwd": {"bytes_per_launch_pair": round(per_pair),
                                   "source": os.path.basename(path),
                                   "metric": "dram__bytes_read.sum + dram__bytes_write.sum"}}
json.dump(data, open(out, "w"), indent=1)
