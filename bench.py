"""Benchmark: document-masked CP attention fwd+bwd on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload auto|128k] [--shape llama7b|llama70b-gqa]

With --gpus N > 1 and no torchrun environment, the script re-launches itself
under `torch.distributed.run --nproc-per-node N` (one process per GPU).

One step = the hot path over one synthetic global batch: the 8 long-tail
sequences `generate_synthetic_stream(SyntheticSpec(T, T), seed=0, n_batches=8)`
(BASELINE.md 3), each a micro-batch that is sharded + strategy-selected on
the GPU (one batched `wlb_shard_plan` launch), then run through CP
document-masked attention forward and backward (tcgen05 kernels, NCCL
all-gather / reduce-scatter for N > 1).

Workloads (BASELINE.json configs), `--workload auto` (default): N = 1 ->
config 2, Llama-7B attention (32 q / 32 kv heads, d = 128), seq 32K, CP = 1;
N > 1 -> config 3 shape at seq 128K, CP = N (one process per GPU).
`--workload 128k` runs the same 8 x 128K sequences at CP = N for every N,
including N = 1, so N = 1/2/4/8 is a strong-scaling curve of fixed work.

FLOPs are algorithmic and unmasked: 14 * D * Hq * pairs, pairs = sum over
documents of L(L+1)/2 (`attention_workload`, workload.py:196-198).
`value` = whole-job TFLOP/s = step FLOPs / max-over-ranks step time.
"""

from __future__ import annotations

import argparse
import json
import os
import select
import statistics
import subprocess
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200.attention import attn_backward, attn_forward  # noqa: E402
from paper_2503_17924_b200.hoststream import HostStreamedStep  # noqa: E402
from paper_2503_17924_b200.cp import (CPStepPipeline, NcclExchange, SymmExchange,  # noqa: E402
                                      build_cp_shards)

N_SEQ = 8
METRIC = "doc-masked attn TFLOP/s/GPU & CP rank imbalance (max/mean) at CP=1/2/4/8"


def _peaks():
    """(burst, sustained, kind) dense bf16 TFLOP/s.  The attention kernels run
    inside a long step (seconds of back-to-back tensor work under the 1 kW cap),
    so the roofline denominator is the SUSTAINED figure; burst is reported too."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        p = json.load(open(path))
        return p["bf16_tflops"], p.get("bf16_tflops_sustained") or p["bf16_tflops"], "measured"
    return 1590.0, 1400.0, "fallback"


def _workload(n, shape="llama7b", workload="auto"):
    """BASELINE configs: 2 (7B 32x128, 32K, CP=1) at N=1, 3 (7B, 128K, CP=N) at
    N>1; --shape llama70b-gqa gives config 4 (64 query / 8 KV heads x 128);
    --workload 128k keeps the 128K sequences at every N (CP = N, N = 1 too)."""
    hq, hkv = (64, 8) if shape == "llama70b-gqa" else (32, 32)
    tag = "llama70b-gqa" if shape == "llama70b-gqa" else "llama7b"
    if n == 1 and workload == "auto":
        return dict(name=f"{tag}-attn-32k-cp1", window=32768, hq=hq, hkv=hkv, d=128, cp=1)
    return dict(name=f"{tag}-attn-128k-cp{n}", window=131072, hq=hq, hkv=hkv, d=128, cp=n)


def _cpu_model():
    """`lscpu` model name of the host (BASELINE.md 4 asks for it with the core count)."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return None


def _host_steps(lengths_list, cp):
    """Reference host-side steps on this host's CPU:
    pad_for_cp + per-sequence / per-document sharding + model latencies +
    adaptive selection of every micro-batch, through the oracle port of
    sharding.py:86-188 (the reference's Python cannot travel to the GPU box).
    Returns ms per micro-batch (median of 3 passes).
    TEST/BASELINE ONLY: the checker is never the thing measured for `value`."""
    from oracle import shard_oracle as so
    import paper_2503_17924_b200 as pkg
    prof = pkg.CostProfile()
    cq = [q for q, _ in prof.tflops_curve]
    cv = [v for _, v in prof.tflops_curve]
    passes = []
    for _ in range(3):
        t0 = time.perf_counter()
        for ls in lengths_list:
            ls = so.pad_lengths_for_cp(ls, cp)
            strat = so.adaptive(ls, cp, prof.tile_size, cq, cv, prof.op_scale)
            so.shard(ls, cp, strat)              # the reference rebuilds the winner
        passes.append((time.perf_counter() - t0) * 1e3 / len(lengths_list))
    return statistics.median(passes)


def _lengths(window):
    spec = wl.SyntheticSpec(context_window=window, tokens_per_global_batch=window)
    return [[d.length for d in b] for b in wl.generate_synthetic_stream(spec, 0, N_SEQ)]


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index, period_ms=500):
        self.index = index
        self.period_ms = period_ms
        self.proc = None

    def __enter__(self):
        if self.period_ms <= 0:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        self.first = []  # pre-timed-region sample, not reported
        if self.proc is not None:
            # block until nvidia-smi is live, so its samples cover the timed region
            ready, _, _ = select.select([self.proc.stdout], [], [], 10.0)
            line = self.proc.stdout.readline() if ready else ""
            if line.strip():
                self.first.append(line)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.05)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in getattr(self, "lines", []):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        busy = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _bounded(lengths, max_pairs):
    """Documents in order, the last one cut to a prefix, so that the sample's
    causal pairs stay <= max_pairs (a prefix of a document is exact
    document-prefix attention of its own)."""
    out, used = [], 0
    for x in lengths:
        room = max_pairs - used
        if room <= 0:
            break
        if x * (x + 1) // 2 > room:
            x = max(1, int(((8 * room + 1) ** 0.5 - 1) // 2))
        out.append(x)
        used += x * (x + 1) // 2
    return out


def _cpu_sample(lengths_list, hq_sample, d, budget_s, first=0, max_pairs=1_500_000_000):
    """Oracle (torch-CPU fp32) fwd+bwd on head(s) of synthetic sequences, all host
    cores, each sequence bounded to max_pairs causal pairs (~10-15 s of CPU).
    TEST/BASELINE ONLY: the checker is never the thing measured for `value`."""
    from oracle import attention_oracle as ao
    from oracle import shard_oracle as so
    torch.set_num_threads(os.cpu_count())
    flops = secs = 0.0
    done = []
    i = first
    t_start = time.perf_counter()
    while True:
        lengths = so.pad_lengths_for_cp(_bounded(lengths_list[i % len(lengths_list)], max_pairs), 1)
        g = torch.Generator().manual_seed(1000 + i)
        T = sum(lengths)
        q = torch.randn(T, hq_sample, d, generator=g)
        k = torch.randn(T, hq_sample, d, generator=g)
        v = torch.randn(T, hq_sample, d, generator=g)
        do = torch.randn(T, hq_sample, d, generator=g)
        t0 = time.perf_counter()
        ranges = so.per_document(lengths, 1)[0]          # reference CP path (cp=1)
        ao.segment_attention_fwd_bwd(q, k, v, do, lengths, ranges)
        secs += time.perf_counter() - t0
        flops += 14.0 * d * hq_sample * sum(x * (x + 1) // 2 for x in lengths)
        done.append(i % len(lengths_list))
        i += 1
        if time.perf_counter() - t_start > budget_s or len(done) >= len(lengths_list):
            break
    return flops / secs / 1e12, done, secs


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path (oracle port: the reference
    computes no attention; its sharding is Python and cannot travel) on the
    host cores, rank 0 only."""
    if rank != 0:
        return
    wk = _workload(world, args.shape, args.workload)
    lengths = _lengths(wk["window"])
    vals = []
    secs_tot = flops_tot = 0.0
    for s in range(args.warmup + args.steps):
        tflops, done, secs = _cpu_sample(lengths, 1, wk["d"], budget_s=0.0, first=s)
        if s >= args.warmup:
            vals.append(tflops)
            secs_tot += secs
            flops_tot += tflops * 1e12 * secs
    value = flops_tot / secs_tot / 1e12
    line = {
        "impl": "reference", "metric": METRIC,
        "value": round(value, 4), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(secs_tot / args.steps * 1e3, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": wk["name"], "seq_len": wk["window"], "sequences_per_step": N_SEQ,
                   "heads": [wk["hq"], wk["hkv"]], "head_dim": wk["d"], "cp": wk["cp"],
                   "policy": "per_document (CPU sample)", "parallelism": f"cp{wk['cp']}"},
        "cpu_baseline": {"value": round(value, 4), "unit": "TFLOP/s", "cores": os.cpu_count(),
                         "cpu_model": _cpu_model(), "kind": "port",
                         "sample": "per step: head 0 of one synthetic sequence (cycling the 8), "
                                   "documents in order up to 1.5e9 causal pairs (last one "
                                   "prefix-cut), per_document shard + torch-CPU fp32 "
                                   "doc-prefix attention fwd+bwd (oracle/attention_oracle.py)",
                         "host_shard_select_ms_per_mb": round(_host_steps(lengths, wk["cp"]), 3)},
        "e2e": {"value": round(value, 4), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", default="symm", choices=["nccl", "symm"],
                    help="CP K/V + dK/dV exchange: NCCL collectives or one-sided NVLink "
                         "stores/loads on symmetric memory")
    ap.add_argument("--shape", default="llama7b", choices=["llama7b", "llama70b-gqa"],
                    help="attention shape: Llama-7B 32x128 (configs 2/3) or Llama-70B GQA "
                         "64q/8kv x128 (config 4)")
    ap.add_argument("--workload", default="auto", choices=["auto", "128k"],
                    help="auto: 32K CP=1 at N=1 (config 2), 128K CP=N at N>1 (config 3); "
                         "128k: 128K CP=N at every N (fixed total work: strong scaling)")
    ap.add_argument("--clock-ms", type=int, default=100,
                    help="nvidia-smi sampling period during the timed region (0: off)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (the driver launches
        # torchrun itself; a bare `python bench.py --gpus N` lands here)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={29500 + os.getpid() % 1000}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one process per GPU")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    group = None
    wk = _workload(world, args.shape, args.workload)
    cp, hq, hkv, d = wk["cp"], wk["hq"], wk["hkv"], wk["d"]
    lengths = _lengths(wk["window"])
    T = wk["window"]
    tl = T // cp

    # inputs resident in HBM: this rank's local tokens of every sequence
    gen = torch.Generator(device=dev)
    ins = []
    for b in range(N_SEQ):
        gen.manual_seed(1000 + 64 * b + rank)
        mk = lambda h: torch.randn((tl, h, d), generator=gen, device=dev, dtype=torch.bfloat16)
        ins.append((mk(hq), mk(hkv), mk(hkv), mk(hq)))

    ev = lambda: torch.cuda.Event(enable_timing=True)
    launches = [0]

    symm = args.exchange == "symm" and cp > 1
    exchange = SymmExchange(dist.group.WORLD, T, hkv, d, dev) if symm else NcclExchange(group)
    pipe = CPStepPipeline(group, exchange=exchange)

    def mb_launches():
        """Kernel launches of this library per micro-batch (memsets excluded):
        tile list + forward + backward (Delta, KV tiles, backward, dQ
        conversion; + uncovered-row zero fill without the covered pull) and the
        exchange.  Symmetric exchange, G head groups, group-by-group launches:
        per group a flag wait + forward, backward passes + a signal, push +
        signal, wait + pull, plus the two slot barriers."""
        if cp == 1:
            return 1 + 1 + 5
        if not symm:
            return 1 + 1 + 5 + 4                            # 2 row scatters + 2 row gathers
        g = len(exchange.groups)
        if exchange.fused_sync:
            return 1 + 1 + 4 + 2 + 4 * g
        return 1 + 2 * g + 5 * g + 2 + 4 * g

    # CP > 1: per-sequence vs per-document chosen by the measured-latency tile
    # model calibrated on B200 (tilemodel.py); CP = 1 has one sharding, which
    # the reference selector (bit-exact with balsim) picks
    policy = "measured" if cp > 1 else "adaptive"
    model = wl.TileModel.for_shape(hq, hkv, d) if cp > 1 else None

    def step(record=None):
        shards = build_cp_shards(lengths, cp, rank, policy, model=model)
        launches[0] += 1 + N_SEQ * mb_launches()                # plan + per micro-batch

        def timed(b, sh, kernels):
            if record is None:
                return kernels()
            e = [ev() for _ in range(2)]
            e[0].record()
            res = kernels()
            e[1].record()
            record.append((e, sh))
            return res

        # outputs are released micro-batch by micro-batch: holding a whole step's
        # outputs (~20 GB) made the caching allocator free + re-malloc (device syncs)
        pipe.run(shards, ins, on_kernels=timed, keep_outputs=False)
        return shards

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        shards = step()
    barrier()

    # ------------------------------------------------------------ timed loop --
    launches[0] = 0
    recs = []
    t0, t1 = ev(), ev()
    with ClockSampler(local_rank, args.clock_ms) as clk:
        barrier()
        t0.record()
        for _ in range(args.steps):
            shards = step(record=recs)
        t1.record()
        barrier()
    my_ms = t0.elapsed_time(t1)
    alloc_retries = torch.cuda.memory_stats(dev).get("num_alloc_retries", 0)
    kern_each = [e[0].elapsed_time(e[1]) for e, _ in recs]
    # per micro-batch kernel time of this rank, mean over the timed steps
    mb_ms = torch.tensor([sum(kern_each[s * N_SEQ + b] for s in range(args.steps)) / args.steps
                          for b in range(N_SEQ)], device=dev, dtype=torch.float64)
    my_pairs = sum(sh.pairs for sh in shards)
    total_pairs = sum(sum(x * (x + 1) // 2 for x in ls) for ls in lengths)
    step_flops = 14.0 * d * hq * total_pairs
    kern_ms = sum(kern_each)
    stats = torch.tensor([my_ms, kern_ms, float(my_pairs)], device=dev, dtype=torch.float64)
    if world > 1:
        allv = [torch.empty_like(stats) for _ in range(world)]
        dist.all_gather(allv, stats)
        allv = torch.stack(allv).cpu()
        allmb = [torch.empty_like(mb_ms) for _ in range(world)]
        dist.all_gather(allmb, mb_ms)
        allmb = torch.stack(allmb).cpu()
    else:
        allv = stats.cpu()[None]
        allmb = mb_ms.cpu()[None]
    max_ms = float(allv[:, 0].max())
    ms_step = max_ms / args.steps
    value = step_flops * args.steps / (max_ms / 1e3) / 1e12
    kt = allv[:, 1]
    imbalance = float(kt.max() / kt.mean())
    pair_imb = float(allv[:, 2].max() / allv[:, 2].mean())
    strategies = [sh.strategy.value for sh in shards]

    # ------------------------------------------------------------------ e2e --
    # The same step through the public API with host buffers: every step copies
    # each micro-batch's q, k, v, dO from pinned host memory (H2D stream) and
    # reads o, dq, dk, dv back (D2H stream); the copies are pipelined against
    # compute across micro-batches with CUDA events.
    e2e = None
    if not args.no_e2e:
        pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t.cpu())
        host_in = [pin(t) for t in ins[0]]
        host_out = [torch.empty((tl, hq, d), dtype=torch.bfloat16, pin_memory=True),
                    torch.empty((tl, hq, d), dtype=torch.bfloat16, pin_memory=True),
                    torch.empty((tl, hkv, d), dtype=torch.bfloat16, pin_memory=True),
                    torch.empty((tl, hkv, d), dtype=torch.bfloat16, pin_memory=True)]
        # hoststream.HostStreamedStep: copies pipelined against the attention,
        # per KV-head group where the step is PCIe-bound (each group's columns
        # of q, k, v, dO land and its O, dQ, dK, dV leave on their own, so one
        # group's transfer, not one micro-batch's, is exposed at the step's
        # start and end), per micro-batch where the attention dominates
        gsel = os.environ.get("WLB_E2E_GROUPS", "auto")
        streamer = HostStreamedStep(pipe, groups=None if gsel == "mb" else
                                    gsel if gsel == "auto" else int(gsel),
                                    order=os.environ.get("WLB_E2E_ORDER", "given"))

        def e2e_step():
            shards = build_cp_shards(lengths, cp, rank, policy, model=model)
            streamer.run(shards, [host_in] * N_SEQ, ins, [host_out] * N_SEQ)

        e2e_step()
        barrier()
        retries0 = torch.cuda.memory_stats(dev).get("num_alloc_retries", 0)
        a, b_ = ev(), ev()
        n_e2e = args.steps
        marks = []
        a.record()
        for _ in range(n_e2e):
            e2e_step()
            marks.append(ev())
            marks[-1].record()
        b_.record()
        barrier()
        e2e_steps = [round(x.elapsed_time(y), 1) for x, y in zip([a] + marks[:-1], marks)]
        e_ms = torch.tensor([a.elapsed_time(b_)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        h2d = N_SEQ * sum(t.numel() * t.element_size() for t in host_in)
        d2h = N_SEQ * sum(t.numel() * t.element_size() for t in host_out)
        e2e = {"value": round(step_flops * n_e2e / (float(e_ms) / 1e3) / 1e12, 2),
               "unit": "TFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(float(e_ms) / n_e2e, 2),
               "granularity": ("micro-batch" if streamer.last_groups is None else
                               f"{streamer.last_groups} KV-head groups"),
               "order": streamer.last_order, "rank0_step_ms": e2e_steps,
               "alloc_retries": torch.cuda.memory_stats(dev).get("num_alloc_retries", 0) - retries0,
               "note": "every micro-batch: H2D k,v,q then dO from pinned host, D2H o "
                       "(during the backward) then dq,dk,dv, copy streams pipelined against "
                       "the attention (hoststream.HostStreamedStep); shard plan + attention "
                       "through the public API"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_sus, peak_kind = _peaks()
    # dominant kernel: the attention fwd+bwd pair of each micro-batch (CUDA events
    # on the launching stream around exactly those launches)
    dom = ("attn_fwd+bwd", 14.0 * d * hq * my_pairs * args.steps, kern_ms)
    achieved = dom[1] / (dom[2] / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(wk["name"], {}).get(dom[0])
    line = {
        "metric": METRIC,
        "value": round(value, 2), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "value_basis": "whole job: step FLOPs (all ranks) / max-over-ranks step time; "
                       "per GPU in tflops_per_gpu",
        "config": {"workload": wk["name"], "seq_len": T, "sequences_per_step": N_SEQ,
                   "heads": [hq, hkv], "head_dim": d, "cp": cp, "policy": policy,
                   "workload_rule": "N=1: config 2 (32K, CP=1); N>1: config 3 (128K, CP=N); "
                                    "--workload 128k: 128K at CP=N for every N"
                                    if args.workload == "auto" else "128K at CP=N for every N",
                   "strategies": strategies, "l2": "inputs > L2 (256 MiB per tensor)",
                   "parallelism": f"cp{cp}",
                   "exchange": args.exchange if cp > 1 else "none"},
        "tflops_per_gpu": round(value / world, 2),
        "frac_of_peak": round(value / world / peak_sus, 4),
        "frac_of_burst_peak": round(value / world / peak, 4),
        "imbalance": round(imbalance, 4),
        "pair_imbalance": round(pair_imb, 5),
        "rank_kernel_ms": [round(float(x), 3) for x in kt],
        "rank_mb_kernel_ms": [[round(float(x), 2) for x in row] for row in allmb],
        "kernel_ms": round(kern_ms, 3),
        "roofline": {"kernel": dom[0], "bound": "tensor", "achieved": round(achieved, 1),
                     "peak": peak_sus, "unit": "TFLOP/s", "frac": round(achieved / peak_sus, 4),
                     "frac_burst": round(achieved / peak, 4),
                     "peak_kind": f"{peak_kind} sustained bf16 (burst {peak})",
                     "traffic": traffic,
                     "flops_basis": "14*D*Hq*pairs_rank per (fwd+bwd) launch pair"},
        "gpu_launches": launches[0],
        "alloc_retries": alloc_retries,
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if world == 1 and not args.no_cpu_baseline:
        tflops, done, secs = _cpu_sample(lengths, 1, d, budget_s=15.0)
        line["cpu_baseline"] = {
            "value": round(tflops, 4), "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "port",
            "cpu_model": _cpu_model(),
            "sample": f"head 0 of synthetic sequences {done}, each bounded to 1.5e9 causal "
                      f"pairs ({secs:.1f} s): per_document shard + torch-CPU fp32 "
                      "doc-prefix attention fwd+bwd (oracle)",
            "host_shard_select_ms_per_mb": round(_host_steps(lengths, cp), 3),
            "gpu_shard_select": "one wlb_shard_plan launch per step (all micro-batches)"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
