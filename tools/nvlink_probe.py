"""NVLink throughput of the CP exchange kernels (full push / full pull, so
the bytes are exact): one 128K micro-batch, 7B shape, under torchrun.
Remote bytes per rank: push (cp-1)/cp * T/cp rows * cp ranks... i.e. every
local row to the cp-1 peers; pull: this rank's T/cp rows from cp-1 peers.

    python -m torch.distributed.run --nproc-per-node 4 tools/nvlink_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200.cp import SymmExchange, shard_for_rank  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    os.environ["WLB_XCHG_PUSH"] = "all"
    os.environ["WLB_XCHG_PULL"] = "all"
    spec = wl.SyntheticSpec(context_window=131072, tokens_per_global_batch=131072)
    lengths = [d.length for d in wl.generate_synthetic_stream(spec, 0, 3)[2]]
    plan = wl.build_shard_plan([lengths], world, "per_document")
    sh = shard_for_rank(plan, 0, rank)
    tl, T, hkv, d = sh.gather_local.numel(), sum(lengths), 32, 128
    k = torch.randn(tl, hkv, d, device=dev, dtype=torch.bfloat16)
    v = torch.randn_like(k)
    res = {"world": world, "rows_per_rank": tl}
    for G in (1, 4):
        ex = SymmExchange(dist.group.WORLD, T, hkv, d, dev, groups=G)
        dk_out, dv_out = ex.dkv_out(sh, 0, torch.cuda.current_stream())
        dk_out.zero_()
        dv_out.zero_()
        best_push = best_pull = 1e9
        for _ in range(4):
            dist.barrier()
            torch.cuda.synchronize()
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record()
            ex.gather(k, v, sh, 0)
            for gi in range(len(ex.groups)):
                ex.wait_kv(0, gi)
            b.record()
            for gi in range(len(ex.groups)):
                ex.signal_dkv(0, gi)
            ex.scatter(dk_out, dv_out, sh, 0)
            c.record()
            c.synchronize()
            best_push = min(best_push, a.elapsed_time(b))
            best_pull = min(best_pull, b.elapsed_time(c))
        kv_row = hkv * d * 2 * 2                    # K + V bf16
        dkv_row = hkv * d * 4 * 2                   # dK + dV fp32 partials
        push_remote = tl * kv_row * (world - 1)
        pull_remote = tl * dkv_row * (world - 1)
        res[f"g{G}"] = {"push_ms": round(best_push, 3), "pull_ms": round(best_pull, 3),
                        "push_remote_GB": round(push_remote / 1e9, 3),
                        "pull_remote_GB": round(pull_remote / 1e9, 3),
                        "push_GBps": round(push_remote / best_push / 1e6, 1),
                        "pull_GBps": round(pull_remote / best_pull / 1e6, 1)}
        del ex
    t = torch.tensor([res["g1"]["push_ms"], res["g1"]["pull_ms"]], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
