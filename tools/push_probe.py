"""Time the K/V push alone (kernel vs copy engines) for one 128K micro-batch
under torchrun: python -m torch.distributed.run --nproc-per-node 4 tools/push_probe.py"""
import json
import os
import sys
import time

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
    seq = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    spec = wl.SyntheticSpec(context_window=131072, tokens_per_global_batch=131072)
    lengths = [d.length for d in wl.generate_synthetic_stream(spec, 0, seq + 1)[seq]]
    plan = wl.build_shard_plan([lengths], world, "measured")
    sh = shard_for_rank(plan, 0, rank)
    tl, T = sh.gather_local.numel(), sum(lengths)
    k = torch.randn(tl, 32, 128, device=dev, dtype=torch.bfloat16)
    v = torch.randn_like(k)
    res = {"world": world, "seq": seq, "runs": None}
    for mode in ("covered", "dma"):
        os.environ["WLB_XCHG_PUSH"] = mode
        for G in (1, 4):
            ex = SymmExchange(dist.group.WORLD, T, 32, 128, dev, groups=G)
            if mode == "dma":
                res["runs"] = len(ex._runs(sh))
            ts = []
            for _ in range(3):
                dist.barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                ex.gather(k, v, sh, 0)
                for gi in range(len(ex.groups)):
                    ex.wait_kv(0, gi)
                b.record()
                b.synchronize()
                ts.append((a.elapsed_time(b), (time.perf_counter() - t0) * 1e3))
            res[f"{mode}_g{G}_ms"] = [round(x, 2) for x in min(ts)]
            del ex
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
