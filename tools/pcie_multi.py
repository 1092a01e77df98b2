"""Development aid: per-GPU pinned-host copy rates with every rank copying at
once (H2D and D2H together), under torchrun."""
import os
import time

import torch
import torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
dev = torch.device("cuda", torch.cuda.current_device())
dist.init_process_group("nccl", device_id=dev)
n = 1 << 30
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(n, dtype=torch.uint8, device=dev)
d_out = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for mode in ("h2d", "d2h", "both"):
    for rep in range(3):
        dist.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(2):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d_in.copy_(h_in, non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h_out.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize()
        res[mode] = 2 * n / (time.perf_counter() - t) / 1e9
out = [None] * world
dist.all_gather_object(out, res)
if rank == 0:
    for r, x in enumerate(out):
        print(f"world {world} rank {r}: H2D {x['h2d']:.1f} GB/s | D2H {x['d2h']:.1f} | both, each {x['both']:.1f}")
dist.destroy_process_group()
