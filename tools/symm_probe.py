"""Feasibility probe: torch symmetric memory + peer stores across GPUs (dev aid)."""
import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank); dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
buf = symm.empty(1 << 20, dtype=torch.float32, device=dev)
h = symm.rendezvous(buf, dist.group.WORLD)
buf.fill_(-1.0)
h.barrier()
peer = (rank + 1) % world
# write our rank id into the peer's buffer through its mapped pointer
remote = h.get_buffer(peer, (1 << 20,), torch.float32)
remote.fill_(float(rank))
h.barrier()
torch.cuda.synchronize()
expect = float((rank - 1) % world)
print(f"rank {rank}: ptrs={len(h.buffer_ptrs)} got {buf[0].item()} expect {expect} ok={bool((buf == expect).all())}", flush=True)
dist.destroy_process_group()
