"""Development aid: pinned-host <-> device copy bandwidth (alone and concurrent)."""
import torch, time
n = 256 << 20
dev = torch.device("cuda")
h_in = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
h_out = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
d = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(8)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=4):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                for i in range(4): d[i].copy_(h_in[i], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                for i in range(4): h_out[i].copy_(d[4 + i], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    return reps * 4 * n / dt / 1e9
run(True, True, 1)
print(f"H2D alone {run(True, False):.1f} GB/s | D2H alone {run(False, True):.1f} GB/s | "
      f"concurrent each {run(True, True):.1f} GB/s")
import os
print("cpus", os.cpu_count(), "numa", open('/sys/devices/system/node/online').read().strip() if os.path.exists('/sys/devices/system/node/online') else '?')
