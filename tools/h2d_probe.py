"""Host->device copy bandwidth probe (pinned, 1 vs 2 vs 4 streams) used to size
the host-buffer C ABI's transfer pipeline (e2e)."""
import time
import torch

N = 1 << 30
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = N // ns
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"H2D streams={ns}: {N / dt / 1e9:.1f} GB/s")
hd = torch.empty(N, dtype=torch.uint8, pin_memory=True)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hd.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"D2H: {N / dt / 1e9:.1f} GB/s")
