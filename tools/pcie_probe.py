"""PCIe probe for the e2e leg: H2D alone, D2H alone, and both at once
(full duplex) for the bench's per-step volume (8 x 64 MiB each way)."""
import time

import torch

n, size = 8, 64 << 20
dev = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in range(n)]
dev2 = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in range(n)]
hin = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
hout = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
a, b = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if h2d:
            with torch.cuda.stream(a):
                for d, h in zip(dev, hin):
                    d.copy_(h, non_blocking=True)
        if d2h:
            with torch.cuda.stream(b):
                for d, h in zip(dev2, hout):
                    h.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


gb = n * size / 1e9
th = run(True, False)
td = run(False, True)
tb = run(True, True)
print(f"H2D {gb / th:.1f} GB/s ({th * 1e3:.2f} ms); D2H {gb / td:.1f} GB/s ({td * 1e3:.2f} ms); "
      f"both {tb * 1e3:.2f} ms (duplex efficiency {max(th, td) / tb:.2f})")
