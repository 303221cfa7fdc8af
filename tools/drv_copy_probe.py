"""Profile target: the driver's same-device copy kernel (cudaMemcpyAsync D2D)
at 1 GiB, to compare its launch shape and SASS with tma_items_kernel."""
import torch

n = 1 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda").random_()
b = torch.empty_like(a)
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(10):
    e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(f"memcpy 1GiB best {best*1e3:.1f} us -> {2*n/best/1e6:.1f} GB/s")
