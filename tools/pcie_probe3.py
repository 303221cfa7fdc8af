"""PCIe duplex with k streams per direction (8 x 64 MiB each way): does
spreading each direction over more copy engines beat one stream each?"""
import torch

n, size = 8, 64 << 20
dev = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in range(n)]
dev2 = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in range(n)]
hin = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
hout = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(n)]


def run(k, reps=5, split=1):
    hs = [torch.cuda.Stream() for _ in range(k)]
    ds = [torch.cuda.Stream() for _ in range(k)]
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for st in hs + ds:
            st.wait_event(e0)
        for i in range(n):
            for p in range(split):
                lo, hi = p * size // split, (p + 1) * size // split
                with torch.cuda.stream(hs[(i * split + p) % k]):
                    dev[i][lo:hi].copy_(hin[i][lo:hi], non_blocking=True)
                with torch.cuda.stream(ds[(i * split + p) % k]):
                    hout[i][lo:hi].copy_(dev2[i][lo:hi], non_blocking=True)
        for st in hs + ds:
            ev = torch.cuda.Event()
            ev.record(st)
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


for k in (1, 2, 4, 8):
    t = run(k)
    print(f"streams/direction {k}: both {t:.3f} ms ({2 * n * size / t / 1e6:.1f} GB/s combined)", flush=True)
t = run(4, split=4)
print(f"streams/direction 4, 16 MiB pieces: both {t:.3f} ms ({2 * n * size / t / 1e6:.1f} GB/s combined)")
