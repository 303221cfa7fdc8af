"""PCIe duplex probe for the e2e leg (bench.py): 8 x 64 MiB host->device and
8 x 64 MiB device->host per step, both directions at once, varying the
number of streams per direction (copy engines in use) and the copy size.
Prints the best per-step time of each variant (CUDA events, 5 repetitions)."""
import json
import sys

import torch

n, size = 8, 64 << 20
dev_in = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in range(n)]
dev_out = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in range(n)]
hin = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
hout = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
streams = {k: [torch.cuda.Stream() for _ in range(4)] for k in ("h2d", "d2h")}


def step(h2d, d2h, nst, piece):
    jobs_in = [(d[o:o + piece], h[o:o + piece]) for d, h in zip(dev_in, hin) for o in range(0, size, piece)]
    jobs_out = [(h[o:o + piece], d[o:o + piece]) for d, h in zip(dev_out, hout) for o in range(0, size, piece)]
    if h2d:
        for k, (dst, src) in enumerate(jobs_in):
            with torch.cuda.stream(streams["h2d"][k % nst]):
                dst.copy_(src, non_blocking=True)
    if d2h:
        for k, (dst, src) in enumerate(jobs_out):
            with torch.cuda.stream(streams["d2h"][k % nst]):
                dst.copy_(src, non_blocking=True)


def timed(h2d, d2h, nst, piece, reps=5):
    cur = torch.cuda.current_stream()
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for st in streams["h2d"] + streams["d2h"]:
            st.wait_event(e0)
        step(h2d, d2h, nst, piece)
        for st in streams["h2d"] + streams["d2h"]:
            cur.wait_stream(st)
        e1.record(cur)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


res = {}
for nst in (1, 2, 4):
    for piece in (64 << 20, 8 << 20):
        key = f"streams{nst}_piece{piece >> 20}MiB"
        res[key] = {"h2d_ms": round(timed(True, False, nst, piece), 3), "d2h_ms": round(timed(False, True, nst, piece), 3),
                    "both_ms": round(timed(True, True, nst, piece), 3)}
        print(key, res[key], flush=True)
json.dump(res, sys.stdout)
print()
