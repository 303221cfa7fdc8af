"""Can the SM mover fill the device->host direction of PCIe better than a
copy engine while a copy engine fills host->device? 8 co-resident ranks,
all-to-all of 8 x 64 MiB (the headline workload):
  ce_h2d        copy engine, 512 MiB host -> device
  ce_d2h        copy engine, 512 MiB device -> host
  ce_both       both at once (two streams)
  sm_to_host    the collective writing its result straight into pinned host
                memory (SM stores over PCIe, no HBM write of recv)
  ce_h2d+sm     ce_h2d concurrently with sm_to_host
Prints ms (median of 5)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_06605_b200 as cc  # noqa: E402

n, s = 8, 8 << 20
comms = cc.Comm.init_all([0] * n)
dev_in = [torch.randint(0, 256, (n * s,), dtype=torch.uint8, device="cuda") for _ in range(n)]
dev_out = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
host_in = [torch.empty(n * s, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
host_out = [torch.empty(n * s, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
a, b, c = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for st in (a, b, c):
            st.wait_event(e0)
        fn()
        for st in (a, b, c):
            ev = torch.cuda.Event()
            ev.record(st)
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def ce_h2d():
    with torch.cuda.stream(a):
        for h, d in zip(host_in, dev_in):
            d.copy_(h, non_blocking=True)


def ce_d2h():
    with torch.cuda.stream(b):
        for h, d in zip(host_out, dev_out):
            h.copy_(d, non_blocking=True)


def sm_to_host(impl="sm"):
    cc.all_to_all(comms, dev_in, host_out, s, impl=impl, streams=c)


for impl in ("sm", "pcpy"):
    sm_to_host(impl)
    torch.cuda.synchronize()
    ok = all(torch.equal(host_out[j][i * s:(i + 1) * s].cuda(), dev_in[i][j * s:(j + 1) * s])
             for i in range(n) for j in (0, n - 1))
    print(f"parity collective->host ({impl}): {ok}")
res = {
    "ce_h2d": timed(ce_h2d),
    "ce_d2h": timed(ce_d2h),
    "ce_both": timed(lambda: (ce_h2d(), ce_d2h())),
    "sm_to_host": timed(lambda: sm_to_host("sm")),
    "ce_h2d+sm_to_host": timed(lambda: (ce_h2d(), sm_to_host("sm"))),
    "pcpy_to_host": timed(lambda: sm_to_host("pcpy")),
    "ce_h2d+pcpy_to_host": timed(lambda: (ce_h2d(), sm_to_host("pcpy"))),
}
for k, v in res.items():
    print(f"{k:22s} {v:8.3f} ms  ({n * n * s / v / 1e6:6.1f} GB/s per direction-equivalent)")
cc.destroy_all(comms)
