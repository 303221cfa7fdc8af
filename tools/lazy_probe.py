"""Does a lazily loaded kernel's first launch wait behind an armed prelaunch
plan? Arms an explicit plan, then launches torch kernels never used before
in this process and times them (run under `timeout`)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2511_06605_b200 as cc

n, s = 2, 4096
cs = cc.Comm.init_all([0] * n)
sends = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
recvs = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
stream = torch.cuda.current_stream()
plan = cc.Plan(cs, "alltoall", sends, recvs, s, impl=sys.argv[1] if len(sys.argv) > 1 else "prelaunch_pcpy")
plan.launch([stream] * n)
stream.synchronize()  # the next instance is armed now
print("armed", flush=True)
for name, fn in [("cumsum f64", lambda: torch.arange(1000, device="cuda", dtype=torch.float64).cumsum(0)),
                 ("sort i16", lambda: torch.randint(0, 100, (5000,), device="cuda", dtype=torch.int16).sort()),
                 ("fft", lambda: torch.fft.fft(torch.randn(256, device="cuda")))]:
    t0 = time.time()
    fn()
    stream.synchronize()
    print(f"{name}: {time.time() - t0:.3f} s", flush=True)
plan.launch([stream] * n)
stream.synchronize()
plan.destroy()
cc.destroy_all(cs)
print("done", flush=True)
