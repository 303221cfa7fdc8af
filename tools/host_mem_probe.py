"""Host DRAM bandwidth on the GPU box vs the e2e leg's traffic: is the N = 1
end-to-end bound the PCIe link or host memory, which both arms share?
   python tools/host_mem_probe.py
Prints: CPU copy bandwidth (read + write, torch CPU copy_, all threads, pinned
and pageable buffers), and the same host bytes moved by the copy engines
(H2D alone, D2H alone, both at once) for 512 MiB per direction."""
import os
import sys
import time

import torch

MiB = 1 << 20
n = 512 * MiB


def cpu_copy(a, b, reps=5):
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        b.copy_(a)
        best = min(best, time.perf_counter() - t0)
    return 2 * a.numel() / best / 1e9


def ev_time(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


print(f"# host cores {os.cpu_count()}, torch threads {torch.get_num_threads()}")
for pinned in (False, True):
    a = torch.empty(n, dtype=torch.uint8, pin_memory=pinned).fill_(1)
    b = torch.empty(n, dtype=torch.uint8, pin_memory=pinned)
    print(f"cpu copy_ {'pinned' if pinned else 'pageable'} 512 MiB: {cpu_copy(a, b):.1f} GB/s (read + write)")
for th in (1, 4, 8, 16):
    torch.set_num_threads(th)
    a = torch.empty(n, dtype=torch.uint8).fill_(1)
    b = torch.empty(n, dtype=torch.uint8)
    print(f"cpu copy_ pageable, {th} threads: {cpu_copy(a, b):.1f} GB/s (read + write)")
torch.set_num_threads(os.cpu_count())
hi = torch.empty(n, dtype=torch.uint8, pin_memory=True).fill_(1)
ho = torch.empty(n, dtype=torch.uint8, pin_memory=True)
di = torch.empty(n, dtype=torch.uint8, device="cuda")
do = torch.empty(n, dtype=torch.uint8, device="cuda").fill_(2)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2d = ev_time(lambda: di.copy_(hi, non_blocking=True))
d2h = ev_time(lambda: ho.copy_(do, non_blocking=True))


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


bt = ev_time(both)
print(f"H2D alone {n / h2d / 1e9:.1f} GB/s, D2H alone {n / d2h / 1e9:.1f} GB/s, both at once {bt * 1e3:.2f} ms "
      f"= {2 * n / bt / 1e9:.1f} GB/s of host memory traffic")
# the e2e's host traffic while the CPU is also streaming memory (does a busy host slow the copy engines?)
import threading  # noqa: E402

stop = False


def hog():
    a = torch.empty(n, dtype=torch.uint8).fill_(1)
    b = torch.empty(n, dtype=torch.uint8)
    while not stop:
        b.copy_(a)


torch.set_num_threads(8)
th = threading.Thread(target=hog)
th.start()
time.sleep(0.5)
bt2 = ev_time(both)
stop = True
th.join()
print(f"both at once beside an 8-thread CPU copy: {bt2 * 1e3:.2f} ms = {2 * n / bt2 / 1e9:.1f} GB/s")
