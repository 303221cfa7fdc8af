"""L2 / DRAM disturbance of a concurrent GEMM by a collective (north star:
"L2 hit-rate disturbance to the concurrent GEMM"; BASELINE configs[4]).

ncu's kernel replay serialises kernels, so the interference is measured with
range replay: each phase below is one cudaProfilerStart/Stop range whose
kernels run concurrently as in the application, and ncu reports DRAM bytes
and the L2 hit rate over the whole range. The collective's own DRAM bytes
come from its range alone; the GEMM's extra DRAM traffic caused by the
collective is (together) - (GEMM alone) - (collective alone).

   ncu --replay-mode range --metrics dram__bytes_read.sum,dram__bytes_write.sum,\\
       lts__t_sector_hit_rate.pct,gpu__time_duration.sum --csv python tools/l2_disturb.py [impl] [chunk_MiB]
(without ncu the script just runs the phases and prints their device times)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_06605_b200 as cc  # noqa: E402

impl = sys.argv[1] if len(sys.argv) > 1 else "sm"
s = (int(sys.argv[2]) if len(sys.argv) > 2 else 64) << 20
budget = int(sys.argv[3]) if len(sys.argv) > 3 else 0
host = len(sys.argv) > 4 and sys.argv[4] == "host"  # recv buffers in pinned host memory (copy engines over PCIe)
n = 8
N = 8192
G = 8  # GEMMs per phase
C = 2  # collectives per phase

comms = cc.Comm.init_all([0] * n)
if budget:
    comms[0].set_sm_budget(budget)
a = torch.randn(N, N, device="cuda", dtype=torch.bfloat16)
b = torch.randn(N, N, device="cuda", dtype=torch.bfloat16)
c = torch.empty(N, N, device="cuda", dtype=torch.bfloat16)
sends = [torch.randint(0, 256, (s,), dtype=torch.uint8, device="cuda") for _ in range(n)]
recvs = [torch.empty(n * s, dtype=torch.uint8, pin_memory=True) if host else
         torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
gs, cs = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()


def gemms():
    with torch.cuda.stream(gs):
        for _ in range(G):
            torch.matmul(a, b, out=c)


def colls():
    for _ in range(C):
        cc.all_gather(comms, sends, recvs, s, impl=impl, streams=cs)


# a phase needs at least one kernel in its range: a tiny marker kernel per phase
marker = torch.zeros(1, device="cuda")


# warm up (plans built, graphs recorded, cuBLAS heuristics) outside the ranges
for _ in range(2):
    gemms()
    colls()
torch.cuda.synchronize()


def phase(name, fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    e0.record()
    marker.add_(1)
    fn()
    gs.synchronize()
    cs.synchronize()
    e1.record()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"phase {name}: {e0.elapsed_time(e1):.3f} ms", flush=True)


phase("gemm", gemms)
phase("collective", colls)
phase("together", lambda: (gemms(), colls()))
cc.destroy_all(comms)
