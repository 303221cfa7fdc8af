"""Threading contract of include/cecoll.h: different worlds may be driven
from different host threads at the same time (ctypes releases the GIL, so
the library really runs concurrently here). Two threads each own a world of
four co-resident ranks on cuda:0 and their own stream, and run collectives of
every implementation family back to back; every result is checked against
the reference byte layout (compiler.cpp:115-126) restated in torch."""
import threading

import pytest

import paper_2511_06605_b200 as cc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

N = 4
S = 64 << 10
IMPLS = ["pcpy", "b2b", "sm", "prelaunch_pcpy", "hybrid", "pull"]


def expected(kind, sends):
    if kind == "allgather":
        full = torch.cat(sends)
        return [full for _ in sends]
    return [torch.cat([sends[j][r * S:(r + 1) * S] for j in range(N)]) for r in range(N)]


def worker(tid, iters, errors, worlds):
    try:
        comms = cc.Comm.init_all([0] * N)
        worlds.append(comms)
        stream = torch.cuda.Stream()
        g = torch.Generator(device="cuda")
        g.manual_seed(1000 + tid)
        with torch.cuda.stream(stream):
            for it in range(iters):
                impl = IMPLS[(it + tid) % len(IMPLS)]
                kind = "allgather" if it % 2 else "alltoall"
                in_bytes = S if kind == "allgather" else N * S
                sends = [torch.randint(0, 256, (in_bytes,), dtype=torch.uint8, device="cuda", generator=g)
                         for _ in range(N)]
                recvs = [torch.full((N * S,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(N)]
                fn = cc.all_gather if kind == "allgather" else cc.all_to_all
                fn(comms, sends, recvs, S, impl=impl, streams=stream)
                for r, (got, want) in enumerate(zip(recvs, expected(kind, sends))):
                    if not torch.equal(got, want):
                        errors.append((tid, it, impl, kind, r))
                        return
        stream.synchronize()
    except Exception as e:  # reported by the main thread
        errors.append((tid, repr(e)))


def test_two_worlds_from_two_threads():
    # torch's own kernels loaded once up front: the test is about the
    # library's threads, not about lazy module loading
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    x = torch.randint(0, 256, (N * S,), dtype=torch.uint8, device="cuda", generator=g)
    y = torch.full((N * S,), 0xA5, dtype=torch.uint8, device="cuda")
    torch.equal(torch.cat([x[:S], y[:S]]), torch.cat([y[:S], x[:S]]))  # loads cat, eq, all
    torch.cuda.synchronize()
    errors, worlds = [], []
    threads = [threading.Thread(target=worker, args=(t, 48, errors, worlds)) for t in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=240)
    assert not any(t.is_alive() for t in threads), "a worker thread hung"
    # Destroyed here, not in the workers: destroy synchronises the device,
    # which must not overlap another thread's collectives (include/cecoll.h).
    for comms in worlds:
        cc.destroy_all(comms)
    assert errors == []

