"""One process per GPU (comm_init_rank / comm_init_ranks).

CPU: the init exchange over torch.distributed (gloo, world size 2) — blob
marshaling through the C callback and validation of the processes' rank
ranges — runs without a GPU (cecoll_exchange_check).
GPU: two processes on cuda:0 owning two ranks each (4 ranks), flag pages and
symmetric windows mapped through CUDA IPC across the processes, every
implementation checked against the oracle.
"""
import os
import socket
import traceback

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    return dist


def _exchange_worker(rank, world, port, out):
    try:
        dist = _init(rank, world, port)
        import paper_2511_06605_b200 as cc

        ex = cc.torch_exchange()
        devs = cc.exchange_check(4, rank * 2, 2, 10 + rank, ex)
        # Overlapping ranges are rejected on every process (no hang: the
        # exchange completes, validation fails everywhere).
        try:
            cc.exchange_check(4, 0, 2, 0, ex)
            bad = "accepted"
        except cc.InvalidArgument as e:
            bad = str(e)
        # Uneven ownership is rejected before the exchange.
        try:
            cc.exchange_check(4, 0, 3, 0, ex)
            uneven = "accepted"
        except cc.InvalidArgument:
            uneven = "rejected"
        out.put((rank, devs, bad, uneven))
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        out.put((rank, traceback.format_exc(), None, None))


def test_exchange_over_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, devs, bad, uneven in res:
        assert devs == [10, 10, 11, 11], devs
        assert "owned by two processes" in bad or "owned by no process" in bad, bad
        assert uneven == "rejected"


def _gpu_worker(rank, world, port, out, force_remote=False):
    try:
        if force_remote:  # every cross-process signal down the other-device path (signal kernels)
            os.environ["CECOLL_FORCE_REMOTE_SIGNALS"] = "1"
        dist = _init(rank, world, port)
        import numpy as np
        import torch

        import paper_2511_06605_b200 as cc
        from oracle import oracle as ora

        nranks, nlocal = 4, 2
        first = rank * nlocal
        comms = cc.Comm.init_ranks(nranks, first, nlocal, 0, cc.torch_exchange())
        O = ora.Oracle()
        s = 65536 + 64
        results = []
        for kind, impls in (("alltoall", ["sm", "pcpy", "b2b", "prelaunch_pcpy", "swap", "hybrid", "pull"]),
                            ("allgather", ["sm", "pcpy", "bcst", "prelaunch_b2b", "pull"])):
            in_bytes = s if kind == "allgather" else nranks * s
            # One symmetric window per rank: [send | recv].
            wins = [torch.full((in_bytes + nranks * s,), 0xA5, dtype=torch.uint8, device="cuda") for _ in comms]
            for c, w in zip(comms, wins):
                c.register(w)
            for it, impl in enumerate(impls):
                seed = 40 + it
                host_all = [ora.splitmix_pattern(in_bytes, r, seed) for r in range(nranks)]
                sends, recvs = [], []
                for k, w in enumerate(wins):
                    w[:in_bytes].copy_(torch.from_numpy(host_all[first + k]))
                    w[in_bytes:].fill_(0xA5)
                    sends.append(w[:in_bytes])
                    recvs.append(sends[-1] if impl.endswith("swap") else w[in_bytes:])
                torch.cuda.synchronize()
                dist.barrier()
                fn = cc.all_gather if kind == "allgather" else cc.all_to_all
                fn(comms, sends, recvs, s, impl=impl, streams=torch.cuda.current_stream())
                torch.cuda.synchronize()
                dist.barrier()
                mine = [t.cpu().numpy() for t in recvs]
                # Check this process's ranks against the oracle's full result.
                full = [np.zeros(nranks * s, np.uint8) for _ in range(nranks)]
                O.reference_result(kind, s, nranks, host_all, full)
                ok = all(np.array_equal(mine[k], full[first + k]) for k in range(nlocal))
                results.append((kind, impl, ok))
        # reduce-scatter (SM path: every rank reads its chunk from every peer's
        # registered send window), bf16 sum, against the oracle's rank-order fold
        count = 4096 + 8
        ins = [ora.splitmix_pattern(nranks * count * 2, r, 90) for r in range(nranks)]
        for b in ins:  # finite bf16 values: clear the exponent MSB
            b.view(np.uint16)[:] &= np.uint16(0xBFFF)
        want = O.reduce_scatter(1, 0, count, ins)
        wins = [torch.empty(nranks * count * 2, dtype=torch.uint8, device="cuda") for _ in comms]
        for c, w in zip(comms, wins):
            c.register(w)
        for k, w in enumerate(wins):
            w.copy_(torch.from_numpy(ins[first + k]))
        recvs = [torch.full((count * 2,), 0xA5, dtype=torch.uint8, device="cuda") for _ in comms]
        torch.cuda.synchronize()
        dist.barrier()
        for _ in range(2):
            cc.reduce_scatter(comms, wins, recvs, count, dtype="bf16", op="sum", impl="sm",
                              streams=torch.cuda.current_stream())
        torch.cuda.synchronize()
        dist.barrier()
        results.append(("reduce_scatter", "sm",
                        all(np.array_equal(recvs[k].cpu().numpy(), want[first + k]) for k in range(nlocal))))
        out.put((rank, results))
        torch.cuda.synchronize()
        for c in comms:
            c.destroy()
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        out.put((rank, traceback.format_exc()))


def _alloc_worker(rank, world, port, out):
    """Windows from cecoll_mem_alloc (auto-registered), freed and allocated
    again between collectives."""
    try:
        dist = _init(rank, world, port)
        import numpy as np
        import torch

        import paper_2511_06605_b200 as cc
        from oracle import oracle as ora

        nranks, nlocal = 4, 2
        first = rank * nlocal
        comms = cc.Comm.init_ranks(nranks, first, nlocal, 0, cc.torch_exchange())
        O = ora.Oracle()
        s = 3 * 65536 + 48
        results = []
        for cycle, impl in enumerate(["sm", "pcpy", "b2b", "sm"]):
            wins = [c.mem_alloc(2 * nranks * s) for c in comms]
            host_all = [ora.splitmix_pattern(nranks * s, r, 70 + cycle) for r in range(nranks)]
            sends, recvs = [], []
            for k, w in enumerate(wins):
                w[: nranks * s].copy_(torch.from_numpy(host_all[first + k]))
                w[nranks * s:].fill_(0xA5)
                sends.append(w[: nranks * s])
                recvs.append(w[nranks * s: 2 * nranks * s])
            torch.cuda.synchronize()
            dist.barrier()
            cc.all_to_all(comms, sends, recvs, s, impl=impl, streams=torch.cuda.current_stream())
            torch.cuda.synchronize()
            dist.barrier()
            full = [np.zeros(nranks * s, np.uint8) for _ in range(nranks)]
            O.reference_result("alltoall", s, nranks, host_all, full)
            ok = all(np.array_equal(recvs[k].cpu().numpy(), full[first + k]) for k in range(nlocal))
            results.append((cycle, impl, ok))
            del sends, recvs
            for c, w in zip(comms, wins):
                c.mem_free(w)
        # Freeing twice (or a foreign pointer) is an error, not a crash.
        try:
            comms[0].mem_free(wins[0])
            results.append(("double free", "", False))
        except cc.CecollError:
            results.append(("double free", "", True))
        out.put((rank, results))
        for c in comms:
            c.destroy()
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        out.put((rank, traceback.format_exc()))


def _run2(target):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return res


@pytest.mark.gpu
def test_two_processes_mem_alloc_windows():
    for rank, results in _run2(_alloc_worker):
        assert isinstance(results, list), results
        assert len(results) == 5
        assert all(r[2] for r in results), (rank, results)


@pytest.mark.gpu
@pytest.mark.parametrize("force_remote", [False, True])
def test_two_processes_share_one_gpu_through_ipc(force_remote):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q, force_remote)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, results in res:
        assert isinstance(results, list), results
        bad = [r for r in results if not r[2]]
        assert not bad, (rank, bad)
        assert len(results) == 13


def _asymmetric_failure_worker(rank, world, port, out):
    """Rank 0 registers a host pointer (its local step fails before the
    exchange); rank 1 a valid device window. Collective calls fail
    collectively: both must raise, neither may hang in the exchange."""
    try:
        dist = _init(rank, world, port)
        import torch

        import paper_2511_06605_b200 as cc

        comms = cc.Comm.init_ranks(2, rank, 1, 0, cc.torch_exchange())
        buf = torch.empty(1 << 20, dtype=torch.uint8) if rank == 0 else \
            torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
        try:
            comms[0].register(buf)
            res = "registered"
        except cc.CecollError as e:
            res = "error: " + str(e)[:80]
        # the communicator stays usable for a good registration afterwards
        good = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
        comms[0].register(good)
        out.put((rank, res))
        torch.cuda.synchronize()
        comms[0].destroy()
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        out.put((rank, traceback.format_exc()))


@pytest.mark.gpu
@pytest.mark.timeout(240)
def test_registration_fails_on_every_process_together():
    res = dict(_run2(_asymmetric_failure_worker))
    assert res[0].startswith("error"), res
    assert res[1].startswith("error") and "another process" in res[1], res


def _stress_worker(rank, world, port, out, force_remote):
    """Back-to-back collectives across two processes without host
    synchronisation (DESIGN.md §3.2 across CUDA IPC): per local rank its own
    stream; per iteration a random spin, the input reload, the collective, a
    random spin and the copy-out; the processes meet only at the start."""
    try:
        if force_remote:
            os.environ["CECOLL_FORCE_REMOTE_SIGNALS"] = "1"
        dist = _init(rank, world, port)
        import random

        import numpy as np
        import torch

        import paper_2511_06605_b200 as cc
        from oracle import oracle as ora

        nranks, nlocal, iters = 4, 2, 10
        first = rank * nlocal
        comms = cc.Comm.init_ranks(nranks, first, nlocal, 0, cc.torch_exchange())
        s = 24576 + 32
        streams = [torch.cuda.Stream() for _ in range(nlocal)]
        wins = [torch.zeros(2 * nranks * s, dtype=torch.uint8, device="cuda") for _ in comms]
        for c, w in zip(comms, wins):
            c.register(w)
        results = []
        for impl in ["sm", "pcpy", "b2b", "swap", "pull", "hybrid", "prelaunch_pcpy", "prelaunch_b2b"]:
            rng = random.Random(f"{impl}-{rank}")
            in_place = impl.endswith("swap")
            hosts = [[ora.splitmix_pattern(nranks * s, r, 7000 + it) for r in range(nranks)] for it in range(iters)]
            inputs = [[torch.from_numpy(hosts[it][first + k]).cuda() for k in range(nlocal)] for it in range(iters)]
            outs = [[torch.empty(nranks * s, dtype=torch.uint8, device="cuda") for _ in range(nlocal)]
                    for _ in range(iters)]
            sends = [w[:nranks * s] for w in wins]
            recvs = sends if in_place else [w[nranks * s:] for w in wins]
            torch.cuda.synchronize()
            dist.barrier()
            for it in range(iters):
                for k, st in enumerate(streams):
                    with torch.cuda.stream(st):
                        if rng.random() < 0.5:
                            torch.cuda._sleep(rng.randint(1000, 100000))
                        sends[k].copy_(inputs[it][k])
                cc.all_to_all(comms, sends, recvs, s, impl=impl, streams=streams)
                for k, st in enumerate(streams):
                    with torch.cuda.stream(st):
                        if rng.random() < 0.5:
                            torch.cuda._sleep(rng.randint(1000, 100000))
                        outs[it][k].copy_(recvs[k])
            torch.cuda.synchronize()
            bad = []
            for it in range(iters):
                for k in range(nlocal):
                    r = first + k
                    want = np.concatenate([hosts[it][j][r * s:(r + 1) * s] for j in range(nranks)])
                    if not np.array_equal(outs[it][k].cpu().numpy(), want):
                        bad.append((it, r))
            results.append((impl, bad))
            dist.barrier()
        err = comms[0].async_error()
        results.append(("async_error", [] if err is None else [str(err)]))
        out.put((rank, results))
        torch.cuda.synchronize()
        for c in comms:
            c.destroy()
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        out.put((rank, traceback.format_exc()))


@pytest.mark.gpu
@pytest.mark.timeout(400)
@pytest.mark.parametrize("force_remote", [False, True])
def test_two_processes_back_to_back_without_host_sync(force_remote):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stress_worker, args=(r, 2, port, q, force_remote)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=360) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, results in res:
        assert isinstance(results, list), results
        assert len(results) == 9
        bad = [(impl, b) for impl, b in results if b]
        assert not bad, (rank, bad)
