"""Measured selector (cecoll_tune, csrc/tune.cpp): the reference's run_sweep +
winner_grid (sweep.cpp:71-218) executed on the machine, driving
CECOLL_IMPL_AUTO. GPU: 8 co-resident ranks in one process, and two processes
on one GPU that must install identical tables (agreed through the init
exchange). Every collective AUTO runs after tuning is checked byte for byte
(postcondition, verifier.cpp:143-169)."""
import os
import sys

import numpy as np
import pytest
import torch

import paper_2511_06605_b200 as cc

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from test_multiprocess import _init, _run2  # noqa: E402

N = 8


@pytest.fixture(scope="module")
def comms():
    cs = cc.Comm.init_all([0] * N)
    yield cs
    cc.destroy_all(cs)


def _check_auto(comms, kind, s, stream):
    in_bytes = s if kind == "allgather" else N * s
    sends = [torch.randint(0, 256, (in_bytes,), dtype=torch.uint8, device="cuda") for _ in range(N)]
    recvs = [torch.full((N * s,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(N)]
    torch.cuda.synchronize()
    fn = cc.all_gather if kind == "allgather" else cc.all_to_all
    fn(comms, sends, recvs, s, impl="auto", streams=stream)
    torch.cuda.synchronize()
    for i in range(N):
        for j in range(N):
            src = sends[i][:s] if kind == "allgather" else sends[i][j * s:(j + 1) * s]
            assert torch.equal(recvs[j][i * s:(i + 1) * s], src), (kind, s, i, j)
    return comms[0].last_plan_info()["impl"]


@pytest.mark.gpu
def test_tune_installs_a_table_that_auto_follows(comms):
    stream = torch.cuda.Stream()
    assert comms[0].tuned_table() == []
    cc.tune(comms, max_chunk=1 << 20, streams=stream)
    table = comms[0].tuned_table()
    sizes = [4096 << (2 * k) for k in range(5)]
    for kind in ("allgather", "alltoall"):
        rows = [(s, i) for k, s, i in table if k == kind]
        assert [s for s, _ in rows] == sizes, table
        for s, impl in rows:
            assert impl in cc.IMPLS_FOR[kind] + ["sm", "hybrid", "pull"], (kind, s, impl)
            assert _check_auto(comms, kind, s, stream) == impl
    # every communicator of the world sees the same table; the report holds
    # every candidate's time and the same winners
    assert all(c.tuned_table() == table for c in comms)
    rep = comms[0].tune_report()
    assert sorted(rep) == sorted((k, s) for k, s, _ in table)
    for k, s, impl in table:
        assert rep[(k, s)]["winner"] == impl
        assert rep[(k, s)]["us"][impl] > 0
        assert "sm" in rep[(k, s)]["us"] and "pcpy" in rep[(k, s)]["us"]
    # an SM budget hands AUTO back to the static policy
    comms[0].set_sm_budget(16)
    try:
        assert _check_auto(comms, "alltoall", 65536, stream) == cc.select("alltoall", 65536, N, 1, sm_budget=16)
    finally:
        comms[0].set_sm_budget(0)
    comms[0].load_tuned([])
    assert comms[0].tuned_table() == []
    assert _check_auto(comms, "alltoall", 65536, stream) == cc.select("alltoall", 65536, N, 1)


@pytest.mark.gpu
def test_loaded_table_nearest_size_on_a_log_scale(comms):
    stream = torch.cuda.Stream()
    comms[0].load_tuned([("alltoall", 4096, "b2b"), ("alltoall", 1 << 20, "pcpy"), ("allgather", 65536, "bcst")])
    try:
        assert _check_auto(comms, "alltoall", 4096, stream) == "b2b"
        assert _check_auto(comms, "alltoall", 16384, stream) == "b2b"      # 2^28 < 4 KiB * 1 MiB
        assert _check_auto(comms, "alltoall", 65536, stream) == "pcpy"     # the geometric midpoint goes up
        assert _check_auto(comms, "alltoall", 4 << 20, stream) == "pcpy"   # above the table: its last entry
        assert _check_auto(comms, "allgather", 4096, stream) == "bcst"     # below: its first entry
        # in-place all-to-all stays swap (a different call)
        sends = [torch.randint(0, 256, (N * 4096,), dtype=torch.uint8, device="cuda") for _ in range(N)]
        want = [t.clone() for t in sends]
        torch.cuda.synchronize()
        cc.all_to_all(comms, sends, sends, 4096, impl="auto", streams=stream)
        torch.cuda.synchronize()
        assert comms[0].last_plan_info()["impl"] == "swap"
        assert all(torch.equal(sends[j][i * 4096:(i + 1) * 4096], want[i][j * 4096:(j + 1) * 4096])
                   for i in range(N) for j in range(N))
    finally:
        comms[0].load_tuned([])


@pytest.mark.gpu
@pytest.mark.parametrize("text", ["alltoall 4096 bcst\n", "reduce 4096 sm\n", "alltoall -4 sm\n", "alltoall x sm\n",
                                  "alltoall 4096 nope\n"])
def test_bad_tables_are_rejected(comms, text):
    with pytest.raises(cc.CecollError):
        comms[0].load_tuned(text)
    assert comms[0].tuned_table() == []


def _tune_worker(rank, world, port, out):
    import traceback

    try:
        dist = _init(rank, world, port)
        import paper_2511_06605_b200 as cc  # noqa: F811

        nranks, nlocal = 4, 2
        first = rank * nlocal
        comms = cc.Comm.init_ranks(nranks, first, nlocal, 0, cc.torch_exchange())
        cc.tune(comms, max_chunk=65536, streams=torch.cuda.current_stream())
        table = comms[0].tuned_table()
        # AUTO after tuning, on registered windows, checked against the sources
        s = 16384
        wins = [c.mem_alloc(2 * nranks * s) for c in comms]
        g = torch.Generator().manual_seed(5)
        host = [torch.randint(0, 256, (nranks * s,), dtype=torch.uint8, generator=g) for _ in range(nranks)]
        sends, recvs = [], []
        for k, w in enumerate(wins):
            w[: nranks * s].copy_(host[first + k])
            w[nranks * s:].fill_(0xA5)
            sends.append(w[: nranks * s])
            recvs.append(w[nranks * s:])
        torch.cuda.synchronize()
        dist.barrier()
        cc.all_to_all(comms, sends, recvs, s, impl="auto", streams=torch.cuda.current_stream())
        torch.cuda.synchronize()
        dist.barrier()
        ok = all(np.array_equal(recvs[k][i * s:(i + 1) * s].cpu().numpy(), host[i][(first + k) * s:(first + k + 1) * s].numpy())
                 for k in range(nlocal) for i in range(nranks))
        impl = comms[0].last_plan_info()["impl"]
        del sends, recvs
        for c, w in zip(comms, wins):
            c.mem_free(w)
        out.put((rank, table, ok, impl))
        for c in comms:
            c.destroy()
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        out.put((rank, traceback.format_exc(), None, None))


@pytest.mark.gpu
def test_two_processes_install_the_same_table():
    res = sorted(_run2(_tune_worker), key=lambda r: r[0])
    for rank, table, ok, impl in res:
        assert isinstance(table, list), table
        assert len(table) == 2 * 3, table  # 4, 16, 64 KiB for both collectives
        assert ok, (rank, impl)
    assert res[0][1] == res[1][1]
    assert res[0][3] == res[1][3] == dict((s, i) for k, s, i in res[0][1] if k == "alltoall")[16384]
