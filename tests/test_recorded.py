"""Recorded command lists: non-prelaunch plans replay as one CUDA graph per
unit from their second launch (include/cecoll.h). Every
replay is checked against the oracle; the counters show that the replays
happened. Also: a caller capturing an eager collective into its own CUDA
graph (the library then submits into the capture)."""
import numpy as np
import pytest

import paper_2511_06605_b200 as cc
from oracle import oracle as ora

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

IMPLS = {"allgather": ["sm", "pcpy", "b2b", "bcst", "hybrid", "pull"],
         "alltoall": ["sm", "pcpy", "b2b", "swap", "hybrid", "pull"]}
CASES = [(k, i) for k in IMPLS for i in IMPLS[k]]


def _bufs(kind, n, s, impl):
    in_bytes = s if kind == "allgather" else n * s
    sends = [torch.empty(in_bytes, dtype=torch.uint8, device="cuda") for _ in range(n)]
    recvs = sends if impl.endswith("swap") else [torch.empty(n * s, dtype=torch.uint8, device="cuda")
                                                 for _ in range(n)]
    return in_bytes, sends, recvs


def _load(sends, recvs, in_bytes, n, seed, in_place):
    host = [ora.splitmix_pattern(in_bytes, r, seed) for r in range(n)]
    for t, h in zip(sends, host):
        t.copy_(torch.from_numpy(h))
    if not in_place:
        for t in recvs:
            t.fill_(0xA5)
    return host


@pytest.mark.parametrize("n", [4, 8])
@pytest.mark.parametrize("kind,impl", CASES)
def test_eager_calls_replay_recorded_lists(kind, impl, n):
    s = 8192 + 16
    comms = cc.Comm.init_all([0] * n)
    O = ora.Oracle()
    st = torch.cuda.Stream()
    in_place = impl.endswith("swap")
    try:
        in_bytes, sends, recvs = _bufs(kind, n, s, impl)
        fn = cc.all_gather if kind == "allgather" else cc.all_to_all
        c0 = comms[0].counters()
        for it in range(5):
            host = _load(sends, recvs, in_bytes, n, 300 + it, in_place)
            torch.cuda.synchronize()
            fn(comms, sends, recvs, s, impl=impl, streams=st)
            st.synchronize()
            res = [t.cpu().numpy() for t in recvs]
            assert O.check(kind, s, n, in_place, host, res) == -1, (kind, impl, it)
        c1 = comms[0].counters()
        # first call eager, calls 2..5 replay one recorded graph (one unit);
        # the one-unit SM path too (a one-node graph)
        assert c1["recorded_launches"] - c0["recorded_launches"] == 4
        assert c1["collectives"] - c0["collectives"] == 5
    finally:
        torch.cuda.synchronize()
        cc.destroy_all(comms)


@pytest.mark.parametrize("kind,impl", [("alltoall", "pcpy"), ("alltoall", "sm"), ("allgather", "b2b")])
def test_explicit_plan_replays_and_rebinds_streams(kind, impl):
    n, s = 4, 65536 + 48
    comms = cc.Comm.init_all([0] * n)
    O = ora.Oracle()
    try:
        in_bytes, sends, recvs = _bufs(kind, n, s, impl)
        plan = cc.Plan(comms, kind, sends, recvs, s, impl=impl)
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        for it in range(6):
            host = _load(sends, recvs, in_bytes, n, 400 + it, False)
            torch.cuda.synchronize()
            st = streams[it % 2]  # a replay may run on another stream than the recording
            plan.launch(st)
            st.synchronize()
            res = [t.cpu().numpy() for t in recvs]
            assert O.check(kind, s, n, False, host, res) == -1, (kind, impl, it)
        plan.destroy()
    finally:
        torch.cuda.synchronize()
        cc.destroy_all(comms)


def test_per_rank_streams_stay_eager():
    # Several units on one device keep the phase-ordered submission.
    n, s = 4, 4096
    comms = cc.Comm.init_all([0] * n)
    try:
        sends = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
        recvs = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
        streams = [torch.cuda.Stream() for _ in range(n)]
        c0 = comms[0].counters()
        for _ in range(3):
            cc.all_to_all(comms, sends, recvs, s, impl="pcpy", streams=streams)
        torch.cuda.synchronize()
        assert comms[0].counters()["recorded_launches"] == c0["recorded_launches"]
    finally:
        cc.destroy_all(comms)


@pytest.mark.parametrize("impl", ["sm", "pcpy", "b2b"])
def test_caller_captures_eager_collective(impl):
    n, s = 4, 32768
    comms = cc.Comm.init_all([0] * n)
    O = ora.Oracle()
    try:
        in_bytes, sends, recvs = _bufs("alltoall", n, s, impl)
        st = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        _load(sends, recvs, in_bytes, n, 1, False)
        # warm-up outside the capture: the plan (device tables) is built here
        cc.all_to_all(comms, sends, recvs, s, impl=impl, streams=st)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            cc.all_to_all(comms, sends, recvs, s, impl=impl, streams=st)
        for it in range(3):
            host = _load(sends, recvs, in_bytes, n, 500 + it, False)
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            res = [t.cpu().numpy() for t in recvs]
            assert O.check("alltoall", s, n, False, host, res) == -1, (impl, it)
        del g
    finally:
        torch.cuda.synchronize()
        cc.destroy_all(comms)


@pytest.mark.timeout(180)
@pytest.mark.parametrize("impl", ["sm", "prelaunch_b2b", "prelaunch_pcpy"])
@pytest.mark.parametrize("s", [256 << 10, 1 << 20])
def test_many_units_back_to_back(impl, s):
    """Eight units on one GPU (one stream per rank: flags between all of
    them), many collectives in flight. Regression for a resource deadlock: a
    full-grid mover spinning on flags inside an armed prelaunch graph could
    hold every SM that a caller-stream poll kernel needed;
    the SM path's fused kernel is safe by stream order (§3.5)."""
    n = 8
    comms = cc.Comm.init_all([0] * n)
    O = ora.Oracle()
    try:
        in_bytes, sends, recvs = _bufs("allgather", n, s, impl)
        host = _load(sends, recvs, in_bytes, n, 600, False)
        streams = [torch.cuda.Stream() for _ in range(n)]
        torch.cuda.synchronize()
        for _ in range(30):
            cc.all_gather(comms, sends, recvs, s, impl=impl, streams=streams)
        torch.cuda.synchronize()
        res = [t.cpu().numpy() for t in recvs]
        assert O.check("allgather", s, n, False, host, res) == -1
    finally:
        torch.cuda.synchronize()
        cc.destroy_all(comms)


@pytest.mark.parametrize("pct", [0, 25, 50, 100])
@pytest.mark.parametrize("kind", ["allgather", "alltoall"])
@pytest.mark.parametrize("stream_mode", ["shared", "per_rank"])
def test_hybrid_split_against_oracle(kind, pct, stream_mode, monkeypatch):
    """Every chunk split between a copy-engine lane and the SM mover at the
    given SM share (odd chunk size: misaligned split points), explicit plans
    launched repeatedly, with one stream or one stream per rank (flags)."""
    monkeypatch.setenv("CECOLL_HYBRID_SM_PCT", str(pct))
    n, s = 4, 3 * 65536 + 40
    comms = cc.Comm.init_all([0] * n)
    O = ora.Oracle()
    try:
        in_bytes, sends, recvs = _bufs(kind, n, s, "hybrid")
        plan = cc.Plan(comms, kind, sends, recvs, s, impl="hybrid")
        streams = torch.cuda.Stream() if stream_mode == "shared" else [torch.cuda.Stream() for _ in range(n)]
        for it in range(3):
            host = _load(sends, recvs, in_bytes, n, 700 + it, False)
            torch.cuda.synchronize()
            plan.launch(streams)
            torch.cuda.synchronize()
            res = [t.cpu().numpy() for t in recvs]
            assert O.check(kind, s, n, False, host, res) == -1, (kind, pct, it)
        plan.destroy()
    finally:
        torch.cuda.synchronize()
        cc.destroy_all(comms)


@pytest.mark.parametrize("impl", ["pcpy", "b2b", "bcst", "swap", "sm", "hybrid", "pull", "prelaunch_pcpy",
                                  "prelaunch_b2b", "prelaunch_swap"])
def test_other_device_signal_path_on_one_gpu(impl, monkeypatch):
    """CECOLL_FORCE_REMOTE_SIGNALS=1 sends every cross-unit signal down the
    other-device path (signal kernels with st.release.sys; the lanes' done
    signals as one kernel per unit after the join) — the path a multi-GPU
    node takes — with one stream per rank so every transfer is flagged."""
    monkeypatch.setenv("CECOLL_FORCE_REMOTE_SIGNALS", "1")
    n, s = 4, 65536 + 32
    kinds = ["allgather"] if impl.endswith("bcst") else ["alltoall"] if impl.endswith("swap") else \
        ["allgather", "alltoall"]
    comms = cc.Comm.init_all([0] * n)
    O = ora.Oracle()
    try:
        for kind in kinds:
            in_place = impl.endswith("swap")
            in_bytes, sends, recvs = _bufs(kind, n, s, impl)
            streams = [torch.cuda.Stream() for _ in range(n)]
            fn = cc.all_gather if kind == "allgather" else cc.all_to_all
            for it in range(4):
                host = _load(sends, recvs, in_bytes, n, 800 + it, in_place)
                torch.cuda.synchronize()
                fn(comms, sends, recvs, s, impl=impl, streams=streams)
                torch.cuda.synchronize()
                res = [t.cpu().numpy() for t in recvs]
                assert O.check(kind, s, n, in_place, host, res) == -1, (kind, impl, it)
    finally:
        torch.cuda.synchronize()
        cc.destroy_all(comms)


@pytest.mark.timeout(300)
def test_plan_cache_eviction_with_recorded_graphs():
    """More distinct calls than the eager-call plan cache holds (64): every
    plan is recorded (second call) and the oldest are evicted with their
    graphs; results stay exact, including for sizes evicted and re-created."""
    n = 4
    comms = cc.Comm.init_all([0] * n)
    O = ora.Oracle()
    st = torch.cuda.Stream()
    try:
        sizes = [4096 + 16 * k for k in range(70)] + [4096, 4096 + 16]  # the last two were evicted
        sends = [torch.empty(n * sizes[-3], dtype=torch.uint8, device="cuda") for _ in range(n)]
        recvs = [torch.empty(n * sizes[-3], dtype=torch.uint8, device="cuda") for _ in range(n)]
        for i, s in enumerate(sizes):
            snd = [t[:n * s] for t in sends]
            rcv = [t[:n * s] for t in recvs]
            host = _load(snd, rcv, n * s, n, 900 + i, False)
            torch.cuda.synchronize()
            for _ in range(2):  # eager, then recorded replay
                cc.all_to_all(comms, snd, rcv, s, impl="pcpy", streams=st)
            st.synchronize()
            if i % 7 == 0 or i >= len(sizes) - 3:
                res = [t.cpu().numpy() for t in rcv]
                assert O.check("alltoall", s, n, False, host, res) == -1, (i, s)
    finally:
        torch.cuda.synchronize()
        cc.destroy_all(comms)


@pytest.mark.timeout(180)
@pytest.mark.parametrize("impl", ["sm", "pcpy", "b2b", "swap", "pull", "hybrid"])
def test_caller_graph_with_many_collectives_on_rank_streams(impl):
    """A caller's own CUDA graph holding K collectives on per-rank streams
    (forked once from the capture stream, joined once): input reload,
    collective, copy-out per iteration, flags between the four units inside
    the graph; replayed twice back to back, three times (tools/caller_graph_probe.py)."""
    n, s, K = 4, 16384 + 16, 4
    comms = cc.Comm.init_all([0] * n)
    try:
        in_place = impl.endswith("swap")
        hosts = [[ora.splitmix_pattern(n * s, r, 900 + it) for r in range(n)] for it in range(K)]
        inputs = [[torch.from_numpy(hosts[it][r]).cuda() for r in range(n)] for it in range(K)]
        sends = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
        recvs = sends if in_place else [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
        outs = [[torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)] for _ in range(K)]
        main = torch.cuda.Stream()
        rs = [torch.cuda.Stream() for _ in range(n)]

        def body():
            for r in range(n):
                rs[r].wait_stream(main)
            for it in range(K):
                for r in range(n):
                    with torch.cuda.stream(rs[r]):
                        sends[r].copy_(inputs[it][r])
                cc.all_to_all(comms, sends, recvs, s, impl=impl, streams=rs)
                for r in range(n):
                    with torch.cuda.stream(rs[r]):
                        outs[it][r].copy_(recvs[r])
            for r in range(n):
                main.wait_stream(rs[r])

        with torch.cuda.stream(main):
            body()  # eager warm-up: the plan is built outside the capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=main):
            body()
        for rep in range(3):
            for it in range(K):
                for t in outs[it]:
                    t.zero_()
            torch.cuda.synchronize()
            g.replay()
            g.replay()
            torch.cuda.synchronize()
            for it in range(K):
                for r in range(n):
                    want = np.concatenate([hosts[it][j][r * s:(r + 1) * s] for j in range(n)])
                    assert np.array_equal(outs[it][r].cpu().numpy(), want), (impl, rep, it, r)
        assert comms[0].async_error() is None
        del g
    finally:
        torch.cuda.synchronize()
        cc.destroy_all(comms)
