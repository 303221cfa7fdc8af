"""Hardware timelines in the reference's trace-event format (sim.cpp:523-544):
well-formed B/E pairs per (pid, tid), one span per command the program holds,
results still bit-exact while tracing."""
import collections
import ctypes

import numpy as np
import pytest

import paper_2511_06605_b200 as cc
from oracle import oracle as ora

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

N, S = 4, 3 * 65536 + 16


@pytest.fixture(scope="module")
def comms():
    cs = cc.Comm.init_all([0] * N)
    yield cs
    cc.destroy_all(cs)


def spans(events):
    """Pairs B/E per (name, pid, tid) in order; asserts the nesting is sane."""
    open_ = collections.defaultdict(list)
    out = []
    for e in events:
        assert set(e) == {"name", "ph", "ts", "pid", "tid"}, e
        key = (e["name"], e["pid"], e["tid"])
        if e["ph"] == "B":
            open_[key].append(e["ts"])
        else:
            assert e["ph"] == "E" and open_[key], e
            b = open_[key].pop()
            assert e["ts"] >= b
            out.append((e["name"], e["pid"], e["tid"], b, e["ts"]))
    assert not any(open_.values())
    return out


def traced_call(comms, kind, impl, seed):
    in_bytes = S if kind == "allgather" else N * S
    host = [ora.splitmix_pattern(in_bytes, r, seed) for r in range(N)]
    sends = [torch.from_numpy(h).cuda() for h in host]
    recvs = sends if impl.endswith("swap") else [
        torch.full((N * S,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(N)]
    streams = [torch.cuda.Stream() for _ in range(N)]
    for st in streams:
        st.wait_stream(torch.cuda.current_stream())
    torch.cuda.synchronize()
    fn = cc.all_gather if kind == "allgather" else cc.all_to_all
    fn(comms, sends, recvs, S, impl=impl, streams=streams)  # plan built outside the trace
    torch.cuda.synchronize()
    with cc.Trace(comms[0]) as t:
        fn(comms, sends if not impl.endswith("swap") else recvs, recvs, S, impl=impl, streams=streams)
        torch.cuda.synchronize()
    res = [r.cpu().numpy() for r in recvs]
    if impl.endswith("swap"):  # applied twice: an involution
        assert all(np.array_equal(a, b) for a, b in zip(res, host))
    else:
        want = [np.zeros(N * S, np.uint8) for _ in range(N)]
        ora.Oracle().reference_result(kind, S, N, host, want)
        assert all(np.array_equal(a, b) for a, b in zip(res, want))
    return spans(t.events)


def count(sp, name, lanes_only=True):
    return sum(1 for n, pid, tid, _, _ in sp if n == name and (tid >= 0 or not lanes_only))


def test_pcpy_one_copy_per_lane(comms):
    sp = traced_call(comms, "alltoall", "pcpy", 3)
    assert count(sp, "copy:copy") == N * (N - 1)
    assert count(sp, "poll:poll") == N * (N - 1)  # every lane waits for its destination's rdy
    assert count(sp, "sync:signal") == N * (N - 1)
    assert sum(1 for n, *_ in sp if n == "control") >= N * (N - 1)
    assert {pid for _, pid, tid, _, _ in sp if pid >= 0} == set(range(N))


def test_b2b_copies_back_to_back(comms):
    sp = traced_call(comms, "allgather", "b2b", 4)
    per_lane = collections.defaultdict(list)
    for n, pid, tid, b, e in sp:
        if n == "copy:copy" and tid >= 0:
            per_lane[(pid, tid)].append((b, e))
    assert len(per_lane) == N and all(len(v) == N - 1 for v in per_lane.values())
    for v in per_lane.values():  # one engine queue: copies never overlap
        v.sort()
        assert all(v[i][1] <= v[i + 1][0] + 1e-3 for i in range(len(v) - 1))


@pytest.mark.parametrize("kind,impl,name", [("allgather", "bcst", "copy:broadcast"),
                                            ("alltoall", "swap", "copy:swap")])
def test_item_kernels_are_spans(comms, kind, impl, name):
    sp = traced_call(comms, kind, impl, 5)
    assert count(sp, name) >= N - 1


@pytest.mark.parametrize("kind", ["allgather", "alltoall"])
def test_sm_kernel_span(comms, kind):
    sp = traced_call(comms, kind, "sm", 6)
    assert sum(1 for n, *_ in sp if n.startswith("kernel:")) == N  # one per unit (per-rank streams)


def test_prelaunch_graph_spans(comms):
    sp = traced_call(comms, "alltoall", "prelaunch_pcpy", 7)
    assert count(sp, "copy:graph") == N
    assert sum(1 for n, *_ in sp if n == "trigger") == N


def test_begin_twice_is_rejected_and_empty_trace_is_empty(comms):
    n = ctypes.c_size_t()
    L = cc.lib()
    assert L.cecoll_trace_begin(comms[0]._h) == 0
    assert L.cecoll_trace_begin(comms[0]._h) != 0  # already tracing
    assert L.cecoll_trace_end(comms[0]._h, None, 0, ctypes.byref(n)) == 0
    assert n.value == 2  # "[]": nothing was issued
    buf = ctypes.create_string_buffer(8)
    assert L.cecoll_trace_end(comms[0]._h, buf, 8, ctypes.byref(n)) == 0
    assert buf.value == b"[]"
