"""GPU parity: every implementation, through the C ABI, bit-exact against the
reference's golden digests (tests/golden/digests.json, produced from the
reference's own compile() output by oracle/make_golden.py) and against the
oracle at larger sizes. Ranks are co-resident on cuda:0 (devlist repeats the
device), so every chunk transfer is a real device copy through the executor
that would cross NVLink on a multi-GPU node.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2511_06605_b200 as cc
from oracle import oracle as ora

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLDEN, "digests.json")) as _f:
    DIGESTS = json.load(_f)

_COMMS = {}


def comms(n):
    if n not in _COMMS:
        _COMMS[n] = cc.Comm.init_all([0] * n)
    return _COMMS[n]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(a.tobytes()).hexdigest()


def run(kind, impl, s, n, seed, stream_mode="shared", sends=None, recvs=None):
    in_bytes = s if kind == "allgather" else n * s
    in_place = impl.endswith("swap")
    host_in = [ora.splitmix_pattern(in_bytes, r, seed) for r in range(n)]
    if sends is None:
        sends = [torch.empty(in_bytes, dtype=torch.uint8, device="cuda") for _ in range(n)]
    for t, h in zip(sends, host_in):
        t.copy_(torch.from_numpy(h))
    if in_place:
        recvs = sends
    elif recvs is None:
        recvs = [torch.full((n * s,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(n)]
    else:
        for t in recvs:
            t.fill_(0xA5)
    if stream_mode == "shared":
        streams = torch.cuda.current_stream()
    else:
        streams = [torch.cuda.Stream() for _ in range(n)]
        for st in streams:
            st.wait_stream(torch.cuda.current_stream())
    torch.cuda.synchronize()
    fn = cc.all_gather if kind == "allgather" else cc.all_to_all
    fn(comms(n), sends, recvs, s, impl=impl, streams=streams)
    torch.cuda.synchronize()
    return host_in, [t.cpu().numpy() for t in recvs], sends, recvs


CASES = [d for d in DIGESTS if d["n"] in (2, 3, 4, 8)]


@pytest.mark.parametrize("stream_mode", ["shared", "per_rank"])
@pytest.mark.parametrize("d", CASES, ids=lambda d: f"{d['kind']}-{d['impl']}-n{d['n']}-s{d['s']}-seed{d['seed']}")
def test_matches_reference_digest(d, stream_mode):
    _, res, _, _ = run(d["kind"], d["impl"], d["s"], d["n"], d["seed"], stream_mode)
    assert [sha(r) for r in res] == d["sha256"]


SM_CASES = [d for d in CASES if d["impl"] == "pcpy"]


@pytest.mark.parametrize("stream_mode", ["shared", "per_rank"])
@pytest.mark.parametrize("d", SM_CASES, ids=lambda d: f"{d['kind']}-sm-n{d['n']}-s{d['s']}-seed{d['seed']}")
def test_sm_path_matches_reference_digest(d, stream_mode):
    # Every implementation of a collective has the same postcondition
    # (verifier.cpp:143-169); the SM path is checked against pcpy's digest.
    _, res, _, _ = run(d["kind"], "sm", d["s"], d["n"], d["seed"], stream_mode)
    assert [sha(r) for r in res] == d["sha256"]


@pytest.mark.parametrize("impl", ["hybrid", "pull"])
@pytest.mark.parametrize("stream_mode", ["shared", "per_rank"])
@pytest.mark.parametrize("d", SM_CASES, ids=lambda d: f"{d['kind']}-n{d['n']}-s{d['s']}-seed{d['seed']}")
def test_b200_executors_match_reference_digest(d, stream_mode, impl):
    # The hybrid (copy-engine lane + SM share per chunk) and pull (destination-
    # issued reads) executors against the same reference digests.
    _, res, _, _ = run(d["kind"], impl, d["s"], d["n"], d["seed"], stream_mode)
    assert [sha(r) for r in res] == d["sha256"]


@pytest.mark.parametrize("impl", ["pcpy", "b2b", "bcst", "swap", "prelaunch_pcpy", "prelaunch_b2b",
                                  "prelaunch_bcst", "prelaunch_swap", "sm", "hybrid", "pull"])
@pytest.mark.parametrize("stream_mode", ["shared", "per_rank"])
def test_repeated_calls_reuse_plans_and_flags(impl, stream_mode):
    n, s = 4, 8192 + 16
    kind = "allgather" if impl.endswith("bcst") else "alltoall"
    if impl in ("pcpy", "b2b", "prelaunch_pcpy", "prelaunch_b2b", "sm", "hybrid", "pull"):
        kinds = ["allgather", "alltoall"]
    else:
        kinds = [kind]
    O = ora.Oracle()
    for kind in kinds:
        sends = recvs = None
        for it in range(5):
            host_in, res, sends, recvs = run(kind, impl, s, n, seed=100 + it, stream_mode=stream_mode,
                                             sends=sends, recvs=recvs)
            assert O.check(kind, s, n, impl.endswith("swap"), host_in, res) == -1, (kind, impl, it)


@pytest.mark.parametrize("kind,impl,s", [
    ("alltoall", "sm", 8 << 20),
    ("alltoall", "pcpy", 8 << 20),
    ("alltoall", "b2b", 8 << 20),
    ("alltoall", "prelaunch_pcpy", 8 << 20),
    ("alltoall", "swap", 8 << 20),
    ("alltoall", "hybrid", 8 << 20),
    ("allgather", "hybrid", 16 << 20),
    ("alltoall", "pull", 8 << 20),
    ("allgather", "pull", 16 << 20),
    ("allgather", "sm", 64 << 20),
    ("allgather", "bcst", 16 << 20),
    ("allgather", "prelaunch_pcpy", 16 << 20),
])
def test_large_against_oracle(kind, impl, s):
    n = 8
    O = ora.Oracle()
    host_in, res, _, _ = run(kind, impl, s, n, seed=5)
    assert O.check(kind, s, n, impl.endswith("swap"), host_in, res) == -1


def test_alltoall_twice_is_identity_at_full_size():
    # Size-independent property: alltoall is an involution of the rank/chunk
    # layout, so applying it twice restores every send buffer.
    n, s = 8, 8 << 20
    cs = comms(n)
    g = torch.Generator(device="cuda").manual_seed(0)
    sends = [torch.randint(0, 256, (n * s,), dtype=torch.uint8, device="cuda", generator=g) for _ in range(n)]
    mid = [torch.empty_like(t) for t in sends]
    back = [torch.empty_like(t) for t in sends]
    for impl in ("sm", "pcpy", "prelaunch_pcpy"):
        cc.all_to_all(cs, sends, mid, s, impl=impl)
        cc.all_to_all(cs, mid, back, s, impl=impl)
        torch.cuda.synchronize()
        assert all(torch.equal(a, b) for a, b in zip(sends, back)), impl


def test_allgather_ranks_agree_at_full_size():
    n, s = 8, 64 << 20
    cs = comms(n)
    sends = [torch.full((s,), r + 1, dtype=torch.uint8, device="cuda") for r in range(n)]
    recvs = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
    cc.all_gather(cs, sends, recvs, s, impl="auto")
    torch.cuda.synchronize()
    for r in range(n):
        assert torch.equal(recvs[r], recvs[0])
        for i in range(n):
            assert int(recvs[r][i * s]) == i + 1 and int(recvs[r][(i + 1) * s - 1]) == i + 1


def test_explicit_prelaunch_plan_rearms_and_cancels():
    n, s = 4, 65536
    cs = comms(n)
    O = ora.Oracle()
    sends = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
    recvs = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
    plan = cc.Plan(cs, "alltoall", sends, recvs, s, impl="prelaunch_pcpy")
    stream = torch.cuda.current_stream()
    for it in range(4):
        host_in = [ora.splitmix_pattern(n * s, r, 50 + it) for r in range(n)]
        for t, h in zip(sends, host_in):
            t.copy_(torch.from_numpy(h))
        plan.launch([stream] * n)
        stream.synchronize()  # stream sync, not device sync: the next instance is armed
        res = [t.cpu().numpy() for t in recvs]
        assert O.check("alltoall", s, n, False, host_in, res) == -1, it
    plan.destroy()  # cancels the armed instance
    torch.cuda.synchronize()


def test_single_process_requires_group():
    cs = comms(2)
    a = torch.zeros(2048, dtype=torch.uint8, device="cuda")
    b = torch.zeros(2048, dtype=torch.uint8, device="cuda")
    L = cc.lib()
    st = L.cecoll_alltoall(a.data_ptr(), b.data_ptr(), 1024, 0, cs[0]._h, None)
    assert st == 1


def test_inplace_alltoall_needs_swap():
    cs = comms(2)
    bufs = [torch.zeros(2048, dtype=torch.uint8, device="cuda") for _ in range(2)]
    with pytest.raises(cc.InvalidArgument):
        cc.all_to_all(cs, bufs, bufs, 1024, impl="pcpy")


def test_counters_track_commands():
    n, s = 8, 4096
    cs = cc.Comm.init_all([0] * n)
    try:
        sends = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
        recvs = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
        streams = [torch.cuda.Stream() for _ in range(n)]
        c0 = cs[0].counters()
        cc.all_to_all(cs, sends, recvs, s, impl="pcpy", streams=streams)
        c1 = cs[0].counters()
        # static_metrics identities (test_program.cpp:29-43): 56 copies + 8
        # local placements; with one unit per rank every copy is signalled.
        assert c1["copies"] - c0["copies"] == 56 + 8
        assert c1["flag_writes"] - c0["flag_writes"] >= 56
        cc.all_to_all(cs, sends, recvs, s, impl="b2b", streams=streams)
        c2 = cs[0].counters()
        assert c2["copies"] - c1["copies"] == 56 + 8
        torch.cuda.synchronize()
    finally:
        cc.destroy_all(cs)


with open(os.path.join(GOLDEN, "programs.json")) as _f:
    REF_DUMPS = [e for e in json.load(_f)["programs"] if "dump" in e]


@pytest.mark.parametrize("e", REF_DUMPS, ids=lambda e: f"{e['kind']}-{e['impl']}-n{e['n']}")
def test_executes_the_reference_program_text(e):
    """The reference's own compile() output (dump_program text, golden) run as
    is on the GPU through cecoll_program_parse + cecoll_plan_create_program."""
    kind, n, s = e["kind"], e["n"], e["s"]
    prog = cc.Program.parse(e["dump"], kind, s, n)
    in_place = e["impl"].endswith("swap")
    in_bytes = s if kind == "allgather" else n * s
    host_in = [ora.splitmix_pattern(in_bytes, r, 11) for r in range(n)]
    sends = [torch.from_numpy(h).cuda() for h in host_in]
    recvs = sends if in_place else [torch.full((n * s,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(n)]
    plan = cc.Plan(comms(n), kind, sends, recvs, program=prog)
    plan.launch([torch.cuda.current_stream()] * n)
    torch.cuda.current_stream().synchronize()
    res = [t.cpu().numpy() for t in recvs]
    plan.destroy()
    torch.cuda.synchronize()
    assert ora.Oracle().check(kind, s, n, in_place, host_in, res) == -1


def test_auto_picks_swap_for_inplace_alltoall():
    n, s = 4, 4096
    O = ora.Oracle()
    host_in = [ora.splitmix_pattern(n * s, r, 77) for r in range(n)]
    bufs = [torch.from_numpy(h).cuda() for h in host_in]
    cc.all_to_all(comms(n), bufs, bufs, s, impl="auto")
    torch.cuda.synchronize()
    assert O.check("alltoall", s, n, True, host_in, [b.cpu().numpy() for b in bufs]) == -1


@pytest.mark.parametrize("impl", ["sm", "pcpy", "b2b", "prelaunch_b2b", "bcst", "swap"])
@pytest.mark.parametrize("n", [16, 32])
def test_many_ranks(impl, n):
    """Up to kMaxRanks co-resident ranks (the reference tests n up to 16,
    acceptance.cpp:89-143); per-rank streams exercise every flag pair."""
    kind = "allgather" if impl == "bcst" else "alltoall"
    s = 4096 + 48
    O = ora.Oracle()
    host_in, res, _, _ = run(kind, impl, s, n, seed=3, stream_mode="per_rank" if n == 16 else "shared")
    assert O.check(kind, s, n, impl.endswith("swap"), host_in, res) == -1


@pytest.mark.parametrize("impl", ["sm", "pcpy", "b2b", "prelaunch_pcpy", "swap", "prelaunch_swap"])
def test_flag_protocol_under_random_delays(impl):
    """Stress of the rdy/done protocol: one stream per rank,
    random spin delays injected into random ranks' streams before each
    collective, 25 back-to-back collectives on the same buffers, every result
    checked. A lost or early flag shows up as a mismatch (or a hang, bounded
    by the test timeout)."""
    import random

    n, s = 6, 12288
    cs = comms(n)
    O = ora.Oracle()
    rng = random.Random(impl)
    streams = [torch.cuda.Stream() for _ in range(n)]
    sends = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
    recvs = sends if impl.endswith("swap") else [torch.empty(n * s, dtype=torch.uint8, device="cuda")
                                                 for _ in range(n)]
    for it in range(25):
        host_in = [ora.splitmix_pattern(n * s, r, 1000 + it) for r in range(n)]
        torch.cuda.synchronize()
        for t, h in zip(sends, host_in):
            t.copy_(torch.from_numpy(h))
        torch.cuda.synchronize()
        for st in streams:
            if rng.random() < 0.5:
                with torch.cuda.stream(st):
                    torch.cuda._sleep(rng.randint(1000, 200000))
        cc.all_to_all(cs, sends, recvs, s, impl=impl, streams=streams)
        torch.cuda.synchronize()
        res = [t.cpu().numpy() for t in recvs]
        assert O.check("alltoall", s, n, impl.endswith("swap"), host_in, res) == -1, it


@pytest.mark.parametrize("kind,impl", [("allgather", "sm"), ("allgather", "bcst"), ("alltoall", "sm"),
                                       ("alltoall", "prelaunch_pcpy")])
def test_mem_alloc_buffers(kind, impl):
    """cecoll_mem_alloc: library-owned registered buffers used as send/recv,
    then freed; a second free is rejected."""
    n, s = 8, 2 * 65536 + 80
    cs = comms(n)
    in_bytes = s if kind == "allgather" else n * s
    sends = [c.mem_alloc(in_bytes) for c in cs]
    recvs = [c.mem_alloc(n * s) for c in cs]
    assert all(t.numel() == in_bytes for t in sends)
    assert all(t.data_ptr() % (2 << 20) == 0 for t in sends + recvs)
    try:
        host_in, res, _, _ = run(kind, impl, s, n, 91, sends=sends, recvs=recvs)
        want = [np.zeros(n * s, np.uint8) for _ in range(n)]
        ora.Oracle().reference_result(kind, s, n, host_in, want)
        assert all(np.array_equal(a, b) for a, b in zip(res, want))
    finally:
        torch.cuda.synchronize()
        for c, a, b in zip(cs, sends, recvs):
            c.mem_free(a)
            c.mem_free(b)
    with pytest.raises(cc.CecollError):
        cs[0].mem_free(sends[0])


@pytest.mark.timeout(300)
@pytest.mark.parametrize("impl", ["sm", "pcpy", "b2b", "hybrid", "pull", "swap", "prelaunch_pcpy", "prelaunch_b2b"])
def test_back_to_back_collectives_without_host_sync(impl, fresh=False):
    """Flag reuse across collectives in flight: one stream
    per rank; per iteration each rank's stream loads a fresh input, runs the
    collective and copies its result out, with random spin delays — no host
    synchronisation until the end. A destination overwritten before it
    copied out the previous result (rdy), or a send buffer reloaded before
    every peer finished reading it (done), changes some iteration's result."""
    import random

    n, s, iters = 4, 12288 + 16, 12
    cs = cc.Comm.init_all([0] * n) if fresh else comms(n)
    O = ora.Oracle()
    rng = random.Random("b2b-" + impl)
    in_place = impl.endswith("swap")
    streams = [torch.cuda.Stream() for _ in range(n)]
    hosts = [[ora.splitmix_pattern(n * s, r, 5000 + it) for r in range(n)] for it in range(iters)]
    inputs = [[torch.from_numpy(hosts[it][r]).cuda() for r in range(n)] for it in range(iters)]
    sends = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
    recvs = sends if in_place else [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
    outs = [[torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)] for _ in range(iters)]
    torch.cuda.synchronize()
    for it in range(iters):
        for r, st in enumerate(streams):
            with torch.cuda.stream(st):
                if rng.random() < 0.5:
                    torch.cuda._sleep(rng.randint(1000, 100000))
                sends[r].copy_(inputs[it][r])
        cc.all_to_all(cs, sends, recvs, s, impl=impl, streams=streams)
        for r, st in enumerate(streams):
            with torch.cuda.stream(st):
                if rng.random() < 0.5:
                    torch.cuda._sleep(rng.randint(1000, 100000))
                outs[it][r].copy_(recvs[r])
    torch.cuda.synchronize()
    for it in range(iters):
        res = [t.cpu().numpy() for t in outs[it]]
        assert O.check("alltoall", s, n, in_place, hosts[it], res) == -1, (impl, it)
    if fresh:
        cc.destroy_all(cs)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("impl", ["sm", "pcpy", "pull", "prelaunch_b2b"])
def test_back_to_back_through_the_other_device_signal_path(impl, monkeypatch):
    """The same, with every cross-unit signal on the other-device path
    (signal kernels, folded start signals are not used: several units)."""
    monkeypatch.setenv("CECOLL_FORCE_REMOTE_SIGNALS", "1")
    test_back_to_back_collectives_without_host_sync(impl, fresh=True)


def test_misrouted_program_fails_parity_on_the_gpu():
    """Negative control for every parity test here (test_verifier.cpp:35-49
    on hardware): the reference's own program text with one copy misrouted
    (rank 0's chunk for rank 1 written to slot 2 instead of slot 0) executes
    fine — and the byte check must catch it, exactly at the bytes it broke."""
    kind, n, s = "allgather", 4, 4096
    with open(os.path.join(GOLDEN, "programs.json")) as f:
        text = next(e["dump"] for e in json.load(f)["programs"]
                    if (e["kind"], e["impl"], e["s"], e["n"]) == (kind, "pcpy", s, n) and "dump" in e)
    lines = [line.split("\t") for line in text.splitlines()]
    hits = 0
    for f in lines:
        if f[2] == "copy" and f[3].startswith("g0.in") and f[4] == f"g1.out[0+{s}]":
            f[4] = f"g1.out[{2 * s}+{s}]"  # slot 2 instead of slot 0
            hits += 1
    assert hits == 1
    bad = "\n".join("\t".join(f) for f in lines) + "\n"
    host_in = [ora.splitmix_pattern(s, r, 21) for r in range(n)]
    O = ora.Oracle()
    for txt, want_ok in ((text, True), (bad, False)):
        sends = [torch.from_numpy(h).cuda() for h in host_in]
        recvs = [torch.full((n * s,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(n)]
        plan = cc.Plan(comms(n), kind, sends, recvs, program=cc.Program.parse(txt, kind, s, n))
        plan.launch([torch.cuda.current_stream()] * n)
        torch.cuda.current_stream().synchronize()
        res = [t.cpu().numpy() for t in recvs]
        plan.destroy()
        torch.cuda.synchronize()
        bad_at = O.check(kind, s, n, False, host_in, res)
        assert (bad_at == -1) == want_ok, (want_ok, bad_at)


@pytest.mark.parametrize("kind,impl", [("alltoall", "prelaunch_pcpy"), ("alltoall", "prelaunch_b2b"),
                                       ("allgather", "prelaunch_bcst"), ("alltoall", "prelaunch_swap"),
                                       ("allgather", "pcpy"), ("alltoall", "sm")])
def test_plan_arm_and_trigger(kind, impl):
    """SURVEY §8(b) plan_arm / plan_trigger: arm ahead (idempotent), trigger
    without re-arming — after which device-wide synchronisation returns —,
    disarm then trigger (re-arms inside), and every result byte-checked."""
    n, s = 4, 12288
    O = ora.Oracle()
    in_place = impl.endswith("swap")
    in_bytes = s if kind == "allgather" else n * s
    sends = [torch.empty(in_bytes, dtype=torch.uint8, device="cuda") for _ in range(n)]
    recvs = sends if in_place else [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
    plan = cc.Plan(comms(n), kind, sends, recvs, s, impl=impl)
    stream = torch.cuda.current_stream()
    for it, steps in enumerate((["arm", "arm", "trigger"], ["trigger"], ["arm", "disarm", "trigger"])):
        host_in = [ora.splitmix_pattern(in_bytes, r, 300 + it) for r in range(n)]
        if not in_place:
            for t in recvs:
                t.fill_(0xA5)
        for t, h in zip(sends, host_in):
            t.copy_(torch.from_numpy(h))
        torch.cuda.synchronize()
        for step in steps:
            if step == "trigger":
                plan.trigger([stream] * n)
            else:
                getattr(plan, step)()
        torch.cuda.synchronize()  # nothing is left armed after a trigger
        res = [t.cpu().numpy() for t in recvs]
        assert O.check(kind, s, n, in_place, host_in, res) == -1, (impl, steps)
    plan.destroy()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("impl", ["sm", "pcpy", "b2b", "bcst", "prelaunch_bcst", "prelaunch_pcpy", "hybrid", "pull"])
def test_allgather_back_to_back_without_host_sync(impl):
    """The all-gather side of the flag-reuse stress (bcst's two-destination
    items included): one stream per rank, random spin delays, input reload,
    collective, copy-out, no host synchronisation until the end."""
    import random

    n, s, iters = 4, 12288 + 16, 12
    cs = comms(n)
    rng = random.Random("ag-" + impl)
    streams = [torch.cuda.Stream() for _ in range(n)]
    hosts = [[ora.splitmix_pattern(s, r, 6000 + it) for r in range(n)] for it in range(iters)]
    inputs = [[torch.from_numpy(hosts[it][r]).cuda() for r in range(n)] for it in range(iters)]
    sends = [torch.empty(s, dtype=torch.uint8, device="cuda") for _ in range(n)]
    recvs = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
    outs = [[torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)] for _ in range(iters)]
    torch.cuda.synchronize()
    for it in range(iters):
        for r, st in enumerate(streams):
            with torch.cuda.stream(st):
                if rng.random() < 0.5:
                    torch.cuda._sleep(rng.randint(1000, 100000))
                sends[r].copy_(inputs[it][r])
        cc.all_gather(cs, sends, recvs, s, impl=impl, streams=streams)
        for r, st in enumerate(streams):
            with torch.cuda.stream(st):
                if rng.random() < 0.5:
                    torch.cuda._sleep(rng.randint(1000, 100000))
                outs[it][r].copy_(recvs[r])
    torch.cuda.synchronize()
    for it in range(iters):
        want = np.concatenate(hosts[it])
        for r in range(n):
            assert np.array_equal(outs[it][r].cpu().numpy(), want), (impl, it, r)
