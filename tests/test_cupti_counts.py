"""Structural counts from CUPTI activity records: the copy
commands the driver actually executed for one eager collective equal the
reference's static_metrics identities (test_program.cpp:29-52) plus the
local placements — an account independent of the library's own counters.
torch.profiler collects the CUPTI activities."""
import pytest

import paper_2511_06605_b200 as cc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _device_activities(fn):
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    memcpy = sum(e.count for e in prof.key_averages() if "Memcpy" in e.key and "DtoD" in e.key)
    kernels = sum(e.count for e in prof.key_averages() if "items_kernel" in e.key or "signal_kernel" in e.key
                  or "poll_kernel" in e.key)
    return memcpy, kernels


@pytest.mark.parametrize("impl", ["pcpy", "b2b"])
def test_copy_commands_match_static_metrics(impl):
    n, s = 8, 65536
    comms = cc.Comm.init_all([0] * n)
    try:
        sends = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
        recvs = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
        streams = [torch.cuda.Stream() for _ in range(n)]  # one unit per rank: eager, every copy its own command
        cc.all_to_all(comms, sends, recvs, s, impl=impl, streams=streams)  # plan built outside the capture
        torch.cuda.synchronize()
        c0 = comms[0].counters()
        memcpy, _ = _device_activities(lambda: cc.all_to_all(comms, sends, recvs, s, impl=impl, streams=streams))
        c1 = comms[0].counters()
        # n(n-1) = 56 route copies (static_metrics: pcpy 56 queues of one copy,
        # b2b 8 queues of 7) + n local placements (verifier.cpp:40-44)
        assert c1["copies"] - c0["copies"] == 56 + 8
        # every copy is an individual copy activity: pcpy's one per lane, b2b's
        # n-1 back to back on one lane (the driver's batched-copy entry point
        # is not used)
        assert memcpy == 56 + 8, memcpy
    finally:
        torch.cuda.synchronize()
        cc.destroy_all(comms)


def test_broadcast_commands_are_kernels():
    # bcst: CUDA has no copy-engine broadcast; the 24 two-destination commands
    # run as item kernels (one per lane with flags), the 8 single copies and 8
    # placements as copies (static_metrics bcst: 32 data commands at n = 8).
    n, s = 8, 65536
    comms = cc.Comm.init_all([0] * n)
    try:
        sends = [torch.zeros(s, dtype=torch.uint8, device="cuda") for _ in range(n)]
        recvs = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
        streams = [torch.cuda.Stream() for _ in range(n)]
        cc.all_gather(comms, sends, recvs, s, impl="bcst", streams=streams)
        torch.cuda.synchronize()
        memcpy, kernels = _device_activities(
            lambda: cc.all_gather(comms, sends, recvs, s, impl="bcst", streams=streams))
        assert memcpy == 8 + 8, memcpy
        assert kernels >= 8 * 3, kernels  # 3 broadcast lanes per rank, each its own item kernel
    finally:
        torch.cuda.synchronize()
        cc.destroy_all(comms)
