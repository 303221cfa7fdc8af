"""Edge cases of the byte layout (compiler.cpp:115-126), through the C ABI on
cuda:0, checked against the oracle: tiny and ragged chunks (1..33 bytes),
odd rank counts, buffers that are not 16-byte aligned (the movers' bytewise
heads/tails and the TMA gating), one stream per rank, and the argument
errors the reference raises as std::invalid_argument (compiler.cpp:142-145,
program.cpp:31-38)."""
import pytest

import paper_2511_06605_b200 as cc
from oracle import oracle as ora

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

_C = {}


def comms(n):
    if n not in _C:
        _C[n] = cc.Comm.init_all([0] * n)
    return _C[n]


def kinds_for(impl):
    if impl.endswith("bcst"):
        return ["allgather"]
    if impl.endswith("swap"):
        return ["alltoall"]
    return ["allgather", "alltoall"]


def run_case(kind, impl, s, n, seed, offset=0, per_rank=False):
    in_place = impl.endswith("swap")
    in_bytes = s if kind == "allgather" else n * s
    host = [ora.splitmix_pattern(in_bytes, r, seed) for r in range(n)]
    # slices at `offset` bytes into larger allocations: misaligned pointers
    sbase = [torch.zeros(in_bytes + 64, dtype=torch.uint8, device="cuda") for _ in range(n)]
    sends = [b[offset:offset + in_bytes] for b in sbase]
    for t, h in zip(sends, host):
        t.copy_(torch.from_numpy(h))
    if in_place:
        recvs = sends
    else:
        rbase = [torch.full((n * s + 64,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(n)]
        recvs = [b[offset:offset + n * s] for b in rbase]
    streams = [torch.cuda.Stream() for _ in range(n)] if per_rank else torch.cuda.Stream()
    torch.cuda.synchronize()
    fn = cc.all_gather if kind == "allgather" else cc.all_to_all
    for _ in range(2):  # second call: recorded replay where it applies
        if not in_place:
            for t in recvs:
                t.fill_(0xA5)
        else:
            for t, h in zip(sends, host):
                t.copy_(torch.from_numpy(h))
        torch.cuda.synchronize()
        fn(comms(n), sends, recvs, s, impl=impl, streams=streams)
        torch.cuda.synchronize()
        res = [t.cpu().numpy() for t in recvs]
        assert ora.Oracle().check(kind, s, n, in_place, host, res) == -1, (kind, impl, s, n, offset)


IMPLS = ["sm", "pcpy", "b2b", "bcst", "swap", "hybrid", "pull", "prelaunch_b2b", "prelaunch_swap"]


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("s", [1, 3, 15, 17, 33])
def test_tiny_ragged_chunks_odd_ranks(impl, s):
    for kind in kinds_for(impl):
        run_case(kind, impl, s, 3, seed=1000 + s)


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("offset", [1, 3, 8])
def test_misaligned_buffers(impl, offset):
    for kind in kinds_for(impl):
        run_case(kind, impl, 65536 + 5, 4, seed=2000 + offset, offset=offset)


@pytest.mark.parametrize("impl", ["sm", "pcpy", "hybrid", "pull", "prelaunch_pcpy"])
def test_ragged_two_ranks_per_rank_streams(impl):
    for kind in kinds_for(impl):
        run_case(kind, impl, 40961, 2, seed=3000, per_rank=True)


def test_argument_errors():
    n = 2
    cs = comms(n)
    buf = [torch.zeros(64, dtype=torch.uint8, device="cuda") for _ in range(n)]
    out = [torch.zeros(128, dtype=torch.uint8, device="cuda") for _ in range(n)]
    with pytest.raises(cc.InvalidArgument):
        cc.all_to_all(cs, buf, out, 0, impl="pcpy")  # chunk size must be positive (program.cpp:31-38)
    for impl in ("pcpy", "b2b", "sm", "hybrid", "pull"):
        with pytest.raises(cc.InvalidArgument):
            cc.all_to_all(cs, buf, buf, 32, impl=impl)  # in place only for swap (compiler.cpp:209-210)
    with pytest.raises(cc.InvalidArgument):
        cc.all_gather(cs, buf, out, 64, impl="swap")  # swap is all-to-all only (compiler.cpp:70-75)
    with pytest.raises(cc.InvalidArgument):
        cc.all_to_all(cs, buf, out, 64, impl="bcst")  # bcst is all-gather only
    with pytest.raises(cc.InvalidArgument):
        cc.all_to_all(cs, buf, out, 64, impl="nope")
    torch.cuda.synchronize()
