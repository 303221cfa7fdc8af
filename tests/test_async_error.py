"""A peer that never signals (the reference's untriggered-poll deadlock,
sim.cpp:227-242, raised there as std::runtime_error) surfaces as
CECOLL_TIMEOUT through cecoll_comm_get_async_error and the communicator's
destroy — not as a silent wrong answer. Rank 1's stream is held busy for
longer than the device-side poll bound (20 s, flags.cuh kPollTimeoutNs), so
rank 0's kernel gives up waiting for rank 1's readiness flag."""
import pytest

import paper_2511_06605_b200 as cc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.timeout(180)
def test_a_peer_that_never_signals_surfaces_as_timeout():
    n, s = 2, 4096
    cs = cc.Comm.init_all([0] * n)
    sends = [torch.randint(0, 256, (n * s,), dtype=torch.uint8, device="cuda") for _ in range(n)]
    recvs = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
    streams = [torch.cuda.Stream() for _ in range(n)]
    cc.all_to_all(cs, sends, recvs, s, impl="sm", streams=streams)
    torch.cuda.synchronize()
    assert cs[0].async_error() is None and cs[1].async_error() is None
    with torch.cuda.stream(streams[1]):
        torch.cuda._sleep(int(2.0e9 * 24))  # ~24 s at the B200's 1.965 GHz: rank 1 signals too late
    cc.all_to_all(cs, sends, recvs, s, impl="sm", streams=streams)
    torch.cuda.synchronize()
    e = cs[0].async_error()
    assert e is not None and e.status == 4, e  # CECOLL_TIMEOUT
    assert "timed out" in str(e)
    assert cs[1].async_error() is not None  # per world, sticky
    cs[0].destroy()
    with pytest.raises(cc.CecollError, match="timed out"):
        cs[1].destroy()  # the last communicator of the world reports it
