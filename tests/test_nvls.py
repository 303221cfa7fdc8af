"""NVLS (switch multicast) all-gather readiness — SURVEY §8(f)2, the multicast
form of the reference's broadcast command (compiler.cpp:166-205).

Where the node refuses multicast objects (every one-GPU box so far,
profiles/mc_probe_r01.txt) the window must fail cleanly with
CECOLL_UNSUPPORTED and leave the communicator usable. Where it accepts them,
the window's all-gather result is checked byte for byte against the oracle
(ora_check, the postcondition of verifier.cpp:143-169).
"""
import pytest

import paper_2511_06605_b200 as cc
from oracle import oracle as ora

pytestmark = pytest.mark.gpu


def _one_rank_world():
    return cc.Comm.init_rank(1, 0, 0, lambda mine: [mine])


def test_multicast_window_refuses_cleanly_or_matches_the_oracle():
    torch = pytest.importorskip("torch")
    comm = _one_rank_world()
    s = 65536 + 16 * 7
    try:
        try:
            mc = cc.McWindow(comm, s)
        except cc.CecollError as e:
            assert e.status == 2, e  # CECOLL_UNSUPPORTED, never a CUDA error or a hang
            assert "multicast" in str(e)
            # the communicator still works after the refusal
            host = ora.splitmix_pattern(s, 0, 3)
            send = torch.from_numpy(host).cuda()
            recv = torch.full((s,), 0xA5, dtype=torch.uint8, device="cuda")
            cc.all_gather([comm], [send], [recv], s, impl="sm")
            torch.cuda.synchronize()
            assert torch.equal(recv.cpu(), torch.from_numpy(host))
            return
        try:
            for seed in (0, 1):
                host = [ora.splitmix_pattern(s, 0, seed)]
                send = torch.from_numpy(host[0]).cuda()
                torch.cuda.synchronize()
                mc.allgather(send, s, torch.cuda.current_stream())
                torch.cuda.synchronize()
                res = [mc.recv[: s].cpu().numpy()]
                assert ora.Oracle().check("allgather", s, 1, False, host, res) == -1
        finally:
            mc.destroy()
    finally:
        comm.destroy()


def test_multicast_rejects_single_process_worlds():
    """The window needs one process per GPU (comm_init_rank): a
    comm_init_all world gets CECOLL_UNSUPPORTED, not a partial window."""
    comms = cc.Comm.init_all([0, 0])
    try:
        with pytest.raises(cc.CecollError) as ei:
            cc.McWindow(comms[0], 4096)
        assert ei.value.status == 2
    finally:
        cc.destroy_all(comms)
