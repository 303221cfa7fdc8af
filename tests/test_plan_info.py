"""cecoll_plan_info / cecoll_comm_last_plan_info: what a plan turned into
(the fields every bench line carries, so a number cannot be misread: a
prelaunch plan that fell back to eager, a command list that is not recorded,
the mover and the flag path of every unit)."""
import pytest

import paper_2511_06605_b200 as cc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

N = 8


@pytest.fixture(scope="module")
def comms():
    cs = cc.Comm.init_all([0] * N)
    yield cs
    cc.destroy_all(cs)


def _bufs(s, kind="alltoall"):
    in_bytes = s if kind == "allgather" else N * s
    return ([torch.randint(0, 256, (in_bytes,), dtype=torch.uint8, device="cuda") for _ in range(N)],
            [torch.zeros(N * s, dtype=torch.uint8, device="cuda") for _ in range(N)])


def test_single_unit_sm_is_one_kernel_recorded(comms):
    """One kernel per collective, replayed as a one-node graph from the second
    launch (cheaper on the host than a direct launch, exec.cpp graph_eligible)."""
    sends, recvs = _bufs(4096)
    st = torch.cuda.Stream()
    c0 = comms[0].counters()
    for _ in range(3):
        cc.all_to_all(comms, sends, recvs, 4096, impl="sm", streams=st)
    c1 = comms[0].counters()
    info = comms[0].last_plan_info()
    assert info["impl"] == "sm" and info["recorded"] and info["record_note"] == ""
    assert c1["kernels"] - c0["kernels"] == 3 and c1["recorded_launches"] - c0["recorded_launches"] == 2
    assert len(info["units"]) == 1 and info["units"][0]["mover"] in ("tma", "reg")
    assert info["units"][0]["ranks"] == list(range(N))
    torch.cuda.synchronize()


@pytest.mark.parametrize("impl", ["pcpy", "b2b", "hybrid"])
def test_copy_engine_plans_record_from_the_second_launch(comms, impl):
    sends, recvs = _bufs(65536)
    st = torch.cuda.Stream()
    cc.all_to_all(comms, sends, recvs, 65536, impl=impl, streams=st)
    assert not comms[0].last_plan_info()["recorded"]
    cc.all_to_all(comms, sends, recvs, 65536, impl=impl, streams=st)
    info = comms[0].last_plan_info()
    assert info["recorded"] and info["record_note"] == "", info
    torch.cuda.synchronize()


@pytest.mark.parametrize("fold", ["0", "1"])
@pytest.mark.parametrize("impl,s,small", [("prelaunch_b2b", 4096, True), ("prelaunch_swap", 4096, True),
                                          ("prelaunch_pcpy", 8 << 20, False)])
def test_prelaunch_plans_report_their_body(comms, impl, s, small, fold, monkeypatch):
    """The folded single-kernel body is opt-in (CECOLL_PRELAUNCH_FOLD=1) and
    only for small collectives; every launch is byte-checked, three times
    (instances consume posts 0, 1, 2 through their kernel parameters)."""
    monkeypatch.setenv("CECOLL_PRELAUNCH_FOLD", fold)
    sends, recvs = _bufs(s)
    if impl.endswith("swap"):
        recvs = sends
    plan = cc.Plan(comms, "alltoall", sends, recvs, s, impl=impl)
    info = plan.info()
    assert info["prelaunch"] and info["graph_fallback"] == ""
    assert info["prelaunch_folded"] == (small and fold == "1"), info
    st = torch.cuda.current_stream()
    # Results are compared on the host: while the next instance is armed, a
    # torch kernel launched for the first time in the process would wait
    # behind the armed gate for its lazy module load.
    host_sends = [t.cpu() for t in sends]
    for it in range(3):
        want = None
        if not impl.endswith("swap"):
            want = [torch.cat([host_sends[j][r * s:(r + 1) * s] for j in range(N)]) for r in range(N)]
        plan.launch(st)
        st.synchronize()  # the next instance is armed: no device-wide sync
        if want is not None:
            assert all(torch.equal(a.cpu(), b) for a, b in zip(recvs, want)), (impl, it)
    plan.destroy()
    torch.cuda.synchronize()


def test_sm_budget_caps_the_grid(comms):
    sends, recvs = _bufs(8 << 20)
    comms[0].set_sm_budget(16)
    try:
        plan = cc.Plan(comms, "alltoall", sends, recvs, 8 << 20, impl="sm")
        info = plan.info()
        assert info["sm_budget"] == 16 and info["units"][0]["grid"] == 16
        plan.launch(torch.cuda.current_stream())
        torch.cuda.synchronize()
        for i in range(N):
            for j in range(N):
                s = 8 << 20
                assert torch.equal(recvs[j][i * s:(i + 1) * s], sends[i][j * s:(j + 1) * s])
        plan.destroy()
    finally:
        comms[0].set_sm_budget(0)


@pytest.mark.parametrize("kind,s,tile,tiles,grid", [
    ("allgather", 65536, 4096, 128, 128),         # 8 fan items: smallest tile leaving <= 1 tile per SM
    ("allgather", 262144, 15360, 144, 144),       # 8 x ceil(256 KiB / 15 KiB) = 144 <= 148
    ("alltoall", 65536, 32768, 128, 128),         # 64 items x 2 tiles already fit one wave
    ("alltoall", 1 << 20, 16384, 64 * 64, 1366),        # up to 16384 tiles: 3 tiles per CTA
    ("alltoall", 8 << 20, 16384, 64 * 512, 64 * 256),  # the headline: 16 KiB tiles, 2 tiles per CTA
    ("allgather", 8 << 20, 8192, 8 * 1024, 8 * 1024),  # fan: 8 KiB tiles, one tile per CTA
])
def test_tma_tile_size_follows_the_table(comms, kind, s, tile, tiles, grid):
    """kernels.cu table_tile / mover_grid_for: one tile per CTA while the table
    fits one wave of one CTA per SM (a 64 KiB all-gather 8.2 -> 4.1 us per
    collective); above, short-lived CTAs of the table kind's shape (copy: 16
    KiB tiles, 3 per CTA up to 16384 tiles and 2 above; fan: 8 KiB tiles, 1
    per CTA)."""
    sends, recvs = _bufs(s, kind)
    torch.cuda.synchronize()  # the inputs are written on the default stream
    fn = cc.all_gather if kind == "allgather" else cc.all_to_all
    fn(comms, sends, recvs, s, impl="sm", streams=torch.cuda.Stream())
    torch.cuda.synchronize()
    u = comms[0].last_plan_info()["units"][0]
    assert u["mover"] == "tma" and u["tile_bytes"] == tile and u["tiles"] == tiles, u
    assert u["grid"] == grid, u
    ok = all(torch.equal(recvs[j][i * s:(i + 1) * s], sends[i] if kind == "allgather" else sends[i][j * s:(j + 1) * s])
             for i in range(N) for j in range(N))
    assert ok
    torch.cuda.synchronize()


def test_grid_cap_loops_over_the_remaining_tiles(comms):
    """A table of more tiles than kMaxGrid CTAs (2^19: fused_finish counts CTAs
    in 20 bits) launches the capped grid and every CTA loops over its further
    tiles: an all-gather of 1 GiB chunks is 2^20 fan tiles of 8 KiB."""
    s = 1 << 30
    sends = [torch.randint(0, 256, (s,), dtype=torch.uint8, device="cuda") for _ in range(N)]
    recvs = [torch.empty(N * s, dtype=torch.uint8, device="cuda") for _ in range(N)]
    try:
        torch.cuda.synchronize()
        cc.all_gather(comms, sends, recvs, s, impl="sm", streams=torch.cuda.Stream())
        torch.cuda.synchronize()
        u = comms[0].last_plan_info()["units"][0]
        assert u["tiles"] == 8 * (s // 8192) and u["grid"] == 1 << 19, u
        for j in range(N):
            for i in range(N):
                assert torch.equal(recvs[j][i * s:(i + 1) * s], sends[i]), (i, j)
    finally:
        del sends, recvs
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
