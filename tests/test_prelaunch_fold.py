"""The folded prelaunch body (CECOLL_PRELAUNCH_FOLD=1): one
mover kernel that is its own gate. Opt-in (the two-kernel body measured
faster on one B200), so the flag-protocol stresses of test_gpu_parity run
again here with it on: repeated calls on one stream and on one stream per
rank (several folded units on one device), random delays, back-to-back
collectives without host synchronisation, arm / trigger / disarm."""
import pytest

import test_gpu_parity as P  # noqa: E402 (tests/ is on sys.path under pytest)

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _fold(monkeypatch):
    monkeypatch.setenv("CECOLL_PRELAUNCH_FOLD", "1")


@pytest.mark.parametrize("impl", ["prelaunch_pcpy", "prelaunch_b2b", "prelaunch_bcst", "prelaunch_swap"])
@pytest.mark.parametrize("stream_mode", ["shared", "per_rank"])
def test_repeated_calls(impl, stream_mode):
    P.test_repeated_calls_reuse_plans_and_flags(impl, stream_mode)


@pytest.mark.parametrize("impl", ["prelaunch_pcpy", "prelaunch_swap"])
def test_random_delays(impl):
    P.test_flag_protocol_under_random_delays(impl)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("impl", ["prelaunch_pcpy", "prelaunch_b2b"])
def test_back_to_back(impl):
    P.test_back_to_back_collectives_without_host_sync(impl, fresh=True)


@pytest.mark.parametrize("kind,impl", [("alltoall", "prelaunch_b2b"), ("allgather", "prelaunch_bcst"),
                                       ("alltoall", "prelaunch_swap")])
def test_arm_and_trigger(kind, impl):
    P.test_plan_arm_and_trigger(kind, impl)


def test_explicit_plan_rearms_and_cancels():
    P.test_explicit_prelaunch_plan_rearms_and_cancels()
