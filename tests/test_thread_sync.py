"""Recording is crash-free under a concurrent device synchronisation.

Round 1 recorded command lists by stream capture, and a cudaDeviceSynchronize
from another thread during a capture crashed inside the CUDA runtime
(DESIGN.md §3.2). Graphs are now built node by node (csrc/sink.cpp GraphSink),
so no stream is ever in capture mode. tools/thread_sync_probe.py runs cold —
every plan is recorded for the first time inside the race, 10 fresh worlds
per run — while another thread synchronises the device in a loop; every
result is checked (the reference arm of the SPEC: programs are values shared
across threads, sweep.cpp:113-124).
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.timeout(900)
@pytest.mark.parametrize("impls", ["pcpy", "b2b", "hybrid,pull", "sm", "prelaunch_pcpy,prelaunch_b2b"])
def test_cold_recording_races_device_synchronize(impls):
    env = dict(os.environ)
    env.pop("PROBE_WARM", None)
    env.pop("PROBE_SYNC", None)
    r = subprocess.run([sys.executable, "-X", "faulthandler", os.path.join(ROOT, "tools", "thread_sync_probe.py"),
                        "10", impls], cwd=ROOT, env=env, capture_output=True, text=True, timeout=800)
    assert r.returncode == 0, (r.returncode, r.stdout[-3000:], r.stderr[-3000:])
    assert r.stdout.count("parity=True") == 10, r.stdout[-3000:]
