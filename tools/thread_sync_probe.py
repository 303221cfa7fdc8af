"""One thread synchronises the device in a loop while another runs eager
prelaunch collectives (tests/test_threads.py); repeated, with faulthandler.
Usage: python -X faulthandler tools/thread_sync_probe.py [reps] [impl]
PROBE_SYNC=stream: the other thread synchronises an idle stream instead.
PROBE_WARM=1: every plan is recorded (launched three times) before the race.
Exit status: 0 clean; 3 a thread hung; 4 an error or a parity failure; a
signal (e.g. -11) if the process crashed. tests/test_thread_sync.py runs it
cold (no warming) for the recorded and prelaunch implementations."""
import faulthandler
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.enable(all_threads=True)
import torch

import paper_2511_06605_b200 as cc

N, S = 4, 64 << 10
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
impls = sys.argv[2].split(",") if len(sys.argv) > 2 else ["prelaunch_pcpy", "prelaunch_b2b"]
for rep in range(reps):
    comms = cc.Comm.init_all([0] * N)
    sends = [torch.randint(0, 256, (N * S,), dtype=torch.uint8, device="cuda") for _ in range(N)]
    recvs = [torch.empty(N * S, dtype=torch.uint8, device="cuda") for _ in range(N)]
    stream = torch.cuda.Stream()
    if os.environ.get("PROBE_WARM") == "1":  # record every plan before the race
        for impl in impls:
            for _ in range(3):
                cc.all_to_all(comms, sends, recvs, S, impl=impl, streams=stream)
    torch.cuda.synchronize()
    done = threading.Event()
    errors = []

    other = torch.cuda.Stream()

    def syncer():
        while not done.is_set():
            if os.environ.get("PROBE_SYNC") == "stream":
                other.synchronize()
            else:
                torch.cuda.synchronize()

    def runner():
        try:
            for it in range(200):
                cc.all_to_all(comms, sends, recvs, S, impl=impls[it % len(impls)], streams=stream)
            stream.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))
        finally:
            done.set()

    ts = [threading.Thread(target=syncer), threading.Thread(target=runner)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=60)
    alive = any(t.is_alive() for t in ts)
    want = [torch.cat([sends[j][r * S:(r + 1) * S] for j in range(N)]) for r in range(N)]
    ok = all(torch.equal(r, w) for r, w in zip(recvs, want)) if not alive else None
    print(f"rep {rep}: alive={alive} errors={errors} parity={ok}", flush=True)
    if alive:
        faulthandler.dump_traceback(all_threads=True)
        os._exit(3)
    cc.destroy_all(comms)
    if errors or not ok:
        sys.exit(4)
print("done", flush=True)
