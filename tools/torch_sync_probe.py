"""Control for tools/thread_sync_probe.py without this library: one thread
synchronises the device in a loop while another replays a CUDA graph holding
a kernel (mode graph) or launches kernels eagerly (mode eager)."""
import faulthandler
import sys
import threading

faulthandler.enable(all_threads=True)
import torch

mode = sys.argv[1] if len(sys.argv) > 1 else "graph"
x = torch.zeros(1 << 20, device="cuda")
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    x.add_(1)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    x.add_(1)
torch.cuda.synchronize()
for rep in range(6):
    done = threading.Event()

    def syncer():
        while not done.is_set():
            torch.cuda.synchronize()

    def runner():
        with torch.cuda.stream(s):
            for _ in range(2000):
                if mode == "graph":
                    g.replay()
                elif mode == "capturing":
                    for _ in range(20):
                        torch.cuda.is_current_stream_capturing()  # cudaStreamIsCapturing
                    x.add_(1)
                else:
                    x.add_(1)
        s.synchronize()
        done.set()

    ts = [threading.Thread(target=syncer), threading.Thread(target=runner)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    print(f"rep {rep} ok", flush=True)
print("done", flush=True)
