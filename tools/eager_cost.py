"""Start-up time and device memory of a process under the current
CUDA_MODULE_LOADING mode (torch init + the package's first collective)."""
import os
import sys
import time

t0 = time.time()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2511_06605_b200 as cc

x = torch.ones(1, device="cuda")
torch.cuda.synchronize()
t1 = time.time()
cs = cc.Comm.init_all([0, 0])
a = [torch.zeros(8192, dtype=torch.uint8, device="cuda") for _ in range(2)]
b = [torch.zeros(8192, dtype=torch.uint8, device="cuda") for _ in range(2)]
cc.all_to_all(cs, a, b, 4096, impl="pcpy")
torch.cuda.synchronize()
t2 = time.time()
free, total = torch.cuda.mem_get_info()
print(f"mode={os.environ.get('CUDA_MODULE_LOADING', 'LAZY(default)')} torch_init={t1 - t0:.2f}s "
      f"first_collective={t2 - t1:.2f}s device_used={(total - free) / 2**30:.2f} GiB", flush=True)
