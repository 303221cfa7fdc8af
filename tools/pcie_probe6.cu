// PCIe duplex floor of the e2e leg (512 MiB host->device + 512 MiB
// device->host at once, one copy per direction) for different kinds of pinned
// host memory: cudaHostAlloc default, write-combined source, and
// transparent-huge-page memory registered with cudaHostRegister.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -cudart static tools/pcie_probe6.cu -o tools/pcie_probe6
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

static void* thp_alloc(size_t bytes) {
  void* p = nullptr;
  if (posix_memalign(&p, size_t(2) << 20, bytes) != 0) return nullptr;
  madvise(p, bytes, MADV_HUGEPAGE);
  std::memset(p, 1, bytes);
  if (cudaHostRegister(p, bytes, cudaHostRegisterDefault) != cudaSuccess) return nullptr;
  return p;
}

int main() {
  const size_t bytes = size_t(512) << 20;
  void *d_in, *d_out;
  cudaMalloc(&d_in, bytes);
  cudaMalloc(&d_out, bytes);
  cudaMemset(d_out, 1, bytes);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, ea, eb;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&ea);
  cudaEventCreate(&eb);
  auto run = [&](const char* name, void* h_in, void* h_out, bool h2d, bool d2h) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, 0);
      cudaStreamWaitEvent(a, e0, 0);
      cudaStreamWaitEvent(b, e0, 0);
      if (h2d) cudaMemcpyAsync(d_in, h_in, bytes, cudaMemcpyHostToDevice, a);
      if (d2h) cudaMemcpyAsync(h_out, d_out, bytes, cudaMemcpyDeviceToHost, b);
      cudaEventRecord(ea, a);
      cudaEventRecord(eb, b);
      cudaStreamWaitEvent(0, ea, 0);
      cudaStreamWaitEvent(0, eb, 0);
      cudaEventRecord(e1, 0);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    std::printf("%-40s %8.3f ms\n", name, best);
  };
  void *p_in, *p_out, *wc_in, *thp_in, *thp_out;
  cudaHostAlloc(&p_in, bytes, cudaHostAllocDefault);
  cudaHostAlloc(&p_out, bytes, cudaHostAllocDefault);
  cudaHostAlloc(&wc_in, bytes, cudaHostAllocWriteCombined);
  std::memset(p_in, 1, bytes);
  std::memset(p_out, 1, bytes);
  std::memset(wc_in, 1, bytes);
  thp_in = thp_alloc(bytes);
  thp_out = thp_alloc(bytes);
  run("default: h2d", p_in, p_out, true, false);
  run("default: d2h", p_in, p_out, false, true);
  run("default: both", p_in, p_out, true, true);
  run("write-combined src: h2d", wc_in, p_out, true, false);
  run("write-combined src: both", wc_in, p_out, true, true);
  if (thp_in && thp_out) {
    run("thp registered: h2d", thp_in, thp_out, true, false);
    run("thp registered: d2h", thp_in, thp_out, false, true);
    run("thp registered: both", thp_in, thp_out, true, true);
  } else {
    std::printf("thp registration failed\n");
  }
  std::printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
