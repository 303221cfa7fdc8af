// PCIe duplex with the SMs on one direction: host->device moved by a kernel
// that loads pinned host memory directly (zero-copy reads over PCIe) while a
// copy engine moves device->host, against both directions on copy engines
// (the e2e leg of bench.py: 512 MiB each way per step).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -cudart static tools/pcie_probe5.cu -o tools/pcie_probe5
#include <cuda_runtime.h>

#include <cstdio>

__global__ void __launch_bounds__(512) pull_kernel(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {  // four 16-byte loads in flight per thread
    int4 a = __ldg(src + i), b = __ldg(src + i + stride), c = __ldg(src + i + 2 * stride), d = __ldg(src + i + 3 * stride);
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = __ldg(src + i);
}

int main() {
  const size_t bytes = size_t(512) << 20;
  void *h_in, *h_out, *d_in, *d_out;
  cudaHostAlloc(&h_in, bytes, cudaHostAllocMapped);
  cudaHostAlloc(&h_out, bytes, cudaHostAllocMapped);
  cudaMalloc(&d_in, bytes);
  cudaMalloc(&d_out, bytes);
  cudaMemset(d_out, 1, bytes);
  for (size_t i = 0; i < bytes; i += 4096) static_cast<char*>(h_in)[i] = 1;
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, ea, eb;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&ea);
  cudaEventCreate(&eb);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const char* name, bool k_h2d, bool ce_h2d, bool ce_d2h, int grid) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, 0);
      cudaStreamWaitEvent(a, e0, 0);
      cudaStreamWaitEvent(b, e0, 0);
      if (k_h2d) pull_kernel<<<grid, 512, 0, a>>>(static_cast<const int4*>(h_in), static_cast<int4*>(d_in), bytes / 16);
      if (ce_h2d) cudaMemcpyAsync(d_in, h_in, bytes, cudaMemcpyHostToDevice, a);
      if (ce_d2h) cudaMemcpyAsync(h_out, d_out, bytes, cudaMemcpyDeviceToHost, b);
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
    std::printf("%-34s grid %4d  %8.3f ms  (%.1f GB/s per direction-equivalent)\n", name, grid, best,
                bytes / (best * 1e-3) / 1e9);
  };
  run("ce_h2d", false, true, false, 0);
  run("ce_d2h", false, false, true, 0);
  run("ce_both", false, true, true, 0);
  for (int g : {sms / 4, sms / 2, sms, 2 * sms}) {
    run("kernel_h2d (zero-copy loads)", true, false, false, g);
    run("kernel_h2d + ce_d2h", true, false, true, g);
  }
  const cudaError_t err = cudaGetLastError();
  std::printf("last error: %s\n", cudaGetErrorString(err));
  return 0;
}
