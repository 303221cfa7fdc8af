// Host cost of a kernel launch: triple-chevron vs cudaLaunchKernel with the
// same kernel and arguments (the KernelCall path of csrc/kernels.cu), and the
// cost of cudaGetDevice / cudaStreamIsCapturing / cudaGetLastError.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -cudart static tools/launch_probe.cu -o tools/launch_probe
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>

struct Big {
  void* p[12];
  int x[4];
};

__global__ void k_small(const int* a, int n, int m, int e, Big f) {
  if (threadIdx.x == 0 && n < 0) printf("%d %d %d %p\n", m, e, f.x[0], a);
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  Big f = {};
  int n = 1, m = 2, e = 3;
  const int* a = nullptr;
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) k_small<<<32, 32, 0, s>>>(a, n, m, e, f);
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    void* args[] = {&a, &n, &m, &e, &f};
    auto t2 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i)
      cudaLaunchKernel(reinterpret_cast<const void*>(k_small), dim3(32), dim3(32), args, 0, s);
    auto t3 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    int dev;
    auto t4 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) cudaGetDevice(&dev);
    auto t5 = std::chrono::steady_clock::now();
    cudaStreamCaptureStatus cs;
    for (int i = 0; i < iters; ++i) cudaStreamIsCapturing(s, &cs);
    auto t6 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) cudaGetLastError();
    auto t7 = std::chrono::steady_clock::now();
    auto us = [&](auto a_, auto b_) { return std::chrono::duration<double, std::micro>(b_ - a_).count() / iters; };
    std::printf("chevron %.3f us  cudaLaunchKernel %.3f us  cudaGetDevice %.3f us  IsCapturing %.3f us  "
                "GetLastError %.3f us\n", us(t0, t1), us(t2, t3), us(t4, t5), us(t5, t6), us(t6, t7));
  }
  return 0;
}
