// Copy-engine probe, part 2: which same-device copy APIs run on a copy
// engine (finish while every SM is held by a spinning kernel) and which are
// driver SM kernels; plus device-side flag round-trip latency.
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <vector>
#include <unistd.h>

#include "../paper_2511_06605_b200/csrc/cu_driver.hpp"

using namespace cecoll;

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

static const DriverApi* drv;

__global__ void spin_kernel(long long ns) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > ns) break;
  }
}

// Two single-CTA kernels ping-pong through a flag pair in global memory.
__global__ void pingpong(volatile unsigned long long* mine, volatile unsigned long long* theirs, int iters,
                         int first, unsigned long long* out_ns) {
  if (threadIdx.x != 0) return;
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; ++i) {
    if (first) {
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(theirs), "l"((unsigned long long)i) : "memory");
      unsigned long long v;
      do { asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory"); } while (v < (unsigned long long)i);
    } else {
      unsigned long long v;
      do { asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory"); } while (v < (unsigned long long)i);
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(theirs), "l"((unsigned long long)i) : "memory");
    }
  }
  long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (first) *out_ns = (unsigned long long)(t1 - t0);
}

__global__ void empty_kernel() {}

typedef void (*copy_fn)(char* dst, const char* src, size_t bytes, cudaStream_t s);

static void test_under_spin(const char* name, copy_fn fn, char* dst, const char* src, size_t bytes,
                            cudaStream_t spin_s, cudaStream_t copy_s, int sms) {
  cudaEvent_t c0, c1, s1;
  CK(cudaEventCreate(&c0));
  CK(cudaEventCreate(&c1));
  CK(cudaEventCreate(&s1));
  // Alone first.
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(c0, copy_s));
  fn(dst, src, bytes, copy_s);
  CK(cudaEventRecord(c1, copy_s));
  CK(cudaDeviceSynchronize());
  float alone;
  CK(cudaEventElapsedTime(&alone, c0, c1));
  // Under a one-wave all-SM spin of 20 ms.
  spin_kernel<<<sms * 2, 1024, 0, spin_s>>>(20000000LL);
  CK(cudaEventRecord(s1, spin_s));
  usleep(2000);
  CK(cudaEventRecord(c0, copy_s));
  fn(dst, src, bytes, copy_s);
  CK(cudaEventRecord(c1, copy_s));
  CK(cudaDeviceSynchronize());
  float under, before_end;
  CK(cudaEventElapsedTime(&under, c0, c1));
  CK(cudaEventElapsedTime(&before_end, c1, s1));
  cudaError_t e = cudaGetLastError();
  printf("%-28s bytes=%zu alone_ms=%.4f (%.0f GB/s rd+wr) under_spin_ms=%.4f finished_before_spin_end_ms=%.3f -> %s %s\n",
         name, bytes, alone, 2.0 * bytes / alone / 1e6, under, before_end, before_end > 1.0 ? "COPY-ENGINE" : "SM",
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

static void f_memcpy(char* d, const char* s, size_t b, cudaStream_t st) {
  CK(cudaMemcpyAsync(d, s, b, cudaMemcpyDeviceToDevice, st));
}
static void f_memcpy_default(char* d, const char* s, size_t b, cudaStream_t st) {
  CK(cudaMemcpyAsync(d, s, b, cudaMemcpyDefault, st));
}
static void f_peer(char* d, const char* s, size_t b, cudaStream_t st) { CK(cudaMemcpyPeerAsync(d, 0, s, 0, b, st)); }
static void f_2d(char* d, const char* s, size_t b, cudaStream_t st) {
  size_t w = 1 << 20;
  CK(cudaMemcpy2DAsync(d, w, s, w, w, b / w, cudaMemcpyDeviceToDevice, st));
}
static void f_2d_pitched(char* d, const char* s, size_t b, cudaStream_t st) {
  size_t w = 1 << 20;
  CK(cudaMemcpy2DAsync(d, w + 4096, s, w + 4096, w, b / (w + 4096), cudaMemcpyDeviceToDevice, st));
}
static void batch_flags(char* d, const char* s, size_t b, cudaStream_t st, unsigned flags, int count) {
  std::vector<CUdeviceptr> dd(count), ss(count);
  std::vector<size_t> sz(count, b / count);
  for (int i = 0; i < count; ++i) {
    dd[i] = (CUdeviceptr)(d + i * (b / count));
    ss[i] = (CUdeviceptr)(s + i * (b / count));
  }
  CUmemcpyAttributes attr = {};
  attr.srcAccessOrder = CU_MEMCPY_SRC_ACCESS_ORDER_STREAM;
  attr.flags = flags;
  size_t idx = 0, fail = 0;
  CUresult r = drv->MemcpyBatchAsync(dd.data(), ss.data(), sz.data(), count, &attr, &idx, 1, &fail, (CUstream)st);
  if (r != CUDA_SUCCESS) printf("batch rc=%d\n", (int)r);
}
static void f_batch_overlap(char* d, const char* s, size_t b, cudaStream_t st) {
  batch_flags(d, s, b, st, CU_MEMCPY_FLAG_PREFER_OVERLAP_WITH_COMPUTE, 1);
}
static void f_batch_overlap7(char* d, const char* s, size_t b, cudaStream_t st) {
  batch_flags(d, s, b, st, CU_MEMCPY_FLAG_PREFER_OVERLAP_WITH_COMPUTE, 7);
}
static void f_batch_default(char* d, const char* s, size_t b, cudaStream_t st) { batch_flags(d, s, b, st, 0, 1); }

int main() {
  alarm(300);
  drv = driver_api();
  CK(cudaSetDevice(0));
  int sms = 148;
  const size_t bytes = 256ull << 20;
  char *src, *dst;
  CK(cudaMalloc(&src, 2 * bytes));
  CK(cudaMalloc(&dst, 2 * bytes));
  CK(cudaMemset(src, 3, 2 * bytes));
  cudaStream_t a, b;
  CK(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
  test_under_spin("cudaMemcpyAsync D2D", f_memcpy, dst, src, bytes, a, b, sms);
  test_under_spin("cudaMemcpyAsync Default", f_memcpy_default, dst, src, bytes, a, b, sms);
  test_under_spin("cudaMemcpyPeerAsync 0->0", f_peer, dst, src, bytes, a, b, sms);
  test_under_spin("cudaMemcpy2DAsync", f_2d, dst, src, bytes, a, b, sms);
  test_under_spin("cudaMemcpy2DAsync pitched", f_2d_pitched, dst, src, bytes, a, b, sms);
  test_under_spin("batch PREFER_OVERLAP x1", f_batch_overlap, dst, src, bytes, a, b, sms);
  test_under_spin("batch PREFER_OVERLAP x7", f_batch_overlap7, dst, src, bytes, a, b, sms);
  test_under_spin("batch default x1", f_batch_default, dst, src, bytes, a, b, sms);
  // Small sizes: does PREFER_OVERLAP change latency?
  for (size_t sz : {4096ul, 1ul << 20, 8ul << 20, 64ul << 20}) {
    test_under_spin("batch PREFER_OVERLAP small", f_batch_overlap, dst, src, sz, a, b, sms);
    test_under_spin("cudaMemcpy2DAsync small", f_2d, dst, src, sz < (1 << 20) ? (1 << 20) : sz, a, b, sms);
  }
  // Concurrency scaling of CE batch copies across streams (if CE).
  {
    std::vector<cudaStream_t> st(16);
    for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    std::vector<cudaEvent_t> ev(16);
    for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (int k : {1, 2, 4, 7, 8, 16}) {
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0, st[0]));
        for (int i = 1; i < k; ++i) CK(cudaStreamWaitEvent(st[i], e0));
        size_t per = (2 * bytes) / k / 4096 * 4096;
        for (int i = 0; i < k; ++i) f_batch_overlap(dst + i * per, src + i * per, per, st[i]);
        for (int i = 1; i < k; ++i) {
          CK(cudaEventRecord(ev[i], st[i]));
          CK(cudaStreamWaitEvent(st[0], ev[i]));
        }
        CK(cudaEventRecord(e1, st[0]));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
      }
      printf("batch_overlap streams=%d total=%zu ms=%.4f GBps(rd+wr)=%.1f\n", k, 2 * bytes, best,
             2.0 * 2 * bytes / best / 1e6);
    }
  }
  // Device-side flag ping-pong between two concurrently running kernels.
  {
    unsigned long long* flags;
    CK(cudaMalloc(&flags, 4096));
    CK(cudaMemset(flags, 0, 4096));
    unsigned long long* out;
    CK(cudaMallocManaged(&out, 8));
    const int iters = 10000;
    pingpong<<<1, 32, 0, a>>>(flags, flags + 16, iters, 1, out);
    pingpong<<<1, 32, 0, b>>>(flags + 16, flags, iters, 0, out);
    CK(cudaDeviceSynchronize());
    printf("kernel_flag_pingpong round_trip_ns=%.1f\n", (double)*out / iters);
  }
  // Empty kernel launch rate and latency.
  {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, a));
    auto h0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 2000; ++i) empty_kernel<<<1, 32, 0, a>>>();
    auto h1 = std::chrono::steady_clock::now();
    CK(cudaEventRecord(e1, a));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("empty_kernel gpu_us_per=%.3f host_us_per=%.3f\n", ms * 1000 / 2000,
           std::chrono::duration<double, std::micro>(h1 - h0).count() / 2000);
  }
  printf("probe2 done\n");
  return 0;
}
