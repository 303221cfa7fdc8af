// Copy-engine probe for one B200 (sm_100a).
//
// Answers the questions SURVEY.md §7 "Hard parts" leaves open before the
// executor is designed: how many async engines the driver reports, how
// same-device D2D memcpy bandwidth scales with the number of concurrent
// streams, whether memcpy occupies SMs (it must not, for the offload claim),
// what a small CE copy and a stream flag round trip cost, and whether stream
// memory operations and cuMemcpyBatchAsync capture into CUDA graphs.
//
// Build: make -C tools ce_probe   Run (GPU box): tools/ce_probe
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
#define CU(x)                                                                       \
  do {                                                                              \
    CUresult r_ = (x);                                                              \
    if (r_ != CUDA_SUCCESS) {                                                       \
      const char* s_ = "?";                                                         \
      drv->GetErrorString(r_, &s_);                                                 \
      printf("CU error %d %s at %s:%d\n", (int)r_, s_, __FILE__, __LINE__);          \
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

__global__ void copy_v4(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    int4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  alarm(300);
  drv = driver_api();
  if (!drv) { printf("no driver\n"); return 1; }
  CK(cudaSetDevice(0));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int attrs[] = {CU_DEVICE_ATTRIBUTE_ASYNC_ENGINE_COUNT, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS,
                 CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED,
                 CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT,
                 CU_DEVICE_ATTRIBUTE_CAN_USE_HOST_POINTER_FOR_REGISTERED_MEM};
  const char* names[] = {"async_engine_count", "mem_ops_64", "flush_remote_writes", "multicast",
                         "wait_nor", "sm_count", "host_ptr_registered"};
  printf("device %s cc %d.%d\n", prop.name, prop.major, prop.minor);
  for (int i = 0; i < 7; ++i) {
    int v = -1;
    drv->DeviceGetAttribute(&v, (CUdevice_attribute)attrs[i], 0);
    printf("attr %s = %d\n", names[i], v);
  }
  const char* conn = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
  printf("CUDA_DEVICE_MAX_CONNECTIONS=%s batch_memcpy=%d\n", conn ? conn : "(unset)", (int)drv->has_batch_memcpy);

  const size_t total = 1ull << 30;
  char *src, *dst;
  CK(cudaMalloc(&src, total));
  CK(cudaMalloc(&dst, total));
  CK(cudaMemset(src, 1, total));
  CK(cudaMemset(dst, 0, total));
  std::vector<cudaStream_t> streams(64);
  for (auto& s : streams) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<cudaEvent_t> evs(64);
  for (auto& e : evs) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));

  // B. D2D memcpy bandwidth vs concurrent streams (1 GiB total).
  for (int k : {1, 2, 4, 7, 8, 14, 16, 32, 56}) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0, streams[0]));
      for (int i = 1; i < k; ++i) CK(cudaStreamWaitEvent(streams[i], e0));
      size_t per = total / k / 4096 * 4096;
      for (int i = 0; i < k; ++i)
        CK(cudaMemcpyAsync(dst + i * per, src + i * per, per, cudaMemcpyDeviceToDevice, streams[i]));
      for (int i = 1; i < k; ++i) {
        CK(cudaEventRecord(evs[i], streams[i]));
        CK(cudaStreamWaitEvent(streams[0], evs[i]));
      }
      CK(cudaEventRecord(e1, streams[0]));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    size_t per = total / k / 4096 * 4096;
    printf("memcpy_d2d streams=%d bytes=%zu ms=%.4f GBps(rd+wr)=%.1f\n", k, per * k, best,
           2.0 * per * k / best / 1e6);
  }

  // D. SM copy kernel bandwidth.
  for (int blocks : {148, 296, 592, 1184}) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(e0, streams[0]));
      copy_v4<<<blocks, 512, 0, streams[0]>>>((const int4*)src, (int4*)dst, total / 16);
      CK(cudaEventRecord(e1, streams[0]));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    printf("sm_copy blocks=%d ms=%.4f GBps(rd+wr)=%.1f\n", blocks, best, 2.0 * total / best / 1e6);
  }

  // C. Does memcpy need SMs? Spin all SMs for 50 ms, memcpy 256 MiB concurrently.
  {
    CK(cudaDeviceSynchronize());
    cudaEvent_t m0, m1;
    CK(cudaEventCreate(&m0));
    CK(cudaEventCreate(&m1));
    spin_kernel<<<prop.multiProcessorCount * 8, 1024, 0, streams[1]>>>(50000000LL);
    usleep(5000);
    CK(cudaEventRecord(m0, streams[2]));
    CK(cudaMemcpyAsync(dst, src, 256 << 20, cudaMemcpyDeviceToDevice, streams[2]));
    CK(cudaEventRecord(m1, streams[2]));
    CK(cudaEventRecord(e1, streams[1]));
    CK(cudaDeviceSynchronize());
    float ms_copy, ms_spin_to_copy;
    CK(cudaEventElapsedTime(&ms_copy, m0, m1));
    CK(cudaEventElapsedTime(&ms_spin_to_copy, m1, e1));
    printf("memcpy_under_full_sm_spin ms=%.4f (copy finished %.2f ms before spin end; CE if >0)\n", ms_copy,
           ms_spin_to_copy);
  }

  // E. Small copy latency: back-to-back 4 KiB memcpys on one stream.
  for (size_t sz : {4096ul, 65536ul, 1048576ul}) {
    const int iters = 1000;
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0, streams[0]));
    double h0 = now_us();
    for (int i = 0; i < iters; ++i)
      CK(cudaMemcpyAsync(dst, src, sz, cudaMemcpyDeviceToDevice, streams[0]));
    double h1 = now_us();
    CK(cudaEventRecord(e1, streams[0]));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("memcpy_serial size=%zu gpu_us_per=%.3f host_us_per_submit=%.3f\n", sz, ms * 1000 / iters,
           (h1 - h0) / iters);
    CK(cudaEventRecord(e0, streams[0]));
    for (int i = 0; i < iters; ++i)
      copy_v4<<<(unsigned)((sz / 16 + 511) / 512), 512, 0, streams[0]>>>((const int4*)src, (int4*)dst, sz / 16);
    CK(cudaEventRecord(e1, streams[0]));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("kernel_serial size=%zu gpu_us_per=%.3f\n", sz, ms * 1000 / iters);
  }

  // Flags: ping-pong between two streams with write/wait value.
  uint64_t* flags;
  CK(cudaMalloc(&flags, 4096));
  CK(cudaMemset(flags, 0, 4096));
  {
    CUdeviceptr fa = (CUdeviceptr)flags, fb = (CUdeviceptr)(flags + 8);
    const int iters = 1000;
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0, streams[0]));
    CK(cudaStreamWaitEvent(streams[1], e0));
    for (int i = 1; i <= iters; ++i) {
      CU(drv->StreamWriteValue64((CUstream)streams[0], fa, i, 0));
      CU(drv->StreamWaitValue64((CUstream)streams[1], fa, i, CU_STREAM_WAIT_VALUE_GEQ));
      CU(drv->StreamWriteValue64((CUstream)streams[1], fb, i, 0));
      CU(drv->StreamWaitValue64((CUstream)streams[0], fb, i, CU_STREAM_WAIT_VALUE_GEQ));
    }
    CK(cudaEventRecord(e1, streams[0]));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("flag_pingpong round_trip_us=%.3f\n", ms * 1000 / iters);
  }
  // memcpy + writeValue on lane, waitValue on main, repeated (one pcpy lane).
  for (size_t sz : {4096ul, 1048576ul}) {
    CUdeviceptr fa = (CUdeviceptr)(flags + 16);
    CK(cudaMemset(flags, 0, 4096));
    const int iters = 500;
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0, streams[0]));
    for (int i = 1; i <= iters; ++i) {
      CK(cudaEventRecord(evs[0], streams[0]));
      CK(cudaStreamWaitEvent(streams[1], evs[0]));
      CK(cudaMemcpyAsync(dst, src, sz, cudaMemcpyDeviceToDevice, streams[1]));
      CU(drv->StreamWriteValue64((CUstream)streams[1], fa, i, 0));
      CU(drv->StreamWaitValue64((CUstream)streams[0], fa, i, CU_STREAM_WAIT_VALUE_GEQ));
    }
    CK(cudaEventRecord(e1, streams[0]));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("lane_copy_signal size=%zu us_per=%.3f\n", sz, ms * 1000 / iters);
  }

  // F. batch memcpy vs 7 memcpys.
  if (drv->has_batch_memcpy) {
    for (size_t sz : {4096ul, 262144ul, 8388608ul}) {
      std::vector<CUdeviceptr> d(7), s(7);
      std::vector<size_t> sizes(7, sz);
      for (int i = 0; i < 7; ++i) {
        d[i] = (CUdeviceptr)(dst + i * sz * 2);
        s[i] = (CUdeviceptr)(src + i * sz * 2);
      }
      CUmemcpyAttributes attr = {};
      attr.srcAccessOrder = CU_MEMCPY_SRC_ACCESS_ORDER_STREAM;
      attr.flags = CU_MEMCPY_FLAG_PREFER_OVERLAP_WITH_COMPUTE;
      size_t idx = 0, fail = 0;
      const int iters = 300;
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0, streams[0]));
      double h0 = now_us();
      for (int i = 0; i < iters; ++i)
        CU(drv->MemcpyBatchAsync(d.data(), s.data(), sizes.data(), 7, &attr, &idx, 1, &fail,
                                 (CUstream)streams[0]));
      double h1 = now_us();
      CK(cudaEventRecord(e1, streams[0]));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("batch7 size=%zu gpu_us_per=%.3f host_us_per=%.3f GBps(rd+wr)=%.1f\n", sz, ms * 1000 / iters,
             (h1 - h0) / iters, 2.0 * 7 * sz * iters / ms / 1e6);
      CK(cudaEventRecord(e0, streams[0]));
      h0 = now_us();
      for (int i = 0; i < iters; ++i)
        for (int j = 0; j < 7; ++j)
          CK(cudaMemcpyAsync((void*)d[j], (void*)s[j], sz, cudaMemcpyDeviceToDevice, streams[0]));
      h1 = now_us();
      CK(cudaEventRecord(e1, streams[0]));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("serial7 size=%zu gpu_us_per=%.3f host_us_per=%.3f GBps(rd+wr)=%.1f\n", sz, ms * 1000 / iters,
             (h1 - h0) / iters, 2.0 * 7 * sz * iters / ms / 1e6);
    }
  }

  // G. Graph capture of wait/write value + batch memcpy + memcpy.
  {
    CK(cudaMemset(flags, 0, 4096));
    cudaGraph_t g;
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    CK(cudaStreamBeginCapture(streams[3], mode));
    CUstreamBatchMemOpParams ops[2] = {};
    ops[0].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
    ops[0].waitValue.address = (CUdeviceptr)(flags + 32);
    ops[0].waitValue.value64 = 1;
    ops[0].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
    ops[1].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
    ops[1].writeValue.address = (CUdeviceptr)(flags + 32);
    ops[1].writeValue.value64 = 0;
    ops[1].writeValue.flags = 0;
    CUresult r1 = drv->StreamBatchMemOp((CUstream)streams[3], 2, ops, 0);
    CUresult r2 = CUDA_SUCCESS;
    if (drv->has_batch_memcpy) {
      CUdeviceptr d0 = (CUdeviceptr)dst, s0 = (CUdeviceptr)src;
      size_t sz = 4096, idx = 0, fail = 0;
      CUmemcpyAttributes attr = {};
      attr.srcAccessOrder = CU_MEMCPY_SRC_ACCESS_ORDER_STREAM;
      r2 = drv->MemcpyBatchAsync(&d0, &s0, &sz, 1, &attr, &idx, 1, &fail, (CUstream)streams[3]);
    }
    cudaError_t r3 = cudaMemcpyAsync(dst, src, 4096, cudaMemcpyDeviceToDevice, streams[3]);
    CUresult r4 = drv->StreamWriteValue64((CUstream)streams[3], (CUdeviceptr)(flags + 40), 7, 0);
    cudaError_t rc = cudaStreamEndCapture(streams[3], &g);
    printf("capture batchmemop=%d batchmemcpy=%d memcpy=%d writevalue=%d end=%s\n", (int)r1, (int)r2, (int)r3,
           (int)r4, cudaGetErrorString(rc));
    cudaGetLastError();
    if (rc == cudaSuccess) {
      cudaGraphExec_t ge;
      cudaError_t ri = cudaGraphInstantiate(&ge, g, 0);
      printf("instantiate=%s\n", cudaGetErrorString(ri));
      if (ri == cudaSuccess) {
        CK(cudaGraphLaunch(ge, streams[3]));
        usleep(1000);
        uint64_t one = 1;
        CK(cudaMemcpyAsync(flags + 32, &one, 8, cudaMemcpyHostToDevice, streams[4]));
        CK(cudaStreamSynchronize(streams[3]));
        uint64_t v[9];
        CK(cudaMemcpy(v, flags + 32, 72, cudaMemcpyDeviceToHost));
        printf("graph ran: trigger reset=%llu signal=%llu\n", (unsigned long long)v[0], (unsigned long long)v[8]);
        // Graph replay latency when triggered from the host.
        const int iters = 200;
        float tot = 0;
        for (int i = 0; i < iters; ++i) {
          CK(cudaGraphLaunch(ge, streams[3]));
          CK(cudaEventRecord(e0, streams[4]));
          CK(cudaMemcpyAsync(flags + 32, &one, 8, cudaMemcpyHostToDevice, streams[4]));
          CK(cudaEventRecord(e1, streams[3]));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          tot += ms;
        }
        printf("graph_triggered_latency_us=%.3f\n", tot * 1000 / iters);
      }
    }
  }
  // H. waitValue on pinned host memory, host-side trigger.
  {
    uint64_t* hflag;
    CK(cudaHostAlloc(&hflag, 4096, cudaHostAllocMapped));
    hflag[0] = 0;
    uint64_t* dflag;
    CK(cudaHostGetDevicePointer(&dflag, hflag, 0));
    CK(cudaDeviceSynchronize());
    const int iters = 200;
    double tot = 0;
    for (int i = 1; i <= iters; ++i) {
      CU(drv->StreamWaitValue64((CUstream)streams[5], (CUdeviceptr)dflag, i, CU_STREAM_WAIT_VALUE_GEQ));
      CK(cudaMemcpyAsync(dst, src, 4096, cudaMemcpyDeviceToDevice, streams[5]));
      CU(drv->StreamWriteValue64((CUstream)streams[5], (CUdeviceptr)(dflag + 8), i, 0));
      usleep(200);
      double t0 = now_us();
      __atomic_store_n(&hflag[0], (uint64_t)i, __ATOMIC_RELEASE);
      while (__atomic_load_n(&hflag[8], __ATOMIC_ACQUIRE) < (uint64_t)i) {
      }
      tot += now_us() - t0;
    }
    CK(cudaDeviceSynchronize());
    printf("host_trigger_copy_observe_us=%.3f\n", tot / iters);
  }
  printf("probe done\n");
  return 0;
}
