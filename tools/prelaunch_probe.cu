// Floor of the prelaunch trigger protocol on one B200, without the library:
// what a caller stream pays per back-to-back collective when the mover is
// (a) launched on the caller stream (the `sm` path), (b) a gated graph
// (gate kernel -> mover, caller: memop write + event wait, the two-kernel
// body), (c) a gated graph whose completion is a done word (caller: memop
// write + memop wait), (d) a self-gated mover (one kernel: CTA 0 polls the
// ready word, the others wait on CTA 0), (e) a persistent mover that serves
// every trigger of the run (the trigger -> observe -> move -> signal ->
// observe floor). 64 chunks of CHUNK bytes are copied per collective.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/prelaunch_probe.cu -o tools/prelaunch_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
      std::exit(1);                                                                      \
    }                                                                                    \
  } while (0)
#define CD(x)                                                        \
  do {                                                               \
    CUresult r_ = (x);                                               \
    if (r_ != CUDA_SUCCESS) {                                        \
      std::printf("CU %d at %s:%d\n", int(r_), __FILE__, __LINE__);  \
      std::exit(1);                                                  \
    }                                                                \
  } while (0)

constexpr int kChunks = 64;

__device__ __forceinline__ uint64_t ld_acq(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// every CTA copies its share of the chunks (int4 granularity)
__device__ __forceinline__ void move(const int4* src, int4* dst, size_t nvec) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec; i += stride) dst[i] = src[i];
}

__global__ void mover(const int4* src, int4* dst, size_t nvec) { move(src, dst, nvec); }

// last CTA (ticket) writes *done = epoch
__device__ __forceinline__ void finish(unsigned* ctr, uint64_t* done, uint64_t epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    const unsigned t = atomicAdd(ctr, 1u);
    if (t == gridDim.x - 1) {
      *ctr = 0;
      st_rel(done, epoch);
    }
  }
}

__global__ void mover_done(const int4* src, int4* dst, size_t nvec, unsigned* ctr, uint64_t* done,
                           uint64_t* epoch_ctr) {
  move(src, dst, nvec);
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    const unsigned t = atomicAdd(ctr, 1u);
    if (t == gridDim.x - 1) {
      *ctr = 0;
      const uint64_t e = *epoch_ctr + 1;
      *epoch_ctr = e;
      st_rel(done, e);
    }
  }
}

__global__ void gate(uint64_t* ready) {
  if (threadIdx.x == 0) {
    while (ld_acq(ready) < 1) __nanosleep(32);
    *ready = 0;
  }
}

// self-gated: CTA 0 takes the ready word, publishes it in a device word
__global__ void folded(const int4* src, int4* dst, size_t nvec, uint64_t* ready, uint64_t* go, uint64_t* go_seen,
                       unsigned* ctr, uint64_t* done, uint64_t* epoch_ctr) {
  __shared__ uint64_t e;
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      while (ld_acq(ready) < 1) __nanosleep(32);
      *ready = 0;
      const uint64_t n = *epoch_ctr + 1;
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(go), "l"(n) : "memory");
      e = n;
    } else {
      const uint64_t want = *go_seen + 1;  // instances run one at a time
      uint64_t v;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(go) : "memory");
      } while (v < want);
      e = v;
    }
  }
  __syncthreads();
  move(src, dst, nvec);
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    const unsigned t = atomicAdd(ctr, 1u);
    if (t == gridDim.x - 1) {
      *ctr = 0;
      *epoch_ctr = e;
      *go_seen = e;
      st_rel(done, e);
    }
  }
}

// persistent: serves `iters` triggers; trigger k writes ready = k
__global__ void persistent(const int4* src, int4* dst, size_t nvec, const uint64_t* ready, uint64_t* go,
                           unsigned* ctr, uint64_t* done, int iters) {
  __shared__ int dummy;
  for (int k = 1; k <= iters; ++k) {
    if (threadIdx.x == 0) {
      if (blockIdx.x == 0) {
        while (ld_acq(ready) < uint64_t(k)) {
        }
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(go), "l"(uint64_t(k)) : "memory");
      } else {
        uint64_t v;
        do {
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(go) : "memory");
        } while (v < uint64_t(k));
      }
      dummy = k;
    }
    __syncthreads();
    move(src, dst, nvec);
    finish(ctr, done, uint64_t(k));
  }
  (void)dummy;
}


// ---- small-collective mover variants: 64 items of CHUNK bytes, one CTA per
// item; the item table in global memory (one dependent load) or in the
// kernel's parameter space.
struct ProbeItem {
  const char* src;
  char* dst;
  long long bytes;
};
struct ParamTable {
  ProbeItem it[kChunks];
};

__global__ void table_mover(const ProbeItem* items) {
  const ProbeItem it = items[blockIdx.x];
  const int4* s = reinterpret_cast<const int4*>(it.src);
  int4* d = reinterpret_cast<int4*>(it.dst);
  for (long long i = threadIdx.x; i < it.bytes / 16; i += blockDim.x) d[i] = s[i];
}

__global__ void param_mover(const __grid_constant__ ParamTable t) {
  const ProbeItem& it = t.it[blockIdx.x];
  const int4* s = reinterpret_cast<const int4*>(it.src);
  int4* d = reinterpret_cast<int4*>(it.dst);
  for (long long i = threadIdx.x; i < it.bytes / 16; i += blockDim.x) d[i] = s[i];
}

// one warp, TMA bulk load -> mbarrier -> bulk store -> wait_group 0
__global__ void tma_param_mover(const __grid_constant__ ParamTable t) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x != 0) return;
  const ProbeItem& it = t.it[blockIdx.x];
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  const uint32_t r = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint32_t bytes = static_cast<uint32_t>(it.bytes);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(r),
               "l"(it.src), "r"(bytes), "r"(b)
               : "memory");
  asm volatile("{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(b),
               "r"(0)
               : "memory");
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(it.dst), "r"(r), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// (k)-(m): the library TMA mover's ingredients added one at a time to (i):
// template flags: table in global memory, createpolicy + L2 cache hints,
// a 4-stage mbarrier ring with 128 KiB of dynamic shared memory.
template <bool kGlobal, bool kHint, bool kRing>
__global__ void tma_variant(const __grid_constant__ ParamTable t, const ProbeItem* items) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t bars[4];
  if (threadIdx.x != 0) return;
  const ProbeItem it = kGlobal ? items[blockIdx.x] : t.it[blockIdx.x];
  const int nb = kRing ? 4 : 1;
  for (int i = 0; i < nb; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bars[i]))));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bars[0]));
  const uint32_t r = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const uint32_t bytes = static_cast<uint32_t>(it.bytes);
  uint64_t policy = 0;
  if (kHint) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(policy));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  if (kHint)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(r),
                 "l"(it.src), "r"(bytes), "r"(b), "l"(policy)
                 : "memory");
  else
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(r),
                 "l"(it.src), "r"(bytes), "r"(b)
                 : "memory");
  asm volatile("{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(b),
               "r"(0)
               : "memory");
  if (kHint)
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(it.dst), "r"(r),
                 "r"(bytes), "l"(policy)
                 : "memory");
  else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(it.dst), "r"(r), "r"(bytes)
                 : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const size_t chunk = argc > 1 ? std::strtoull(argv[1], nullptr, 0) : 4096;
  const int iters = argc > 2 ? std::atoi(argv[2]) : 2000;
  const int grid = argc > 3 ? std::atoi(argv[3]) : 16;
  CK(cudaSetDevice(0));
  CD(cuInit(0));
  const size_t bytes = chunk * kChunks;
  const size_t nvec = bytes / 16;
  int4 *src, *dst;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMalloc(&dst, bytes));
  uint64_t* words;  // ready, done, go, epoch, go_seen, ctr...
  CK(cudaMalloc(&words, 4096));
  CK(cudaMemset(words, 0, 4096));
  uint64_t* ready = words + 0;
  uint64_t* done = words + 8;
  uint64_t* go = words + 16;
  uint64_t* epoch = words + 24;
  uint64_t* go_seen = words + 32;
  unsigned* ctr = reinterpret_cast<unsigned*>(words + 40);
  cudaStream_t cs, as;
  CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&as, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, gdone;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreateWithFlags(&gdone, cudaEventDisableTiming));

  auto reset = [&] {
    CK(cudaDeviceSynchronize());
    CK(cudaMemset(words, 0, 4096));
    CK(cudaDeviceSynchronize());
  };
  auto report = [&](const char* name, double host_us) {
    float ms = 0;
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::printf("%-44s chunk %8zu grid %3d  device %7.2f us/coll  host %6.2f us/call\n", name, chunk, grid,
                ms * 1e3 / iters, host_us);
  };
  using clk = std::chrono::steady_clock;
  auto hus = [&](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double, std::micro>(b - a).count() / iters;
  };

  // (a) mover on the caller stream
  for (int rep = 0; rep < 2; ++rep) {
    reset();
    CK(cudaEventRecord(e0, cs));
    auto t0 = clk::now();
    for (int i = 0; i < iters; ++i) mover<<<grid, 512, 0, cs>>>(src, dst, nvec);
    auto t1 = clk::now();
    CK(cudaEventRecord(e1, cs));
    if (rep) report("(a) sm: mover on caller stream", hus(t0, t1));
  }
  // (a') the same as a one-node graph
  {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(as, cudaStreamCaptureModeRelaxed));
    mover<<<grid, 512, 0, as>>>(src, dst, nvec);
    CK(cudaStreamEndCapture(as, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int rep = 0; rep < 2; ++rep) {
      reset();
      CK(cudaEventRecord(e0, cs));
      auto t0 = clk::now();
      for (int i = 0; i < iters; ++i) CK(cudaGraphLaunch(ge, cs));
      auto t1 = clk::now();
      CK(cudaEventRecord(e1, cs));
      if (rep) report("(a') sm: one-node graph on caller stream", hus(t0, t1));
    }
  }
  // (g)/(h)/(i): small-collective movers as one-node graphs (caller stream)
  {
    ParamTable pt;
    for (int i = 0; i < kChunks; ++i)
      pt.it[i] = {reinterpret_cast<const char*>(src) + i * chunk, reinterpret_cast<char*>(dst) + i * chunk,
                  static_cast<long long>(chunk)};
    ProbeItem* dtab;
    CK(cudaMalloc(&dtab, sizeof(pt)));
    CK(cudaMemcpy(dtab, &pt, sizeof(pt), cudaMemcpyHostToDevice));
    const int smem = static_cast<int>(chunk);
    CK(cudaFuncSetAttribute(tma_param_mover, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int variant = 0; variant < 4; ++variant) {
      if (variant >= 2 && chunk > 128 * 1024) continue;
      cudaGraph_t g;
      cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(as, cudaStreamCaptureModeRelaxed));
      if (variant == 0) table_mover<<<kChunks, 256, 0, as>>>(dtab);
      if (variant == 1) param_mover<<<kChunks, 256, 0, as>>>(pt);
      if (variant == 2) tma_param_mover<<<kChunks, 32, smem, as>>>(pt);
      if (variant == 3) tma_param_mover<<<kChunks, 32, 128 * 1024, as>>>(pt);
      CK(cudaStreamEndCapture(as, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      for (int rep = 0; rep < 2; ++rep) {
        reset();
        CK(cudaEventRecord(e0, cs));
        auto t0 = clk::now();
        for (int i = 0; i < iters; ++i) CK(cudaGraphLaunch(ge, cs));
        auto t1 = clk::now();
        CK(cudaEventRecord(e1, cs));
        if (rep)
          report(variant == 0   ? "(g) table in global, 1 CTA/item"
                 : variant == 1 ? "(h) table in params, 1 CTA/item"
                 : variant == 2 ? "(i) TMA, table in params, 1 warp/item"
                                : "(j) as (i) with 128 KiB dynamic smem",
                 hus(t0, t1));
      }
    }
    // (k)-(m)
    {
      auto kk = tma_variant<true, false, false>;
      auto kl = tma_variant<true, true, false>;
      auto km = tma_variant<true, true, true>;
      CK(cudaFuncSetAttribute(km, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024));
      for (int variant = 0; variant < 3 && chunk <= 32 * 1024; ++variant) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(as, cudaStreamCaptureModeRelaxed));
        if (variant == 0) kk<<<kChunks, 32, smem, as>>>(pt, dtab);
        if (variant == 1) kl<<<kChunks, 32, smem, as>>>(pt, dtab);
        if (variant == 2) km<<<kChunks, 32, 128 * 1024, as>>>(pt, dtab);
        CK(cudaStreamEndCapture(as, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        for (int rep = 0; rep < 2; ++rep) {
          reset();
          CK(cudaEventRecord(e0, cs));
          auto t0 = clk::now();
          for (int i = 0; i < iters; ++i) CK(cudaGraphLaunch(ge, cs));
          auto t1 = clk::now();
          CK(cudaEventRecord(e1, cs));
          if (rep)
            report(variant == 0   ? "(k) (i) + table in global"
                   : variant == 1 ? "(l) (k) + L2 cache hints"
                                  : "(m) (l) + 4 mbarriers, 128 KiB smem",
                   hus(t0, t1));
        }
      }
    }
  }
  // (b) gated graph: gate -> mover on the arm stream; caller writes ready,
  // waits on the graph's completion event. (c) same, caller waits on the
  // mover's done word with a memop.
  for (int variant = 0; variant < 2; ++variant) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(as, cudaStreamCaptureModeRelaxed));
    gate<<<1, 32, 0, as>>>(ready);
    if (variant == 0) mover<<<grid, 512, 0, as>>>(src, dst, nvec);
    else mover_done<<<grid, 512, 0, as>>>(src, dst, nvec, ctr, done, epoch);
    CK(cudaStreamEndCapture(as, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int rep = 0; rep < 2; ++rep) {
      reset();
      CK(cudaGraphLaunch(ge, as));  // armed instance 1
      CK(cudaEventRecord(gdone, as));
      CK(cudaEventRecord(e0, cs));
      auto t0 = clk::now();
      for (int i = 0; i < iters; ++i) {
        CD(cuStreamWriteValue64(cs, reinterpret_cast<CUdeviceptr>(ready), 1, 0));
        if (variant == 0) {
          CK(cudaStreamWaitEvent(cs, gdone, 0));
        } else {
          CD(cuStreamWaitValue64(cs, reinterpret_cast<CUdeviceptr>(done), uint64_t(i + 1), CU_STREAM_WAIT_VALUE_GEQ));
        }
        if (i + 1 < iters) {
          CK(cudaGraphLaunch(ge, as));  // re-arm (queued behind the running instance)
          CK(cudaEventRecord(gdone, as));
        }
      }
      auto t1 = clk::now();
      CK(cudaEventRecord(e1, cs));
      if (rep)
        report(variant == 0 ? "(b) gate->mover graph, event wait" : "(c) gate->mover graph, done-word memop wait",
               hus(t0, t1));
    }
  }
  // (b2) two gated graphs alternating on two arm streams (own ready words):
  // the instance for collective i+1 is already spinning while i runs.
  {
    cudaStream_t as2;
    CK(cudaStreamCreateWithFlags(&as2, cudaStreamNonBlocking));
    cudaStream_t arm[2] = {as, as2};
    uint64_t* rdy[2] = {ready, words + 48};
    cudaEvent_t gd[2];
    CK(cudaEventCreateWithFlags(&gd[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&gd[1], cudaEventDisableTiming));
    cudaGraphExec_t ge[2];
    for (int k = 0; k < 2; ++k) {
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(arm[k], cudaStreamCaptureModeRelaxed));
      gate<<<1, 32, 0, arm[k]>>>(rdy[k]);
      mover<<<grid, 512, 0, arm[k]>>>(src, dst, nvec);
      CK(cudaStreamEndCapture(arm[k], &g));
      CK(cudaGraphInstantiate(&ge[k], g, 0));
    }
    for (int rep = 0; rep < 2; ++rep) {
      reset();
      for (int k = 0; k < 2; ++k) {
        CK(cudaGraphLaunch(ge[k], arm[k]));
        CK(cudaEventRecord(gd[k], arm[k]));
      }
      CK(cudaEventRecord(e0, cs));
      auto t0 = clk::now();
      for (int i = 0; i < iters; ++i) {
        const int k = i & 1;
        CD(cuStreamWriteValue64(cs, reinterpret_cast<CUdeviceptr>(rdy[k]), 1, 0));
        CK(cudaStreamWaitEvent(cs, gd[k], 0));
        if (i + 2 < iters) {
          CK(cudaGraphLaunch(ge[k], arm[k]));
          CK(cudaEventRecord(gd[k], arm[k]));
        }
      }
      auto t1 = clk::now();
      CK(cudaEventRecord(e1, cs));
      if (rep) report("(b2) two gated graphs alternating", hus(t0, t1));
    }
  }
  // (d) self-gated mover (one kernel per collective), caller memop write +
  // memop wait
  for (int rep = 0; rep < 2; ++rep) {
    reset();
    folded<<<grid, 512, 0, as>>>(src, dst, nvec, ready, go, go_seen, ctr, done, epoch);
    CK(cudaEventRecord(e0, cs));
    auto t0 = clk::now();
    for (int i = 0; i < iters; ++i) {
      CD(cuStreamWriteValue64(cs, reinterpret_cast<CUdeviceptr>(ready), 1, 0));
      CD(cuStreamWaitValue64(cs, reinterpret_cast<CUdeviceptr>(done), uint64_t(i + 1), CU_STREAM_WAIT_VALUE_GEQ));
      if (i + 1 < iters) folded<<<grid, 512, 0, as>>>(src, dst, nvec, ready, go, go_seen, ctr, done, epoch);
    }
    auto t1 = clk::now();
    CK(cudaEventRecord(e1, cs));
    if (rep) report("(d) self-gated mover, memop write + wait", hus(t0, t1));
  }
  // (e) persistent mover serving every trigger
  for (int rep = 0; rep < 2; ++rep) {
    reset();
    persistent<<<grid, 512, 0, as>>>(src, dst, nvec, ready, go, ctr, done, iters);
    CK(cudaEventRecord(e0, cs));
    auto t0 = clk::now();
    for (int i = 0; i < iters; ++i) {
      CD(cuStreamWriteValue64(cs, reinterpret_cast<CUdeviceptr>(ready), uint64_t(i + 1), 0));
      CD(cuStreamWaitValue64(cs, reinterpret_cast<CUdeviceptr>(done), uint64_t(i + 1), CU_STREAM_WAIT_VALUE_GEQ));
    }
    auto t1 = clk::now();
    CK(cudaEventRecord(e1, cs));
    if (rep) report("(e) persistent mover, memop write + wait", hus(t0, t1));
  }
  // (f) memop round trip alone: write ready, a persistent one-CTA echo
  // kernel copies it to done -- no data
  CK(cudaDeviceSynchronize());
  std::printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
