// HBM ceilings for the SM all-gather's fan pattern (one read, n writes):
// is the fan mover (kernels.cu tma_items_kernel, kItemFan) below the copy
// peak because of the kernel or because HBM writes alone are slower?
//   tools/fan_probe [src_MiB] [fan]
// Variants, each timed best-of-5 with CUDA events on one stream:
//   write_st       : st.global.v4 zeros over the destination (256 thr/CTA)
//   write_tma      : bulk stores of one zeroed shared tile (1 thr/CTA)
//   read_ld        : ld.global.v4 over the source, xor-reduced
//   copy_tma       : TMA ring, one store per tile (fan = 1)
//   fan_tma<lag>   : TMA ring, `fan` stores per tile; lag 0 refills a stage
//                    after wait_group.read 0, lag 1 after wait_group.read 1
//   fan_st         : registers: one 16-byte load, `fan` 16-byte stores
// GB/s counts algorithmic bytes: reads + writes.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void write_st(int4* dst, int64_t n16) {
  const int4 z = make_int4(0, 0, 0, 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    __stcs(dst + i, z);
}

__global__ void read_ld(const int4* src, int64_t n16, int* sink) {
  int acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 v = __ldcs(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) *sink = acc;
}

template <int kTile>
__global__ void __launch_bounds__(32, 1) write_tma(char* dst, int64_t bytes) {
  extern __shared__ __align__(128) unsigned char tile[];
  for (int i = threadIdx.x; i < kTile / 16; i += 32) reinterpret_cast<int4*>(tile)[i] = make_int4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (threadIdx.x) return;
  const int64_t ntiles = bytes / kTile;
  int outstanding = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + t * kTile), "r"(sa(tile)),
                 "r"(kTile)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (++outstanding >= 8) asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// fan stores per tile; dst region f is dst + f * bytes.
template <int kStages, int kTile, int kLag>
__global__ void __launch_bounds__(32, 1) fan_tma(const char* src, char* dst, int64_t bytes, int fan, int64_t stride) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[kStages];
  if (threadIdx.x) return;
  for (int i = 0; i < kStages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t ntiles = bytes / kTile;
  const int mine = blockIdx.x < ntiles ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  auto off = [&](int k) { return (blockIdx.x + (int64_t)k * gridDim.x) * kTile; };
  auto load = [&](int st, int k) {
    const uint32_t bar = sa(&full[st]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kTile) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(ring + st * kTile)),
                 "l"(src + off(k)), "r"(kTile), "r"(bar)
                 : "memory");
  };
  int issued = 0;
  for (; issued < kStages && issued < mine; ++issued) load(issued, issued);
  uint32_t phase = 0;
  for (int k = 0; k < mine; ++k) {
    const int st = k % kStages;
    asm volatile("{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(
                     sa(&full[st])),
                 "r"((phase >> st) & 1u)
                 : "memory");
    phase ^= 1u << st;
    for (int f = 0; f < fan; ++f)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + f * stride + off(k)),
                   "r"(sa(ring + st * kTile)), "r"(kTile)
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (kLag == 0) {
      if (issued < mine) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        load(st, issued++);
      }
    } else {
      // refill the previous iteration's stage once its stores have read it
      if (k >= 1 && issued < mine) {
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        load((k - 1) % kStages, issued++);
      }
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void fan_st(const int4* src, int4* dst, int64_t n16, int fan) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 v = __ldcs(src + i);
    for (int f = 0; f < fan; ++f) __stcs(dst + f * n16 + i, v);
  }
}

template <typename F>
static double best_ms(F f) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  double best = 1e30;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  CK(cudaGetLastError());
  return best;
}

static void report(const char* name, int grid, double ms, double rd, double wr) {
  printf("%-28s grid %5d  %8.3f ms  %7.1f GB/s (rd %.0f MiB, wr %.0f MiB)\n", name, grid, ms, (rd + wr) / ms / 1e6,
         rd / 1048576.0, wr / 1048576.0);
}

static int64_t g_stride = 0;
static int g_mults[4] = {1, 2, 0, 0};
template <int kStages, int kTile, int kLag>
static void run_fan(const char* name, const char* src, char* dst, int64_t S, int fan, int sms) {
  const int smem = kStages * kTile;
  CK(cudaFuncSetAttribute(fan_tma<kStages, kTile, kLag>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fan_tma<kStages, kTile, kLag>, 32, smem));
  const int64_t stride = g_stride ? g_stride : S;
  for (int mult : g_mults) {
    if (!mult) continue;
    const int grid = sms * per * mult;
    const double ms = best_ms([&] { fan_tma<kStages, kTile, kLag><<<grid, 32, smem>>>(src, dst, S, fan, stride); });
    char buf[64];
    snprintf(buf, sizeof buf, "%s s%d t%dK x%d%s", name, kStages, kTile / 1024, per, g_stride ? " pad" : "");
    report(buf, grid, ms, (double)S, (double)S * fan);
  }
}

int main(int argc, char** argv) {
  const int64_t S = (argc > 1 ? atoll(argv[1]) : 512) << 20;
  const int fan = argc > 2 ? atoi(argv[2]) : 8;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  char *src, *dst;
  int* sink;
  CK(cudaMalloc(&src, S));
  CK(cudaMalloc(&dst, S * fan + 64 * 40960));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(src, 1, S));
  CK(cudaMemset(dst, 0, S * fan));
  printf("# fan_probe: src %lld MiB, fan %d, %d SMs\n", (long long)(S >> 20), fan, sms);
  const int64_t W = S * fan;
  for (int per : {4, 8}) {
    const int grid = sms * per;
    report("write_st", grid, best_ms([&] { write_st<<<grid, 256>>>((int4*)dst, W / 16); }), 0, (double)W);
    report("read_ld", grid, best_ms([&] { read_ld<<<grid, 256>>>((const int4*)src, S / 16, sink); }), (double)S, 0);
    report("copy_st (fan_st 1)", grid, best_ms([&] { fan_st<<<grid, 256>>>((const int4*)src, (int4*)dst, S / 16, 1); }),
           (double)S, (double)S);
    report("fan_st", grid, best_ms([&] { fan_st<<<grid, 256>>>((const int4*)src, (int4*)dst, S / 16, fan); }),
           (double)S, (double)W);
  }
  CK(cudaFuncSetAttribute(write_tma<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
  for (int per : {1, 2, 4}) {
    const int grid = sms * per;
    report("write_tma t32K", grid, best_ms([&] { write_tma<32768><<<grid, 32, 32768>>>(dst, W); }), 0, (double)W);
  }
  const int mode = argc > 3 ? atoi(argv[3]) : 0;
  if (mode == 0) {
    // copy (fan 1) for the same kernel family
    run_fan<4, 32768, 0>("copy_tma", src, dst, S, 1, sms);
    run_fan<4, 32768, 0>("fan_tma lag0", src, dst, S, fan, sms);
    run_fan<4, 32768, 1>("fan_tma lag1", src, dst, S, fan, sms);
    run_fan<2, 65536, 0>("fan_tma lag0", src, dst, S, fan, sms);
  }
  // tile / occupancy / wave matrix, contiguous and padded destination regions
  g_mults[0] = 1; g_mults[1] = 2; g_mults[2] = 3; g_mults[3] = 4;
  if (mode == 2) {  // the same matrix for plain copies (fan 1)
    run_fan<4, 8192, 1>("copy_tma lag1", src, dst, S, 1, sms);
    run_fan<2, 16384, 0>("copy_tma lag0", src, dst, S, 1, sms);
    run_fan<4, 16384, 1>("copy_tma lag1", src, dst, S, 1, sms);
    run_fan<4, 32768, 0>("copy_tma lag0", src, dst, S, 1, sms);
    run_fan<4, 32768, 1>("copy_tma lag1", src, dst, S, 1, sms);
  }
  for (int pad = 0; pad < (mode == 2 ? 0 : 2); ++pad) {
    g_stride = pad ? S + 40960 : 0;
    run_fan<4, 4096, 1>("fan_tma lag1", src, dst, S, fan, sms);
    run_fan<2, 8192, 0>("fan_tma lag0", src, dst, S, fan, sms);
    run_fan<4, 8192, 1>("fan_tma lag1", src, dst, S, fan, sms);
    run_fan<8, 8192, 1>("fan_tma lag1", src, dst, S, fan, sms);
    run_fan<2, 16384, 0>("fan_tma lag0", src, dst, S, fan, sms);
    run_fan<4, 16384, 1>("fan_tma lag1", src, dst, S, fan, sms);
    run_fan<4, 32768, 0>("fan_tma lag0", src, dst, S, fan, sms);
  }
  CK(cudaDeviceSynchronize());
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
