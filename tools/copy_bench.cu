// Copy-kernel variant bench for the SM path (one B200).
//
// Workload = the bench config: 64 chunk copies of 8 MiB (8 co-resident ranks,
// all-to-all, local placement included), 1 GiB of algorithmic traffic.
// Variants: register-staged LDG/STG copies with different tile shapes and
// occupancy, cache hints, and a TMA bulk (cp.async.bulk) shared-memory
// pipeline. Reports GB/s (read+write) per variant against cudaMemcpyAsync.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <unistd.h>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

struct Item {
  const char* src;
  char* dst;
  int64_t bytes;
  int first_tile;
  int pad;
};

template <int kLoad>
__device__ __forceinline__ int4 ld(const int4* p) {
  int4 r;
  if (kLoad == 0)
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  else if (kLoad == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  else
    asm volatile("ld.global.cs.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int kStore>
__device__ __forceinline__ void st(int4* p, const int4& v) {
  if (kStore == 0)
    asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else if (kStore == 1)
    asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

template <int kThreads, int kVec, int kMinBlocks, int kLoad, int kStore>
__global__ void __launch_bounds__(kThreads, kMinBlocks) reg_copy(const Item* __restrict__ items, int nitems, int ntiles) {
  constexpr int64_t kTile = (int64_t)kThreads * kVec * 16;
  __shared__ int first[1024];
  for (int i = threadIdx.x; i < nitems; i += kThreads) first[i] = items[i].first_tile;
  __syncthreads();
  int cur = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    while (cur + 1 < nitems && first[cur + 1] <= tile) ++cur;
    const Item it = items[cur];
    const int64_t off = (int64_t)(tile - it.first_tile) * kTile;
    const int4* s = reinterpret_cast<const int4*>(it.src + off);
    int4* d = reinterpret_cast<int4*>(it.dst + off);
    int4 r[kVec];
#pragma unroll
    for (int k = 0; k < kVec; ++k) r[k] = ld<kLoad>(s + threadIdx.x + k * kThreads);
#pragma unroll
    for (int k = 0; k < kVec; ++k) st<kStore>(d + threadIdx.x + k * kThreads, r[k]);
  }
}

template <int kThreads, int kVec, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks) reg_copy_ranges(const Item* __restrict__ items, int nitems, int ntiles) {
  constexpr int64_t kTile = (int64_t)kThreads * kVec * 16;
  __shared__ int first[1024];
  for (int i = threadIdx.x; i < nitems; i += kThreads) first[i] = items[i].first_tile;
  __syncthreads();
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(ntiles, t0 + per);
  int cur = 0;
  for (int tile = t0; tile < t1; ++tile) {
    while (cur + 1 < nitems && first[cur + 1] <= tile) ++cur;
    const Item it = items[cur];
    const int64_t off = (int64_t)(tile - it.first_tile) * kTile;
    const int4* s = reinterpret_cast<const int4*>(it.src + off);
    int4* d = reinterpret_cast<int4*>(it.dst + off);
    int4 r[kVec];
#pragma unroll
    for (int k = 0; k < kVec; ++k) r[k] = ld<0>(s + threadIdx.x + k * kThreads);
#pragma unroll
    for (int k = 0; k < kVec; ++k) st<0>(d + threadIdx.x + k * kThreads, r[k]);
  }
}

// TMA bulk pipeline: one elected thread per CTA streams tiles through kStages
// shared-memory buffers: cp.async.bulk G->S (mbarrier complete_tx), then
// cp.async.bulk S->G (bulk_group), reusing a stage once its store has read it.
template <int kStages, int kTileBytes>
__global__ void __launch_bounds__(32, 1) tma_copy(const Item* __restrict__ items, int nitems, int ntiles) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[kStages];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < kStages; ++i) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[i]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  int my_tiles = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) ++my_tiles;
  auto tile_of = [&](int k) { return blockIdx.x + k * gridDim.x; };
  int cur_item = 0;
  auto locate = [&](int tile, const char** src, char** dst) {
    while (cur_item + 1 < nitems && items[cur_item + 1].first_tile <= tile) ++cur_item;
    const Item it = items[cur_item];
    const int64_t off = (int64_t)(tile - it.first_tile) * kTileBytes;
    *src = it.src + off;
    *dst = it.dst + off;
  };
  const char* srcs[kStages];
  char* dsts[kStages];
  uint32_t phase = 0;
  // prologue
  int issued = 0;
  for (; issued < kStages && issued < my_tiles; ++issued) {
    locate(tile_of(issued), &srcs[issued], &dsts[issued]);
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[issued]);
    uint32_t s = (uint32_t)__cvta_generic_to_shared(smem + issued * kTileBytes);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kTileBytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s),
                 "l"(srcs[issued]), "r"(kTileBytes), "r"(b)
                 : "memory");
  }
  for (int k = 0; k < my_tiles; ++k) {
    const int st_ = k % kStages;
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[st_]);
    uint32_t par = (phase >> st_) & 1;
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(b), "r"(par)
        : "memory");
    phase ^= (1u << st_);
    uint32_t s = (uint32_t)__cvta_generic_to_shared(smem + st_ * kTileBytes);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dsts[st_]), "r"(s), "r"(kTileBytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (issued < my_tiles) {
      // stage st_ is reused by tile `issued`: wait until its store has read smem
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      locate(tile_of(issued), &srcs[st_], &dsts[st_]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kTileBytes));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s),
                   "l"(srcs[st_]), "r"(kTileBytes), "r"(b)
                   : "memory");
      ++issued;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  alarm(240);
  const int n = 8;
  const int64_t s = 8 << 20;
  std::vector<char*> send(n), recv(n);
  for (int r = 0; r < n; ++r) {
    CK(cudaMalloc(&send[r], n * s));
    CK(cudaMalloc(&recv[r], n * s));
    CK(cudaMemset(send[r], r + 1, n * s));
  }
  auto build = [&](int64_t tile) {
    std::vector<Item> items;
    int t = 0;
    for (int r = 0; r < n; ++r)
      for (int d = 0; d < n; ++d) {
        int j = (r + d) % n;
        Item it{send[r] + j * s, recv[j] + r * s, s, t, 0};
        t += (int)((s + tile - 1) / tile);
        items.push_back(it);
      }
    Item* dev;
    CK(cudaMalloc(&dev, sizeof(Item) * items.size()));
    CK(cudaMemcpy(dev, items.data(), sizeof(Item) * items.size(), cudaMemcpyHostToDevice));
    return std::make_pair(dev, t);
  };
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double bytes = 2.0 * n * n * s;
  auto timeit = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    float best = 1e9, tot = 0;
    const int iters = 50;
    for (int i = 0; i < iters; ++i) {
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
      tot += ms;
    }
    CK(cudaGetLastError());
    printf("%-44s best %.4f ms (%.0f GB/s)  mean %.4f ms (%.0f GB/s)\n", name, best, bytes / best / 1e6, tot / iters,
           bytes / (tot / iters) / 1e6);
  };
  timeit("cudaMemcpyAsync x64", [&] {
    for (int r = 0; r < n; ++r)
      for (int j = 0; j < n; ++j) CK(cudaMemcpyAsync(recv[j] + r * s, send[r] + j * s, s, cudaMemcpyDeviceToDevice));
  });
#define REG(TH, V, MB, LD, ST, GRIDMUL)                                                                   \
  {                                                                                                       \
    auto [items, nt] = build((int64_t)TH * V * 16);                                                      \
    char name[96];                                                                                        \
    snprintf(name, sizeof name, "reg th=%d v=%d minb=%d ld=%d st=%d grid=148x%d", TH, V, MB, LD, ST, GRIDMUL); \
    timeit(name, [&] { reg_copy<TH, V, MB, LD, ST><<<148 * GRIDMUL, TH>>>(items, 64, nt); });           \
    cudaFree(items);                                                                                      \
  }
  REG(512, 8, 3, 0, 0, 16);
  REG(256, 8, 8, 0, 0, 32);
  {
    char *a, *b;
    CK(cudaMalloc(&a, 512 << 20));
    CK(cudaMalloc(&b, 512 << 20));
    timeit("contig memcpy 512MiB", [&] { CK(cudaMemcpyAsync(b, a, 512 << 20, cudaMemcpyDeviceToDevice)); });
    cudaFree(a); cudaFree(b);
  }
#define TMA(ST, TB, CTAS)                                                                        \
  {                                                                                              \
    auto [items, nt] = build(TB);                                                                \
    auto k = tma_copy<ST, TB>;                                                                   \
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * TB));           \
    char name[96];                                                                               \
    snprintf(name, sizeof name, "tma stages=%d tile=%d ctas/sm=%d", ST, TB, CTAS);              \
    timeit(name, [&] { k<<<148 * CTAS, 32, ST * TB>>>(items, 64, nt); });                       \
    cudaFree(items);                                                                             \
  }
  TMA(4, 32768, 1);
  TMA(4, 32768, 2);
  TMA(3, 32768, 2);
  TMA(6, 16384, 2);
  TMA(8, 16384, 2);
  TMA(5, 32768, 1);
  TMA(2, 65536, 2);
  TMA(3, 65536, 1);
  TMA(4, 16384, 3);
  TMA(3, 16384, 4);
  TMA(4, 32768, 4);
  printf("copy_bench done\n");
  return 0;
}
