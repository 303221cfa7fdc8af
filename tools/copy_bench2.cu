// TMA mover variants at several chunk sizes (8 co-resident ranks, all-to-all
// item pattern): ring depth, tile size, grid, L2 evict-first hints.
//   tools/copy_bench2 <s_bytes>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <algorithm>
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

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int kStages, int kTile, bool kHint>
__global__ void __launch_bounds__(32, 1) tma_copy(const Item* __restrict__ items, int nitems, int ntiles) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ int first[1024];
  for (int i = threadIdx.x; i < nitems; i += 32) first[i] = items[i].first_tile;
  __syncwarp();
  if (threadIdx.x != 0) return;
  for (int i = 0; i < kStages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t pol = 0;
  if (kHint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  int cur = 0;
  auto locate = [&](int k, const char** src, char** dst) {
    const int tile = blockIdx.x + k * gridDim.x;
    while (cur + 1 < nitems && first[cur + 1] <= tile) ++cur;
    const Item& it = items[cur];
    const int64_t off = (int64_t)(tile - it.first_tile) * kTile;
    *src = it.src + off;
    *dst = it.dst + off;
  };
  auto load = [&](int st, const char* src) {
    const uint32_t bar = sa(&full[st]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kTile) : "memory");
    if (kHint)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
              sa(ring + st * kTile)),
          "l"(src), "r"(kTile), "r"(bar), "l"(pol)
          : "memory");
    else
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(ring + st * kTile)),
                   "l"(src), "r"(kTile), "r"(bar)
                   : "memory");
  };
  char* dst[kStages];
  int issued = 0;
  for (; issued < kStages && issued < mine; ++issued) {
    const char* s;
    locate(issued, &s, &dst[issued]);
    load(issued, s);
  }
  uint32_t phase = 0;
  for (int k = 0; k < mine; ++k) {
    const int st = k % kStages;
    asm volatile("{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(
                     sa(&full[st])),
                 "r"((phase >> st) & 1u)
                 : "memory");
    phase ^= 1u << st;
    if (kHint)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst[st]),
                   "r"(sa(ring + st * kTile)), "r"(kTile), "l"(pol)
                   : "memory");
    else
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst[st]),
                   "r"(sa(ring + st * kTile)), "r"(kTile)
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (issued < mine) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      const char* s;
      locate(issued, &s, &dst[st]);
      load(st, s);
      ++issued;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  alarm(240);
  const int n = 8;
  const int64_t s = argc > 1 ? atoll(argv[1]) : (8 << 20);
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
        items.push_back(Item{send[r] + j * s, recv[j] + r * s, s, t, 0});
        t += (int)((s + tile - 1) / tile);
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
    std::vector<float> v;
    const int iters = s >= (64 << 20) ? 10 : 40;
    for (int i = 0; i < iters; ++i) {
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      v.push_back(ms);
    }
    CK(cudaGetLastError());
    std::sort(v.begin(), v.end());
    printf("s=%lld %-40s median %.4f ms (%.0f GB/s) best %.0f GB/s\n", (long long)s, name, v[v.size() / 2],
           bytes / v[v.size() / 2] / 1e6, bytes / v[0] / 1e6);
  };
  timeit("cudaMemcpyAsync x64", [&] {
    for (int r = 0; r < n; ++r)
      for (int j = 0; j < n; ++j) CK(cudaMemcpyAsync(recv[j] + r * s, send[r] + j * s, s, cudaMemcpyDeviceToDevice));
  });
#define T(ST, TB, HINT, GRID)                                                                   \
  {                                                                                             \
    auto [items, nt] = build(TB);                                                               \
    auto k = tma_copy<ST, TB, HINT>;                                                            \
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * TB));          \
    char name[96];                                                                              \
    snprintf(name, sizeof name, "tma st=%d tile=%d hint=%d grid=%d", ST, TB, (int)HINT, GRID); \
    timeit(name, [&] { k<<<GRID, 32, ST * TB>>>(items, 64, nt); });                            \
    cudaFree(items);                                                                            \
  }
  T(4, 32768, false, 296);
  T(4, 32768, true, 296);
  T(4, 32768, false, 148);
  T(6, 32768, false, 148);
  T(6, 32768, true, 148);
  T(3, 65536, false, 148);
  T(8, 16384, false, 296);
  T(8, 16384, true, 296);
  T(4, 32768, false, 444);
  T(12, 16384, false, 148);
  printf("done\n");
  return 0;
}
