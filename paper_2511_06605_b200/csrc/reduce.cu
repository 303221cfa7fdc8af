// Reduce-scatter reduction kernel (§6.1 hybrid).
//
// dst[e] = op(src_0[e], src_1[e], ..., src_{n-1}[e]) with the sources folded
// in order into an fp32 accumulator and one round-to-nearest-even at the end,
// exactly the order of the oracle (oracle/cecoll_oracle.c ora_reduce_scatter),
// so results are bit-exact for every dtype.
//
// Roofline: HBM (or NVLink for peer sources): per output element nsrc reads
// and one write. Each thread owns 16 consecutive elements of a 4096-element
// tile and issues four sources' 16-byte loads before folding them.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "kernels.hpp"

namespace cecoll {

namespace {

#include "flags.cuh"

constexpr int kRedThreads = 256;
constexpr int kElemsPerThread = static_cast<int>(kRedTileElems / kRedThreads);  // 16

template <int kDtype>
struct Elem;
template <>
struct Elem<kF32> {
  using T = float;
  static __device__ __forceinline__ float to_f(T x) { return x; }
  static __device__ __forceinline__ T from_f(float x) { return x; }
};
template <>
struct Elem<kBF16> {
  using T = __nv_bfloat16;
  static __device__ __forceinline__ float to_f(T x) { return __bfloat162float(x); }
  static __device__ __forceinline__ T from_f(float x) { return __float2bfloat16_rn(x); }
};
template <>
struct Elem<kF16> {
  using T = __half;
  static __device__ __forceinline__ float to_f(T x) { return __half2float(x); }
  static __device__ __forceinline__ T from_f(float x) { return __float2half_rn(x); }
};

template <int kOp>
__device__ __forceinline__ float fold(float acc, float x) {
  if (kOp == kSum) return acc + x;
  if (kOp == kMax) return (x > acc) ? x : acc;
  return (x < acc) ? x : acc;
}

// Sources whose loads are in flight together: 4 (with 2 tiles per CTA,
// exec.cpp plan_red_grid, 16-256 MiB chunks 0.89-0.95 -> 1.0-1.06 of the copy
// peak; 8 sources at once drop to 0.41-0.50, profiles/tma_shape_r02.md).
constexpr int kBatch = 4;

template <int kDtype, int kOp>
__global__ void __launch_bounds__(kRedThreads) reduce_kernel(const RedItem* __restrict__ items, int nitems,
                                                              int ntiles, FlagSet flags) {
  using E = Elem<kDtype>;
  using T = typename E::T;
  constexpr int kVecElems = 16 / static_cast<int>(sizeof(T));            // elements per 16-byte vector
  constexpr int kVecs = kElemsPerThread / kVecElems;                       // vectors per thread
  __shared__ int first[kMaxItemsSmem];
  const uint64_t sk = threadIdx.x < 32 ? read_skip(flags) : 0;
  for (int i = threadIdx.x; i < nitems; i += kRedThreads) first[i] = items[i].first_tile;
  // Fused flags (kernels.hpp FlagSet): every source rank's send is ready.
  __shared__ int cta_state;
  if (threadIdx.x < 32) {
    const int st = (flags.npoll || flags.npre || flags.epoch || flags.skip) ? fused_wait(flags, sk) : kGo;
    if (threadIdx.x == 0) cta_state = st;
  }
  __syncthreads();
  const int state = cta_state;
  const bool moved = state == kGo;
  int cur = 0;
  for (int tile = moved ? blockIdx.x : ntiles; tile < ntiles; tile += gridDim.x) {
    while (cur + 1 < nitems && first[cur + 1] <= tile) ++cur;
    const RedItem it = items[cur];
    const int64_t base = static_cast<int64_t>(tile - it.first_tile) * kRedTileElems + threadIdx.x * kElemsPerThread;
    if (base >= it.elems) continue;
    float acc[kElemsPerThread];
    const bool full = base + kElemsPerThread <= it.elems;
    if (it.vec && full) {
      // kBatch sources' loads in flight before any is folded (the fold order
      // stays source 0, 1, ..., n-1)
      for (int s0 = 0; s0 < it.nsrc; s0 += kBatch) {
        int4 v[kBatch][kVecs];
#pragma unroll
        for (int b = 0; b < kBatch; ++b)
          if (s0 + b < it.nsrc) {
            const int4* p = reinterpret_cast<const int4*>(it.srcs[s0 + b] + base * sizeof(T));
#pragma unroll
            for (int k = 0; k < kVecs; ++k) v[b][k] = __ldg(p + k);
          }
#pragma unroll
        for (int b = 0; b < kBatch; ++b)
          if (s0 + b < it.nsrc) {
#pragma unroll
            for (int k = 0; k < kVecs; ++k) {
              const T* x = reinterpret_cast<const T*>(&v[b][k]);
#pragma unroll
              for (int e = 0; e < kVecElems; ++e) {
                const float f = E::to_f(x[e]);
                acc[k * kVecElems + e] = s0 + b == 0 ? f : fold<kOp>(acc[k * kVecElems + e], f);
              }
            }
          }
      }
      int4 out[kVecs];
#pragma unroll
      for (int k = 0; k < kVecs; ++k) {
        T* y = reinterpret_cast<T*>(&out[k]);
#pragma unroll
        for (int e = 0; e < kVecElems; ++e) y[e] = E::from_f(acc[k * kVecElems + e]);
      }
      int4* q = reinterpret_cast<int4*>(it.dst + base * sizeof(T));
#pragma unroll
      for (int k = 0; k < kVecs; ++k) q[k] = out[k];
    } else {
      const int64_t m = it.elems - base < kElemsPerThread ? it.elems - base : kElemsPerThread;
      for (int s = 0; s < it.nsrc; ++s) {
        const T* p = reinterpret_cast<const T*>(it.srcs[s]) + base;
        for (int e = 0; e < m; ++e) {
          const float f = E::to_f(p[e]);
          acc[e] = s == 0 ? f : fold<kOp>(acc[e], f);
        }
      }
      T* q = reinterpret_cast<T*>(it.dst) + base;
      for (int e = 0; e < m; ++e) q[e] = E::from_f(acc[e]);
    }
  }
  if (flags.ctr) {  // every source read: tell the source ranks (last CTA)
    __syncthreads();
    if (threadIdx.x == 0) fused_finish(flags, state);
  }
}

template <int kDtype>
const void* kernel_for(int op) {
  switch (op) {
    case kSum: return reinterpret_cast<const void*>(reduce_kernel<kDtype, kSum>);
    case kMax: return reinterpret_cast<const void*>(reduce_kernel<kDtype, kMax>);
    case kMin: return reinterpret_cast<const void*>(reduce_kernel<kDtype, kMin>);
    default: return nullptr;
  }
}

}  // namespace

KernelCall reduce_call(const RedTable& t, int grid, const FlagSet* fp) {
  KernelCall k;
  if (t.nitems <= 0 || t.ntiles <= 0 || t.nitems > kMaxItemsSmem) return k;
  if (grid > t.ntiles) grid = t.ntiles;
  switch (t.dtype) {
    case kF32: k.func = kernel_for<kF32>(t.op); break;
    case kBF16: k.func = kernel_for<kBF16>(t.op); break;
    case kF16: k.func = kernel_for<kF16>(t.op); break;
    default: break;
  }
  if (!k.func) return k;
  k.grid = dim3(grid);
  k.block = dim3(kRedThreads);
  k.push(static_cast<const RedItem*>(t.items));
  k.push(t.nitems);
  k.push(t.ntiles);
  k.push(fp ? *fp : FlagSet{});
  return k;
}

cudaError_t launch_reduce(const RedTable& t, int grid, cudaStream_t stream, const FlagSet* fp) {
  if (t.nitems <= 0 || t.ntiles <= 0) return cudaSuccess;
  const KernelCall k = reduce_call(t, grid, fp);
  if (!k.func) return cudaErrorInvalidValue;
  return launch(k, stream);
}

// Loads every reduction kernel on the current device (see preload_kernels,
// kernels.cu: a lazy module load can wait behind a spinning armed gate).
cudaError_t preload_reduce_kernels() {
  cudaFuncAttributes a;
  const void* fns[] = {
      kernel_for<kF32>(kSum),  kernel_for<kF32>(kMax),  kernel_for<kF32>(kMin),
      kernel_for<kBF16>(kSum), kernel_for<kBF16>(kMax), kernel_for<kBF16>(kMin),
      kernel_for<kF16>(kSum),  kernel_for<kF16>(kMax),  kernel_for<kF16>(kMin),
  };
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace cecoll
