// sm_100a item mover: copies, two-destination broadcasts and in-place swaps.
//
// Roofline: pure data movement, bound by HBM (same-device destinations) or by
// NVLink (peer destinations). Algorithmic bytes per item: copy 2*bytes
// (1 read + 1 write), bcst 3*bytes (1 read + 2 writes), swap 4*bytes.
//
// Each CTA of 256 threads moves 32 KiB tiles: every thread issues eight
// independent 128-bit loads before its eight 128-bit stores, so 128 KiB per SM
// (at 4 CTAs/SM) are in flight, enough to cover HBM and NVLink latency.
// Source loads bypass L1 (ld.global.nc.L1::no_allocate); the data is touched
// once.
#include <cstdint>

#include "kernels.hpp"

namespace cecoll {

namespace {

constexpr int kVecPerThread = static_cast<int>(kTileBytes / 16 / kCopyThreads);  // 8
static_assert(kVecPerThread * 16 * kCopyThreads == kTileBytes, "tile shape");

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ int4 ld_plain(const int4* p) {
  int4 r;
  asm volatile("ld.global.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_vec(int4* p, const int4& v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Full, 16-byte aligned tile body: nvec vectors starting at vector 0.
__device__ __forceinline__ void move_vectors(const Item& it, int64_t off, int64_t nvec) {
  const int t = threadIdx.x;
  if (it.kind == kItemSwap) {
    int4* a = reinterpret_cast<int4*>(it.dst + off);
    int4* b = reinterpret_cast<int4*>(const_cast<char*>(it.src) + off);
    int4 va[kVecPerThread], vb[kVecPerThread];
#pragma unroll
    for (int k = 0; k < kVecPerThread; ++k) {
      const int64_t v = t + (int64_t)k * kCopyThreads;
      if (v < nvec) {
        va[k] = ld_plain(a + v);
        vb[k] = ld_plain(b + v);
      }
    }
#pragma unroll
    for (int k = 0; k < kVecPerThread; ++k) {
      const int64_t v = t + (int64_t)k * kCopyThreads;
      if (v < nvec) {
        st_vec(a + v, vb[k]);
        st_vec(b + v, va[k]);
      }
    }
    return;
  }
  const int4* s = reinterpret_cast<const int4*>(it.src + off);
  int4* d = reinterpret_cast<int4*>(it.dst + off);
  int4 r[kVecPerThread];
  if (nvec == kTileBytes / 16) {
#pragma unroll
    for (int k = 0; k < kVecPerThread; ++k) r[k] = ld_stream(s + t + k * kCopyThreads);
#pragma unroll
    for (int k = 0; k < kVecPerThread; ++k) st_vec(d + t + k * kCopyThreads, r[k]);
    if (it.kind == kItemBcst) {
      int4* d2 = reinterpret_cast<int4*>(it.dst2 + off);
#pragma unroll
      for (int k = 0; k < kVecPerThread; ++k) st_vec(d2 + t + k * kCopyThreads, r[k]);
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < kVecPerThread; ++k) {
    const int64_t v = t + (int64_t)k * kCopyThreads;
    if (v < nvec) r[k] = ld_stream(s + v);
  }
#pragma unroll
  for (int k = 0; k < kVecPerThread; ++k) {
    const int64_t v = t + (int64_t)k * kCopyThreads;
    if (v < nvec) st_vec(d + v, r[k]);
  }
  if (it.kind == kItemBcst) {
    int4* d2 = reinterpret_cast<int4*>(it.dst2 + off);
#pragma unroll
    for (int k = 0; k < kVecPerThread; ++k) {
      const int64_t v = t + (int64_t)k * kCopyThreads;
      if (v < nvec) st_vec(d2 + v, r[k]);
    }
  }
}

// Byte-granular path for [off, off+len) (misaligned heads/tails, or items
// whose source and destination disagree modulo 16).
__device__ __forceinline__ void move_bytes(const Item& it, int64_t off, int64_t len) {
  for (int64_t b = threadIdx.x; b < len; b += kCopyThreads) {
    const int64_t o = off + b;
    if (it.kind == kItemSwap) {
      char* a = it.dst + o;
      char* c = const_cast<char*>(it.src) + o;
      const char x = *a, y = *c;
      *a = y;
      *c = x;
    } else {
      const char x = it.src[o];
      it.dst[o] = x;
      if (it.kind == kItemBcst) it.dst2[o] = x;
    }
  }
}

__device__ __forceinline__ void move_tile(const Item& it, int64_t off, int64_t len) {
  const uintptr_t d = reinterpret_cast<uintptr_t>(it.dst + off);
  const uintptr_t s = reinterpret_cast<uintptr_t>(it.src + off);
  uintptr_t mis = (d ^ s) & 15;
  if (it.kind == kItemBcst) mis |= (d ^ reinterpret_cast<uintptr_t>(it.dst2 + off)) & 15;
  if (mis) {
    move_bytes(it, off, len);
    return;
  }
  const int64_t head = static_cast<int64_t>((16 - (d & 15)) & 15) < len ? static_cast<int64_t>((16 - (d & 15)) & 15)
                                                                         : len;
  if (head) move_bytes(it, off, head);
  const int64_t body = (len - head) & ~static_cast<int64_t>(15);
  if (body) move_vectors(it, off + head, body / 16);
  const int64_t tail = len - head - body;
  if (tail) move_bytes(it, off + head + body, tail);
}

__global__ void __launch_bounds__(kCopyThreads) items_kernel(const Item* __restrict__ items, int nitems,
                                                              int ntiles) {
  __shared__ int first[kMaxItemsSmem];
  for (int i = threadIdx.x; i < nitems; i += kCopyThreads) first[i] = items[i].first_tile;
  __syncthreads();
  int cur = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    while (cur + 1 < nitems && first[cur + 1] <= tile) ++cur;
    const Item it = items[cur];
    const int64_t off = static_cast<int64_t>(tile - it.first_tile) * kTileBytes;
    const int64_t rem = it.bytes - off;
    move_tile(it, off, rem < kTileBytes ? rem : kTileBytes);
  }
}

constexpr unsigned long long kPollTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void poll_kernel(uint64_t* const* flags, int n, uint64_t* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t* f = flags[i];
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys(f) < 1) {
    if (globaltimer() - t0 > kPollTimeoutNs) {
      atomicOr(reinterpret_cast<unsigned long long*>(err), 1ull);
      return;
    }
    __nanosleep(64);
  }
  *f = 0;
}

__global__ void signal_kernel(uint64_t* const* flags, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  __threadfence_system();
  st_release_sys(flags[i], 1);
}

// Gate of a recorded prelaunch graph. The host posts triggers/cancels into
// pinned memory: posted[0] is a monotonic count, posted[1 + k % 64] the kind
// of post k (1 = go, 2 = cancel). `consumed` (device memory) counts the posts
// already taken by earlier instances; instances run one at a time on the arm
// stream, so the read-modify-write needs no atomics.
__global__ void gate_kernel(volatile uint64_t* posted, uint64_t* consumed, cudaGraphConditionalHandle handle,
                            uint64_t* err) {
  if (threadIdx.x != 0) return;
  const uint64_t c = *consumed;
  while (posted[0] <= c) __nanosleep(256);
  const uint64_t kind = posted[1 + (c % 64)];
  *consumed = c + 1;
  __threadfence_system();
  if (kind != 1 && kind != 2) atomicOr(reinterpret_cast<unsigned long long*>(err), 2ull);
  cudaGraphSetConditional(handle, kind == 1 ? 1u : 0u);
}

}  // namespace

cudaError_t launch_poll(uint64_t* const* flags, int n, uint64_t* err, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  poll_kernel<<<(n + 127) / 128, 128, 0, stream>>>(flags, n, err);
  return cudaGetLastError();
}

cudaError_t launch_signal(uint64_t* const* flags, int n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  signal_kernel<<<(n + 127) / 128, 128, 0, stream>>>(flags, n);
  return cudaGetLastError();
}

cudaError_t launch_gate(volatile uint64_t* posted, uint64_t* consumed, cudaGraphConditionalHandle handle,
                        uint64_t* err, cudaStream_t stream) {
  gate_kernel<<<1, 32, 0, stream>>>(posted, consumed, handle, err);
  return cudaGetLastError();
}

int64_t tiles_for(int64_t bytes) { return (bytes + kTileBytes - 1) / kTileBytes; }

cudaError_t launch_items(const Item* items, int nitems, int ntiles, int grid, cudaStream_t stream) {
  if (nitems <= 0 || ntiles <= 0) return cudaSuccess;
  if (nitems > kMaxItemsSmem) return cudaErrorInvalidValue;
  if (grid > ntiles) grid = ntiles;
  items_kernel<<<grid, kCopyThreads, 0, stream>>>(items, nitems, ntiles);
  return cudaGetLastError();
}

}  // namespace cecoll
