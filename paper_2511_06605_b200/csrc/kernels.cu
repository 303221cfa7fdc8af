// sm_100a item movers (copies, two-destination broadcasts, in-place swaps)
// and the flag kernels of recorded graphs.
//
// Roofline: pure data movement, bound by HBM (same-device destinations) or by
// NVLink (peer destinations). Algorithmic bytes per item: copy 2*bytes
// (1 read + 1 write), bcst 3*bytes (1 read + 2 writes), swap 4*bytes.
// Variant choice (tile shape, occupancy, TMA vs registers) was measured with
// tools/copy_bench.cu on the bench workload (profiles/copy_bench_r01.txt).
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "kernels.hpp"

namespace cecoll {

namespace {

#include "flags.cuh"

// ---------------------------------------------------------------------------
// Register mover
// ---------------------------------------------------------------------------

constexpr int kRegThreads = 512;
constexpr int kRegVec = 8;  // 16-byte vectors per thread per tile
constexpr int64_t kRegTile = int64_t{kRegThreads} * kRegVec * 16;  // 64 KiB

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ int4 ld_plain(const int4* p) {
  int4 r;
  asm volatile("ld.global.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ void st_vec(int4* p, const int4& v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// 16-byte aligned body of nvec vectors.
template <int kKinds>
__device__ __forceinline__ void move_vectors(const Item& it, int64_t off, int64_t nvec) {
  const int t = threadIdx.x;
  const bool full = nvec == kRegTile / 16;
  if ((kKinds & (1 << kItemSwap)) && it.kind == kItemSwap) {
    int4* a = reinterpret_cast<int4*>(it.dst + off);
    int4* b = reinterpret_cast<int4*>(const_cast<char*>(it.src) + off);
    int4 va[kRegVec], vb[kRegVec];
#pragma unroll
    for (int k = 0; k < kRegVec; ++k) {
      const int64_t v = t + int64_t{k} * kRegThreads;
      if (full || v < nvec) {
        va[k] = ld_plain(a + v);
        vb[k] = ld_plain(b + v);
      }
    }
#pragma unroll
    for (int k = 0; k < kRegVec; ++k) {
      const int64_t v = t + int64_t{k} * kRegThreads;
      if (full || v < nvec) {
        st_vec(a + v, vb[k]);
        st_vec(b + v, va[k]);
      }
    }
    return;
  }
  const int4* s = reinterpret_cast<const int4*>(it.src + off);
  int4* d = reinterpret_cast<int4*>(it.dst + off);
  int4 r[kRegVec];
#pragma unroll
  for (int k = 0; k < kRegVec; ++k) {
    const int64_t v = t + int64_t{k} * kRegThreads;
    if (full || v < nvec) r[k] = ld_stream(s + v);
  }
#pragma unroll
  for (int k = 0; k < kRegVec; ++k) {
    const int64_t v = t + int64_t{k} * kRegThreads;
    if (full || v < nvec) st_vec(d + v, r[k]);
  }
  if ((kKinds & (1 << kItemBcst)) && it.kind == kItemBcst) {
    int4* d2 = reinterpret_cast<int4*>(it.dst2 + off);
#pragma unroll
    for (int k = 0; k < kRegVec; ++k) {
      const int64_t v = t + int64_t{k} * kRegThreads;
      if (full || v < nvec) st_vec(d2 + v, r[k]);
    }
  }
  if ((kKinds & (1 << kItemFan)) && it.kind == kItemFan) {
    for (int f = 1; f < it.nfan; ++f) {  // fan[0] is it.dst, already written
      int4* df = reinterpret_cast<int4*>(it.fan[f] + off);
#pragma unroll
      for (int k = 0; k < kRegVec; ++k) {
        const int64_t v = t + int64_t{k} * kRegThreads;
        if (full || v < nvec) st_vec(df + v, r[k]);
      }
    }
  }
}

// Byte-granular path for [off, off+len): unaligned heads/tails, or items
// whose source and destination disagree modulo 16.
__device__ __forceinline__ void move_bytes(const Item& it, int64_t off, int64_t len) {
  for (int64_t b = threadIdx.x; b < len; b += kRegThreads) {
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
      if (it.kind == kItemFan)
        for (int f = 1; f < it.nfan; ++f) it.fan[f][o] = x;
    }
  }
}

template <int kKinds>
__device__ __forceinline__ void move_tile(const Item& it, int64_t off, int64_t len) {
  const uintptr_t d = reinterpret_cast<uintptr_t>(it.dst + off);
  const uintptr_t s = reinterpret_cast<uintptr_t>(it.src + off);
  uintptr_t mis = (d ^ s) & 15;
  if (it.kind == kItemBcst) mis |= (d ^ reinterpret_cast<uintptr_t>(it.dst2 + off)) & 15;
  if (it.kind == kItemFan)
    for (int f = 1; f < it.nfan; ++f) mis |= (d ^ reinterpret_cast<uintptr_t>(it.fan[f] + off)) & 15;
  if (mis) {
    move_bytes(it, off, len);
    return;
  }
  int64_t head = static_cast<int64_t>((16 - (d & 15)) & 15);
  if (head > len) head = len;
  if (head) move_bytes(it, off, head);
  const int64_t body = (len - head) & ~int64_t{15};
  if (body) move_vectors<kKinds>(it, off + head, body / 16);
  const int64_t tail = len - head - body;
  if (tail) move_bytes(it, off + head + body, tail);
}

// Last item whose first tile is <= tile (binary search over the prefix in
// shared memory; CTAs then advance monotonically).
__device__ __forceinline__ int find_item(const int* first, int nitems, int tile) {
  int lo = 0, hi = nitems - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (first[mid] <= tile) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

template <int kKinds, int kMinBlocks>
__global__ void __launch_bounds__(kRegThreads, kMinBlocks)
    reg_items_kernel(const Item* __restrict__ items, int nitems, int ntiles, int uniform, FlagSet flags) {
  // uniform > 0: every item has `uniform` tiles, so tile t belongs to item
  // t / uniform and the first-tile prefix (a global load round trip before
  // any data moves) is not needed.
  __shared__ int first[kMaxItemsSmem];
  __shared__ int cta_state;
  // no-op unless launched behind a programmatic edge (see gate_poll_kernel)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint64_t sk = threadIdx.x < 32 ? read_skip(flags) : 0;
  if (!uniform)
    for (int i = threadIdx.x; i < nitems; i += kRegThreads) first[i] = items[i].first_tile;
  if (threadIdx.x < 32) {
    const int st = (flags.npoll || flags.npre || flags.epoch || flags.skip) ? fused_wait(flags, sk) : kGo;
    if (threadIdx.x == 0) cta_state = st;
  }
  __syncthreads();
  const int state = cta_state;
  const bool moved = state == kGo;
  int cur = uniform ? 0 : find_item(first, nitems, blockIdx.x);
  for (int tile = moved ? blockIdx.x : ntiles; tile < ntiles; tile += gridDim.x) {
    if (uniform) cur = tile / uniform;
    else
      while (cur + 1 < nitems && first[cur + 1] <= tile) ++cur;
    const Item it = items[cur];
    const int64_t off = static_cast<int64_t>(tile - it.first_tile) * kRegTile;
    const int64_t rem = it.bytes - off;
    move_tile<kKinds>(it, off, rem < kRegTile ? rem : kRegTile);
  }
  if (flags.ctr) {
    __syncthreads();  // every thread's stores (peer stores over NVLink included) precede thread 0's fence
    if (threadIdx.x == 0) fused_finish(flags, state);
  }
}

// ---------------------------------------------------------------------------
// TMA bulk mover (copy items, 16-byte aligned, sizes multiple of 16)
// ---------------------------------------------------------------------------

#ifndef CECOLL_TMA_STAGES
#define CECOLL_TMA_STAGES 4
#endif
constexpr int kTmaStages = CECOLL_TMA_STAGES;
constexpr int kTmaTile = 32 * 1024;  // largest tile
constexpr int kTmaSmem = kTmaStages * kTmaTile;
// The ring is sized per launch (kTmaStages x the table's tile). CTAs of the
// TMA mover resident per SM at a tile size: 228 KiB of shared memory per SM,
// 1 KiB reserved per CTA, the kernel's static shared memory (the mbarriers
// and the first-tile table), at most 32 CTAs per SM.
constexpr int kTmaStaticSmem = kTmaStages * 8 + kMaxItemsSmem * 4 + 256;  // ptxas: 4224 B

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// kLag 0: a stage is refilled as soon as its own stores have read it
// (wait_group.read 0); kLag 1: the previous iteration's stage is refilled
// after the current stores are issued (wait_group.read 1), so one tile's
// stores are always in flight while the next load is issued.
template <int kLag>
// opts: bit 0 L2 evict-first, bit 1 a swap table (every item kItemSwap: a
// stage holds both sides of the exchange, tile_bytes each, and its stores
// write them crosswise).
__global__ void __launch_bounds__(32, 1) tma_items_kernel(const Item* __restrict__ items, int nitems, int ntiles,
                                                          int tile_bytes, int uniform, int opts,
                                                          FlagSet flags) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[kTmaStages];
  __shared__ int first[kMaxItemsSmem];
  asm volatile("griddepcontrol.wait;" ::: "memory");  // see reg_items_kernel
  const uint64_t sk = read_skip(flags);
  if (!uniform)  // see reg_items_kernel
    for (int i = threadIdx.x; i < nitems; i += 32) first[i] = items[i].first_tile;
  __syncwarp();
  // the CTA is one warp: fused_wait's result is already warp-uniform
  const int state = (flags.npoll || flags.npre || flags.epoch || flags.skip) ? fused_wait(flags, sk) : kGo;
  if (threadIdx.x != 0) return;
  if (state != kGo) {
    if (flags.ctr) fused_finish(flags, state);
    return;
  }
  for (int i = 0; i < kTmaStages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");

  const bool swp = opts & 2;
  const int stride = swp ? 2 * tile_bytes : tile_bytes;  // bytes of ring per stage
  const int mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  int cur = uniform ? 0 : find_item(first, nitems, blockIdx.x);
  // Tile k of this CTA is global tile blockIdx.x + k * gridDim.x.
  auto locate = [&](int k, const char** src, int* item, int64_t* off_out, uint32_t* bytes) {
    const int tile = blockIdx.x + k * gridDim.x;
    if (uniform) cur = tile / uniform;
    else
      while (cur + 1 < nitems && first[cur + 1] <= tile) ++cur;
    const Item& it = items[cur];
    const int64_t off = static_cast<int64_t>(tile - it.first_tile) * tile_bytes;
    const int64_t rem = it.bytes - off;
    *src = it.src + off;
    *item = cur;
    *off_out = off;
    *bytes = static_cast<uint32_t>(rem < tile_bytes ? rem : tile_bytes);
  };
  // L2 policy of the bulk copies. Evict-first helped the isolated mover by
  // 1-5% at 1-8 MiB chunks (profiles/copy_bench2_r01.txt) but cost 3-4% in
  // the bench step (profiles/tma_hint_ab_r01.txt), so evict-normal is the
  // default; CECOLL_TMA_EVICT_FIRST=1 selects evict-first.
  uint64_t policy;
  if (opts & 1)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(policy));
  // src2: the other side of a swap item (loaded behind src in the stage)
  auto load = [&](int stage, const char* src, uint32_t bytes, const char* src2) {
    const uint32_t bar = smem_addr(&full[stage]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(swp ? 2 * bytes : bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_addr(ring + stage * stride)),
        "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
    if (swp)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
              "r"(smem_addr(ring + stage * stride + tile_bytes)),
          "l"(src2), "r"(bytes), "r"(bar), "l"(policy)
          : "memory");
  };
  auto other = [&](int item, int64_t off) -> const char* { return swp ? items[item].dst + off : nullptr; };
  int sitem[kTmaStages];
  int64_t soff[kTmaStages];
  uint32_t nbytes[kTmaStages];
  int issued = 0;
  for (; issued < kTmaStages && issued < mine; ++issued) {
    const char* src;
    locate(issued, &src, &sitem[issued], &soff[issued], &nbytes[issued]);
    load(issued, src, nbytes[issued], other(sitem[issued], soff[issued]));
  }
  uint32_t phase = 0;
  for (int k = 0; k < mine; ++k) {
    const int st = k % kTmaStages;
    const uint32_t bar = smem_addr(&full[st]);
    const uint32_t parity = (phase >> st) & 1u;
    asm volatile(
        "{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
    phase ^= 1u << st;
    const Item& it = items[sitem[st]];
    const uint32_t from = smem_addr(ring + st * stride);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                     it.dst + soff[st]),
                 "r"(from), "r"(nbytes[st]), "l"(policy)
                 : "memory");
    if (swp)  // the exchange's other half: what was at dst goes to src
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                       const_cast<char*>(it.src) + soff[st]),
                   "r"(from + tile_bytes), "r"(nbytes[st]), "l"(policy)
                   : "memory");
    if (it.kind == kItemFan)
      for (int f = 1; f < it.nfan; ++f)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                         it.fan[f] + soff[st]),
                     "r"(from), "r"(nbytes[st]), "l"(policy)
                     : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (kLag == 0) {
      if (issued < mine) {
        // The stage is refilled once its store has finished reading it.
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        const char* src;
        locate(issued, &src, &sitem[st], &soff[st], &nbytes[st]);
        load(st, src, nbytes[st], other(sitem[st], soff[st]));
        ++issued;
      }
    } else if (k >= 1 && issued < mine) {
      // Tile `issued` goes to stage issued % kTmaStages == (k - 1) % kTmaStages,
      // whose stores (issued last iteration) have read it once every group
      // but the newest has.
      const int pst = (k - 1) % kTmaStages;
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      const char* src;
      locate(issued, &src, &sitem[pst], &soff[pst], &nbytes[pst]);
      load(pst, src, nbytes[pst], other(sitem[pst], soff[pst]));
      ++issued;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (flags.ctr) {
    // The bulk stores are complete; order them (async proxy) before the
    // generic-proxy fence and ticket that publish them.
    asm volatile("fence.proxy.async.global;" ::: "memory");
    fused_finish(flags, kGo);
  }
}

// ---------------------------------------------------------------------------
// Flag kernels
// ---------------------------------------------------------------------------

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

// Gate of a recorded prelaunch graph with a conditional body: takes the
// unit's trigger word (take_trigger, flags.cuh) and opens the body on "go".
__global__ void gate_kernel(uint64_t* trigger, const volatile uint64_t* cancel, uint64_t* seen,
                            cudaGraphConditionalHandle handle, uint64_t* err) {
  if (threadIdx.x != 0) return;
  const uint64_t kind = take_trigger(trigger, cancel, seen, err);
  cudaGraphSetConditional(handle, kind == 1 ? 1u : 0u);
}

__global__ void gate_poll_kernel(uint64_t* const* flags, int n, const volatile uint64_t* cancel, uint64_t* seen,
                                 uint64_t* skip, uint64_t* err) {
  // flags[0] is the unit's trigger word: lane 0 takes it; on "go" the warp
  // polls the other flags in parallel (lane i: flags 1+i, 33+i, ...) and
  // resets them.
  __shared__ uint64_t kind;
  if (threadIdx.x == 0) kind = take_trigger(flags[0], cancel, seen, err);
  __syncwarp();
  if (kind != 1) {
    if (threadIdx.x == 0) *skip = 1;
    return;
  }
  bool ok = true;
  for (int i = 1 + threadIdx.x; i < n; i += 32) {
    if (wait_flag(flags[i], err)) *flags[i] = 0;
    else ok = false;
  }
  // a poll that timed out keeps the mover from writing into a buffer the
  // peer never released (skip = 2: no data, signals still written; the
  // world's error is sticky from here on)
  ok = __all_sync(0xffffffffu, ok);
  // A mover behind a programmatic edge (CECOLL_PRELAUNCH_PDL=1) may launch
  // now; it still waits (griddepcontrol.wait) until this grid has finished
  // and its skip word is visible.
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0) *skip = ok ? 0 : 2;
}

__global__ void __launch_bounds__(kRegThreads) mc_store_kernel(const int4* __restrict__ src, char* mc_dst,
                                                                int64_t nvec, uint64_t* mc_flag, uint64_t epoch,
                                                                unsigned* ctr) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kRegThreads;
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * kRegThreads + threadIdx.x; v < nvec; v += stride) {
    const int4 x = ld_stream(src + v);
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc_dst + v * 16),
                 "f"(__int_as_float(x.x)), "f"(__int_as_float(x.y)), "f"(__int_as_float(x.z)),
                 "f"(__int_as_float(x.w))
                 : "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  unsigned ticket;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(ticket) : "l"(ctr) : "memory");
  if (ticket != gridDim.x - 1) return;
  *ctr = 0;
  asm volatile("multimem.st.release.sys.global.u64 [%0], %1;" ::"l"(mc_flag), "l"(epoch) : "memory");
}

}  // namespace

int64_t mover_tile_bytes(Mover m) { return m == Mover::Tma ? kTmaTile : kRegTile; }

namespace {
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}
// TMA mover shape (tools/fan_probe.cu, tools/r2_tma_ab.sh,
// profiles/tma_shape_r02.md):
//  * one-wave tables: the smallest tile that leaves one tile per CTA, with
//    one resident CTA per SM counted (CECOLL_TMA_ONEWAVE_RES=0 counts the
//    residency at each tile size instead);
//  * larger copy tables (all-to-all): 16 KiB tiles, 3 tiles per CTA up to
//    16384 tiles (a 256 MiB table), 2 above (tools/latency with LAT_MIN /
//    LAT_STEP: 256 KiB 8.2 -> 6.2 us, 1 MiB 25.8 -> 24.6, 4 MiB 85.6 -> 83.9;
//    2 per CTA stays 1-2% faster from the headline's 32768 tiles up);
//  * larger fan tables (all-gather: one read, n writes): 8 KiB tiles, one
//    tile per CTA.
// Short-lived CTAs, the hardware block scheduler refilling the SMs, beat a
// persistent grid that walks each CTA through a strided band of tiles: the
// 8-rank all-to-all at 16-256 MiB chunks 0.95 -> 1.07-1.09 of the measured
// copy peak, the headline 64 x 8 MiB 0.163 -> 0.161 ms, the all-gather fan
// at 16-256 MiB 0.89-0.90 -> 0.99-1.02. (Round 1's shape — 32 KiB tiles on
// 2 waves of one CTA per SM — is CECOLL_TMA_TILE=32768 CECOLL_TMA_TPC=0.)
// CECOLL_TMA_{TILE,WAVES,LAG,TPC} override the copy shape,
// CECOLL_TMA_FAN_{TILE,WAVES,LAG,TPC} the fan shape (TPC 0: WAVES waves of
// resident CTAs instead of tiles per CTA).
struct TmaShape {
  int tile, waves, lag;
  int tpc;  // > 0: ceil(tiles / tpc) CTAs (tiles per CTA) instead of `waves`
  int tpc_small = 0, small_tiles = 0;  // tables of at most small_tiles tiles: tpc_small per CTA
};
struct TmaPolicy {
  bool onewave_res1 = env_int("CECOLL_TMA_ONEWAVE_RES", 1) == 1;
  TmaShape copy{env_int("CECOLL_TMA_TILE", 16384), env_int("CECOLL_TMA_WAVES", 2), env_int("CECOLL_TMA_LAG", 0),
                env_int("CECOLL_TMA_TPC", 2), env_int("CECOLL_TMA_TPC_SMALL", 3),
                env_int("CECOLL_TMA_SMALL_TILES", 16384)};
  TmaShape fan{env_int("CECOLL_TMA_FAN_TILE", 8192), env_int("CECOLL_TMA_FAN_WAVES", 4),
               env_int("CECOLL_TMA_FAN_LAG", 1), env_int("CECOLL_TMA_FAN_TPC", 1)};
  bool fixed = env_int("CECOLL_TMA_FIXED_TILE", 0) == 1;
  const TmaShape& shape(bool has_fan) const { return has_fan ? fan : copy; }
};
const TmaPolicy& tma_policy() {
  static const TmaPolicy p;
  return p;
}
int clamp_tile(int t) {
  t = (t / 1024) * 1024;
  return t < 4096 ? 4096 : (t > kTmaTile ? kTmaTile : t);
}
}  // namespace

int tma_resident(int tile) {
  const int per = (228 * 1024) / (kTmaStages * tile + kTmaStaticSmem + 1024);
  return per < 1 ? 1 : (per > 32 ? 32 : per);
}

int table_tile(Mover m, const std::vector<int64_t>& sizes, int sms, int budget, bool has_fan, bool swap) {
  if (m != Mover::Tma) return static_cast<int>(kRegTile);
  const TmaPolicy& pol = tma_policy();
  if (swap) {
    // a stage holds both sides: the tile is half the copy tables' ring stage
    // (one-wave tables: the smallest tile leaving one tile per CTA, as below)
    for (int t = 4096; t <= kTmaTile / 2; t += 1024) {
      int64_t slots = int64_t{pol.onewave_res1 ? 1 : tma_resident(2 * t)} * sms;
      if (budget > 0) slots = std::min<int64_t>(slots, budget);
      int64_t n = 0;
      for (int64_t b : sizes) n += (b + t - 1) / t;
      if (n <= slots) return t;
    }
    return budget > 0 ? kTmaTile / 2 : std::min(kTmaTile / 2, clamp_tile(pol.copy.tile) / 2);
  }
  if (pol.fixed) return kTmaTile;
  // The smallest tile (1 KiB steps, at least 4 KiB) that still gives every
  // resident CTA at most one tile: at these sizes parallelism wins over
  // pipelining inside a CTA (tools/latency: a 64 KiB all-gather 8.2 -> 4.1
  // us). An SM budget caps the CTAs that count.
  for (int t = 4096; t <= kTmaTile; t += 1024) {
    int64_t slots = int64_t{pol.onewave_res1 ? 1 : tma_resident(t)} * sms;
    if (budget > 0) slots = std::min<int64_t>(slots, budget);
    int64_t n = 0;
    for (int64_t b : sizes) n += (b + t - 1) / t;
    if (n <= slots) return t;
  }
  // Streaming tables. A budgeted plan keeps the largest ring (most bytes in
  // flight per CTA it is allowed).
  if (budget > 0) return kTmaTile;
  return clamp_tile(pol.shape(has_fan).tile);
}

// Grids. TMA mover: ceil(tiles / tpc) CTAs of the table's shape (TmaPolicy;
// a one-wave table launches one CTA per tile: items_call caps the grid at the
// tile count). Register mover: one tile per CTA, or a persistent 2 CTAs per
// SM for swap tables (mover_grid). Beside compute, the mover's SM footprint
// is a policy: the plan's SM budget (cecoll_comm_set_sm_budget) or
// CECOLL_SM_GRID=<ctas> caps the grid, CECOLL_SM_TILES_PER_CTA=<k> launches
// short-lived CTAs of k tiles so the block scheduler can interleave a
// higher-priority stream's CTAs (profiles/interference_r01.json).
int mover_grid(Mover m, int sms) {
  (void)m;
  static const int cap = env_int("CECOLL_SM_GRID", 0);
  return cap > 0 ? cap : 2 * sms;
}

int mover_grid_for(const ItemTable& t, int sms) {
  static const int per_cta = env_int("CECOLL_SM_TILES_PER_CTA", 0);
  if (per_cta > 0) return std::min((t.ntiles + per_cta - 1) / per_cta, kMaxGrid);
  if (t.mover == Mover::Tma) {
    static const int cap = env_int("CECOLL_SM_GRID", 0);
    const TmaPolicy& pol = tma_policy();
    const int tile = (t.tile > 0 ? t.tile : kTmaTile) * (t.kinds == (1 << kItemSwap) ? 2 : 1);
    const TmaShape& sh = pol.shape(t.kinds & (1 << kItemFan));
    const int64_t one_wave = int64_t{tma_resident(tile)} * sms;
    int64_t g = std::max(1, sh.waves) * one_wave;
    // a table that fits one wave keeps one tile per CTA (items_call caps the
    // grid at the tile count); larger ones get ceil(tiles / tpc) CTAs
    if (sh.tpc > 0 && t.ntiles > one_wave) {
      const int tpc = sh.tpc_small > 0 && t.ntiles <= sh.small_tiles ? sh.tpc_small : sh.tpc;
      g = (t.ntiles + tpc - 1) / tpc;
    }
    // fused_finish counts CTAs in 20 bits (flags.cuh): larger tables loop
    g = std::min<int64_t>(g, kMaxGrid);
    return cap > 0 ? std::min<int>(cap, static_cast<int>(g)) : static_cast<int>(g);
  }
  // Register mover: one 64 KiB tile per CTA (at least the persistent grid's
  // CTA count), the TMA mover's finding again: forced onto aligned tables
  // (CECOLL_MOVER=reg) it goes from 0.83 / 0.91 of the copy peak (all-gather
  // / all-to-all, 64 MiB chunks, persistent 2 CTAs per SM) to 0.99 / 1.06,
  // and prelaunch_bcst's broadcast items from 0.86 to 0.99-1.02 at 16-64 MiB
  // (profiles/reg_shape_r02.txt). Tables with in-place swap items keep the
  // persistent grid (1-3% faster there). CECOLL_REG_TPC=k sets k tiles per
  // CTA; 0 restores the persistent grid everywhere.
  static const int reg_tpc = env_int("CECOLL_REG_TPC", 1);
  static const int reg_cap = env_int("CECOLL_SM_GRID", 0);  // a process-wide cap wins
  if (reg_tpc > 0 && reg_cap <= 0 && !(t.kinds & (1 << kItemSwap)))
    return std::max(mover_grid(t.mover, sms), std::min((t.ntiles + reg_tpc - 1) / reg_tpc, kMaxGrid));
  return mover_grid(t.mover, sms);
}

KernelCall items_call(const ItemTable& t, int grid, const FlagSet* fp) {
  KernelCall k;
  if (t.nitems <= 0 || t.ntiles <= 0 || t.nitems > kMaxItemsSmem) return k;
  if (grid > t.ntiles) grid = t.ntiles;
  k.grid = dim3(grid);
  if (t.mover == Mover::Tma) {
    // The attribute is per device; set it once per device (any thread may
    // launch, so the flags are atomic; devices beyond 64 set it every time).
    // Graph kernel nodes need it too: it is set here, before the node exists.
    static std::atomic<bool> configured[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64 || !configured[dev].load(std::memory_order_acquire)) {
      if (cudaFuncSetAttribute(tma_items_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem) !=
              cudaSuccess ||
          cudaFuncSetAttribute(tma_items_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem) !=
              cudaSuccess)
        return KernelCall{};
      if (dev < 64) configured[dev].store(true, std::memory_order_release);
    }
    static const int evict_first = [] {
      const char* e = std::getenv("CECOLL_TMA_EVICT_FIRST");
      return e ? std::atoi(e) : 0;
    }();
    const bool lag = tma_policy().shape(t.kinds & (1 << kItemFan)).lag == 1;
    const bool swp = t.kinds == (1 << kItemSwap);
    k.func = lag ? reinterpret_cast<const void*>(tma_items_kernel<1>) : reinterpret_cast<const void*>(tma_items_kernel<0>);
    k.block = dim3(32);
    k.smem = kTmaStages * (t.tile > 0 ? t.tile : kTmaTile) * (swp ? 2 : 1);
    k.push(static_cast<const Item*>(t.items));
    k.push(t.nitems);
    k.push(t.ntiles);
    k.push(t.tile > 0 ? t.tile : kTmaTile);
    k.push(t.uniform);
    k.push((evict_first ? 1 : 0) | (swp ? 2 : 0));
    k.push(fp ? *fp : FlagSet{});
    return k;
  }
  if (t.kinds == (1 << kItemCopy))
    k.func = reinterpret_cast<const void*>(reg_items_kernel<(1 << kItemCopy), 2>);
  else if (!(t.kinds & ((1 << kItemSwap) | (1 << kItemFan))))
    k.func = reinterpret_cast<const void*>(reg_items_kernel<(1 << kItemCopy) | (1 << kItemBcst), 2>);
  else
    k.func = reinterpret_cast<const void*>(reg_items_kernel<15, 1>);
  k.block = dim3(kRegThreads);
  k.push(static_cast<const Item*>(t.items));
  k.push(t.nitems);
  k.push(t.ntiles);
  k.push(t.uniform);
  k.push(fp ? *fp : FlagSet{});
  return k;
}

cudaError_t launch(const KernelCall& k, cudaStream_t stream) {
  if (!k.func) return cudaSuccess;
  void* args[12];
  k.params(args);
  return cudaLaunchKernel(k.func, k.grid, k.block, args, k.smem, stream);
}

cudaError_t launch_items(const ItemTable& t, int grid, cudaStream_t stream, const FlagSet* fp) {
  if (t.nitems <= 0 || t.ntiles <= 0) return cudaSuccess;
  if (t.nitems > kMaxItemsSmem) return cudaErrorInvalidValue;
  const KernelCall k = items_call(t, grid, fp);
  if (!k.func) return cudaErrorInvalidValue;
  return launch(k, stream);
}

cudaError_t launch_mc_store(const char* src, char* mc_dst, int64_t bytes, uint64_t* mc_flag, uint64_t epoch,
                            unsigned* ctr, int grid, cudaStream_t stream) {
  const int64_t nvec = bytes / 16;
  const int64_t need = (nvec + kRegThreads - 1) / kRegThreads;
  if (grid > need) grid = static_cast<int>(need > 0 ? need : 1);
  mc_store_kernel<<<grid, kRegThreads, 0, stream>>>(reinterpret_cast<const int4*>(src), mc_dst, nvec, mc_flag, epoch,
                                                     ctr);
  return cudaGetLastError();
}

KernelCall poll_call(uint64_t* const* flags, int n, uint64_t* err) {
  KernelCall k;
  if (n <= 0) return k;
  k.func = reinterpret_cast<const void*>(poll_kernel);
  k.grid = dim3((n + 127) / 128);
  k.block = dim3(128);
  k.push(flags);
  k.push(n);
  k.push(err);
  return k;
}

KernelCall signal_call(uint64_t* const* flags, int n) {
  KernelCall k;
  if (n <= 0) return k;
  k.func = reinterpret_cast<const void*>(signal_kernel);
  k.grid = dim3((n + 127) / 128);
  k.block = dim3(128);
  k.push(flags);
  k.push(n);
  return k;
}

KernelCall gate_call(uint64_t* trigger, const volatile uint64_t* cancel, uint64_t* seen,
                     cudaGraphConditionalHandle handle, uint64_t* err) {
  KernelCall k;
  k.func = reinterpret_cast<const void*>(gate_kernel);
  k.block = dim3(32);
  k.push(trigger);
  k.push(cancel);
  k.push(seen);
  k.push(handle);
  k.push(err);
  return k;
}

KernelCall gate_poll_call(uint64_t* const* flags, int n, const volatile uint64_t* cancel, uint64_t* seen,
                          uint64_t* skip, uint64_t* err) {
  KernelCall k;
  k.func = reinterpret_cast<const void*>(gate_poll_kernel);
  k.block = dim3(32);
  k.push(flags);
  k.push(n);
  k.push(cancel);
  k.push(seen);
  k.push(skip);
  k.push(err);
  return k;
}

cudaError_t launch_poll(uint64_t* const* flags, int n, uint64_t* err, cudaStream_t stream) {
  return launch(poll_call(flags, n, err), stream);
}

cudaError_t launch_signal(uint64_t* const* flags, int n, cudaStream_t stream) {
  return launch(signal_call(flags, n), stream);
}

// Loads every kernel of this file on the current device (and sets the TMA
// mover's shared-memory attribute). With CUDA's lazy module loading (the
// default) a kernel's first launch loads its module, and that load can wait
// behind kernels already running on the device: an armed prelaunch gate
// spinning on a trigger that this host thread has yet to post. Measured on
// B200: the first eager collective with signal kernels stalled until a 20 s
// flag poll timed out (tools/b2b_stress.py). Called for every device of a
// world at init, so no launch of ours ever loads a module.
cudaError_t preload_kernels() {
  cudaFuncAttributes a;
  const void* fns[] = {
      reinterpret_cast<const void*>(reg_items_kernel<(1 << kItemCopy), 2>),
      reinterpret_cast<const void*>(reg_items_kernel<(1 << kItemCopy) | (1 << kItemBcst), 2>),
      reinterpret_cast<const void*>(reg_items_kernel<15, 1>),
      reinterpret_cast<const void*>(tma_items_kernel<0>),
      reinterpret_cast<const void*>(tma_items_kernel<1>),
      reinterpret_cast<const void*>(poll_kernel),
      reinterpret_cast<const void*>(signal_kernel),
      reinterpret_cast<const void*>(gate_kernel),
      reinterpret_cast<const void*>(gate_poll_kernel),
      reinterpret_cast<const void*>(mc_store_kernel),
  };
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaFuncSetAttribute(tma_items_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(tma_items_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
}

}  // namespace cecoll
