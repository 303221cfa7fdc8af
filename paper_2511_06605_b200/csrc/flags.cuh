// Device side of the flag protocol, shared by the movers
// (kernels.cu) and the reduce-scatter kernel (reduce.cu). Internal linkage:
// included inside each translation unit's anonymous namespace.
#pragma once

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

// One flag: spin (ld.acquire.sys, 20 s bound) until *p >= 1.
__device__ __forceinline__ void wait_flag(const uint64_t* p, uint64_t* err) {
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys(p) < 1) {
    if (globaltimer() - t0 > kPollTimeoutNs) {
      atomicOr(reinterpret_cast<unsigned long long*>(err), 1ull);
      return;
    }
    __nanosleep(32);
  }
}

// Fused prologue, one full warp of a CTA (warp-level polling): CTA 0 first
// writes the folded start signals, then lane i waits for flags i, i+32, ...
// The closing __syncwarp orders every lane's acquire before the warp's (and,
// after the caller's __syncthreads, the CTA's) data accesses.
__device__ __forceinline__ void fused_wait(const FlagSet& f) {
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0)
    for (int i = lane; i < f.npre; i += 32) st_release_sys(f.pre[i], 1);
  for (int i = lane; i < f.npoll; i += 32) wait_flag(f.polls[i], f.err);
  __syncwarp();
}

// Fused epilogue (thread 0 of a CTA, after the CTA's data writes are
// complete: bar.sync for the register mover, bulk wait_group + proxy fence
// for TMA). With outgoing signals the CTA's writes are published by one
// system-scope release fence before its ticket; the last CTA's acq_rel
// ticket then orders every CTA's writes (and its own resets) before the
// st.release.sys signals — the barrier-then-one-thread-fence pattern, no
// fence per thread. Without signals nothing outside this unit waits on the
// data, and the kernel boundary publishes it: no system fence at all (they
// cost several microseconds each when every CTA issues them).
__device__ __forceinline__ void fused_finish(const FlagSet& f) {
  if (f.nsig) asm volatile("fence.acq_rel.sys;" ::: "memory");
  unsigned ticket;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(ticket) : "l"(f.ctr) : "memory");
  if (ticket != gridDim.x - 1) return;
  *f.ctr = 0;
  // Every CTA passed its polls before taking its ticket: reset them for the
  // next collective (its writers only write again after our signals).
  for (int i = 0; i < f.npoll; ++i) *f.polls[i] = 0;
  for (int i = 0; i < f.nsig; ++i) st_release_sys(f.sigs[i], 1);
}

