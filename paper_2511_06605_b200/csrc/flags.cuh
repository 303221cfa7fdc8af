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

__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// One flag: spin (ld.acquire.sys, 20 s bound) until *p >= 1. Returns false
// (and sets bit 0 of *err) on timeout.
__device__ __forceinline__ bool wait_flag(const uint64_t* p, uint64_t* err) {
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys(p) < 1) {
    if (globaltimer() - t0 > kPollTimeoutNs) {
      atomicOr(reinterpret_cast<unsigned long long*>(err), 1ull);
      return false;
    }
    __nanosleep(32);
  }
  return true;
}

// What a CTA may do after its prologue.
enum : int { kGo = 0, kTimedOut = 1, kCancelled = 2 };

// Trigger of a prelaunch unit. The caller stream writes 1 ("go") into the
// unit's device trigger word when it triggers the unit; the gate spins on
// that word and takes it by resetting it to 0 (the next trigger is only
// written after this instance completes). A cancel comes from the host
// without any stream (a stream could share a hardware queue with the armed
// graph and never run): the host raises a count in pinned memory
// (`cancel`, exec.cpp cancel_armed) and the gate compares it with the count
// it has already honoured (`seen`, device) once every 256 polls — PCIe reads
// of host memory stay off the go path (round 1's gate read a host post on
// every trigger: ~2 us per prelaunch collective, tools/prelaunch_probe.cu).
// No bound: an armed instance waits as long as its caller leaves it armed.
// Returns 1 (go) or 2 (cancel).
__device__ __forceinline__ uint64_t take_trigger(uint64_t* p, const volatile uint64_t* cancel, uint64_t* seen,
                                                 uint64_t* err) {
  uint64_t v;
  for (unsigned i = 1;; ++i) {
    v = ld_acquire_sys(p);
    if (v) break;
    if ((i & 255) == 0) {
      const uint64_t c = *cancel;
      if (c > *seen) {
        *seen = c;
        return 2;
      }
    }
    __nanosleep(32);
  }
  *p = 0;
  if (v != 1) atomicOr(reinterpret_cast<unsigned long long*>(err), 2ull);
  return v;
}

// Folded prelaunch gate (FlagSet::epoch, one full warp of every CTA). CTA 0
// alone takes the unit's trigger word (f.polls[0]), writes the folded start
// signals, polls the other flags (one set of system-scope pollers) and resets
// them — their writers only write again after this instance completes or
// signals — then publishes the outcome in the device word *gate =
// (epoch + 1) * 4 + state; every other CTA waits for that word (device
// scope). *epoch counts completed instances: instances run one at a time on
// the unit's arm stream and the previous one's last CTA advanced it, so every
// CTA of this instance reads the same value (no per-instance kernel
// parameters, so arming is a plain graph launch). CTA 0's system-scope
// acquire of the flags followed by its release of the gate word orders the
// flag writers' data before every CTA's accesses.
__device__ __forceinline__ int folded_gate(const FlagSet& f) {
  const int lane = threadIdx.x & 31;
  uint64_t base = 0;
  if (lane == 0) base = (*reinterpret_cast<const volatile uint64_t*>(f.epoch) + 1) * 4;
  base = __shfl_sync(0xffffffffu, base, 0);
  int state;
  if (blockIdx.x == 0) {
    uint64_t kind = 0;
    if (lane == 0) kind = take_trigger(f.polls[0], f.cancel, f.seen, f.err);
    kind = __shfl_sync(0xffffffffu, kind, 0);
    if (kind != 1) {
      state = kCancelled;
    } else {
      for (int i = lane; i < f.npre; i += 32) st_release_sys(f.pre[i], 1);
      bool ok = true;
      for (int i = 1 + lane; i < f.npoll; i += 32) {
        const bool got = wait_flag(f.polls[i], f.err);
        if (got) *f.polls[i] = 0;
        ok &= got;
      }
      state = __all_sync(0xffffffffu, ok) ? kGo : kTimedOut;
    }
    if (lane == 0) st_release_gpu(f.gate, base + state);
  } else {
    uint64_t v = 0;
    if (lane == 0)
      while ((v = ld_acquire_gpu(f.gate)) < base) __nanosleep(64);
    v = __shfl_sync(0xffffffffu, v, 0);
    state = static_cast<int>(v - base);
  }
  return state;
}

// Fused prologue, one full warp of a CTA (warp-level polling): the folded
// gate if any, then CTA 0 writes the folded start signals, then lane i waits
// for flags i, i+32, ... The closing vote orders every lane's acquire before
// the warp's (and, after the caller's __syncthreads, the CTA's) data
// accesses. Returns (warp-uniform):
//  kGo        move the data;
//  kTimedOut  a poll gave up after 20 s: the peer never released its buffer,
//             so nothing may be written into it — but the done signals are
//             still written (fused_finish), so peers waiting on them (stream
//             memory-operation waits have no bound) do not hang; the error
//             word makes the world's failure sticky;
//  kCancelled a cancelled prelaunch instance: no data, no signals.
// When a skip word is set (a gate_poll kernel ran first) it decides instead;
// the kernels read it at entry (read_skip), in parallel with their table
// loads, and pass the value in.
__device__ __forceinline__ uint64_t read_skip(const FlagSet& f) {
  return f.skip ? *reinterpret_cast<const volatile uint64_t*>(f.skip) : 0;
}

__device__ __forceinline__ int fused_wait(const FlagSet& f, uint64_t sk) {
  const int lane = threadIdx.x & 31;
  if (f.skip) return sk == 0 ? kGo : sk == 1 ? kCancelled : kTimedOut;
  if (f.epoch) return folded_gate(f);
  if (blockIdx.x == 0)
    for (int i = lane; i < f.npre; i += 32) st_release_sys(f.pre[i], 1);
  bool ok = true;
  for (int i = lane; i < f.npoll; i += 32) ok &= wait_flag(f.polls[i], f.err);
  return __all_sync(0xffffffffu, ok) ? kGo : kTimedOut;
}

// Fused epilogue (thread 0 of a CTA, after the CTA's data writes are
// complete: bar.sync for the register mover, bulk wait_group + proxy fence
// for TMA). With outgoing signals the CTA's writes are published by one
// system-scope release fence before its ticket; the last CTA's acq_rel
// ticket then orders every CTA's writes (and its own resets) before the
// st.release.sys signals — the barrier-then-one-thread-fence pattern, no
// fence per thread. Without signals nothing outside this unit waits on the
// data, and the kernel boundary publishes it: no system fence at all (they
// cost several microseconds each when every CTA issues them). `state` is
// the CTA's fused_wait result: the last CTA resets the polls only if every
// CTA passed them, and signals unless the instance was cancelled.
__device__ __forceinline__ void fused_finish(const FlagSet& f, int state) {
  if (f.nsig && state == kGo) asm volatile("fence.acq_rel.sys;" ::: "memory");
  unsigned ticket;
  // tickets count up by 1 per CTA; a CTA whose poll timed out adds 1 << 20
  // as well, so the last CTA sees whether anyone did (grids stay below 2^20)
  const unsigned add = state == kTimedOut ? (1u << 20) + 1u : 1u;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(ticket) : "l"(f.ctr), "r"(add) : "memory");
  if ((ticket & 0xFFFFFu) != gridDim.x - 1) return;
  *f.ctr = 0;
  if (f.epoch) *f.epoch += 1;       // a folded body: this instance is complete
  if (state == kCancelled) return;  // uniform: every CTA read the same gate / skip word
  // Every CTA passed its polls before taking its ticket: reset them for the
  // next collective (its writers only write again after our signals). A
  // folded gate has reset them already.
  if (state == kGo && (ticket >> 20) == 0 && !f.epoch)
    for (int i = 0; i < f.npoll; ++i) *f.polls[i] = 0;
  for (int i = 0; i < f.nsig; ++i) st_release_sys(f.sigs[i], 1);
}
