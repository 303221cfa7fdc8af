// sm_100a data-movement kernels shared by the SM path and by the command
// types a copy engine cannot execute (two-destination broadcast, in-place
// swap; compiler.cpp:166-239), plus the flag kernels of recorded graphs.
#pragma once

#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

namespace cecoll {

// A kernel launch as data: launched on a stream (eager submission) or added
// to a graph as a kernel node (recorded command lists and prelaunch bodies
// are built node by node, never by stream capture; exec.cpp GraphSink).
// func == nullptr means there is nothing to launch.
struct KernelCall {
  const void* func = nullptr;
  dim3 grid{1, 1, 1};
  dim3 block{1, 1, 1};
  unsigned smem = 0;
  int nargs = 0;
  unsigned used = 0;
  unsigned short off[12] = {};
  alignas(16) unsigned char buf[384] = {};

  template <class T>
  void push(const T& v) {
    const unsigned o = (used + alignof(T) - 1) & ~static_cast<unsigned>(alignof(T) - 1);
    std::memcpy(buf + o, &v, sizeof(T));
    off[nargs++] = static_cast<unsigned short>(o);
    used = o + sizeof(T);
  }
  // kernelParams for cudaLaunchKernel / cudaKernelNodeParams (pointers into buf).
  void params(void** out) const {
    for (int i = 0; i < nargs; ++i) out[i] = const_cast<unsigned char*>(buf + off[i]);
  }
};

cudaError_t launch(const KernelCall& k, cudaStream_t stream);

enum ItemKind : int32_t { kItemCopy = 0, kItemBcst = 1, kItemSwap = 2, kItemFan = 3 };

// One transfer. Copy: src -> dst. Bcst: src -> dst and dst2 (one read).
// Swap: dst <-> src exchanged in place (both read before either is written,
// per element, so the exchange has no observable intermediate state,
// verifier.cpp:126-137). Fan: src -> fan[0..nfan) with one read — the
// all-gather source chunk written to every rank's slot (the n-destination
// generalisation of the reference's two-destination broadcast,
// compiler.cpp:166-205; on a multi-GPU node the NVLS multicast analog).
struct Item {
  const char* src;
  char* dst;
  char* dst2;
  char* const* fan;  // device array of nfan destinations (kItemFan)
  int64_t bytes;
  int32_t kind;
  int32_t first_tile;  // prefix sum of tiles over the item table
  int32_t nfan;
  int32_t pad;
};
constexpr int kMaxFan = 32;

// Which kernel moves a table:
//  Reg: 512-thread CTAs, 64 KiB tiles staged through registers (eight 16-byte
//       loads in flight per thread), any alignment, any item kind.
//  Tma: copy / fan tables and pure swap tables whose items are 16-byte
//       aligned with sizes that are multiples of 16: one elected thread per
//       CTA streams 4-32 KiB tiles (swap: both sides of a 4-16 KiB exchange
//       per stage) through a 4-stage shared-memory ring with cp.async.bulk
//       (global->shared on an mbarrier, shared->global as a bulk group; a
//       fan tile is loaded once and stored once per destination).
enum class Mover : int { Reg = 0, Tma = 1 };

struct ItemTable {
  Item* items = nullptr;  // device memory
  int nitems = 0;
  int ntiles = 0;
  Mover mover = Mover::Reg;
  int kinds = 1;  // bitmask of (1 << ItemKind) present
  int tile = 0;     // bytes per tile (0: the mover's default)
  int uniform = 0;  // tiles per item when every item has the same count, else 0
};

constexpr int kMaxItemsSmem = 1024;
// Largest grid of an item or reduction kernel: fused_finish's tickets count
// CTAs in 20 bits (flags.cuh); CTAs past the grid loop over further tiles.
constexpr int kMaxGrid = 1 << 19;

int64_t mover_tile_bytes(Mover m);
// Tile size of a table of items of `sizes` bytes on a device with `sms` SMs
// (budget: the plan's SM budget in CTAs, 0 = none): the register mover uses
// 64 KiB tiles; the TMA mover the smallest tile (4-32 KiB) that leaves at
// most one tile per resident CTA, else its streaming tile (kernels.cu
// TmaPolicy; 32 KiB under a budget).
int table_tile(Mover m, const std::vector<int64_t>& sizes, int sms, int budget = 0, bool has_fan = false,
               bool swap = false);
// CTAs of the TMA mover resident per SM when its ring holds `tile`-byte stages.
int tma_resident(int tile);
// Tiles of one item of `bytes` at `tile` bytes per tile.
inline int64_t tiles_of(int64_t bytes, int tile) { return (bytes + tile - 1) / tile; }
// Grid that fills the device for mover m (multiple of the SM count).
int mover_grid(Mover m, int sms);
// Grid for one table (honours CECOLL_SM_TILES_PER_CTA).
int mover_grid_for(const ItemTable& t, int sms);

// Flag work fused into an item kernel (one launch instead of poll kernel /
// memops -> mover -> signal kernel / memops). Before moving, thread 0 of
// every CTA waits for polls[i] >= 1 (ld.acquire.sys, 20 s bound: on timeout
// *err |= 1 and it proceeds). After its tiles, every CTA fences (system
// scope) and takes a ticket on *ctr; the last CTA resets *ctr and every
// polls[i] to 0 (all CTAs have passed their polls by then), then writes
// sigs[i] = 1 with st.release.sys. Tables and ctr live in device memory;
// ctr starts at 0.
struct FlagSet {
  // Written (= 1, st.release.sys) by thread 0 of CTA 0 before anything else:
  // the unit's start signals ("my buffers may be used"), when folded in.
  uint64_t* const* pre = nullptr;
  int npre = 0;
  uint64_t* const* polls = nullptr;
  int npoll = 0;
  uint64_t* const* sigs = nullptr;
  int nsig = 0;
  unsigned* ctr = nullptr;
  uint64_t* err = nullptr;
  // Non-null: written by a gate_poll kernel before the mover — 0 move, 1 a
  // cancelled prelaunch instance (no data, no signals), 2 a poll timed out
  // (no data, signals still written).
  const uint64_t* skip = nullptr;
  // Folded prelaunch gate (a single-kernel prelaunch body):
  // a non-null `epoch` (device word: instances of this body completed so far)
  // makes the kernel itself the gate. polls[0] is then the unit's trigger
  // word (1 go, 2 cancel; flags.cuh take_trigger). CTA 0 takes the trigger,
  // writes the start signals, polls and resets the other flags, and
  // publishes the outcome in *gate (device word: (epoch + 1) * 4 + state)
  // for the other CTAs; a cancel makes every CTA skip data and signals. The
  // last CTA (finish ticket, always present here) advances *epoch.
  uint64_t* epoch = nullptr;
  const volatile uint64_t* cancel = nullptr;  // host cancel count (flags.cuh take_trigger)
  uint64_t* seen = nullptr;                   // cancels honoured (device)
  uint64_t* gate = nullptr;
};

cudaError_t launch_items(const ItemTable& t, int grid, cudaStream_t stream, const FlagSet* flags = nullptr);
KernelCall items_call(const ItemTable& t, int grid, const FlagSet* flags = nullptr);

// Reduce-scatter reduction: dst[e] = op over srcs[0..nsrc)
// in source order of src[e], accumulated in fp32 and rounded once (RNE) to
// the element type — the same order as the oracle (ora_reduce_scatter).
enum Dtype : int32_t { kF32 = 0, kBF16 = 1, kF16 = 2 };
enum RedOp : int32_t { kSum = 0, kMax = 1, kMin = 2 };

inline int dtype_bytes(int dtype) { return dtype == kF32 ? 4 : 2; }

struct RedItem {
  const char* const* srcs;  // device array of nsrc pointers
  char* dst;
  int64_t elems;
  int32_t nsrc;
  int32_t first_tile;
  int32_t vec;  // all pointers 16-byte aligned: vectorised body
  int32_t pad;
};

struct RedTable {
  RedItem* items = nullptr;
  int nitems = 0;
  int ntiles = 0;
  int dtype = kF32;
  int op = kSum;
};

constexpr int64_t kRedTileElems = 4096;
cudaError_t launch_reduce(const RedTable& t, int grid, cudaStream_t stream, const FlagSet* flags = nullptr);
KernelCall reduce_call(const RedTable& t, int grid, const FlagSet* flags = nullptr);

// Flag kernels used inside recorded (prelaunch) graphs, where stream memory
// operations are not allowed in conditional bodies.
//  poll:   every flags[i] >= 1, then reset to 0 (ld.acquire.sys spin with a
//          globaltimer bound; on timeout *err |= 1 and the kernel exits).
//  signal: flags[i] = 1 with st.release.sys after a system-scope fence.
//  gate:   take the unit's trigger (flags.cuh take_trigger: the device
//          trigger word, or a host cancel): "go" opens the conditional body,
//          "cancel" skips it.
// Load every kernel of the library on the current device (called at world
// init for each device; see kernels.cu).
cudaError_t preload_kernels();
cudaError_t preload_reduce_kernels();
cudaError_t launch_poll(uint64_t* const* flags, int n, uint64_t* err, cudaStream_t stream);
cudaError_t launch_signal(uint64_t* const* flags, int n, cudaStream_t stream);
//  gate_poll: the gate of a kernel-only prelaunch body (no conditional node):
//          takes the trigger (word flags[0]); on "go" polls flags[1..n) (>= 1,
//          reset to 0, as poll) and writes *skip = 0; on "cancel" writes
//          *skip = 1 so the mover after it returns at once.
KernelCall poll_call(uint64_t* const* flags, int n, uint64_t* err);
KernelCall signal_call(uint64_t* const* flags, int n);
KernelCall gate_call(uint64_t* trigger, const volatile uint64_t* cancel, uint64_t* seen,
                     cudaGraphConditionalHandle handle, uint64_t* err);
KernelCall gate_poll_call(uint64_t* const* flags, int n, const volatile uint64_t* cancel, uint64_t* seen,
                          uint64_t* skip, uint64_t* err);

// NVLS multicast all-gather store (mcast.cpp, experimental): src (bytes, a
// multiple of 16, 16-byte aligned) -> mc_dst with multimem.st (the switch
// writes every GPU of the multicast group); after every CTA's stores, the
// last CTA publishes *mc_flag = epoch with multimem.st.release.sys. ctr is a
// zeroed device word (restored to 0).
cudaError_t launch_mc_store(const char* src, char* mc_dst, int64_t bytes, uint64_t* mc_flag, uint64_t epoch,
                            unsigned* ctr, int grid, cudaStream_t stream);

}  // namespace cecoll
