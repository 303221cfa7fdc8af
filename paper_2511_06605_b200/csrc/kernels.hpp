// sm_100a data-movement kernels shared by the SM path and by the command
// types a copy engine cannot execute (two-destination broadcast, in-place
// swap; compiler.cpp:166-239).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cecoll {

enum ItemKind : int32_t { kItemCopy = 0, kItemBcst = 1, kItemSwap = 2 };

// One transfer. Copy: src -> dst. Bcst: src -> dst and dst2 (one read).
// Swap: dst <-> src exchanged in place (both read before either is written,
// per element, so the exchange has no observable intermediate state,
// verifier.cpp:126-137).
struct Item {
  const char* src;
  char* dst;
  char* dst2;
  int64_t bytes;
  int32_t kind;
  int32_t first_tile;  // prefix sum of tiles over the item table
};

// Bytes per tile: one CTA moves one tile per step (256 threads x 8 x 16 B).
constexpr int64_t kTileBytes = 32 * 1024;
constexpr int kCopyThreads = 256;
constexpr int kMaxItemsSmem = 1024;

// Moves every item of `items` (device-resident table) with a grid-stride loop
// over tiles. `ntiles` is items[nitems-1].first_tile + tiles of the last item.
cudaError_t launch_items(const Item* items, int nitems, int ntiles, int grid, cudaStream_t stream);

int64_t tiles_for(int64_t bytes);

// Flag kernels used inside recorded (prelaunch) graphs, where stream memory
// operations are not allowed in conditional bodies.
//  poll:   every flags[i] >= 1, then reset to 0 (ld.acquire.sys spin with a
//          globaltimer bound; on timeout *err |= 1 and the kernel exits).
//  signal: flags[i] = 1 with st.release.sys after a system-scope fence.
//  gate:   wait for the next host post (pinned memory, see kernels.cu); a
//          "go" post opens the conditional body, a "cancel" post skips it.
cudaError_t launch_poll(uint64_t* const* flags, int n, uint64_t* err, cudaStream_t stream);
cudaError_t launch_signal(uint64_t* const* flags, int n, cudaStream_t stream);
cudaError_t launch_gate(volatile uint64_t* posted, uint64_t* consumed, cudaGraphConditionalHandle handle,
                        uint64_t* err, cudaStream_t stream);

}  // namespace cecoll
