// Helpers shared by the runtime's translation units (world.cpp, lower.cpp,
// exec.cpp, util.cpp). Not part of the C ABI.
#pragma once

#include <string>
#include <vector>

#include "runtime.hpp"

namespace cecoll {

Status fail(int code, const std::string& msg);
Status cuda_fail(cudaError_t e, const char* what, const char* file, int line);
Status cu_fail(CUresult r, const char* what, const char* file, int line);

#define CUDA_TRY(expr)                                      \
  do {                                                      \
    cudaError_t e_ = (expr);                                \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr, __FILE__, __LINE__); \
  } while (0)

#define CU_TRY(expr)                                       \
  do {                                                     \
    CUresult r_ = (expr);                                  \
    if (r_ != CUDA_SUCCESS) return cu_fail(r_, #expr, __FILE__, __LINE__); \
  } while (0)

#define STATUS_TRY(expr)         \
  do {                           \
    Status s_ = (expr);          \
    if (!s_.ok()) return s_;     \
  } while (0)

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev_);
    if (dev >= 0 && dev != prev_) cudaSetDevice(dev);
  }
  ~DeviceGuard() { cudaSetDevice(prev_); }

 private:
  int prev_ = 0;
};

CUstreamBatchMemOpParams op_write(uint64_t* addr, uint64_t v);
CUstreamBatchMemOpParams op_wait(uint64_t* addr, uint64_t v);
// Poll + reset of one slot (the reset keeps graph replays value-constant).
void add_poll(MemOps& ops, uint64_t* addr);
// cuStreamBatchMemOp in batches of at most 255 operations.
Status submit(World* w, cudaStream_t s, const MemOps& ops);
// Copy commands: one cuMemcpyBatchAsync (allow_batch, non-legacy stream) or
// one cudaMemcpyAsync per copy.
Status issue_copies(World* w, const std::vector<Copy>& copies, cudaStream_t s, bool allow_batch);
Status ensure_lanes(RankState* rs, int n);
// Signal kernel for flags on other devices (see split_remote in lower.cpp).
Status signal_remote(World* w, uint64_t** tab, size_t n, cudaStream_t s);
// Tracing (trace.cpp); every call is a no-op unless the world traces.
// trace_mark records a timing event on `s` (nullptr when not tracing).
cudaEvent_t trace_mark(World* w, int device, cudaStream_t s);
void trace_span(World* w, const std::string& name, int pid, int tid, int device, cudaEvent_t b, cudaEvent_t e);
double trace_host_now(World* w);
void trace_host_span(World* w, const std::string& name, double b_us);
// Records a unit's prelaunch graph (lower.cpp).
Status build_graph(World* w, Plan* p, Unit& u);

}  // namespace cecoll
