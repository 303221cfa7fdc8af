// Helpers shared by the runtime's translation units (world.cpp, lower.cpp,
// exec.cpp, util.cpp). Not part of the C ABI.
#pragma once

#include <algorithm>
#include <map>
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
// Writes a plan table (src, or zeros when src is null) into device memory of
// the current device and returns once the bytes have landed: on a private
// per-device stream, synchronised. Plain cudaMemcpy from pageable memory may
// return before its DMA completes and cudaMemset is asynchronous, both on the
// legacy stream that the callers' non-blocking streams do not wait for — a
// plan's first kernel could read the table before it is written (seen once
// in eight fresh two-process runs, tools/pull_race_probe.py).
Status write_device(void* dst, const void* src, size_t bytes);
// Copy commands: one cudaMemcpyAsync per copy, in order on stream s.
Status issue_copies(World* w, const std::vector<Copy>& copies, cudaStream_t s);
Status ensure_lanes(RankState* rs, int n);
// Where an executor's commands go (sink.cpp): StreamSink
// submits them to their streams now; GraphSink adds them as explicit nodes of
// per-unit graphs (recorded command lists, prelaunch bodies) with stream
// order and event record/wait turned into node dependencies. Both count the
// commands in the world's counters.
class Sink {
 public:
  virtual ~Sink() = default;
  virtual bool graph() const = 0;
  virtual Status memops(World* w, cudaStream_t s, const MemOps& ops) = 0;
  virtual Status copies(World* w, const std::vector<Copy>& c, cudaStream_t s) = 0;
  virtual Status kernel(World* w, cudaStream_t s, const KernelCall& k) = 0;
  virtual Status record(World* w, cudaEvent_t e, cudaStream_t s) = 0;
  virtual Status wait(World* w, cudaStream_t s, cudaEvent_t e) = 0;
  // Tracing (no-ops unless the world traces): a timing event in stream order
  // (an event-record node in a graph), and a host span of the submission
  // (none while building a graph: the host cost is the graph launch's).
  virtual cudaEvent_t mark(World* w, int device, cudaStream_t s) = 0;
  virtual void host_span(World* w, const std::string& name, double b_us) = 0;
};

class StreamSink : public Sink {
 public:
  bool graph() const override { return false; }
  Status memops(World* w, cudaStream_t s, const MemOps& ops) override;
  Status copies(World* w, const std::vector<Copy>& c, cudaStream_t s) override;
  Status kernel(World* w, cudaStream_t s, const KernelCall& k) override;
  Status record(World* w, cudaEvent_t e, cudaStream_t s) override;
  Status wait(World* w, cudaStream_t s, cudaEvent_t e) override;
  cudaEvent_t mark(World* w, int device, cudaStream_t s) override;
  void host_span(World* w, const std::string& name, double b_us) override;
};

class GraphSink : public Sink {
 public:
  // Streams not mapped to another graph add their nodes to graphs[0].
  explicit GraphSink(std::vector<cudaGraph_t> graphs);
  void map(cudaStream_t s, int graph);
  bool graph() const override { return true; }
  Status memops(World* w, cudaStream_t s, const MemOps& ops) override;
  Status copies(World* w, const std::vector<Copy>& c, cudaStream_t s) override;
  Status kernel(World* w, cudaStream_t s, const KernelCall& k) override;
  Status record(World* w, cudaEvent_t e, cudaStream_t s) override;
  Status wait(World* w, cudaStream_t s, cudaEvent_t e) override;
  cudaEvent_t mark(World* w, int device, cudaStream_t s) override;
  void host_span(World*, const std::string&, double) override {}
  // Any other node type (the prelaunch conditional node), in stream order.
  Status add_node(cudaStream_t s, cudaGraphNodeParams* params, cudaGraphNode_t* out);
  const std::vector<cudaGraphNode_t>& tail(cudaStream_t s);
  int nodes() const { return nodes_; }

 private:
  struct Tail {
    int graph = 0;
    std::vector<cudaGraphNode_t> deps;
  };
  Tail& tail_of(cudaStream_t s);
  Status added(Tail& t, cudaGraphNode_t node);
  std::vector<cudaGraph_t> graphs_;
  std::map<cudaStream_t, Tail> tails_;
  std::map<cudaEvent_t, Tail> events_;
  int nodes_ = 0;
};

// The signal kernel for other devices' flags (see split_remote in lower.cpp).
Status signal_remote(World* w, Sink& sink, uint64_t** tab, size_t n, cudaStream_t s);
// Tracing (trace.cpp); every call is a no-op unless the world traces.
// trace_mark records a timing event on `s` (nullptr when not tracing).
cudaEvent_t trace_mark(World* w, int device, cudaStream_t s);
void trace_span(World* w, const std::string& name, int pid, int tid, int device, cudaEvent_t b, cudaEvent_t e);
double trace_host_now(World* w);
void trace_host_span(World* w, const std::string& name, double b_us);
// Records a unit's prelaunch graph (lower.cpp).
Status build_graph(World* w, Plan* p, Unit& u);

}  // namespace cecoll
