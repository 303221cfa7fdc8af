// Where the executors' commands go.
//
// StreamSink submits every command to its CUDA stream now (eager launches).
// GraphSink turns the same command sequence into explicit graph nodes —
// memcpy nodes for copies, batch-mem-op nodes for stream memory operations
// (flag polls and writes), kernel nodes for the movers and flag kernels —
// tracking per stream the nodes that the next command depends on, and per
// event the nodes it was recorded behind, exactly as stream order and
// cudaEventRecord / cudaStreamWaitEvent would order them. No stream is ever
// put in capture mode, so a device-wide synchronisation in another thread
// cannot race a recording (the round-1 crash).
#include <cstring>

#include "internal.hpp"

namespace cecoll {

// ---------------------------------------------------------------------------
// StreamSink
// ---------------------------------------------------------------------------

Status StreamSink::memops(World* w, cudaStream_t s, const MemOps& ops) { return submit(w, s, ops); }

Status StreamSink::copies(World* w, const std::vector<Copy>& c, cudaStream_t s) {
  return issue_copies(w, c, s);
}

Status StreamSink::kernel(World* w, cudaStream_t s, const KernelCall& k) {
  if (!k.func) return {};
  CUDA_TRY(launch(k, s));
  ++w->counters[kCtrKernels];
  ++w->counters[kCtrApiCalls];
  return {};
}

Status StreamSink::record(World* w, cudaEvent_t e, cudaStream_t s) {
  CUDA_TRY(cudaEventRecord(e, s));
  ++w->counters[kCtrApiCalls];
  return {};
}

Status StreamSink::wait(World* w, cudaStream_t s, cudaEvent_t e) {
  CUDA_TRY(cudaStreamWaitEvent(s, e, 0));
  ++w->counters[kCtrApiCalls];
  return {};
}

cudaEvent_t StreamSink::mark(World* w, int device, cudaStream_t s) { return trace_mark(w, device, s); }

void StreamSink::host_span(World* w, const std::string& name, double b_us) { trace_host_span(w, name, b_us); }

// ---------------------------------------------------------------------------
// GraphSink
// ---------------------------------------------------------------------------

// While the world traces, a timing event becomes an event-record node in
// stream order: every replay of the graph re-records it (a traced graph is
// launched once per trace, exec.cpp launch_traced).
cudaEvent_t GraphSink::mark(World* w, int device, cudaStream_t s) {
  if (!w->tracer) return nullptr;
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  w->tracer->events.push_back({e, device});
  Tail& t = tail_of(s);
  cudaGraphNode_t node = nullptr;
  if (cudaGraphAddEventRecordNode(&node, graphs_[t.graph], t.deps.data(), t.deps.size(), e) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  added(t, node);
  return e;
}

GraphSink::GraphSink(std::vector<cudaGraph_t> graphs) : graphs_(std::move(graphs)) {}

void GraphSink::map(cudaStream_t s, int graph) { tails_[s].graph = graph; }

GraphSink::Tail& GraphSink::tail_of(cudaStream_t s) {
  auto it = tails_.find(s);
  if (it == tails_.end()) it = tails_.emplace(s, Tail{}).first;
  return it->second;
}

const std::vector<cudaGraphNode_t>& GraphSink::tail(cudaStream_t s) { return tail_of(s).deps; }

Status GraphSink::added(Tail& t, cudaGraphNode_t node) {
  t.deps.assign(1, node);
  ++nodes_;
  return {};
}

Status GraphSink::memops(World* w, cudaStream_t s, const MemOps& ops) {
  if (ops.empty()) return {};
  const DriverApi* d = driver_api();
  if (!d) return fail(CECOLL_NO_DEVICE, "no CUDA driver");
  CUcontext ctx = nullptr;
  CU_TRY(d->CtxGetCurrent(&ctx));
  Tail& t = tail_of(s);
  size_t i = 0;
  while (i < ops.size()) {  // one node per batch of at most 255 operations, as submit()
    const unsigned count = static_cast<unsigned>(std::min<size_t>(255, ops.size() - i));
    CUDA_BATCH_MEM_OP_NODE_PARAMS np;
    std::memset(&np, 0, sizeof(np));
    np.ctx = ctx;
    np.count = count;
    np.paramArray = const_cast<CUstreamBatchMemOpParams*>(ops.data() + i);
    np.flags = 0;
    CUgraphNode node = nullptr;
    CU_TRY(d->GraphAddBatchMemOpNode(&node, graphs_[t.graph], t.deps.data(), t.deps.size(), &np));
    STATUS_TRY(added(t, node));
    for (unsigned k = 0; k < count; ++k) {
      if (ops[i + k].operation == CU_STREAM_MEM_OP_WRITE_VALUE_64) ++w->counters[kCtrFlagWrites];
      else ++w->counters[kCtrFlagWaits];
    }
    ++w->counters[kCtrApiCalls];
    i += count;
  }
  return {};
}

Status GraphSink::copies(World* w, const std::vector<Copy>& c, cudaStream_t s) {
  // a recorded lane keeps its copies back to back as a chain of memcpy nodes
  Tail& t = tail_of(s);
  for (const Copy& cp : c) {
    cudaGraphNode_t node = nullptr;
    CUDA_TRY(cudaGraphAddMemcpyNode1D(&node, graphs_[t.graph], t.deps.data(), t.deps.size(), cp.dst, cp.src,
                                      static_cast<size_t>(cp.bytes), cudaMemcpyDefault));
    STATUS_TRY(added(t, node));
    ++w->counters[kCtrCopies];
    ++w->counters[kCtrApiCalls];
  }
  return {};
}

Status GraphSink::kernel(World* w, cudaStream_t s, const KernelCall& k) {
  if (!k.func) return {};
  Tail& t = tail_of(s);
  void* args[12];
  k.params(args);
  cudaKernelNodeParams kp;
  std::memset(&kp, 0, sizeof(kp));
  kp.func = const_cast<void*>(k.func);
  kp.gridDim = k.grid;
  kp.blockDim = k.block;
  kp.sharedMemBytes = k.smem;
  kp.kernelParams = args;
  cudaGraphNode_t node = nullptr;
  CUDA_TRY(cudaGraphAddKernelNode(&node, graphs_[t.graph], t.deps.data(), t.deps.size(), &kp));
  STATUS_TRY(added(t, node));
  ++w->counters[kCtrKernels];
  ++w->counters[kCtrApiCalls];
  return {};
}

Status GraphSink::record(World* w, cudaEvent_t e, cudaStream_t s) {
  Tail& t = tail_of(s);
  events_[e] = t;
  ++w->counters[kCtrApiCalls];
  return {};
}

Status GraphSink::wait(World* w, cudaStream_t s, cudaEvent_t e) {
  Tail& t = tail_of(s);
  auto it = events_.find(e);
  ++w->counters[kCtrApiCalls];
  if (it == events_.end() || it->second.deps.empty()) return {};  // nothing recorded inside this graph yet
  if (it->second.graph != t.graph)
    return fail(CECOLL_INTERNAL, "recording: an event joins the command lists of two units");
  for (cudaGraphNode_t n : it->second.deps)
    if (std::find(t.deps.begin(), t.deps.end(), n) == t.deps.end()) t.deps.push_back(n);
  return {};
}

Status GraphSink::add_node(cudaStream_t s, cudaGraphNodeParams* params, cudaGraphNode_t* out) {
  Tail& t = tail_of(s);
  cudaGraphNode_t node = nullptr;
  CUDA_TRY(cudaGraphAddNode(&node, graphs_[t.graph], t.deps.data(), t.deps.size(), params));
  STATUS_TRY(added(t, node));
  if (out) *out = node;
  return {};
}

}  // namespace cecoll
