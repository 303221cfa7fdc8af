// Error reporting, stream memory operations and copy submission shared by
// the executors.
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>

#include "internal.hpp"

namespace cecoll {

namespace {
thread_local std::string g_error;

std::string base_name(const char* path) {
  std::string p(path);
  const size_t k = p.find_last_of('/');
  return k == std::string::npos ? p : p.substr(k + 1);
}
}  // namespace

Status fail(int code, const std::string& msg) {
  g_error = msg;
  return Status{code, msg};
}

Status cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  return fail(CECOLL_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e) + " (" + base_name(file) + ":" +
                                     std::to_string(line) + ")");
}

Status cu_fail(CUresult r, const char* what, const char* file, int line) {
  const char* s = "?";
  if (driver_api()) driver_api()->GetErrorString(r, &s);
  return fail(CECOLL_CUDA_ERROR, std::string(what) + ": " + s + " (" + base_name(file) + ":" + std::to_string(line) + ")");
}



CUstreamBatchMemOpParams op_write(uint64_t* addr, uint64_t v) {
  CUstreamBatchMemOpParams op;
  std::memset(&op, 0, sizeof(op));
  op.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
  op.writeValue.address = reinterpret_cast<CUdeviceptr>(addr);
  op.writeValue.value64 = v;
  op.writeValue.flags = 0;  // with the default memory barrier: prior copies are visible first
  return op;
}

CUstreamBatchMemOpParams op_wait(uint64_t* addr, uint64_t v) {
  CUstreamBatchMemOpParams op;
  std::memset(&op, 0, sizeof(op));
  op.waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
  op.waitValue.address = reinterpret_cast<CUdeviceptr>(addr);
  op.waitValue.value64 = v;
  op.waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
  return op;
}

// Poll + reset of one slot (the reset keeps graph replays value-constant).
void add_poll(MemOps& ops, uint64_t* addr) {
  ops.push_back(op_wait(addr, 1));
  ops.push_back(op_write(addr, 0));
}

Status submit(World* w, cudaStream_t s, const MemOps& ops) {
  const DriverApi* d = driver_api();
  size_t i = 0;
  while (i < ops.size()) {
    const unsigned count = static_cast<unsigned>(std::min<size_t>(255, ops.size() - i));
    CU_TRY(d->StreamBatchMemOp(reinterpret_cast<CUstream>(s), count,
                               const_cast<CUstreamBatchMemOpParams*>(ops.data() + i), 0));
    for (unsigned k = 0; k < count; ++k) {
      if (ops[i + k].operation == CU_STREAM_MEM_OP_WRITE_VALUE_64) ++w->counters[kCtrFlagWrites];
      else ++w->counters[kCtrFlagWaits];
    }
    ++w->counters[kCtrApiCalls];
    i += count;
  }
  return {};
}

Status write_device(void* dst, const void* src, size_t bytes) {
  if (!bytes) return {};
  static std::mutex mu;
  static std::map<int, cudaStream_t> streams;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  cudaStream_t s = nullptr;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = streams.find(dev);
    if (it == streams.end()) {
      CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      streams[dev] = s;
    } else {
      s = it->second;
    }
    // one writer at a time per device stream (the synchronise below is
    // per call)
    if (src) CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    else CUDA_TRY(cudaMemsetAsync(dst, 0, bytes, s));
    CUDA_TRY(cudaStreamSynchronize(s));
  }
  return {};
}

Status issue_copies(World* w, const std::vector<Copy>& copies, cudaStream_t s) {
  // One cudaMemcpyAsync per copy: a b2b lane's n-1 copies go out back to back
  // on its stream (the driver's batched-copy entry point is not used: it
  // faulted GPUs on the round-2 pool).
  for (const Copy& c : copies) {
    CUDA_TRY(cudaMemcpyAsync(c.dst, c.src, static_cast<size_t>(c.bytes), cudaMemcpyDefault, s));
    ++w->counters[kCtrCopies];
    ++w->counters[kCtrApiCalls];
  }
  return {};
}

Status ensure_lanes(RankState* rs, int n) {
  DeviceGuard g(rs->device);
  while (static_cast<int>(rs->lanes.size()) < n) {
    cudaStream_t s;
    cudaEvent_t e;
    CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    rs->lanes.push_back(s);
    rs->lane_done.push_back(e);
  }
  return {};
}

// The signal kernel for other-device flags.
Status signal_remote(World* w, Sink& sink, uint64_t** tab, size_t n, cudaStream_t s) {
  if (!n) return {};
  STATUS_TRY(sink.kernel(w, s, signal_call(tab, static_cast<int>(n))));
  w->counters[kCtrFlagWrites] += static_cast<int64_t>(n);
  return {};
}

void set_error(const std::string& msg) { g_error = msg; }
const char* last_error() { return g_error.c_str(); }

}  // namespace cecoll
