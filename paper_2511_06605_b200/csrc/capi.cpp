// extern "C" boundary (include/cecoll.h). Exceptions never cross it: the
// reference's std::invalid_argument sites become CECOLL_INVALID_ARGUMENT /
// CECOLL_UNSUPPORTED and the message is kept for cecoll_last_error().
#include <algorithm>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "cecoll.h"
#include "internal.hpp"
#include "model.hpp"
#include "program.hpp"
#include "runtime.hpp"

using namespace cecoll;

struct cecoll_program {
  Program program;
};

namespace {

struct PendingCall {
  cecoll_comm_t comm;
  Kind kind;
  const void* send;
  void* recv;
  int64_t chunk;  // bytes (AG/AA) or elements (reduce-scatter)
  Impl impl;
  cudaStream_t stream;
  int dtype = 0;
  int op = 0;
};

thread_local int g_group_depth = 0;
thread_local std::vector<PendingCall> g_pending;

cecoll_status_t st(const Status& s) { return static_cast<cecoll_status_t>(s.code); }

cecoll_status_t err(cecoll_status_t code, const std::string& msg) {
  set_error(msg);
  return code;
}

bool impl_ok(cecoll_impl_t impl) { return impl >= CECOLL_IMPL_AUTO && impl <= CECOLL_IMPL_PULL; }

cecoll_status_t flush_group(std::vector<PendingCall>& calls) {
  // Group the calls per world and validate every group before anything is
  // submitted: a rejected group must not leave other worlds' collectives
  // half issued (their peers would wait on flags forever).
  std::vector<std::vector<size_t>> groups;
  std::vector<bool> done(calls.size(), false);
  for (size_t i = 0; i < calls.size(); ++i) {
    if (done[i]) continue;
    World* w = calls[i].comm->world;
    groups.emplace_back();
    for (size_t j = i; j < calls.size(); ++j) {
      if (done[j] || calls[j].comm->world != w) continue;
      if (calls[j].kind != calls[i].kind || calls[j].chunk != calls[i].chunk || calls[j].impl != calls[i].impl ||
          calls[j].dtype != calls[i].dtype || calls[j].op != calls[i].op)
        return err(CECOLL_INVALID_ARGUMENT, "group: one collective per communicator set (kind, size and impl must match)");
      groups.back().push_back(j);
      done[j] = true;
    }
  }
  cecoll_status_t result = CECOLL_SUCCESS;
  for (const auto& g : groups) {
    const PendingCall& c = calls[g[0]];
    std::vector<CallArgs> args;
    for (size_t j : g) args.push_back({calls[j].comm->rank, calls[j].send, calls[j].recv, calls[j].stream});
    Status s = c.kind == Kind::ReduceScatter ? run_reduce_scatter(c.comm->world, c.impl, c.chunk, c.dtype, c.op, args)
                                             : run_collective(c.comm->world, c.kind, c.impl, c.chunk, args);
    if (!s.ok() && result == CECOLL_SUCCESS) result = st(s);
  }
  return result;
}

cecoll_status_t enqueue(Kind kind, const void* send, void* recv, size_t chunk, cecoll_impl_t impl, cecoll_comm_t comm,
                        void* stream, int dtype = 0, int op = 0) {
  if (!comm || !comm->world) return err(CECOLL_INVALID_ARGUMENT, "null communicator");
  if (!impl_ok(impl)) return err(CECOLL_INVALID_ARGUMENT, "unknown implementation");
  if (!send || !recv) return err(CECOLL_INVALID_ARGUMENT, "collective: null send or recv buffer");
  if (chunk == 0) return err(CECOLL_INVALID_ARGUMENT, "collective: chunk size must be positive");
  PendingCall c{comm,   kind, send, recv, static_cast<int64_t>(chunk), static_cast<Impl>(impl),
                static_cast<cudaStream_t>(stream), dtype, op};
  if (g_group_depth > 0) {
    g_pending.push_back(c);
    return CECOLL_SUCCESS;
  }
  World* w = comm->world;
  if (!w->multiprocess && w->nranks > 1)
    return err(CECOLL_INVALID_ARGUMENT,
               "single-process communicator with several ranks: call every rank inside cecoll_group_start/end");
  std::vector<PendingCall> one{c};
  return flush_group(one);
}

}  // namespace

extern "C" {

const char* cecoll_strerror(cecoll_status_t s) {
  switch (s) {
    case CECOLL_SUCCESS: return "success";
    case CECOLL_INVALID_ARGUMENT: return "invalid argument";
    case CECOLL_UNSUPPORTED: return "unsupported";
    case CECOLL_CUDA_ERROR: return "CUDA error";
    case CECOLL_TIMEOUT: return "timeout";
    case CECOLL_NO_DEVICE: return "no CUDA device";
    case CECOLL_NOT_REGISTERED: return "buffer not registered";
    case CECOLL_INTERNAL: return "internal error";
  }
  return "unknown status";
}

const char* cecoll_impl_name(cecoll_impl_t impl) { return impl_name(static_cast<Impl>(impl)); }

cecoll_impl_t cecoll_parse_impl(const char* name) {
  Impl out;
  if (!name || !parse_impl(name, &out)) return static_cast<cecoll_impl_t>(-2);
  return static_cast<cecoll_impl_t>(out);
}

int cecoll_impl_valid_for(cecoll_impl_t impl, cecoll_kind_t kind) {
  if (impl == CECOLL_IMPL_SM || impl == CECOLL_IMPL_HYBRID || impl == CECOLL_IMPL_PULL || impl == CECOLL_IMPL_AUTO)
    return 1;
  if (!impl_ok(impl)) return 0;
  return valid_for(static_cast<Impl>(impl), static_cast<Kind>(kind)) ? 1 : 0;
}

const char* cecoll_last_error(void) { return last_error(); }

cecoll_status_t cecoll_program_compile(cecoll_kind_t kind, cecoll_impl_t impl, int64_t chunk_bytes, int nranks,
                                       int lanes_per_rank, cecoll_program_t* out) {
  if (!out) return err(CECOLL_INVALID_ARGUMENT, "null output");
  *out = nullptr;
  if (kind != CECOLL_ALLGATHER && kind != CECOLL_ALLTOALL) return err(CECOLL_INVALID_ARGUMENT, "unknown collective");
  if (impl < CECOLL_IMPL_PCPY || impl > CECOLL_IMPL_PRELAUNCH_B2B)
    return err(CECOLL_INVALID_ARGUMENT, "no command program for this implementation");
  if (!valid_for(static_cast<Impl>(impl), static_cast<Kind>(kind)))
    return err(CECOLL_UNSUPPORTED, std::string(impl_name(static_cast<Impl>(impl))) + " does not apply to " +
                                       (kind == CECOLL_ALLGATHER ? "allgather" : "alltoall"));
  Spec spec;
  spec.kind = static_cast<Kind>(kind);
  spec.chunk = chunk_bytes;
  spec.nranks = nranks;
  try {
    auto* p = new cecoll_program{compile(static_cast<Impl>(impl), spec, lanes_per_rank)};
    *out = p;
    return CECOLL_SUCCESS;
  } catch (const std::invalid_argument& e) {
    return err(CECOLL_INVALID_ARGUMENT, e.what());
  }
}

int64_t cecoll_program_dump(cecoll_program_t program, char* buf, size_t cap) {
  if (!program) return -1;
  std::string text = dump(program->program);
  if (!buf || text.size() + 1 > cap) return -1;
  std::memcpy(buf, text.c_str(), text.size() + 1);
  return static_cast<int64_t>(text.size());
}

cecoll_status_t cecoll_program_metrics(cecoll_program_t program, int64_t out5[5]) {
  if (!program || !out5) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  Metrics m = metrics(program->program);
  out5[0] = m.data;
  out5[1] = m.sync;
  out5[2] = m.poll;
  out5[3] = m.engines;
  out5[4] = m.doorbells;
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_program_traffic(cecoll_program_t program, int64_t out3[3], int64_t* rr, int64_t* rw) {
  if (!program || !out3) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  Traffic t = traffic(program->program);
  out3[0] = t.read;
  out3[1] = t.write;
  out3[2] = t.link;
  for (size_t i = 0; i < t.rank_read.size(); ++i) {
    if (rr) rr[i] = t.rank_read[i];
    if (rw) rw[i] = t.rank_write[i];
  }
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_program_validate(cecoll_program_t program, int lanes_per_rank) {
  if (!program) return err(CECOLL_INVALID_ARGUMENT, "null program");
  std::string v = validate(program->program, lanes_per_rank);
  if (v.empty()) return CECOLL_SUCCESS;
  return err(CECOLL_INVALID_ARGUMENT, v);
}

void cecoll_program_free(cecoll_program_t program) { delete program; }

cecoll_status_t cecoll_program_parse(const char* text, cecoll_kind_t kind, int64_t chunk_bytes, int nranks,
                                     cecoll_program_t* out) {
  if (!text || !out) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (kind != CECOLL_ALLGATHER && kind != CECOLL_ALLTOALL) return err(CECOLL_INVALID_ARGUMENT, "unknown collective");
  try {
    *out = new cecoll_program{parse_dump(text, static_cast<Kind>(kind), chunk_bytes, nranks)};
    return CECOLL_SUCCESS;
  } catch (const std::invalid_argument& e) {
    return err(CECOLL_INVALID_ARGUMENT, e.what());
  }
}

cecoll_impl_t cecoll_reference_select(cecoll_kind_t kind, int64_t chunk_bytes) {
  try {
    return static_cast<cecoll_impl_t>(reference_select(static_cast<Kind>(kind), chunk_bytes));
  } catch (const std::invalid_argument& e) {
    set_error(e.what());
    return static_cast<cecoll_impl_t>(-2);
  }
}

cecoll_impl_t cecoll_select(cecoll_kind_t kind, int64_t chunk_bytes, int nranks, int ndevices) {
  return static_cast<cecoll_impl_t>(select(static_cast<Kind>(kind), chunk_bytes, nranks, ndevices));
}

cecoll_status_t cecoll_tune(const cecoll_comm_t* comms, int n, int64_t max_chunk_bytes, void* const* streams) {
  if (!comms || n <= 0 || !comms[0] || !comms[0]->world) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  if (g_group_depth > 0) return err(CECOLL_INVALID_ARGUMENT, "cecoll_tune: not inside a group");
  World* w = comms[0]->world;
  std::vector<int> ranks;
  for (int i = 0; i < n; ++i) {
    if (!comms[i] || comms[i]->world != w) return err(CECOLL_INVALID_ARGUMENT, "cecoll_tune: communicators of one world");
    ranks.push_back(comms[i]->rank);
  }
  if (static_cast<int>(ranks.size()) != (w->multiprocess ? w->nlocal : w->nranks))
    return err(CECOLL_INVALID_ARGUMENT, "cecoll_tune: pass every local communicator of the world");
  std::vector<cudaStream_t> ss(ranks.size(), nullptr);
  std::map<int, cudaStream_t> own;  // one private stream per device
  for (size_t k = 0; k < ranks.size(); ++k) {
    if (streams && streams[k]) {
      ss[k] = static_cast<cudaStream_t>(streams[k]);
      continue;
    }
    const int dev = w->device[ranks[k]];
    if (!own.count(dev)) {
      DeviceGuard g(dev);
      cudaStream_t s = nullptr;
      if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
        return err(CECOLL_CUDA_ERROR, "cecoll_tune: stream creation failed");
      own[dev] = s;
    }
    ss[k] = own[dev];
  }
  std::string report;
  Status s = world_tune(w, ranks, max_chunk_bytes, ss, &report);
  for (auto& kv : own) {
    DeviceGuard g(kv.first);
    cudaStreamSynchronize(kv.second);
    cudaStreamDestroy(kv.second);
  }
  return st(s);
}

cecoll_status_t cecoll_tune_table(cecoll_comm_t comm, char* buf, size_t cap, size_t* len) {
  if (!comm || !comm->world) return err(CECOLL_INVALID_ARGUMENT, "null communicator");
  const std::string t = tuned_text(comm->world);
  if (len) *len = t.size() + 1;
  if (buf && cap) {
    const size_t m = std::min(cap - 1, t.size());
    std::memcpy(buf, t.data(), m);
    buf[m] = 0;
  }
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_tune_report(cecoll_comm_t comm, char* buf, size_t cap, size_t* len) {
  if (!comm || !comm->world) return err(CECOLL_INVALID_ARGUMENT, "null communicator");
  const std::string& t = comm->world->tune_report;
  if (len) *len = t.size() + 1;
  if (buf && cap) {
    const size_t m = std::min(cap - 1, t.size());
    std::memcpy(buf, t.data(), m);
    buf[m] = 0;
  }
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_tune_load(cecoll_comm_t comm, const char* text) {
  if (!comm || !comm->world || !text) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  return st(tuned_load(comm->world, text));
}

cecoll_status_t cecoll_comm_init_all(cecoll_comm_t* comms, int nranks, const int* devlist) {
  if (!comms || !devlist) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  World* w = nullptr;
  Status s = world_init_all(nranks, devlist, &w);
  if (!s.ok()) return st(s);
  for (int r = 0; r < nranks; ++r) comms[r] = new cecoll_comm{w, r};
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_comm_init_rank(cecoll_comm_t* comm, int nranks, int rank, int device,
                                      cecoll_exchange_fn exchange, void* ctx) {
  return cecoll_comm_init_ranks(comm, nranks, rank, 1, device, exchange, ctx);
}

cecoll_status_t cecoll_comm_init_ranks(cecoll_comm_t* comms, int nranks, int first_rank, int nlocal, int device,
                                       cecoll_exchange_fn exchange, void* ctx) {
  if (!comms) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  World* w = nullptr;
  Status s = world_init_ranks(nranks, first_rank, nlocal, device, exchange, ctx, &w);
  if (!s.ok()) return st(s);
  for (int k = 0; k < nlocal; ++k) comms[k] = new cecoll_comm{w, first_rank + k};
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_exchange_check(int nranks, int first_rank, int nlocal, int device, cecoll_exchange_fn exchange,
                                      void* ctx, int32_t* out_devices) {
  std::vector<ProcInfoView> procs;
  Status s = gather_procs(nranks, first_rank, nlocal, device, nullptr, exchange, ctx, &procs);
  if (!s.ok()) return st(s);
  if (out_devices)
    for (const ProcInfoView& p : procs)
      for (int k = 0; k < p.nlocal; ++k) out_devices[p.first + k] = p.device;
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_comm_destroy(cecoll_comm_t comm) {
  if (!comm) return err(CECOLL_INVALID_ARGUMENT, "null communicator");
  World* w = comm->world;
  delete comm;
  if (--w->live_comms == 0) {
    const Status s = world_release(w);
    if (!s.ok()) return err(st(s), s.msg);
  }
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_comm_get_async_error(cecoll_comm_t comm, cecoll_status_t* async_error) {
  if (!comm || !async_error) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  const Status s = world_async_error(comm->world);
  *async_error = st(s);
  if (!s.ok()) set_error(s.msg);
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_comm_info(cecoll_comm_t comm, int* rank, int* nranks, int* device) {
  if (!comm) return err(CECOLL_INVALID_ARGUMENT, "null communicator");
  if (rank) *rank = comm->rank;
  if (nranks) *nranks = comm->world->nranks;
  if (device) *device = comm->world->device[comm->rank];
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_register(cecoll_comm_t comm, void* ptr, size_t bytes) {
  if (!comm || !ptr || !bytes) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  World* w = comm->world;
  return st(world_register(w, comm->rank, ptr, bytes, w->exchange, w->exchange_ctx));
}

cecoll_status_t cecoll_deregister(cecoll_comm_t comm, void* ptr) {
  if (!comm) return err(CECOLL_INVALID_ARGUMENT, "null communicator");
  return st(world_deregister(comm->world, ptr));
}

cecoll_status_t cecoll_mem_alloc(cecoll_comm_t comm, size_t bytes, void** ptr) {
  if (!comm || !ptr || !bytes) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  *ptr = nullptr;
  return st(world_mem_alloc(comm->world, comm->rank, bytes, ptr));
}

cecoll_status_t cecoll_mem_free(cecoll_comm_t comm, void* ptr) {
  if (!comm || !ptr) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  return st(world_mem_free(comm->world, ptr));
}

cecoll_status_t cecoll_allgather(const void* send, void* recv, size_t chunk_bytes, cecoll_impl_t impl,
                                 cecoll_comm_t comm, void* stream) {
  return enqueue(Kind::AllGather, send, recv, chunk_bytes, impl, comm, stream);
}

cecoll_status_t cecoll_alltoall(const void* send, void* recv, size_t chunk_bytes, cecoll_impl_t impl,
                                cecoll_comm_t comm, void* stream) {
  return enqueue(Kind::AllToAll, send, recv, chunk_bytes, impl, comm, stream);
}

cecoll_status_t cecoll_reduce_scatter(const void* send, void* recv, size_t count, cecoll_dtype_t dtype,
                                      cecoll_redop_t op, cecoll_impl_t impl, cecoll_comm_t comm, void* stream) {
  if (dtype < CECOLL_F32 || dtype > CECOLL_F16 || op < CECOLL_SUM || op > CECOLL_MIN)
    return err(CECOLL_INVALID_ARGUMENT, "reduce-scatter: unknown dtype or op");
  return enqueue(Kind::ReduceScatter, send, recv, count, impl, comm, stream, dtype, op);
}

cecoll_status_t cecoll_reduce_scatter_n(const cecoll_comm_t* comms, int n, const void* const* sends,
                                        void* const* recvs, size_t count, cecoll_dtype_t dtype, cecoll_redop_t op,
                                        cecoll_impl_t impl, void* const* streams) {
  if (!comms || n <= 0 || !sends || !recvs) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  if (dtype < CECOLL_F32 || dtype > CECOLL_F16 || op < CECOLL_SUM || op > CECOLL_MIN)
    return err(CECOLL_INVALID_ARGUMENT, "reduce-scatter: unknown dtype or op");
  if (!impl_ok(impl)) return err(CECOLL_INVALID_ARGUMENT, "unknown implementation");
  if (count == 0) return err(CECOLL_INVALID_ARGUMENT, "reduce-scatter: count must be positive");
  std::vector<PendingCall> calls;
  for (int i = 0; i < n; ++i) {
    if (!comms[i] || !sends[i] || !recvs[i]) return err(CECOLL_INVALID_ARGUMENT, "null argument");
    calls.push_back({comms[i], Kind::ReduceScatter, sends[i], recvs[i], static_cast<int64_t>(count),
                     static_cast<Impl>(impl), streams ? static_cast<cudaStream_t>(streams[i]) : nullptr, dtype, op});
  }
  if (g_group_depth > 0) {
    g_pending.insert(g_pending.end(), calls.begin(), calls.end());
    return CECOLL_SUCCESS;
  }
  return flush_group(calls);
}

cecoll_status_t cecoll_collective_n(cecoll_kind_t kind, const cecoll_comm_t* comms, int n, const void* const* sends,
                                    void* const* recvs, size_t chunk_bytes, cecoll_impl_t impl,
                                    void* const* streams) {
  if (!comms || n <= 0 || !sends || !recvs) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  if (kind != CECOLL_ALLGATHER && kind != CECOLL_ALLTOALL) return err(CECOLL_INVALID_ARGUMENT, "unknown collective");
  if (!impl_ok(impl)) return err(CECOLL_INVALID_ARGUMENT, "unknown implementation");
  if (chunk_bytes == 0) return err(CECOLL_INVALID_ARGUMENT, "collective: chunk size must be positive");
  std::vector<PendingCall> calls;
  calls.reserve(n);
  for (int i = 0; i < n; ++i) {
    if (!comms[i] || !sends[i] || !recvs[i]) return err(CECOLL_INVALID_ARGUMENT, "null argument");
    calls.push_back({comms[i], static_cast<Kind>(kind), sends[i], recvs[i], static_cast<int64_t>(chunk_bytes),
                     static_cast<Impl>(impl), streams ? static_cast<cudaStream_t>(streams[i]) : nullptr});
  }
  if (g_group_depth > 0) {
    g_pending.insert(g_pending.end(), calls.begin(), calls.end());
    return CECOLL_SUCCESS;
  }
  return flush_group(calls);
}

cecoll_status_t cecoll_group_start(void) {
  ++g_group_depth;
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_group_end(void) {
  if (g_group_depth <= 0) return err(CECOLL_INVALID_ARGUMENT, "group_end without group_start");
  if (--g_group_depth > 0) return CECOLL_SUCCESS;
  std::vector<PendingCall> calls;
  calls.swap(g_pending);
  return flush_group(calls);
}

cecoll_status_t cecoll_plan_create(const cecoll_comm_t* comms, int ncomms, cecoll_kind_t kind,
                                   const void* const* sends, void* const* recvs, size_t chunk_bytes,
                                   cecoll_impl_t impl, cecoll_plan_t* out) {
  if (!comms || ncomms <= 0 || !sends || !recvs || !out) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  if (!impl_ok(impl)) return err(CECOLL_INVALID_ARGUMENT, "unknown implementation");
  if (kind != CECOLL_ALLGATHER && kind != CECOLL_ALLTOALL) return err(CECOLL_INVALID_ARGUMENT, "unknown collective");
  for (int i = 0; i < ncomms; ++i)
    if (!comms[i]) return err(CECOLL_INVALID_ARGUMENT, "null communicator");
  World* w = comms[0]->world;
  std::vector<CallArgs> args;
  // Streams are bound at launch; plan units are formed per (device, rank)
  // with a placeholder stream equal to the rank index, resolved at launch.
  for (int i = 0; i < ncomms; ++i) {
    if (comms[i]->world != w) return err(CECOLL_INVALID_ARGUMENT, "plan: communicators of one world only");
    args.push_back({comms[i]->rank, sends[i], recvs[i], nullptr});
  }
  Plan* p = nullptr;
  Status s = plan_create(w, static_cast<Kind>(kind), static_cast<Impl>(impl), static_cast<int64_t>(chunk_bytes),
                         args, &p);
  if (!s.ok()) return st(s);
  w->explicit_plans.push_back(p);
  *out = new cecoll_plan{w, p};
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_plan_create_program(const cecoll_comm_t* comms, int ncomms, cecoll_program_t program,
                                           const void* const* sends, void* const* recvs, cecoll_plan_t* out) {
  if (!comms || ncomms <= 0 || !program || !sends || !recvs || !out)
    return err(CECOLL_INVALID_ARGUMENT, "null argument");
  for (int i = 0; i < ncomms; ++i)
    if (!comms[i]) return err(CECOLL_INVALID_ARGUMENT, "null communicator");
  World* w = comms[0]->world;
  std::vector<CallArgs> args;
  for (int i = 0; i < ncomms; ++i) {
    if (comms[i]->world != w) return err(CECOLL_INVALID_ARGUMENT, "plan: communicators of one world only");
    args.push_back({comms[i]->rank, sends[i], recvs[i], nullptr});
  }
  const Program& prog = program->program;
  Plan* p = nullptr;
  Status s = plan_create(w, prog.spec.kind, prog.impl, prog.spec.chunk, args, &p, &prog);
  if (!s.ok()) return st(s);
  w->explicit_plans.push_back(p);
  *out = new cecoll_plan{w, p};
  return CECOLL_SUCCESS;
}

namespace {
// Units were formed per device (streams are bound at launch): each unit runs
// on the stream given for its lowest rank.
void bind_streams(Plan* p, void* const* streams) {
  for (Unit& u : p->units) {
    cudaStream_t s = nullptr;
    for (size_t i = 0; i < p->key_rank.size(); ++i)
      if (p->key_rank[i] == u.ranks[0] && streams) s = static_cast<cudaStream_t>(streams[i]);
    u.stream = s;
  }
}
}  // namespace

cecoll_status_t cecoll_plan_launch(cecoll_plan_t plan, void* const* streams) {
  if (!plan) return err(CECOLL_INVALID_ARGUMENT, "null plan");
  bind_streams(plan->plan, streams);
  return st(plan_launch(plan->world, plan->plan, true));
}

cecoll_status_t cecoll_plan_arm(cecoll_plan_t plan) {
  if (!plan) return err(CECOLL_INVALID_ARGUMENT, "null plan");
  return st(plan_arm(plan->world, plan->plan));
}

cecoll_status_t cecoll_plan_trigger(cecoll_plan_t plan, void* const* streams) {
  if (!plan) return err(CECOLL_INVALID_ARGUMENT, "null plan");
  bind_streams(plan->plan, streams);
  return st(plan_launch(plan->world, plan->plan, false));
}

cecoll_status_t cecoll_plan_destroy(cecoll_plan_t plan) {
  if (!plan) return err(CECOLL_INVALID_ARGUMENT, "null plan");
  auto& v = plan->world->explicit_plans;
  v.erase(std::remove(v.begin(), v.end(), plan->plan), v.end());
  Status s = plan_destroy(plan->world, plan->plan);
  delete plan->plan;
  delete plan;
  return st(s);
}

cecoll_status_t cecoll_plan_disarm(cecoll_plan_t plan) {
  if (!plan) return err(CECOLL_INVALID_ARGUMENT, "null plan");
  return st(plan_disarm(plan->world, plan->plan));
}

cecoll_status_t cecoll_trace_begin(cecoll_comm_t comm) {
  if (!comm) return err(CECOLL_INVALID_ARGUMENT, "null communicator");
  return st(trace_begin(comm->world));
}

cecoll_status_t cecoll_trace_end(cecoll_comm_t comm, char* json, size_t capacity, size_t* length) {
  if (!comm || !length) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  World* w = comm->world;
  if (w->tracer) {
    std::string out;
    cecoll_status_t r = st(trace_end(w, &out));
    w->trace_json = std::move(out);
    if (r != CECOLL_SUCCESS) return r;
  }
  *length = w->trace_json.size();
  if (!json || capacity < w->trace_json.size() + 1) return CECOLL_SUCCESS;  // size query: keep the trace
  std::memcpy(json, w->trace_json.c_str(), w->trace_json.size() + 1);
  w->trace_json.clear();
  return CECOLL_SUCCESS;
}

namespace {
cecoll_status_t copy_out(const std::string& text, char* buf, size_t capacity, size_t* length) {
  *length = text.size();
  if (buf && capacity >= text.size() + 1) std::memcpy(buf, text.c_str(), text.size() + 1);
  return CECOLL_SUCCESS;
}
}  // namespace

cecoll_status_t cecoll_plan_info(cecoll_plan_t plan, char* json, size_t capacity, size_t* length) {
  if (!plan || !length) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  return copy_out(plan_info(plan->world, plan->plan), json, capacity, length);
}

cecoll_status_t cecoll_comm_last_plan_info(cecoll_comm_t comm, char* json, size_t capacity, size_t* length) {
  if (!comm || !length) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  const Plan* p = comm->world->last_plan;
  return copy_out(p ? plan_info(comm->world, p) : std::string("{}"), json, capacity, length);
}

cecoll_status_t cecoll_comm_set_sm_budget(cecoll_comm_t comm, int max_ctas) {
  if (!comm || max_ctas < 0) return err(CECOLL_INVALID_ARGUMENT, "null communicator or negative budget");
  comm->world->sm_budget = max_ctas;
  return CECOLL_SUCCESS;
}

cecoll_impl_t cecoll_select_budget(cecoll_kind_t kind, int64_t chunk_bytes, int nranks, int ndevices, int sm_budget) {
  return static_cast<cecoll_impl_t>(select(static_cast<Kind>(kind), chunk_bytes, nranks, ndevices, sm_budget));
}

namespace {
B200Model from_c(const cecoll_model_t* c) {
  B200Model m;
  m.t_kernel = c->t_kernel;
  m.t_graph = c->t_graph;
  m.t_branch = c->t_branch;
  m.t_node = c->t_node;
  m.t_trigger = c->t_trigger;
  m.bw_copy = c->bw_copy;
  m.bw_fan = c->bw_fan;
  m.bw_ce = c->bw_ce;
  m.bw_lanes = c->bw_lanes;
  m.bw_swap = c->bw_swap;
  m.l2_boost = c->l2_boost;
  m.l2_bytes = c->l2_bytes;
  m.folded_max_bytes = c->folded_max_bytes;
  m.prelaunch_gain_threshold = c->prelaunch_gain_threshold;
  m.t_stream = c->t_stream;
  m.stream_min_bytes = c->stream_min_bytes;
  m.l2_boost_swap = c->l2_boost_swap;
  return m;
}
void to_c(const B200Model& m, cecoll_model_t* c) {
  c->t_kernel = m.t_kernel;
  c->t_graph = m.t_graph;
  c->t_branch = m.t_branch;
  c->t_node = m.t_node;
  c->t_trigger = m.t_trigger;
  c->bw_copy = m.bw_copy;
  c->bw_fan = m.bw_fan;
  c->bw_ce = m.bw_ce;
  c->bw_lanes = m.bw_lanes;
  c->bw_swap = m.bw_swap;
  c->l2_boost = m.l2_boost;
  c->l2_bytes = m.l2_bytes;
  c->folded_max_bytes = m.folded_max_bytes;
  c->prelaunch_gain_threshold = m.prelaunch_gain_threshold;
  c->t_stream = m.t_stream;
  c->stream_min_bytes = m.stream_min_bytes;
  c->l2_boost_swap = m.l2_boost_swap;
}
}  // namespace

void cecoll_model_default(cecoll_model_t* m) {
  if (m) to_c(default_model(), m);
}

cecoll_status_t cecoll_model_predict(const cecoll_model_t* m, cecoll_kind_t kind, cecoll_impl_t impl,
                                     int64_t chunk_bytes, int nranks, double* ns) {
  if (!m || !ns) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  if (!impl_ok(impl) || impl == CECOLL_IMPL_AUTO) return err(CECOLL_INVALID_ARGUMENT, "unknown implementation");
  try {
    if (impl != CECOLL_IMPL_SM && !valid_for(static_cast<Impl>(impl), static_cast<Kind>(kind)))
      return err(CECOLL_UNSUPPORTED, "implementation does not apply to the collective");
    *ns = predict_ns(from_c(m), static_cast<Kind>(kind), static_cast<Impl>(impl), chunk_bytes, nranks);
  } catch (const std::invalid_argument& e) {
    return err(CECOLL_INVALID_ARGUMENT, e.what());
  }
  return CECOLL_SUCCESS;
}

cecoll_impl_t cecoll_model_winner(const cecoll_model_t* m, cecoll_kind_t kind, int64_t chunk_bytes, int nranks) {
  if (!m) return static_cast<cecoll_impl_t>(-2);
  try {
    return static_cast<cecoll_impl_t>(model_winner(from_c(m), static_cast<Kind>(kind), chunk_bytes, nranks));
  } catch (const std::invalid_argument&) {
    return static_cast<cecoll_impl_t>(-2);
  }
}

cecoll_status_t cecoll_model_fit(const int* kinds, const int* impls, const int64_t* chunk_bytes, const int* nranks,
                                 const double* ns, int count, uint64_t seed, int iterations, cecoll_model_t* out,
                                 double* residual, char* report, size_t capacity) {
  if (!kinds || !impls || !chunk_bytes || !nranks || !ns || count < 0 || !out)
    return err(CECOLL_INVALID_ARGUMENT, "null argument");
  std::vector<Measurement> meas;
  for (int i = 0; i < count; ++i) {
    if (impls[i] < 0 || impls[i] > CECOLL_IMPL_PULL || kinds[i] < 0 || kinds[i] > 1) continue;
    meas.push_back({static_cast<Kind>(kinds[i]), static_cast<Impl>(impls[i]), chunk_bytes[i], nranks[i], ns[i]});
  }
  const FitResult r = calibrate_b200(meas, seed, iterations);
  to_c(r.model, out);
  if (residual) *residual = r.residual;
  if (report && capacity) {
    const size_t k = std::min(capacity - 1, r.report.size());
    std::memcpy(report, r.report.data(), k);
    report[k] = 0;
  }
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_comm_counters(cecoll_comm_t comm, int64_t out8[8]) {
  if (!comm || !out8) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  for (int i = 0; i < kNumCounters; ++i) out8[i] = comm->world->counters[i].load();
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_mc_window_create(cecoll_comm_t comm, size_t chunk_capacity, cecoll_mc_t* out, void** recv) {
  if (!comm || !out) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  McWindow* m = nullptr;
  Status s = mc_create(comm->world, comm->rank, static_cast<int64_t>(chunk_capacity), &m);
  if (!s.ok()) return st(s);
  *out = new cecoll_mc{m};
  if (recv) *recv = mc_recv(m);
  return CECOLL_SUCCESS;
}

cecoll_status_t cecoll_mc_allgather(cecoll_mc_t mc, const void* send, size_t chunk_bytes, void* stream) {
  if (!mc || !send) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  return st(mc_allgather(mc->m, send, static_cast<int64_t>(chunk_bytes), static_cast<cudaStream_t>(stream)));
}

const char* cecoll_mc_handle_type(cecoll_mc_t mc) { return mc ? mc_how(mc->m) : ""; }

cecoll_status_t cecoll_mc_window_destroy(cecoll_mc_t mc) {
  if (!mc) return err(CECOLL_INVALID_ARGUMENT, "null argument");
  mc_release(mc->m);
  delete mc;
  return CECOLL_SUCCESS;
}

}  // extern "C"
