// Executors: copy-engine lanes (pcpy / b2b / bcst / swap), the SM path,
// prelaunch triggers, plan lifetime and the eager-call plan cache.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <set>

#include "internal.hpp"

namespace cecoll {

Status run_reduce_scatter(World* w, Impl impl, int64_t count, int dtype, int op, const std::vector<CallArgs>& args) {
  if (impl == Impl::Auto) impl = Impl::Sm;
  const int64_t s = count * dtype_bytes(dtype);
  Plan* p = nullptr;
  for (auto& cand : w->plans) {
    Plan* c = cand.get();
    if (c->kind != Kind::ReduceScatter || c->impl != impl || c->chunk != s || c->dtype != dtype || c->op != op ||
        c->key_rank.size() != args.size())
      continue;
    bool same = true;
    for (size_t i = 0; i < args.size() && same; ++i)
      same = c->key_rank[i] == args[i].rank && c->key_send[i] == args[i].send && c->key_recv[i] == args[i].recv &&
             c->key_stream[i] == args[i].stream;
    if (same) {
      p = c;
      break;
    }
  }
  if (!p) {
    STATUS_TRY(plan_create_rs(w, impl, count, dtype, op, args, &p));
    w->plans.emplace_back(p);
  }
  return plan_launch(w, p, false);
}

// ---------------------------------------------------------------------------
// Execution
// ---------------------------------------------------------------------------

namespace {

const char* table_name(const ItemTable& t) {
  if (t.kinds & (1 << kItemSwap)) return "copy:swap";
  if (t.kinds & ((1 << kItemBcst) | (1 << kItemFan))) return "copy:broadcast";
  return "copy:copy";
}

// Traced copy submission: one call per copy, each bracketed by events.
Status issue_copies_traced(World* w, const std::vector<Copy>& copies, cudaStream_t s, bool allow_batch, int device,
                           int pid, int tid) {
  if (!w->tracer) return issue_copies(w, copies, s, allow_batch);
  for (const Copy& c : copies) {
    cudaEvent_t b = trace_mark(w, device, s);
    STATUS_TRY(issue_copies(w, {c}, s, false));
    trace_span(w, "copy:copy", pid, tid, device, b, trace_mark(w, device, s));
  }
  return {};
}

// Stream memory operations (+ the signal kernel for other devices' flags)
// bracketed as one traced span when tracing and the batch is not empty.
Status submit_traced(World* w, cudaStream_t s, const MemOps& ops, uint64_t** remote_tab, size_t nremote,
                     const char* name, int device, int pid, int tid) {
  if (ops.empty() && nremote == 0) return {};
  cudaEvent_t b = trace_mark(w, device, s);
  STATUS_TRY(submit(w, s, ops));
  STATUS_TRY(signal_remote(w, remote_tab, nremote, s));
  trace_span(w, name, pid, tid, device, b, trace_mark(w, device, s));
  return {};
}

Status run_ce(World* w, Plan* p) {
  // Phase 1: every unit announces readiness (rdy), forks its lanes and places
  // its own chunk. Phase 2: lanes poll rdy, copy, signal done. Phase 3: units
  // poll done and join their lanes. Every poll is submitted after the signal
  // it waits for, so streams that share a hardware queue cannot deadlock.
  for (Unit& u : p->units) {
    DeviceGuard g(u.device);
    const double h0 = trace_host_now(w);
    const int pid = u.ranks[0];
    STATUS_TRY(issue_copies_traced(w, u.precopy, u.stream, true, u.device, pid, -1));
    STATUS_TRY(submit_traced(w, u.stream, u.start, u.start_remote_tab, u.start_remote.size(), "sync:signal",
                             u.device, pid, -1));
    for (int r : u.ranks) {
      CUDA_TRY(cudaEventRecord(w->local[r]->start, u.stream));
      ++w->counters[kCtrApiCalls];
    }
    STATUS_TRY(issue_copies_traced(w, u.placement, u.stream, true, u.device, pid, -1));
    if (u.table.nitems) {  // the lanes' merged item-kernel commands (lower.cpp lower_program)
      cudaEvent_t b = trace_mark(w, u.device, u.stream);
      CUDA_TRY(launch_items(u.table, mover_grid_for(u.table, p->sms), u.stream));
      ++w->counters[kCtrKernels];
      ++w->counters[kCtrApiCalls];
      trace_span(w, table_name(u.table), pid, -1, u.device, b, trace_mark(w, u.device, u.stream));
    }
    trace_host_span(w, "control", h0);
  }
  for (LaneExec& l : p->lanes) {
    RankState* rs = w->local[l.rank].get();
    DeviceGuard g(rs->device);
    const double h0 = trace_host_now(w);
    cudaStream_t s = rs->lanes[l.lane];
    CUDA_TRY(cudaStreamWaitEvent(s, rs->start, 0));
    ++w->counters[kCtrApiCalls];
    STATUS_TRY(submit_traced(w, s, l.pre, nullptr, 0, "poll:poll", rs->device, l.rank, l.lane));
    STATUS_TRY(issue_copies_traced(w, l.copies, s, true, rs->device, l.rank, l.lane));
    if (l.table.nitems) {
      cudaEvent_t b = trace_mark(w, rs->device, s);
      CUDA_TRY(launch_items(l.table, mover_grid_for(l.table, p->sms), s));
      ++w->counters[kCtrKernels];
      ++w->counters[kCtrApiCalls];
      trace_span(w, table_name(l.table), l.rank, l.lane, rs->device, b, trace_mark(w, rs->device, s));
    }
    STATUS_TRY(submit_traced(w, s, l.post, nullptr, 0, "sync:signal", rs->device, l.rank, l.lane));
    CUDA_TRY(cudaEventRecord(rs->lane_done[l.lane], s));
    ++w->counters[kCtrApiCalls];
    trace_host_span(w, "control", h0);
  }
  for (Unit& u : p->units) {
    // Join the lanes, signal other-device destinations (one kernel), then
    // wait for the incoming chunks.
    DeviceGuard g(u.device);
    for (const LaneExec& l : p->lanes) {
      if (std::find(u.ranks.begin(), u.ranks.end(), l.rank) == u.ranks.end()) continue;
      CUDA_TRY(cudaStreamWaitEvent(u.stream, w->local[l.rank]->lane_done[l.lane], 0));
      ++w->counters[kCtrApiCalls];
    }
    STATUS_TRY(submit_traced(w, u.stream, {}, u.lanes_remote_tab, u.lanes_remote.size(), "sync:signal", u.device,
                             u.ranks[0], -1));
    STATUS_TRY(submit_traced(w, u.stream, u.finish, nullptr, 0, "poll:poll", u.device, u.ranks[0], -1));
  }
  return {};
}

Status run_sm(World* w, Plan* p) {
  for (Unit& u : p->units) {  // phase 1: readiness to sources in other units
    if (u.start_folded) {     // written by the fused kernel itself
      w->counters[kCtrFlagWrites] += u.sm_flags.npre;
      continue;
    }
    DeviceGuard g(u.device);
    STATUS_TRY(submit_traced(w, u.stream, u.start, u.start_remote_tab, u.start_remote.size(), "sync:signal",
                             u.device, u.ranks[0], -1));
  }
  for (Unit& u : p->units) {  // phase 2: wait destinations, move, signal
    DeviceGuard g(u.device);
    const double h0 = trace_host_now(w);
    const int pid = u.ranks[0];
    if (!u.fused) STATUS_TRY(submit_traced(w, u.stream, u.sm_pre, nullptr, 0, "poll:poll", u.device, pid, -1));
    // Hybrid: the copy-engine shares fork after the rdy polls and join
    // before the done signals.
    std::vector<const LaneExec*> forked;
    if (p->hybrid) {
      cudaEvent_t fork = w->local[u.ranks[0]]->start;
      CUDA_TRY(cudaEventRecord(fork, u.stream));
      ++w->counters[kCtrApiCalls];
      for (const LaneExec& l : p->lanes) {
        if (std::find(u.ranks.begin(), u.ranks.end(), l.rank) == u.ranks.end()) continue;
        RankState* rs = w->local[l.rank].get();
        cudaStream_t ls = rs->lanes[l.lane];
        CUDA_TRY(cudaStreamWaitEvent(ls, fork, 0));
        STATUS_TRY(issue_copies_traced(w, l.copies, ls, false, rs->device, l.rank, l.lane));
        CUDA_TRY(cudaEventRecord(rs->lane_done[l.lane], ls));
        w->counters[kCtrApiCalls] += 2;
        forked.push_back(&l);
      }
    }
    if (u.table.nitems) {
      cudaEvent_t b = trace_mark(w, u.device, u.stream);
      CUDA_TRY(launch_items(u.table, mover_grid_for(u.table, p->sms), u.stream, u.fused ? &u.sm_flags : nullptr));
      if (u.fused) {
        w->counters[kCtrFlagWrites] += u.sm_flags.nsig;
        w->counters[kCtrFlagWaits] += u.sm_flags.npoll;
      }
      ++w->counters[kCtrKernels];
      ++w->counters[kCtrApiCalls];
      trace_span(w, std::string("kernel:") + (table_name(u.table) + 5), pid, -1, u.device, b,
                 trace_mark(w, u.device, u.stream));
    }
    if (u.red.nitems) {
      cudaEvent_t b = trace_mark(w, u.device, u.stream);
      CUDA_TRY(launch_reduce(u.red, 4 * p->sms, u.stream, u.fused ? &u.sm_flags : nullptr));
      if (u.fused) {
        w->counters[kCtrFlagWrites] += u.sm_flags.nsig;
        w->counters[kCtrFlagWaits] += u.sm_flags.npoll;
      }
      ++w->counters[kCtrKernels];
      ++w->counters[kCtrApiCalls];
      trace_span(w, "kernel:reduce", pid, -1, u.device, b, trace_mark(w, u.device, u.stream));
    }
    for (const LaneExec* l : forked) {
      CUDA_TRY(cudaStreamWaitEvent(u.stream, w->local[l->rank]->lane_done[l->lane], 0));
      ++w->counters[kCtrApiCalls];
    }
    if (!u.fused)
      STATUS_TRY(submit_traced(w, u.stream, u.sm_post, u.sm_post_remote_tab, u.sm_post_remote.size(), "sync:signal",
                               u.device, pid, -1));
    trace_host_span(w, "control", h0);
  }
  for (Unit& u : p->units) {  // phase 3: incoming chunks
    DeviceGuard g(u.device);
    STATUS_TRY(submit_traced(w, u.stream, u.finish, nullptr, 0, "poll:poll", u.device, u.ranks[0], -1));
  }
  return {};
}

Status post_gate(Unit& u, uint64_t kind) {
  const uint64_t k = u.posts++;
  volatile uint64_t* posted = u.posted;
  posted[1 + (k % 64)] = kind;
  __atomic_thread_fence(__ATOMIC_SEQ_CST);
  posted[0] = k + 1;
  __atomic_thread_fence(__ATOMIC_SEQ_CST);
  return {};
}

Status arm_unit(World* w, Unit& u) {
  DeviceGuard g(u.device);
  CUDA_TRY(cudaGraphLaunch(u.exec, u.arm));
  CUDA_TRY(cudaEventRecord(u.graph_done, u.arm));
  ++w->counters[kCtrGraphLaunches];
  w->counters[kCtrApiCalls] += 2;
  u.armed = true;
  return {};
}

// Trigger phase 1 (signals): the unit's start / ready writes and the host
// post that opens its armed graph.
Status trigger_signal(World* w, Unit& u, cudaEvent_t* span_begin) {
  DeviceGuard g(u.device);
  const double h0 = trace_host_now(w);
  const int pid = u.ranks[0];
  STATUS_TRY(issue_copies_traced(w, u.precopy, u.stream, true, u.device, pid, -1));
  MemOps ops = u.start;
  ops.push_back(op_write(u.ready_flag, 1));
  *span_begin = trace_mark(w, u.device, u.stream);
  STATUS_TRY(submit_traced(w, u.stream, ops, u.start_remote_tab, u.start_remote.size(), "trigger:signal", u.device,
                           pid, -1));
  STATUS_TRY(post_gate(u, 1));
  u.armed = false;
  trace_host_span(w, "trigger", h0);
  return {};
}

// Trigger phase 2 (polls): incoming done flags and the graph's completion.
// Submitted for every unit only after every unit's phase 1, so a poll never
// sits ahead of a signal it waits for in a shared hardware queue (§3.2).
Status trigger_wait(World* w, Unit& u, cudaEvent_t span_begin) {
  DeviceGuard g(u.device);
  const int pid = u.ranks[0];
  if (u.nfin) {
    cudaEvent_t pb = trace_mark(w, u.device, u.stream);
    CUDA_TRY(launch_poll(u.fin_tab, u.nfin, u.err, u.stream));
    ++w->counters[kCtrKernels];
    ++w->counters[kCtrApiCalls];
    trace_span(w, "poll:poll", pid, -1, u.device, pb, trace_mark(w, u.device, u.stream));
  }
  CUDA_TRY(cudaStreamWaitEvent(u.stream, u.graph_done, 0));
  ++w->counters[kCtrApiCalls];
  // The gated graph body (polls, copies, signals) runs on the arm stream; its
  // span is taken from the trigger to its completion as seen by the caller.
  trace_span(w, "copy:graph", pid, 0, u.device, span_begin, trace_mark(w, u.device, u.stream));
  return {};
}

// Recorded command lists. A plan qualifies when every unit
// has its own device (two units on one device keep the phase-ordered eager
// submission, which never lets a poll block the queue of the signal it waits
// for), its stream is an explicit, non-capturing stream, and nothing traces.
bool graph_mode_wanted(World* w, Plan* p) {
  static const bool off = [] {
    const char* e = std::getenv("CECOLL_GRAPH");
    return e && std::string(e) == "0";
  }();
  if (off || p->prelaunch || w->tracer) return false;
  // A submission of exactly one kernel launch (the SM path with one unit and
  // no flags) gains nothing from a graph, and skipping the recording keeps
  // its stream out of capture mode (open issue).
  if (p->sm && !p->hybrid && p->units.size() == 1) {
    const Unit& u = p->units[0];
    if (u.start.empty() && u.start_remote.empty() && u.sm_pre.empty() && u.sm_post.empty() &&
        u.sm_post_remote.empty() && u.finish.empty())
      return false;
  }
  std::set<int> devs;
  for (const Unit& u : p->units) {
    if (!u.stream || u.stream == cudaStreamLegacy || u.stream == cudaStreamPerThread) return false;
    if (!devs.insert(u.device).second) return false;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(u.stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return false;
  }
  return true;
}

void drop_recording(Plan* p) {
  for (Unit& u : p->units) {
    DeviceGuard g(u.device);
    if (u.rec_exec) cudaGraphExecDestroy(u.rec_exec);
    if (u.rec_graph) cudaGraphDestroy(u.rec_graph);
    u.rec_exec = nullptr;
    u.rec_graph = nullptr;
  }
  p->recorded = false;
}

// Captures the plan's eager submission (run_ce / run_sm) on every unit stream
// at once — one graph per unit; lane streams join through the start / lane_done
// events — and instantiates the graphs. Nothing executes while recording.
Status record_plan(World* w, Plan* p) {
  int64_t before[kNumCounters];
  for (int i = 0; i < kNumCounters; ++i) before[i] = w->counters[i];
  size_t begun = 0;
  Status st;
  for (Unit& u : p->units) {
    DeviceGuard g(u.device);
    cudaError_t e = cudaStreamBeginCapture(u.stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
      st = cuda_fail(e, "cudaStreamBeginCapture", __FILE__, __LINE__);
      break;
    }
    ++begun;
  }
  w->capturing = true;
  if (st.ok()) st = p->sm ? run_sm(w, p) : run_ce(w, p);
  w->capturing = false;
  for (size_t i = 0; i < begun; ++i) {
    Unit& u = p->units[i];
    DeviceGuard g(u.device);
    cudaGraph_t gph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(u.stream, &gph);
    if (e != cudaSuccess && st.ok()) st = cuda_fail(e, "cudaStreamEndCapture", __FILE__, __LINE__);
    u.rec_graph = gph;
  }
  for (Unit& u : p->units) {
    if (!st.ok()) break;
    DeviceGuard g(u.device);
    const cudaError_t e = cudaGraphInstantiate(&u.rec_exec, u.rec_graph, 0);
    if (e != cudaSuccess) st = cuda_fail(e, "cudaGraphInstantiate", __FILE__, __LINE__);
  }
  for (int i = 0; i < kNumCounters; ++i) {
    p->rec_delta[i] = w->counters[i] - before[i];
    w->counters[i] = before[i];  // recording submitted nothing
  }
  if (!st.ok()) {
    drop_recording(p);
    cudaGetLastError();
    p->record_note = st.msg.empty() ? "recording failed" : st.msg;
    return st;
  }
  p->recorded = true;
  return {};
}

Status launch_recorded(World* w, Plan* p) {
  for (Unit& u : p->units) {
    DeviceGuard g(u.device);
    CUDA_TRY(cudaGraphLaunch(u.rec_exec, u.stream));
    ++w->counters[kCtrRecordedLaunches];
    ++w->counters[kCtrApiCalls];
  }
  for (int i : {kCtrCopies, kCtrFlagWrites, kCtrFlagWaits, kCtrKernels}) w->counters[i] += p->rec_delta[i];
  return {};
}

bool same_call(const Plan* p, Kind kind, Impl impl, int64_t s, const std::vector<CallArgs>& args) {
  if (p->kind != kind || p->chunk != s || p->key_rank.size() != args.size()) return false;
  if (p->impl != impl) return false;
  for (size_t i = 0; i < args.size(); ++i)
    if (p->key_rank[i] != args[i].rank || p->key_send[i] != args[i].send || p->key_recv[i] != args[i].recv ||
        p->key_stream[i] != args[i].stream)
      return false;
  return true;
}

}  // namespace

// Cancels armed instances (the next launch re-arms): after this, device-wide
// synchronisation returns.
Status plan_disarm(World* w, Plan* p) {
  if (p->inner) STATUS_TRY(plan_disarm(w, p->inner.get()));
  for (Unit& u : p->units) {
    if (!u.armed) continue;
    DeviceGuard g(u.device);
    STATUS_TRY(post_gate(u, 2));
    CUDA_TRY(cudaStreamSynchronize(u.arm));
    u.armed = false;
  }
  return {};
}

Status plan_arm(World* w, Plan* p) {
  if (p->inner) return plan_arm(w, p->inner.get());
  if (!p->prelaunch) return {};
  for (Unit& u : p->units)
    if (!u.armed) STATUS_TRY(arm_unit(w, u));
  return {};
}

Status plan_launch(World* w, Plan* p, bool rearm) {
  if (p->inner) {  // reduce-scatter over copy engines: gather, then reduce
    for (size_t i = 0; i < p->units.size(); ++i) p->inner->units[i].stream = p->units[i].stream;
    STATUS_TRY(plan_launch(w, p->inner.get(), rearm));
    for (Unit& u : p->units) {
      DeviceGuard g(u.device);
      CUDA_TRY(launch_reduce(u.red, 4 * p->sms, u.stream));
      ++w->counters[kCtrKernels];
      ++w->counters[kCtrApiCalls];
    }
    return {};
  }
  ++w->counters[kCtrCollectives];
  if (!p->prelaunch) {
    // First launch eager; from the second on, one recorded graph per unit.
    const bool want = graph_mode_wanted(w, p);
    if (p->recorded && want) return launch_recorded(w, p);
    if (!p->recorded && want && p->launches++ >= 1 && p->record_note.empty() && record_plan(w, p).ok())
      return launch_recorded(w, p);
    return p->sm ? run_sm(w, p) : run_ce(w, p);
  }
  // prelaunch: trigger every unit, then wait; re-arm if asked. A unit that
  // is not armed yet (eager calls, a plan's first launch) gets its post and
  // ready flag before its gated instance is launched: that instance never
  // waits on the host, so no CUDA call of this thread or another (a lazy
  // module load, a device synchronisation) can end up waiting behind a gate
  // whose trigger it blocks.
  const size_t nu = p->units.size();
  std::vector<bool> was_armed(nu);
  for (size_t i = 0; i < nu; ++i) was_armed[i] = p->units[i].armed;
  std::vector<cudaEvent_t> spans(nu, nullptr);
  for (size_t i = 0; i < nu; ++i) STATUS_TRY(trigger_signal(w, p->units[i], &spans[i]));
  for (size_t i = 0; i < nu; ++i) {
    if (was_armed[i]) continue;
    STATUS_TRY(arm_unit(w, p->units[i]));  // consumes the post just made
    p->units[i].armed = false;
  }
  for (size_t i = 0; i < nu; ++i) STATUS_TRY(trigger_wait(w, p->units[i], spans[i]));
  if (rearm) STATUS_TRY(plan_arm(w, p));
  return {};
}

namespace {
Status err_status(uint64_t err) {
  return fail(CECOLL_TIMEOUT, (err & 1) ? "a flag poll timed out (20 s): a peer never signalled"
                                        : "gate received an unknown post");
}
}  // namespace

Status plan_poll_errors(Plan* p) {
  if (p->inner) STATUS_TRY(plan_poll_errors(p->inner.get()));
  for (Unit& u : p->units) {
    if (!u.err) continue;
    DeviceGuard g(u.device);
    cudaStream_t s = nullptr;
    CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    uint64_t err = 0;
    cudaError_t e = cudaMemcpyAsync(&err, u.err, sizeof(err), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    CUDA_TRY(e);
    if (err) return err_status(err);
  }
  return {};
}

void note_async(World* w, const Status& s) {
  if (!s.ok() && w->async_error.ok()) w->async_error = s;
}

Status world_async_error(World* w) {
  if (!w->async_error.ok()) return w->async_error;
  for (auto& p : w->plans) note_async(w, plan_poll_errors(p.get()));
  for (Plan* p : w->explicit_plans) note_async(w, plan_poll_errors(p));
  return w->async_error;
}

Status plan_destroy(World* w, Plan* p) {
  Status result;
  if (p->inner) result = plan_destroy(w, p->inner.get());
  drop_recording(p);
  for (Unit& u : p->units) {
    DeviceGuard g(u.device);
    if (u.armed) {
      post_gate(u, 2);  // cancel: the gate skips the body
      cudaStreamSynchronize(u.arm);
      u.armed = false;
    }
    if (u.err) {  // kernel-side polls report timeouts here (kernels.cu poll_kernel)
      if (u.arm) cudaStreamSynchronize(u.arm);
      uint64_t err = 0;
      if (cudaMemcpy(&err, u.err, sizeof(err), cudaMemcpyDeviceToHost) == cudaSuccess && err && result.ok())
        result = err_status(err);
    }
    // Idempotent: every handle is cleared once released.
    if (u.exec) cudaGraphExecDestroy(u.exec);
    if (u.graph) cudaGraphDestroy(u.graph);
    if (u.arm) {
      cudaStreamSynchronize(u.arm);
      cudaStreamDestroy(u.arm);
    }
    if (u.graph_done) cudaEventDestroy(u.graph_done);
    if (u.posted) cudaFreeHost(u.posted);
    u.exec = nullptr;
    u.graph = nullptr;
    u.arm = nullptr;
    u.graph_done = nullptr;
    u.posted = nullptr;
    u.err = nullptr;
  }
  for (size_t i = 0; i < p->dev_allocs.size(); ++i) {
    DeviceGuard g(p->dev_alloc_device[i]);
    cudaFree(p->dev_allocs[i]);
  }
  p->dev_allocs.clear();
  return result;
}

Status run_collective(World* w, Kind kind, Impl impl, int64_t s, const std::vector<CallArgs>& args) {
  if (impl == Impl::Auto) {
    bool in_place = kind == Kind::AllToAll;
    for (const CallArgs& a : args) in_place &= a.send == a.recv;
    impl = in_place ? Impl::Swap : select(kind, s, w->nranks, w->ndevices);
  }
  Plan* p = nullptr;
  for (auto& cand : w->plans)
    if (same_call(cand.get(), kind, impl, s, args)) {
      p = cand.get();
      break;
    }
  if (!p) {
    const double h0 = trace_host_now(w);
    STATUS_TRY(plan_create(w, kind, impl, s, args, &p));
    trace_host_span(w, "control:compile", h0);
    w->plans.emplace_back(p);
    if (w->plans.size() > 64) {  // bounded cache: drop the oldest plan
      for (Unit& u : w->plans.front()->units) {
        DeviceGuard g(u.device);
        cudaStreamSynchronize(u.stream);
      }
      note_async(w, plan_destroy(w, w->plans.front().get()));
      w->plans.erase(w->plans.begin());
    }
  }
  // Eager calls never leave an instance armed after returning (a waiting
  // graph would block device-wide synchronisation); explicit plans do.
  return plan_launch(w, p, false);
}

}  // namespace cecoll
