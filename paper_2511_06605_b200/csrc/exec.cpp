// Executors: copy-engine lanes (pcpy / b2b / bcst / swap), the SM path,
// prelaunch triggers, plan lifetime and the eager-call plan cache.
#include <algorithm>
#include <atomic>
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
    cache_plan(w, p);
  }
  w->last_plan = p;
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

// Copy submission; when tracing (eager only) one call per copy, each
// bracketed by events.
Status issue_copies_traced(World* w, Sink& sink, const std::vector<Copy>& copies, cudaStream_t s,
                           int device, int pid, int tid) {
  if (!w->tracer) return sink.copies(w, copies, s);
  for (const Copy& c : copies) {
    cudaEvent_t b = sink.mark(w, device, s);
    STATUS_TRY(sink.copies(w, {c}, s));
    trace_span(w, "copy:copy", pid, tid, device, b, sink.mark(w, device, s));
  }
  return {};
}

// Stream memory operations (+ the signal kernel for other devices' flags)
// bracketed as one traced span when tracing and the batch is not empty.
Status submit_traced(World* w, Sink& sink, cudaStream_t s, const MemOps& ops, uint64_t** remote_tab, size_t nremote,
                     const char* name, int device, int pid, int tid) {
  if (ops.empty() && nremote == 0) return {};
  cudaEvent_t b = sink.mark(w, device, s);
  STATUS_TRY(sink.memops(w, s, ops));
  STATUS_TRY(signal_remote(w, sink, remote_tab, nremote, s));
  trace_span(w, name, pid, tid, device, b, sink.mark(w, device, s));
  return {};
}

Status kernel_traced(World* w, Sink& sink, cudaStream_t s, const KernelCall& k, const std::string& name, int device,
                     int pid, int tid) {
  if (!k.func) return {};
  cudaEvent_t b = sink.mark(w, device, s);
  STATUS_TRY(sink.kernel(w, s, k));
  trace_span(w, name, pid, tid, device, b, sink.mark(w, device, s));
  return {};
}

Status run_ce(World* w, Plan* p, Sink& sink) {
  // Phase 1: every unit announces readiness (rdy), forks its lanes and places
  // its own chunk. Phase 2: lanes poll rdy, copy, signal done. Phase 3: units
  // poll done and join their lanes. Every poll is submitted after the signal
  // it waits for, so streams that share a hardware queue cannot deadlock.
  for (Unit& u : p->units) {
    DeviceGuard g(u.device);
    const double h0 = trace_host_now(w);
    const int pid = u.ranks[0];
    STATUS_TRY(issue_copies_traced(w, sink, u.precopy, u.stream, u.device, pid, -1));
    STATUS_TRY(submit_traced(w, sink, u.stream, u.start, u.start_remote_tab, u.start_remote.size(), "sync:signal",
                             u.device, pid, -1));
    for (int r : u.ranks) STATUS_TRY(sink.record(w, w->local[r]->start, u.stream));
    STATUS_TRY(issue_copies_traced(w, sink, u.placement, u.stream, u.device, pid, -1));
    if (u.table.nitems)  // the lanes' merged item-kernel commands (lower.cpp lower_program)
      STATUS_TRY(kernel_traced(w, sink, u.stream, items_call(u.table, plan_grid(p, u.table)), table_name(u.table),
                               u.device, pid, -1));
    sink.host_span(w, "control", h0);
  }
  for (LaneExec& l : p->lanes) {
    RankState* rs = w->local[l.rank].get();
    DeviceGuard g(rs->device);
    const double h0 = trace_host_now(w);
    cudaStream_t s = rs->lanes[l.lane];
    STATUS_TRY(sink.wait(w, s, rs->start));
    STATUS_TRY(submit_traced(w, sink, s, l.pre, nullptr, 0, "poll:poll", rs->device, l.rank, l.lane));
    STATUS_TRY(issue_copies_traced(w, sink, l.copies, s, rs->device, l.rank, l.lane));
    if (l.table.nitems)
      STATUS_TRY(kernel_traced(w, sink, s, items_call(l.table, plan_grid(p, l.table)), table_name(l.table), rs->device,
                               l.rank, l.lane));
    STATUS_TRY(submit_traced(w, sink, s, l.post, nullptr, 0, "sync:signal", rs->device, l.rank, l.lane));
    STATUS_TRY(sink.record(w, rs->lane_done[l.lane], s));
    sink.host_span(w, "control", h0);
  }
  for (Unit& u : p->units) {
    // Join the lanes, signal other-device destinations (one kernel), then
    // wait for the incoming chunks.
    DeviceGuard g(u.device);
    for (const LaneExec& l : p->lanes) {
      if (std::find(u.ranks.begin(), u.ranks.end(), l.rank) == u.ranks.end()) continue;
      STATUS_TRY(sink.wait(w, u.stream, w->local[l.rank]->lane_done[l.lane]));
    }
    STATUS_TRY(submit_traced(w, sink, u.stream, {}, u.lanes_remote_tab, u.lanes_remote.size(), "sync:signal",
                             u.device, u.ranks[0], -1));
    STATUS_TRY(submit_traced(w, sink, u.stream, u.finish, nullptr, 0, "poll:poll", u.device, u.ranks[0], -1));
  }
  return {};
}

Status run_sm(World* w, Plan* p, Sink& sink) {
  for (Unit& u : p->units) {  // phase 1: readiness to sources in other units
    if (u.start_folded) {     // written by the fused kernel itself
      w->counters[kCtrFlagWrites] += u.sm_flags.npre;
      continue;
    }
    DeviceGuard g(u.device);
    STATUS_TRY(submit_traced(w, sink, u.stream, u.start, u.start_remote_tab, u.start_remote.size(), "sync:signal",
                             u.device, u.ranks[0], -1));
  }
  for (Unit& u : p->units) {  // phase 2: wait destinations, move, signal
    DeviceGuard g(u.device);
    const double h0 = trace_host_now(w);
    const int pid = u.ranks[0];
    if (!u.fused) STATUS_TRY(submit_traced(w, sink, u.stream, u.sm_pre, nullptr, 0, "poll:poll", u.device, pid, -1));
    // Hybrid: the copy-engine shares fork after the rdy polls and join
    // before the done signals.
    std::vector<const LaneExec*> forked;
    if (p->hybrid) {
      cudaEvent_t fork = w->local[u.ranks[0]]->start;
      STATUS_TRY(sink.record(w, fork, u.stream));
      for (const LaneExec& l : p->lanes) {
        if (std::find(u.ranks.begin(), u.ranks.end(), l.rank) == u.ranks.end()) continue;
        RankState* rs = w->local[l.rank].get();
        cudaStream_t ls = rs->lanes[l.lane];
        STATUS_TRY(sink.wait(w, ls, fork));
        STATUS_TRY(issue_copies_traced(w, sink, l.copies, ls, rs->device, l.rank, l.lane));
        STATUS_TRY(sink.record(w, rs->lane_done[l.lane], ls));
        forked.push_back(&l);
      }
    }
    const FlagSet* fs = u.fused ? &u.sm_flags : nullptr;
    if (u.table.nitems) {
      STATUS_TRY(kernel_traced(w, sink, u.stream, items_call(u.table, plan_grid(p, u.table), fs),
                               std::string("kernel:") + (table_name(u.table) + 5), u.device, pid, -1));
      if (u.fused) {
        w->counters[kCtrFlagWrites] += u.sm_flags.nsig;
        w->counters[kCtrFlagWaits] += u.sm_flags.npoll;
      }
    }
    if (u.red.nitems) {
      STATUS_TRY(kernel_traced(w, sink, u.stream, reduce_call(u.red, plan_red_grid(p, u.red), fs), "kernel:reduce", u.device,
                               pid, -1));
      if (u.fused) {
        w->counters[kCtrFlagWrites] += u.sm_flags.nsig;
        w->counters[kCtrFlagWaits] += u.sm_flags.npoll;
      }
    }
    for (const LaneExec* l : forked) STATUS_TRY(sink.wait(w, u.stream, w->local[l->rank]->lane_done[l->lane]));
    if (!u.fused)
      STATUS_TRY(submit_traced(w, sink, u.stream, u.sm_post, u.sm_post_remote_tab, u.sm_post_remote.size(),
                               "sync:signal", u.device, pid, -1));
    sink.host_span(w, "control", h0);
  }
  for (Unit& u : p->units) {  // phase 3: incoming chunks
    DeviceGuard g(u.device);
    STATUS_TRY(submit_traced(w, sink, u.stream, u.finish, nullptr, 0, "poll:poll", u.device, u.ranks[0], -1));
  }
  return {};
}

// Cancels a unit's armed instance: raises the unit's cancel count in pinned
// host memory (no stream: a stream memory operation could land in the same
// hardware queue as the armed graph and wait behind it forever — round 2's
// first version did, and an 8-rank latency run hung in plan_destroy), then
// waits for the instance to finish; its gate sees the raise and skips the
// body.
Status cancel_armed(World* w, Unit& u) {
  (void)w;
  volatile uint64_t* c = u.cancel_host;
  *c = ++u.cancels;
  __atomic_thread_fence(__ATOMIC_SEQ_CST);
  CUDA_TRY(cudaStreamSynchronize(u.arm));
  return {};
}

// Process-wide count of armed prelaunch units: device-synchronising calls
// (cudaFree, cudaFreeHost) wait behind an armed gate, so plan memory is only
// released while nothing is armed (release_retired).
std::atomic<int> g_armed{0};

void set_armed(Unit& u, bool armed) {
  if (u.armed == armed) return;
  u.armed = armed;
  g_armed.fetch_add(armed ? 1 : -1);
}

Status arm_unit(World* w, Unit& u) {
  DeviceGuard g(u.device);
  CUDA_TRY(cudaGraphLaunch(u.exec, u.arm));
  CUDA_TRY(cudaEventRecord(u.graph_done, u.arm));
  ++w->counters[kCtrGraphLaunches];
  w->counters[kCtrApiCalls] += 2;
  set_armed(u, true);
  return {};
}

// Trigger phase 1 (signals): the unit's start signals and its trigger word
// (ready = 1), written by the caller stream: the armed graph's gate opens when
// the caller stream reaches this point (stream-ordered behind the producer).
Status trigger_signal(World* w, Unit& u, cudaEvent_t* span_begin) {
  DeviceGuard g(u.device);
  StreamSink sink;
  const double h0 = trace_host_now(w);
  const int pid = u.ranks[0];
  STATUS_TRY(issue_copies_traced(w, sink, u.precopy, u.stream, u.device, pid, -1));
  MemOps ops = u.start;
  // CECOLL_TRIGGER_KERNEL=1: the trigger word is written by a one-thread
  // signal kernel instead of a stream memory operation (A/B).
  static const bool kernel_trigger = [] {
    const char* e = std::getenv("CECOLL_TRIGGER_KERNEL");
    return e && std::string(e) == "1";
  }();
  if (!kernel_trigger) ops.push_back(op_write(u.ready_flag, 1));
  *span_begin = trace_mark(w, u.device, u.stream);
  STATUS_TRY(submit_traced(w, sink, u.stream, ops, u.start_remote_tab, u.start_remote.size(), "trigger:signal",
                           u.device, pid, -1));
  if (kernel_trigger) STATUS_TRY(sink.kernel(w, u.stream, signal_call(u.ready_tab, 1)));
  set_armed(u, false);
  trace_host_span(w, "trigger", h0);
  return {};
}

// Trigger phase 2 (polls): incoming done flags and the graph's completion.
// Submitted for every unit only after every unit's phase 1, so a poll never
// sits ahead of a signal it waits for in a shared hardware queue (§3.2).
Status trigger_wait(World* w, Unit& u, cudaEvent_t span_begin) {
  DeviceGuard g(u.device);
  StreamSink sink;
  const int pid = u.ranks[0];
  if (u.nfin)
    STATUS_TRY(kernel_traced(w, sink, u.stream, poll_call(u.fin_tab, u.nfin, u.err), "poll:poll", u.device, pid, -1));
  STATUS_TRY(sink.wait(w, u.stream, u.graph_done));
  // The gated graph body (polls, copies, signals) runs on the arm stream; its
  // span is taken from the trigger to its completion as seen by the caller.
  trace_span(w, "copy:graph", pid, 0, u.device, span_begin, trace_mark(w, u.device, u.stream));
  return {};
}

// Recorded command lists. A plan qualifies when every unit
// has its own device (two units on one device keep the phase-ordered eager
// submission, which never lets a poll block the queue of the signal it waits
// for), its stream is an explicit stream that the caller is not capturing,
// and nothing traces.
bool graph_eligible(World* w, Plan* p) {
  (void)w;
  static const bool off = [] {
    const char* e = std::getenv("CECOLL_GRAPH");
    return e && std::string(e) == "0";
  }();
  if (off || p->prelaunch) return false;
  // A submission of exactly one kernel launch (the SM path with one unit and
  // no flags) is recorded too: on the round-2 boxes a one-node graph launch
  // costs the host 1.3 µs against 3-5 µs for the direct launch
  // (profiles/latency_r02_n8.csv: swap's recorded single kernel vs sm), and
  // back-to-back small collectives are host-bound. CECOLL_RECORD_SINGLE=0
  // keeps such plans on direct launches.
  static const bool single_off = [] {
    const char* e = std::getenv("CECOLL_RECORD_SINGLE");
    return e && std::string(e) == "0";
  }();
  if (single_off && p->sm && !p->hybrid && p->units.size() == 1) {
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

// Builds the plan's command list explicitly — the same commands run_ce /
// run_sm submit eagerly, as memcpy, batch-mem-op and kernel nodes of one
// graph per unit (GraphSink; the unit's lane streams map to its graph) — and
// instantiates the graphs. Nothing executes and no stream enters capture
// mode while recording.
Status record_plan(World* w, Plan* p) {
  int64_t before[kNumCounters];
  for (int i = 0; i < kNumCounters; ++i) before[i] = w->counters[i];
  Status st;
  std::vector<cudaGraph_t> graphs;
  for (Unit& u : p->units) {
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaGraphCreate(&g, 0);
    if (e != cudaSuccess) {
      st = cuda_fail(e, "cudaGraphCreate", __FILE__, __LINE__);
      break;
    }
    u.rec_graph = g;
    graphs.push_back(g);
  }
  if (st.ok()) {
    GraphSink sink(graphs);
    for (size_t i = 0; i < p->units.size(); ++i) {
      Unit& u = p->units[i];
      sink.map(u.stream, static_cast<int>(i));
      for (int r : u.ranks)
        for (cudaStream_t ls : w->local[r]->lanes) sink.map(ls, static_cast<int>(i));
    }
    st = p->sm ? run_sm(w, p, sink) : run_ce(w, p, sink);
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

// A traced launch of a recorded plan (cecoll_trace_begin): the same command
// list built once more with an event-record node around every command
// (GraphSink::mark), launched once and released; the per-command spans then
// show the replayed graph's timeline, not an eager stand-in.
Status launch_traced(World* w, Plan* p) {
  const int64_t api0 = w->counters[kCtrApiCalls];
  std::vector<cudaGraph_t> graphs;
  Status st;
  for (size_t i = 0; i < p->units.size() && st.ok(); ++i) {
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaGraphCreate(&g, 0);
    if (e != cudaSuccess) st = cuda_fail(e, "cudaGraphCreate", __FILE__, __LINE__);
    else graphs.push_back(g);
  }
  if (st.ok()) {
    GraphSink sink(graphs);
    for (size_t i = 0; i < p->units.size(); ++i) {
      Unit& u = p->units[i];
      sink.map(u.stream, static_cast<int>(i));
      for (int r : u.ranks)
        for (cudaStream_t ls : w->local[r]->lanes) sink.map(ls, static_cast<int>(i));
    }
    st = p->sm ? run_sm(w, p, sink) : run_ce(w, p, sink);
  }
  w->counters[kCtrApiCalls] = api0;
  for (size_t i = 0; i < graphs.size(); ++i) {
    Unit& u = p->units[i];
    DeviceGuard g(u.device);
    if (st.ok()) {
      cudaGraphExec_t exec = nullptr;
      cudaError_t e = cudaGraphInstantiate(&exec, graphs[i], 0);
      const double h0 = trace_host_now(w);
      if (e == cudaSuccess) e = cudaGraphLaunch(exec, u.stream);
      trace_host_span(w, "control", h0);
      if (exec) cudaGraphExecDestroy(exec);  // freed once the launch completes
      if (e != cudaSuccess) st = cuda_fail(e, "traced graph launch", __FILE__, __LINE__);
      ++w->counters[kCtrRecordedLaunches];
      ++w->counters[kCtrApiCalls];
    }
    cudaGraphDestroy(graphs[i]);
  }
  return st;
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

bool same_call(const Plan* p, Kind kind, Impl impl, int64_t s, const std::vector<CallArgs>& args, int budget) {
  if (p->kind != kind || p->chunk != s || p->key_rank.size() != args.size()) return false;
  if (p->impl != impl || p->sm_budget != budget) return false;
  for (size_t i = 0; i < args.size(); ++i)
    if (p->key_rank[i] != args[i].rank || p->key_send[i] != args[i].send || p->key_recv[i] != args[i].recv ||
        p->key_stream[i] != args[i].stream)
      return false;
  return true;
}

}  // namespace

int armed_units() { return g_armed.load(); }

int plan_grid(const Plan* p, const ItemTable& t) {
  const int g = mover_grid_for(t, p->sms);
  return p->sm_budget > 0 ? std::min(g, p->sm_budget) : g;
}

// Reduction kernel grid: ceil(tiles / 2) short-lived CTAs, at least 4 per SM
// (the TMA mover's shape policy, kernels.cu TmaPolicy). With four sources'
// loads in flight (reduce.cu) 16-256 MiB chunks went from 0.89-0.95 of the
// copy peak (persistent grid, one source at a time) to 1.0-1.06
// (profiles/tma_shape_r02.md); CECOLL_RED_TPC=0 restores the persistent grid.
int plan_red_grid(const Plan* p, const RedTable& t) {
  static const int tpc = [] {
    const char* e = std::getenv("CECOLL_RED_TPC");
    return e ? std::atoi(e) : 2;
  }();
  int g = 4 * p->sms;
  if (tpc > 0) g = std::max(g, std::min((t.ntiles + tpc - 1) / tpc, kMaxGrid));
  return p->sm_budget > 0 ? std::min(g, p->sm_budget) : g;
}

// Cancels armed instances (the next launch re-arms): after this, device-wide
// synchronisation returns.
Status plan_disarm(World* w, Plan* p) {
  if (p->inner) STATUS_TRY(plan_disarm(w, p->inner.get()));
  for (Unit& u : p->units) {
    if (!u.armed) continue;
    DeviceGuard g(u.device);
    STATUS_TRY(cancel_armed(w, u));
    set_armed(u, false);
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
    StreamSink sink;
    for (Unit& u : p->units) {
      DeviceGuard g(u.device);
      STATUS_TRY(sink.kernel(w, u.stream, reduce_call(u.red, plan_red_grid(p, u.red))));
    }
    return {};
  }
  ++w->counters[kCtrCollectives];
  if (!p->prelaunch) {
    // First launch eager; from the second on, one recorded graph per unit.
    const int launch_no = p->launches++;
    if (launch_no >= 1 && graph_eligible(w, p)) {
      if (w->tracer) return launch_traced(w, p);
      if (!p->recorded && p->record_note.empty()) record_plan(w, p);
      if (p->recorded) return launch_recorded(w, p);
    }
    StreamSink sink;
    return p->sm ? run_sm(w, p, sink) : run_ce(w, p, sink);
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
    set_armed(p->units[i], false);
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
  for (auto& p : w->retired) note_async(w, plan_poll_errors(p.get()));
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
      const Status c = cancel_armed(w, u);  // the gate skips the body
      if (!c.ok() && result.ok()) result = c;
      set_armed(u, false);
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
    if (u.cancel_host) cudaFreeHost(u.cancel_host);
    u.cancel_host = nullptr;
    u.exec = nullptr;
    u.graph = nullptr;
    u.arm = nullptr;
    u.graph_done = nullptr;
    u.err = nullptr;
  }
  for (size_t i = 0; i < p->dev_allocs.size(); ++i) {
    DeviceGuard g(p->dev_alloc_device[i]);
    cudaFree(p->dev_allocs[i]);
  }
  p->dev_allocs.clear();
  return result;
}

// A plan leaving the eager cache (eviction, deregistration) is not destroyed
// on the collective path: its release frees device and pinned memory, which
// synchronises the device and would wait behind any armed prelaunch gate —
// possibly one whose trigger this very thread is about to post. Retired plans
// are released once no unit in the process is armed, or at world release.
void retire_plan(World* w, std::unique_ptr<Plan> p) {
  w->retired.push_back(std::move(p));
  release_retired(w, false);
}

void release_retired(World* w, bool force) {
  if (w->retired.empty() || (!force && armed_units() > 0)) return;
  // plan_destroy's frees synchronise the device, so the plan's last launches
  // have finished before its memory goes (its caller streams may be gone).
  for (auto& p : w->retired) note_async(w, plan_destroy(w, p.get()));
  w->retired.clear();
}

void cache_plan(World* w, Plan* p) {
  w->plans.emplace_back(p);
  if (w->plans.size() > kPlanCacheSize) {  // bounded cache: retire the oldest plan
    std::unique_ptr<Plan> old = std::move(w->plans.front());
    w->plans.erase(w->plans.begin());
    if (w->last_plan == old.get()) w->last_plan = nullptr;
    retire_plan(w, std::move(old));
  }
}

namespace {
const char* mover_name(const ItemTable& t) {
  if (!t.nitems) return "none";
  return t.mover == Mover::Tma ? "tma" : "reg";
}
}  // namespace

// What a plan turned into (cecoll_plan_info): the evidence a benchmark line
// needs to be read correctly — whether the prelaunch graph exists or the plan
// fell back to its eager program, whether the command list is recorded (and
// why not), which mover each unit uses and how flags between units travel.
std::string plan_info(World* w, const Plan* p) {
  std::string j = "{";
  auto kv = [&](const char* k, const std::string& v, bool quote) {
    if (j.size() > 1) j += ",";
    j += "\"" + std::string(k) + "\":" + (quote ? "\"" + v + "\"" : v);
  };
  auto esc = [](std::string v) {
    std::string o;
    for (char c : v) {
      if (c == '"' || c == '\\') o += '\\';
      if (static_cast<unsigned char>(c) >= 0x20) o += c;
    }
    return o;
  };
  const char* rs = std::getenv("CECOLL_REMOTE_SIGNAL");
  kv("impl", impl_name(p->impl), true);
  kv("kind", p->kind == Kind::AllGather ? "allgather" : p->kind == Kind::AllToAll ? "alltoall" : "reduce_scatter",
     true);
  kv("chunk_bytes", std::to_string(p->chunk), false);
  kv("prelaunch", p->prelaunch ? "true" : "false", false);
  kv("prelaunch_folded", p->folded ? "true" : "false", false);
  kv("graph_fallback", esc(p->graph_fallback), true);
  kv("recorded", p->recorded ? "true" : "false", false);
  kv("record_note", esc(p->record_note), true);
  kv("launches", std::to_string(p->launches), false);
  kv("sm_budget", std::to_string(p->sm_budget), false);
  kv("remote_signals", (rs && std::string(rs) == "memop") ? "memop" : "kernel", true);
  std::string units = "[";
  for (size_t i = 0; i < p->units.size(); ++i) {
    const Unit& u = p->units[i];
    std::string ranks;
    for (int r : u.ranks) ranks += (ranks.empty() ? "" : ",") + std::to_string(r);
    int lanes = 0;
    for (const LaneExec& l : p->lanes)
      if (std::find(u.ranks.begin(), u.ranks.end(), l.rank) != u.ranks.end() && !l.copies.empty()) ++lanes;
    const size_t remote = u.start_remote.size() + u.sm_post_remote.size() + u.lanes_remote.size();
    const size_t local = u.start.size() + u.sm_post.size();
    units += std::string(i ? "," : "") + "{\"device\":" + std::to_string(u.device) + ",\"ranks\":[" + ranks +
             "],\"mover\":\"" + (u.red.nitems ? "reduce" : mover_name(u.table)) +
             "\",\"grid\":" + std::to_string(u.table.nitems ? std::min(plan_grid(p, u.table), u.table.ntiles) : 0) +
             ",\"tile_bytes\":" + std::to_string(u.table.nitems ? u.table.tile : 0) +
             ",\"tiles\":" + std::to_string(u.table.ntiles) +
             ",\"ce_lanes\":" + std::to_string(lanes) + ",\"fused_flags\":" + (u.fused ? "true" : "false") +
             ",\"start_folded\":" + (u.start_folded ? "true" : "false") +
             ",\"flag_writes_memop\":" + std::to_string(local) +
             ",\"flag_writes_kernel\":" + std::to_string(remote) + "}";
  }
  units += "]";
  kv("units", units, false);
  (void)w;
  return j + "}";
}

Status run_collective(World* w, Kind kind, Impl impl, int64_t s, const std::vector<CallArgs>& args) {
  if (impl == Impl::Auto) {
    bool in_place = kind == Kind::AllToAll;
    for (const CallArgs& a : args) in_place &= a.send == a.recv;
    impl = in_place ? Impl::Swap : select_for(w, kind, s);
  }
  Plan* p = nullptr;
  for (auto& cand : w->plans)
    if (same_call(cand.get(), kind, impl, s, args, w->sm_budget)) {
      p = cand.get();
      break;
    }
  if (!p) {
    const double h0 = trace_host_now(w);
    STATUS_TRY(plan_create(w, kind, impl, s, args, &p));
    trace_host_span(w, "control:compile", h0);
    cache_plan(w, p);
  }
  w->last_plan = p;
  // Eager calls never leave an instance armed after returning (a waiting
  // graph would block device-wide synchronisation); explicit plans do.
  return plan_launch(w, p, false);
}

}  // namespace cecoll
