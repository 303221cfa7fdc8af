// Executors: copy-engine lanes (pcpy / b2b / bcst / swap), the SM path,
// prelaunch triggers, plan lifetime and the eager-call plan cache.
#include <algorithm>
#include <cstring>

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

Status run_ce(World* w, Plan* p) {
  const DriverApi* d = driver_api();
  (void)d;
  // Phase 1: every unit announces readiness (rdy), forks its lanes and places
  // its own chunk. Phase 2: lanes poll rdy, copy, signal done. Phase 3: units
  // poll done and join their lanes. Every poll is submitted after the signal
  // it waits for, so streams that share a hardware queue cannot deadlock.
  for (Unit& u : p->units) {
    DeviceGuard g(u.device);
    STATUS_TRY(issue_copies(w, u.precopy, u.stream, true));
    STATUS_TRY(submit(w, u.stream, u.start));
    STATUS_TRY(signal_remote(w, u.start_remote_tab, u.start_remote.size(), u.stream));
    for (int r : u.ranks) {
      CUDA_TRY(cudaEventRecord(w->local[r]->start, u.stream));
      ++w->counters[6];
    }
    STATUS_TRY(issue_copies(w, u.placement, u.stream, true));
  }
  for (LaneExec& l : p->lanes) {
    RankState* rs = w->local[l.rank].get();
    DeviceGuard g(rs->device);
    cudaStream_t s = rs->lanes[l.lane];
    CUDA_TRY(cudaStreamWaitEvent(s, rs->start, 0));
    ++w->counters[6];
    STATUS_TRY(submit(w, s, l.pre));
    STATUS_TRY(issue_copies(w, l.copies, s, true));
    if (l.table.nitems) {
      CUDA_TRY(launch_items(l.table, mover_grid_for(l.table, p->sms), s));
      ++w->counters[4];
      ++w->counters[6];
    }
    STATUS_TRY(submit(w, s, l.post));
    STATUS_TRY(signal_remote(w, l.post_remote_tab, l.post_remote.size(), s));
    CUDA_TRY(cudaEventRecord(rs->lane_done[l.lane], s));
    ++w->counters[6];
  }
  for (Unit& u : p->units) {
    DeviceGuard g(u.device);
    STATUS_TRY(submit(w, u.stream, u.finish));
    for (const LaneExec& l : p->lanes) {
      if (std::find(u.ranks.begin(), u.ranks.end(), l.rank) == u.ranks.end()) continue;
      CUDA_TRY(cudaStreamWaitEvent(u.stream, w->local[l.rank]->lane_done[l.lane], 0));
      ++w->counters[6];
    }
  }
  return {};
}

Status run_sm(World* w, Plan* p) {
  for (Unit& u : p->units) {  // phase 1: readiness to sources in other units
    DeviceGuard g(u.device);
    STATUS_TRY(submit(w, u.stream, u.start));
    STATUS_TRY(signal_remote(w, u.start_remote_tab, u.start_remote.size(), u.stream));
  }
  for (Unit& u : p->units) {  // phase 2: wait destinations, move, signal
    DeviceGuard g(u.device);
    STATUS_TRY(submit(w, u.stream, u.sm_pre));
    if (u.table.nitems) {
      CUDA_TRY(launch_items(u.table, mover_grid_for(u.table, p->sms), u.stream));
      ++w->counters[4];
      ++w->counters[6];
    }
    if (u.red.nitems) {
      CUDA_TRY(launch_reduce(u.red, 4 * p->sms, u.stream));
      ++w->counters[4];
      ++w->counters[6];
    }
    STATUS_TRY(submit(w, u.stream, u.sm_post));
    STATUS_TRY(signal_remote(w, u.sm_post_remote_tab, u.sm_post_remote.size(), u.stream));
  }
  for (Unit& u : p->units) {  // phase 3: incoming chunks
    DeviceGuard g(u.device);
    STATUS_TRY(submit(w, u.stream, u.finish));
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
  ++w->counters[5];
  w->counters[6] += 2;
  u.armed = true;
  return {};
}

Status trigger_unit(World* w, Plan* p, Unit& u) {
  DeviceGuard g(u.device);
  STATUS_TRY(issue_copies(w, u.precopy, u.stream, true));
  MemOps ops = u.start;
  ops.push_back(op_write(u.ready_flag, 1));
  STATUS_TRY(submit(w, u.stream, ops));
  STATUS_TRY(signal_remote(w, u.start_remote_tab, u.start_remote.size(), u.stream));
  STATUS_TRY(post_gate(u, 1));
  u.armed = false;
  if (u.nfin) {
    CUDA_TRY(launch_poll(u.fin_tab, u.nfin, u.err, u.stream));
    ++w->counters[4];
    ++w->counters[6];
  }
  CUDA_TRY(cudaStreamWaitEvent(u.stream, u.graph_done, 0));
  ++w->counters[6];
  (void)p;
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
      ++w->counters[4];
      ++w->counters[6];
    }
    return {};
  }
  ++w->counters[0];
  if (p->sm) return run_sm(w, p);
  if (!p->prelaunch) return run_ce(w, p);
  // prelaunch: make sure every unit is armed, trigger all, re-arm if asked.
  STATUS_TRY(plan_arm(w, p));
  for (Unit& u : p->units) STATUS_TRY(trigger_unit(w, p, u));
  if (rearm) STATUS_TRY(plan_arm(w, p));
  return {};
}

Status plan_destroy(World* w, Plan* p) {
  Status result;
  if (p->inner) result = plan_destroy(w, p->inner.get());
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
        result = fail(CECOLL_TIMEOUT, (err & 1) ? "a flag poll timed out (20 s): a peer never signalled"
                                                : "gate received an unknown post");
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
    STATUS_TRY(plan_create(w, kind, impl, s, args, &p));
    w->plans.emplace_back(p);
    if (w->plans.size() > 64) {  // bounded cache: drop the oldest plan
      for (Unit& u : w->plans.front()->units) {
        DeviceGuard g(u.device);
        cudaStreamSynchronize(u.stream);
      }
      plan_destroy(w, w->plans.front().get());
      w->plans.erase(w->plans.begin());
    }
  }
  // Eager calls never leave an instance armed after returning (a waiting
  // graph would block device-wide synchronisation); explicit plans do.
  return plan_launch(w, p, false);
}

}  // namespace cecoll
