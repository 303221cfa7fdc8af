// Hardware timelines in the reference's trace-event format (
// export_trace_json, sim.cpp:523-544): a JSON array of {"name":
// "<phase>:<command>", "ph": "B"|"E", "ts": µs, "pid": rank (-1 host),
// "tid": lane (-1 the caller stream, 0 host)}.
//
// While a world traces (cecoll_trace_begin), the executors bracket every
// command with CUDA events on the stream that runs it: lane polls, each copy
// (copies are then submitted one call each, so a b2b lane shows its n-1
// copies back to back), broadcast/swap item kernels, signals, the SM mover
// kernel, prelaunch graph bodies; the host side records one control span per
// submission. Device times are measured from a per-device base event recorded
// and synchronised at trace_begin, host times from the host clock read right
// after that synchronisation, so both timelines start at the same instant
// (within the synchronisation latency, a few µs).
#include <algorithm>
#include <chrono>
#include <cstdio>

#include "internal.hpp"

namespace cecoll {

namespace {

double host_us(const Tracer* t) {
  using namespace std::chrono;
  return duration<double, std::micro>(steady_clock::now() - t->host0).count();
}

}  // namespace

Status trace_begin(World* w) {
  if (w->tracer) return fail(CECOLL_INVALID_ARGUMENT, "cecoll_trace_begin: already tracing");
  auto t = std::make_unique<Tracer>();
  for (auto& rs : w->local) {
    if (!rs || t->base.count(rs->device)) continue;
    DeviceGuard g(rs->device);
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    CUDA_TRY(cudaEventRecord(e, nullptr));
    t->base[rs->device] = e;
  }
  for (auto& kv : t->base) {
    DeviceGuard g(kv.first);
    CUDA_TRY(cudaEventSynchronize(kv.second));
  }
  t->host0 = std::chrono::steady_clock::now();
  w->tracer = std::move(t);
  return {};
}

cudaEvent_t trace_mark(World* w, int device, cudaStream_t s) {
  Tracer* t = w->tracer.get();
  if (!t) return nullptr;
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  if (cudaEventRecord(e, s) != cudaSuccess) {
    cudaEventDestroy(e);
    return nullptr;
  }
  t->events.push_back({e, device});
  return e;
}

void trace_span(World* w, const std::string& name, int pid, int tid, int device, cudaEvent_t b, cudaEvent_t e) {
  Tracer* t = w->tracer.get();
  if (!t || !b || !e) return;
  t->spans.push_back({name, pid, tid, device, b, e});
}

double trace_host_now(World* w) { return w->tracer ? host_us(w->tracer.get()) : 0.0; }

void trace_host_span(World* w, const std::string& name, double b_us) {
  Tracer* t = w->tracer.get();
  if (!t) return;
  t->host.push_back({name, b_us, host_us(t)});
}

Status trace_end(World* w, std::string* json) {
  Tracer* t = w->tracer.get();
  if (!t) return fail(CECOLL_INVALID_ARGUMENT, "cecoll_trace_end: not tracing");
  struct Ev {
    double ts;
    int order;
    std::string line;
  };
  std::vector<Ev> evs;
  char buf[256];
  auto add = [&](const std::string& name, bool begin, double ts, int pid, int tid) {
    std::snprintf(buf, sizeof(buf), "{\"name\":\"%s\",\"ph\":\"%s\",\"ts\":%.3f,\"pid\":%d,\"tid\":%d}", name.c_str(),
                  begin ? "B" : "E", ts, pid, tid);
    evs.push_back({ts, static_cast<int>(evs.size()), buf});
  };
  Status result;
  for (const auto& sp : t->spans) {
    DeviceGuard g(sp.device);
    float b = 0, e = 0;
    cudaError_t r1 = cudaEventSynchronize(sp.e);
    cudaError_t r2 = cudaEventElapsedTime(&b, t->base[sp.device], sp.b);
    cudaError_t r3 = cudaEventElapsedTime(&e, t->base[sp.device], sp.e);
    if (r1 != cudaSuccess || r2 != cudaSuccess || r3 != cudaSuccess) {
      if (result.ok()) result = fail(CECOLL_CUDA_ERROR, "cecoll_trace_end: a traced event did not complete");
      continue;
    }
    add(sp.name, true, b * 1e3, sp.pid, sp.tid);
    add(sp.name, false, e * 1e3, sp.pid, sp.tid);
  }
  for (const auto& h : t->host) {
    add(h.name, true, h.b_us, -1, 0);
    add(h.name, false, h.e_us, -1, 0);
  }
  std::stable_sort(evs.begin(), evs.end(), [](const Ev& a, const Ev& b) { return a.ts < b.ts; });
  std::string out = "[";
  for (size_t i = 0; i < evs.size(); ++i) {
    out += i ? ",\n " : "\n ";
    out += evs[i].line;
  }
  out += evs.empty() ? "]" : "\n]";
  for (const auto& ev : t->events) {
    DeviceGuard g(ev.second);
    cudaEventDestroy(ev.first);
  }
  for (auto& kv : t->base) {
    DeviceGuard g(kv.first);
    cudaEventDestroy(kv.second);
  }
  w->tracer.reset();
  *json = std::move(out);
  return result;
}

}  // namespace cecoll
