// Runtime winner grid (cecoll_tune) — SURVEY §8(a) a10 on the machine the
// communicator runs on.
//
// The reference picks an implementation from a table (select_implementation,
// compiler.cpp:305-318) whose thresholds its sweep derives from simulated
// winners (run_sweep + winner_grid, sweep.cpp:71-218). The static B200
// selector (program.cpp select) is measured on one GPU only; on a node whose
// NVLink / copy-engine behaviour was never measured its cut-offs are a guess.
// cecoll_tune runs the sweep for real on the world's own devices and buffers:
// every applicable implementation at 4 KiB x 4^k chunk sizes, timed on the
// device (CUDA events on each rank's stream, max over ranks and processes),
// winner per size by winner_grid's rule (the plain variant wins a near tie
// with its prelaunch form, prelaunch_gain_threshold; cost_model.hpp:30), and
// a small stability margin for the static choice. The grid then drives
// CECOLL_IMPL_AUTO for this world (nearest tuned size on a log scale) until
// cleared. In a multi-process world every process calls it with the same
// arguments; times are agreed through the init exchange, so every rank holds
// the same table and AUTO picks the same program everywhere.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <sstream>

#include "internal.hpp"
#include "runtime.hpp"

namespace cecoll {

namespace {

constexpr double kPrelaunchGain = 0.002;  // winner_grid's tie-break (cost_model.hpp:30)
constexpr double kStaticMargin = 1.03;    // the static selector's pick keeps ties within 3%

std::vector<Impl> tune_candidates(Kind kind) {
  std::vector<Impl> c = {Impl::Sm, Impl::Pcpy, Impl::B2b, Impl::Hybrid, Impl::Pull, Impl::PrelaunchPcpy,
                         Impl::PrelaunchB2b};
  if (kind == Kind::AllGather) {
    c.push_back(Impl::Bcst);
    c.push_back(Impl::PrelaunchBcst);
  }
  return c;
}

// Element-wise max over every process (failures, -1, win); single-process: as is.
Status agree_max(World* w, std::vector<double>& v) {
  if (!w->multiprocess) return {};
  const int procs = w->nranks / std::max(1, w->nlocal);
  std::vector<double> all(static_cast<size_t>(procs) * v.size());
  if (w->exchange(w->exchange_ctx, v.data(), v.size() * sizeof(double), all.data()) != 0)
    return fail(CECOLL_INTERNAL, "cecoll_tune: exchange failed");
  for (size_t i = 0; i < v.size(); ++i) {
    double m = 0;
    bool failed = false;
    for (int p = 0; p < procs; ++p) {
      const double x = all[static_cast<size_t>(p) * v.size() + i];
      failed |= x < 0;
      m = std::max(m, x);
    }
    v[i] = failed ? -1.0 : m;
  }
  return {};
}

// Device time of one collective (µs), back to back: max over the local ranks
// of their streams' event spans. -1 when the implementation is rejected.
double time_one(World* w, Kind kind, Impl impl, int64_t s, const std::vector<CallArgs>& args, int iters) {
  for (int i = 0; i < 2; ++i)
    if (!run_collective(w, kind, impl, s, args).ok()) return -1;
  std::vector<cudaEvent_t> b(args.size()), e(args.size());
  for (size_t r = 0; r < args.size(); ++r) {
    DeviceGuard g(w->device[args[r].rank]);
    cudaEventCreate(&b[r]);
    cudaEventCreate(&e[r]);
    cudaStreamSynchronize(args[r].stream);
  }
  for (size_t r = 0; r < args.size(); ++r) {
    DeviceGuard g(w->device[args[r].rank]);
    cudaEventRecord(b[r], args[r].stream);
  }
  bool ok = true;
  for (int i = 0; i < iters && ok; ++i) ok = run_collective(w, kind, impl, s, args).ok();
  double worst = 0;
  for (size_t r = 0; r < args.size(); ++r) {
    DeviceGuard g(w->device[args[r].rank]);
    cudaEventRecord(e[r], args[r].stream);
    cudaEventSynchronize(e[r]);
    float ms = 0;
    if (cudaEventElapsedTime(&ms, b[r], e[r]) != cudaSuccess) ok = false;
    worst = std::max(worst, static_cast<double>(ms) * 1e3 / iters);
    cudaEventDestroy(b[r]);
    cudaEventDestroy(e[r]);
  }
  cudaGetLastError();
  return ok ? worst : -1;
}

Impl pick(Kind kind, int64_t s, const World* w, const std::vector<Impl>& cands, const std::vector<double>& us) {
  int best = -1;
  for (size_t i = 0; i < cands.size(); ++i)
    if (us[i] > 0 && (best < 0 || us[i] < us[best])) best = static_cast<int>(i);
  if (best < 0) return Impl::Auto;
  Impl win = cands[best];
  auto time_of = [&](Impl c) {
    for (size_t i = 0; i < cands.size(); ++i)
      if (cands[i] == c) return us[i];
    return -1.0;
  };
  // winner_grid (sweep.cpp:206-214): the plain variant wins a near tie
  if (is_prelaunched(win)) {
    const double plain = time_of(base_of(win));
    if (plain > 0 && plain <= us[best] * (1 + kPrelaunchGain)) win = base_of(win);
  }
  // measurement noise must not flip the table between near-equal programs:
  // the static selector's choice keeps a tie within kStaticMargin
  const Impl stat = select(kind, s, w->nranks, w->ndevices, 0);
  const double ts = time_of(stat);
  if (ts > 0 && ts <= us[best] * kStaticMargin) win = stat;
  return win;
}

}  // namespace

Impl tuned_select(const World* w, Kind kind, int64_t s) {
  auto it = w->tuned.find(static_cast<int>(kind));
  if (it == w->tuned.end() || it->second.empty()) return Impl::Auto;
  const auto& t = it->second;  // ascending sizes
  if (s <= t.front().first) return t.front().second;
  if (s >= t.back().first) return t.back().second;
  for (size_t i = 1; i < t.size(); ++i) {
    if (s > t[i].first) continue;
    const double a = static_cast<double>(t[i - 1].first), b = static_cast<double>(t[i].first);
    // nearest tuned size on a log scale
    return static_cast<double>(s) * static_cast<double>(s) < a * b ? t[i - 1].second : t[i].second;
  }
  return t.back().second;
}

Status world_tune(World* w, const std::vector<int>& ranks, int64_t max_chunk, const std::vector<cudaStream_t>& streams,
                  std::string* report) {
  if (armed_units() > 0)
    return fail(CECOLL_INVALID_ARGUMENT, "cecoll_tune: a prelaunch plan is armed (its gate would stall the sweep)");
  if (max_chunk <= 0) max_chunk = int64_t{64} << 20;
  const int n = w->nranks;
  std::vector<int64_t> sizes;
  for (int64_t s = 4096; s <= max_chunk; s *= 4) sizes.push_back(s);
  if (sizes.empty()) return fail(CECOLL_INVALID_ARGUMENT, "cecoll_tune: max_chunk_bytes below 4 KiB");
  const int64_t top = sizes.back();
  // scratch buffers, allocated in the same order in every process (registered
  // windows in multi-process worlds: the allocation is collective)
  std::vector<void*> send(ranks.size(), nullptr), recv(ranks.size(), nullptr);
  Status st;
  for (size_t k = 0; k < ranks.size() && st.ok(); ++k) st = world_mem_alloc(w, ranks[k], n * top, &send[k]);
  for (size_t k = 0; k < ranks.size() && st.ok(); ++k) st = world_mem_alloc(w, ranks[k], n * top, &recv[k]);
  std::map<int, std::vector<std::pair<int64_t, Impl>>> table;
  std::ostringstream log;
  if (st.ok()) {
    for (size_t k = 0; k < ranks.size(); ++k) {
      DeviceGuard g(w->device[ranks[k]]);
      cudaMemsetAsync(send[k], k & 0xff, n * top, streams[k]);
    }
    for (Kind kind : {Kind::AllGather, Kind::AllToAll}) {
      const std::vector<Impl> cands = tune_candidates(kind);
      for (int64_t s : sizes) {
        std::vector<CallArgs> args;
        for (size_t k = 0; k < ranks.size(); ++k) args.push_back({ranks[k], send[k], recv[k], streams[k]});
        const int64_t bytes = int64_t{n} * n * s;
        const int iters = static_cast<int>(std::clamp<int64_t>((int64_t{256} << 20) / bytes, 3, 50));
        std::vector<double> us;
        for (Impl c : cands) us.push_back(time_one(w, kind, c, s, args, iters));
        st = agree_max(w, us);
        if (!st.ok()) break;
        const Impl win = pick(kind, s, w, cands, us);
        log << (kind == Kind::AllGather ? "allgather" : "alltoall") << " " << s;
        for (size_t i = 0; i < cands.size(); ++i) log << " " << impl_name(cands[i]) << "=" << us[i];
        log << " -> " << (win == Impl::Auto ? "none" : impl_name(win)) << "\n";
        if (win != Impl::Auto) table[static_cast<int>(kind)].push_back({s, win});
      }
      if (!st.ok()) break;
    }
  }
  // drop the plans built on the scratch buffers, then free them
  std::vector<std::unique_ptr<Plan>> keep;
  for (auto& p : w->plans) {
    bool scratch = false;
    for (const void* k : p->key_send) scratch |= std::find(send.begin(), send.end(), k) != send.end();
    if (scratch) {
      if (w->last_plan == p.get()) w->last_plan = nullptr;
      retire_plan(w, std::move(p));
    } else {
      keep.push_back(std::move(p));
    }
  }
  w->plans.swap(keep);
  for (size_t k = 0; k < ranks.size(); ++k) {
    DeviceGuard g(w->device[ranks[k]]);
    cudaStreamSynchronize(streams[k]);
  }
  for (void* p : send)
    if (p) world_mem_free(w, p);
  for (void* p : recv)
    if (p) world_mem_free(w, p);
  if (!st.ok()) return st;
  w->tuned = std::move(table);
  w->tune_report = log.str();
  if (report) *report = w->tune_report;
  return {};
}

std::string tuned_text(const World* w) {
  std::ostringstream o;
  for (const auto& kv : w->tuned)
    for (const auto& e : kv.second)
      o << (static_cast<Kind>(kv.first) == Kind::AllGather ? "allgather" : "alltoall") << " " << e.first << " "
        << impl_name(e.second) << "\n";
  return o.str();
}

Status tuned_load(World* w, const std::string& text) {
  std::map<int, std::vector<std::pair<int64_t, Impl>>> table;
  std::istringstream in(text);
  std::string kind, impl;
  int64_t s = 0;
  while (in >> kind >> s >> impl) {
    Kind k;
    if (kind == "allgather") k = Kind::AllGather;
    else if (kind == "alltoall") k = Kind::AllToAll;
    else return fail(CECOLL_INVALID_ARGUMENT, "cecoll_tune_load: unknown collective '" + kind + "'");
    Impl i;
    if (!parse_impl(impl, &i) || i == Impl::Auto || !(valid_for(i, k) || i == Impl::Sm || i == Impl::Hybrid ||
                                                       i == Impl::Pull))
      return fail(CECOLL_INVALID_ARGUMENT, "cecoll_tune_load: '" + impl + "' does not apply to " + kind);
    if (s <= 0) return fail(CECOLL_INVALID_ARGUMENT, "cecoll_tune_load: chunk size must be positive");
    table[static_cast<int>(k)].push_back({s, i});
  }
  if (!in.eof()) return fail(CECOLL_INVALID_ARGUMENT, "cecoll_tune_load: expected '<collective> <bytes> <impl>' lines");
  for (auto& kv : table) std::sort(kv.second.begin(), kv.second.end(), [](auto& a, auto& b) { return a.first < b.first; });
  w->tuned = std::move(table);
  return {};
}

}  // namespace cecoll
