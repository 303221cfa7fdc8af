// C shim over the reference's own library — TEST INFRASTRUCTURE ONLY.
//
// Compiled by oracle/Makefile together with the reference's unmodified
// sources (/root/reference/proj/src/{program,compiler,topology,verifier}.cpp)
// into oracle/_ref/libdmasim_ref.so. It exposes the reference's compile(),
// dump_program(), static_metrics(), account_traffic(), verify_collective(),
// validate_program() and select_implementation() through a C ABI so that
// oracle/make_golden.py can record golden vectors and tests can pin the C
// restatement (oracle/cecoll_oracle.c) against the reference itself.
//
// ref_execute() is the byte-level executor the reference lacks (its verifier
// is symbolic, verifier.cpp:11-23): it runs the reference's CommandProgram
// with memcpy semantics after the local placement of verifier.cpp:40-44.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "dmasim/compiler.hpp"
#include "dmasim/program.hpp"
#include "dmasim/topology.hpp"
#include "dmasim/verifier.hpp"

using namespace dmasim;

namespace {

bool build(const char* kind, const char* impl, std::int64_t s, int n, CommandProgram& out) {
  auto k = parse_collective(kind);
  auto im = parse_implementation(impl);
  if (!k || !im) return false;
  try {
    NodeTopology topo = build_topology(n);
    CollectiveSpec spec{*k, s, n, false};
    out = compile(*im, spec, topo);
    return true;
  } catch (const std::invalid_argument&) {
    return false;
  }
}

std::uint8_t* region(const CommandProgram& p, std::uint8_t** in, std::uint8_t** out, const BufferRef& r) {
  bool input = p.metadata.spec.in_place || r.buffer == BufferId::Input;
  return (input ? in[r.gpu] : out[r.gpu]) + r.offset;
}

}  // namespace

extern "C" {

int ref_compile_dump(const char* kind, const char* impl, std::int64_t s, int n, char* buf, std::size_t cap) {
  CommandProgram p;
  if (!build(kind, impl, s, n, p)) return -1;
  std::string text = dump_program(p);
  if (text.size() + 1 > cap) return -2;
  std::memcpy(buf, text.c_str(), text.size() + 1);
  return static_cast<int>(text.size());
}

int ref_metrics(const char* kind, const char* impl, std::int64_t s, int n, int* out5) {
  CommandProgram p;
  if (!build(kind, impl, s, n, p)) return -1;
  MetricsReport m = static_metrics(p);
  out5[0] = m.data_commands;
  out5[1] = m.sync_commands;
  out5[2] = m.poll_commands;
  out5[3] = m.engines_used;
  out5[4] = m.doorbells;
  return 0;
}

int ref_traffic(const char* kind, const char* impl, std::int64_t s, int n, std::int64_t* out3,
                std::int64_t* per_gpu_read, std::int64_t* per_gpu_write) {
  CommandProgram p;
  if (!build(kind, impl, s, n, p)) return -1;
  TrafficReport t = account_traffic(p);
  out3[0] = t.total_read_bytes;
  out3[1] = t.total_write_bytes;
  out3[2] = t.total_link_bytes;
  for (int g = 0; g < n; ++g) {
    auto it = t.per_gpu.find(g);
    per_gpu_read[g] = it == t.per_gpu.end() ? 0 : it->second.hbm_read_bytes;
    per_gpu_write[g] = it == t.per_gpu.end() ? 0 : it->second.hbm_write_bytes;
  }
  return 0;
}

int ref_validate(const char* kind, const char* impl, std::int64_t s, int n) {
  CommandProgram p;
  if (!build(kind, impl, s, n, p)) return -1;
  return validate_program(p, build_topology(n)).ok ? 0 : 1;
}

// Returns VerdictKind (0 ok, 1 mismatch, 2 hazard, 3 invalid) or -1.
int ref_verify(const char* kind, const char* impl, std::int64_t s, int n, std::uint64_t seed) {
  CommandProgram p;
  if (!build(kind, impl, s, n, p)) return -1;
  VerifyOptions opts;
  opts.seed = seed;
  return static_cast<int>(verify_collective(p, p.metadata.spec, opts).kind);
}

int ref_select(const char* kind, std::int64_t size, char* buf, std::size_t cap) {
  auto k = parse_collective(kind);
  if (!k) return -1;
  try {
    std::string name = to_string(select_implementation(*k, size));
    if (name.size() + 1 > cap) return -2;
    std::memcpy(buf, name.c_str(), name.size() + 1);
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

namespace {

void run_queue(const CommandProgram& p, const CommandQueue& q, std::uint8_t** in, std::uint8_t** out,
               std::vector<std::uint8_t>& tmp) {
  for (const auto& c : q.commands) {
    switch (c.kind) {
      case CommandKind::Copy:
        std::memcpy(region(p, in, out, c.dst), region(p, in, out, c.src), c.size);
        break;
      case CommandKind::Broadcast:
        std::memcpy(region(p, in, out, c.dst), region(p, in, out, c.src), c.size);
        std::memcpy(region(p, in, out, c.dst2), region(p, in, out, c.src), c.size);
        break;
      case CommandKind::Swap:
        tmp.resize(c.size);
        std::memcpy(tmp.data(), region(p, in, out, c.src), c.size);
        std::memcpy(region(p, in, out, c.src), region(p, in, out, c.peer), c.size);
        std::memcpy(region(p, in, out, c.peer), tmp.data(), c.size);
        break;
      default:
        break;
    }
  }
}

}  // namespace

// Executes the reference's program with `nthreads` host threads: queues are
// independent (every destination region has one writer, verifier.cpp:202-235),
// so they are distributed round-robin, like the reference's own thread pool
// over independent work (sweep.cpp:113-124).
int ref_execute_mt(const char* kind, const char* impl, std::int64_t s, int n, std::uint8_t** in,
                   std::uint8_t** out, int nthreads) {
  CommandProgram p;
  if (!build(kind, impl, s, n, p)) return -1;
  const CollectiveSpec& spec = p.metadata.spec;
  if (nthreads < 1) nthreads = 1;
  auto work = [&](int t) {
    std::vector<std::uint8_t> tmp;
    if (!spec.in_place)
      for (int g = t; g < n; g += nthreads)
        std::memcpy(out[g] + g * s, in[g] + (spec.kind == CollectiveKind::AllGather ? 0 : g * s), s);
    for (size_t qi = t; qi < p.queues.size(); qi += nthreads) run_queue(p, p.queues[qi], in, out, tmp);
  };
  if (nthreads == 1) {
    work(0);
    return 0;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < nthreads; ++t) pool.emplace_back(work, t);
  for (auto& th : pool) th.join();
  return 0;
}

int ref_execute(const char* kind, const char* impl, std::int64_t s, int n, std::uint8_t** in,
                std::uint8_t** out) {
  return ref_execute_mt(kind, impl, s, n, in, out, 1);
}

}  // extern "C"
