// compile(): collective → per-lane command program.
//
// Each implementation is expressed as a lane policy over the same set of
// routes. A route is one (source rank → destination rank) chunk transfer;
// rank i's routes are visited in the rotation j = (i + d) % n, d = 1..n-1
// (compiler.cpp:149-150, 251-252), which makes every lane index a permutation
// of destinations across ranks (no incast on a lane).
#include "program.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>
#include <sstream>
#include <stdexcept>

namespace cecoll {

namespace {
constexpr int kTriggerBase = 100000;  // apply_prelaunch slot base (compiler.cpp:89)

const char* const kNames[] = {"pcpy",           "bcst",           "swap",           "b2b",
                              "prelaunch_pcpy", "prelaunch_bcst", "prelaunch_swap", "prelaunch_b2b",
                              "sm",             "hybrid",         "pull"};
}  // namespace

const char* impl_name(Impl impl) {
  int i = static_cast<int>(impl);
  if (impl == Impl::Auto) return "auto";
  return (i >= 0 && i <= 10) ? kNames[i] : "?";
}

bool parse_impl(const std::string& name, Impl* out) {
  if (name == "baseline") {  // compiler.cpp:25
    *out = Impl::Pcpy;
    return true;
  }
  if (name == "auto") {
    *out = Impl::Auto;
    return true;
  }
  for (int i = 0; i <= 10; ++i)
    if (name == kNames[i]) {
      *out = static_cast<Impl>(i);
      return true;
    }
  return false;
}

bool is_prelaunched(Impl impl) { return impl >= Impl::PrelaunchPcpy && impl <= Impl::PrelaunchB2b; }

Impl base_of(Impl impl) {
  return is_prelaunched(impl) ? static_cast<Impl>(static_cast<int>(impl) - 4) : impl;
}

bool valid_for(Impl impl, Kind kind) {
  Impl b = base_of(impl);
  if (b == Impl::Bcst) return kind == Kind::AllGather;
  if (b == Impl::Swap) return kind == Kind::AllToAll;
  return true;
}

namespace {

void check_spec(const Spec& s) {  // validate_spec, program.cpp:31-38
  if (s.chunk <= 0) throw std::invalid_argument("collective: chunk size must be positive");
  if (s.nranks < 2) throw std::invalid_argument("collective: gpu_count must be >= 2");
  if (s.kind == Kind::AllGather && s.in_place)
    throw std::invalid_argument("collective: allgather forbids in_place");
}

// Source of rank i's transfer to rank j, and its landing slot at j.
Region route_src(const Spec& s, int i, int j) {
  if (s.kind == Kind::AllGather) return {i, Buf::Input, 0, s.chunk};
  return {i, Buf::Input, j * s.chunk, s.chunk};
}
Region landing(const Spec& s, int j, int i) {
  return {j, s.in_place ? Buf::Input : Buf::Output, i * s.chunk, s.chunk};
}

class Emitter {
 public:
  explicit Emitter(Program& p) : p_(p) {}
  Lane& lane(int rank) {
    Lane l;
    l.rank = rank;
    l.index = next_lane_[rank]++;
    p_.lanes.push_back(std::move(l));
    return p_.lanes.back();
  }
  void close(Lane& l) {  // every data lane ends with exactly one signal
    Command c;
    c.op = Op::Signal;
    c.signal_slot = next_signal_++;
    l.cmds.push_back(c);
    p_.completion_signals.push_back(c.signal_slot);
  }

 private:
  Program& p_;
  std::map<int, int> next_lane_;
  int next_signal_ = 0;
};

Command copy_cmd(const Region& src, const Region& dst) {
  Command c;
  c.op = Op::Copy;
  c.src = src;
  c.dst = dst;
  c.size = src.len;
  return c;
}

// pcpy (compiler.cpp:139-164): one lane per route.
void lanes_pcpy(Program& p, int lanes_per_rank) {
  const Spec& s = p.spec;
  if (s.in_place) throw std::invalid_argument("pcpy compiles out-of-place only");
  if (lanes_per_rank < s.nranks - 1) throw std::invalid_argument("pcpy needs n-1 engines per gpu");
  Emitter e(p);
  for (int i = 0; i < s.nranks; ++i)
    for (int d = 1; d < s.nranks; ++d) {
      const int j = (i + d) % s.nranks;
      Lane& l = e.lane(i);
      l.cmds.push_back(copy_cmd(route_src(s, i, j), landing(s, j, i)));
      e.close(l);
    }
}

// b2b (compiler.cpp:241-265): all routes of a rank back to back on one lane.
void lanes_b2b(Program& p) {
  const Spec& s = p.spec;
  if (s.in_place) throw std::invalid_argument("b2b compiles out-of-place only");
  Emitter e(p);
  for (int i = 0; i < s.nranks; ++i) {
    Lane& l = e.lane(i);
    for (int d = 1; d < s.nranks; ++d) {
      const int j = (i + d) % s.nranks;
      l.cmds.push_back(copy_cmd(route_src(s, i, j), landing(s, j, i)));
    }
    e.close(l);
  }
}

// bcst (compiler.cpp:166-205): routes d=(2k+1, 2k+2) fused into one
// two-destination command; with even n the last route d=n-1 stays a copy.
void lanes_bcst(Program& p, int lanes_per_rank) {
  const Spec& s = p.spec;
  if (s.kind == Kind::AllToAll) throw std::invalid_argument("bcst applies to allgather only");
  const int n = s.nranks;
  const int pairs = (n - 1) / 2;
  const bool odd_route = n % 2 == 0;
  if (lanes_per_rank < pairs + (odd_route ? 1 : 0))
    throw std::invalid_argument("bcst needs ceil((n-1)/2) engines per gpu");
  Emitter e(p);
  for (int i = 0; i < n; ++i) {
    for (int k = 0; k < pairs; ++k) {
      Lane& l = e.lane(i);
      Command c;
      c.op = Op::Broadcast;
      c.src = route_src(s, i, i);
      c.dst = landing(s, (i + 2 * k + 1) % n, i);
      c.dst2 = landing(s, (i + 2 * k + 2) % n, i);
      c.size = s.chunk;
      l.cmds.push_back(c);
      e.close(l);
    }
    if (odd_route) {
      Lane& l = e.lane(i);
      l.cmds.push_back(copy_cmd(route_src(s, i, i), landing(s, (i + n - 1) % n, i)));
      e.close(l);
    }
  }
}

// swap (compiler.cpp:207-239): one in-place exchange per unordered pair,
// issued by the lower rank when the forward distance is at most n/2.
void lanes_swap(Program& p, int lanes_per_rank) {
  Spec& s = p.spec;
  s.in_place = true;
  check_spec(s);
  if (s.kind != Kind::AllToAll) throw std::invalid_argument("swap applies to alltoall only");
  const int n = s.nranks;
  std::vector<std::vector<int>> owned(n);
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const bool lower_owns = (j - i) <= n / 2;
      owned[lower_owns ? i : j].push_back(lower_owns ? j : i);
    }
  if (lanes_per_rank < n / 2) throw std::invalid_argument("swap needs ceil((n-1)/2) engines per gpu");
  Emitter e(p);
  for (int g = 0; g < n; ++g)
    for (int peer : owned[g]) {
      Lane& l = e.lane(g);
      Command c;
      c.op = Op::Swap;
      c.src = route_src(s, g, peer);
      c.peer = route_src(s, peer, g);
      c.size = s.chunk;
      l.cmds.push_back(c);
      e.close(l);
    }
}

// apply_prelaunch (compiler.cpp:267-285): one trigger poll heads each lane.
void prelaunch(Program& p) {
  if (p.prelaunched) throw std::invalid_argument("program is already prelaunched");
  int slot = kTriggerBase;
  for (Lane& l : p.lanes) {
    if (l.cmds.empty()) continue;
    Command c;
    c.op = Op::Poll;
    c.poll_slot = slot++;
    c.expected = 1;
    l.cmds.insert(l.cmds.begin(), c);
    p.trigger_slots.push_back(c.poll_slot);
  }
  p.prelaunched = true;
}

}  // namespace

Program compile(Impl impl, const Spec& spec, int lanes_per_rank) {
  if (impl == Impl::Auto || impl == Impl::Sm || static_cast<int>(impl) < 0 || static_cast<int>(impl) > 8)
    throw std::invalid_argument("compile: no command program for this implementation");
  if (!valid_for(impl, spec.kind))
    throw std::invalid_argument(std::string(impl_name(impl)) + " does not apply to " +
                                (spec.kind == Kind::AllGather ? "allgather" : "alltoall"));
  Program p;
  p.spec = spec;
  p.spec.in_place = base_of(impl) == Impl::Swap;
  p.impl = base_of(impl);
  check_spec(p.spec);
  switch (base_of(impl)) {
    case Impl::Pcpy: lanes_pcpy(p, lanes_per_rank); break;
    case Impl::Bcst: lanes_bcst(p, lanes_per_rank); break;
    case Impl::Swap: lanes_swap(p, lanes_per_rank); break;
    default: lanes_b2b(p); break;
  }
  if (is_prelaunched(impl)) {
    prelaunch(p);
    p.impl = impl;
  }
  return p;
}

namespace {
std::string region_str(const Region& r) {
  std::ostringstream o;
  o << "g" << r.rank << (r.buf == Buf::Input ? ".in[" : ".out[") << r.off << "+" << r.len << "]";
  return o.str();
}
}  // namespace

// dump_program format (program.cpp:218-254): tab-separated, one line per command.
std::string dump(const Program& p) {
  static const char* ops[] = {"copy", "broadcast", "swap", "signal", "poll", "timestamp"};
  std::ostringstream o;
  for (size_t li = 0; li < p.lanes.size(); ++li) {
    const Lane& l = p.lanes[li];
    for (size_t ci = 0; ci < l.cmds.size(); ++ci) {
      const Command& c = l.cmds[ci];
      o << "q" << li << "(g" << l.rank << "e" << l.index << ")\t" << ci << "\t" << ops[static_cast<int>(c.op)]
        << "\t";
      switch (c.op) {
        case Op::Copy: o << region_str(c.src) << "\t" << region_str(c.dst) << "\t" << c.size << "\t-"; break;
        case Op::Broadcast:
          o << region_str(c.src) << "\t" << region_str(c.dst) << "," << region_str(c.dst2) << "\t" << c.size
            << "\t-";
          break;
        case Op::Swap: o << region_str(c.src) << "\t" << region_str(c.peer) << "\t" << c.size << "\t-"; break;
        case Op::Signal: o << "-\t-\t0\t" << c.signal_slot; break;
        case Op::Poll: o << "-\t-\t0\t" << c.poll_slot; break;
        case Op::Timestamp: o << "-\t-\t0\t-"; break;
      }
      o << "\n";
    }
  }
  return o.str();
}

Metrics metrics(const Program& p) {  // static_metrics, program.cpp:40-65
  Metrics m;
  for (const Lane& l : p.lanes) {
    if (l.cmds.empty()) continue;
    m.engines += 1;
    m.doorbells += l.doorbells;
    for (const Command& c : l.cmds) {
      if (c.moves_data()) ++m.data;
      else if (c.op == Op::Signal) ++m.sync;
      else if (c.op == Op::Poll) ++m.poll;
    }
  }
  return m;
}

Traffic traffic(const Program& p) {  // account_traffic, verifier.cpp:281-327
  Traffic t;
  const int n = p.spec.nranks;
  t.rank_read.assign(n, 0);
  t.rank_write.assign(n, 0);
  // Parsed programs may reference gpus outside [0, n) (validate() reports
  // them); their bytes count in the totals only.
  auto rd = [&](int r, int64_t b) {
    t.read += b;
    if (r >= 0 && r < n) t.rank_read[r] += b;
  };
  auto wr = [&](int r, int64_t b) {
    t.write += b;
    if (r >= 0 && r < n) t.rank_write[r] += b;
  };
  for (const Lane& l : p.lanes)
    for (const Command& c : l.cmds) {
      switch (c.op) {
        case Op::Copy:
          rd(c.src.rank, c.size);
          wr(c.dst.rank, c.size);
          if (c.src.rank != c.dst.rank) t.link += c.size;
          break;
        case Op::Broadcast:
          rd(c.src.rank, c.size);
          wr(c.dst.rank, c.size);
          wr(c.dst2.rank, c.size);
          t.link += (c.src.rank != c.dst.rank ? c.size : 0) + (c.src.rank != c.dst2.rank ? c.size : 0);
          break;
        case Op::Swap:
          rd(c.src.rank, c.size);
          rd(c.peer.rank, c.size);
          wr(c.src.rank, c.size);
          wr(c.peer.rank, c.size);
          t.link += 2 * c.size;
          break;
        default: break;
      }
    }
  return t;
}

namespace {
bool overlap(const Region& a, const Region& b) {
  return a.rank == b.rank && a.buf == b.buf && a.off < b.off + b.len && b.off < a.off + a.len;
}
}  // namespace

// Structural invariants of validate_program (program.cpp:98-205).
std::string validate(const Program& p, int lanes_per_rank) {
  const Spec& s = p.spec;
  std::set<std::pair<int, int>> seen;
  std::map<int, int> per_rank;
  std::set<int> trailing, polls;
  auto in_bounds = [&](const Region& r) {
    if (r.rank < 0 || r.rank >= s.nranks) return std::string("buffer ref on unknown gpu");
    if (r.off < 0 || r.len <= 0) return std::string("buffer region must have positive length");
    int64_t cap = r.buf == Buf::Input ? s.input_bytes() : s.output_bytes();
    if (s.in_place) cap = s.output_bytes();
    if (r.off + r.len > cap) return std::string("buffer region out of declared bounds");
    return std::string();
  };
  for (size_t li = 0; li < p.lanes.size(); ++li) {
    const Lane& l = p.lanes[li];
    const std::string where = " (queue " + std::to_string(li) + ")";
    if (l.rank < 0 || l.rank >= s.nranks) return "queue on unknown gpu" + where;
    if (l.index < 0 || l.index >= lanes_per_rank)
      return "engine overflow: local index exceeds engines_per_gpu" + where;
    if (!seen.insert({l.rank, l.index}).second) return "two queues share one engine" + where;
    if (l.cmds.empty()) continue;
    if (++per_rank[l.rank] > lanes_per_rank) return "engine overflow: too many engines used on one gpu" + where;
    if (l.doorbells < 1) return "unrung queue: doorbell_count must be >= 1" + where;
    bool saw_data = false;
    int signals = 0;
    for (const Command& c : l.cmds) {
      std::string err;
      switch (c.op) {
        case Op::Copy:
          if (c.size <= 0) return "copy with nonpositive size" + where;
          if (c.src.len != c.size || c.dst.len != c.size) return "copy src/dst size mismatch" + where;
          if (overlap(c.src, c.dst)) return "copy src and dst overlap" + where;
          if (!(err = in_bounds(c.src)).empty() || !(err = in_bounds(c.dst)).empty()) return err + where;
          saw_data = true;
          break;
        case Op::Broadcast:
          if (c.size <= 0) return "broadcast with nonpositive size" + where;
          if (c.src.len != c.size || c.dst.len != c.size || c.dst2.len != c.size)
            return "broadcast region size mismatch" + where;
          if (c.dst.rank == c.dst2.rank) return "broadcast destinations must be on distinct gpus" + where;
          for (const Region* r : {&c.src, &c.dst, &c.dst2})
            if (!(err = in_bounds(*r)).empty()) return err + where;
          saw_data = true;
          break;
        case Op::Swap:
          if (c.size <= 0) return "swap with nonpositive size" + where;
          if (c.src.len != c.size || c.peer.len != c.size) return "swap region size mismatch" + where;
          if (c.src.rank == c.peer.rank) return "swap regions must be on distinct gpus" + where;
          if (!(err = in_bounds(c.src)).empty() || !(err = in_bounds(c.peer)).empty()) return err + where;
          saw_data = true;
          break;
        case Op::Signal:
          if (c.signal_slot < 0) return "signal without a target slot" + where;
          ++signals;
          break;
        case Op::Poll:
          if (c.poll_slot < 0) return "poll without a slot" + where;
          if (saw_data) return "poll must precede the commands it gates" + where;
          polls.insert(c.poll_slot);
          break;
        case Op::Timestamp: break;
      }
    }
    if (saw_data) {
      if (signals != 1 || l.cmds.back().op != Op::Signal)
        return "unsignaled queue: data queue must end with exactly one AtomicSignal" + where;
      trailing.insert(l.cmds.back().signal_slot);
    }
  }
  if (std::set<int>(p.completion_signals.begin(), p.completion_signals.end()) != trailing)
    return "completion_signals do not match trailing signal targets";
  if (p.prelaunched && p.trigger_slots.empty()) return "prelaunched program without trigger slots";
  if (!p.prelaunched && !p.trigger_slots.empty()) return "trigger slots on a non-prelaunched program";
  if (std::set<int>(p.trigger_slots.begin(), p.trigger_slots.end()) != polls)
    return "trigger_slots do not match the poll slots used";
  return std::string();
}

namespace {

Region parse_region(const std::string& tok) {
  // g<rank>.in[<off>+<len>] | g<rank>.out[<off>+<len>]
  Region r;
  long long rank = 0, off = 0, len = 0;
  char buf[8] = {0};
  if (std::sscanf(tok.c_str(), "g%lld.%3[a-z][%lld+%lld]", &rank, buf, &off, &len) != 4)
    throw std::invalid_argument("parse_dump: bad region '" + tok + "'");
  const std::string b(buf);
  if (b != "in" && b != "out") throw std::invalid_argument("parse_dump: bad buffer '" + tok + "'");
  r.rank = static_cast<int>(rank);
  r.buf = b == "in" ? Buf::Input : Buf::Output;
  r.off = off;
  r.len = len;
  return r;
}

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : s) {
    if (c == sep) {
      out.push_back(cur);
      cur.clear();
    } else {
      cur += c;
    }
  }
  out.push_back(cur);
  return out;
}

}  // namespace

Program parse_dump(const std::string& text, Kind kind, int64_t chunk, int nranks) {
  if (nranks < 1 || nranks > 1024) throw std::invalid_argument("parse_dump: gpu_count out of range");
  if (kind != Kind::AllGather && kind != Kind::AllToAll) throw std::invalid_argument("parse_dump: unknown collective");
  Program p;
  p.spec.kind = kind;
  p.spec.chunk = chunk;
  p.spec.nranks = nranks;
  int last_q = -1;
  for (const std::string& line : split(text, '\n')) {
    if (line.empty()) continue;
    const auto f = split(line, '\t');
    if (f.size() != 7) throw std::invalid_argument("parse_dump: expected 7 fields: " + line);
    int q = -1, g = -1, e = -1;
    if (std::sscanf(f[0].c_str(), "q%d(g%de%d)", &q, &g, &e) != 3)
      throw std::invalid_argument("parse_dump: bad queue '" + f[0] + "'");
    if (q != last_q) {
      if (q != last_q + 1) throw std::invalid_argument("parse_dump: queues must be listed in order");
      Lane l;
      l.rank = g;
      l.index = e;
      p.lanes.push_back(l);
      last_q = q;
    }
    Command c;
    const std::string& op = f[2];
    if (op == "copy") {
      c.op = Op::Copy;
      c.src = parse_region(f[3]);
      c.dst = parse_region(f[4]);
    } else if (op == "broadcast") {
      c.op = Op::Broadcast;
      c.src = parse_region(f[3]);
      const auto d = split(f[4], ',');
      if (d.size() != 2) throw std::invalid_argument("parse_dump: broadcast needs two destinations");
      c.dst = parse_region(d[0]);
      c.dst2 = parse_region(d[1]);
    } else if (op == "swap") {
      c.op = Op::Swap;
      c.src = parse_region(f[3]);
      c.peer = parse_region(f[4]);
      p.spec.in_place = true;
    } else if (op == "signal") {
      c.op = Op::Signal;
      c.signal_slot = std::atoi(f[6].c_str());
      p.completion_signals.push_back(c.signal_slot);
    } else if (op == "poll") {
      c.op = Op::Poll;
      c.poll_slot = std::atoi(f[6].c_str());
      c.expected = 1;
      p.trigger_slots.push_back(c.poll_slot);
      p.prelaunched = true;
    } else if (op == "timestamp") {
      c.op = Op::Timestamp;
    } else {
      throw std::invalid_argument("parse_dump: unknown command '" + op + "'");
    }
    c.size = std::atoll(f[5].c_str());
    p.lanes.back().cmds.push_back(c);
  }
  bool bcst = false, swap = false, multi = false;
  for (const Lane& l : p.lanes) {
    int data = 0;
    for (const Command& c : l.cmds) {
      bcst |= c.op == Op::Broadcast;
      swap |= c.op == Op::Swap;
      data += c.moves_data();
    }
    multi |= data > 1;
  }
  Impl base = swap ? Impl::Swap : bcst ? Impl::Bcst : multi ? Impl::B2b : Impl::Pcpy;
  p.impl = p.prelaunched ? static_cast<Impl>(static_cast<int>(base) + 4) : base;
  return p;
}

// The reference's prescribed table (compiler.cpp:305-318, PAPER Tables 1-2).
Impl reference_select(Kind kind, int64_t size) {
  if (size < (1ll << 10)) throw std::invalid_argument("select_implementation: size below 1KB");
  if (kind == Kind::AllGather) {
    if (size < (256ll << 10)) return Impl::PrelaunchB2b;
    if (size < (1ll << 20)) return Impl::PrelaunchBcst;
    if (size < (512ll << 20)) return Impl::PrelaunchPcpy;
    return Impl::Pcpy;
  }
  if (size < (64ll << 10)) return Impl::PrelaunchB2b;
  if (size < (4ll << 20)) return Impl::PrelaunchSwap;
  if (size < (1ll << 30)) return Impl::PrelaunchPcpy;
  return Impl::Pcpy;
}

// B200 selector (the winner_grid analog, sweep.cpp:186-218). One device
// (co-resident ranks), from profiles/latency_r02_n{8,2}_final.csv and
// profiles/sweep_r02_plan_n{8,2}_final.csv: the SM path wins or ties every
// size of both collectives since the mover runs short-lived CTAs (kernels.cu
// TmaPolicy; round 1's persistent grid lost to the driver's back-to-back
// copies, b2b, by ~5% above 16 MiB all-to-all chunks). Several devices: not
// measured yet — the SM path for latency-bound chunks, per-peer copies (copy
// engines over NVLink, one lane per peer) above; their plans replay as
// recorded graphs (exec.cpp), which beat the gated prelaunch graphs at every
// measured size on one GPU (profiles/sweep_r01_plan_n8_recorded.csv).
// CECOLL_SM_MAX_BYTES overrides the SM cutoff. (bench_mgpu.py measures every
// implementation per size on the multi-GPU node and reports the winner grid.)
Impl select(Kind kind, int64_t size, int nranks, int ndevices, int sm_budget) {
  (void)nranks;
  int64_t sm_max;
  (void)kind;
  if (ndevices <= 1) sm_max = INT64_MAX;
  else sm_max = int64_t{1} << 20;
  // With an SM budget the caller keeps the SMs for its own compute: across
  // devices every transfer above the latency regime goes to the copy engines
  // (per-peer lanes, 0 SMs). On one device the driver itself runs
  // device-local copies on SMs (profiles/ce_probe2_r01.txt), so the budgeted
  // SM mover stays the choice there.
  if (sm_budget > 0 && ndevices > 1) sm_max = int64_t{64} << 10;
  if (const char* env = std::getenv("CECOLL_SM_MAX_BYTES")) sm_max = std::atoll(env);
  if (size <= sm_max) return Impl::Sm;
  return ndevices <= 1 ? Impl::B2b : Impl::Pcpy;
}

}  // namespace cecoll
