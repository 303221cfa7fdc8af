// Command programs: the B200 library's compile() stage.
//
// A Program is the per-rank, per-lane command list that the executors in
// exec.cpp lower onto CUDA streams, graphs and sm_100a kernels. It keeps the
// reference's command IR (proj/include/dmasim/program.hpp:36-87) so that the
// exact program the hardware runs can be dumped in the reference's
// dump_program format and compared with it (tests/golden/programs.json).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace cecoll {

// ReduceScatter is the B200 extension of SURVEY §8(f)4 (no reference program).
enum class Kind : int { AllGather = 0, AllToAll = 1, ReduceScatter = 2 };

// Implementation ids follow compiler.hpp:12-21; Sm is the B200 SM path.
enum class Impl : int {
  Auto = -1,
  Pcpy = 0,
  Bcst = 1,
  Swap = 2,
  B2b = 3,
  PrelaunchPcpy = 4,
  PrelaunchBcst = 5,
  PrelaunchSwap = 6,
  PrelaunchB2b = 7,
  Sm = 8,
  // B200 hybrid: each chunk is split between a copy-engine lane (the pcpy
  // rotation, compiler.cpp:150) and the SM mover (SURVEY §7 "hybrid CE + SM
  // lanes" fallback when copy engines alone cannot fill NVLink).
  Hybrid = 9,
  // B200 pull: the destination's copy-engine lanes read every source's chunk
  // (lane d-1 of rank r reads from (r+d)%n), SURVEY §7's push-vs-pull question.
  Pull = 10,
};

const char* impl_name(Impl impl);
bool parse_impl(const std::string& name, Impl* out);
bool is_prelaunched(Impl impl);
Impl base_of(Impl impl);
bool valid_for(Impl impl, Kind kind);

enum class Buf : int { Input = 0, Output = 1 };

struct Region {
  int rank = 0;
  Buf buf = Buf::Input;
  int64_t off = 0;
  int64_t len = 0;
};

enum class Op : int { Copy = 0, Broadcast, Swap, Signal, Poll, Timestamp };

struct Command {
  Op op = Op::Copy;
  Region src, dst, dst2, peer;
  int64_t size = 0;
  int signal_slot = -1;
  int poll_slot = -1;
  uint64_t expected = 0;
  bool moves_data() const { return op == Op::Copy || op == Op::Broadcast || op == Op::Swap; }
};

// One lane = one copy-engine queue (reference CommandQueue, program.hpp:68-72).
struct Lane {
  int rank = 0;
  int index = 0;  // engine local index
  int doorbells = 1;
  std::vector<Command> cmds;
};

struct Spec {
  Kind kind = Kind::AllGather;
  int64_t chunk = 0;  // s
  int nranks = 0;     // n
  bool in_place = false;
  int64_t input_bytes() const { return kind == Kind::AllGather ? chunk : chunk * nranks; }
  int64_t output_bytes() const { return chunk * nranks; }
};

struct Program {
  Spec spec;
  Impl impl = Impl::Pcpy;
  bool prelaunched = false;
  std::vector<Lane> lanes;  // ordered by (rank, lane index)
  std::vector<int> completion_signals;
  std::vector<int> trigger_slots;
};

struct Metrics {
  int64_t data = 0, sync = 0, poll = 0, engines = 0, doorbells = 0;
};

struct Traffic {
  int64_t read = 0, write = 0, link = 0;
  std::vector<int64_t> rank_read, rank_write;
};

// Throws std::invalid_argument exactly where the reference does.
Program compile(Impl impl, const Spec& spec, int lanes_per_rank);
std::string dump(const Program& p);
Metrics metrics(const Program& p);
Traffic traffic(const Program& p);
// Empty string when valid, else the first violation (program.cpp:98-205).
std::string validate(const Program& p, int lanes_per_rank);
// Inverse of dump(): reads the reference's dump_program text (any program the
// reference's compile() produced, or a hand-made one) so that it can be
// executed as is. Throws std::invalid_argument on malformed text.
Program parse_dump(const std::string& text, Kind kind, int64_t chunk, int nranks);

Impl reference_select(Kind kind, int64_t size);
Impl select(Kind kind, int64_t size, int nranks, int ndevices, int sm_budget = 0);

}  // namespace cecoll
