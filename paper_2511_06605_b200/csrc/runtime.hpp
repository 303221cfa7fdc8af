// Communicator, plans and executors (world.cpp, lower.cpp, exec.cpp).
//
// Execution model:
//  * A World is every rank this process can address. comm_init_all builds one
//    World whose ranks are all local (one host thread drives every device, the
//    reference's single host process); comm_init_rank builds one
//    local rank per process and maps the peers' flag pages and registered
//    windows through CUDA IPC.
//  * A unit is the set of local ranks that share a device and a caller
//    stream; stream order already orders their readiness and completion.
//    Between units synchronisation is flag based (§2.4 atomic and
//    poll commands; program.hpp:47): every rank owns a page of u64 slots in
//    device memory. rdy[j] in rank r's page is written by rank j when j's
//    destination buffer may be written by r; done[i] in rank r's page is
//    written after rank i's chunk landed in r. Waiters reset a slot to 0 in
//    the same batch, so recorded graphs replay with constant values, and a
//    slot's next write is always causally after its reset.
//  * A Plan is a Program (program.hpp) lowered onto concrete buffers: per lane
//    the polls, the copy-engine copies or kernel items, and the signals; per
//    unit the start/finish flag operations, the SM item table and, for
//    prelaunch_*, the recorded graph. Plans are cached per call signature.
#pragma once

#include <atomic>
#include <chrono>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "cecoll.h"
#include "cu_driver.hpp"
#include "kernels.hpp"
#include "program.hpp"

namespace cecoll {

constexpr int kMaxRanks = 32;
constexpr int kMaxLanes = 32;
// Flag page layout (u64 slots).
constexpr int kSlotRdy = 0;             // rdy[j], j < kMaxRanks
constexpr int kSlotDone = kMaxRanks;    // done[i]
constexpr size_t kFlagBytes = 4096;

// World::counters (exported by cecoll_comm_counters in this order).
enum Counter : int {
  kCtrCollectives = 0,
  kCtrCopies = 1,            // copy commands issued (CE memcpys)
  kCtrFlagWrites = 2,
  kCtrFlagWaits = 3,
  kCtrKernels = 4,
  kCtrGraphLaunches = 5,     // prelaunch graphs
  kCtrApiCalls = 6,          // host CUDA calls issued by the executors
  kCtrRecordedLaunches = 7,  // replays of a recorded command list
  kNumCounters = 8,
};

struct Status {
  int code = 0;
  std::string msg;
  bool ok() const { return code == 0; }
};

struct RankState {
  int rank = -1;
  int device = -1;
  std::vector<cudaStream_t> lanes;
  std::vector<cudaEvent_t> lane_done;
  cudaEvent_t start = nullptr;
  uint64_t* flags = nullptr;  // own flag page (device memory)
  bool owns_flags = true;
};

struct Window {  // a symmetric registered window: its base in every rank, as mapped here
  size_t bytes = 0;
  std::vector<char*> rank_base;
  bool live = true;  // false once any local rank deregistered it
};

struct ProcInfoView {
  int first = 0, nlocal = 0, device = -1;
  cudaIpcMemHandle_t flags;
  unsigned char uuid[16];
};

struct Plan;

// Trace recording state (trace.cpp): CUDA event pairs per traced command and
// host spans, turned into the reference's trace-event JSON at trace_end.
struct Tracer {
  struct Span {
    std::string name;
    int pid, tid, device;
    cudaEvent_t b, e;
  };
  struct HostSpan {
    std::string name;
    double b_us, e_us;
  };
  std::vector<Span> spans;
  std::vector<HostSpan> host;
  std::vector<std::pair<cudaEvent_t, int>> events;  // every recorded event, for release
  std::map<int, cudaEvent_t> base;                  // per device: time zero
  std::chrono::steady_clock::time_point host0;
};

struct World {
  int nranks = 0;
  bool multiprocess = false;
  int ndevices = 1;
  std::vector<int> device;           // per rank
  std::vector<uint64_t*> flag_page;  // per rank, usable from this process
  std::vector<std::unique_ptr<RankState>> local;  // by rank; null if remote
  std::atomic<int64_t> counters[kNumCounters];
  std::vector<std::unique_ptr<Plan>> plans;  // eager-call plan cache
  // Plans evicted from the cache (or dropped at deregistration) wait here
  // until no prelaunch unit of the process is armed (exec.cpp retire_plan).
  std::vector<std::unique_ptr<Plan>> retired;
  // SM budget for plans created from now on (cecoll_comm_set_sm_budget): the
  // most CTAs any mover / reduction kernel of a plan may launch (0: a full
  // persistent grid), and the AUTO selector prefers copy-engine lanes.
  int sm_budget = 0;
  // Measured winner grid (cecoll_tune / cecoll_tune_load, tune.cpp): per
  // collective kind, ascending (chunk bytes, implementation); when present
  // and no SM budget is set it drives CECOLL_IMPL_AUTO for this world.
  std::map<int, std::vector<std::pair<int64_t, Impl>>> tuned;
  std::string tune_report;  // the last cecoll_tune's measurements, one line per size
  Plan* last_plan = nullptr;  // the cached plan of the latest eager call (cecoll_comm_last_plan_info)
  std::vector<Plan*> explicit_plans;         // cecoll_plan_create; cancelled at release
  std::vector<Window> windows;
  std::vector<int> reg_rounds;  // per local index
  std::vector<void*> ipc_opened;
  std::vector<std::pair<void*, int>> allocs;  // cecoll_mem_alloc: pointer, device
  std::map<std::string, void*> ipc_by_handle;
  void* flag_block = nullptr;
  int first_local = 0, nlocal = 0;
  cecoll_exchange_fn exchange = nullptr;  // multi-process: kept for registration
  void* exchange_ctx = nullptr;
  int live_comms = 0;
  // First failure of a cached plan found at its release or by
  // cecoll_comm_get_async_error (a device-side flag poll timed out); sticky,
  // returned by the communicator's destroy.
  Status async_error;
  std::unique_ptr<Tracer> tracer;  // non-null between cecoll_trace_begin and _end
  std::string trace_json;          // last finished trace, until read through the C ABI
  World() {
    for (auto& c : counters) c = 0;
  }
};

struct Copy {
  char* dst;
  const char* src;
  int64_t bytes;
};

using MemOps = std::vector<CUstreamBatchMemOpParams>;

struct LaneExec {
  int rank = 0;
  int lane = 0;
  MemOps pre;                 // rdy polls (+ resets) for destinations in other units
  std::vector<Copy> copies;   // copy commands
  ItemTable table;            // Broadcast / Swap commands (no copy-engine form)
  MemOps post;                // done signals to destinations in other units (same device)
  // (signals whose flag page lives on another device are the unit's
  // lanes_remote: one signal kernel after the lanes join)
};

struct Unit {
  int device = -1;
  cudaStream_t stream = nullptr;  // shared caller stream
  std::vector<int> ranks;         // local ranks, ascending
  MemOps start;                   // rdy signals to sources in other units
  MemOps finish;                  // done polls (+ resets) from sources in other units
  MemOps sm_pre, sm_post;         // SM path: rdy polls / done signals
  std::vector<uint64_t*> start_remote, sm_post_remote;  // other-device flags (signal kernel)
  uint64_t** start_remote_tab = nullptr;
  uint64_t** sm_post_remote_tab = nullptr;
  // The lanes' done signals to other-device flags, written by one signal
  // kernel on the unit stream after the lanes join (one kernel per unit
  // instead of one per lane; a destination waits for all its sources anyway).
  std::vector<uint64_t*> lanes_remote;
  uint64_t** lanes_remote_tab = nullptr;
  // SM path with the flag work fused into the item kernel (kernels.hpp
  // FlagSet): device tables of the sm_pre poll and sm_post signal addresses.
  bool fused = false;
  bool start_folded = false;  // the start signals are the fused kernel's `pre` writes
  FlagSet sm_flags;
  std::vector<Copy> placement;    // local-slot placement (verifier.cpp:40-44)
  std::vector<Copy> precopy;      // swap with send != recv: send -> recv first
  ItemTable table;                // SM path: every chunk of the unit's ranks
  RedTable red;                   // reduce-scatter: one reduction per local rank
  // prelaunch graph
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t arm = nullptr;
  cudaEvent_t graph_done = nullptr;
  uint64_t* err = nullptr;         // device
  uint64_t** poll_tab = nullptr;   // device array of flag pointers
  uint64_t** sig_tab = nullptr;
  uint64_t** fin_tab = nullptr;
  int npoll = 0, nsig = 0, nfin = 0;
  // Trigger word (device memory owned by the plan, one per unit, so armed
  // plans never share one): the caller stream writes 1 to trigger; the gate
  // takes it.
  uint64_t* ready_flag = nullptr;
  uint64_t** ready_tab = nullptr;  // {ready_flag} in device memory (CECOLL_TRIGGER_KERNEL=1)
  // Cancels: a count in pinned host memory (written by the host, no stream)
  // and its device alias; the gate honours each raise once.
  uint64_t* cancel_host = nullptr;
  uint64_t* cancel_dev = nullptr;
  uint64_t cancels = 0;
  bool armed = false;
  // Recorded command list of a non-prelaunch plan (exec.cpp record_plan):
  // the unit's whole submission (flags, lanes, copies, kernels) as one graph.
  cudaGraph_t rec_graph = nullptr;
  cudaGraphExec_t rec_exec = nullptr;
};

struct Plan {
  Kind kind = Kind::AllGather;
  Impl impl = Impl::Pcpy;
  int64_t chunk = 0;
  std::vector<const void*> key_send;
  std::vector<void*> key_recv;
  std::vector<cudaStream_t> key_stream;
  std::vector<int> key_rank;
  std::vector<LaneExec> lanes;
  std::vector<Unit> units;
  std::vector<void*> dev_allocs;
  std::vector<int> dev_alloc_device;
  Program program;
  bool sm = false;       // SM path flag structure (sm, hybrid)
  bool hybrid = false;   // + copy-engine lanes for each chunk's CE share
  bool pull = false;     // lanes belong to the destination and read the sources
  int64_t hybrid_sm_bytes = 0;  // SM share of every chunk (16-byte multiple)
  bool prelaunch = false;
  int sms = 148;
  int sm_budget = 0;              // max CTAs per kernel of this plan (0: full grid)
  bool folded = false;            // prelaunch body is one kernel that is its own gate
  int dtype = 0, op = 0;          // reduce-scatter element type / operator
  std::unique_ptr<Plan> inner;    // reduce-scatter over copy engines: the all-to-all into staging
  std::string graph_fallback;     // why a prelaunch plan runs without its graph (empty: it has one)
  // Non-prelaunch plans are recorded into one CUDA graph per unit at their
  // second launch and replayed afterwards (command scheduling paid once).
  int launches = 0;
  bool recorded = false;
  std::string record_note;        // why recording failed (then the plan stays eager)
  int64_t rec_delta[kNumCounters] = {};      // counter increments of one recorded launch
};

void set_error(const std::string& msg);
const char* last_error();

Status world_init_all(int nranks, const int* devlist, World** out);
Status world_init_ranks(int nranks, int first, int nlocal, int device, cecoll_exchange_fn fn, void* ctx,
                        World** out);
// The init exchange on its own (host only; no CUDA calls): validates that the
// processes' rank ranges tile [0, nranks) and returns them.
Status gather_procs(int nranks, int first, int nlocal, int device, const cudaIpcMemHandle_t* flags,
                    cecoll_exchange_fn fn, void* ctx, std::vector<ProcInfoView>* out,
                    const unsigned char* uuid = nullptr, int32_t local_status = 0);
Status world_release(World* w);  // the world's async error, if any
// Sticky async error of the world, refreshed from every live plan's device
// error words (read on a private stream: never waits for armed graphs).
Status world_async_error(World* w);
void note_async(World* w, const Status& s);
Status world_register(World* w, int rank, void* ptr, size_t bytes, cecoll_exchange_fn fn, void* ctx);
Status world_deregister(World* w, void* ptr);
Status world_mem_alloc(World* w, int rank, size_t bytes, void** out);
Status world_mem_free(World* w, void* ptr);

struct CallArgs {
  int rank;
  const void* send;
  void* recv;
  cudaStream_t stream;
};

Status run_collective(World* w, Kind kind, Impl impl, int64_t chunk, const std::vector<CallArgs>& args);

// `given`: execute this program (e.g. parsed from the reference's
// dump_program text) instead of compiling one.
// `no_placement`: skip the local-slot placement copies (the reduce-scatter's
// copy-engine gather reads each rank's own chunk in place).
Status plan_create(World* w, Kind kind, Impl impl, int64_t chunk, const std::vector<CallArgs>& args, Plan** out,
                   const Program* given = nullptr, bool no_placement = false);
// Reduce-scatter: count elements of `dtype` per rank chunk.
// impl Sm: one kernel per unit reads every rank's chunk (peer loads over
// NVLink); pcpy / b2b / prelaunch_*: an all-to-all over the copy engines into
// a per-rank staging buffer, then one reduction kernel per unit (§6.1).
Status plan_create_rs(World* w, Impl impl, int64_t count, int dtype, int op, const std::vector<CallArgs>& args,
                      Plan** out);
Status run_reduce_scatter(World* w, Impl impl, int64_t count, int dtype, int op, const std::vector<CallArgs>& args);
Status plan_arm(World* w, Plan* p);
Status plan_disarm(World* w, Plan* p);
Status plan_launch(World* w, Plan* p, bool rearm);
Status plan_destroy(World* w, Plan* p);
Status plan_poll_errors(Plan* p);  // CECOLL_TIMEOUT if a kernel-side poll of the plan timed out
// Plan cache and deferred release (exec.cpp).
constexpr size_t kPlanCacheSize = 64;
void cache_plan(World* w, Plan* p);
void retire_plan(World* w, std::unique_ptr<Plan> p);
void release_retired(World* w, bool force);
int armed_units();  // prelaunch units armed in this process
// Kernel grids under the plan's SM budget.
int plan_grid(const Plan* p, const ItemTable& t);
int plan_red_grid(const Plan* p, const RedTable& t);
std::string plan_info(World* w, const Plan* p);
// AUTO selection for the world (its device count and SM budget).
Impl select_for(World* w, Kind kind, int64_t s);

// tune.cpp: the measured winner grid. world_tune sweeps every applicable
// implementation over 4 KiB x 4^k chunks up to max_chunk on the local ranks
// `ranks` (streams[k] for ranks[k]) and installs the table; tuned_select
// returns Impl::Auto when the world has no table for `kind`.
Status world_tune(World* w, const std::vector<int>& ranks, int64_t max_chunk, const std::vector<cudaStream_t>& streams,
                  std::string* report);
Impl tuned_select(const World* w, Kind kind, int64_t s);
std::string tuned_text(const World* w);
Status tuned_load(World* w, const std::string& text);

// NVLS multicast all-gather windows (mcast.cpp, experimental).
struct McWindow;
Status mc_create(World* w, int rank, int64_t chunk_capacity, McWindow** out);
Status mc_allgather(McWindow* m, const void* send, int64_t chunk, cudaStream_t stream);
void mc_release(McWindow* m);
void* mc_recv(McWindow* m);
const char* mc_how(McWindow* m);

Status trace_begin(World* w);
Status trace_end(World* w, std::string* json);

}  // namespace cecoll

struct cecoll_comm {
  cecoll::World* world;
  int rank;
};

struct cecoll_mc {
  cecoll::McWindow* m;
};

struct cecoll_plan {
  cecoll::World* world;
  cecoll::Plan* plan;
};
