/*
 * cecoll — B200-native copy-engine collectives (all-gather, all-to-all).
 *
 * Thin C ABI (plain pointers and sizes; streams are cudaStream_t passed as
 * void*). Every entry point below names the reference interface it replaces
 * or realises; paths are relative to /root/reference/proj.
 *
 * Vocabulary kept from the reference:
 *   - chunk_bytes is the per-peer chunk s (program.hpp:20-31, README.md:29-30).
 *   - all-gather: recv holds n*s bytes, rank i's chunk at [i*s, (i+1)*s)
 *     (compiler.cpp:115-122). all-to-all: send holds n*s bytes, chunk j goes to
 *     rank j's slot `rank` (compiler.cpp:124-126, 156-157).
 *   - implementations pcpy / bcst / swap / b2b and their prelaunch_ variants
 *     (compiler.hpp:12-21); swap is in place (compiler.cpp:207-210, 293).
 *
 * Errors are status codes; the reference's std::invalid_argument sites map to
 * CECOLL_INVALID_ARGUMENT / CECOLL_UNSUPPORTED and its untriggered-poll
 * deadlock (sim.cpp:227-242) to CECOLL_TIMEOUT.
 */
#ifndef CECOLL_H
#define CECOLL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CECOLL_VERSION 1

typedef enum {
  CECOLL_SUCCESS = 0,
  CECOLL_INVALID_ARGUMENT = 1, /* std::invalid_argument (compiler.cpp:142-145, program.cpp:31-38) */
  CECOLL_UNSUPPORTED = 2,      /* impl not valid for the collective (compiler.cpp:70-75, 289-291) */
  CECOLL_CUDA_ERROR = 3,
  CECOLL_TIMEOUT = 4, /* a poll that is never triggered (sim.cpp:237-240) */
  CECOLL_NO_DEVICE = 5,
  CECOLL_NOT_REGISTERED = 6, /* buffer not reachable from a peer rank */
  CECOLL_INTERNAL = 7
} cecoll_status_t;

typedef enum { CECOLL_ALLGATHER = 0, CECOLL_ALLTOALL = 1 } cecoll_kind_t; /* CollectiveKind, program.hpp:13 */

/* Implementation (compiler.hpp:12-21) plus the B200 SM path and AUTO. */
typedef enum {
  CECOLL_IMPL_AUTO = -1, /* cecoll_select() */
  CECOLL_IMPL_PCPY = 0,
  CECOLL_IMPL_BCST = 1,
  CECOLL_IMPL_SWAP = 2,
  CECOLL_IMPL_B2B = 3,
  CECOLL_IMPL_PRELAUNCH_PCPY = 4,
  CECOLL_IMPL_PRELAUNCH_BCST = 5,
  CECOLL_IMPL_PRELAUNCH_SWAP = 6,
  CECOLL_IMPL_PRELAUNCH_B2B = 7,
  CECOLL_IMPL_SM = 8, /* one-shot sm_100a push kernel (latency regime) */
  CECOLL_IMPL_HYBRID = 9 /* each chunk split: copy-engine lane (pcpy rotation) + sm_100a mover;
                            SM share CECOLL_HYBRID_SM_PCT percent (default 50), read per plan */,
  CECOLL_IMPL_PULL = 10 /* destination-issued copy-engine reads, one lane per source (pcpy rotation) */
} cecoll_impl_t;

typedef struct cecoll_comm* cecoll_comm_t;
typedef struct cecoll_program* cecoll_program_t;
typedef struct cecoll_plan* cecoll_plan_t;

const char* cecoll_strerror(cecoll_status_t status);
/* to_string / parse_implementation (compiler.cpp:8-37; "baseline" = pcpy). */
const char* cecoll_impl_name(cecoll_impl_t impl);
cecoll_impl_t cecoll_parse_impl(const char* name); /* returns -2 when unknown */
/* valid_for (compiler.cpp:70-75) */
int cecoll_impl_valid_for(cecoll_impl_t impl, cecoll_kind_t kind);
/* Last error message recorded on this thread (first violation found). */
const char* cecoll_last_error(void);

/* ---------------------------------------------------------------------
 * Command programs (CPU only; no GPU required).
 * Replaces compile(Implementation, CollectiveSpec, NodeTopology)
 * (compiler.hpp:55-56, compiler.cpp:287-303) with the node model reduced to
 * `lanes_per_rank` (engines_per_gpu, topology.hpp:34); the returned program has
 * the reference's queue/command structure exactly.
 * ------------------------------------------------------------------- */
cecoll_status_t cecoll_program_compile(cecoll_kind_t kind, cecoll_impl_t impl, int64_t chunk_bytes,
                                       int nranks, int lanes_per_rank, cecoll_program_t* out);
/* dump_program text (program.cpp:218-254). Returns the length (excluding the
 * NUL) or -1 when cap is too small. */
int64_t cecoll_program_dump(cecoll_program_t program, char* buf, size_t cap);
/* static_metrics (program.cpp:40-65): data, sync, poll, engines, doorbells. */
cecoll_status_t cecoll_program_metrics(cecoll_program_t program, int64_t out5[5]);
/* account_traffic (verifier.cpp:281-327): total read, write, link bytes;
 * per-rank arrays (nranks entries) may be NULL. */
cecoll_status_t cecoll_program_traffic(cecoll_program_t program, int64_t out3[3], int64_t* per_rank_read,
                                       int64_t* per_rank_write);
/* validate_program (program.cpp:98-205): CECOLL_SUCCESS or INVALID_ARGUMENT
 * with cecoll_last_error() naming the first violation. */
cecoll_status_t cecoll_program_validate(cecoll_program_t program, int lanes_per_rank);
void cecoll_program_free(cecoll_program_t program);
/* Inverse of dump: reads dump_program text (program.cpp:218-254) produced by
 * the reference's own compile() — or any hand-made program — so that the
 * exact reference program can be executed with cecoll_plan_create_program.
 * The program is validated (validate_program rules, buffer bounds) at plan
 * creation. */
cecoll_status_t cecoll_program_parse(const char* dump_text, cecoll_kind_t kind, int64_t chunk_bytes, int nranks,
                                     cecoll_program_t* out);

/* select_implementation (compiler.cpp:305-318), the reference's MI300X table. */
cecoll_impl_t cecoll_reference_select(cecoll_kind_t kind, int64_t chunk_bytes);
/* B200 selector: measured thresholds for nranks ranks on ndevices devices;
 * overridable with CECOLL_SM_MAX_BYTES. */
cecoll_impl_t cecoll_select(cecoll_kind_t kind, int64_t chunk_bytes, int nranks, int ndevices);
/* The selector under an SM budget (cecoll_comm_set_sm_budget): with a budget
 * and more than one device, everything above 64 KiB chunks goes to the copy
 * engines (per-peer lanes, no SMs); on one device the driver runs
 * device-local copies on SMs anyway, so the budgeted SM path is kept. */
cecoll_impl_t cecoll_select_budget(cecoll_kind_t kind, int64_t chunk_bytes, int nranks, int ndevices, int sm_budget);

/* ---------------------------------------------------------------------
 * B200 cost model (csrc/model.cpp). The reference's CostModel
 * (cost_model.hpp:14-33) prices MI300X phases; this one prices the B200
 * executor's structure — kernel boundaries, recorded-graph launches and
 * parallel branches, serial memcpy nodes, the prelaunch trigger — plus three
 * bandwidths of algorithmic HBM bytes, for n co-resident ranks on one B200.
 * cecoll_model_fit is the reference's calibrate() (calibrate.cpp:67-181):
 * seeded multiplicative log-normal hill-climb, deterministic given the seed,
 * scored by mean squared log error over the measurements plus the reference's
 * one-binary-step boundary rule on the winner grid (calibrate.cpp:44-62).
 * Times in ns, bandwidths in bytes/s. CPU only.
 * ------------------------------------------------------------------- */
typedef struct {
  double t_kernel, t_graph, t_branch, t_node, t_trigger;
  double bw_copy, bw_fan, bw_ce, bw_lanes, bw_swap;
  double l2_boost, l2_bytes; /* bandwidth factor when the buffers fit in L2 */
  double folded_max_bytes, prelaunch_gain_threshold;
  /* SM mover tables larger than one wave of 32 KiB tiles on one CTA per SM
   * (stream_min_bytes, fixed): pipeline fill and drain of the short-lived
   * CTAs (kernels.cu TmaPolicy), added once per collective */
  double t_stream, stream_min_bytes;
  /* in-place swap items whose buffers fit in L2: their writes land on lines
   * the same items just read, so they gain more than l2_boost */
  double l2_boost_swap;
} cecoll_model_t;
void cecoll_model_default(cecoll_model_t* model);
cecoll_status_t cecoll_model_predict(const cecoll_model_t* model, cecoll_kind_t kind, cecoll_impl_t impl,
                                     int64_t chunk_bytes, int nranks, double* ns);
/* winner_grid's choice at one size (sweep.cpp:186-218): the fastest of sm and
 * the reference's six implementations, the plain variant winning a near tie
 * with its prelaunch form. Returns -2 on error. */
cecoll_impl_t cecoll_model_winner(const cecoll_model_t* model, cecoll_kind_t kind, int64_t chunk_bytes, int nranks);
/* Fits *out to `count` measurements (kinds[i], impls[i], chunk_bytes[i],
 * nranks[i] -> ns[i], device time back to back). report (optional) gets the
 * per-boundary log. */
cecoll_status_t cecoll_model_fit(const int* kinds, const int* impls, const int64_t* chunk_bytes, const int* nranks,
                                 const double* ns, int count, uint64_t seed, int iterations, cecoll_model_t* out,
                                 double* residual, char* report, size_t capacity);

/* ---------------------------------------------------------------------
 * Communicators. The reference models one host process driving every GPU
 * (SPEC.md:61); cecoll_comm_init_all is that model (like
 * ncclCommInitAll). devlist may repeat a device: several ranks then share
 * one B200 ("co-resident ranks") and their transfers are intra-HBM.
 *
 * Threads: the communicators of one cecoll_comm_init_all / init_ranks call
 * (one "world"), and the plans built on them, are driven by one host thread
 * at a time, as with an NCCL communicator. Different worlds may be used from
 * different threads concurrently. cecoll_last_error and the group state
 * (cecoll_group_start/end) are per thread. Eager calls never leave a gate
 * waiting on the host, even for prelaunch_* implementations: each instance is
 * launched after its trigger is posted. An explicit plan armed ahead is
 * different. It blocks device-wide synchronisation and lazy module loads in
 * every thread of the process until it is launched or disarmed (see
 * cecoll_plan_disarm).
 * Recorded command lists and prelaunch graphs are built node by node (no
 * stream capture), so a device-wide synchronisation in another thread can
 * run at any time, including while a plan records (tests/test_thread_sync.py;
 * round 1's capture-based recording crashed in that race). Destroy a world
 * only while no other thread is issuing collectives on it.
 * ------------------------------------------------------------------- */
cecoll_status_t cecoll_comm_init_all(cecoll_comm_t* comms, int nranks, const int* devlist);
/* Multi-process: one process per GPU owning one rank. `exchange` must
 * all-gather `bytes` from every rank into `all` (rank-major); the Python
 * layer passes torch.distributed. Buffers are mapped through CUDA IPC. */
typedef int (*cecoll_exchange_fn)(void* ctx, const void* mine, size_t bytes, void* all);
cecoll_status_t cecoll_comm_init_rank(cecoll_comm_t* comm, int nranks, int rank, int device,
                                      cecoll_exchange_fn exchange, void* ctx);
/* A process owning `nlocal` consecutive ranks [first_rank, first_rank+nlocal)
 * on `device` (every process owns the same count). comms receives nlocal
 * handles. The exchange callback is kept for cecoll_register and must stay
 * valid for the communicator's lifetime. */
cecoll_status_t cecoll_comm_init_ranks(cecoll_comm_t* comms, int nranks, int first_rank, int nlocal, int device,
                                       cecoll_exchange_fn exchange, void* ctx);
/* Host-only check of the init exchange (no CUDA): validates that the
 * processes' rank ranges tile [0, nranks) and writes every rank's device. */
cecoll_status_t cecoll_exchange_check(int nranks, int first_rank, int nlocal, int device, cecoll_exchange_fn exchange,
                                      void* ctx, int32_t* out_devices);
/* Returns the world's async error when the last communicator of a world is
 * destroyed (see cecoll_comm_get_async_error); everything is released anyway. */
cecoll_status_t cecoll_comm_destroy(cecoll_comm_t comm);
/* Like ncclCommGetAsyncError. Device-side flag polls (kernels: the SM path,
 * fused flags, prelaunch bodies, flag kernels) give up after 20 s (the
 * reference's untriggered-poll deadlock, sim.cpp:227-242), record it in the
 * plan's error word and skip the data movement and signals that depended on
 * the flag (nothing is written into a buffer its owner never released).
 * Stream memory-operation waits (cuStreamWaitValue64: the copy-engine paths'
 * rdy/done polls, eager and recorded) have no timeout and no error word: a
 * peer that never signals leaves that stream waiting. Collectives are
 * asynchronous, so a kernel-side failure is reported here: *async_error = CECOLL_TIMEOUT (message in
 * cecoll_last_error) once any plan of the communicator's world has timed
 * out, else CECOLL_SUCCESS. Sticky: a world that timed out has flags out of
 * phase and must be destroyed. Reads the error words on a private stream, so
 * it never waits for armed plans or running collectives. */
cecoll_status_t cecoll_comm_get_async_error(cecoll_comm_t comm, cecoll_status_t* async_error);
cecoll_status_t cecoll_comm_info(cecoll_comm_t comm, int* rank, int* nranks, int* device);
/* Interference policy (BASELINE configs[4]: a collective beside a GEMM). Plans
 * created after this call — explicit or behind the eager calls — launch at
 * most max_ctas CTAs per mover / reduction kernel (0, the default: the
 * movers' own grids, short-lived CTAs, fastest alone), and CECOLL_IMPL_AUTO
 * selects with cecoll_select_budget. Applies to the communicator's whole
 * world; cached plans of another budget are not reused. */
cecoll_status_t cecoll_comm_set_sm_budget(cecoll_comm_t comm, int max_ctas);

/* Measured selector (csrc/tune.cpp; the reference's run_sweep + winner_grid,
 * sweep.cpp:71-218, executed on this machine). Times every applicable
 * all-gather and all-to-all implementation (sm, pcpy, b2b, bcst, hybrid,
 * pull, prelaunch_*) at 4 KiB x 4^k chunks up to max_chunk_bytes (0: 64 MiB)
 * on scratch buffers, device time per collective back to back, max over
 * ranks; picks the winner per size (the plain variant wins a near tie with
 * its prelaunch form, prelaunch_gain_threshold; the static selector's choice
 * keeps a tie within 3%) and installs the table: CECOLL_IMPL_AUTO on this
 * world then uses the nearest tuned size (log scale) while no SM budget is
 * set. comms: every local communicator of one world (all ranks of a
 * cecoll_comm_init_all world; a process's own ranks otherwise — every
 * process calls it with the same max_chunk_bytes, and the times are agreed
 * through the init exchange so every rank installs the same table).
 * streams: one per comm, or NULL for one private stream per device. Needs
 * 2 * nranks * max_chunk_bytes of device memory per rank while it runs;
 * refused while a prelaunch plan is armed. Collective, blocking. */
cecoll_status_t cecoll_tune(const cecoll_comm_t* comms, int n, int64_t max_chunk_bytes, void* const* streams);
/* The installed table as text, one "<allgather|alltoall> <chunk_bytes> <impl>"
 * line per tuned size; *len = bytes needed (with the terminating NUL). */
cecoll_status_t cecoll_tune_table(cecoll_comm_t comm, char* buf, size_t cap, size_t* len);
/* The last cecoll_tune's measurements: per kind and size, every candidate's
 * device µs per collective (-1: rejected) and the winner, one line each. */
cecoll_status_t cecoll_tune_report(cecoll_comm_t comm, char* buf, size_t cap, size_t* len);
/* Installs a table in that text form (e.g. saved from an earlier run on the
 * same node; load the same text on every process); "" clears it. */
cecoll_status_t cecoll_tune_load(cecoll_comm_t comm, const char* text);

/* Buffer registration (≙ BufferId::Input/Output being addressable on every
 * GPU, program.hpp:36). Single-process: optional no-op. Multi-process:
 * collective (each process registers its local ranks in the same order);
 * windows are symmetric — same size on every rank — and a collective's
 * buffers must sit at the same offset inside every rank's window. */
cecoll_status_t cecoll_register(cecoll_comm_t comm, void* ptr, size_t bytes);
/* Multi-process: `ptr` must be a registered window base; the window stops
 * translating and cached plans are dropped (IPC mappings stay open until
 * cecoll_comm_destroy). Explicit plans on the window must be destroyed first. */
cecoll_status_t cecoll_deregister(cecoll_comm_t comm, void* ptr);
/* Library-owned buffers (SURVEY §8(b) cecoll_mem_alloc): device memory on the
 * rank's B200, rounded up to whole 2 MiB pages and registered as a window
 * (collective in multi-process mode, like cecoll_register). cecoll_mem_free
 * deregisters and frees (waits for work still using it); buffers left
 * allocated are freed by cecoll_comm_destroy of the last communicator. */
cecoll_status_t cecoll_mem_alloc(cecoll_comm_t comm, size_t bytes, void** ptr);
cecoll_status_t cecoll_mem_free(cecoll_comm_t comm, void* ptr);

/* ---------------------------------------------------------------------
 * Collectives (the runtime the reference simulates, sim.cpp:470).
 * In single-process mode call once per rank inside group_start/group_end
 * (all ranks of the communicator must participate); a lone call outside a
 * group is only valid for multi-process communicators.
 * Ordering: the collectives and plan launches of one world share its flag
 * slots (one rdy and one done word per rank pair). Each rank's calls must
 * therefore be ordered on the device: issue them on the same stream per
 * rank, or order the streams with events. As with NCCL, two collectives of
 * one world must not be in flight on unordered streams of the same rank.
 * Every rank must also issue the world's collectives in the same order.
 * ------------------------------------------------------------------- */
cecoll_status_t cecoll_allgather(const void* send, void* recv, size_t chunk_bytes, cecoll_impl_t impl,
                                 cecoll_comm_t comm, void* stream);
/* recv may equal send only for CECOLL_IMPL_SWAP / PRELAUNCH_SWAP (in place). */
cecoll_status_t cecoll_alltoall(const void* send, void* recv, size_t chunk_bytes, cecoll_impl_t impl,
                                cecoll_comm_t comm, void* stream);
cecoll_status_t cecoll_group_start(void);
cecoll_status_t cecoll_group_end(void);

/* Reduce-scatter — the third collective (§6.1; not in
 * the reference). send holds n*count elements, recv count
 * elements: recv of rank j = op over ranks i = 0..n-1 (in rank order) of
 * send_i[j*count, (j+1)*count), accumulated in fp32 with one
 * round-to-nearest-even, so results are deterministic and bit-exact against
 * the oracle. impl: CECOLL_IMPL_SM / AUTO (one kernel reading every rank's
 * chunk), or PCPY / B2B / PRELAUNCH_PCPY / PRELAUNCH_B2B (copy-engine gather
 * into a staging buffer, then an SM reduction; single-process). */
typedef enum { CECOLL_F32 = 0, CECOLL_BF16 = 1, CECOLL_F16 = 2 } cecoll_dtype_t;
typedef enum { CECOLL_SUM = 0, CECOLL_MAX = 1, CECOLL_MIN = 2 } cecoll_redop_t;
cecoll_status_t cecoll_reduce_scatter(const void* send, void* recv, size_t count, cecoll_dtype_t dtype,
                                      cecoll_redop_t op, cecoll_impl_t impl, cecoll_comm_t comm, void* stream);
cecoll_status_t cecoll_reduce_scatter_n(const cecoll_comm_t* comms, int n, const void* const* sends,
                                        void* const* recvs, size_t count, cecoll_dtype_t dtype, cecoll_redop_t op,
                                        cecoll_impl_t impl, void* const* streams);
/* The n per-rank calls of one group in a single call (same semantics as
 * group_start; n x allgather/alltoall; group_end). streams may be NULL
 * (legacy stream for every rank). */
cecoll_status_t cecoll_collective_n(cecoll_kind_t kind, const cecoll_comm_t* comms, int n, const void* const* sends,
                                    void* const* recvs, size_t chunk_bytes, cecoll_impl_t impl,
                                    void* const* streams);

/* ---------------------------------------------------------------------
 * Explicit prelaunch plans (≙ apply_prelaunch, compiler.cpp:267-285, and the
 * producer→collective sync chain, sim.cpp:475-499). A plan binds the ranks'
 * buffers once, builds the command lists as CUDA graphs gated on a per-unit
 * device trigger word, and keeps one instance armed ahead of the trigger.
 * The trigger is stream-ordered: cecoll_plan_launch has each caller stream
 * write the word (a stream memory operation), so the armed instance starts
 * when that stream reaches the call — behind a producer kernel queued before
 * it, with no host round trip.
 * Plans of the other implementations (and the cached plans behind the eager
 * calls) are recorded too (built explicitly, node by node — never by stream
 * capture): from their second launch on, each unit's whole
 * submission — flag operations, lanes, copies, kernels — replays as one CUDA
 * graph launched on the caller stream (one host call per collective). This
 * applies when every unit of the plan has its own device and an explicit,
 * non-capturing stream (a one-unit SM plan, a single kernel, is recorded too:
 * a one-node graph launch costs the host less than the direct launch;
 * CECOLL_RECORD_SINGLE=0 opts out); otherwise, or with CECOLL_GRAPH=0,
 * commands are submitted one by one on every launch.
 * ------------------------------------------------------------------- */
cecoll_status_t cecoll_plan_create(const cecoll_comm_t* comms, int ncomms, cecoll_kind_t kind,
                                   const void* const* sends, void* const* recvs, size_t chunk_bytes,
                                   cecoll_impl_t impl, cecoll_plan_t* out);
/* A plan that executes a given command program (the reference's interpreter
 * seam: simulate(program) / verify_collective(program) → run on hardware). */
cecoll_status_t cecoll_plan_create_program(const cecoll_comm_t* comms, int ncomms, cecoll_program_t program,
                                           const void* const* sends, void* const* recvs, cecoll_plan_t* out);
/* Trigger the armed instance from each rank's stream (streams[i] for
 * comms[i]; NULL entries = the legacy default stream) and make each stream
 * wait for completion; re-arms the next instance off the critical path. */
cecoll_status_t cecoll_plan_launch(cecoll_plan_t plan, void* const* streams);
/* The two halves of cecoll_plan_launch, for callers that schedule the arming
 * themselves (SURVEY §8(b) plan_arm / plan_trigger). cecoll_plan_arm launches
 * the gated instance of every unit now (no-op for plans that are not
 * prelaunch_* and for units already armed); cecoll_plan_trigger opens the
 * armed instance exactly as cecoll_plan_launch does (arming first if needed)
 * but leaves nothing armed behind, so device-wide synchronisation returns
 * once the collective completes. */
cecoll_status_t cecoll_plan_arm(cecoll_plan_t plan);
cecoll_status_t cecoll_plan_trigger(cecoll_plan_t plan, void* const* streams);
/* Cancels the armed instance (the next launch re-arms). While a plan is
 * armed its gate kernel waits on the device, so device-wide synchronisation
 * (cudaDeviceSynchronize) only returns after disarm, destroy or a launch —
 * and so does anything that synchronises the device implicitly or loads
 * code: cudaFree, library plan creation (a cuFFT plan, measured), and under
 * CUDA's default lazy module loading the first launch of any kernel not yet
 * loaded in the process (tools/lazy_probe.py: a first torch kernel launched
 * behind an armed plan never returned; CUDA_MODULE_LOADING=EAGER cures the
 * kernel case, not the cuFFT one). Run such work before arming, disarm
 * around it, or use cecoll_plan_trigger, which leaves nothing armed. */
cecoll_status_t cecoll_plan_disarm(cecoll_plan_t plan);
/* Destroy plans before their communicators; cecoll_comm_destroy cancels any
 * plan still armed (its handle must not be used afterwards). */
cecoll_status_t cecoll_plan_destroy(cecoll_plan_t plan);
/* What the plan turned into, as one JSON object: impl, prelaunch (and whether
 * its body is a single folded kernel), graph_fallback (non-empty: the
 * prelaunch graph could not be built and the plan runs its program without
 * prelaunch), recorded / record_note (the recorded command list and why it
 * is missing), sm_budget, remote_signals ("kernel" or "memop") and per unit:
 * device, ranks, mover ("tma", "reg", "reduce", "none"), grid, ce_lanes,
 * fused_flags, start_folded, flag_writes_memop / flag_writes_kernel. Call
 * with json == NULL to get *length (excluding the NUL). */
cecoll_status_t cecoll_plan_info(cecoll_plan_t plan, char* json, size_t capacity, size_t* length);
/* The same for the cached plan behind the communicator world's latest eager
 * collective ("{}" before the first). */
cecoll_status_t cecoll_comm_last_plan_info(cecoll_comm_t comm, char* json, size_t capacity, size_t* length);

/* Hardware timelines in the reference's trace-event format (sim.cpp:523-544,
 * export_trace_json): between trace_begin and trace_end every collective of
 * the communicator's world is recorded per command with CUDA events (copies
 * are then submitted one call each). trace_end stops recording and returns
 * the JSON array ({"name": "<phase>:<command>", "ph": "B"|"E", "ts" µs,
 * "pid": rank or -1 for the host, "tid": lane, -1 for the caller stream}):
 * call it with json == NULL (or too small a capacity) to get *length; the
 * trace is kept until it has been copied out. */
cecoll_status_t cecoll_trace_begin(cecoll_comm_t comm);
cecoll_status_t cecoll_trace_end(cecoll_comm_t comm, char* json, size_t capacity, size_t* length);

/* Counters since comm creation: [0] collectives, [1] copy commands issued
 * (CE memcpys), [2] flag writes, [3] flag waits, [4] kernel launches,
 * [5] prelaunch graph launches, [6] host API calls issued, [7] replays of a
 * recorded command list (whose copies, flags and kernels count in [1]-[4]). */
cecoll_status_t cecoll_comm_counters(cecoll_comm_t comm, int64_t out8[8]);

/* ---------------------------------------------------------------------
 * EXPERIMENTAL: NVLS (switch multicast) all-gather, SURVEY §8(f)2 — the
 * multicast analogue of the reference's broadcast command
 * (compiler.cpp:166-205): each rank's chunk is read once and stored once to
 * a multicast address; the NVSwitch writes it into every GPU's window.
 * One process per GPU (cecoll_comm_init_rank). window_create is collective
 * over the processes (it uses the communicator's exchange callback) and
 * returns, in *recv, this rank's window: after cecoll_mc_allgather with
 * chunk s (<= chunk_capacity, 16-byte multiple) it holds rank i's chunk at
 * [i*s, (i+1)*s) (compiler.cpp:115-122), ordered on `stream`. Returns
 * CECOLL_UNSUPPORTED wherever the node offers no multicast objects (e.g. the
 * one-GPU development boxes). Not yet executed on hardware that accepts
 * multicast objects.
 * Reuse: the window has no ready flags (unlike the copy-engine and SM
 * paths). A call's stores land in every rank's window as soon as that rank
 * issues it, so every rank must have consumed the previous result (or copied
 * it out) before any rank starts the next call on the same window (e.g. a
 * barrier). Back-to-back calls with unchanged inputs, as in a timing loop,
 * are safe. Completion flags are per-call epochs that only grow.
 * ------------------------------------------------------------------- */
typedef struct cecoll_mc* cecoll_mc_t;
cecoll_status_t cecoll_mc_window_create(cecoll_comm_t comm, size_t chunk_capacity, cecoll_mc_t* out, void** recv);
cecoll_status_t cecoll_mc_allgather(cecoll_mc_t mc, const void* send, size_t chunk_bytes, void* stream);
const char* cecoll_mc_handle_type(cecoll_mc_t mc); /* "fabric" or "posix_fd" */
cecoll_status_t cecoll_mc_window_destroy(cecoll_mc_t mc);

#ifdef __cplusplus
}
#endif
#endif /* CECOLL_H */
