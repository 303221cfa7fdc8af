// Communicator, plan lowering and the three executors:
//   CE       pcpy / b2b / bcst / swap: per-lane streams of copy commands,
//            bracketed by batched flag memops (cuStreamBatchMemOp).
//   graph    prelaunch_*: the same lanes recorded once per unit into a CUDA
//            graph whose body sits behind a gate (conditional node), launched
//            ahead and opened by a host post (apply_prelaunch,
//            compiler.cpp:267-285).
//   SM       one sm_100a item kernel per unit moving every chunk of the unit's
//            ranks (latency regime).
#include "runtime.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <stdexcept>

namespace cecoll {

namespace {

thread_local std::string g_error;

Status fail(int code, const std::string& msg) {
  g_error = msg;
  return Status{code, msg};
}

Status cuda_fail(cudaError_t e, const char* what, int line) {
  return fail(CECOLL_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e) + " (runtime.cpp:" +
                                     std::to_string(line) + ")");
}

Status cu_fail(CUresult r, const char* what, int line) {
  const char* s = "?";
  if (driver_api()) driver_api()->GetErrorString(r, &s);
  return fail(CECOLL_CUDA_ERROR, std::string(what) + ": " + s + " (runtime.cpp:" + std::to_string(line) + ")");
}

#define CUDA_TRY(expr)                                      \
  do {                                                      \
    cudaError_t e_ = (expr);                                \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr, __LINE__); \
  } while (0)

#define CU_TRY(expr)                                       \
  do {                                                     \
    CUresult r_ = (expr);                                  \
    if (r_ != CUDA_SUCCESS) return cu_fail(r_, #expr, __LINE__); \
  } while (0)

#define STATUS_TRY(expr)         \
  do {                           \
    Status s_ = (expr);          \
    if (!s_.ok()) return s_;     \
  } while (0)

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev_);
    if (dev >= 0 && dev != prev_) cudaSetDevice(dev);
  }
  ~DeviceGuard() { cudaSetDevice(prev_); }

 private:
  int prev_ = 0;
};

CUstreamBatchMemOpParams op_write(uint64_t* addr, uint64_t v) {
  CUstreamBatchMemOpParams op;
  std::memset(&op, 0, sizeof(op));
  op.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
  op.writeValue.address = reinterpret_cast<CUdeviceptr>(addr);
  op.writeValue.value64 = v;
  op.writeValue.flags = 0;  // with the default memory barrier: prior copies are visible first
  return op;
}

CUstreamBatchMemOpParams op_wait(uint64_t* addr, uint64_t v) {
  CUstreamBatchMemOpParams op;
  std::memset(&op, 0, sizeof(op));
  op.waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
  op.waitValue.address = reinterpret_cast<CUdeviceptr>(addr);
  op.waitValue.value64 = v;
  op.waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
  return op;
}

// Poll + reset of one slot (the reset keeps graph replays value-constant).
void add_poll(MemOps& ops, uint64_t* addr) {
  ops.push_back(op_wait(addr, 1));
  ops.push_back(op_write(addr, 0));
}

Status submit(World* w, cudaStream_t s, const MemOps& ops) {
  const DriverApi* d = driver_api();
  size_t i = 0;
  while (i < ops.size()) {
    const unsigned count = static_cast<unsigned>(std::min<size_t>(255, ops.size() - i));
    CU_TRY(d->StreamBatchMemOp(reinterpret_cast<CUstream>(s), count,
                               const_cast<CUstreamBatchMemOpParams*>(ops.data() + i), 0));
    for (unsigned k = 0; k < count; ++k) {
      if (ops[i + k].operation == CU_STREAM_MEM_OP_WRITE_VALUE_64) ++w->counters[2];
      else ++w->counters[3];
    }
    ++w->counters[6];
    i += count;
  }
  return {};
}

Status issue_copies(World* w, const std::vector<Copy>& copies, cudaStream_t s, bool allow_batch) {
  const DriverApi* d = driver_api();
  // cuMemcpyBatchAsync rejects the legacy NULL stream.
  const bool legacy = s == nullptr || s == cudaStreamLegacy;
  if (copies.size() > 1 && allow_batch && d->has_batch_memcpy && !legacy) {
    std::vector<CUdeviceptr> dst, src;
    std::vector<size_t> sz;
    for (const Copy& c : copies) {
      dst.push_back(reinterpret_cast<CUdeviceptr>(c.dst));
      src.push_back(reinterpret_cast<CUdeviceptr>(c.src));
      sz.push_back(static_cast<size_t>(c.bytes));
    }
    CUmemcpyAttributes attr;
    std::memset(&attr, 0, sizeof(attr));
    attr.srcAccessOrder = CU_MEMCPY_SRC_ACCESS_ORDER_STREAM;
    attr.flags = CU_MEMCPY_FLAG_PREFER_OVERLAP_WITH_COMPUTE;
    size_t idx = 0, fail_idx = 0;
    CU_TRY(d->MemcpyBatchAsync(dst.data(), src.data(), sz.data(), copies.size(), &attr, &idx, 1, &fail_idx,
                               reinterpret_cast<CUstream>(s)));
    w->counters[1] += static_cast<int64_t>(copies.size());
    ++w->counters[6];
    return {};
  }
  for (const Copy& c : copies) {
    CUDA_TRY(cudaMemcpyAsync(c.dst, c.src, static_cast<size_t>(c.bytes), cudaMemcpyDefault, s));
    ++w->counters[1];
    ++w->counters[6];
  }
  return {};
}

Status make_rank(World* w, int rank, int device, uint64_t* page = nullptr) {
  DeviceGuard g(device);
  auto rs = std::make_unique<RankState>();
  rs->rank = rank;
  rs->device = device;
  CUDA_TRY(cudaEventCreateWithFlags(&rs->start, cudaEventDisableTiming));
  if (page) {
    rs->flags = page;
    rs->owns_flags = false;
  } else {
    CUDA_TRY(cudaMalloc(&rs->flags, kFlagBytes));
    CUDA_TRY(cudaMemset(rs->flags, 0, kFlagBytes));
    CUDA_TRY(cudaDeviceSynchronize());
  }
  w->flag_page[rank] = rs->flags;
  w->local[rank] = std::move(rs);
  return {};
}

Status ensure_lanes(RankState* rs, int n) {
  DeviceGuard g(rs->device);
  while (static_cast<int>(rs->lanes.size()) < n) {
    cudaStream_t s;
    cudaEvent_t e;
    CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    rs->lanes.push_back(s);
    rs->lane_done.push_back(e);
  }
  return {};
}

int count_devices(const std::vector<int>& dev) {
  std::set<int> s(dev.begin(), dev.end());
  return static_cast<int>(s.size());
}

}  // namespace

void set_error(const std::string& msg) { g_error = msg; }
const char* last_error() { return g_error.c_str(); }

Status world_init_all(int nranks, const int* devlist, World** out) {
  if (!driver_api()) return fail(CECOLL_NO_DEVICE, "no CUDA driver / device");
  if (nranks < 1 || nranks > kMaxRanks)
    return fail(CECOLL_INVALID_ARGUMENT, "nranks must be in [1, " + std::to_string(kMaxRanks) + "]");
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  for (int r = 0; r < nranks; ++r)
    if (devlist[r] < 0 || devlist[r] >= ndev)
      return fail(CECOLL_INVALID_ARGUMENT, "device " + std::to_string(devlist[r]) + " out of range");
  auto w = std::make_unique<World>();
  w->nranks = nranks;
  w->device.assign(devlist, devlist + nranks);
  w->flag_page.assign(nranks, nullptr);
  w->local.resize(nranks);
  w->ndevices = count_devices(w->device);
  // Peer access between every pair of distinct devices (NVLink / NVSwitch).
  std::set<int> devs(w->device.begin(), w->device.end());
  for (int a : devs)
    for (int b : devs) {
      if (a == b) continue;
      int can = 0;
      CUDA_TRY(cudaDeviceCanAccessPeer(&can, a, b));
      if (!can) return fail(CECOLL_UNSUPPORTED, "no peer access between devices");
      DeviceGuard g(a);
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "EnablePeerAccess", __LINE__);
      cudaGetLastError();
    }
  for (int r = 0; r < nranks; ++r) STATUS_TRY(make_rank(w.get(), r, w->device[r]));
  w->live_comms = nranks;
  w->first_local = 0;
  w->nlocal = nranks;
  *out = w.release();
  return {};
}

namespace {

// One blob per process in the init exchange.
struct ProcInfo {
  int32_t first;   // first global rank owned by the process
  int32_t nlocal;  // ranks owned (consecutive)
  int32_t device;
  int32_t pid;
  cudaIpcMemHandle_t flags;  // nlocal flag pages, kFlagBytes apart
};

// One blob per process in a registration round.
struct RegInfo {
  int32_t rank;
  int32_t pad;
  uint64_t offset;  // of the window inside its allocation
  uint64_t bytes;
  cudaIpcMemHandle_t handle;  // of the allocation
};

Status open_ipc(World* w, const cudaIpcMemHandle_t& h, void** out) {
  std::string key(reinterpret_cast<const char*>(&h), sizeof(h));
  auto it = w->ipc_by_handle.find(key);
  if (it != w->ipc_by_handle.end()) {
    *out = it->second;
    return {};
  }
  CUDA_TRY(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  w->ipc_opened.push_back(*out);
  w->ipc_by_handle[key] = *out;
  return {};
}

}  // namespace

Status gather_procs(int nranks, int first, int nlocal, int device, const cudaIpcMemHandle_t* flags,
                    cecoll_exchange_fn fn, void* ctx, std::vector<ProcInfoView>* out) {
  if (nranks < 1 || nranks > kMaxRanks || nlocal < 1 || first < 0 || first + nlocal > nranks || !fn)
    return fail(CECOLL_INVALID_ARGUMENT, "bad rank range / exchange");
  if (nranks % nlocal != 0)
    return fail(CECOLL_INVALID_ARGUMENT, "every process must own the same number of ranks");
  const int procs = nranks / nlocal;
  ProcInfo mine;
  std::memset(&mine, 0, sizeof(mine));
  mine.first = first;
  mine.nlocal = nlocal;
  mine.device = device;
  if (flags) mine.flags = *flags;
  std::vector<ProcInfo> all(procs);
  if (fn(ctx, &mine, sizeof(ProcInfo), all.data()) != 0) return fail(CECOLL_INTERNAL, "exchange failed");
  std::vector<int> owner(nranks, -1);
  out->clear();
  for (int p = 0; p < procs; ++p) {
    const ProcInfo& pi = all[p];
    if (pi.nlocal != nlocal || pi.first < 0 || pi.first + pi.nlocal > nranks)
      return fail(CECOLL_INVALID_ARGUMENT, "inconsistent rank ranges across processes");
    for (int k = 0; k < pi.nlocal; ++k) {
      if (owner[pi.first + k] >= 0) return fail(CECOLL_INVALID_ARGUMENT, "a rank is owned by two processes");
      owner[pi.first + k] = p;
    }
    ProcInfoView v;
    v.first = pi.first;
    v.nlocal = pi.nlocal;
    v.device = pi.device;
    std::memcpy(&v.flags, &pi.flags, sizeof(v.flags));
    out->push_back(v);
  }
  for (int r = 0; r < nranks; ++r)
    if (owner[r] < 0) return fail(CECOLL_INVALID_ARGUMENT, "rank " + std::to_string(r) + " is owned by no process");
  return {};
}

Status world_init_ranks(int nranks, int first, int nlocal, int device, cecoll_exchange_fn fn, void* ctx,
                        World** out) {
  if (!driver_api()) return fail(CECOLL_NO_DEVICE, "no CUDA driver / device");
  if (nranks < 1 || nranks > kMaxRanks || nlocal < 1 || first < 0 || first + nlocal > nranks || !fn)
    return fail(CECOLL_INVALID_ARGUMENT, "bad rank range / exchange");
  DeviceGuard g(device);
  auto w = std::make_unique<World>();
  w->nranks = nranks;
  w->multiprocess = true;
  w->first_local = first;
  w->nlocal = nlocal;
  w->device.assign(nranks, -1);
  w->flag_page.assign(nranks, nullptr);
  w->local.resize(nranks);
  // One allocation holds the flag pages of every local rank (one IPC handle).
  void* block = nullptr;
  CUDA_TRY(cudaMalloc(&block, kFlagBytes * nlocal));
  CUDA_TRY(cudaMemset(block, 0, kFlagBytes * nlocal));
  CUDA_TRY(cudaDeviceSynchronize());
  w->flag_block = block;
  for (int k = 0; k < nlocal; ++k)
    STATUS_TRY(make_rank(w.get(), first + k, device,
                         reinterpret_cast<uint64_t*>(static_cast<char*>(block) + k * kFlagBytes)));
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, block));
  std::vector<ProcInfoView> procs;
  STATUS_TRY(gather_procs(nranks, first, nlocal, device, &h, fn, ctx, &procs));
  for (const ProcInfoView& pv : procs) {
    char* base = nullptr;
    if (pv.first != first) {
      void* opened = nullptr;
      STATUS_TRY(open_ipc(w.get(), pv.flags, &opened));
      base = static_cast<char*>(opened);
    }
    for (int k = 0; k < pv.nlocal; ++k) {
      const int r = pv.first + k;
      w->device[r] = pv.device;
      if (pv.first != first) w->flag_page[r] = reinterpret_cast<uint64_t*>(base + k * kFlagBytes);
    }
  }
  w->ndevices = count_devices(w->device);
  w->live_comms = nlocal;
  w->reg_rounds.assign(nlocal, 0);
  w->exchange = fn;
  w->exchange_ctx = ctx;
  *out = w.release();
  return {};
}

// Registration is collective: each process registers its local ranks in the
// same order; round i of local index k fills window i for ranks first_p + k
// of every process p. Windows are symmetric (same size on every rank) and a
// collective's buffers must sit at the same offset in every rank's window.
Status world_register(World* w, int rank, void* ptr, size_t bytes, cecoll_exchange_fn fn, void* ctx) {
  if (!w->multiprocess) return {};  // single process: UVA pointers are used as is
  if (!fn) return fail(CECOLL_INVALID_ARGUMENT, "multi-process registration needs the exchange callback");
  DeviceGuard g(w->device[rank]);
  const int k = rank - w->first_local;
  const int round = w->reg_rounds[k]++;
  if (static_cast<int>(w->windows.size()) <= round) {
    Window win;
    win.bytes = bytes;
    win.rank_base.assign(w->nranks, nullptr);
    w->windows.push_back(win);
  }
  Window& win = w->windows[round];
  if (win.bytes != bytes)
    return fail(CECOLL_INVALID_ARGUMENT, "cecoll_register: windows must be symmetric (same size on every rank)");
  CUdeviceptr base = 0;
  size_t size = 0;
  CU_TRY(driver_api()->MemGetAddressRange(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)));
  RegInfo mine;
  std::memset(&mine, 0, sizeof(mine));
  mine.rank = rank;
  mine.offset = reinterpret_cast<uint64_t>(ptr) - base;
  mine.bytes = bytes;
  CUDA_TRY(cudaIpcGetMemHandle(&mine.handle, reinterpret_cast<void*>(base)));
  const int procs = w->nranks / w->nlocal;
  std::vector<RegInfo> all(procs);
  if (fn(ctx, &mine, sizeof(RegInfo), all.data()) != 0) return fail(CECOLL_INTERNAL, "exchange failed");
  for (const RegInfo& ri : all) {
    if (ri.bytes != bytes)
      return fail(CECOLL_INVALID_ARGUMENT, "cecoll_register: windows must be symmetric (same size on every rank)");
    if (ri.rank < 0 || ri.rank >= w->nranks) return fail(CECOLL_INVALID_ARGUMENT, "bad rank in registration");
    if (ri.rank == rank) {
      win.rank_base[ri.rank] = static_cast<char*>(ptr);
      continue;
    }
    void* opened = nullptr;
    STATUS_TRY(open_ipc(w, ri.handle, &opened));
    win.rank_base[ri.rank] = static_cast<char*>(opened) + ri.offset;
  }
  return {};
}

Status world_deregister(World* w, void* ptr) {
  (void)ptr;
  // Windows stay mapped until the communicator is destroyed (mappings are
  // shared by every plan built on them).
  return w->multiprocess ? Status{} : Status{};
}

void world_release(World* w) {
  for (auto& p : w->plans) plan_destroy(w, p.get());
  w->plans.clear();
  // Armed explicit plans would keep their gate kernels waiting (and the
  // device synchronisation below would never return): cancel them. Their
  // cecoll_plan handles must not be used afterwards.
  for (Plan* p : w->explicit_plans) plan_destroy(w, p);
  w->explicit_plans.clear();
  for (auto& rs : w->local) {
    if (!rs) continue;
    DeviceGuard g(rs->device);
    cudaDeviceSynchronize();
    for (auto s : rs->lanes) cudaStreamDestroy(s);
    for (auto e : rs->lane_done) cudaEventDestroy(e);
    if (rs->start) cudaEventDestroy(rs->start);
    if (rs->flags && rs->owns_flags) cudaFree(rs->flags);
  }
  for (void* p : w->ipc_opened) cudaIpcCloseMemHandle(p);
  if (w->flag_block) cudaFree(w->flag_block);
  delete w;
}

// ---------------------------------------------------------------------------
// Plan lowering
// ---------------------------------------------------------------------------

namespace {

struct Addressing {
  std::vector<const char*> send;  // per rank, usable in this process
  std::vector<char*> recv;
};

// Address of `mine` (a pointer of local rank `me`) in rank `target`'s
// registered window at the same offset.
char* translate(World* w, int me, int target, const void* mine, bool* ok) {
  const char* p = static_cast<const char*>(mine);
  for (const Window& win : w->windows) {
    const char* b = win.rank_base[me];
    if (b && p >= b && p < b + win.bytes && win.rank_base[target]) return win.rank_base[target] + (p - b);
  }
  *ok = false;
  return nullptr;
}

uint64_t* slot(World* w, int rank, int index) { return w->flag_page[rank] + index; }

Item make_item(ItemKind kind, const char* src, char* dst, char* dst2, int64_t bytes) {
  Item it;
  std::memset(&it, 0, sizeof(it));
  it.kind = kind;
  it.src = src;
  it.dst = dst;
  it.dst2 = dst2;
  it.bytes = bytes;
  return it;
}

// A host-side item plus, for kItemFan, its destination list. `remote`: some
// destination is another device's memory (NVLink); such tables use the
// register mover (plain st.global to peer-mapped addresses) rather than TMA
// bulk stores.
struct HostItem {
  Item item;
  std::vector<char*> fan;
  bool remote = false;
};

// Chooses the mover (TMA for aligned copy/fan tables unless
// CECOLL_MOVER=reg), numbers the tiles, uploads the fan lists and the table.
Status upload_items(Plan* p, int device, std::vector<HostItem>& host, ItemTable* out) {
  if (host.empty()) return {};
  if (host.size() > static_cast<size_t>(kMaxItemsSmem))
    return fail(CECOLL_INVALID_ARGUMENT, "too many chunk transfers for one launch");
  DeviceGuard g(device);
  bool tma = true;
  int kinds = 0;
  size_t nfan = 0;
  for (const HostItem& h : host) {
    const Item& it = h.item;
    kinds |= 1 << it.kind;
    uintptr_t a = reinterpret_cast<uintptr_t>(it.src) | reinterpret_cast<uintptr_t>(it.dst);
    for (char* f : h.fan) a |= reinterpret_cast<uintptr_t>(f);
    tma &= (it.kind == kItemCopy || it.kind == kItemFan) && (a & 15) == 0 && (it.bytes & 15) == 0 && !h.remote;
    nfan += h.fan.size();
  }
  const char* env = std::getenv("CECOLL_MOVER");
  if (env && std::string(env) == "reg") tma = false;
  out->mover = tma ? Mover::Tma : Mover::Reg;
  out->kinds = kinds;
  char** fan_dev = nullptr;
  if (nfan) {
    std::vector<char*> flat;
    for (const HostItem& h : host) flat.insert(flat.end(), h.fan.begin(), h.fan.end());
    void* d = nullptr;
    CUDA_TRY(cudaMalloc(&d, sizeof(char*) * flat.size()));
    CUDA_TRY(cudaMemcpy(d, flat.data(), sizeof(char*) * flat.size(), cudaMemcpyHostToDevice));
    p->dev_allocs.push_back(d);
    p->dev_alloc_device.push_back(device);
    fan_dev = static_cast<char**>(d);
  }
  std::vector<Item> items;
  int64_t tiles = 0;
  size_t fan_at = 0;
  for (HostItem& h : host) {
    Item it = h.item;
    it.first_tile = static_cast<int32_t>(tiles);
    tiles += tiles_for(it.bytes, out->mover);
    if (it.kind == kItemFan) {
      it.fan = fan_dev + fan_at;
      it.nfan = static_cast<int32_t>(h.fan.size());
      it.dst = h.fan[0];
      fan_at += h.fan.size();
    }
    items.push_back(it);
  }
  if (tiles > INT32_MAX) return fail(CECOLL_INVALID_ARGUMENT, "collective too large for one launch");
  void* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, sizeof(Item) * items.size()));
  CUDA_TRY(cudaMemcpy(d, items.data(), sizeof(Item) * items.size(), cudaMemcpyHostToDevice));
  p->dev_allocs.push_back(d);
  p->dev_alloc_device.push_back(device);
  out->items = static_cast<Item*>(d);
  out->nitems = static_cast<int>(items.size());
  out->ntiles = static_cast<int>(tiles);
  return {};
}

Status upload_ptrs(Plan* p, int device, const std::vector<uint64_t*>& ptrs, uint64_t*** out) {
  *out = nullptr;
  if (ptrs.empty()) return {};
  DeviceGuard g(device);
  void* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, sizeof(uint64_t*) * ptrs.size()));
  CUDA_TRY(cudaMemcpy(d, ptrs.data(), sizeof(uint64_t*) * ptrs.size(), cudaMemcpyHostToDevice));
  p->dev_allocs.push_back(d);
  p->dev_alloc_device.push_back(device);
  *out = static_cast<uint64_t**>(d);
  return {};
}

// Device holding the flag page that contains addr (-1 if none).
int flag_device(World* w, const uint64_t* addr) {
  for (int r = 0; r < w->nranks; ++r) {
    const uint64_t* b = w->flag_page[r];
    if (b && addr >= b && addr < b + kFlagBytes / sizeof(uint64_t)) return w->device[r];
  }
  return -1;
}

// Moves the writes in `ops` that target another device's flag page into
// `remote`: those are issued by a signal kernel (st.release.sys to the
// peer-mapped page) rather than a stream memory operation, the portable way
// to signal across NVLink. Same-device pages (also across processes) keep
// the memop.
void split_writes(World* w, int device, MemOps& ops, std::vector<uint64_t*>& remote) {
  MemOps keep;
  for (const auto& op : ops) {
    if (op.operation == CU_STREAM_MEM_OP_WRITE_VALUE_64) {
      uint64_t* a = reinterpret_cast<uint64_t*>(op.writeValue.address);
      const int d = flag_device(w, a);
      if (d >= 0 && d != device) {
        remote.push_back(a);
        continue;
      }
    }
    keep.push_back(op);
  }
  ops.swap(keep);
}

Status split_remote(World* w, Plan* p) {
  for (Unit& u : p->units) {
    split_writes(w, u.device, u.start, u.start_remote);
    split_writes(w, u.device, u.sm_post, u.sm_post_remote);
    STATUS_TRY(upload_ptrs(p, u.device, u.start_remote, &u.start_remote_tab));
    STATUS_TRY(upload_ptrs(p, u.device, u.sm_post_remote, &u.sm_post_remote_tab));
  }
  for (LaneExec& l : p->lanes) {
    const int dev = w->device[l.rank];
    split_writes(w, dev, l.post, l.post_remote);
    STATUS_TRY(upload_ptrs(p, dev, l.post_remote, &l.post_remote_tab));
  }
  return {};
}

// Stream memops, then the signal kernel for other-device flags.
Status signal_remote(World* w, uint64_t** tab, size_t n, cudaStream_t s) {
  if (!n) return {};
  CUDA_TRY(launch_signal(tab, static_cast<int>(n), s));
  ++w->counters[4];
  ++w->counters[6];
  w->counters[2] += static_cast<int64_t>(n);
  return {};
}

}  // namespace

Status build_graph(World* w, Plan* p, Unit& u);

Status plan_create(World* w, Kind kind, Impl impl, int64_t s, const std::vector<CallArgs>& args, Plan** out,
                   const Program* given) {
  const int n = w->nranks;
  if (s <= 0) return fail(CECOLL_INVALID_ARGUMENT, "collective: chunk size must be positive");
  auto plan = std::make_unique<Plan>();
  Plan* p = plan.get();
  p->kind = kind;
  p->chunk = s;
  for (const CallArgs& a : args) {
    p->key_rank.push_back(a.rank);
    p->key_send.push_back(a.send);
    p->key_recv.push_back(a.recv);
    p->key_stream.push_back(a.stream);
  }
  if (given) {
    if (given->spec.kind != kind || given->spec.chunk != s || given->spec.nranks != n)
      return fail(CECOLL_INVALID_ARGUMENT, "program spec does not match the communicator / call");
    const std::string v = validate(*given, kMaxLanes);
    if (!v.empty()) return fail(CECOLL_INVALID_ARGUMENT, "program rejected: " + v);
    impl = given->impl;
  }
  if (impl == Impl::Auto) {
    bool in_place = kind == Kind::AllToAll;
    for (const CallArgs& a : args) in_place &= a.send == a.recv;
    impl = in_place ? Impl::Swap : select(kind, s, n, w->ndevices);
  }
  if (impl != Impl::Sm && !valid_for(impl, kind))
    return fail(CECOLL_UNSUPPORTED, std::string(impl_name(impl)) + " does not apply to " +
                                         (kind == Kind::AllGather ? "allgather" : "alltoall"));
  const bool in_place_impl = base_of(impl) == Impl::Swap;
  p->impl = impl;
  p->sm = impl == Impl::Sm;
  p->prelaunch = is_prelaunched(impl);

  // Addresses of every rank's buffers as usable from this process.
  Addressing ad;
  ad.send.assign(n, nullptr);
  ad.recv.assign(n, nullptr);
  std::vector<bool> have(n, false);
  for (const CallArgs& a : args) {
    if (a.rank < 0 || a.rank >= n || !w->local[a.rank]) return fail(CECOLL_INVALID_ARGUMENT, "rank not local");
    if (have[a.rank]) return fail(CECOLL_INVALID_ARGUMENT, "rank appears twice in one group");
    have[a.rank] = true;
    ad.send[a.rank] = static_cast<const char*>(a.send);
    ad.recv[a.rank] = static_cast<char*>(a.recv);
  }
  if (!w->multiprocess) {
    for (int r = 0; r < n; ++r)
      if (!have[r])
        return fail(CECOLL_INVALID_ARGUMENT,
                    "single-process communicator: every rank must take part (use cecoll_group_start/end)");
  } else {
    if (static_cast<int>(args.size()) != w->nlocal)
      return fail(CECOLL_INVALID_ARGUMENT, "multi-process: every local rank must take part (group calls)");
    const CallArgs& a = args[0];
    for (int r = 0; r < n; ++r) {
      if (have[r]) continue;
      bool ok = true;
      ad.send[r] = translate(w, a.rank, r, a.send, &ok);
      ad.recv[r] = translate(w, a.rank, r, a.recv, &ok);
      if (!ok) return fail(CECOLL_NOT_REGISTERED, "send/recv must lie in a window registered with cecoll_register");
    }
  }
  for (const CallArgs& a : args) {
    const bool aliased = a.send == a.recv;
    if (kind == Kind::AllToAll && aliased && !in_place_impl)
      return fail(CECOLL_INVALID_ARGUMENT, "alltoall in place requires the swap implementation");
  }

  // Units: local ranks sharing (device, stream).
  std::vector<int> unit_of(n, -1);
  for (const CallArgs& a : args) {
    int found = -1;
    for (size_t u = 0; u < p->units.size(); ++u)
      if (p->units[u].device == w->device[a.rank] && p->units[u].stream == a.stream) found = static_cast<int>(u);
    if (found < 0) {
      Unit u;
      u.device = w->device[a.rank];
      u.stream = a.stream;
      p->units.push_back(u);
      found = static_cast<int>(p->units.size()) - 1;
    }
    p->units[found].ranks.push_back(a.rank);
    unit_of[a.rank] = found;
  }
  for (Unit& u : p->units) std::sort(u.ranks.begin(), u.ranks.end());
  auto same_unit = [&](int a, int b) { return unit_of[a] >= 0 && unit_of[a] == unit_of[b]; };

  // Buffer of a program region. In-place programs (swap) address the
  // in-place buffer as Input (compiler.cpp:119-122); it is `recv`.
  auto base = [&](int rank, Buf b) -> char* {
    if (in_place_impl || b == Buf::Output) return ad.recv[rank];
    return const_cast<char*>(ad.send[rank]);
  };
  auto addr = [&](const Region& r) { return base(r.rank, r.buf) + r.off; };

  // Edges writer -> destination and the flag operations they imply.
  std::vector<std::pair<int, int>> edges;
  if (p->sm) {
    for (int r = 0; r < n; ++r)
      for (int d = 1; d < n; ++d) edges.push_back({r, (r + d) % n});
  } else {
    if (n < 2) return fail(CECOLL_INVALID_ARGUMENT, "collective: gpu_count must be >= 2");
    Spec spec;
    spec.kind = kind;
    spec.chunk = s;
    spec.nranks = n;
    try {
      p->program = given ? *given : compile(impl, spec, kMaxLanes);
    } catch (const std::invalid_argument& e) {
      return fail(CECOLL_INVALID_ARGUMENT, e.what());
    }
    for (const Lane& l : p->program.lanes)
      for (const Command& c : l.cmds) {
        if (!c.moves_data()) continue;
        const Region* ds[3] = {&c.dst, c.op == Op::Broadcast ? &c.dst2 : nullptr, nullptr};
        if (c.op == Op::Swap) ds[0] = &c.peer;
        for (const Region* d : ds)
          if (d && d->rank != l.rank) edges.push_back({l.rank, d->rank});
      }
  }
  for (auto [r, j] : edges) {
    if (same_unit(r, j)) continue;
    if (unit_of[j] >= 0) {  // j is local: it announces readiness and waits for r's data
      Unit& u = p->units[unit_of[j]];
      u.start.push_back(op_write(slot(w, r, kSlotRdy + j), 1));
      add_poll(u.finish, slot(w, j, kSlotDone + r));
    }
    if (unit_of[r] >= 0 && p->sm) {  // r is local: wait for j, then signal it
      Unit& u = p->units[unit_of[r]];
      add_poll(u.sm_pre, slot(w, r, kSlotRdy + j));
      u.sm_post.push_back(op_write(slot(w, j, kSlotDone + r), 1));
    }
  }

  // Local-slot placement (verifier.cpp:40-44) and the swap pre-copy.
  for (Unit& u : p->units)
    for (int r : u.ranks) {
      if (in_place_impl) {
        if (ad.send[r] != ad.recv[r])
          u.precopy.push_back({ad.recv[r], ad.send[r], s * n});
        continue;
      }
      const char* src = ad.send[r] + (kind == Kind::AllGather ? 0 : r * s);
      char* dst = ad.recv[r] + r * s;
      if (src != dst) u.placement.push_back({dst, src, s});
    }

  if (p->sm) {
    for (Unit& u : p->units) {
      std::vector<HostItem> items;
      for (int r : u.ranks) {
        if (kind == Kind::AllGather) {
          // One read of the source chunk, one write per rank's slot r (local
          // slot first, then the pcpy rotation): n*s + n*n*s bytes instead
          // of 2*n*n*s for n separate copies.
          HostItem h{make_item(kItemFan, ad.send[r], nullptr, nullptr, s), {}};
          for (int d = 0; d < n; ++d) {
            char* dst = ad.recv[(r + d) % n] + r * s;
            if (dst != ad.send[r]) h.fan.push_back(dst);
            h.remote |= w->device[(r + d) % n] != u.device;
          }
          if (h.fan.size() == 1) h.item = make_item(kItemCopy, ad.send[r], h.fan[0], nullptr, s), h.fan.clear();
          if (!h.fan.empty() || h.item.kind == kItemCopy) items.push_back(h);
          continue;
        }
        for (const Copy& c : u.placement)
          if (c.dst == ad.recv[r] + r * s) items.push_back({make_item(kItemCopy, c.src, c.dst, nullptr, c.bytes), {}});
        for (int d = 1; d < n; ++d) {
          const int j = (r + d) % n;
          items.push_back({make_item(kItemCopy, ad.send[r] + j * s, ad.recv[j] + r * s, nullptr, s), {},
                           w->device[j] != u.device});
        }
      }
      u.placement.clear();
      STATUS_TRY(upload_items(p, u.device, items, &u.table));
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->units[0].device);
    p->sms = sms;
  } else {
    // A recorded (prelaunch) graph moves its same-device chunks with one item
    // kernel per unit instead of one memcpy node per copy: the driver runs
    // same-device memcpy on SMs anyway (profiles/ce_probe2_r01.txt) and every
    // graph node costs launch latency. Cross-device copies stay memcpy nodes
    // (copy engines over NVLink). CECOLL_GRAPH_MEMCPY=1 keeps every copy a
    // memcpy node.
    const char* gm = std::getenv("CECOLL_GRAPH_MEMCPY");
    const bool merge = p->prelaunch && !(gm && std::string(gm) == "1");
    std::vector<std::vector<HostItem>> unit_items(p->units.size());
    if (merge)
      for (size_t ui = 0; ui < p->units.size(); ++ui) {
        for (const Copy& c : p->units[ui].placement)
          unit_items[ui].push_back({make_item(kItemCopy, c.src, c.dst, nullptr, c.bytes), {}});
        p->units[ui].placement.clear();
      }
    // Lanes of the command program owned by local ranks.
    for (const Lane& l : p->program.lanes) {
      if (unit_of[l.rank] < 0) continue;
      LaneExec le;
      le.rank = l.rank;
      le.lane = l.index;
      std::set<int> dests;
      std::vector<HostItem> items;
      const int dev = w->device[l.rank];
      for (const Command& c : l.cmds) {
        const bool local_cmd = w->device[c.src.rank] == dev && w->device[c.dst.rank] == dev &&
                               (c.op != Op::Broadcast || w->device[c.dst2.rank] == dev) &&
                               (c.op != Op::Swap || w->device[c.peer.rank] == dev);
        std::vector<HostItem>& sink = merge && local_cmd ? unit_items[unit_of[l.rank]] : items;
        switch (c.op) {
          case Op::Copy:
            if (merge && local_cmd) sink.push_back({make_item(kItemCopy, addr(c.src), addr(c.dst), nullptr, c.size), {}});
            else le.copies.push_back({addr(c.dst), addr(c.src), c.size});
            dests.insert(c.dst.rank);
            break;
          case Op::Broadcast:
            sink.push_back({make_item(kItemBcst, addr(c.src), addr(c.dst), addr(c.dst2), c.size), {}, !local_cmd});
            dests.insert(c.dst.rank);
            dests.insert(c.dst2.rank);
            break;
          case Op::Swap:
            sink.push_back({make_item(kItemSwap, addr(c.peer), addr(c.src), nullptr, c.size), {}, !local_cmd});
            dests.insert(c.peer.rank);
            break;
          default: break;  // Signal / Poll: realised by the flag operations below
        }
      }
      dests.erase(l.rank);
      for (int j : dests) {
        if (same_unit(l.rank, j)) continue;
        add_poll(le.pre, slot(w, l.rank, kSlotRdy + j));
        le.post.push_back(op_write(slot(w, j, kSlotDone + l.rank), 1));
      }
      STATUS_TRY(upload_items(p, w->device[l.rank], items, &le.table));
      STATUS_TRY(ensure_lanes(w->local[l.rank].get(), l.index + 1));
      p->lanes.push_back(std::move(le));
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->units[0].device);
    p->sms = sms;
    for (size_t ui = 0; ui < p->units.size(); ++ui)
      STATUS_TRY(upload_items(p, p->units[ui].device, unit_items[ui], &p->units[ui].table));
  }
  STATUS_TRY(split_remote(w, p));
  if (p->prelaunch)
    for (Unit& u : p->units) {
      const Status gs = build_graph(w, p, u);
      if (gs.ok()) continue;
      if (given) return gs;  // a given program keeps its polls: no eager form
      // A graph this driver cannot record or instantiate (e.g. a copy-engine
      // memcpy node between devices inside a conditional body): run the same
      // command program without prelaunch rather than fail the collective.
      std::string why = gs.msg;
      plan_destroy(w, p);
      Plan* eager = nullptr;
      STATUS_TRY(plan_create(w, kind, base_of(impl), s, args, &eager, given));
      eager->impl = impl;
      eager->graph_fallback = why;
      *out = eager;
      return {};
    }
  *out = plan.release();
  return {};
}

namespace {

// Uploads a reduction table: the items plus one flat array of source pointers.
Status upload_red(Plan* p, int device, std::vector<RedItem>& items, const std::vector<std::vector<const char*>>& srcs,
                  int dtype, int op, RedTable* out) {
  if (items.empty()) return {};
  if (items.size() > static_cast<size_t>(kMaxItemsSmem))
    return fail(CECOLL_INVALID_ARGUMENT, "too many reductions for one launch");
  DeviceGuard g(device);
  std::vector<const char*> flat;
  for (const auto& v : srcs) flat.insert(flat.end(), v.begin(), v.end());
  void* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, sizeof(char*) * flat.size()));
  CUDA_TRY(cudaMemcpy(d, flat.data(), sizeof(char*) * flat.size(), cudaMemcpyHostToDevice));
  p->dev_allocs.push_back(d);
  p->dev_alloc_device.push_back(device);
  int64_t tiles = 0;
  size_t at = 0;
  for (size_t i = 0; i < items.size(); ++i) {
    items[i].srcs = static_cast<const char* const*>(d) + at;
    at += srcs[i].size();
    items[i].first_tile = static_cast<int32_t>(tiles);
    tiles += (items[i].elems + kRedTileElems - 1) / kRedTileElems;
  }
  if (tiles > INT32_MAX) return fail(CECOLL_INVALID_ARGUMENT, "reduce-scatter too large for one launch");
  void* t = nullptr;
  CUDA_TRY(cudaMalloc(&t, sizeof(RedItem) * items.size()));
  CUDA_TRY(cudaMemcpy(t, items.data(), sizeof(RedItem) * items.size(), cudaMemcpyHostToDevice));
  p->dev_allocs.push_back(t);
  p->dev_alloc_device.push_back(device);
  out->items = static_cast<RedItem*>(t);
  out->nitems = static_cast<int>(items.size());
  out->ntiles = static_cast<int>(tiles);
  out->dtype = dtype;
  out->op = op;
  return {};
}

RedItem make_red(char* dst, int64_t elems, const std::vector<const char*>& srcs, int esize) {
  RedItem r;
  std::memset(&r, 0, sizeof(r));
  r.dst = dst;
  r.elems = elems;
  r.nsrc = static_cast<int32_t>(srcs.size());
  uintptr_t a = reinterpret_cast<uintptr_t>(dst);
  for (const char* s : srcs) a |= reinterpret_cast<uintptr_t>(s);
  r.vec = (a & 15) == 0 && esize > 0;
  return r;
}

}  // namespace

Status plan_create_rs(World* w, Impl impl, int64_t count, int dtype, int op, const std::vector<CallArgs>& args,
                      Plan** out) {
  const int n = w->nranks;
  if (count <= 0) return fail(CECOLL_INVALID_ARGUMENT, "reduce-scatter: count must be positive");
  if (dtype < kF32 || dtype > kF16 || op < kSum || op > kMin)
    return fail(CECOLL_INVALID_ARGUMENT, "reduce-scatter: unknown dtype or op");
  if (impl == Impl::Auto) impl = Impl::Sm;
  if (impl != Impl::Sm && impl != Impl::Pcpy && impl != Impl::B2b && impl != Impl::PrelaunchPcpy &&
      impl != Impl::PrelaunchB2b)
    return fail(CECOLL_UNSUPPORTED, "reduce-scatter: sm, pcpy, b2b, prelaunch_pcpy or prelaunch_b2b");
  const int esize = dtype_bytes(dtype);
  const int64_t s = count * esize;
  auto plan = std::make_unique<Plan>();
  Plan* p = plan.get();
  p->kind = Kind::ReduceScatter;
  p->impl = impl;
  p->chunk = s;
  p->dtype = dtype;
  p->op = op;
  p->sm = impl == Impl::Sm;
  for (const CallArgs& a : args) {
    p->key_rank.push_back(a.rank);
    p->key_send.push_back(a.send);
    p->key_recv.push_back(a.recv);
    p->key_stream.push_back(a.stream);
  }
  std::vector<const char*> send(n, nullptr);
  std::vector<char*> recv(n, nullptr);
  std::vector<bool> have(n, false);
  for (const CallArgs& a : args) {
    if (a.rank < 0 || a.rank >= n || !w->local[a.rank]) return fail(CECOLL_INVALID_ARGUMENT, "rank not local");
    if (have[a.rank]) return fail(CECOLL_INVALID_ARGUMENT, "rank appears twice in one group");
    have[a.rank] = true;
    send[a.rank] = static_cast<const char*>(a.send);
    recv[a.rank] = static_cast<char*>(a.recv);
  }
  if (!w->multiprocess) {
    for (int r = 0; r < n; ++r)
      if (!have[r])
        return fail(CECOLL_INVALID_ARGUMENT,
                    "single-process communicator: every rank must take part (use cecoll_group_start/end)");
  } else {
    if (static_cast<int>(args.size()) != w->nlocal)
      return fail(CECOLL_INVALID_ARGUMENT, "multi-process: every local rank must take part (group calls)");
    if (!p->sm) return fail(CECOLL_UNSUPPORTED, "reduce-scatter over copy engines needs a single-process communicator");
    for (int r = 0; r < n; ++r) {
      if (have[r]) continue;
      bool ok = true;
      send[r] = translate(w, args[0].rank, r, args[0].send, &ok);
      if (!ok) return fail(CECOLL_NOT_REGISTERED, "send must lie in a window registered with cecoll_register");
    }
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, w->device[args[0].rank]);
  p->sms = sms;

  if (!p->sm) {
    // Copy-engine gather: chunk j of every rank lands in rank j's staging
    // slot i (an all-to-all into staging), then rank j reduces its staging.
    std::vector<CallArgs> inner_args;
    std::vector<char*> staging(n, nullptr);
    for (const CallArgs& a : args) {
      DeviceGuard g(w->device[a.rank]);
      void* d = nullptr;
      CUDA_TRY(cudaMalloc(&d, static_cast<size_t>(s) * n));
      p->dev_allocs.push_back(d);
      p->dev_alloc_device.push_back(w->device[a.rank]);
      staging[a.rank] = static_cast<char*>(d);
      inner_args.push_back({a.rank, a.send, d, a.stream});
    }
    Plan* inner = nullptr;
    STATUS_TRY(plan_create(w, Kind::AllToAll, impl, s, inner_args, &inner));
    p->inner.reset(inner);
    for (const Unit& iu : inner->units) {
      Unit u;
      u.device = iu.device;
      u.stream = iu.stream;
      u.ranks = iu.ranks;
      std::vector<RedItem> items;
      std::vector<std::vector<const char*>> srcs;
      for (int j : u.ranks) {
        std::vector<const char*> v;
        for (int i = 0; i < n; ++i) v.push_back(staging[j] + i * s);
        items.push_back(make_red(recv[j], count, v, esize));
        srcs.push_back(v);
      }
      STATUS_TRY(upload_red(p, u.device, items, srcs, dtype, op, &u.red));
      p->units.push_back(std::move(u));
    }
    *out = plan.release();
    return {};
  }

  // SM path: units, flags (rank j reads every rank i's send), reductions.
  std::vector<int> unit_of(n, -1);
  for (const CallArgs& a : args) {
    int found = -1;
    for (size_t u = 0; u < p->units.size(); ++u)
      if (p->units[u].device == w->device[a.rank] && p->units[u].stream == a.stream) found = static_cast<int>(u);
    if (found < 0) {
      Unit u;
      u.device = w->device[a.rank];
      u.stream = a.stream;
      p->units.push_back(u);
      found = static_cast<int>(p->units.size()) - 1;
    }
    p->units[found].ranks.push_back(a.rank);
    unit_of[a.rank] = found;
  }
  for (Unit& u : p->units) std::sort(u.ranks.begin(), u.ranks.end());
  for (int r = 0; r < n; ++r)
    for (int d = 1; d < n; ++d) {
      const int j = (r + d) % n;  // r reads j's send
      if (unit_of[r] >= 0 && unit_of[r] == unit_of[j]) continue;
      if (unit_of[j] >= 0) {
        Unit& u = p->units[unit_of[j]];
        u.start.push_back(op_write(slot(w, r, kSlotRdy + j), 1));
        add_poll(u.finish, slot(w, j, kSlotDone + r));
      }
      if (unit_of[r] >= 0) {
        Unit& u = p->units[unit_of[r]];
        add_poll(u.sm_pre, slot(w, r, kSlotRdy + j));
        u.sm_post.push_back(op_write(slot(w, j, kSlotDone + r), 1));
      }
    }
  for (Unit& u : p->units) {
    std::vector<RedItem> items;
    std::vector<std::vector<const char*>> srcs;
    for (int j : u.ranks) {
      std::vector<const char*> v;
      for (int i = 0; i < n; ++i) v.push_back(send[i] + j * s);
      items.push_back(make_red(recv[j], count, v, esize));
      srcs.push_back(v);
    }
    STATUS_TRY(upload_red(p, u.device, items, srcs, dtype, op, &u.red));
  }
  STATUS_TRY(split_remote(w, p));
  *out = plan.release();
  return {};
}

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

// Records one unit's lanes into a graph: [gate kernel] -> IF{ poll kernel ->
// lanes (copies, item kernels) + placement -> signal kernel }.
Status build_graph(World* w, Plan* p, Unit& u) {
  DeviceGuard g(u.device);
  CUDA_TRY(cudaStreamCreateWithFlags(&u.arm, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&u.graph_done, cudaEventDisableTiming));
  void* host = nullptr;
  CUDA_TRY(cudaHostAlloc(&host, 4096, cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(host, 0, 4096);
  u.posted = static_cast<uint64_t*>(host);
  void* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, 64));
  CUDA_TRY(cudaMemset(d, 0, 64));
  p->dev_allocs.push_back(d);
  p->dev_alloc_device.push_back(u.device);
  u.consumed = static_cast<uint64_t*>(d);
  u.err = static_cast<uint64_t*>(d) + 1;
  u.ready_flag = slot(w, u.ranks[0], kSlotReady);

  // Polls: the unit's own readiness word plus rdy from destinations in other
  // units; signals: done to those destinations (from the lanes' memops).
  std::vector<uint64_t*> polls{u.ready_flag}, sigs, fins;
  for (const LaneExec& le : p->lanes) {
    if (std::find(u.ranks.begin(), u.ranks.end(), le.rank) == u.ranks.end()) continue;
    for (const auto& op : le.pre)
      if (op.operation == CU_STREAM_MEM_OP_WAIT_VALUE_64) polls.push_back(reinterpret_cast<uint64_t*>(op.waitValue.address));
    for (const auto& op : le.post) sigs.push_back(reinterpret_cast<uint64_t*>(op.writeValue.address));
    sigs.insert(sigs.end(), le.post_remote.begin(), le.post_remote.end());
  }
  for (const auto& op : u.finish)
    if (op.operation == CU_STREAM_MEM_OP_WAIT_VALUE_64) fins.push_back(reinterpret_cast<uint64_t*>(op.waitValue.address));
  u.npoll = static_cast<int>(polls.size());
  u.nsig = static_cast<int>(sigs.size());
  u.nfin = static_cast<int>(fins.size());
  STATUS_TRY(upload_ptrs(p, u.device, polls, &u.poll_tab));
  STATUS_TRY(upload_ptrs(p, u.device, sigs, &u.sig_tab));
  STATUS_TRY(upload_ptrs(p, u.device, fins, &u.fin_tab));

  CUDA_TRY(cudaGraphCreate(&u.graph, 0));
  cudaGraphConditionalHandle handle;
  CUDA_TRY(cudaGraphConditionalHandleCreate(&handle, u.graph, 0, cudaGraphCondAssignDefault));
  uint64_t* posted_dev = nullptr;
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&posted_dev), u.posted, 0));

  // Root: the gate kernel.
  CUDA_TRY(cudaStreamBeginCaptureToGraph(u.arm, u.graph, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  cudaError_t le = launch_gate(posted_dev, u.consumed, handle, u.err, u.arm);
  cudaGraph_t captured = nullptr;
  cudaError_t ec = cudaStreamEndCapture(u.arm, &captured);
  CUDA_TRY(le);
  CUDA_TRY(ec);
  size_t nnodes = 0;
  CUDA_TRY(cudaGraphGetNodes(u.graph, nullptr, &nnodes));
  std::vector<cudaGraphNode_t> nodes(nnodes);
  CUDA_TRY(cudaGraphGetNodes(u.graph, nodes.data(), &nnodes));
  if (nnodes != 1) return fail(CECOLL_INTERNAL, "gate capture produced an unexpected graph");

  // cudaGraphNodeParams has no default constructor (union with non-trivial
  // members): zero-initialised raw storage, as the runtime expects.
  alignas(cudaGraphNodeParams) unsigned char cp_storage[sizeof(cudaGraphNodeParams)] = {};
  cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(cp_storage);
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  cudaGraphNode_t if_node;
  CUDA_TRY(cudaGraphAddNode(&if_node, u.graph, nodes.data(), 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];

  // Body: poll -> fork lanes -> join -> signal.
  CUDA_TRY(cudaStreamBeginCaptureToGraph(u.arm, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  Status st;
  auto body_ops = [&]() -> Status {
    CUDA_TRY(launch_poll(u.poll_tab, u.npoll, u.err, u.arm));
    for (const Copy& c : u.placement) CUDA_TRY(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDefault, u.arm));
    cudaEvent_t fork;
    CUDA_TRY(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(fork, u.arm));
    std::vector<const LaneExec*> busy;
    for (const LaneExec& l : p->lanes) {
      if (std::find(u.ranks.begin(), u.ranks.end(), l.rank) == u.ranks.end()) continue;
      if (l.copies.empty() && !l.table.nitems) continue;  // its chunks are in the unit kernel
      RankState* rs = w->local[l.rank].get();
      cudaStream_t ls = rs->lanes[l.lane];
      CUDA_TRY(cudaStreamWaitEvent(ls, fork, 0));
      for (const Copy& c : l.copies) CUDA_TRY(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDefault, ls));
      if (l.table.nitems) CUDA_TRY(launch_items(l.table, mover_grid_for(l.table, p->sms), ls));
      CUDA_TRY(cudaEventRecord(rs->lane_done[l.lane], ls));
      busy.push_back(&l);
    }
    // Same-device chunks of every lane of the unit: one item kernel.
    if (u.table.nitems) CUDA_TRY(launch_items(u.table, mover_grid_for(u.table, p->sms), u.arm));
    for (const LaneExec* l : busy)
      CUDA_TRY(cudaStreamWaitEvent(u.arm, w->local[l->rank]->lane_done[l->lane], 0));
    CUDA_TRY(launch_signal(u.sig_tab, u.nsig, u.arm));
    cudaEventDestroy(fork);
    return {};
  };
  st = body_ops();
  cudaGraph_t body_out = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(u.arm, &body_out);
  if (!st.ok()) return st;
  CUDA_TRY(e2);
  CUDA_TRY(cudaGraphInstantiate(&u.exec, u.graph, 0));
  return {};
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
    if (u.exec) cudaGraphExecDestroy(u.exec);
    if (u.graph) cudaGraphDestroy(u.graph);
    if (u.arm) {
      cudaStreamSynchronize(u.arm);
      cudaStreamDestroy(u.arm);
    }
    if (u.graph_done) cudaEventDestroy(u.graph_done);
    if (u.posted) cudaFreeHost(u.posted);
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
