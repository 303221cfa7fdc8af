// Communicators: single-process worlds (every rank local, the reference's
// single host process) and multi-process worlds (CUDA IPC
// mapping of flag pages and symmetric registered windows).
#include <algorithm>
#include <array>
#include <cstring>
#include <set>

#include "internal.hpp"

namespace cecoll {

namespace {

// Zeroes device memory and waits for it on a private stream: never a
// device-wide synchronisation, which would wait for another world's armed
// prelaunch gate.
Status zero_now(void* p, size_t bytes) {
  cudaStream_t s = nullptr;
  CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaError_t e = cudaMemsetAsync(p, 0, bytes, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  CUDA_TRY(e);
  return {};
}

Status make_rank(World* w, int rank, int device, uint64_t* page = nullptr) {
  DeviceGuard g(device);
  // Every kernel loaded now, never lazily behind an armed gate (kernels.cu).
  CUDA_TRY(preload_kernels());
  CUDA_TRY(preload_reduce_kernels());
  auto rs = std::make_unique<RankState>();
  rs->rank = rank;
  rs->device = device;
  CUDA_TRY(cudaEventCreateWithFlags(&rs->start, cudaEventDisableTiming));
  if (page) {
    rs->flags = page;
    rs->owns_flags = false;
  } else {
    CUDA_TRY(cudaMalloc(&rs->flags, kFlagBytes));
    STATUS_TRY(zero_now(rs->flags, kFlagBytes));
  }
  w->flag_page[rank] = rs->flags;
  w->local[rank] = std::move(rs);
  return {};
}

int count_devices(const std::vector<int>& dev) {
  std::set<int> s(dev.begin(), dev.end());
  return static_cast<int>(s.size());
}

}  // namespace

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
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "EnablePeerAccess", __FILE__, __LINE__);
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
  int32_t status;  // the process's local steps before the exchange (0: ok)
  cudaIpcMemHandle_t flags;  // nlocal flag pages, kFlagBytes apart
  unsigned char uuid[16];    // device identity (ordinals differ between processes
                             // when CUDA_VISIBLE_DEVICES differs)
};

// One blob per process in a registration round.
struct RegInfo {
  int32_t rank;
  int32_t pad;      // status of the process's local steps (0: ok)
  uint64_t offset;  // of the window inside its allocation
  uint64_t bytes;
  cudaIpcMemHandle_t handle;  // of the allocation
};

// Collective calls fail collectively: every process exchanges its status
// after its local steps, so a failure on one process (e.g. opening a peer's
// IPC handle) fails the call on all of them instead of leaving the others to
// wait in the next exchange.
Status agree_all(cecoll_exchange_fn fn, void* ctx, int procs, const Status& local, const char* what) {
  int32_t mine = local.code;
  std::vector<int32_t> all(procs);
  if (fn(ctx, &mine, sizeof(mine), all.data()) != 0) return fail(CECOLL_INTERNAL, std::string(what) + ": exchange failed");
  if (!local.ok()) return local;
  for (int32_t c : all)
    if (c != 0) return fail(c, std::string(what) + ": failed on another process");
  return {};
}

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
                    cecoll_exchange_fn fn, void* ctx, std::vector<ProcInfoView>* out, const unsigned char* uuid,
                    int32_t local_status) {
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
  if (uuid) std::memcpy(mine.uuid, uuid, sizeof(mine.uuid));
  mine.status = local_status;
  std::vector<ProcInfo> all(procs);
  if (fn(ctx, &mine, sizeof(ProcInfo), all.data()) != 0) return fail(CECOLL_INTERNAL, "exchange failed");
  if (local_status != 0) return fail(local_status, last_error());  // keep this process's own message
  for (const ProcInfo& pi : all)
    if (pi.status != 0) return fail(pi.status, "comm_init: failed on another process");
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
    std::memcpy(v.uuid, pi.uuid, sizeof(v.uuid));
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
  // Local steps before the exchange report their status through it (a
  // process that fails here must not leave the others waiting in it).
  cudaIpcMemHandle_t h;
  std::memset(&h, 0, sizeof(h));
  std::vector<std::array<unsigned char, 16>> uuids(1);
  auto local_steps = [&]() -> Status {
    // One allocation holds the flag pages of every local rank (one IPC handle).
    void* block = nullptr;
    CUDA_TRY(cudaMalloc(&block, kFlagBytes * nlocal));
    w->flag_block = block;
    STATUS_TRY(zero_now(block, kFlagBytes * nlocal));
    for (int k = 0; k < nlocal; ++k)
      STATUS_TRY(make_rank(w.get(), first + k, device,
                           reinterpret_cast<uint64_t*>(static_cast<char*>(block) + k * kFlagBytes)));
    CUDA_TRY(cudaIpcGetMemHandle(&h, block));
    // Device identity by UUID: a peer process's device is mapped to this
    // process's ordinal for it, or to a unique negative id when this process
    // cannot see it (then it is never mistaken for a local device).
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(CECOLL_INVALID_ARGUMENT, "device out of range");
    uuids.assign(ndev, {});
    for (int d = 0; d < ndev; ++d) {
      cudaDeviceProp prop;
      CUDA_TRY(cudaGetDeviceProperties(&prop, d));
      std::memcpy(uuids[d].data(), prop.uuid.bytes, 16);
    }
    return {};
  };
  const Status pre = local_steps();
  const int dev_index = pre.ok() ? device : 0;
  std::vector<ProcInfoView> procs;
  STATUS_TRY(gather_procs(nranks, first, nlocal, device, &h, fn, ctx, &procs, uuids[dev_index].data(), pre.code));
  for (size_t pi = 0; pi < procs.size(); ++pi) {
    ProcInfoView& pv = procs[pi];
    int local_ordinal = -1000 - static_cast<int>(pi);
    for (size_t d = 0; d < uuids.size(); ++d)
      if (std::memcmp(uuids[d].data(), pv.uuid, 16) == 0) local_ordinal = static_cast<int>(d);
    pv.device = local_ordinal;
  }
  Status opened_all;
  for (const ProcInfoView& pv : procs) {
    char* base = nullptr;
    if (pv.first != first) {
      void* opened = nullptr;
      opened_all = open_ipc(w.get(), pv.flags, &opened);
      if (!opened_all.ok()) break;
      base = static_cast<char*>(opened);
    }
    for (int k = 0; k < pv.nlocal; ++k) {
      const int r = pv.first + k;
      w->device[r] = pv.device;
      if (pv.first != first) w->flag_page[r] = reinterpret_cast<uint64_t*>(base + k * kFlagBytes);
    }
  }
  STATUS_TRY(agree_all(fn, ctx, nranks / nlocal, opened_all, "comm_init_ranks"));
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
  // Local steps report through the exchange (pad = status) rather than
  // returning early: the other processes are about to wait in it.
  RegInfo mine;
  std::memset(&mine, 0, sizeof(mine));
  mine.rank = rank;
  mine.bytes = bytes;
  Status local;
  if (win.bytes != bytes) {
    local = fail(CECOLL_INVALID_ARGUMENT, "cecoll_register: windows must be symmetric (same size on every rank)");
  } else {
    CUdeviceptr base = 0;
    size_t size = 0;
    const CUresult r = driver_api()->MemGetAddressRange(&base, &size, reinterpret_cast<CUdeviceptr>(ptr));
    if (r != CUDA_SUCCESS) {
      local = cu_fail(r, "cuMemGetAddressRange", __FILE__, __LINE__);
    } else {
      mine.offset = reinterpret_cast<uint64_t>(ptr) - base;
      const cudaError_t e = cudaIpcGetMemHandle(&mine.handle, reinterpret_cast<void*>(base));
      if (e != cudaSuccess) local = cuda_fail(e, "cudaIpcGetMemHandle", __FILE__, __LINE__);
    }
  }
  mine.pad = local.code;
  const int procs = w->nranks / w->nlocal;
  std::vector<RegInfo> all(procs);
  if (fn(ctx, &mine, sizeof(RegInfo), all.data()) != 0) return fail(CECOLL_INTERNAL, "exchange failed");
  if (!local.ok()) return agree_all(fn, ctx, procs, local, "cecoll_register");
  for (const RegInfo& ri : all)
    if (ri.pad != 0) return agree_all(fn, ctx, procs, fail(ri.pad, "cecoll_register: failed on another process"),
                                      "cecoll_register");
  Status st;
  for (const RegInfo& ri : all) {
    if (ri.bytes != bytes) {
      st = fail(CECOLL_INVALID_ARGUMENT, "cecoll_register: windows must be symmetric (same size on every rank)");
      break;
    }
    if (ri.rank < 0 || ri.rank >= w->nranks) {
      st = fail(CECOLL_INVALID_ARGUMENT, "bad rank in registration");
      break;
    }
    if (ri.rank == rank) {
      win.rank_base[ri.rank] = static_cast<char*>(ptr);
      continue;
    }
    void* opened = nullptr;
    st = open_ipc(w, ri.handle, &opened);
    if (!st.ok()) break;
    win.rank_base[ri.rank] = static_cast<char*>(opened) + ri.offset;
  }
  return agree_all(fn, ctx, procs, st, "cecoll_register");
}

Status world_deregister(World* w, void* ptr) {
  if (!w->multiprocess) return {};  // nothing was mapped
  // The window stops translating addresses, and cached plans (which hold the
  // peers' mapped addresses) are dropped so a later registration at the same
  // local address cannot reuse stale peer addresses. The IPC mappings
  // themselves stay open until the communicator is destroyed. Explicit plans
  // built on the window must be destroyed by the caller first.
  bool found = false;
  for (Window& win : w->windows) {
    for (int k = 0; k < w->nlocal; ++k) {
      if (win.rank_base[w->first_local + k] == ptr) {
        win.live = false;  // symmetric: the window is gone for every rank
        found = true;
        break;
      }
    }
  }
  if (!found) return fail(CECOLL_NOT_REGISTERED, "cecoll_deregister: pointer is not a registered window base");
  // Released later (exec.cpp retire_plan): freeing plan memory synchronises
  // the device, which must not happen while a prelaunch gate is armed.
  std::vector<std::unique_ptr<Plan>> drop;
  drop.swap(w->plans);
  w->last_plan = nullptr;
  for (auto& p : drop) retire_plan(w, std::move(p));
  return {};
}

Status world_mem_alloc(World* w, int rank, size_t bytes, void** out) {
  RankState* rs = w->local[rank].get();
  if (!rs) return fail(CECOLL_INVALID_ARGUMENT, "cecoll_mem_alloc: rank is not local");
  DeviceGuard g(rs->device);
  // Whole 2 MiB pages: the registered window then covers the allocation
  // exactly (symmetric when every rank asks for the same size).
  constexpr size_t kPage = size_t(2) << 20;
  const size_t padded = (bytes + kPage - 1) / kPage * kPage;
  void* p = nullptr;
  CUDA_TRY(cudaMalloc(&p, padded));
  Status s = world_register(w, rank, p, padded, w->exchange, w->exchange_ctx);
  if (!s.ok()) {
    cudaFree(p);
    return s;
  }
  w->allocs.push_back({p, rs->device});
  *out = p;
  return {};
}

Status world_mem_free(World* w, void* ptr) {
  auto it = std::find_if(w->allocs.begin(), w->allocs.end(), [&](const auto& a) { return a.first == ptr; });
  if (it == w->allocs.end()) return fail(CECOLL_INVALID_ARGUMENT, "cecoll_mem_free: not a cecoll_mem_alloc pointer");
  // cudaFree synchronises the device: behind an armed prelaunch gate (any
  // world of the process) it would wait for a trigger that may never come.
  if (armed_units() > 0)
    return fail(CECOLL_INVALID_ARGUMENT,
                "cecoll_mem_free: a prelaunch plan is armed (disarm or launch it first; cudaFree would wait for it)");
  STATUS_TRY(world_deregister(w, ptr));
  DeviceGuard g(it->second);
  CUDA_TRY(cudaFree(ptr));  // synchronises with work still reading the buffer
  w->allocs.erase(it);
  return {};
}

Status world_release(World* w) {
  if (w->tracer) {
    std::string discard;
    trace_end(w, &discard);
  }
  for (auto& p : w->plans) note_async(w, plan_destroy(w, p.get()));
  w->plans.clear();
  // Armed explicit plans would keep their gate kernels waiting (and the
  // device synchronisation below would never return): cancel them. Their
  // cecoll_plan handles must not be used afterwards.
  for (Plan* p : w->explicit_plans) note_async(w, plan_destroy(w, p));
  w->explicit_plans.clear();
  release_retired(w, true);
  for (auto& rs : w->local) {
    if (!rs) continue;
    DeviceGuard g(rs->device);
    cudaDeviceSynchronize();
    for (auto s : rs->lanes) cudaStreamDestroy(s);
    for (auto e : rs->lane_done) cudaEventDestroy(e);
    if (rs->start) cudaEventDestroy(rs->start);
    if (rs->flags && rs->owns_flags) cudaFree(rs->flags);
  }
  for (auto& a : w->allocs) {
    DeviceGuard g(a.second);
    cudaFree(a.first);
  }
  for (void* p : w->ipc_opened) cudaIpcCloseMemHandle(p);
  if (w->flag_block) cudaFree(w->flag_block);
  const Status result = w->async_error;
  delete w;
  return result;
}

}  // namespace cecoll
