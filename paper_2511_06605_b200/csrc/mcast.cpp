// NVLS (switch multicast) all-gather — SURVEY §8(f)2, the multicast analogue
// of the reference's two-destination broadcast command (compiler.cpp:166-205,
// verifier.cpp:304-312): one read of each source chunk and one store stream
// per GPU, replicated by the NVSwitch to every GPU of the group.
//
// EXPERIMENTAL. The one-GPU development boxes refuse cuMulticastCreate for
// every handle type (profiles/mc_probe_r01.txt), so this path has only been
// compiled, never executed; bench_mgpu.py tries it on the multi-GPU node
// under its consensus + parity protocol. Every failure is a status, never a
// crash.
//
// Window layout (one per process, nlocal == 1): a multicast object of
// `padded` bytes bound to `padded` bytes of this GPU's memory; data region
// [0, n*cap) (rank i's chunk at [i*s, (i+1)*s) — compiler.cpp:115-122), then
// one flag per rank at data_bytes + i*128. A collective with epoch e: every
// rank multicasts its chunk, then multicasts flag[rank] = e (release); the
// caller stream waits (stream memops, GEQ) until its local copy of every flag
// is >= e. Flags only grow, so nothing is reset.
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>

#include "internal.hpp"

#ifndef SYS_pidfd_open
#define SYS_pidfd_open 434
#endif
#ifndef SYS_pidfd_getfd
#define SYS_pidfd_getfd 438
#endif

namespace cecoll {

struct McWindow {
  World* world = nullptr;
  int rank = 0;
  int device = 0;
  int64_t cap = 0;
  size_t data_bytes = 0;
  size_t padded = 0;
  CUmemGenericAllocationHandle mc = 0, phys = 0;
  bool have_mc = false, have_phys = false, bound = false;
  CUdeviceptr mc_va = 0, uc_va = 0;
  bool mc_mapped = false, uc_mapped = false;
  int imported_fd = -1, exported_fd = -1;
  unsigned* ctr = nullptr;
  uint64_t epoch = 0;
  std::string how;  // handle type used
};

namespace {

struct McBlob {
  int32_t first;   // process's first rank
  int32_t status;  // 0 ok
  int32_t type;    // CUmemAllocationHandleType used by process 0
  int32_t pid;
  int32_t fd;
  int32_t pad;
  CUmemFabricHandle fabric;
};

// All-gather of one status code per process: the first failure anywhere
// fails every process at the same step (no process is left waiting).
Status agree(World* w, const Status& local, const char* step) {
  const int procs = w->nranks / w->nlocal;
  int32_t mine = local.code;
  std::vector<int32_t> all(procs);
  if (w->exchange(w->exchange_ctx, &mine, sizeof(mine), all.data()) != 0)
    return fail(CECOLL_INTERNAL, std::string("multicast: exchange failed at ") + step);
  if (!local.ok()) return local;
  for (int32_t c : all)
    if (c != 0) return fail(CECOLL_UNSUPPORTED, std::string("multicast: a peer process failed at ") + step);
  return {};
}

Status cu_step(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return {};
  const char* s = "?";
  if (driver_api()) driver_api()->GetErrorString(r, &s);
  return fail(CECOLL_UNSUPPORTED, std::string("multicast: ") + what + ": " + s);
}

}  // namespace

void mc_release(McWindow* m) {
  if (!m) return;
  const DriverApi* d = driver_api();
  DeviceGuard g(m->device);
  cudaDeviceSynchronize();
  if (d) {
    if (m->mc_mapped) d->MemUnmap(m->mc_va, m->padded);
    if (m->mc_va) d->MemAddressFree(m->mc_va, m->padded);
    if (m->uc_mapped) d->MemUnmap(m->uc_va, m->padded);
    if (m->uc_va) d->MemAddressFree(m->uc_va, m->padded);
    if (m->bound) {
      CUdevice cud;
      if (d->DeviceGet(&cud, m->device) == CUDA_SUCCESS) d->MulticastUnbind(m->mc, cud, 0, m->padded);
    }
    if (m->have_phys) d->MemRelease(m->phys);
    if (m->have_mc) d->MemRelease(m->mc);
  }
  if (m->ctr) cudaFree(m->ctr);
  if (m->imported_fd >= 0) close(m->imported_fd);
  if (m->exported_fd >= 0) close(m->exported_fd);
  delete m;
}

Status mc_create(World* w, int rank, int64_t cap, McWindow** out) {
  *out = nullptr;
  const DriverApi* d = driver_api();
  if (!w->multiprocess || w->nlocal != 1)
    return fail(CECOLL_UNSUPPORTED, "multicast window: one process per GPU (comm_init_rank) only");
  if (cap <= 0 || cap % 16) return fail(CECOLL_INVALID_ARGUMENT, "multicast window: capacity must be a positive multiple of 16");
  auto m = new McWindow;
  m->world = w;
  m->rank = rank;
  m->device = w->device[rank];
  m->cap = cap;
  DeviceGuard g(m->device);
  const int n = w->nranks;
  Status st;
  int supported = 0;
  if (!d || !d->has_multicast) st = fail(CECOLL_UNSUPPORTED, "multicast: driver entry points missing");
  if (st.ok()) {
    CUdevice cud;
    st = cu_step(d->DeviceGet(&cud, m->device), "cuDeviceGet");
    if (st.ok()) st = cu_step(d->DeviceGetAttribute(&supported, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cud),
                              "multicast attribute");
    if (st.ok() && !supported) st = fail(CECOLL_UNSUPPORTED, "multicast: device reports no switch multicast support");
  }
  // Sizes: the multicast and the physical allocation granularities.
  CUmulticastObjectProp prop;
  std::memset(&prop, 0, sizeof(prop));
  prop.numDevices = static_cast<unsigned>(n);
  m->data_bytes = static_cast<size_t>(n) * static_cast<size_t>(cap);
  prop.size = m->data_bytes + static_cast<size_t>(n) * 128;
  CUmemAllocationProp ap;
  std::memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = m->device;
  size_t gran = 0;
  if (st.ok()) {
    size_t g_mc = 0, g_ph = 0;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    st = cu_step(d->MulticastGetGranularity(&g_mc, &prop, CU_MULTICAST_GRANULARITY_MINIMUM), "granularity");
    if (st.ok()) st = cu_step(d->MemGetAllocationGranularity(&g_ph, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM), "granularity");
    gran = std::max(g_mc, g_ph);
    if (gran == 0) gran = size_t(2) << 20;
    m->padded = (prop.size + gran - 1) / gran * gran;
    prop.size = m->padded;
  }

  // Process 0 creates the object and exports it: a fabric handle (a plain
  // blob) when the node supports it, else a POSIX fd fetched by the other
  // processes with pidfd_getfd.
  McBlob mine;
  std::memset(&mine, 0, sizeof(mine));
  mine.first = w->first_local;
  if (st.ok() && w->first_local == 0) {
    Status cs = fail(CECOLL_UNSUPPORTED, "multicast: cuMulticastCreate refused every handle type");
    for (CUmemAllocationHandleType t : {CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR}) {
      CUmulticastObjectProp p2 = prop;
      p2.handleTypes = t;
      CUmemGenericAllocationHandle h;
      CUresult r = d->MulticastCreate(&h, &p2);
      if (r != CUDA_SUCCESS) {
        cs = cu_step(r, t == CU_MEM_HANDLE_TYPE_FABRIC ? "cuMulticastCreate(fabric)" : "cuMulticastCreate(posix fd)");
        continue;
      }
      m->mc = h;
      m->have_mc = true;
      mine.type = static_cast<int32_t>(t);
      if (t == CU_MEM_HANDLE_TYPE_FABRIC) {
        cs = cu_step(d->MemExportToShareableHandle(&mine.fabric, h, t, 0), "export fabric handle");
        m->how = "fabric";
      } else {
        int fd = -1;
        cs = cu_step(d->MemExportToShareableHandle(&fd, h, t, 0), "export posix fd");
        m->exported_fd = fd;
        mine.pid = static_cast<int32_t>(getpid());
        mine.fd = fd;
        m->how = "posix_fd";
      }
      if (cs.ok()) break;
      d->MemRelease(h);
      m->have_mc = false;
    }
    st = cs;
  }
  mine.status = st.code;
  const int procs = w->nranks / w->nlocal;
  std::vector<McBlob> all(procs);
  if (w->exchange(w->exchange_ctx, &mine, sizeof(mine), all.data()) != 0) {
    mc_release(m);
    return fail(CECOLL_INTERNAL, "multicast: exchange failed");
  }
  const McBlob* root = nullptr;
  for (const McBlob& b : all)
    if (b.first == 0) root = &b;
  bool any_failed = false;
  for (const McBlob& b : all) any_failed |= b.status != 0;
  if (!root || any_failed) {
    Status r = st.ok() ? fail(CECOLL_UNSUPPORTED, "multicast: the creating process failed") : st;
    mc_release(m);
    return r;
  }
  // Import on the other processes.
  if (w->first_local != 0) {
    const auto t = static_cast<CUmemAllocationHandleType>(root->type);
    if (t == CU_MEM_HANDLE_TYPE_FABRIC) {
      CUmemFabricHandle fh = root->fabric;
      st = cu_step(d->MemImportFromShareableHandle(&m->mc, &fh, t), "import fabric handle");
      m->how = "fabric";
    } else {
      const long pidfd = syscall(SYS_pidfd_open, root->pid, 0);
      const long fd = pidfd >= 0 ? syscall(SYS_pidfd_getfd, pidfd, root->fd, 0) : -1;
      if (pidfd >= 0) close(static_cast<int>(pidfd));
      if (fd < 0) {
        st = fail(CECOLL_UNSUPPORTED, "multicast: pidfd_getfd of the exported fd failed (ptrace policy?)");
      } else {
        m->imported_fd = static_cast<int>(fd);
        st = cu_step(d->MemImportFromShareableHandle(&m->mc, reinterpret_cast<void*>(static_cast<intptr_t>(fd)), t),
                     "import posix fd");
      }
      m->how = "posix_fd";
    }
    m->have_mc = st.ok();
  }
  st = agree(w, st, "import");
  if (st.ok()) {
    CUdevice cud;
    st = cu_step(d->DeviceGet(&cud, m->device), "cuDeviceGet");
    if (st.ok()) st = cu_step(d->MulticastAddDevice(m->mc, cud), "cuMulticastAddDevice");
  }
  st = agree(w, st, "add device");  // every device added before any binding
  if (st.ok()) {
    st = cu_step(d->MemCreate(&m->phys, m->padded, &ap, 0), "cuMemCreate");
    m->have_phys = st.ok();
    if (st.ok()) st = cu_step(d->MulticastBindMem(m->mc, 0, m->phys, 0, m->padded, 0), "cuMulticastBindMem");
    m->bound = st.ok();
  }
  st = agree(w, st, "bind");
  if (st.ok()) {
    CUmemAccessDesc acc;
    std::memset(&acc, 0, sizeof(acc));
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = m->device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    st = cu_step(d->MemAddressReserve(&m->mc_va, m->padded, gran, 0, 0), "reserve multicast VA");
    if (st.ok()) st = cu_step(d->MemMap(m->mc_va, m->padded, 0, m->mc, 0), "map multicast");
    m->mc_mapped = st.ok();
    if (st.ok()) st = cu_step(d->MemSetAccess(m->mc_va, m->padded, &acc, 1), "multicast access");
    if (st.ok()) st = cu_step(d->MemAddressReserve(&m->uc_va, m->padded, gran, 0, 0), "reserve unicast VA");
    if (st.ok()) st = cu_step(d->MemMap(m->uc_va, m->padded, 0, m->phys, 0), "map unicast");
    m->uc_mapped = st.ok();
    if (st.ok()) st = cu_step(d->MemSetAccess(m->uc_va, m->padded, &acc, 1), "unicast access");
    if (st.ok()) {
      cudaError_t e = cudaMemset(reinterpret_cast<void*>(m->uc_va), 0, m->padded);
      if (e == cudaSuccess) e = cudaMalloc(&m->ctr, 64);
      if (e == cudaSuccess) e = cudaMemset(m->ctr, 0, 64);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (e != cudaSuccess) st = cuda_fail(e, "multicast window init", __FILE__, __LINE__);
    }
  }
  st = agree(w, st, "map");  // every window zeroed before anyone stores into it
  if (!st.ok()) {
    mc_release(m);
    return st;
  }
  *out = m;
  return {};
}

Status mc_allgather(McWindow* m, const void* send, int64_t s, cudaStream_t stream) {
  if (s <= 0 || s > m->cap || s % 16 || reinterpret_cast<uintptr_t>(send) % 16)
    return fail(CECOLL_INVALID_ARGUMENT, "multicast all-gather: 0 < s <= capacity, s and send 16-byte aligned");
  World* w = m->world;
  DeviceGuard g(m->device);
  const uint64_t e = ++m->epoch;
  char* mc_base = reinterpret_cast<char*>(m->mc_va);
  char* uc_base = reinterpret_cast<char*>(m->uc_va);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device);
  CUDA_TRY(launch_mc_store(static_cast<const char*>(send), mc_base + static_cast<int64_t>(m->rank) * s, s,
                           reinterpret_cast<uint64_t*>(mc_base + m->data_bytes + m->rank * 128), e, m->ctr, 2 * sms,
                           stream));
  ++w->counters[kCtrKernels];
  MemOps waits;
  for (int i = 0; i < w->nranks; ++i)
    waits.push_back(op_wait(reinterpret_cast<uint64_t*>(uc_base + m->data_bytes + i * 128), e));
  return submit(w, stream, waits);
}

void* mc_recv(McWindow* m) { return reinterpret_cast<void*>(m->uc_va); }
const char* mc_how(McWindow* m) { return m->how.c_str(); }

}  // namespace cecoll
