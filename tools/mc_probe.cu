// Multicast (NVLS) and VMM probe: which handle types and multicast features
// does this B200 expose, and does a multimem.st through a one-device
// multicast object land in the bound physical memory?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mc_probe tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    CUresult r_ = (x);                                                         \
    if (r_ != CUDA_SUCCESS) {                                                  \
      const char* s_ = nullptr;                                                \
      cuGetErrorString(r_, &s_);                                               \
      std::printf("FAIL %s -> %d %s\n", #x, (int)r_, s_ ? s_ : "?");           \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__global__ void mc_store(uint4* mc, size_t n16, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t a = seed ^ (uint32_t)i, b = a * 2654435761u, c = b ^ 0x9e3779b9u, d = c + 7u;
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "r"(a), "r"(b), "r"(c),
                 "r"(d)
                 : "memory");
  }
}

__global__ void uc_store(uint4* p, size_t n16, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t a = seed ^ (uint32_t)i, b = a * 2654435761u, c = b ^ 0x9e3779b9u, d = c + 7u;
    p[i] = make_uint4(a, b, c, d);
  }
}

__global__ void check(const uint4* p, size_t n16, uint32_t seed, unsigned long long* bad) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t a = seed ^ (uint32_t)i, b = a * 2654435761u, c = b ^ 0x9e3779b9u, d = c + 7u;
    uint4 v = p[i];
    if (v.x != a || v.y != b || v.z != c || v.w != d) atomicAdd(bad, 1ull);
  }
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  int ndev = 0;
  cuDeviceGetCount(&ndev);
  struct {
    const char* name;
    CUdevice_attribute a;
  } attrs[] = {
      {"MULTICAST_SUPPORTED", CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED},
      {"VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED", CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED},
      {"HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED", CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED},
      {"HANDLE_TYPE_FABRIC_SUPPORTED", CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED},
      {"GPU_DIRECT_RDMA_WITH_CUDA_VMM_SUPPORTED", CU_DEVICE_ATTRIBUTE_GPU_DIRECT_RDMA_WITH_CUDA_VMM_SUPPORTED},
  };
  std::printf("devices %d\n", ndev);
  int mc_ok = 0;
  for (auto& x : attrs) {
    int v = -1;
    cuDeviceGetAttribute(&v, x.a, dev);
    std::printf("%s %d\n", x.name, v);
    if (x.a == CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED) mc_ok = v;
  }

  // VMM allocation (always available on B200): granularity and a mapped buffer.
  const size_t bytes = 256ull << 20;
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0, gran_rec = 0;
  CK(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  CK(cuMemGetAllocationGranularity(&gran_rec, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  std::printf("vmm granularity min %zu recommended %zu\n", gran, gran_rec);
  CUmemGenericAllocationHandle phys;
  CK(cuMemCreate(&phys, bytes, &prop, 0));
  CUdeviceptr uc = 0;
  CK(cuMemAddressReserve(&uc, bytes, 0, 0, 0));
  CK(cuMemMap(uc, bytes, 0, phys, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, bytes, &acc, 1));
  int fd = -1;
  CUresult er = cuMemExportToShareableHandle(&fd, phys, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  std::printf("export posix fd -> %d (fd %d)\n", (int)er, fd);

  unsigned long long* bad;
  cudaMalloc(&bad, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t n16 = bytes / 16;
  float ms = 0;
  for (int it = 0; it < 3; ++it) {
    cudaEventRecord(e0);
    uc_store<<<148 * 8, 512>>>((uint4*)uc, n16, 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  cudaEventElapsedTime(&ms, e0, e1);
  std::printf("unicast store 256 MiB: %.1f us (%.0f GB/s)\n", ms * 1e3, bytes / (ms * 1e-3) / 1e9);

  if (!mc_ok) {
    std::printf("multicast unsupported on this device: stop\n");
    return 0;
  }
  CUmulticastObjectProp mp{};
  mp.numDevices = 1;
  mp.size = bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t mgran = 0, mgran_rec = 0;
  CK(cuMulticastGetGranularity(&mgran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CK(cuMulticastGetGranularity(&mgran_rec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  std::printf("multicast granularity min %zu recommended %zu\n", mgran, mgran_rec);
  CUmemGenericAllocationHandle mc;
  {
    CUresult best = CUDA_ERROR_UNKNOWN;
    const unsigned long long types[] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC, 0};
    for (unsigned long long t : types)
      for (unsigned nd : {1u, 2u}) {
        for (size_t sz : {bytes, mgran_rec}) {
          CUmulticastObjectProp q = mp;
          q.handleTypes = t;
          q.numDevices = nd;
          q.size = sz;
          CUmemGenericAllocationHandle h;
          CUresult r = cuMulticastCreate(&h, &q);
          std::printf("cuMulticastCreate handleTypes=%llu numDevices=%u size=%zu -> %d\n", t, nd, sz, (int)r);
          if (r == CUDA_SUCCESS) {
            if (nd == 1 && sz == bytes && best != CUDA_SUCCESS) {
              mc = h;
              best = r;
              mp = q;
            } else {
              cuMemRelease(h);
            }
          }
        }
      }
    if (best != CUDA_SUCCESS) {
      std::printf("no one-device multicast object: stop\n");
      return 0;
    }
  }
  CK(cuMulticastAddDevice(mc, dev));
  CK(cuMulticastBindMem(mc, 0, phys, 0, bytes, 0));
  CUdeviceptr mva = 0;
  CK(cuMemAddressReserve(&mva, bytes, mgran_rec, 0, 0));
  CK(cuMemMap(mva, bytes, 0, mc, 0));
  CK(cuMemSetAccess(mva, bytes, &acc, 1));
  for (int it = 0; it < 3; ++it) {
    cudaEventRecord(e0);
    mc_store<<<148 * 8, 512>>>((uint4*)mva, n16, 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  cudaError_t ce = cudaGetLastError();
  cudaEventElapsedTime(&ms, e0, e1);
  std::printf("multimem.st 256 MiB (1 device): %.1f us (%.0f GB/s) err %s\n", ms * 1e3,
              bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(ce));
  cudaMemset(bad, 0, 8);
  check<<<148 * 8, 512>>>((const uint4*)uc, n16, 2, bad);
  unsigned long long hb = 0;
  cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
  std::printf("multicast store visible through unicast mapping: %s (%llu bad vectors)\n", hb ? "NO" : "yes", hb);
  return 0;
}
