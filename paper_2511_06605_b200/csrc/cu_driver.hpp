// Driver-API entry points resolved at runtime through cudart.
//
// libcecoll links cudart statically and never links libcuda, so the shared
// library loads (and its CPU-side planner runs) on a machine without a GPU
// driver. The stream memory operations (cuStreamWaitValue64 /
// cuStreamWriteValue64 / cuStreamBatchMemOp) have no cudart equivalent;
// they are looked up once with cudaGetDriverEntryPointByVersion the first
// time a communicator is created.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

namespace cecoll {

struct DriverApi {
  CUresult (*StreamWaitValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned) = nullptr;
  CUresult (*StreamWriteValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned) = nullptr;
  CUresult (*StreamWaitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned) = nullptr;
  CUresult (*StreamWriteValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned) = nullptr;
  CUresult (*StreamBatchMemOp)(CUstream, unsigned, CUstreamBatchMemOpParams*, unsigned) = nullptr;
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*MemGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
  // Switch multicast (NVLS) and virtual memory management (mcast.cpp).
  CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                               unsigned long long) = nullptr;
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long) = nullptr;
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) =
      nullptr;
  CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
  // Explicit graph construction (exec.cpp GraphSink): stream memory operations
  // as batch-mem-op graph nodes, in the context current on the calling thread.
  CUresult (*GraphAddBatchMemOpNode)(CUgraphNode*, CUgraph, const CUgraphNode*, size_t,
                                     const CUDA_BATCH_MEM_OP_NODE_PARAMS*) = nullptr;
  CUresult (*CtxGetCurrent)(CUcontext*) = nullptr;
  bool has_multicast = false;
  bool loaded = false;
};

// Returns the process-wide table, loading it on first use. Returns nullptr
// when the CUDA driver is absent (CPU-only machine).
const DriverApi* driver_api();

}  // namespace cecoll
