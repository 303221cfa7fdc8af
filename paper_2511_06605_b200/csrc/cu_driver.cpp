#include "cu_driver.hpp"

#include <mutex>

namespace cecoll {

namespace {

template <typename F>
bool load(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion(name, &p, 12090, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || p == nullptr) {
    cudaGetLastError();
    return false;
  }
  fn = reinterpret_cast<F>(p);
  return true;
}

}  // namespace

const DriverApi* driver_api() {
  static DriverApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
      cudaGetLastError();
      return;
    }
    bool ok = true;
    ok &= load("cuStreamWaitValue64", api.StreamWaitValue64);
    ok &= load("cuStreamWriteValue64", api.StreamWriteValue64);
    ok &= load("cuStreamWaitValue32", api.StreamWaitValue32);
    ok &= load("cuStreamWriteValue32", api.StreamWriteValue32);
    ok &= load("cuStreamBatchMemOp", api.StreamBatchMemOp);
    ok &= load("cuDeviceGetAttribute", api.DeviceGetAttribute);
    ok &= load("cuGetErrorString", api.GetErrorString);
    ok &= load("cuGraphAddBatchMemOpNode", api.GraphAddBatchMemOpNode);
    ok &= load("cuCtxGetCurrent", api.CtxGetCurrent);
    bool mc = load("cuMulticastCreate", api.MulticastCreate);
    mc &= load("cuMulticastGetGranularity", api.MulticastGetGranularity);
    mc &= load("cuMulticastAddDevice", api.MulticastAddDevice);
    mc &= load("cuMulticastBindMem", api.MulticastBindMem);
    mc &= load("cuMulticastUnbind", api.MulticastUnbind);
    mc &= load("cuMemCreate", api.MemCreate);
    mc &= load("cuMemRelease", api.MemRelease);
    mc &= load("cuMemExportToShareableHandle", api.MemExportToShareableHandle);
    mc &= load("cuMemImportFromShareableHandle", api.MemImportFromShareableHandle);
    mc &= load("cuMemAddressReserve", api.MemAddressReserve);
    mc &= load("cuMemAddressFree", api.MemAddressFree);
    mc &= load("cuMemMap", api.MemMap);
    mc &= load("cuMemUnmap", api.MemUnmap);
    mc &= load("cuMemSetAccess", api.MemSetAccess);
    mc &= load("cuMemGetAllocationGranularity", api.MemGetAllocationGranularity);
    mc &= load("cuDeviceGet", api.DeviceGet);
    api.has_multicast = mc;
    ok &= load("cuMemGetAddressRange", api.MemGetAddressRange);
    api.loaded = ok;
  });
  return api.loaded ? &api : nullptr;
}

}  // namespace cecoll
