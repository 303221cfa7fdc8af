// Back-to-back cadence of a small copy kernel (the 8-rank 4 KiB all-to-all's
// 256 KiB of items) with and without programmatic dependent launch (PDL):
// can the next collective's launch and prologue overlap the previous one's
// tail on B200?
//   tools/pdl_probe [bytes] [reps]
// Variants (device time per kernel, CUDA events around `reps` launches):
//   plain          : cudaLaunchKernel back to back
//   pdl            : cudaLaunchKernelEx with programmatic stream
//                    serialisation; the kernel waits (griddepcontrol.wait)
//                    before its first global access and lets dependents
//                    launch at entry (griddepcontrol.launch_dependents)
//   pdl_late       : as pdl, dependents released only after the copy
//   graph1         : one-kernel graph, launched `reps` times
//   graph_chain    : one graph of `reps` kernels with ordinary edges
//   graph_chain_pdl: the same chain captured from PDL launches
//                    (programmatic edges)
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

template <int kMode>  // 0 plain, 1 pdl early trigger, 2 pdl late trigger
__global__ void copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n16) {
  if (kMode) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (kMode == 1) asm volatile("griddepcontrol.launch_dependents;");
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  if (kMode == 2) asm volatile("griddepcontrol.launch_dependents;");
}

template <int kMode>
static void launch(const int4* s, int4* d, int64_t n16, int grid, cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, copy_kernel<kMode>, s, d, n16));
}

template <typename F>
static double per_us(F f, int reps, cudaStream_t st) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaStreamSynchronize(st));
  double best = 1e30;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(a, st));
    f();
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  return best * 1000.0 / reps;
}

int main(int argc, char** argv) {
  const int64_t bytes = argc > 1 ? atoll(argv[1]) : 256 * 1024;
  const int reps = argc > 2 ? atoi(argv[2]) : 1000;
  const int64_t n16 = bytes / 16;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int grid = (int)((n16 + 255) / 256);
  if (grid > 2 * sms) grid = 2 * sms;
  int4 *s, *d;
  CK(cudaMalloc(&s, bytes));
  CK(cudaMalloc(&d, bytes));
  CK(cudaMemset(s, 1, bytes));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  printf("# pdl_probe: %lld bytes, grid %d, %d reps\n", (long long)bytes, grid, reps);
  printf("plain            %.3f us\n", per_us([&] { for (int i = 0; i < reps; ++i) launch<0>(s, d, n16, grid, st, false); }, reps, st));
  printf("pdl              %.3f us\n", per_us([&] { for (int i = 0; i < reps; ++i) launch<1>(s, d, n16, grid, st, true); }, reps, st));
  printf("pdl_late         %.3f us\n", per_us([&] { for (int i = 0; i < reps; ++i) launch<2>(s, d, n16, grid, st, true); }, reps, st));
  printf("pdl_kernel_plain %.3f us\n", per_us([&] { for (int i = 0; i < reps; ++i) launch<1>(s, d, n16, grid, st, false); }, reps, st));

  auto capture = [&](int count, bool pdl) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < count; ++i) {
      if (pdl) launch<1>(s, d, n16, grid, st, true);
      else launch<0>(s, d, n16, grid, st, false);
    }
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    return ge;
  };
  cudaGraphExec_t g1 = capture(1, false);
  printf("graph1           %.3f us\n", per_us([&] { for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(g1, st)); }, reps, st));
  cudaGraphExec_t g1p = capture(1, true);
  printf("graph1_pdlkernel %.3f us\n", per_us([&] { for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(g1p, st)); }, reps, st));
  const int chain = 100;
  cudaGraphExec_t gc = capture(chain, false);
  printf("graph_chain      %.3f us\n", per_us([&] { for (int i = 0; i < reps / chain; ++i) CK(cudaGraphLaunch(gc, st)); }, reps, st));
  cudaGraphExec_t gcp = capture(chain, true);
  printf("graph_chain_pdl  %.3f us\n", per_us([&] { for (int i = 0; i < reps / chain; ++i) CK(cudaGraphLaunch(gcp, st)); }, reps, st));
  CK(cudaDeviceSynchronize());
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
