// B200 phase latencies in the reference's cost-model vocabulary
// (proj/include/dmasim/cost_model.hpp:14-33): measures each phase of one
// copy offload on this GPU/driver/host and prints a key=value file that the
// reference's load_cost_model() accepts (cost_model.cpp:77-123), so that the
// reference simulator can be re-run with B200 parameters.
//
//   tools/phase_probe > profiles/b200_cost_model.conf
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <vector>
#include <unistd.h>

#include "../paper_2511_06605_b200/csrc/cu_driver.hpp"

using namespace cecoll;

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

static double now_ns() {
  return std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  alarm(120);
  const DriverApi* d = driver_api();
  if (!d) return 1;
  CK(cudaSetDevice(0));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  char *src, *dst;
  CK(cudaMalloc(&src, 1 << 20));
  CK(cudaMalloc(&dst, 1 << 20));
  uint64_t* host;
  CK(cudaHostAlloc(&host, 4096, cudaHostAllocMapped));
  uint64_t* hdev;
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hdev), host, 0));
  volatile uint64_t* h = host;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int K = 400;
  uint64_t gate = 0;

  // Block the stream on a host gate so that enqueue cost (host) and execution
  // cost (device) are measured separately.
  auto block = [&]() {
    ++gate;
    d->StreamWaitValue64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(hdev), gate,
                         CU_STREAM_WAIT_VALUE_GEQ);
  };
  auto release = [&]() { h[0] = gate; };

  // t_ctl: host cost of creating + enqueueing one copy command.
  block();
  CK(cudaEventRecord(e0, s));
  double t0 = now_ns();
  for (int i = 0; i < K; ++i) CK(cudaMemcpyAsync(dst, src, 4096, cudaMemcpyDeviceToDevice, s));
  double t_ctl = (now_ns() - t0) / K;
  CK(cudaEventRecord(e1, s));
  release();
  CK(cudaStreamSynchronize(s));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  // fetch + fixed per 4 KiB copy executed back to back (host far ahead).
  const double t_copy_fixed = ms * 1e6 / K;

  // t_sig: device cost of one signal (stream memory write).
  block();
  CK(cudaEventRecord(e0, s));
  for (int i = 0; i < K; ++i)
    d->StreamWriteValue64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(hdev + 8), i, 0);
  CK(cudaEventRecord(e1, s));
  release();
  CK(cudaStreamSynchronize(s));
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double t_sig = ms * 1e6 / K;

  // Trigger -> poll -> copy -> signal -> host observe round trip (prelaunch
  // chain), with the poll armed well ahead.
  std::vector<double> rt;
  for (int i = 0; i < 200; ++i) {
    block();
    CK(cudaMemcpyAsync(dst, src, 4096, cudaMemcpyDeviceToDevice, s));
    d->StreamWriteValue64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(hdev + 16), gate, 0);
    usleep(300);
    const double a = now_ns();
    release();
    while (h[16] < gate) {
    }
    rt.push_back(now_ns() - a);
  }
  CK(cudaStreamSynchronize(s));
  std::sort(rt.begin(), rt.end());
  const double roundtrip = rt[rt.size() / 2];
  // Same chain without the copy: isolates the poll latency + signal + observe.
  std::vector<double> rt2;
  for (int i = 0; i < 200; ++i) {
    block();
    d->StreamWriteValue64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(hdev + 16), gate, 0);
    usleep(300);
    const double a = now_ns();
    release();
    while (h[16] < gate) {
    }
    rt2.push_back(now_ns() - a);
  }
  CK(cudaStreamSynchronize(s));
  std::sort(rt2.begin(), rt2.end());
  const double flag_rt = rt2[rt2.size() / 2];
  // Host scan of an additional completion slot and a trigger write.
  double scan0 = now_ns();
  uint64_t acc = 0;
  for (int i = 0; i < 100000; ++i) acc += h[(i % 64) + 64];
  const double t_scan = (now_ns() - scan0) / 100000;
  double trig0 = now_ns();
  for (int i = 0; i < 100000; ++i) h[200 + (i % 64)] = i;
  const double t_trig = (now_ns() - trig0) / 100000;

  // Split the flag round trip: poll wake-up, signal, host observation.
  const double t_poll_lat = (flag_rt - t_sig) / 2;
  const double t_obs = flag_rt - t_sig - t_poll_lat;
  // Copy engine cap: a single large same-device copy stream.
  CK(cudaFree(dst));
  CK(cudaFree(src));
  const size_t big = size_t{1} << 30;
  CK(cudaMalloc(&src, big));
  CK(cudaMalloc(&dst, big));
  CK(cudaMemcpyAsync(dst, src, big, cudaMemcpyDeviceToDevice, s));
  CK(cudaEventRecord(e0, s));
  CK(cudaMemcpyAsync(dst, src, big, cudaMemcpyDeviceToDevice, s));
  CK(cudaEventRecord(e1, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double cap = big / (ms * 1e-3);

  printf("# B200 phase latencies measured by tools/phase_probe.cu (one GPU, same-device copies)\n");
  printf("# copy+signal+observe round trip after a host trigger: %.0f ns; flag-only round trip: %.0f ns\n",
         roundtrip, flag_rt);
  printf("# t_db folded into t_ctl (a CUDA enqueue rings its own doorbell); t_fetch folded into t_copy_fixed\n");
  printf("t_ctl_ns=%.1f\n", t_ctl);
  printf("t_db_ns=0\n");
  printf("t_fetch_ns=0\n");
  printf("t_copy_fixed_ns=%.1f\n", t_copy_fixed);
  printf("t_sig_ns=%.1f\n", t_sig);
  printf("t_obs_ns=%.1f\n", t_obs);
  printf("t_scan_ns=%.1f\n", t_scan);
  printf("t_trig_ns=%.1f\n", t_trig);
  printf("t_poll_lat_ns=%.1f\n", t_poll_lat);
  printf("engine_throughput_cap_bytes_per_s=%.6g\n", cap);
  printf("# acc=%llu\n", (unsigned long long)acc);
  return 0;
}
