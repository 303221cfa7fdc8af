// Small-message latency of every implementation through the C ABI, from C++
// (no Python in the loop): the library's own control cost per collective.
//
//   tools/latency [nranks] [iters] [per_rank_streams] [impl-filter]
//     (env LAT_MIN / LAT_MAX / LAT_STEP: size grid, default 4 KiB..1 MiB x4)
//     (GPU box; ranks co-resident on GPU 0; per_rank_streams=1 gives every
//      rank its own stream: one unit per rank, flags between all of them)
//
// Prints CSV: api,impl,collective,size_bytes,device_us_b2b,device_us_isolated (median of 50),host_us,
// isolated_p10_us,isolated_p90_us (median plus p10 / p90)
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../include/cecoll.h"

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                       \
    }                                                                                     \
  } while (0)
#define CC(x)                                                                                \
  do {                                                                                       \
    cecoll_status_t s_ = (x);                                                                \
    if (s_ != CECOLL_SUCCESS) {                                                              \
      std::printf("cecoll error %s (%s) at %s:%d\n", cecoll_strerror(s_), cecoll_last_error(), \
                  __FILE__, __LINE__);                                                       \
      std::exit(1);                                                                          \
    }                                                                                        \
  } while (0)

int main(int argc, char** argv) {
  // As the Python package does: give the driver its maximum number of
  // hardware queues before the context exists.
  setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);
  const int n = argc > 1 ? std::atoi(argv[1]) : 8;
  const int iters = argc > 2 ? std::atoi(argv[2]) : 500;
  const bool per_rank = argc > 3 && std::atoi(argv[3]) != 0;
  const std::string only = argc > 4 ? argv[4] : "";
  CK(cudaSetDevice(0));
  std::vector<int> devs(n, 0);
  std::vector<cecoll_comm_t> comms(n);
  CC(cecoll_comm_init_all(comms.data(), n, devs.data()));
  cudaStream_t stream;
  CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  std::vector<void*> streams(n, stream);
  std::vector<cudaEvent_t> joins(n);
  for (int r = 0; r < n; ++r) {
    CK(cudaEventCreateWithFlags(&joins[r], cudaEventDisableTiming));
    if (per_rank && r > 0) {
      cudaStream_t sr;
      CK(cudaStreamCreateWithFlags(&sr, cudaStreamNonBlocking));
      streams[r] = sr;
    }
  }
  // Fork the rank streams off `stream` after e0 / join them before e1.
  auto fork = [&]() {
    if (!per_rank) return;
    CK(cudaEventRecord(joins[0], stream));
    for (int r = 1; r < n; ++r) CK(cudaStreamWaitEvent(static_cast<cudaStream_t>(streams[r]), joins[0], 0));
  };
  // Not cudaDeviceSynchronize: an armed prelaunch plan keeps its gate kernel
  // waiting on the device until the next launch.
  auto sync_all = [&]() {
    for (int r = 0; r < n; ++r) CK(cudaStreamSynchronize(static_cast<cudaStream_t>(streams[r])));
  };
  auto join = [&]() {
    if (!per_rank) return;
    for (int r = 1; r < n; ++r) {
      CK(cudaEventRecord(joins[r], static_cast<cudaStream_t>(streams[r])));
      CK(cudaStreamWaitEvent(stream, joins[r], 0));
    }
  };
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const size_t max_s = std::getenv("LAT_MAX") ? std::strtoull(std::getenv("LAT_MAX"), nullptr, 0) : size_t(1) << 20;
  // LAT_MIN / LAT_STEP: first size and multiplier of the size grid (4 KiB, x4)
  const size_t min_s = std::getenv("LAT_MIN") ? std::strtoull(std::getenv("LAT_MIN"), nullptr, 0) : size_t(4096);
  const size_t step = std::getenv("LAT_STEP") ? std::strtoull(std::getenv("LAT_STEP"), nullptr, 0) : size_t(4);
  std::vector<void*> send(n), recv(n);
  for (int r = 0; r < n; ++r) {
    CK(cudaMalloc(&send[r], n * max_s));
    CK(cudaMalloc(&recv[r], n * max_s));
    CK(cudaMemset(send[r], r, n * max_s));
  }
  std::printf("api,impl,collective,size_bytes,device_us_b2b,device_us_isolated,host_us,isolated_p10_us,isolated_p90_us\n");
  const char* names[] = {"sm", "pcpy", "b2b", "bcst", "swap", "prelaunch_pcpy", "prelaunch_b2b", "prelaunch_bcst",
                         "prelaunch_swap", "hybrid", "pull"};
  for (int kind = 0; kind < 2; ++kind) {
    for (size_t s = min_s; s <= max_s; s *= step) {
      for (const char* name : names) {
        if (!only.empty() && only != name) continue;
        const cecoll_impl_t impl = cecoll_parse_impl(name);
        if (!cecoll_impl_valid_for(impl, static_cast<cecoll_kind_t>(kind))) continue;
        const bool in_place = std::string(name).find("swap") != std::string::npos;
        std::vector<void*> rv = in_place ? send : recv;
        for (int api = 0; api < 2; ++api) {  // 0: plan, 1: eager collective_n
          cecoll_plan_t plan = nullptr;
          auto call = [&]() {
            if (api == 0) {
              CC(cecoll_plan_launch(plan, streams.data()));
            } else {
              CC(cecoll_collective_n(static_cast<cecoll_kind_t>(kind), comms.data(), n, send.data(), rv.data(), s,
                                     impl, streams.data()));
            }
          };
          if (api == 0)
            CC(cecoll_plan_create(comms.data(), n, static_cast<cecoll_kind_t>(kind), send.data(), rv.data(), s, impl,
                                  &plan));
          for (int i = 0; i < 10; ++i) call();
          sync_all();
          auto h0 = std::chrono::steady_clock::now();
          CK(cudaEventRecord(e0, stream));
          fork();
          for (int i = 0; i < iters; ++i) call();
          join();
          CK(cudaEventRecord(e1, stream));
          auto h1 = std::chrono::steady_clock::now();
          CK(cudaStreamSynchronize(stream));
          float ms_b2b = 0;
          CK(cudaEventElapsedTime(&ms_b2b, e0, e1));
          std::vector<float> iso;
          for (int i = 0; i < 50; ++i) {
            sync_all();
            CK(cudaEventRecord(e0, stream));
            fork();
            call();
            join();
            CK(cudaEventRecord(e1, stream));
            CK(cudaStreamSynchronize(stream));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            iso.push_back(ms);
          }
          std::sort(iso.begin(), iso.end());
          const double host_us = std::chrono::duration<double, std::micro>(h1 - h0).count() / iters;
          std::printf("%s,%s,%s,%zu,%.2f,%.2f,%.2f,%.2f,%.2f\n", api == 0 ? "plan" : "eager", name,
                      kind == 0 ? "allgather" : "alltoall", s, ms_b2b * 1000 / iters, iso[iso.size() / 2] * 1000,
                      host_us, iso[iso.size() / 10] * 1000, iso[iso.size() * 9 / 10] * 1000);
          std::fflush(stdout);
          if (plan) CC(cecoll_plan_destroy(plan));
          sync_all();
        }
      }
    }
  }
  // Reduce-scatter (bf16 sum, eager collective call): chunk s bytes per rank.
  const char* rs_names[] = {"sm", "pcpy", "b2b", "prelaunch_pcpy"};
  for (size_t s = min_s; s <= max_s; s *= step) {
    for (const char* name : rs_names) {
      if (!only.empty() && only != name) continue;
      const cecoll_impl_t impl = cecoll_parse_impl(name);
      const size_t count = s / 2;
      auto call = [&]() {
        CC(cecoll_reduce_scatter_n(comms.data(), n, send.data(), recv.data(), count, CECOLL_BF16, CECOLL_SUM, impl,
                                   streams.data()));
      };
      for (int i = 0; i < 10; ++i) call();
      sync_all();
      auto h0 = std::chrono::steady_clock::now();
      CK(cudaEventRecord(e0, stream));
      fork();
      for (int i = 0; i < iters; ++i) call();
      join();
      CK(cudaEventRecord(e1, stream));
      auto h1 = std::chrono::steady_clock::now();
      CK(cudaStreamSynchronize(stream));
      float ms_b2b = 0;
      CK(cudaEventElapsedTime(&ms_b2b, e0, e1));
      std::vector<float> iso;
      for (int i = 0; i < 50; ++i) {
        sync_all();
        CK(cudaEventRecord(e0, stream));
        fork();
        call();
        join();
        CK(cudaEventRecord(e1, stream));
        CK(cudaStreamSynchronize(stream));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        iso.push_back(ms);
      }
      std::sort(iso.begin(), iso.end());
      const double host_us = std::chrono::duration<double, std::micro>(h1 - h0).count() / iters;
      std::printf("eager,%s,reduce_scatter_bf16_sum,%zu,%.2f,%.2f,%.2f,%.2f,%.2f\n", name, s, ms_b2b * 1000 / iters,
                  iso[iso.size() / 2] * 1000, host_us, iso[iso.size() / 10] * 1000, iso[iso.size() * 9 / 10] * 1000);
      std::fflush(stdout);
      sync_all();
    }
  }
  for (auto c : comms) CC(cecoll_comm_destroy(c));
  return 0;
}
