// Multi-process self-test of the C ABI from C++ alone (no Python, no torch):
// N forked processes, one rank each (GPU rank % device_count), exchange their
// init / registration blobs through POSIX shared memory with a
// process-shared barrier (the cecoll_exchange_fn contract), register a
// library-owned window (cecoll_mem_alloc), and run all-to-all and all-gather
// through every implementation — three calls each, so recorded command lists
// replay — checking every byte against the rank/chunk layout
// (compiler.cpp:115-126).
//
//   tools/mp_selftest [nprocs] [chunk_bytes]      exit code = failures
#include <cuda_runtime.h>
#include <pthread.h>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../include/cecoll.h"

namespace {

constexpr int kMaxProcs = 32;
constexpr size_t kSlot = 4096;

struct Shared {
  pthread_barrier_t barrier;
  char slots[kMaxProcs][kSlot];
};

struct Ctx {
  Shared* shm;
  int rank, nprocs;
};

// All-gather of one fixed-size blob per process (cecoll_exchange_fn).
int exchange(void* ctx, const void* mine, size_t bytes, void* all) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (bytes > kSlot) return 1;
  std::memcpy(c->shm->slots[c->rank], mine, bytes);
  pthread_barrier_wait(&c->shm->barrier);
  for (int p = 0; p < c->nprocs; ++p) std::memcpy(static_cast<char*>(all) + p * bytes, c->shm->slots[p], bytes);
  pthread_barrier_wait(&c->shm->barrier);
  return 0;
}

void barrier(Ctx* c) { pthread_barrier_wait(&c->shm->barrier); }

// Byte k of the chunk rank i sends to rank j (all-gather: j = 0).
uint8_t pattern(int i, int j, int64_t k, int salt) {
  uint64_t z = (static_cast<uint64_t>(i) << 48) ^ (static_cast<uint64_t>(j) << 40) ^ static_cast<uint64_t>(k / 8) ^
               (static_cast<uint64_t>(salt) << 56);
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  return static_cast<uint8_t>(z >> (8 * (k % 8)));
}

#define CK(x)                                                                                     \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) {                                                                      \
      std::fprintf(stderr, "rank %d: CUDA %s at %s:%d\n", c.rank, cudaGetErrorString(e_), __FILE__, \
                   __LINE__);                                                                     \
      return 100;                                                                                 \
    }                                                                                             \
  } while (0)

int child(Ctx c, int64_t s) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const int dev = c.rank % ndev;
  CK(cudaSetDevice(dev));
  const int n = c.nprocs;
  cecoll_comm_t comm;
  if (cecoll_comm_init_rank(&comm, n, c.rank, dev, exchange, &c) != CECOLL_SUCCESS) {
    std::fprintf(stderr, "rank %d: init: %s\n", c.rank, cecoll_last_error());
    return 101;
  }
  void* win = nullptr;  // [send n*s | recv n*s], registered on every rank (collective)
  if (cecoll_mem_alloc(comm, static_cast<size_t>(2 * n * s), &win) != CECOLL_SUCCESS) {
    std::fprintf(stderr, "rank %d: mem_alloc: %s\n", c.rank, cecoll_last_error());
    return 102;
  }
  char* send = static_cast<char*>(win);
  char* recv = send + n * s;
  cudaStream_t stream;
  CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  std::vector<uint8_t> host(static_cast<size_t>(n * s)), got(static_cast<size_t>(n * s));
  const char* impls[] = {"sm", "pcpy", "b2b", "hybrid", "pull", "prelaunch_pcpy", "prelaunch_b2b", "bcst", "swap"};
  int failures = 0;
  for (int kind = 0; kind < 2; ++kind) {
    for (const char* name : impls) {
      const cecoll_impl_t impl = cecoll_parse_impl(name);
      if (!cecoll_impl_valid_for(impl, static_cast<cecoll_kind_t>(kind))) continue;
      const bool in_place = std::string(name).find("swap") != std::string::npos;
      const int64_t in_bytes = kind == CECOLL_ALLGATHER ? s : n * s;
      bool ok = true;
      for (int call = 0; call < 3 && ok; ++call) {
        const int salt = call + 3 * kind;
        for (int64_t k = 0; k < in_bytes; ++k)
          host[k] = kind == CECOLL_ALLGATHER ? pattern(c.rank, 0, k, salt) : pattern(c.rank, static_cast<int>(k / s), k % s, salt);
        CK(cudaMemcpy(in_place ? recv : send, host.data(), in_bytes, cudaMemcpyHostToDevice));
        if (!in_place) CK(cudaMemset(recv, 0xA5, n * s));
        CK(cudaDeviceSynchronize());
        barrier(&c);  // every rank's input is in place before anyone's collective
        const cecoll_status_t st = kind == CECOLL_ALLGATHER
                                       ? cecoll_allgather(send, recv, s, impl, comm, stream)
                                       : cecoll_alltoall(in_place ? recv : send, recv, s, impl, comm, stream);
        if (st != CECOLL_SUCCESS) {
          std::fprintf(stderr, "rank %d: %s: %s\n", c.rank, name, cecoll_last_error());
          ok = false;
        }
        CK(cudaStreamSynchronize(stream));
        barrier(&c);  // every rank done reading before inputs change
        CK(cudaMemcpy(got.data(), recv, n * s, cudaMemcpyDeviceToHost));
        for (int i = 0; i < n && ok; ++i)
          for (int64_t k = 0; k < s; ++k) {
            const uint8_t want = kind == CECOLL_ALLGATHER ? pattern(i, 0, k, salt) : pattern(i, c.rank, k, salt);
            if (got[i * s + k] != want) {
              std::fprintf(stderr, "rank %d: %s %s call %d: slot %d byte %lld differs\n", c.rank,
                           kind ? "alltoall" : "allgather", name, call, i, static_cast<long long>(k));
              ok = false;
              break;
            }
          }
      }
      if (c.rank == 0) {
        std::printf("%-9s %-15s %s\n", kind ? "alltoall" : "allgather", name, ok ? "PASS" : "FAIL");
        std::fflush(stdout);  // the child leaves through _exit
      }
      failures += ok ? 0 : 1;
    }
  }
  // Measured selection from C (cecoll_tune, csrc/tune.cpp): every process
  // must install the same table (times agreed through the exchange).
  {
    bool ok = cecoll_tune(&comm, 1, 65536, nullptr) == CECOLL_SUCCESS;
    std::string table;
    if (ok) {
      size_t len = 0;
      cecoll_tune_table(comm, nullptr, 0, &len);
      table.assign(len, '\0');
      cecoll_tune_table(comm, &table[0], len, &len);
      table.resize(std::strlen(table.c_str()));
    } else {
      std::fprintf(stderr, "rank %d: tune: %s\n", c.rank, cecoll_last_error());
    }
    uint64_t h = 1469598103934665603ull;  // FNV-1a of the table text
    for (char ch : table) h = (h ^ static_cast<uint8_t>(ch)) * 1099511628211ull;
    std::vector<uint64_t> all(static_cast<size_t>(n));
    exchange(&c, &h, sizeof(h), all.data());
    for (uint64_t x : all) ok &= x == all[0];
    ok &= std::count(table.begin(), table.end(), '\n') == 6;  // 4, 16, 64 KiB for both collectives
    if (c.rank == 0) {
      std::printf("%-9s %-15s %s\n", "tune", "same table", ok ? "PASS" : "FAIL");
      std::fflush(stdout);
    }
    failures += ok ? 0 : 1;
  }
  CK(cudaStreamDestroy(stream));
  cecoll_mem_free(comm, win);
  cecoll_comm_destroy(comm);
  return failures;
}

}  // namespace

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 2;
  const int64_t s = argc > 2 ? std::atoll(argv[2]) : 65536 + 48;
  if (n < 2 || n > kMaxProcs) return 2;
  setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);  // before any CUDA call
  auto* shm = static_cast<Shared*>(
      mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED | MAP_ANONYMOUS, -1, 0));
  if (shm == MAP_FAILED) return 3;
  pthread_barrierattr_t attr;
  pthread_barrierattr_init(&attr);
  pthread_barrierattr_setpshared(&attr, PTHREAD_PROCESS_SHARED);
  pthread_barrier_init(&shm->barrier, &attr, static_cast<unsigned>(n));
  std::vector<pid_t> kids;
  for (int r = 0; r < n; ++r) {
    const pid_t pid = fork();
    if (pid == 0) _exit(child(Ctx{shm, r, n}, s));  // no CUDA in the parent: fork is safe
    kids.push_back(pid);
  }
  int failures = 0;
  for (pid_t pid : kids) {
    int status = 0;
    waitpid(pid, &status, 0);
    failures += WIFEXITED(status) ? WEXITSTATUS(status) : 1;
  }
  std::printf("mp_selftest: %d processes, chunk %lld bytes: %s\n", n, static_cast<long long>(s),
              failures ? "FAILED" : "all implementations bit-exact");
  return failures ? 1 : 0;
}
