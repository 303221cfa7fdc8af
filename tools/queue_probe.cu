// Does an armed gated graph block other streams that share its hardware
// queue? A graph (gate kernel spinning on a word -> second kernel) is launched
// on an "arm" stream; then the word is written with a stream memory
// operation from each of 64 fresh streams in turn (more streams than the 32
// hardware queues of CUDA_DEVICE_MAX_CONNECTIONS=32, so some share the arm
// stream's queue). A write that has not landed after 200 ms is counted as
// blocked; the host then releases the gate itself (the word is pinned host
// memory) and the stream's write completes later.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/queue_probe.cu -o tools/queue_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>

__global__ void gate(volatile uint64_t* w, uint64_t want) {
  if (threadIdx.x == 0)
    while (*w < want) __nanosleep(100);
}
__global__ void body(int* x) {
  if (threadIdx.x == 0) ++*x;
}

int main(int argc, char** argv) {
  const bool plain = argc > 1 && argv[1][0] == 'p';  // two kernel launches instead of a graph
  setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 1);
  cuInit(0);
  cudaSetDevice(0);
  volatile uint64_t* w;
  cudaHostAlloc((void**)&w, 64, cudaHostAllocMapped);
  *w = 0;
  uint64_t* wd;
  cudaHostGetDevicePointer((void**)&wd, (void*)w, 0);
  int* x;
  cudaMalloc(&x, 4);
  cudaStream_t arm;
  cudaStreamCreateWithFlags(&arm, cudaStreamNonBlocking);
  int blocked = 0, tried = 0;
  for (int i = 0; i < 64; ++i) {
    const uint64_t want = i + 1;
    cudaGraphExec_t ge = nullptr;
    if (!plain) {
      cudaGraph_t g;
      cudaStreamBeginCapture(arm, cudaStreamCaptureModeRelaxed);
      gate<<<1, 32, 0, arm>>>(w, want);
      body<<<1, 32, 0, arm>>>(x);
      cudaStreamEndCapture(arm, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, arm);
    } else {
      gate<<<1, 32, 0, arm>>>(w, want);
      body<<<1, 32, 0, arm>>>(x);
    }
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cuStreamWriteValue64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(wd), want, 0);
    auto t0 = std::chrono::steady_clock::now();
    bool done = false;
    while (std::chrono::steady_clock::now() - t0 < std::chrono::milliseconds(200)) {
      if (cudaStreamQuery(arm) == cudaSuccess) {
        done = true;
        break;
      }
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    ++tried;
    if (!done) {
      ++blocked;
      std::printf("stream %d: write did not land within 200 ms (shares the armed queue?)\n", i);
      *w = want;  // release from the host
    }
    cudaStreamSynchronize(arm);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (ge) cudaGraphExecDestroy(ge);
  }
  std::printf("%s: %d of %d trigger streams blocked behind the armed %s\n", plain ? "plain launches" : "graph",
              blocked, tried, plain ? "kernels" : "graph");
  std::printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
