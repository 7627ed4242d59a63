// ipc_probe.cu — checks that two processes sharing ONE GPU make progress
// when a kernel of one spins on a flag the other writes through CUDA IPC
// memory (time-sliced contexts), and measures the ping-pong round trip.
// This is the mechanism the multi-rank PCG uses for its halo / reduction
// flags; on one gpurun box (1 GPU) it is how the N>1 path is exercised.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/ipc_probe tools/ipc_probe.cu
//   /tmp/ipc_probe 0 /tmp/h & /tmp/ipc_probe 1 /tmp/h
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <thread>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

// flags[0] written by rank 0, flags[1] by rank 1 (both live in rank 0's memory)
__global__ void pingpong(unsigned* flags, int rank, int rounds, long long timeout_cycles, int* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const long long t0 = clock64();
  for (int k = 1; k <= rounds; ++k) {
    if (rank == 0) {
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flags), "r"((unsigned)k) : "memory");
    }
    unsigned v = 0;
    unsigned* wait_on = rank == 0 ? flags + 1 : flags;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(wait_on) : "memory");
      if (clock64() - t0 > timeout_cycles) {
        *status = -k;
        return;
      }
    } while (v < (unsigned)k);
    if (rank == 1) {
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flags + 1), "r"((unsigned)k) : "memory");
    }
  }
  *status = rounds;
}

int main(int argc, char** argv) {
  const int rank = atoi(argv[1]);
  const char* path = argv[2];
  const int rounds = argc > 3 ? atoi(argv[3]) : 200;
  CK(cudaSetDevice(0));
  unsigned* flags = nullptr;
  if (rank == 0) {
    CK(cudaMalloc(&flags, 256));
    CK(cudaMemset(flags, 0, 256));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, flags));
    std::ofstream f(std::string(path) + ".tmp", std::ios::binary);
    f.write(reinterpret_cast<const char*>(&h), sizeof(h));
    f.close();
    std::rename((std::string(path) + ".tmp").c_str(), path);
  } else {
    cudaIpcMemHandle_t h;
    for (;;) {
      std::ifstream f(path, std::ios::binary);
      if (f && f.read(reinterpret_cast<char*>(&h), sizeof(h))) break;
      std::this_thread::sleep_for(std::chrono::milliseconds(10));
    }
    CK(cudaIpcOpenMemHandle(reinterpret_cast<void**>(&flags), h, cudaIpcMemLazyEnablePeerAccess));
  }
  int* status;
  CK(cudaMallocManaged(&status, sizeof(int)));
  *status = 0;
  const auto t0 = std::chrono::steady_clock::now();
  pingpong<<<1, 32>>>(flags, rank, rounds, 20LL * 2000000000LL, status);
  CK(cudaDeviceSynchronize());
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  printf("rank %d: status %d (rounds %d) in %.1f ms -> %.3f ms per round trip\n", rank, *status, rounds, ms,
         ms / rounds);
  if (rank == 0) {
    std::this_thread::sleep_for(std::chrono::milliseconds(500));
    std::remove(path);
  }
  return *status == rounds ? 0 : 2;
}
