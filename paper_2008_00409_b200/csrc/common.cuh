// common.cuh — shared device/host infrastructure for libweft_gpu.so.
//
// The whole library is compiled with -fmad=false: every FP64 expression is
// evaluated as separately rounded multiplies and adds in the association the
// reference uses (see oracle/shim/Eigen/Dense), which is what makes the
// assembled matrix and the SpMV bitwise equal to the CPU reference.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/weft_gpu.h"

namespace weft_gpu {

// Error carrying a weft_status; converted at the C-ABI boundary.
struct Error : std::runtime_error {
  weft_status status;
  Error(weft_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void cuda_check(cudaError_t e, const char* what, int device) {
  if (e != cudaSuccess) {
    // ExecError wording of the reference (proj/src/exec.cpp:164).
    throw Error(WEFT_ERR_EXEC, "device " + std::to_string(device) + " failed: " + what + ": " +
                                   cudaGetErrorString(e));
  }
}

#define WG_CUDA(call) ::weft_gpu::cuda_check((call), #call, ::weft_gpu::current_device())

inline int current_device() {
  int d = -1;
  cudaGetDevice(&d);
  return d;
}

// Growable device buffer (capacity never shrinks; memory is plentiful on a
// 180 GB part, re-allocation per step is not).
template <class T>
struct DBuf {
  T* ptr = nullptr;
  size_t cap = 0;
  size_t n = 0;
  bool ext = false;  // view of memory owned elsewhere (the peer window)
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (ptr && !ext) cudaFree(ptr);
  }
  // Turns the buffer into a fixed-capacity view of `count` elements at p.
  void attach(T* p, size_t count) {
    if (ptr && !ext) cudaFree(ptr);
    ptr = p;
    cap = n = count;
    ext = true;
  }
  void resize(size_t count) {
    if (count > cap) {
      if (ext) throw std::runtime_error("window buffer too small (vertex count changed after weft_gpu_comm_export)");
      if (ptr) WG_CUDA(cudaFree(ptr));
      ptr = nullptr;
      size_t c = count + count / 8 + 16;
      WG_CUDA(cudaMalloc(&ptr, c * sizeof(T)));
      cap = c;
    }
    n = count;
  }
  T* data() const { return ptr; }
  size_t size() const { return n; }
  size_t bytes() const { return n * sizeof(T); }
  void upload(const T* src, size_t count, cudaStream_t s) {
    resize(count);
    if (count) WG_CUDA(cudaMemcpyAsync(ptr, src, count * sizeof(T), cudaMemcpyDefault, s));
  }
  void download(T* dst, size_t count, cudaStream_t s) const {
    if (count) WG_CUDA(cudaMemcpyAsync(dst, ptr, count * sizeof(T), cudaMemcpyDefault, s));
  }
  void zero(cudaStream_t s) {
    if (n) WG_CUDA(cudaMemsetAsync(ptr, 0, n * sizeof(T), s));
  }
};

constexpr int kSlice = 32;  // sliced-ELL slice height (one warp of rows)
constexpr int kMaxParts = 8;

// PartitionMap::owner (proj/include/weft/assembly.hpp:27-31).
struct PartMap {
  int p = 0, n = 1, base = 0, extra = 0;
  __host__ __device__ int owner(int v) const {
    const int split = extra * (base + 1);
    if (v < split) return v / (base + 1);
    return extra + (v - split) / (base > 1 ? base : 1);
  }
  __host__ __device__ int begin(int d) const { return d * base + (d < extra ? d : extra); }
  __host__ __device__ int end(int d) const { return begin(d) + base + (d < extra ? 1 : 0); }
  static PartMap make(int p, int n) {
    PartMap m;
    m.p = p;
    m.n = n;
    m.base = p / n;
    m.extra = p % n;
    return m;
  }
};

// Per-partition processing order of column owners: qpos[d][o] = position of
// owner o in device d's accumulation order (0 = own sub-block, k = k-th
// work-queue node; proj/include/weft/sparse.hpp:89-95).
struct GroupOrder {
  int n = 1;
  int8_t qpos[kMaxParts][kMaxParts];
};

inline int div_up(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// ---------------------------------------------------------------------------
// Peer-memory synchronisation between ranks (one process per GPU, windows
// mapped through CUDA IPC; NVLink P2P on a multi-GPU node). Flags are
// monotonically increasing 64-bit sequence numbers written by their owner
// rank with a system-scope release and polled with a system-scope acquire.
// ---------------------------------------------------------------------------
constexpr int kMaxRanks = 8;
constexpr unsigned long long kSpinTimeoutNs = 30ull * 1000 * 1000 * 1000;  // 30 s

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spins until *flag >= target; false after kSpinTimeoutNs (a dead peer must
// not hang the GPU: the caller records the failure and the host throws).
__device__ __forceinline__ bool wait_flag(const unsigned long long* flag, unsigned long long target) {
  if (ld_acquire_sys(flag) >= target) return true;
  const unsigned long long t0 = global_ns();
  for (;;) {
    __nanosleep(64);
    if (ld_acquire_sys(flag) >= target) return true;
    if (global_ns() - t0 > kSpinTimeoutNs) return false;
  }
}

// The peer-visible part of a rank's context (one cudaMalloc, exported as a
// CUDA IPC handle). Written remotely by peers: the ready flags (slot = the
// writer's rank) and the reduction slots of the writer's partitions.
struct CommHeader {
  unsigned long long vec_ready[kMaxRanks];    // PCG / SpMV gather vectors published
  unsigned long long red_ready[kMaxRanks];    // reduction partials published
  unsigned long long state_ready[kMaxRanks];  // sim state (v, x_cand) rows published
  unsigned long long hits_ready[kMaxRanks];   // narrow-phase hits of the writer's share published
  long long hit_count[kMaxRanks];             // ... their count (unique within the share)
  long long pair_count[kMaxRanks];            // ... and the share's candidate pairs
  double red[2][kMaxParts][4];                // [sequence parity][partition][value]
};

// Kernel-side view of the rank group (by value in kernel arguments).
struct CommView {
  int world = 1, rank = 0;
  int ppr = 1;                            // partitions per rank
  CommHeader* hdr[kMaxRanks] = {};        // every rank's header (own = local)
  const double* z[kMaxRanks] = {};        // every rank's gather vectors (global row index)
  const double* p[kMaxRanks] = {};
  char* base[kMaxRanks] = {};             // every rank's window base
  unsigned long long* seq = nullptr;      // own counters: [0] vec, [1] red, [2] state, [3] error, [4] hits
};

}  // namespace weft_gpu
