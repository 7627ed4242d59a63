// sparse.cu — sliced-ELL 3x3-block matrix, SpMV and block-Jacobi PCG.
//
// Reference: BellMatrix::multiply_into/accumulate (proj/src/bell.cpp:87-129),
// spmv_pipelined (proj/include/weft/sparse.hpp:72-101) and pcg_solve
// (proj/include/weft/solver.hpp:36-178).
//
// SpMV is HBM-bound (~0.2 FLOP/B): one thread per block row walks its slots
// (coalesced 256-byte plane loads per warp per component), gathers x from
// L2, and keeps the reference's per-row order exactly: a fresh partial sum
// per partition group, the own group assigned first, the others added in
// work-queue order. The PCG is device-driven: two kernels per iteration,
// (1) SpMV with the search direction p = z + beta p formed on the fly and
// the p.q partial fused into the epilogue, the last block finalising alpha;
// (2) the x/r update, block-Jacobi z = D^-1 r and the r.r / r.z partials,
// the last block finalising the residual test and beta. Dot products are
// reduced per partition in a fixed tree and then summed in ascending
// partition order (Engine::all_reduce_sum, proj/src/exec.cpp:170-174).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include <cooperative_groups.h>

#include <type_traits>

#include "ctx.cuh"

namespace weft_gpu {

// ---------------------------------------------------------------------------
// Matrix view passed to kernels
// ---------------------------------------------------------------------------
struct SellView {
  int rows;  // held rows; the matrix is addressed by POSITION m (SELL-32-sigma),
             // local row perm[m], global row row0 + perm[m]
  int row0;
  int64_t total;
  const int64_t* __restrict__ slice_off;
  const int32_t* __restrict__ rowlen;
  const int32_t* __restrict__ cols;
  const double* __restrict__ vals;
  const int32_t* __restrict__ perm;  // matrix position -> local row
  const float* __restrict__ vals32;  // Precision::Single systems: the values as float
};

static SellView view(const SellMatrix& A) {
  return SellView{A.rows,        A.row0,       A.total,       A.slice_off.data(), A.rowlen.data(),
                  A.cols.data(), A.vals.data(), A.perm.data(), A.vals32.data()};
}

// The value planes of a system in Real = T (driver.hpp:13: Precision::Double
// runs on doubles, Precision::Single on floats).
template <class T>
__device__ __forceinline__ const T* sell_vals(const SellView& A) {
  if constexpr (std::is_same_v<T, float>) return A.vals32;
  else return A.vals;
}

// Blocks are aligned to partitions so that every block's dot partial
// belongs to exactly one partition.
struct PartBlocks {
  int n;   // partitions held by this rank
  int d0;  // global index of the first one
  int bstart[kMaxParts + 1];
  int rbegin[kMaxParts];
  int rend[kMaxParts];
};

static PartBlocks part_blocks(const Ctx& c, int threads) {
  PartBlocks pb{};
  pb.n = c.part_end - c.part_begin;
  pb.d0 = c.part_begin;
  pb.bstart[0] = 0;
  for (int d = 0; d < pb.n; ++d) {
    pb.rbegin[d] = c.pm.begin(pb.d0 + d);
    pb.rend[d] = c.pm.end(pb.d0 + d);
    pb.bstart[d + 1] = pb.bstart[d] + div_up(pb.rend[d] - pb.rbegin[d], threads);
  }
  return pb;
}

__device__ __forceinline__ int block_part(const PartBlocks& pb, int b) {
  int d = 0;
  while (d + 1 < pb.n && b >= pb.bstart[d + 1]) ++d;
  return d;
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// evict_last for a fraction of the lines (by address), evict_unchanged for
// the rest: the gathered vectors keep at most ~60 MB of L2 pinned when they
// are larger than that (frac < 1 from the host, PcgArgs::vec_el_frac).
__device__ __forceinline__ uint64_t l2_policy_evict_last_frac(float frac) {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.L2::evict_unchanged.b64 %0, %1;" : "=l"(pol) : "f"(frac));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double ld_nc_hint(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_nc_hint(const int* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_nc_hint(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_nc_hint(const int16_t* p, uint64_t pol) {
  short v;
  asm volatile("ld.global.nc.L2::cache_hint.s16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_cg_hint(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_cg_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.cg.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ double ld_hint(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
// Single-group row products of the multi-kernel path (k_spmv, k_pcg_spmv:
// one partition, or the interior rows of a rank): the same L2 priorities as
// the persistent kernel (matrix evict_first, gathered vector evict_last).
// Measured on B200, config D, graph PCG: 259 -> 229 us per iteration; the
// multi-group row product measured 3 % slower with them, so it keeps plain
// loads (tools/pcg_ab.py, WEFT_SPMV_HINT=0 turns them off).
#ifndef WEFT_SPMV_HINT
#define WEFT_SPMV_HINT 1
#endif
#if WEFT_SPMV_HINT
#define SP_POLICIES                                  \
  const uint64_t mpol = l2_policy_evict_first(); \
  const uint64_t vpol = l2_policy_evict_last();
#define SP_MLD(p) ld_nc_hint(p, mpol)
#define SP_XLD(p) ld_hint(p, vpol)
#else
#define SP_POLICIES
#define SP_MLD(p) __ldg(p)
#define SP_XLD(p) (*(p))
#endif

// ---------------------------------------------------------------------------
// Row product in the reference order
// ---------------------------------------------------------------------------
// Gathers x[c] (+ beta * pold[c] for PMode 2) for column c. Columns of
// another rank (kRemote, only reached for accumulation groups != 0) are read
// over peer memory once that rank has published the vectors
// (vec_ready >= vexp); `seen` caches which ranks were already waited for.
template <int PMode, bool kRemote, bool kCg = false, class T = double>
__device__ __forceinline__ void gather3(int c, int g, const T* __restrict__ x, const T* __restrict__ pold,
                                        T beta, const CommView& cv, const PartMap& pm, unsigned long long vexp,
                                        unsigned& seen, T& x0, T& x1, T& x2) {
  if constexpr (kRemote && std::is_same_v<T, double>) {
   if (g != 0) {
    const int q = pm.owner(c) / cv.ppr;
    if (q != cv.rank) {
      if (!(seen & (1u << q))) {
        if (!wait_flag(&cv.hdr[cv.rank]->vec_ready[q], vexp)) atomicExch(cv.seq + 3, 1ull);
        seen |= 1u << q;
      }
      const double* zq = cv.z[q];
      x0 = __ldcg(zq + 3 * c);
      x1 = __ldcg(zq + 3 * c + 1);
      x2 = __ldcg(zq + 3 * c + 2);
      if (PMode == 2) {
        const double* pq = cv.p[q];
        x0 = x0 + beta * __ldcg(pq + 3 * c);
        x1 = x1 + beta * __ldcg(pq + 3 * c + 1);
        x2 = x2 + beta * __ldcg(pq + 3 * c + 2);
      }
      return;
    }
   }
  }
  if constexpr (kCg) {  // vectors written earlier in the same (persistent) kernel
    x0 = __ldcg(x + 3 * c);
    x1 = __ldcg(x + 3 * c + 1);
    x2 = __ldcg(x + 3 * c + 2);
    if (PMode == 2) {
      x0 = x0 + beta * __ldcg(pold + 3 * c);
      x1 = x1 + beta * __ldcg(pold + 3 * c + 1);
      x2 = x2 + beta * __ldcg(pold + 3 * c + 2);
    }
    return;
  }
  x0 = x[3 * c];
  x1 = x[3 * c + 1];
  x2 = x[3 * c + 2];
  if (PMode == 2) {
    x0 = x0 + beta * pold[3 * c];
    x1 = x1 + beta * pold[3 * c + 1];
    x2 = x2 + beta * pold[3 * c + 2];
  }
}

#ifndef WEFT_MG_UNROLL
#define WEFT_MG_UNROLL 2
#endif
constexpr int kMgUnroll = WEFT_MG_UNROLL;  // slots per trip of the multi-group row loop

// Row product of LOCAL row lr in the reference order.
// PMode 0: x given. PMode 1: x = z (first PCG iteration, p = z).
// PMode 2: x = z + beta * p_old on the fly (PCG p update).
// T = float: Precision::Single (bell.cpp:87-129 with Real = float; beta is
// cast to Real as the p update of solver.hpp:166 does).
template <int PMode, bool kRemote = false, bool kCg = false, class T = double>
__device__ __forceinline__ void row_product(const SellView& A, int lr, int ngroups, const T* __restrict__ x,
                                            const T* __restrict__ pold, double beta_d, T& y0, T& y1,
                                            T& y2, const CommView& cv = CommView(), const PartMap& pm = PartMap(),
                                            unsigned long long vexp = 0) {
  const T beta = static_cast<T>(beta_d);
  const int len = A.rowlen[lr];
  const int64_t base = A.slice_off[lr >> 5] + (lr & 31);
  const T* __restrict__ vals = sell_vals<T>(A);
  T a0 = 0, a1 = 0, a2 = 0;
  int cg = 0;
  unsigned seen = 0;
  y0 = y1 = y2 = 0.0;
  // the column word of slot k+1 is fetched while slot k is processed, so a
  // slot's gathers only wait on their own round trip (as row_product_1)
  int pn = len > 0 ? __ldg(A.cols + base) : 0;
#pragma unroll kMgUnroll
  for (int k = 0; k < len; ++k) {
    const int64_t at = base + (int64_t)k * kSlice;
    const int packed = pn;
    if (k + 1 < len) pn = __ldg(A.cols + at + kSlice);
    const int c = packed & kColMask;
    const int g = (int)((unsigned)packed >> kGroupShift);
    while (cg < g) {
      if (cg == 0) {
        y0 = a0;
        y1 = a1;
        y2 = a2;
      } else {
        y0 = y0 + a0;
        y1 = y1 + a1;
        y2 = y2 + a2;
      }
      a0 = a1 = a2 = 0;
      ++cg;
    }
    const T* v = vals + vidx(at, lr & 31, 0);
    const T v0 = __ldg(v), v1 = __ldg(v + 32), v2 = __ldg(v + 64);
    const T v3 = __ldg(v + 96), v4 = __ldg(v + 128), v5 = __ldg(v + 160);
    const T v6 = __ldg(v + 192), v7 = __ldg(v + 224), v8 = __ldg(v + 256);
    T x0, x1, x2;
    gather3<PMode, kRemote, kCg, T>(c, g, x, pold, beta, cv, pm, vexp, seen, x0, x1, x2);
    a0 = a0 + ((v0 * x0 + v1 * x1) + v2 * x2);
    a1 = a1 + ((v3 * x0 + v4 * x1) + v5 * x2);
    a2 = a2 + ((v6 * x0 + v7 * x1) + v8 * x2);
  }
  while (cg < ngroups) {
    if (cg == 0) {
      y0 = a0;
      y1 = a1;
      y2 = a2;
    } else {
      y0 = y0 + a0;
      y1 = y1 + a1;
      y2 = y2 + a2;
    }
    a0 = a1 = a2 = 0.0;
    ++cg;
  }
}

// Matrix-stream load: WEFT_LDS(p) (default __ldg; evict-first __ldcs
// measured slower or equal on B200 for this kernel).
#ifndef WEFT_LDS
#define WEFT_LDS(p) __ldg(p)
#endif

// Single accumulation group (n = 1 or interior rows): the column of slot
// k+1 is fetched while slot k is processed, so the x gather of a slot only
// waits on its own round trip; matrix words are streamed with evict-first
// loads (ld.global.cs) so the gathered vectors stay resident in L2.
template <int PMode>
__device__ __forceinline__ void row_product_1(const SellView& A, int r, const double* __restrict__ x,
                                              const double* __restrict__ pold, double beta, double& y0, double& y1,
                                              double& y2) {
  const int len = A.rowlen[r];
  const int64_t base = A.slice_off[r >> 5] + (r & 31);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  SP_POLICIES
  int cn = len > 0 ? (SP_MLD(A.cols + base) & kColMask) : 0;
#pragma unroll 2
  for (int k = 0; k < len; ++k) {
    const int64_t at = base + (int64_t)k * kSlice;
    const int c = cn;
    if (k + 1 < len) cn = SP_MLD(A.cols + at + kSlice) & kColMask;
    const double* v = A.vals + vidx(at, r & 31, 0);
    const double v0 = SP_MLD(v), v1 = SP_MLD(v + 32), v2 = SP_MLD(v + 64);
    const double v3 = SP_MLD(v + 96), v4 = SP_MLD(v + 128), v5 = SP_MLD(v + 160);
    const double v6 = SP_MLD(v + 192), v7 = SP_MLD(v + 224), v8 = SP_MLD(v + 256);
    double x0 = SP_XLD(x + 3 * c), x1 = SP_XLD(x + 3 * c + 1), x2 = SP_XLD(x + 3 * c + 2);
    if (PMode == 2) {
      x0 = x0 + beta * SP_XLD(pold + 3 * c);
      x1 = x1 + beta * SP_XLD(pold + 3 * c + 1);
      x2 = x2 + beta * SP_XLD(pold + 3 * c + 2);
    }
    a0 = a0 + ((v0 * x0 + v1 * x1) + v2 * x2);
    a1 = a1 + ((v3 * x0 + v4 * x1) + v5 * x2);
    a2 = a2 + ((v6 * x0 + v7 * x1) + v8 * x2);
  }
  y0 = a0;
  y1 = a1;
  y2 = a2;
}

// Asks the TMA unit to stream a whole slice (values + column words) into L2
// with one bulk prefetch, so the per-row loads that follow hit L2 instead of
// each paying a DRAM round trip (SASS: UBLKPF.L2).
__device__ __forceinline__ void prefetch_slice_l2(const SellView& A, int slice) {
  const int64_t s0 = A.slice_off[slice], s1 = A.slice_off[slice + 1];
  const int64_t w = s1 - s0;  // slots (32 per row-width unit)
  if (w <= 0) return;
  const char* vals = reinterpret_cast<const char*>(A.vals + 9 * s0);
  const char* cols = reinterpret_cast<const char*>(A.cols + s0);
  const unsigned vbytes = static_cast<unsigned>(72 * w);
  const unsigned cbytes = static_cast<unsigned>(4 * w);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vals), "r"(vbytes) : "memory");
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(cols), "r"(cbytes) : "memory");
}

// Two threads per row (single accumulation group): lane parity q takes
// slots k = 2j + q, so each warp load instruction moves two coalesced
// 128-byte segments (16 rows x slots 2j and 2j+1) and twice as many rows are
// in flight. The even lane accumulates the row in the reference's slot order
// (P_2j from itself, P_2j+1 from its odd partner via a shuffle). All lanes of
// the warp iterate to the warp's longest row so the shuffles stay converged.
template <int PMode>
__device__ __forceinline__ void row_product_pair(const SellView& A, int r, bool valid, const double* __restrict__ x,
                                                 const double* __restrict__ pold, double beta, double& y0,
                                                 double& y1, double& y2) {
  const int par = threadIdx.x & 1;
  const int len = valid ? A.rowlen[r] : 0;
  const int kmax = __reduce_max_sync(0xffffffffu, len);
  const int64_t base = valid ? A.slice_off[r >> 5] + (r & 31) : 0;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  int cn = par < len ? (WEFT_LDS(A.cols + base + (int64_t)par * kSlice) & kColMask) : 0;
  for (int k0 = 0; k0 < kmax; k0 += 2) {
    const int k = k0 + par;
    double p0 = 0.0, p1 = 0.0, p2 = 0.0;
    if (k < len) {
      const int64_t at = base + (int64_t)k * kSlice;
      const int c = cn;
      if (k + 2 < len) cn = WEFT_LDS(A.cols + at + 2 * kSlice) & kColMask;
      const double* v = A.vals + vidx(at, r & 31, 0);
      const double v0 = WEFT_LDS(v), v1 = WEFT_LDS(v + 32), v2 = WEFT_LDS(v + 64);
      const double v3 = WEFT_LDS(v + 96), v4 = WEFT_LDS(v + 128), v5 = WEFT_LDS(v + 160);
      const double v6 = WEFT_LDS(v + 192), v7 = WEFT_LDS(v + 224), v8 = WEFT_LDS(v + 256);
      double x0 = x[3 * c], x1 = x[3 * c + 1], x2 = x[3 * c + 2];
      if (PMode == 2) {
        x0 = x0 + beta * pold[3 * c];
        x1 = x1 + beta * pold[3 * c + 1];
        x2 = x2 + beta * pold[3 * c + 2];
      }
      p0 = (v0 * x0 + v1 * x1) + v2 * x2;
      p1 = (v3 * x0 + v4 * x1) + v5 * x2;
      p2 = (v6 * x0 + v7 * x1) + v8 * x2;
    }
    const double q0 = __shfl_down_sync(0xffffffffu, p0, 1);
    const double q1 = __shfl_down_sync(0xffffffffu, p1, 1);
    const double q2 = __shfl_down_sync(0xffffffffu, p2, 1);
    if (par == 0 && k0 < len) {
      a0 = a0 + p0;
      a1 = a1 + p1;
      a2 = a2 + p2;
      if (k0 + 1 < len) {
        a0 = a0 + q0;
        a1 = a1 + q1;
        a2 = a2 + q2;
      }
    }
  }
  y0 = a0;
  y1 = a1;
  y2 = a2;
}

__global__ void __launch_bounds__(256) k_spmv_pair(SellView A, const double* __restrict__ x, double* __restrict__ y) {
  const int m = blockIdx.x * (blockDim.x >> 1) + (threadIdx.x >> 1);
  double y0, y1, y2;
  row_product_pair<0>(A, m, m < A.rows, x, nullptr, 0.0, y0, y1, y2);
  if (m < A.rows && (threadIdx.x & 1) == 0) {
    const int r = A.perm[m];  // one partition, one rank: row0 == 0
    y[3 * r] = y0;
    y[3 * r + 1] = y1;
    y[3 * r + 2] = y2;
  }
}

template <class T = double>
__global__ void __launch_bounds__(256) k_spmv(SellView A, int ngroups, const T* __restrict__ x,
                                              T* __restrict__ y, CommView cv, PartMap pm) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= A.rows) return;
  const int r = A.row0 + A.perm[m];
  T y0, y1, y2;
  if constexpr (std::is_same_v<T, float>) {  // Precision::Single: one rank
    row_product<0, false, false, float>(A, m, ngroups, x, nullptr, 0.0, y0, y1, y2);
  } else {
    if (ngroups == 1) row_product_1<0>(A, m, x, nullptr, 0.0, y0, y1, y2);
    else if (cv.world > 1) row_product<0, true, false, double>(A, m, ngroups, x, nullptr, 0.0, y0, y1, y2, cv, pm, cv.seq[0]);
    else row_product<0, false, false, double>(A, m, ngroups, x, nullptr, 0.0, y0, y1, y2);
  }
  y[3 * r] = y0;
  y[3 * r + 1] = y1;
  y[3 * r + 2] = y2;
}

// ---------------------------------------------------------------------------
// Rank-group primitives over peer memory (world > 1)
// ---------------------------------------------------------------------------
// "My rows of the gather vectors (z, p) are final": one thread, after the
// writes of the whole grid are ordered before it (kernel boundary or the
// last-block counter with system-scope fences).
__device__ __forceinline__ void publish_vec(const CommView& cv) {
  __threadfence_system();
  const unsigned long long s = cv.seq[0] + 1;
  cv.seq[0] = s;
  for (int q = 0; q < cv.world; ++q) st_release_sys(&cv.hdr[q]->vec_ready[cv.rank], s);
}

__global__ void k_publish_vec(CommView cv) {
  if (threadIdx.x == 0 && blockIdx.x == 0) publish_vec(cv);
}

// Engine::all_reduce_sum (proj/src/exec.cpp:170-174) over ranks: every rank
// stores its partitions' values into every rank's reduction slots, releases
// its flag, waits for all flags, and sums the n partitions in ascending
// order — the same association as a single-rank run with n partitions, so
// all ranks (and the 1-GPU run) get bitwise the same scalar. Thread 0 only.
template <int NV>
__device__ void combine(const CommView& cv, int d0, int nloc, int ntot, const double (&v)[kMaxParts][NV],
                        double (&out)[NV]) {
#pragma unroll
  for (int i = 0; i < NV; ++i) out[i] = 0.0;
  if (cv.world == 1) {
    for (int d = 0; d < nloc; ++d)
#pragma unroll
      for (int i = 0; i < NV; ++i) out[i] = out[i] + v[d][i];
    return;
  }
  const unsigned long long s = cv.seq[1] + 1;
  cv.seq[1] = s;
  const int par = static_cast<int>(s & 1);
  for (int q = 0; q < cv.world; ++q)
    for (int d = 0; d < nloc; ++d)
#pragma unroll
      for (int i = 0; i < NV; ++i) cv.hdr[q]->red[par][d0 + d][i] = v[d][i];
  __threadfence_system();
  for (int q = 0; q < cv.world; ++q) st_release_sys(&cv.hdr[q]->red_ready[cv.rank], s);
  CommHeader* me = cv.hdr[cv.rank];
  for (int q = 0; q < cv.world; ++q)
    if (!wait_flag(&me->red_ready[q], s)) atomicExch(cv.seq + 3, 1ull);
  for (int d = 0; d < ntot; ++d)
#pragma unroll
    for (int i = 0; i < NV; ++i) out[i] = out[i] + __ldcg(&me->red[par][d][i]);
}

// Rank barrier (a reduction of nothing): after it, every rank has finished
// all work it issued before (e.g. reading this rank's window).
__global__ void k_rank_barrier(CommView cv, int ntot) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double v[kMaxParts][1] = {};
  double out[1];
  combine<1>(cv, 0, 0, ntot, v, out);
}

void publish_vectors(Ctx& c) {
  k_publish_vec<<<1, 32, 0, ls(c)>>>(c.comm);
  WG_CUDA(cudaGetLastError());
}

void rank_barrier(Ctx& c) {
  k_rank_barrier<<<1, 32, 0, ls(c)>>>(c.comm, c.nparts);
  WG_CUDA(cudaGetLastError());
}

void spmv_f32(Ctx& c, const float* x_dev, float* y_dev) {
  if (!c.has_matrix || !c.A.f32) throw Error(WEFT_ERR_INVALID, "spmv: no single-precision matrix loaded");
  if (c.A.rows == 0) return;
  k_spmv<float><<<div_up(c.A.rows, 256), 256, 0, ls(c)>>>(view(c.A), c.go.n, x_dev, y_dev, c.comm, c.pm);
  WG_CUDA(cudaGetLastError());
}

void spmv(Ctx& c, const double* x_dev, double* y_dev) {
  if (!c.has_matrix) throw Error(WEFT_ERR_INVALID, "spmv: no matrix loaded");
  if (c.A.f32) throw Error(WEFT_ERR_INVALID, "spmv: single-precision system (use the f32 entry)");
  const int threads = 256;
  if (c.A.rows == 0) return;
  if (c.go.n == 1 && c.spmv_pair) k_spmv_pair<<<div_up(c.A.rows, threads / 2), threads, 0, ls(c)>>>(view(c.A), x_dev, y_dev);
  else k_spmv<<<div_up(c.A.rows, threads), threads, 0, ls(c)>>>(view(c.A), c.go.n, x_dev, y_dev, c.comm, c.pm);
  WG_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Host construction of the SELL layout from a global CSR (set_matrix path)
// ---------------------------------------------------------------------------
void set_rows(Ctx& c, int p) {
  c.pm = PartMap::make(p, c.nparts);
  c.row0 = c.pm.begin(c.part_begin);
  c.row1 = c.pm.end(c.part_end - 1);
}

std::vector<int32_t> sigma_windows(const Ctx& c, int win) {
  std::vector<int32_t> w;
  for (int d = c.part_begin; d < c.part_end; ++d) {
    const int b = c.pm.begin(d) - c.row0, e = c.pm.end(d) - c.row0;
    for (int s = b; s < e; s += win) w.push_back(s);
  }
  w.push_back(c.row1 - c.row0);
  return w;
}

// One block per window: stable sort of its rows by descending length
// (rank = rows that are longer, or as long and earlier).
template <int W>
__global__ void __launch_bounds__(W) k_sigma(const int32_t* __restrict__ wstart, const int32_t* __restrict__ len,
                                             int32_t* __restrict__ perm, int32_t* __restrict__ pos,
                                             int32_t* __restrict__ len_m) {
  __shared__ int32_t sl[W];
  const int a = wstart[blockIdx.x], n = wstart[blockIdx.x + 1] - a;
  const int t = threadIdx.x;
  if (t < n) sl[t] = len[a + t];
  __syncthreads();
  if (t >= n) return;
  const int L = sl[t];
  int rank = 0;
  for (int j = 0; j < n; ++j) rank += (sl[j] > L) || (sl[j] == L && j < t);
  perm[a + rank] = a + t;
  pos[a + t] = a + rank;
  len_m[a + rank] = L;
}

void build_sigma(Ctx& c, const int32_t* len_row) {
  SellMatrix& A = c.A;
  // Contact rows carry up to 3x the slots of grid rows: a wider sorting
  // window groups them into fewer, fuller slices (config D contacts-mode
  // solve 49.0 -> 44.5 ms; the contact-free matrix is best at 256).
  const int win = c.n_contacts > 0 ? kSigmaContacts : kSigma;
  const std::vector<int32_t> w = sigma_windows(c, win);
  DBuf<int32_t>& wd = c.sc_sigma_w;
  wd.upload(w.data(), w.size(), c.stream);
  A.perm.resize(static_cast<size_t>(A.rows) + 1);
  A.pos.resize(static_cast<size_t>(A.rows) + 1);
  A.rowlen.resize(static_cast<size_t>(A.rows) + 1);
  if (w.size() > 1) {
    if (win == kSigmaContacts)
      k_sigma<kSigmaContacts><<<static_cast<int>(w.size()) - 1, kSigmaContacts, 0, ls(c)>>>(
          wd.data(), len_row, A.perm.data(), A.pos.data(), A.rowlen.data());
    else
      k_sigma<kSigma><<<static_cast<int>(w.size()) - 1, kSigma, 0, ls(c)>>>(wd.data(), len_row, A.perm.data(),
                                                                           A.pos.data(), A.rowlen.data());
  }
  WG_CUDA(cudaGetLastError());
  WG_CUDA(cudaStreamSynchronize(c.stream));  // wd dies here
}

// Takes the GLOBAL block CSR (every rank passes the same matrix) and keeps
// this rank's rows [row0, row1) (partition_matrix, sparse.hpp:103-147).
void set_matrix_csr(Ctx& c, int rows, const int64_t* row_ptr, const int32_t* cols, const double* vals) {
  c.A.f32 = false;
  if (rows < 0) throw Error(WEFT_ERR_DIMENSION, "set_matrix: negative row count");
  if (rows >= (1 << 28)) throw Error(WEFT_ERR_DIMENSION, "set_matrix: more than 2^28 block rows");
  if (rows < c.nparts) throw Error(WEFT_ERR_DIMENSION, "set_matrix: fewer rows than partitions");
  set_rows(c, rows);
  SellMatrix& A = c.A;
  const int nloc = c.row1 - c.row0;
  A.rows = nloc;
  A.row0 = c.row0;
  A.nslices = div_up(nloc, kSlice);
  std::vector<int32_t> len(static_cast<size_t>(nloc));
  std::vector<int64_t> soff(static_cast<size_t>(A.nslices) + 1, 0);
  int64_t nnzb = 0;
  int maxlen = 0;
  for (int r = 0; r < rows; ++r)
    if (row_ptr[r + 1] - row_ptr[r] < 0) throw Error(WEFT_ERR_DIMENSION, "set_matrix: row_ptr not monotone");
  // SELL-32-sigma: positions sorted by descending row length per window
  std::vector<int32_t> perm(static_cast<size_t>(nloc)), pos(static_cast<size_t>(nloc));
  {
    const std::vector<int32_t> w = sigma_windows(c);
    std::vector<std::pair<int, int>> v;
    for (size_t k = 0; k + 1 < w.size(); ++k) {
      v.clear();
      for (int lr = w[k]; lr < w[k + 1]; ++lr)
        v.push_back({-static_cast<int>(row_ptr[c.row0 + lr + 1] - row_ptr[c.row0 + lr]), lr});
      std::stable_sort(v.begin(), v.end());
      for (size_t i = 0; i < v.size(); ++i) {
        perm[static_cast<size_t>(w[k]) + i] = v[i].second;
        pos[static_cast<size_t>(v[i].second)] = w[k] + static_cast<int>(i);
      }
    }
  }
  for (int m = 0; m < nloc; ++m) {
    const int r = c.row0 + perm[static_cast<size_t>(m)];
    const int64_t l = row_ptr[r + 1] - row_ptr[r];
    len[static_cast<size_t>(m)] = static_cast<int32_t>(l);
    nnzb += l;
    maxlen = std::max<int>(maxlen, static_cast<int>(l));
  }
  for (int s = 0; s < A.nslices; ++s) {
    int w = 0;
    for (int m = s * kSlice; m < std::min(nloc, (s + 1) * kSlice); ++m) w = std::max(w, len[static_cast<size_t>(m)]);
    soff[static_cast<size_t>(s) + 1] = soff[static_cast<size_t>(s)] + static_cast<int64_t>(w) * kSlice;
  }
  const int64_t total = soff.back();
  std::vector<int32_t> hc(static_cast<size_t>(total), -1);
  std::vector<double> hv(9 * static_cast<size_t>(total), 0.0);
  std::vector<std::pair<int, int64_t>> order;  // (group, csr index)
  for (int lr = 0; lr < nloc; ++lr) {
    const int r = c.row0 + lr;
    const int mp = pos[static_cast<size_t>(lr)];
    const int d = c.pm.owner(r);
    order.clear();
    for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
      const int col = cols[k];
      if (col < 0 || col >= rows) throw Error(WEFT_ERR_DIMENSION, "input vector too short for column index");
      order.push_back({c.go.qpos[d][c.pm.owner(col)], k});
    }
    std::stable_sort(order.begin(), order.end(),
                     [](const auto& a, const auto& b) { return a.first < b.first; });
    const int64_t base = soff[static_cast<size_t>(mp / kSlice)] + mp % kSlice;
    for (size_t s = 0; s < order.size(); ++s) {
      const int64_t at = base + static_cast<int64_t>(s) * kSlice;
      const int64_t k = order[s].second;
      hc[static_cast<size_t>(at)] = cols[k] | (order[s].first << kGroupShift);
      for (int q = 0; q < 9; ++q) hv[static_cast<size_t>(vidx(at, mp % kSlice, q))] = vals[9 * k + q];
    }
  }
  A.total = total;
  A.nnzb = nnzb;
  A.max_len = maxlen;
  A.slice_off.upload(soff.data(), soff.size(), c.stream);
  A.rowlen.upload(len.data(), len.size(), c.stream);
  A.perm.upload(perm.data(), perm.size(), c.stream);
  A.pos.upload(pos.data(), pos.size(), c.stream);
  A.cols.upload(hc.data(), hc.size(), c.stream);
  A.vals.upload(hv.data(), hv.size(), c.stream);
  WG_CUDA(cudaStreamSynchronize(c.stream));
  ++A.layout_id;
  c.has_matrix = true;
  c.has_rhs = false;
  c.have_pattern_for_contacts = false;
}

// This rank's rows [row0, row1) as block CSR with ascending columns
// (gather_matrix, sparse.hpp:149-173; all rows when world == 1).
template <class T>
static void download_csr_t(Ctx& c, int64_t* row_ptr, int32_t* cols, T* vals) {
  SellMatrix& A = c.A;
  std::vector<int64_t> soff(A.slice_off.size());
  std::vector<int32_t> len(static_cast<size_t>(A.rows));
  std::vector<int32_t> hc(static_cast<size_t>(A.total));
  std::vector<int32_t> pos(static_cast<size_t>(A.rows));
  A.slice_off.download(soff.data(), soff.size(), c.stream);
  A.rowlen.download(len.data(), len.size(), c.stream);
  A.pos.download(pos.data(), pos.size(), c.stream);
  A.cols.download(hc.data(), hc.size(), c.stream);
  std::vector<T> hv;
  if (vals) {
    hv.resize(9 * static_cast<size_t>(A.total));
    if constexpr (std::is_same_v<T, float>) A.vals32.download(hv.data(), hv.size(), c.stream);
    else A.vals.download(hv.data(), hv.size(), c.stream);
  }
  WG_CUDA(cudaStreamSynchronize(c.stream));
  int64_t cursor = 0;
  std::vector<std::pair<int, int64_t>> order;
  if (row_ptr) row_ptr[0] = 0;
  for (int r = 0; r < A.rows; ++r) {
    const int mp = pos[static_cast<size_t>(r)];
    const int64_t base = soff[static_cast<size_t>(mp / kSlice)] + mp % kSlice;
    order.clear();
    for (int k = 0; k < len[static_cast<size_t>(mp)]; ++k) {
      const int64_t at = base + static_cast<int64_t>(k) * kSlice;
      order.push_back({hc[static_cast<size_t>(at)] & kColMask, at});
    }
    std::sort(order.begin(), order.end());
    for (const auto& [col, at] : order) {
      if (cols) cols[cursor] = col;
      if (vals)
        for (int q = 0; q < 9; ++q) vals[9 * cursor + q] = hv[static_cast<size_t>(vidx(at, mp % kSlice, q))];
      ++cursor;
    }
    if (row_ptr) row_ptr[r + 1] = cursor;
  }
}

void download_csr(Ctx& c, int64_t* row_ptr, int32_t* cols, double* vals) {
  if (c.A.f32 && vals) throw Error(WEFT_ERR_INVALID, "download_matrix: single-precision system (use the f32 entry)");
  download_csr_t<double>(c, row_ptr, cols, vals);
}
void download_csr_f32(Ctx& c, int64_t* row_ptr, int32_t* cols, float* vals) {
  if (!c.A.f32 && vals) throw Error(WEFT_ERR_INVALID, "download_matrix: double-precision system");
  download_csr_t<float>(c, row_ptr, cols, vals);
}

// ---------------------------------------------------------------------------
// Deterministic block reduction helpers
// ---------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* smem /* NV * 32 */) {
#pragma unroll
  for (int i = 0; i < NV; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] = v[i] + __shfl_xor_sync(0xffffffffu, v[i], o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) smem[i * 32 + warp] = v[i];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double t = lane < nw ? smem[i * 32 + lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t = t + __shfl_xor_sync(0xffffffffu, t, o);
      v[i] = t;
    }
  }
  __syncthreads();
}

// Sums partials[b*NV + i] over the blocks of each held partition (fixed
// strided order + fixed tree), then combines the partitions in ascending
// order across ranks. Called by all threads of the last block; result valid
// in thread 0.
template <int NV>
__device__ void finalize_sums(const PartBlocks& pb, const double* partials, double (&out)[NV], double* smem,
                              const CommView& cv, int ntot) {
  double per[kMaxParts][NV];
  for (int d = 0; d < pb.n; ++d) {
    double v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = 0.0;
    for (int b = pb.bstart[d] + threadIdx.x; b < pb.bstart[d + 1]; b += blockDim.x)
#pragma unroll
      for (int i = 0; i < NV; ++i) v[i] = v[i] + __ldcg(partials + (size_t)b * NV + i);
    block_sum<NV>(v, smem);
#pragma unroll
    for (int i = 0; i < NV; ++i) per[d][i] = v[i];  // only thread 0's value is used
  }
  if (threadIdx.x == 0) combine<NV>(cv, pb.d0, pb.n, ntot, per, out);
}

// ---------------------------------------------------------------------------
// PCG
// ---------------------------------------------------------------------------
struct PcgState {  // read back with read_small (<= 128 bytes)
  double rho, alpha, beta, b_norm, tol, r_norm;
  int iter;       // completed iterations
  int done;       // 1 = stop (converged, error, or max iterations)
  int status;     // 0 ok, 1 non-finite curvature, 2 non-positive, 3 divergence
  int converged;
  int max_iter;
  int first;      // next SpMV uses p = z
  unsigned counter;
};

// Last-block-done: thread 0 publishes the block's partial (caller wrote it
// before), fences once, and counts arrivals; only the last block reduces.
// With peers (sys), the fence is system-scope so the rows this grid wrote
// are visible to other GPUs before the last block releases them.
__device__ __forceinline__ bool last_block(unsigned* counter, bool sys) {
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    if (sys) __threadfence_system();
    else __threadfence();
    const unsigned t = atomicAdd(counter, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

// Global row of thread threadIdx.x in block b under partition-aligned
// blocking (rows of the held partitions only).
__device__ __forceinline__ int block_row(const PartBlocks& pb, int b, int& rend) {
  const int d = block_part(pb, b);
  rend = pb.rend[d];
  return pb.rbegin[d] + (b - pb.bstart[d]) * blockDim.x + threadIdx.x;
}

// dot(u, v) per partition + ascending sum into *out (used for ||b||, rho0).
// Products of Real values taken in double (solver.hpp:91-100).
template <class T = double>
__global__ void __launch_bounds__(256) k_dot2(PartBlocks pb, const T* __restrict__ u, const T* __restrict__ v,
                                              const T* __restrict__ u2, const T* __restrict__ v2,
                                              double* partials, unsigned* counter, double* out, CommView cv,
                                              int ntot) {
  __shared__ double smem[2 * 32];
  int rend;
  const int r = block_row(pb, blockIdx.x, rend);
  double s[2] = {0.0, 0.0};
  auto d = [](T a) { return static_cast<double>(a); };
  if (r < rend) {
    s[0] = (d(u[3 * r]) * d(v[3 * r]) + d(u[3 * r + 1]) * d(v[3 * r + 1])) + d(u[3 * r + 2]) * d(v[3 * r + 2]);
    if (u2)
      s[1] = (d(u2[3 * r]) * d(v2[3 * r]) + d(u2[3 * r + 1]) * d(v2[3 * r + 1])) + d(u2[3 * r + 2]) * d(v2[3 * r + 2]);
  }
  block_sum<2>(s, smem);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = s[0];
    partials[2 * blockIdx.x + 1] = s[1];
  }
  if (!last_block(counter, false)) return;
  double t[2];
  finalize_sums<2>(pb, partials, t, smem, cv, ntot);
  if (threadIdx.x == 0) {
    out[0] = t[0];
    out[1] = t[1];
    *counter = 0;
  }
}

// Block-Jacobi inverse of the diagonal blocks (solver.hpp:49-65) with the
// cofactor inverse of oracle/shim/Eigen/Dense; identity when absent.
// dinv is indexed by global row.
// kPosOut (persistent solve): position order, plus the packed upper
// triangle d6 (6 doubles) and *asym = 1 if any inverse is not bitwise
// symmetric (then the solve reads the 9-double form).
template <bool kPosOut, class T = double>
__global__ void k_dinv(SellView A, double* __restrict__ dinv, double* __restrict__ d6 = nullptr,
                       int* __restrict__ asym = nullptr) {
  const int mp = blockIdx.x * blockDim.x + threadIdx.x;
  if (mp >= A.rows) return;
  const int r = A.row0 + A.perm[mp];
  const int len = A.rowlen[mp];
  const int64_t base = A.slice_off[mp >> 5] + (mp & 31);
  double m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  for (int k = 0; k < len; ++k) {
    const int64_t at = base + (int64_t)k * kSlice;
    if ((A.cols[at] & kColMask) == r) {
      for (int q = 0; q < 9; ++q) m[q] = static_cast<double>(sell_vals<T>(A)[vidx(at, mp & 31, q)]);
      break;
    }
  }
#define M(i, j) m[(i) * 3 + (j)]
#define COF(i, j)                                                                                   \
  (M(((i) + 1) % 3, ((j) + 1) % 3) * M(((i) + 2) % 3, ((j) + 2) % 3) -                              \
   M(((i) + 1) % 3, ((j) + 2) % 3) * M(((i) + 2) % 3, ((j) + 1) % 3))
  const double c00 = COF(0, 0), c10 = COF(1, 0), c20 = COF(2, 0);
  const double det = (c00 * M(0, 0) + c10 * M(1, 0)) + c20 * M(2, 0);
  const double invdet = 1.0 / det;
  double* o = dinv + 9 * (kPosOut ? (size_t)mp : (size_t)r);
  o[0] = c00 * invdet;
  o[1] = c10 * invdet;
  o[2] = c20 * invdet;
  o[3] = COF(0, 1) * invdet;
  o[4] = COF(1, 1) * invdet;
  o[5] = COF(2, 1) * invdet;
  o[6] = COF(0, 2) * invdet;
  o[7] = COF(1, 2) * invdet;
  o[8] = COF(2, 2) * invdet;
  if (kPosOut && d6) {
    // SpdProjected / contact / mass diagonal blocks are bitwise symmetric
    // (sums of outer products in one order), and so are their cofactor
    // inverses: 6 doubles carry the block exactly.
    if (o[1] != o[3] || o[2] != o[6] || o[5] != o[7]) atomicOr(asym, 1);
    double* h = d6 + 6 * (size_t)mp;
    h[0] = o[0];
    h[1] = o[1];
    h[2] = o[2];
    h[3] = o[4];
    h[4] = o[5];
    h[5] = o[8];
  }
#undef COF
#undef M
}

// apply_precond (solver.hpp:67-89): acc = 0; acc += m(i,j) * src[j].
// acc in double, the result cast to Real (solver.hpp:80-86).
template <class T = double>
__device__ __forceinline__ void precond_row(const double* __restrict__ dinv, bool bj, int r, T r0, T r1, T r2,
                                            T& z0, T& z1, T& z2) {
  if (!bj) {
    z0 = r0;
    z1 = r1;
    z2 = r2;
    return;
  }
  const double* m = dinv + 9 * (size_t)r;
  const double d0 = r0, d1 = r1, d2 = r2;
  z0 = static_cast<T>(((0.0 + m[0] * d0) + m[1] * d1) + m[2] * d2);
  z1 = static_cast<T>(((0.0 + m[3] * d0) + m[4] * d1) + m[5] * d2);
  z2 = static_cast<T>(((0.0 + m[6] * d0) + m[7] * d1) + m[8] * d2);
}

// PCG init over the held rows: x = 0, r = b, z = M^-1 r (p = z is formed by
// the first SpMV).
template <class T = double>
__global__ void k_pcg_init(int row0, int rows, const T* __restrict__ b, const double* __restrict__ dinv,
                           bool bj, T* __restrict__ x, T* __restrict__ r, T* __restrict__ z,
                           T* __restrict__ p) {
  const int lr = blockIdx.x * blockDim.x + threadIdx.x;
  if (lr >= rows) return;
  const int i = row0 + lr;
  const T b0 = b[3 * i], b1 = b[3 * i + 1], b2 = b[3 * i + 2];
  T z0, z1, z2;
  precond_row<T>(dinv, bj, i, b0, b1, b2, z0, z1, z2);
  x[3 * i] = x[3 * i + 1] = x[3 * i + 2] = 0;
  r[3 * i] = b0;
  r[3 * i + 1] = b1;
  r[3 * i + 2] = b2;
  z[3 * i] = z0;
  z[3 * i + 1] = z1;
  z[3 * i + 2] = z2;
  p[3 * i] = p[3 * i + 1] = p[3 * i + 2] = 0;
}

// Per-solve arguments, read by the iteration kernels through one device
// pointer so the captured CUDA graph stays valid across solves.
struct PcgArgs {
  SellView A;
  PartBlocks pb;
  PartBlocks pb2;  // blocks of 128 rows (two threads per row, single partition)
  int ngroups;
  int bj;
  const double* dinv;
  double *x, *r, *z, *p, *q, *partials, *hist, *phist;
  CommView cv;
  PartMap pm;
  double* p2;  // persistent solve: second search-direction buffer
  int q_msw;   // persistent solve with q in shared memory: max slices per warp
  const double* dinv6;  // persistent solve: packed symmetric D^-1 (null: 9-double form)
  float vec_el_frac;    // persistent solve: fraction of the gathered z / p lines kept evict_last
  const int16_t* colp16;  // persistent solve: 16-bit column offsets (null: A.cols)
  const uint32_t* mwords;  // persistent solve, kMir: column offset (low 16) | mirror slot delta (high 16)
  unsigned long long* timing;  // dev instrumentation (WEFT_PCG_TIMING=1): ns per phase, summed
};

// Iteration kernel 1: q = A p with p = z (+ beta p) formed on the fly;
// p.q partials; last block: curvature checks and alpha = rho / pq.
// kRemote: columns of other ranks are gathered over peer memory.
template <bool kSingle, bool kPair, bool kRemote>
__global__ void __launch_bounds__(256) k_pcg_spmv(const PcgArgs* __restrict__ args, PcgState* st) {
  __shared__ double smem[32];
  if (st->done) return;
  const PcgArgs& g = *args;
  const SellView A = g.A;
  const double* __restrict__ z = g.z;
  const double* __restrict__ p = g.p;
  double* __restrict__ q = g.q;
  const bool first = st->first != 0;
  const double beta = st->beta;
  int rend;
  double s[1] = {0.0};
  if constexpr (kSingle && kPair) {
    // two threads per row (single partition: rows [0, rows))
    const int m = blockIdx.x * (blockDim.x >> 1) + (threadIdx.x >> 1);
    const bool valid = m < A.rows;
    double y0, y1, y2;
    if (first) row_product_pair<1>(A, m, valid, z, p, beta, y0, y1, y2);
    else row_product_pair<2>(A, m, valid, z, p, beta, y0, y1, y2);
    if (valid && (threadIdx.x & 1) == 0) {
      const int r = A.perm[m];
      q[3 * r] = y0;
      q[3 * r + 1] = y1;
      q[3 * r + 2] = y2;
      double p0 = z[3 * r], p1 = z[3 * r + 1], p2 = z[3 * r + 2];
      if (!first) {
        p0 = p0 + beta * p[3 * r];
        p1 = p1 + beta * p[3 * r + 1];
        p2 = p2 + beta * p[3 * r + 2];
      }
      s[0] = (p0 * y0 + p1 * y1) + p2 * y2;
    }
  }
  // the partition-aligned block layout walks matrix positions; each
  // position's row lies in the same sigma window, hence the same partition
  const int mg = (kSingle && kPair) ? -1 : block_row(g.pb, blockIdx.x, rend);
  if (!(kSingle && kPair) && mg < rend) {
    const int m = mg - A.row0;
    const int r = A.row0 + A.perm[m];
    double y0, y1, y2;
    if constexpr (kSingle) {
      if (first) row_product_1<1>(A, m, z, p, beta, y0, y1, y2);
      else row_product_1<2>(A, m, z, p, beta, y0, y1, y2);
    } else {
      const unsigned long long vexp = kRemote ? g.cv.seq[0] : 0;
      if (first) row_product<1, kRemote>(A, m, g.ngroups, z, p, beta, y0, y1, y2, g.cv, g.pm, vexp);
      else row_product<2, kRemote>(A, m, g.ngroups, z, p, beta, y0, y1, y2, g.cv, g.pm, vexp);
    }
    q[3 * r] = y0;
    q[3 * r + 1] = y1;
    q[3 * r + 2] = y2;
    double p0 = z[3 * r], p1 = z[3 * r + 1], p2 = z[3 * r + 2];
    if (!first) {
      p0 = p0 + beta * p[3 * r];
      p1 = p1 + beta * p[3 * r + 1];
      p2 = p2 + beta * p[3 * r + 2];
    }
    s[0] = (p0 * y0 + p1 * y1) + p2 * y2;
  }
  block_sum<1>(s, smem);
  if (threadIdx.x == 0) g.partials[blockIdx.x] = s[0];
  if (!last_block(&st->counter, false)) return;
  double t[1];
  finalize_sums<1>((kSingle && kPair) ? g.pb2 : g.pb, g.partials, t, smem, g.cv, g.pm.n);
  if (threadIdx.x == 0) {
    st->counter = 0;
    const double pq = t[0];
    const int it = st->iter + 1;
    if (!isfinite(pq)) {
      st->status = 1;
      st->done = 1;
      st->iter = it;
    } else if (pq <= 0.0) {
      st->status = 2;
      st->done = 1;
      st->iter = it;
    } else {
      st->alpha = st->rho / pq;
    }
  }
}

// Iteration kernel 2: p = z + beta p (own rows), x += alpha p,
// r -= alpha q, z = M^-1 r; r.r and r.z partials; last block: residual
// history, convergence test, beta, and (graph mode) the loop condition.
__global__ void __launch_bounds__(256) k_pcg_update(const PcgArgs* __restrict__ args, PcgState* st,
                                                    cudaGraphConditionalHandle cond, int use_cond) {
  __shared__ double smem[2 * 32];
  if (st->done) {
    if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
    return;
  }
  const PcgArgs& g = *args;
  double* __restrict__ x = g.x;
  double* __restrict__ r = g.r;
  double* __restrict__ z = g.z;
  double* __restrict__ p = g.p;
  const double* __restrict__ q = g.q;
  const bool first = st->first != 0;
  const double beta = st->beta, alpha = st->alpha;
  int rend;
  const int i = block_row(g.pb, blockIdx.x, rend);
  double s[2] = {0.0, 0.0};
  if (i < rend) {
    // all loads first (the arrays come through a struct, so the compiler
    // cannot prove they do not alias and would otherwise serialise them)
    double zv[3], pv[3], xv[3], rv[3], qv[3], m[9];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      zv[c] = z[3 * i + c];
      pv[c] = first ? 0.0 : p[3 * i + c];
      xv[c] = x[3 * i + c];
      rv[c] = r[3 * i + c];
      qv[c] = q[3 * i + c];
    }
    if (g.bj) {
#pragma unroll
      for (int k = 0; k < 9; ++k) m[k] = g.dinv[9 * (size_t)i + k];
    }
    double pr[3], rr[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      pr[c] = first ? zv[c] : zv[c] + beta * pv[c];
      xv[c] = xv[c] + alpha * pr[c];
      rr[c] = rv[c] - alpha * qv[c];
    }
    double z0, z1, z2;
    if (g.bj) {  // apply_precond (solver.hpp:67-89)
      z0 = ((0.0 + m[0] * rr[0]) + m[1] * rr[1]) + m[2] * rr[2];
      z1 = ((0.0 + m[3] * rr[0]) + m[4] * rr[1]) + m[5] * rr[2];
      z2 = ((0.0 + m[6] * rr[0]) + m[7] * rr[1]) + m[8] * rr[2];
    } else {
      z0 = rr[0];
      z1 = rr[1];
      z2 = rr[2];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      p[3 * i + c] = pr[c];
      x[3 * i + c] = xv[c];
      r[3 * i + c] = rr[c];
    }
    z[3 * i] = z0;
    z[3 * i + 1] = z1;
    z[3 * i + 2] = z2;
    s[0] = (rr[0] * rr[0] + rr[1] * rr[1]) + rr[2] * rr[2];
    s[1] = (rr[0] * z0 + rr[1] * z1) + rr[2] * z2;
  }
  block_sum<2>(s, smem);
  if (threadIdx.x == 0) {
    g.partials[2 * blockIdx.x] = s[0];
    g.partials[2 * blockIdx.x + 1] = s[1];
  }
  const bool peers = g.cv.world > 1;
  if (!last_block(&st->counter, peers)) return;
  // z and p of the held rows are final: release them to the peers before
  // waiting on the reduction, so their next SpMV can start gathering.
  if (peers && threadIdx.x == 0) publish_vec(g.cv);
  double t[2];
  finalize_sums<2>(g.pb, g.partials, t, smem, g.cv, g.pm.n);
  if (threadIdx.x == 0) {
    st->counter = 0;
    const int it = st->iter + 1;
    st->iter = it;
    st->first = 0;
    const double r_norm = sqrt(t[0]);
    st->r_norm = r_norm;
    if (!isfinite(r_norm)) {
      st->status = 3;
      st->done = 1;
    } else {
      g.hist[it - 1] = r_norm / st->b_norm;
      const double rho_next = t[1];
      g.phist[it - 1] = sqrt(rho_next > 0.0 ? rho_next : 0.0);
      if (r_norm <= st->tol) {
        st->converged = 1;
        st->done = 1;
      } else {
        st->beta = rho_next / st->rho;
        st->rho = rho_next;
        if (it >= st->max_iter) st->done = 1;
      }
    }
    if (use_cond) cudaGraphSetConditional(cond, st->done ? 0 : 1);
  }
}


// ---------------------------------------------------------------------------
// Persistent multi-partition / rank-group PCG: the graph path's two
// iteration kernels (k_pcg_spmv, k_pcg_update) fused into ONE cooperative
// kernel per rank. Each CTA walks the same partition-aligned 256-row
// "virtual blocks" the two kernels use (blockIdx.x, + grid, ...), so every
// block partial, every per-partition sum and every reduction is bitwise the
// graph path's; the kernel boundaries become grid syncs and the last-block
// reductions become redundant per-CTA reductions over the partials. Across
// ranks: block 0 posts this rank's partition sums into every rank's
// reduction slots and releases its flag, every CTA waits for all flags and
// adds the n partitions in ascending order (Engine::all_reduce_sum,
// exec.cpp:170-174), and block 0 publishes z / p after each update so the
// peers' next SpMV can gather the halo columns (dynamic contact columns
// included). Per iteration: 2 grid syncs, 2 flag rounds, no launch.
// ---------------------------------------------------------------------------
template <int NV>
__device__ void partition_sums(const PartBlocks& pb, const double* partials, double (&per)[kMaxParts][NV],
                               double* smem) {
  for (int d = 0; d < pb.n; ++d) {
    double v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = 0.0;
    for (int b = pb.bstart[d] + threadIdx.x; b < pb.bstart[d + 1]; b += blockDim.x)
#pragma unroll
      for (int i = 0; i < NV; ++i) v[i] = v[i] + __ldcg(partials + (size_t)b * NV + i);
    block_sum<NV>(v, smem);
#pragma unroll
    for (int i = 0; i < NV; ++i) per[d][i] = v[i];  // thread 0's value is the sum
  }
}

// combine() split over the CTAs of a persistent grid: `post` (block 0,
// thread 0) stores and releases, every CTA's thread 0 waits and sums. The
// reduction sequence number s is tracked per CTA (identical everywhere).
template <int NV>
__device__ void combine_split(const CommView& cv, int d0, int nloc, int ntot, const double (&v)[kMaxParts][NV],
                              unsigned long long s, bool post, double (&out)[NV]) {
#pragma unroll
  for (int i = 0; i < NV; ++i) out[i] = 0.0;
  if (cv.world == 1) {
    for (int d = 0; d < nloc; ++d)
#pragma unroll
      for (int i = 0; i < NV; ++i) out[i] = out[i] + v[d][i];
    return;
  }
  const int par = static_cast<int>(s & 1);
  if (post) {
    cv.seq[1] = s;
    for (int q = 0; q < cv.world; ++q)
      for (int d = 0; d < nloc; ++d)
#pragma unroll
        for (int i = 0; i < NV; ++i) cv.hdr[q]->red[par][d0 + d][i] = v[d][i];
    __threadfence_system();
    for (int q = 0; q < cv.world; ++q) st_release_sys(&cv.hdr[q]->red_ready[cv.rank], s);
  }
  CommHeader* me = cv.hdr[cv.rank];
  for (int q = 0; q < cv.world; ++q)
    if (!wait_flag(&me->red_ready[q], s)) atomicExch(cv.seq + 3, 1ull);
  for (int d = 0; d < ntot; ++d)
#pragma unroll
    for (int i = 0; i < NV; ++i) out[i] = out[i] + __ldcg(&me->red[par][d][i]);
}

template <bool kRemote, class T = double>
__global__ void __launch_bounds__(256, 2) k_pcg_persistent_rows(const PcgArgs* __restrict__ args, PcgState* st) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double smem[2 * 32];
  __shared__ double bc[2];
  const PcgArgs& g = *args;
  const SellView A = g.A;
  const PartBlocks& pb = g.pb;
  const int nvb = pb.bstart[pb.n];  // virtual blocks (256 rows of one partition)
  // T = float: Precision::Single — Real vectors and matrix, double scalars
  // and dot products, alpha / beta cast to Real in the updates (solver.hpp)
  T* __restrict__ x = reinterpret_cast<T*>(g.x);
  T* __restrict__ r = reinterpret_cast<T*>(g.r);
  T* __restrict__ z = reinterpret_cast<T*>(g.z);
  T* __restrict__ p = reinterpret_cast<T*>(g.p);
  T* __restrict__ q = reinterpret_cast<T*>(g.q);
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const CommView cv = g.cv;
  unsigned long long vseq = kRemote ? cv.seq[0] : 0;  // z / p publications seen so far
  unsigned long long rseq = kRemote ? cv.seq[1] : 0;   // reductions so far (no counters on one rank)
  double rho = st->rho, beta = st->beta;
  const double tol = st->tol, b_norm = st->b_norm;
  const int max_it = st->max_iter;
  int it = st->iter, status = 0, converged = 0;
  bool first = st->first != 0;
  bool done = st->done != 0;
  double r_norm = st->r_norm;
  grid.sync();  // every CTA has read the starting sequence numbers
  while (!done) {
    // ---- k_pcg_spmv: q = A p with p = z (+ beta p) formed on the fly
    for (int vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
      int rend;
      const int mg = block_row(pb, vb, rend);
      double s1[1] = {0.0};
      if (mg < rend) {
        const int m = mg - A.row0;
        const int row = A.row0 + A.perm[m];
        T y0, y1, y2;
        if (first) row_product<1, kRemote, true, T>(A, m, g.ngroups, z, p, beta, y0, y1, y2, cv, g.pm, vseq);
        else row_product<2, kRemote, true, T>(A, m, g.ngroups, z, p, beta, y0, y1, y2, cv, g.pm, vseq);
        __stcg(q + 3 * row, y0);
        __stcg(q + 3 * row + 1, y1);
        __stcg(q + 3 * row + 2, y2);
        T p0 = __ldcg(z + 3 * row), p1 = __ldcg(z + 3 * row + 1), p2 = __ldcg(z + 3 * row + 2);
        if (!first) {
          const T bt = static_cast<T>(beta);
          p0 = p0 + bt * __ldcg(p + 3 * row);
          p1 = p1 + bt * __ldcg(p + 3 * row + 1);
          p2 = p2 + bt * __ldcg(p + 3 * row + 2);
        }
        const double dp0 = p0, dp1 = p1, dp2 = p2, dy0 = y0, dy1 = y1, dy2 = y2;
        s1[0] = (dp0 * dy0 + dp1 * dy1) + dp2 * dy2;
      }
      block_sum<1>(s1, smem);
      if (threadIdx.x == 0) __stcg(g.partials + vb, s1[0]);
    }
    grid.sync();
    if (kRemote && __ldcg(cv.seq + 3)) break;  // a peer timed out: stop everywhere
    {
      double per[kMaxParts][1];
      partition_sums<1>(pb, g.partials, per, smem);
      ++rseq;
      if (threadIdx.x == 0) {
        double t[1];
        combine_split<1>(cv, pb.d0, pb.n, g.pm.n, per, rseq, blockIdx.x == 0, t);
        bc[0] = t[0];
      }
      __syncthreads();
    }
    const double pq = bc[0];
    if (!isfinite(pq)) {
      status = 1;
      ++it;
      break;
    }
    if (pq <= 0.0) {
      status = 2;
      ++it;
      break;
    }
    const double alpha = rho / pq;
    // ---- k_pcg_update: p, x, r, z of the held rows; r.r and r.z
    for (int vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
      int rend;
      const int i = block_row(pb, vb, rend);
      double s2[2] = {0.0, 0.0};
      if (i < rend) {
        T zv[3], pv[3], xv[3], rv[3], qv[3];
        double m[9];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          zv[c] = __ldcg(z + 3 * i + c);
          pv[c] = first ? T(0) : __ldcg(p + 3 * i + c);
          xv[c] = __ldcg(x + 3 * i + c);
          rv[c] = __ldcg(r + 3 * i + c);
          qv[c] = __ldcg(q + 3 * i + c);
        }
        if (g.bj) {
#pragma unroll
          for (int k = 0; k < 9; ++k) m[k] = __ldg(g.dinv + 9 * (size_t)i + k);
        }
        T pr[3], rr[3];
        const T at = static_cast<T>(alpha), bt = static_cast<T>(beta);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          pr[c] = first ? zv[c] : zv[c] + bt * pv[c];
          xv[c] = xv[c] + at * pr[c];
          rr[c] = rv[c] - at * qv[c];
        }
        T z0, z1, z2;
        if (g.bj) {  // apply_precond (solver.hpp:67-89): double acc, cast to Real
          const double d0 = rr[0], d1 = rr[1], d2 = rr[2];
          z0 = static_cast<T>(((0.0 + m[0] * d0) + m[1] * d1) + m[2] * d2);
          z1 = static_cast<T>(((0.0 + m[3] * d0) + m[4] * d1) + m[5] * d2);
          z2 = static_cast<T>(((0.0 + m[6] * d0) + m[7] * d1) + m[8] * d2);
        } else {
          z0 = rr[0];
          z1 = rr[1];
          z2 = rr[2];
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          __stcg(p + 3 * i + c, pr[c]);
          __stcg(x + 3 * i + c, xv[c]);
          __stcg(r + 3 * i + c, rr[c]);
        }
        __stcg(z + 3 * i, z0);
        __stcg(z + 3 * i + 1, z1);
        __stcg(z + 3 * i + 2, z2);
        const double e0 = rr[0], e1 = rr[1], e2 = rr[2], f0 = z0, f1 = z1, f2 = z2;
        s2[0] = (e0 * e0 + e1 * e1) + e2 * e2;
        s2[1] = (e0 * f0 + e1 * f1) + e2 * f2;
      }
      block_sum<2>(s2, smem);
      if (threadIdx.x == 0) {
        __stcg(g.partials + 2 * vb, s2[0]);
        __stcg(g.partials + 2 * vb + 1, s2[1]);
      }
    }
    grid.sync();
    if (kRemote && __ldcg(cv.seq + 3)) break;
    // z and p of the held rows are final: release them to the peers
    if (kRemote) {
      if (lead) publish_vec(cv);
      ++vseq;
    }
    {
      double per[kMaxParts][2];
      partition_sums<2>(pb, g.partials, per, smem);
      ++rseq;
      if (threadIdx.x == 0) {
        double t[2];
        combine_split<2>(cv, pb.d0, pb.n, g.pm.n, per, rseq, blockIdx.x == 0, t);
        bc[0] = t[0];
        bc[1] = t[1];
      }
      __syncthreads();
    }
    ++it;
    first = false;
    r_norm = sqrt(bc[0]);
    if (!isfinite(r_norm)) {
      status = 3;
      break;
    }
    const double rho_next = bc[1];
    if (lead) {
      g.hist[it - 1] = r_norm / b_norm;
      g.phist[it - 1] = sqrt(rho_next > 0.0 ? rho_next : 0.0);
    }
    if (r_norm <= tol) {
      converged = 1;
      break;
    }
    beta = rho_next / rho;
    rho = rho_next;
    if (it >= max_it) break;
  }
  if (lead) {
    st->iter = it;
    st->status = status;
    st->converged = converged;
    st->r_norm = r_norm;
    st->rho = rho;
    st->beta = beta;
    st->first = first ? 1 : 0;
    st->done = 1;
  }
}

// ---------------------------------------------------------------------------
// Persistent PCG (one partition, one rank): the whole solve is ONE cooperative
// kernel. Each warp owns a fixed set of 32-row slices; an iteration is
//   phase A  q = A p_k (p_k = z_k + beta p_{k-1} formed on the fly, two
//            gathers), p_k of the own rows to the other p buffer, p.q
//   grid sync, every block reduces the per-block partials in the same fixed
//            order -> bitwise identical alpha everywhere
//   phase B  x += alpha p, r -= alpha q, z = D^-1 r, r.r and r.z
//   grid sync, reduce -> residual test, beta
// No kernel boundary, no launch gap, no host round trip per iteration. The
// vectors written inside the kernel are read with ld.global.cg (L2, never a
// stale L1 line); the matrix stream uses the read-only path.
// ---------------------------------------------------------------------------
constexpr int kPersistThreads = 256;
#ifndef WEFT_PERSIST_MINB
#define WEFT_PERSIST_MINB 2  // 16 warps/SM, no spills (measured best on B200 vs 3-6)
#endif
// L2 eviction priorities of the persistent kernel: the matrix (streamed
// once per iteration, 0.69 GB at config D) and phase B's own-row streams (r,
// x, D^-1) are loaded with an L2 evict_first policy, the z / p gathers with
// evict_last, so the gathered vectors stay resident in the 126 MB L2 while
// the matrix streams past them. Measured on B200, config D: 200 -> 168 us per
// PCG iteration together with WEFT_PK_UNROLL 1 (tools/pcg_ab.py; knobs:
// WEFT_MAT_EF, WEFT_VEC_EL, WEFT_PB_EF, WEFT_ZP_ST_EL = also store z / p
// with evict_last, measured equal).
#ifndef WEFT_ZP_ST_EL
#define WEFT_ZP_ST_EL 0  // phase A/B stores of p and z (gathered next phase A) with evict_last
#endif
#ifndef WEFT_PB_EF
#define WEFT_PB_EF 1  // phase B streams (r, x, D^-1) with evict_first
#endif
#ifndef WEFT_MAT_EF
#define WEFT_MAT_EF 1
#endif
#ifndef WEFT_VEC_EL
#define WEFT_VEC_EL 1
#endif
#ifndef WEFT_MAT_LD
#if WEFT_MAT_EF
#define WEFT_MAT_LD(p) ld_nc_hint(p, mpol)
#else
#define WEFT_MAT_LD(p) __ldg(p)
#endif
#endif
#if WEFT_VEC_EL
#define WEFT_VEC_LD(p) ld_cg_hint(p, vpol)
#else
#define WEFT_VEC_LD(p) __ldcg(p)
#endif
#ifndef WEFT_PK_UNROLL
#define WEFT_PK_UNROLL 1
#endif
constexpr int kPkUnroll = WEFT_PK_UNROLL;
#ifndef WEFT_DEEP_WIDTH
#define WEFT_DEEP_WIDTH 16
#endif
constexpr int kDeepWidth = WEFT_DEEP_WIDTH;  // slice width (slots) from which the unrolled row loop runs
#ifndef WEFT_PK_PREFETCH
#define WEFT_PK_PREFETCH 0
#endif
#ifndef WEFT_PK_XDEFER
#define WEFT_PK_XDEFER 1
#endif

// Vs = 4: inside the persistent solve the gathered vectors z and p are stored
// 32 bytes per row (xyz + pad), so a column gather is ONE 256-bit load
// (LDG.256, one sector) instead of three 8-byte loads (chosen per solve,
// pcg_solve's v4).
#pragma nv_diag_suppress 550  // the pad lane of the 256-bit loads is never read
__device__ __forceinline__ void ld4_cg(const double* p, uint64_t pol, double& a, double& b, double& c) {
  double d;  // the pad lane
  asm volatile("ld.global.cg.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p), "l"(pol));
  (void)d;
}
__device__ __forceinline__ void ld4_cg(const double* p, double& a, double& b, double& c) {
  double d;  // the pad lane
  asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
  (void)d;
}
#pragma nv_diag_default 550
__device__ __forceinline__ void st4_cg(double* p, double a, double b, double c) {
  asm volatile("st.global.cg.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(0.0) : "memory");
}
// own-row / gathered vector access of the persistent solve (stride Vs)
template <int Vs>
__device__ __forceinline__ void vload3(const double* v, int i, double& a, double& b, double& c) {
  if constexpr (Vs == 4) {
    ld4_cg(v + 4 * (size_t)i, a, b, c);
  } else {
    a = __ldcg(v + 3 * (size_t)i);
    b = __ldcg(v + 3 * (size_t)i + 1);
    c = __ldcg(v + 3 * (size_t)i + 2);
  }
}
template <int Vs>
__device__ __forceinline__ void vstore3(double* v, int i, double a, double b, double c) {
  if constexpr (Vs == 4) {
    st4_cg(v + 4 * (size_t)i, a, b, c);
  } else {
    __stcg(v + 3 * (size_t)i, a);
    __stcg(v + 3 * (size_t)i + 1, b);
    __stcg(v + 3 * (size_t)i + 2, c);
  }
}

// kC16: the column words as 16-bit offsets from the row's own position
// (c16, built per layout when every column of the system is within +-32767
// positions: 2 instead of 4 streamed bytes per block).
//
// kMir: the column word is 32 bits, the 16-bit column offset in the low half
// and in the high half the slot distance to the block's transposed twin
// (0: read the own block). A lower-triangle block that is bitwise the
// transpose of its upper twin is read from the twin, which the wavefront
// order streamed from HBM moments earlier: the second read is an L2 hit, so
// the symmetric part of the matrix crosses HBM once per iteration. Same
// values, same products, same order: bitwise the plain product.
template <int PMode, int kUnroll, int Vs, bool kC16, bool kMir = false>
__device__ __forceinline__ void row_product_cg(const SellView& A, int r, const double* __restrict__ z,
                                               const double* __restrict__ pold, double beta, double& y0, double& y1,
                                               double& y2, float vec_frac, const int16_t* __restrict__ c16,
                                               const uint32_t* __restrict__ cm = nullptr) {
#if WEFT_MAT_EF
  const uint64_t mpol = l2_policy_evict_first();
#endif
#if WEFT_VEC_EL
  const uint64_t vpol = l2_policy_evict_last_frac(vec_frac);
#endif
  const int len = A.rowlen[r];
  const int64_t base = A.slice_off[r >> 5] + (r & 31);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  auto col = [&](int64_t at) -> int {
    if constexpr (kC16) return r + WEFT_MAT_LD(c16 + at);
    else return WEFT_MAT_LD(A.cols + at) & kColMask;
  };
  uint32_t wn = 0;
  int cn = 0;
  if constexpr (kMir) wn = len > 0 ? __ldg(cm + base) : 0u;
  else cn = len > 0 ? col(base) : 0;
#pragma unroll kUnroll
  for (int k = 0; k < len; ++k) {
    const int64_t at = base + (int64_t)k * kSlice;
    int c;
    const double* v;
    int sa = 96, sb = 32;  // element (i, j) of the block at v + sa * i + sb * j
    if constexpr (kMir) {
      const uint32_t w = wn;
      if (k + 1 < len) wn = __ldg(cm + at + kSlice);
      c = r + static_cast<int>(static_cast<int16_t>(w & 0xffffu));
      const int d = static_cast<int>(static_cast<int16_t>(w >> 16));
      v = A.vals + (d ? vidx(at + d, c & 31, 0) : vidx(at, r & 31, 0));
      if (d) {
        sa = 32;
        sb = 96;
      }

    } else {
      c = cn;
      if (k + 1 < len) cn = col(at + kSlice);
      v = A.vals + vidx(at, r & 31, 0);
    }
    // kMir: default L2 policy (an evict_first stream drops the twins before
    // their second read; measured: HBM reads 89.6 vs 141 GB per solve)
    auto mld = [&](const double* q) -> double {
      if constexpr (kMir) return __ldg(q);
      else return WEFT_MAT_LD(q);
    };
    const double v0 = mld(v), v1 = mld(v + sb), v2 = mld(v + 2 * sb);
    const double v3 = mld(v + sa), v4 = mld(v + sa + sb), v5 = mld(v + sa + 2 * sb);
    const double v6 = mld(v + 2 * sa), v7 = mld(v + 2 * sa + sb), v8 = mld(v + 2 * sa + 2 * sb);
#if WEFT_VEC_EL
    double x0, x1, x2;
    if constexpr (Vs == 4) {
      ld4_cg(z + 4 * (size_t)c, vpol, x0, x1, x2);
    if (PMode == 2) {
      double q0, q1, q2;
      ld4_cg(pold + 4 * (size_t)c, vpol, q0, q1, q2);
      x0 = x0 + beta * q0;
      x1 = x1 + beta * q1;
      x2 = x2 + beta * q2;
    }
    } else {
      x0 = WEFT_VEC_LD(z + 3 * c);
      x1 = WEFT_VEC_LD(z + 3 * c + 1);
      x2 = WEFT_VEC_LD(z + 3 * c + 2);
      if (PMode == 2) {
        x0 = x0 + beta * WEFT_VEC_LD(pold + 3 * c);
        x1 = x1 + beta * WEFT_VEC_LD(pold + 3 * c + 1);
        x2 = x2 + beta * WEFT_VEC_LD(pold + 3 * c + 2);
      }
    }
#else
    double x0 = WEFT_VEC_LD(z + Vs * c), x1 = WEFT_VEC_LD(z + Vs * c + 1), x2 = WEFT_VEC_LD(z + Vs * c + 2);
    if (PMode == 2) {
      x0 = x0 + beta * WEFT_VEC_LD(pold + Vs * c);
      x1 = x1 + beta * WEFT_VEC_LD(pold + Vs * c + 1);
      x2 = x2 + beta * WEFT_VEC_LD(pold + Vs * c + 2);
    }
#endif
    a0 = a0 + ((v0 * x0 + v1 * x1) + v2 * x2);
    a1 = a1 + ((v3 * x0 + v4 * x1) + v5 * x2);
    a2 = a2 + ((v6 * x0 + v7 * x1) + v8 * x2);
  }
  y0 = a0;
  y1 = a1;
  y2 = a2;
}

// Sum of partials[i * NV + k] over i < n in a fixed order, result in every
// thread of the block (identical in every block).
template <int NV>
__device__ __forceinline__ void all_blocks_sum(const double* partials, int n, double (&out)[NV], double* smem) {
  double v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = v[k] + __ldcg(partials + (size_t)i * NV + k);
  block_sum<NV>(v, smem);
  __shared__ double bc[NV];
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) bc[k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = bc[k];
  __syncthreads();
}

// kQs: q = A p of the warp's rows stays in shared memory between phase A
// and phase B (phase B then walks the same slice runs): q never touches HBM.
// kUnroll: slots per row-loop trip. Grid rows (<= 13 slots) run best at 1;
// the long contact rows (up to ~40 slots) need the deeper unroll to keep
// enough gathers in flight (config D contacts mode: 44.1 -> 36.9 ms at 4).
// kMir: column words with mirror deltas (row_product_cg).
template <bool kQs, int kUnroll, int Vs, bool kC16, bool kMir = false>
__global__ void __launch_bounds__(kPersistThreads, WEFT_PERSIST_MINB) k_pcg_persistent(const PcgArgs* __restrict__ args, PcgState* st) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double smem[2 * 32];
  extern __shared__ double q_s[];  // kQs: [warp][slice of the run][component][lane]
  const PcgArgs& g = *args;
  const SellView A = g.A;
  const int rows = A.rows;
  const int nslices = (rows + kSlice - 1) / kSlice;
  const int warps = blockDim.x >> 5;
  const int gw = blockIdx.x * warps + (threadIdx.x >> 5), tw = gridDim.x * warps;
  const int lane = threadIdx.x & 31;
  const int G = gridDim.x;
  (void)nslices;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  double* __restrict__ x = g.x;
  double* __restrict__ r = g.r;
  double* __restrict__ z = g.z;
  double* __restrict__ q = g.q;
  double* pcur = g.p;
  double* pnew = g.p2;
  const double* __restrict__ dinv = g.dinv;
  const bool bj = g.bj != 0;
  double rho = st->rho;
  const double tol = st->tol, b_norm = st->b_norm;
  const int max_it = st->max_iter;
  double beta = 0.0, r_norm = st->r_norm;
  int it = 0, status = 0, converged = 0;
  bool done = st->done != 0;
  bool first = true;
  bool x_pending = false;  // x += alpha_prev * p (p in pnew of the last phase B) not applied yet
  double alpha_prev = 0.0;
  // Phase A work split: each warp takes a contiguous run of slices. A run
  // spans whole sigma windows, so every warp gets the same mix of long and
  // short rows (a strided assignment, with tw a multiple of the 8 slices
  // per window, gave some warps only the long window heads). Splitting by
  // equal slot counts instead measured slower on the hot path.
  //
  // kMir: instead, step j deals slices [j tw, (j+1) tw) to the warps,
  // rotated by j (warp gw takes slice j tw + (gw + j) mod tw), so the window
  // position a warp sees changes every step. The whole grid then sweeps the
  // matrix as one front a few tens of MB wide: a block's transposed twin in
  // a row ~nx positions back was streamed moments before (kMir reads it
  // from L2), and the front stays a contiguous HBM stream.
  constexpr bool wave = kMir;  // a runtime switch here costs the default order 11% (measured)
  const int sl_begin = wave ? 0 : static_cast<int>((static_cast<int64_t>(gw) * nslices) / tw);
  const int sl_end = wave ? (nslices + tw - 1) / tw
                          : static_cast<int>((static_cast<int64_t>(gw + 1) * nslices) / tw);
  auto slice_of = [&](int j) -> int { return wave ? j * tw + (gw + j) % tw : j; };
  double* const qw = q_s + static_cast<size_t>(threadIdx.x >> 5) * g.q_msw * 96 + lane;  // kQs: this warp's rows
#if WEFT_ZP_ST_EL
  const uint64_t elpol = l2_policy_evict_last();
#endif
#if WEFT_PB_EF
  const uint64_t efpol = l2_policy_evict_first();
#define PB_LD(p) ld_cg_hint(p, efpol)
#else
#define PB_LD(p) __ldcg(p)
#endif
  while (!done) {
    // ---- phase A: q = A p, p of the own rows, p.q
    unsigned long long tm0 = 0;
    if (g.timing && lead) tm0 = global_ns();
    double s1[1] = {0.0};
    for (int j = sl_begin; j < sl_end; ++j) {
      const int sl = slice_of(j);
#if WEFT_PK_PREFETCH == 1
      // stream this warp's next slice into L2 while this one computes
      if (lane == 0 && j + 1 < sl_end && slice_of(j + 1) < nslices) prefetch_slice_l2(A, slice_of(j + 1));
#elif WEFT_PK_PREFETCH == 2
      // request this slice's whole record stream at once (one bulk L2 prefetch)
      if (lane == 0 && sl < nslices) prefetch_slice_l2(A, sl);
#endif
      const int i = sl * kSlice + lane;  // matrix position == vector index (position space)
      if (sl < nslices && i < rows) {
        double y0, y1, y2;
        // kUnroll > 1 (systems with contacts): only the slices of long
        // (contact) rows take the unrolled loop; grid-row slices keep the
        // tighter single-slot loop (the slice width is warp-uniform)
        const bool deep = kUnroll > 1 && (A.slice_off[sl + 1] - A.slice_off[sl]) > kDeepWidth * kSlice;
        if (deep) {
          if (first)
            row_product_cg<1, kUnroll, Vs, kC16, kMir>(A, i, z, pcur, beta, y0, y1, y2, g.vec_el_frac, g.colp16,
                                                       g.mwords);
          else
            row_product_cg<2, kUnroll, Vs, kC16, kMir>(A, i, z, pcur, beta, y0, y1, y2, g.vec_el_frac, g.colp16,
                                                       g.mwords);
        } else {
          if (first)
            row_product_cg<1, 1, Vs, kC16, kMir>(A, i, z, pcur, beta, y0, y1, y2, g.vec_el_frac, g.colp16,
                                                 g.mwords);
          else
            row_product_cg<2, 1, Vs, kC16, kMir>(A, i, z, pcur, beta, y0, y1, y2, g.vec_el_frac, g.colp16,
                                                 g.mwords);
        }
        double p0, p1, p2;
        vload3<Vs>(z, i, p0, p1, p2);
        if (!first) {
          double o0, o1, o2;
          vload3<Vs>(pcur, i, o0, o1, o2);
          p0 = p0 + beta * o0;
          p1 = p1 + beta * o1;
          p2 = p2 + beta * o2;
        }
        if constexpr (kQs) {
          double* qq = qw + (j - sl_begin) * 96;
          qq[0] = y0;
          qq[32] = y1;
          qq[64] = y2;
        } else {
          __stcg(q + 3 * i, y0);
          __stcg(q + 3 * i + 1, y1);
          __stcg(q + 3 * i + 2, y2);
        }
        vstore3<Vs>(pnew, i, p0, p1, p2);
        s1[0] = s1[0] + ((p0 * y0 + p1 * y1) + p2 * y2);
      }
    }
    block_sum<1>(s1, smem);
    if (threadIdx.x == 0) __stcg(g.partials + blockIdx.x, s1[0]);
    unsigned long long tm1 = 0;
    if (g.timing && lead) tm1 = global_ns();
    grid.sync();
    if (g.timing && lead) {
      const unsigned long long tm2 = global_ns();
      g.timing[0] += tm1 - tm0;  // phase A (block 0's view)
      g.timing[1] += tm2 - tm1;  // grid sync 1
    }
    double pq[1];
    all_blocks_sum<1>(g.partials, G, pq, smem);
    if (!isfinite(pq[0])) {
      status = 1;
      ++it;
      break;
    }
    if (pq[0] <= 0.0) {
      status = 2;
      ++it;
      break;
    }
    const double alpha = rho / pq[0];
    // ---- phase B: x, r, z (coalesced; q and p of phase A are visible after
    // the grid sync, read through L2). The x update of every other iteration
    // is deferred and applied with the next one as (x + a_k p_k) + a_k+1 p_k+1
    // — the same two roundings in the same order, one x round trip fewer.
    const bool x_now = !WEFT_PK_XDEFER || x_pending;
    double s2[2] = {0.0, 0.0};
    // kQs: the rows of this warp's slice run (q from shared memory);
    // otherwise row-linear over the grid
    const int pb_begin = kQs ? sl_begin : blockIdx.x * blockDim.x + threadIdx.x;
    const int pb_end = kQs ? sl_end : rows;
    const int pb_step = kQs ? 1 : gridDim.x * blockDim.x;
    for (int t = pb_begin; t < pb_end; t += pb_step) {
      const int i = kQs ? slice_of(t) * kSlice + lane : t;
      if (kQs && i >= rows) continue;
      double qv[3], rv[3], m[9];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if constexpr (kQs) qv[c] = qw[(t - sl_begin) * 96 + 32 * c];
        else qv[c] = __ldcg(q + 3 * i + c);
        rv[c] = PB_LD(r + 3 * i + c);
      }
      if (x_now) {
        double xv[3], pv[3];
        vload3<Vs>(pnew, i, pv[0], pv[1], pv[2]);
#pragma unroll
        for (int c = 0; c < 3; ++c) xv[c] = PB_LD(x + 3 * i + c);
        if (WEFT_PK_XDEFER) {
          double po[3];
          vload3<Vs>(pcur, i, po[0], po[1], po[2]);
#pragma unroll
          for (int c = 0; c < 3; ++c) xv[c] = xv[c] + alpha_prev * po[c];
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) __stcg(x + 3 * i + c, xv[c] + alpha * pv[c]);
      }
      if (bj) {
        if (g.dinv6) {  // bitwise-symmetric inverses: 48 instead of 72 bytes per row
          const double* h = g.dinv6 + 6 * (size_t)i;
#if WEFT_PB_EF
          m[0] = ld_nc_hint(h, efpol);
          m[1] = m[3] = ld_nc_hint(h + 1, efpol);
          m[2] = m[6] = ld_nc_hint(h + 2, efpol);
          m[4] = ld_nc_hint(h + 3, efpol);
          m[5] = m[7] = ld_nc_hint(h + 4, efpol);
          m[8] = ld_nc_hint(h + 5, efpol);
#else
          m[0] = __ldg(h);
          m[1] = m[3] = __ldg(h + 1);
          m[2] = m[6] = __ldg(h + 2);
          m[4] = __ldg(h + 3);
          m[5] = m[7] = __ldg(h + 4);
          m[8] = __ldg(h + 5);
#endif
        } else {
#pragma unroll
          for (int k = 0; k < 9; ++k) m[k] = __ldg(dinv + 9 * (size_t)i + k);
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) rv[c] = rv[c] - alpha * qv[c];
      double z0, z1, z2;
      if (bj) {  // apply_precond (solver.hpp:67-89)
        z0 = ((0.0 + m[0] * rv[0]) + m[1] * rv[1]) + m[2] * rv[2];
        z1 = ((0.0 + m[3] * rv[0]) + m[4] * rv[1]) + m[5] * rv[2];
        z2 = ((0.0 + m[6] * rv[0]) + m[7] * rv[1]) + m[8] * rv[2];
      } else {
        z0 = rv[0];
        z1 = rv[1];
        z2 = rv[2];
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) __stcg(r + 3 * i + c, rv[c]);
      vstore3<Vs>(z, i, z0, z1, z2);
      s2[0] = s2[0] + ((rv[0] * rv[0] + rv[1] * rv[1]) + rv[2] * rv[2]);
      s2[1] = s2[1] + ((rv[0] * z0 + rv[1] * z1) + rv[2] * z2);
    }
    x_pending = !x_now;
    alpha_prev = alpha;
    block_sum<2>(s2, smem);
    if (threadIdx.x == 0) {
      __stcg(g.partials + G + 2 * blockIdx.x, s2[0]);
      __stcg(g.partials + G + 2 * blockIdx.x + 1, s2[1]);
    }
    unsigned long long tm3 = 0;
    if (g.timing && lead) tm3 = global_ns();
    grid.sync();
    if (g.timing && lead) {
      const unsigned long long tm4 = global_ns();
      g.timing[2] += tm3 - tm0;  // iteration up to sync 2 (A + sync + reduce + B)
      g.timing[3] += tm4 - tm3;  // grid sync 2
    }
    double t[2];
    all_blocks_sum<2>(g.partials + G, G, t, smem);
    ++it;
    r_norm = sqrt(t[0]);
    if (!isfinite(r_norm)) {
      status = 3;
      break;
    }
    if (lead) {
      g.hist[it - 1] = r_norm / b_norm;
      g.phist[it - 1] = sqrt(t[1] > 0.0 ? t[1] : 0.0);
    }
    if (r_norm <= tol) {
      converged = 1;
      break;
    }
    beta = t[1] / rho;
    rho = t[1];
    if (it >= max_it) break;
    double* tmp = pcur;
    pcur = pnew;
    pnew = tmp;
    first = false;
  }
  if (x_pending && status == 0) {
    // the last iteration's deferred x update (its p is in pnew: the swap
    // below the residual test is skipped on exit), over phase B's rows
    const int pb_begin = kQs ? sl_begin : blockIdx.x * blockDim.x + threadIdx.x;
    const int pb_end = kQs ? sl_end : rows;
    const int pb_step = kQs ? 1 : gridDim.x * blockDim.x;
    for (int t = pb_begin; t < pb_end; t += pb_step) {
      const int i = kQs ? slice_of(t) * kSlice + lane : t;
      if (kQs && i >= rows) continue;
      double pv[3];
      vload3<Vs>(pnew, i, pv[0], pv[1], pv[2]);
#pragma unroll
      for (int c = 0; c < 3; ++c) __stcg(x + 3 * i + c, __ldcg(x + 3 * i + c) + alpha_prev * pv[c]);
    }
  }
  if (lead) {
    st->iter = it;
    st->status = status;
    st->converged = converged;
    st->r_norm = r_norm;
    st->rho = rho;
    st->beta = beta;
    st->done = 1;
  }
}

// Position-space column words (one partition: no group bits; padding stays -1).
__global__ void k_colpos(int64_t total, const int32_t* __restrict__ cols, const int32_t* __restrict__ pos,
                         int32_t* __restrict__ colp) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int c = cols[i];
  colp[i] = c < 0 ? c : pos[c & kColMask];
}

// 16-bit position offsets of the column words (slot at of slice s, lane l:
// row position s * 32 + l); *bad = 1 if any live column is out of range.
__global__ void k_colpos16(int nslices, const int64_t* __restrict__ soff, const int32_t* __restrict__ rowlen,
                           const int32_t* __restrict__ colp, int16_t* __restrict__ c16, int* __restrict__ bad) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= nslices * kSlice) return;
  const int len = rowlen[m];
  const int64_t base = soff[m >> 5] + (m & 31);
  for (int k = 0; k < len; ++k) {
    const int d = colp[base + (int64_t)k * kSlice] - m;
    if (d < -32768 || d > 32767) atomicOr(bad, 1);
    c16[base + (int64_t)k * kSlice] = static_cast<int16_t>(d);
  }
}

// Twins of the lower-triangle blocks, once per layout (position space, one
// partition): pair_at[slot of (m, c)] = slot of (c, m) for c < m, else -1.
__global__ void k_pair_at(int nslices, const int64_t* __restrict__ soff, const int32_t* __restrict__ rowlen,
                          const int32_t* __restrict__ colp, int32_t* __restrict__ pair_at) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= nslices * kSlice) return;
  const int len = rowlen[m];
  const int64_t base = soff[m >> 5] + (m & 31);
  for (int k = 0; k < len; ++k) {
    const int64_t at = base + (int64_t)k * kSlice;
    const int c = colp[at];
    int64_t pa = -1;
    if (c >= 0 && c < m) {
      const int lc = rowlen[c];
      const int64_t bc = soff[c >> 5] + (c & 31);
      for (int k2 = 0; k2 < lc; ++k2)
        if (colp[bc + (int64_t)k2 * kSlice] == m) {
          pa = bc + (int64_t)k2 * kSlice;
          break;
        }
    }
    pair_at[at] = static_cast<int32_t>(pa);
  }
}

// Column words of the mirrored persistent solve, per solve (the values
// change every step): low 16 bits the column offset; high 16 bits, for a
// lower block that is BITWISE the transpose of its twin (slot distance
// within +-32767), that distance, else 0. *nmir counts mirrored blocks.
__global__ void k_mirror_words(int nslices, const int64_t* __restrict__ soff, const int32_t* __restrict__ rowlen,
                               const int16_t* __restrict__ c16, const int32_t* __restrict__ pair_at,
                               const double* __restrict__ vals, uint32_t* __restrict__ words,
                               unsigned long long* __restrict__ nmir) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned n = 0;
  if (m < nslices * kSlice) {
    const int len = rowlen[m];
    const int64_t base = soff[m >> 5] + (m & 31);
    for (int k = 0; k < len; ++k) {
      const int64_t at = base + (int64_t)k * kSlice;
      const int off = c16[at];
      uint32_t w = static_cast<uint16_t>(off);
      const int64_t pa = pair_at[at];
      const int64_t d = pa - at;
      if (pa >= 0 && d >= -32767 && d <= 32767) {
        const int c = m + off;
        const double* own = vals + vidx(at, m & 31, 0);
        const double* tw = vals + vidx(pa, c & 31, 0);
        bool eq = true;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j)
            eq = eq && __double_as_longlong(__ldg(own + 96 * i + 32 * j)) ==
                           __double_as_longlong(__ldg(tw + 32 * i + 96 * j));
        if (eq) {
          w |= static_cast<uint32_t>(static_cast<uint16_t>(static_cast<int16_t>(d))) << 16;
          ++n;
        }
      }
      words[at] = w;
    }
  }
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(nmir, static_cast<unsigned long long>(n));
}

// PCG init in position space: r = b[perm], z = M^-1 r, x = 0, p = 0.
__global__ void k_pcg_init_pos(int rows, const int32_t* __restrict__ perm, const double* __restrict__ b,
                               const double* __restrict__ dinv, bool bj, double* __restrict__ x,
                               double* __restrict__ r, double* __restrict__ z, double* __restrict__ p,
                               double* __restrict__ z4, double* __restrict__ p4) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= rows) return;
  const int i = perm[m];
  const double b0 = b[3 * i], b1 = b[3 * i + 1], b2 = b[3 * i + 2];
  double z0, z1, z2;
  precond_row(dinv, bj, m, b0, b1, b2, z0, z1, z2);
  x[3 * m] = x[3 * m + 1] = x[3 * m + 2] = 0.0;
  r[3 * m] = b0;
  r[3 * m + 1] = b1;
  r[3 * m + 2] = b2;
  z[3 * m] = z0;
  z[3 * m + 1] = z1;
  z[3 * m + 2] = z2;
  p[3 * m] = p[3 * m + 1] = p[3 * m + 2] = 0.0;
  if (z4) {  // the persistent solve's 32-byte-per-row copies (v4)
    z4[4 * (size_t)m] = z0;
    z4[4 * (size_t)m + 1] = z1;
    z4[4 * (size_t)m + 2] = z2;
    z4[4 * (size_t)m + 3] = 0.0;
    p4[4 * (size_t)m] = p4[4 * (size_t)m + 1] = p4[4 * (size_t)m + 2] = p4[4 * (size_t)m + 3] = 0.0;
  }
}

// out[perm[m]] = in[m] (3 doubles per row).
__global__ void k_scatter_rows(int rows, const int32_t* __restrict__ perm, const double* __restrict__ in,
                               double* __restrict__ out) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= rows) return;
  const int i = perm[m];
  out[3 * i] = in[3 * m];
  out[3 * i + 1] = in[3 * m + 1];
  out[3 * i + 2] = in[3 * m + 2];
}

void pcg_free(Ctx& c) {
  if (c.pcg_exec) cudaGraphExecDestroy(c.pcg_exec);
  c.pcg_exec = nullptr;
  if (c.pcg) cudaFree(c.pcg);
  if (c.pcg_host) cudaFreeHost(c.pcg_host);
  c.pcg = nullptr;
  c.pcg_host = nullptr;
}

PcgResult pcg_solve(Ctx& c, const double* b_dev, const weft_pcg_config& cfg, double* hist_host,
                    double* phist_host) {
  if (!c.has_matrix) throw Error(WEFT_ERR_INVALID, "pcg: no matrix");
  if (c.A.f32) throw Error(WEFT_ERR_INVALID, "pcg: single-precision system (use the f32 entry)");
  comm_need(c, "pcg");
  const int rows = c.A.rows;                               // held rows
  const size_t len = 3 * static_cast<size_t>(c.pm.p);      // vectors: global row index
  const int threads = 256;
  const bool peers = c.world > 1;
  // One partition on one rank: the whole solve is one persistent kernel in
  // POSITION space (vectors and columns permuted to the SELL-32-sigma order,
  // b gathered in, x scattered out), so every vector access is coalesced.
  const bool persistent = c.go.n == 1 && c.world == 1 && c.use_persistent;
  // otherwise (several partitions or ranks) one cooperative kernel per rank
  // too, in row space (WEFT_PCG_ROWS=0: the graph of two kernels per iteration)
  static const bool rows_off = std::getenv("WEFT_PCG_ROWS") && std::atoi(std::getenv("WEFT_PCG_ROWS")) == 0;
  const bool prows = !persistent && c.use_persistent && !rows_off;
  // z / p at 32 bytes per row inside the persistent solve (one LDG.256 per
  // gather) while 64 B per row of them fit ~100 MB of L2; beyond (the 5-10 M
  // triangle configs) the 24-byte rows move fewer bytes (E5: 97.5 vs 103.6 ms)
  static const int vs_env = std::getenv("WEFT_PCG_VS") ? std::atoi(std::getenv("WEFT_PCG_VS")) : 0;
  const bool v4 = vs_env ? vs_env == 4 : (64.0 * rows <= 100e6);
  if (!c.pcg) {
    WG_CUDA(cudaMalloc(&c.pcg, sizeof(PcgState)));
    WG_CUDA(cudaHostAlloc(&c.pcg_host, sizeof(PcgState), cudaHostAllocDefault));
  }
  for (auto* v : {&c.r, &c.z, &c.pv, &c.q, &c.xs}) v->resize(len);
  const bool bj = cfg.preconditioner == WEFT_PRECOND_BLOCK_JACOBI;
  c.dinv.resize(9 * static_cast<size_t>(c.pm.p) + 9);
  const int max_it = std::max(cfg.max_iterations, 0);
  c.hist.resize(static_cast<size_t>(max_it) + 1);
  c.phist.resize(static_cast<size_t>(max_it) + 1);
  const PartBlocks pb = part_blocks(c, threads);
  const int nblocks = pb.bstart[pb.n];
  c.partials.resize(4 * static_cast<size_t>(nblocks) + 4);
  const SellView A = view(c.A);
  cudaStream_t s = c.stream;

  PcgState init{};
  init.max_iter = max_it;
  init.first = 1;
  WG_CUDA(cudaMemcpyAsync(c.pcg, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  double* dots = reinterpret_cast<double*>(c.scalars.data());
  int* dinv_asym = reinterpret_cast<int*>(c.scalars.data() + 12);
  auto* nmir = reinterpret_cast<unsigned long long*>(c.scalars.data() + 14);
  bool mir = false;
  if (rows > 0) {
    if (persistent) {
      if (c.A.colp_id != c.A.layout_id) {  // position-space column words, once per layout
        c.A.colp.resize(static_cast<size_t>(c.A.total) + 1);
        if (c.A.total)
          k_colpos<<<div_up(c.A.total, 256), 256, 0, ls(c)>>>(c.A.total, c.A.cols.data(), c.A.pos.data(),
                                                               c.A.colp.data());
        // 16-bit offsets when every column is within +-32767 positions of its
        // row (grid meshes: the row bandwidth 2 nx + 1 plus the sigma window)
        static const bool c16_off = std::getenv("WEFT_PCG_C16") && std::atoi(std::getenv("WEFT_PCG_C16")) == 0;
        c.A.colp16_ok = false;
        if (!c16_off && c.A.total) {
          c.A.colp16.resize(static_cast<size_t>(c.A.total) + 1);
          int* bad = reinterpret_cast<int*>(c.scalars.data() + 13);
          WG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
          k_colpos16<<<div_up(c.A.nslices * kSlice, 256), 256, 0, ls(c)>>>(
              c.A.nslices, c.A.slice_off.data(), c.A.rowlen.data(), c.A.colp.data(), c.A.colp16.data(), bad);
          int hbad = 1;
          WG_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
          WG_CUDA(cudaStreamSynchronize(s));
          c.A.colp16_ok = hbad == 0;
        }
        c.A.colp_id = c.A.layout_id;
      }
      // kMir: lower-triangle blocks read from their bitwise-transposed twins
      // (opt-in, WEFT_PCG_MIRROR=1: HBM reads drop 126 -> 90 GB per config-D
      // solve but the solve time does not move, ~27 ms either way — the
      // kernel is latency-bound, not HBM-bound)
      static const bool mir_on = std::getenv("WEFT_PCG_MIRROR") && std::atoi(std::getenv("WEFT_PCG_MIRROR")) == 1;
      mir = mir_on && c.A.colp16_ok && v4 && c.A.total > 0 && c.A.total < (int64_t{1} << 31);
      if (mir) {
        if (c.A.pair_id != c.A.layout_id) {
          c.A.pair_at.resize(static_cast<size_t>(c.A.total) + 1);
          k_pair_at<<<div_up(c.A.nslices * kSlice, 256), 256, 0, ls(c)>>>(
              c.A.nslices, c.A.slice_off.data(), c.A.rowlen.data(), c.A.colp.data(), c.A.pair_at.data());
          c.A.pair_id = c.A.layout_id;
        }
        c.A.mwords.resize(static_cast<size_t>(c.A.total) + 1);
        WG_CUDA(cudaMemsetAsync(nmir, 0, sizeof(unsigned long long), s));
        k_mirror_words<<<div_up(c.A.nslices * kSlice, 256), 256, 0, ls(c)>>>(
            c.A.nslices, c.A.slice_off.data(), c.A.rowlen.data(), c.A.colp16.data(), c.A.pair_at.data(),
            c.A.vals.data(), c.A.mwords.data(), nmir);
      }
      c.xp.resize(len);
      c.dinv6.resize(6 * static_cast<size_t>(rows) + 6);
      WG_CUDA(cudaMemsetAsync(dinv_asym, 0, sizeof(int), s));
      if (bj) k_dinv<true><<<div_up(rows, threads), threads, 0, ls(c)>>>(A, c.dinv.data(), c.dinv6.data(), dinv_asym);
      if (v4) {
        c.z4.resize(4 * static_cast<size_t>(rows) + 4);
        c.p4a.resize(4 * static_cast<size_t>(rows) + 4);
        c.p4b.resize(4 * static_cast<size_t>(rows) + 4);
      }
      k_pcg_init_pos<<<div_up(rows, threads), threads, 0, ls(c)>>>(
          rows, c.A.perm.data(), b_dev, c.dinv.data(), bj, c.xp.data(), c.r.data(), c.z.data(), c.pv.data(),
          v4 ? c.z4.data() : nullptr, v4 ? c.p4a.data() : nullptr);
      // ||b|| and rho = r.z over the permuted r = b
      k_dot2<<<nblocks, threads, 0, ls(c)>>>(pb, c.r.data(), c.r.data(), c.r.data(), c.z.data(), c.partials.data(),
                                         &c.pcg->counter, dots, c.comm, c.nparts);
    } else {
      if (bj) k_dinv<false><<<div_up(rows, threads), threads, 0, ls(c)>>>(A, c.dinv.data());
      k_pcg_init<<<div_up(rows, threads), threads, 0, ls(c)>>>(c.row0, rows, b_dev, c.dinv.data(), bj, c.xs.data(),
                                                           c.r.data(), c.z.data(), c.pv.data());
      if (peers) publish_vectors(c);  // z of the held rows, gathered by the first SpMV
      // ||b|| and rho = r.z (r = b)
      k_dot2<<<nblocks, threads, 0, ls(c)>>>(pb, b_dev, b_dev, c.r.data(), c.z.data(), c.partials.data(),
                                         &c.pcg->counter, dots, c.comm, c.nparts);
    }
    WG_CUDA(cudaGetLastError());
  }
  double hd[2] = {0.0, 0.0};
  int asym = 1;
  if (rows > 0 && persistent && bj)
    read_small(c, s, {dots, hd, sizeof(hd)}, {dinv_asym, &asym, sizeof(int)});
  else if (rows > 0)
    read_small(c, s, {dots, hd, sizeof(hd)});
  else
    WG_CUDA(cudaStreamSynchronize(s));
  comm_check(c);
  PcgResult res;
  const double b_norm = std::sqrt(hd[0]);
  if (b_norm == 0.0) {
    res.converged = 1;
    return res;
  }
  init.b_norm = b_norm;
  init.tol = cfg.rel_tolerance * b_norm;
  init.rho = hd[1];
  init.r_norm = b_norm;
  init.done = max_it == 0 ? 1 : 0;
  WG_CUDA(cudaMemcpyAsync(c.pcg, &init, sizeof(init), cudaMemcpyHostToDevice, s));

  // per-solve argument block (device)
  const PartBlocks pb2 = part_blocks(c, threads / 2);
  const int nblocks2 = pb2.bstart[pb2.n];
  int pgrid = 0, msw = 0;
  size_t qs_bytes = 0;
  static const int unroll_env = std::getenv("WEFT_PCG_UNROLL") ? std::atoi(std::getenv("WEFT_PCG_UNROLL")) : 0;
  const int unroll = (unroll_env ? unroll_env : (c.n_contacts > 0 ? 4 : kPkUnroll)) >= 4 ? 4 : 1;
  const bool c16 = persistent && c.A.colp16_ok;
  auto pick = [&](bool q) -> decltype(&k_pcg_persistent<false, 1, 3, false>) {
    if (mir) {
      if (unroll == 4) return q ? k_pcg_persistent<true, 4, 4, true, true> : k_pcg_persistent<false, 4, 4, true, true>;
      return q ? k_pcg_persistent<true, 1, 4, true, true> : k_pcg_persistent<false, 1, 4, true, true>;
    }
    if (c16) {
      if (v4) {
        if (unroll == 4) return q ? k_pcg_persistent<true, 4, 4, true> : k_pcg_persistent<false, 4, 4, true>;
        return q ? k_pcg_persistent<true, 1, 4, true> : k_pcg_persistent<false, 1, 4, true>;
      }
      if (unroll == 4) return q ? k_pcg_persistent<true, 4, 3, true> : k_pcg_persistent<false, 4, 3, true>;
      return q ? k_pcg_persistent<true, 1, 3, true> : k_pcg_persistent<false, 1, 3, true>;
    }
    if (v4) {
      if (unroll == 4) return q ? k_pcg_persistent<true, 4, 4, false> : k_pcg_persistent<false, 4, 4, false>;
      return q ? k_pcg_persistent<true, 1, 4, false> : k_pcg_persistent<false, 1, 4, false>;
    }
    if (unroll == 4) return q ? k_pcg_persistent<true, 4, 3, false> : k_pcg_persistent<false, 4, 3, false>;
    return q ? k_pcg_persistent<true, 1, 3, false> : k_pcg_persistent<false, 1, 3, false>;
  };

  auto pkern = pick(false);
  if (persistent) {
    // q in shared memory when the warps' slice runs fit at two CTAs per SM
    int sms = 0;
    WG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    const int warps_per_cta = kPersistThreads / 32;
    const int nsl = div_up(rows, kSlice);
    msw = div_up(nsl, static_cast<int64_t>(sms) * WEFT_PERSIST_MINB * warps_per_cta);
    qs_bytes = static_cast<size_t>(warps_per_cta) * msw * 96 * sizeof(double);
    static const bool qs_off = std::getenv("WEFT_PCG_QSMEM") && std::atoi(std::getenv("WEFT_PCG_QSMEM")) == 0;
    // q in shared memory: 29.2 -> 28.0 ms at config D without contacts. With
    // contact elements it first measured slower (52.5 vs 50.3 ms: the 67 KB
    // of q per CTA come out of L1, which the far contact gathers used); since
    // the unrolled row loop runs only in the wide contact slices it is faster
    // there too (34.5 -> 33.3 ms).
    const bool qs = !qs_off && qs_bytes <= 100 * 1024;
    if (qs) {
      pkern = pick(true);
      WG_CUDA(cudaFuncSetAttribute(pkern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(qs_bytes)));
    } else {
      qs_bytes = 0;
    }
    int occ = 0;
    WG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pkern, kPersistThreads, qs_bytes));
    pgrid = std::max(1, occ) * sms;
    if (qs && static_cast<int64_t>(pgrid) * warps_per_cta * msw < nsl)
      throw Error(WEFT_ERR_EXEC, "pcg: persistent grid smaller than planned (" + std::to_string(pgrid) + " CTAs)");
    c.p2.resize(len);
    if (c.partials.size() < 3 * static_cast<size_t>(pgrid) + 4) c.partials.resize(3 * static_cast<size_t>(pgrid) + 4);
  }
  PcgArgs args{A, pb, pb2, c.go.n, bj ? 1 : 0, c.dinv.data(), c.xs.data(), c.r.data(), c.z.data(), c.pv.data(),
               c.q.data(), c.partials.data(), c.hist.data(), c.phist.data(), c.comm, c.pm, c.p2.data()};
  if (persistent) {
    args.A.cols = c.A.colp.data();  // columns as positions
    args.colp16 = c16 ? c.A.colp16.data() : nullptr;
    args.mwords = mir ? c.A.mwords.data() : nullptr;
    args.x = c.xp.data();
    if (v4) {  // gathered vectors 32 bytes per row
      args.z = c.z4.data();
      args.p = c.p4a.data();
      args.p2 = c.p4b.data();
    }
    args.q_msw = msw;
    // z and p (48 B per row) are gathered every iteration: pin them in L2
    // while they fit in ~60 MB of its 126 MB, a proportional fraction beyond
    // (the 5-10 M triangle sweep configs)
    static const double el_budget = std::getenv("WEFT_PCG_EL_MB") ? std::atof(std::getenv("WEFT_PCG_EL_MB")) : 60.0;
    args.vec_el_frac = static_cast<float>(std::min(1.0, el_budget * 1e6 / (48.0 * std::max(rows, 1))));
    static const bool d6_off = std::getenv("WEFT_PCG_DINV6") && std::atoi(std::getenv("WEFT_PCG_DINV6")) == 0;
    args.dinv6 = (bj && !asym && !d6_off) ? c.dinv6.data() : nullptr;
    if (std::getenv("WEFT_PCG_TIMING")) {
      c.timing.resize(8);
      c.timing.zero(s);
      args.timing = c.timing.data();
    }
  }
  c.pcg_args.resize(sizeof(PcgArgs));
  const PcgArgs* dargs = reinterpret_cast<const PcgArgs*>(c.pcg_args.data());
  WG_CUDA(cudaMemcpyAsync(c.pcg_args.data(), &args, sizeof(args), cudaMemcpyHostToDevice, s));
  const bool pair = c.go.n == 1 && c.spmv_pair;
  auto spmv_kernel = c.go.n == 1 ? (pair ? k_pcg_spmv<true, true, false> : k_pcg_spmv<true, false, false>)
                                 : (peers ? k_pcg_spmv<false, false, true> : k_pcg_spmv<false, false, false>);
  auto* hs = static_cast<PcgState*>(c.pcg_host);

  if (persistent) {
    // the whole solve: one cooperative launch (co-resident grid, grid syncs)
    void* kargs[] = {(void*)&dargs, (void*)&c.pcg};
    if (c.profile) WG_CUDA(cudaEventRecord(c.ev[6], s));
    WG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(pkern), dim3(pgrid), dim3(kPersistThreads), kargs,
                                        qs_bytes, s));
    ++c.launches;
    if (c.profile) WG_CUDA(cudaEventRecord(c.ev[7], s));
    k_scatter_rows<<<div_up(rows, threads), threads, 0, ls(c)>>>(rows, c.A.perm.data(), c.xp.data(), c.xs.data());
    read_small(c, s, {c.pcg, hs, sizeof(PcgState)});
    if (args.timing && hs->iter) {
      unsigned long long t[4];
      WG_CUDA(cudaMemcpy(t, args.timing, sizeof(t), cudaMemcpyDeviceToHost));
      std::fprintf(stderr, "[pcg timing] its %d  phaseA %.1f us  sync1 %.1f us  reduce+phaseB %.1f us  sync2 %.1f us\n",
                   hs->iter, t[0] * 1e-3 / hs->iter, t[1] * 1e-3 / hs->iter,
                   (t[2] - t[0] - t[1]) * 1e-3 / hs->iter, t[3] * 1e-3 / hs->iter);
    }
    if (c.profile) {
      float ms = 0.f;
      WG_CUDA(cudaEventElapsedTime(&ms, c.ev[6], c.ev[7]));
      c.pcg_ms += ms;
      c.pcg_iterations += hs->iter;
      ++c.pcg_solves;
      // algorithmic bytes per iteration: 76 per streamed live
      // block; per row phase A 4 + 2*24 gathered + 24 p written (+ 24 q
      // written unless q stays in shared memory), phase B 24 r + 72 D^-1
      // read, 48 r, z written, 48 for x / p every other iteration (+ 24 q
      // read unless shared)
      const double per_row =
          4.0 + 48.0 + 24.0 + 24.0 + (args.dinv6 ? 48.0 : 72.0) + 48.0 + 48.0 + (qs_bytes ? 0.0 : 48.0);
      // kMir: mirrored blocks come from L2, not HBM (their 72 bytes are not
      // counted); the column word is 4 bytes
      // (kMir reads its mirrored blocks from L2: fewer HBM bytes than this
      // algorithmic count, which stays the SURVEY 8(d) figure)
      unsigned long long nm = 0;
      if (mir) WG_CUDA(cudaMemcpy(&nm, nmir, sizeof(nm), cudaMemcpyDeviceToHost));
      c.pcg_mirrored = static_cast<int64_t>(nm);
      c.pcg_bytes += hs->iter * (76.0 * static_cast<double>(c.A.nnzb) + per_row * rows);
    }
  } else if (prows) {
    // several partitions and/or ranks: the two iteration kernels fused into
    // one cooperative launch per rank (bitwise the graph path's iterates)
    auto k = peers ? k_pcg_persistent_rows<true> : k_pcg_persistent_rows<false>;
    int sms = 0, occ = 0;
    WG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    WG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, 0));
    const int grid = std::max(1, std::min(std::max(1, occ) * sms, nblocks));
    void* kargs[] = {(void*)&dargs, (void*)&c.pcg};
    if (c.profile) WG_CUDA(cudaEventRecord(c.ev[6], s));
    WG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k), dim3(grid), dim3(threads), kargs, 0, s));
    ++c.launches;
    if (c.profile) WG_CUDA(cudaEventRecord(c.ev[7], s));
    WG_CUDA(cudaMemcpyAsync(hs, c.pcg, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    if (c.profile) {
      float ms = 0.f;
      WG_CUDA(cudaEventElapsedTime(&ms, c.ev[6], c.ev[7]));
      c.pcg_ms += ms;
      c.pcg_iterations += hs->iter;
      ++c.pcg_solves;
      // SpMV 76 B per streamed block + 4 length + 48 gathered z, p + 24 q
      // written per row; update 288 B per row
      c.pcg_bytes += hs->iter * (76.0 * static_cast<double>(c.A.nnzb) + (76.0 + 288.0) * rows);
    }
  } else if (!c.profile && c.use_graphs) {
    // The whole solve is one graph launch: a conditional WHILE node whose
    // body is the two iteration kernels; the update kernel's last block
    // clears the condition when the solve is done.
    const bool single = c.go.n == 1;
    if (!c.pcg_exec || c.pcg_exec_blocks != nblocks || c.pcg_exec_single != single || c.pcg_exec_pair != pair) {
      if (c.pcg_exec) cudaGraphExecDestroy(c.pcg_exec);
      c.pcg_exec = nullptr;
      cudaGraph_t graph = nullptr;
      bool ok = cudaGraphCreate(&graph, 0) == cudaSuccess;
      cudaGraphConditionalHandle cond = 0;
      cudaGraph_t body = nullptr;
      if (ok) ok = cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault) == cudaSuccess;
      if (ok) {
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = cond;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        ok = cudaGraphAddNode(&node, graph, nullptr, 0, &cp) == cudaSuccess;
        if (ok) body = cp.conditional.phGraph_out[0];
      }
      if (ok) {
        cudaKernelNodeParams k1{};
        void* a1[] = {(void*)&dargs, (void*)&c.pcg};
        k1.func = reinterpret_cast<void*>(spmv_kernel);
        k1.gridDim = dim3(pair ? nblocks2 : nblocks);
        k1.blockDim = dim3(threads);
        k1.kernelParams = a1;
        int use = 1;
        cudaKernelNodeParams k2{};
        void* a2[] = {(void*)&dargs, (void*)&c.pcg, (void*)&cond, (void*)&use};
        k2.func = reinterpret_cast<void*>(k_pcg_update);
        k2.gridDim = dim3(nblocks);
        k2.blockDim = dim3(threads);
        k2.kernelParams = a2;
        cudaGraphNode_t n1, n2;
        ok = cudaGraphAddKernelNode(&n1, body, nullptr, 0, &k1) == cudaSuccess &&
             cudaGraphAddKernelNode(&n2, body, &n1, 1, &k2) == cudaSuccess &&
             cudaGraphInstantiate(&c.pcg_exec, graph, 0) == cudaSuccess;
      }
      if (graph) cudaGraphDestroy(graph);
      if (!ok) {  // no conditional-node support: fall back to host-chunked launches
        cudaGetLastError();
        c.use_graphs = false;
        if (c.pcg_exec) cudaGraphExecDestroy(c.pcg_exec);
        c.pcg_exec = nullptr;
      } else {
        c.pcg_exec_blocks = nblocks;
        c.pcg_exec_single = single;
        c.pcg_exec_pair = pair;
      }
    }
    if (c.pcg_exec) {
      WG_CUDA(cudaGraphLaunch(c.pcg_exec, s));
      c.launches += 2 * max_it;  // upper bound; exact count read back below
      WG_CUDA(cudaMemcpyAsync(hs, c.pcg, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
      WG_CUDA(cudaStreamSynchronize(s));
      c.launches -= 2 * max_it;
      c.launches += 2 * std::max(hs->iter, 1);
    }
  }
  if (!persistent && !prows && (c.profile || !c.use_graphs)) {
    int chunk = 4;
    int iter_before = 0;
    for (;;) {
      if (c.profile && c.prof_ev.size() < 64) {
        c.prof_ev.resize(64);
        for (auto& e : c.prof_ev) WG_CUDA(cudaEventCreate(&e));
      }
      for (int k = 0; k < chunk; ++k) {
        if (c.profile) WG_CUDA(cudaEventRecord(c.prof_ev[2 * k], s));
        spmv_kernel<<<pair ? nblocks2 : nblocks, threads, 0, ls(c)>>>(dargs, c.pcg);
        if (c.profile) WG_CUDA(cudaEventRecord(c.prof_ev[2 * k + 1], s));
        k_pcg_update<<<nblocks, threads, 0, ls(c)>>>(dargs, c.pcg, 0, 0);
      }
      WG_CUDA(cudaGetLastError());
      WG_CUDA(cudaMemcpyAsync(hs, c.pcg, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
      WG_CUDA(cudaStreamSynchronize(s));
      if (c.profile) {
        // Only launches that did work count (kernels early-exit once done).
        const int worked = std::min(chunk, hs->iter - iter_before);
        for (int k = 0; k < worked; ++k) {
          float ms = 0.f;
          WG_CUDA(cudaEventElapsedTime(&ms, c.prof_ev[2 * k], c.prof_ev[2 * k + 1]));
          c.spmv_ms += ms;
          ++c.spmv_launches;
        }
      }
      iter_before = hs->iter;
      if (hs->done) break;
      chunk = std::min(chunk * 2, 32);  // <= 32 (event pool of 64)
    }
  }
  comm_check(c);
  res.iterations = hs->iter;
  res.converged = hs->converged;
  res.rel_residual = hs->r_norm / b_norm;
  if (hs->status == 1)
    throw Error(WEFT_ERR_SOLVER, "pcg: non-finite curvature at iteration " + std::to_string(hs->iter));
  if (hs->status == 2)
    throw Error(WEFT_ERR_SOLVER,
                "pcg: non-positive curvature at iteration " + std::to_string(hs->iter) + " (matrix not SPD)");
  if (hs->status == 3)
    throw Error(WEFT_ERR_SOLVER,
                "pcg: divergence (non-finite residual) at iteration " + std::to_string(hs->iter));
  log_line(c, "event=pcg iterations=" + std::to_string(res.iterations) + " rel_residual=" + fmt_g(res.rel_residual) +
                  " converged=" + std::to_string(res.converged ? 1 : 0));  // solver.hpp:171-175
  if (hist_host && res.iterations)
    WG_CUDA(cudaMemcpyAsync(hist_host, c.hist.data(), sizeof(double) * res.iterations, cudaMemcpyDeviceToHost, s));
  if (phist_host && res.iterations)
    WG_CUDA(cudaMemcpyAsync(phist_host, c.phist.data(), sizeof(double) * res.iterations, cudaMemcpyDeviceToHost, s));
  WG_CUDA(cudaStreamSynchronize(s));
  return res;
}


// pcg_solve<float> (solver.hpp:36-178 with Real = float): the rows solver in
// single precision (one rank; any partition count) — float vectors and
// matrix, double dots, double block-Jacobi inverses of the float diagonal
// blocks, alpha / beta cast to float in the updates.
PcgResult pcg_solve_f32(Ctx& c, const float* b_dev, const weft_pcg_config& cfg, double* hist_host,
                        double* phist_host) {
  if (!c.has_matrix || !c.A.f32) throw Error(WEFT_ERR_INVALID, "pcg: no single-precision matrix");
  if (c.world > 1) throw Error(WEFT_ERR_INVALID, "pcg: Precision::Single runs on one rank");
  const int rows = c.A.rows;
  const size_t len = 3 * static_cast<size_t>(c.pm.p);
  const int threads = 256;
  if (!c.pcg) {
    WG_CUDA(cudaMalloc(&c.pcg, sizeof(PcgState)));
    WG_CUDA(cudaHostAlloc(&c.pcg_host, sizeof(PcgState), cudaHostAllocDefault));
  }
  for (auto* v : {&c.r, &c.z, &c.pv, &c.q, &c.xs}) v->resize(len);  // float views of these
  auto f = [](DBuf<double>& d) { return reinterpret_cast<float*>(d.data()); };
  const bool bj = cfg.preconditioner == WEFT_PRECOND_BLOCK_JACOBI;
  c.dinv.resize(9 * static_cast<size_t>(c.pm.p) + 9);
  const int max_it = std::max(cfg.max_iterations, 0);
  c.hist.resize(static_cast<size_t>(max_it) + 1);
  c.phist.resize(static_cast<size_t>(max_it) + 1);
  const PartBlocks pb = part_blocks(c, threads);
  const int nblocks = pb.bstart[pb.n];
  c.partials.resize(4 * static_cast<size_t>(nblocks) + 4);
  const SellView A = view(c.A);
  cudaStream_t s = c.stream;
  PcgState init{};
  init.max_iter = max_it;
  init.first = 1;
  WG_CUDA(cudaMemcpyAsync(c.pcg, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  double* dots = reinterpret_cast<double*>(c.scalars.data());
  if (rows > 0) {
    if (bj) k_dinv<false, float><<<div_up(rows, threads), threads, 0, ls(c)>>>(A, c.dinv.data());
    k_pcg_init<float><<<div_up(rows, threads), threads, 0, ls(c)>>>(c.row0, rows, b_dev, c.dinv.data(), bj, f(c.xs),
                                                                    f(c.r), f(c.z), f(c.pv));
    k_dot2<float><<<nblocks, threads, 0, ls(c)>>>(pb, b_dev, b_dev, f(c.r), f(c.z), c.partials.data(),
                                                  &c.pcg->counter, dots, c.comm, c.nparts);
    WG_CUDA(cudaGetLastError());
  }
  double hd[2] = {0.0, 0.0};
  if (rows > 0) WG_CUDA(cudaMemcpyAsync(hd, dots, sizeof(hd), cudaMemcpyDeviceToHost, s));
  WG_CUDA(cudaStreamSynchronize(s));
  PcgResult res;
  const double b_norm = std::sqrt(hd[0]);
  if (b_norm == 0.0) {
    res.converged = 1;
    return res;
  }
  init.b_norm = b_norm;
  init.tol = cfg.rel_tolerance * b_norm;
  init.rho = hd[1];
  init.r_norm = b_norm;
  init.done = max_it == 0 ? 1 : 0;
  WG_CUDA(cudaMemcpyAsync(c.pcg, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  PcgArgs args{A, pb, pb, c.go.n, bj ? 1 : 0, c.dinv.data(), c.xs.data(), c.r.data(), c.z.data(), c.pv.data(),
               c.q.data(), c.partials.data(), c.hist.data(), c.phist.data(), c.comm, c.pm, nullptr};
  c.pcg_args.resize(sizeof(PcgArgs));
  const PcgArgs* dargs = reinterpret_cast<const PcgArgs*>(c.pcg_args.data());
  WG_CUDA(cudaMemcpyAsync(c.pcg_args.data(), &args, sizeof(args), cudaMemcpyHostToDevice, s));
  auto k = k_pcg_persistent_rows<false, float>;
  int sms = 0, occ = 0;
  WG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
  WG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, 0));
  const int grid = std::max(1, std::min(std::max(1, occ) * sms, nblocks));
  void* kargs[] = {(void*)&dargs, (void*)&c.pcg};
  WG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k), dim3(grid), dim3(threads), kargs, 0, s));
  ++c.launches;
  auto* hs = static_cast<PcgState*>(c.pcg_host);
  WG_CUDA(cudaMemcpyAsync(hs, c.pcg, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  WG_CUDA(cudaStreamSynchronize(s));
  res.iterations = hs->iter;
  res.converged = hs->converged;
  res.rel_residual = hs->r_norm / b_norm;
  if (hs->status == 1)
    throw Error(WEFT_ERR_SOLVER, "pcg: non-finite curvature at iteration " + std::to_string(hs->iter));
  if (hs->status == 2)
    throw Error(WEFT_ERR_SOLVER,
                "pcg: non-positive curvature at iteration " + std::to_string(hs->iter) + " (matrix not SPD)");
  if (hs->status == 3)
    throw Error(WEFT_ERR_SOLVER,
                "pcg: divergence (non-finite residual) at iteration " + std::to_string(hs->iter));
  log_line(c, "event=pcg iterations=" + std::to_string(res.iterations) + " rel_residual=" + fmt_g(res.rel_residual) +
                  " converged=" + std::to_string(res.converged ? 1 : 0));
  if (hist_host && res.iterations)
    WG_CUDA(cudaMemcpyAsync(hist_host, c.hist.data(), sizeof(double) * res.iterations, cudaMemcpyDeviceToHost, s));
  if (phist_host && res.iterations)
    WG_CUDA(cudaMemcpyAsync(phist_host, c.phist.data(), sizeof(double) * res.iterations, cudaMemcpyDeviceToHost, s));
  WG_CUDA(cudaStreamSynchronize(s));
  return res;
}

// Single-precision systems from a block CSR (values exact in float): the
// double layout is built, then its values are narrowed once on the device.
__global__ void k_narrow_vals(int64_t n, const double* __restrict__ in, float* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = static_cast<float>(in[i]);
}

void set_matrix_csr_f32(Ctx& c, int rows, const int64_t* row_ptr, const int32_t* cols, const float* vals) {
  const int64_t nnz = rows > 0 ? row_ptr[rows] : 0;
  std::vector<double> vd(9 * static_cast<size_t>(nnz));
  for (size_t i = 0; i < vd.size(); ++i) vd[i] = vals[i];
  set_matrix_csr(c, rows, row_ptr, cols, vd.data());
  narrow_to_f32(c);
}

void narrow_to_f32(Ctx& c) {
  SellMatrix& A = c.A;
  const int64_t n = 9 * A.total;
  A.vals32.resize(static_cast<size_t>(n) + 9);
  if (n) k_narrow_vals<<<div_up(n, 256), 256, 0, ls(c)>>>(n, A.vals.data(), A.vals32.data());
  WG_CUDA(cudaGetLastError());
  A.f32 = true;
}

}  // namespace weft_gpu
