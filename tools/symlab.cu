// symlab.cu — dev experiment (not product code): does reading the lower
// triangle's blocks from their upper-triangle mirrors (served from L2, since
// the mirror row was streamed a few hundred rows earlier) cut the SpMV's
// DRAM traffic enough to pay for the gather?
//
// SELL-32 slot-major layout like the product (block (slice, k, lane) at
// (slice_base + k*32 + lane) * 9 doubles). Kernel `plain` streams every slot;
// kernel `mirror` skips the value read of slots whose column is a lower
// neighbour and reads the partner block (transposed) instead, at the address
// held in mirror[slot] (-1 = own). Values are made exactly symmetric so the two
// products must agree bitwise.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace {

template <int kMode>  // 0 plain, 1 mirror (int32 partner address), 2 mirror via byte k' + slice base
__global__ void __launch_bounds__(256) k_spmv(int rows, const int64_t* __restrict__ sbase, const int* __restrict__ slen,
                                              const int* __restrict__ cols, const int* __restrict__ mirror,
                                              const uint8_t* __restrict__ kp, const double* __restrict__ vals,
                                              const double* __restrict__ x, double* __restrict__ y) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const int s = row >> 5, lane = row & 31;
  const int64_t base = sbase[s];
  const int len = slen[row];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int k = 0; k < len; ++k) {
    const int64_t at = base + (int64_t)k * 32 + lane;
    const int c = __ldg(cols + at);
    const double x0 = __ldg(x + 3 * c), x1 = __ldg(x + 3 * c + 1), x2 = __ldg(x + 3 * c + 2);
    int64_t src = at;
    bool tr = false;
    if (kMode == 1) {
      const int m = __ldg(mirror + at);
      if (m >= 0) {
        src = m;
        tr = true;
      }
    } else if (kMode == 2) {
      const int kk = __ldg(kp + at);
      if (kk != 0xff) {
        src = __ldg(sbase + (c >> 5)) + (int64_t)kk * 32 + (c & 31);
        tr = true;
      }
    }
    const double* v = vals + 9 * src;
    double m[9];
    if (!tr) {
#pragma unroll
      for (int e = 0; e < 9; ++e) m[e] = __ldcs(v + e);
    } else {
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int q = 0; q < 3; ++q) m[3 * r + q] = __ldg(v + 3 * q + r);
    }
    a0 = a0 + ((m[0] * x0 + m[1] * x1) + m[2] * x2);
    a1 = a1 + ((m[3] * x0 + m[4] * x1) + m[5] * x2);
    a2 = a2 + ((m[6] * x0 + m[7] * x1) + m[8] * x2);
  }
  y[3 * row] = a0;
  y[3 * row + 1] = a1;
  y[3 * row + 2] = a2;
}

__global__ void k_flush(double* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = p[i] * 0.5 + 1.0;
}

}  // namespace

extern "C" int symlab_run(int rows, int64_t slots, const int64_t* sbase, const int* slen, const int* cols,
                          const int* mirror, const uint8_t* kp, const double* vals, const double* x, double* y_out,
                          float* t) {
  int64_t *d_sbase;
  int *d_slen, *d_cols, *d_mirror;
  uint8_t* d_kp;
  double *d_vals, *d_x, *d_y, *d_flush;
  const int slices = (rows + 31) / 32;
  cudaMalloc(&d_sbase, sizeof(int64_t) * (slices + 1));
  cudaMalloc(&d_slen, sizeof(int) * rows);
  cudaMalloc(&d_cols, sizeof(int) * slots);
  cudaMalloc(&d_mirror, sizeof(int) * slots);
  cudaMalloc(&d_kp, slots);
  cudaMalloc(&d_vals, sizeof(double) * 9 * slots);
  cudaMalloc(&d_x, sizeof(double) * 3 * rows);
  cudaMalloc(&d_y, sizeof(double) * 3 * rows * 3);
  const int64_t nflush = 48ll << 20;  // 384 MB
  cudaMalloc(&d_flush, sizeof(double) * nflush);
  cudaMemset(d_flush, 0, sizeof(double) * nflush);
  cudaMemcpy(d_sbase, sbase, sizeof(int64_t) * (slices + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(d_slen, slen, sizeof(int) * rows, cudaMemcpyHostToDevice);
  cudaMemcpy(d_cols, cols, sizeof(int) * slots, cudaMemcpyHostToDevice);
  cudaMemcpy(d_mirror, mirror, sizeof(int) * slots, cudaMemcpyHostToDevice);
  cudaMemcpy(d_kp, kp, slots, cudaMemcpyHostToDevice);
  cudaMemcpy(d_vals, vals, sizeof(double) * 9 * slots, cudaMemcpyHostToDevice);
  cudaMemcpy(d_x, x, sizeof(double) * 3 * rows, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1, f1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&f1);
  const int grid = (rows + 255) / 256;
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e30f;
    for (int rep = 0; rep < 12; ++rep) {
      k_flush<<<592, 512>>>(d_flush, nflush);
      cudaEventRecord(e0);
      if (mode == 0)
        k_spmv<0><<<grid, 256>>>(rows, d_sbase, d_slen, d_cols, d_mirror, d_kp, d_vals, d_x, d_y);
      else if (mode == 1)
        k_spmv<1><<<grid, 256>>>(rows, d_sbase, d_slen, d_cols, d_mirror, d_kp, d_vals, d_x, d_y + 3 * rows);
      else
        k_spmv<2><<<grid, 256>>>(rows, d_sbase, d_slen, d_cols, d_mirror, d_kp, d_vals, d_x, d_y + 6 * rows);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep >= 2 && ms < best) best = ms;
    }
    t[mode] = best;
  }
  cudaMemcpy(y_out, d_y, sizeof(double) * 9 * rows, cudaMemcpyDeviceToHost);
  const cudaError_t err = cudaGetLastError();
  cudaFree(d_sbase);
  cudaFree(d_slen);
  cudaFree(d_cols);
  cudaFree(d_mirror);
  cudaFree(d_kp);
  cudaFree(d_vals);
  cudaFree(d_x);
  cudaFree(d_y);
  cudaFree(d_flush);
  return err == cudaSuccess ? 0 : (int)err;
}
