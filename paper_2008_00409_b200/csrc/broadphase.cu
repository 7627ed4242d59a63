// broadphase.cu — spatial-hash broad phase for DCD and CCD.
//
// Reference: triangle_query_box (proj/src/collision.cpp:77-91), build_grid
// (:118-179), split_workload (:181-192), min_common_cell (:205-210) and the
// candidate walk of narrow_phase_range (:329-378).
//
// Device pipeline (all sort/scan work on the GPU, no CPU fallback):
//   boxes + diagonals (1 thread / triangle)
//   -> cell size from the SERIAL left-to-right diagonal sum (one warp; the
//      reference's sequential rounding is reproduced exactly, so every
//      floor(lo / cell) and therefore every candidate pair is bit-exact)
//   -> lattice boxes + entry counts -> exclusive scan -> (key, tri) emission
//      in triangle order -> stable radix sort by 63-bit cell key (per-cell
//      triangle lists come out ascending, as the reference's)
//   -> run-length cells, c(c-1)/2 workload prefix
//   -> candidate walk: each thread takes a contiguous chunk of the flattened
//      pair space (the reference's exact pair-range split, at thread
//      granularity) and keeps (t1, t2) iff the smallest common cell of the two
//      lattice boxes is the current cell; two passes (count, write) keep the
//      output in the reference's walk order.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "ctx.cuh"

namespace weft_gpu {

constexpr int64_t kLatBias = int64_t(1) << 20;

__device__ __forceinline__ int clamp_lattice(double v) {
  const double f = floor(v);
  long long i;
  if (!(f >= -9223372036854775808.0 && f < 9223372036854775808.0)) i = LLONG_MIN;  // x86 cvttsd2si
  else i = static_cast<long long>(f);
  if (i < -kLatBias + 1) i = -kLatBias + 1;
  if (i > kLatBias - 1) i = kLatBias - 1;
  return static_cast<int>(i);
}

__device__ __forceinline__ uint64_t pack_cell(int ix, int iy, int iz) {
  return (static_cast<uint64_t>(ix + kLatBias) << 42) | (static_cast<uint64_t>(iy + kLatBias) << 21) |
         static_cast<uint64_t>(iz + kLatBias);
}

void set_soup(Ctx& c, int verts, int ntris, const int32_t* tris) {
  if (verts < 0 || ntris < 0) throw Error(WEFT_ERR_DIMENSION, "set_soup: negative size");
  std::vector<int32_t> h(3 * static_cast<size_t>(ntris));
  if (ntris) WG_CUDA(cudaMemcpy(h.data(), tris, h.size() * sizeof(int32_t), cudaMemcpyDefault));
  for (int32_t v : h)
    if (v < 0 || v >= verts) throw Error(WEFT_ERR_DIMENSION, "triangle vertex index out of range");
  c.soup_verts = verts;
  c.soup_tris = ntris;
  c.tris.upload(h.data(), h.size(), c.stream);
  WG_CUDA(cudaStreamSynchronize(c.stream));
  c.has_grid = false;
}

// triangle_query_box + the diagonal norm (collision.cpp:77-91, 124-133).
__global__ void k_boxes(int ntris, const int32_t* __restrict__ tris, const double* __restrict__ x0,
                        const double* __restrict__ x1, bool ccd, double inflate, double* __restrict__ lo,
                        double* __restrict__ hi, double* __restrict__ diag) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntris) return;
  double l[3] = {1e300, 1e300, 1e300}, h[3] = {-1e300, -1e300, -1e300};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int v = tris[3 * t + k];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double p0 = x0[3 * v + c];
      l[c] = p0 < l[c] ? p0 : l[c];  // cwiseMin
      h[c] = h[c] < p0 ? p0 : h[c];  // cwiseMax
      if (ccd) {
        const double p1 = x1[3 * v + c];
        l[c] = p1 < l[c] ? p1 : l[c];
        h[c] = h[c] < p1 ? p1 : h[c];
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    l[c] = l[c] - inflate;
    h[c] = h[c] + inflate;
    lo[3 * t + c] = l[c];
    hi[3 * t + c] = h[c];
  }
  const double dx = h[0] - l[0], dy = h[1] - l[1], dz = h[2] - l[2];
  diag[t] = sqrt((dx * dx + dy * dy) + dz * dz);
}

// cell = max(cell_scale * (sum_t diag_t) / T, 1e-9) with the sum taken
// strictly left to right (collision.cpp:124-133), reproduced EXACTLY but
// in parallel. While the running sum s stays inside one binade [2^e,
// 2^(e+1)) every double is an integer multiple M of u = 2^(e-52), and
// fl(s + d) = (M + round(d / u)) u: the rounding of each term is
// independent of s except for exact ties, which round the result to an
// even M. Each term is therefore a map M -> M + a[M mod 2] (a0 = a1 unless
// d/u is a tie); such maps compose associatively, so one CTA scans a window
// of 16K terms at a time, advances s by the exact composed offset up to the
// first term whose partial sum would leave the binade, adds that term with a
// plain IEEE add, and continues. Cost: (terms / 16K + binade crossings)
// block scans instead of one dependent add per triangle.
struct ParityMap {
  long long a0, a1;  // offset applied when the running integer is even / odd
};

__device__ __forceinline__ ParityMap compose(ParityMap f, ParityMap g) {  // f, then g
  ParityMap r;
  r.a0 = f.a0 + ((f.a0 & 1) ? g.a1 : g.a0);
  r.a1 = f.a1 + (((1 + f.a1) & 1) ? g.a1 : g.a0);
  return r;
}

constexpr int kSumThreads = 1024;
constexpr int kSumItems = 16;
constexpr long long kTwo53 = 1LL << 53;

__global__ void __launch_bounds__(kSumThreads) k_cell_size(int ntris, const double* __restrict__ diag,
                                                           double cell_scale, double* __restrict__ out) {
  extern __shared__ double sm_d[];  // kSumThreads * kSumItems terms
  __shared__ ParityMap sm_warp[32];
  __shared__ int sm_event;
  __shared__ long long sm_M;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double s = 0.0;  // uniform across the block
  int k = 0;
  while (k < ntris) {
    if (s == 0.0 || !(s >= 0x1p-1000) || !isfinite(s)) {
      // start, tiny or non-finite running sums: plain serial adds
      s = s + diag[k];
      ++k;
      if (!isfinite(s)) {
        for (; k < ntris; ++k) s = s + diag[k];
      }
      continue;
    }
    const int e = ilogb(s);
    const double inv_u = ldexp(1.0, 52 - e);
    const long long ms = static_cast<long long>(s * inv_u);  // exact: s = ms * u
    const int len = min(kSumThreads * kSumItems, ntris - k);
    for (int i = tid; i < len; i += kSumThreads) sm_d[i] = diag[k + i];
    if (tid == 0) sm_event = len;
    __syncthreads();
    // per-thread maps over its contiguous items
    ParityMap loc[kSumItems];
    ParityMap acc{0, 0};
#pragma unroll
    for (int i = 0; i < kSumItems; ++i) {
      const int j = tid * kSumItems + i;
      ParityMap m{0, 0};
      if (j < len) {
        const double x = sm_d[j] * inv_u;  // exact power-of-two scaling
        if (!(x < 0x1p53)) {
          m.a0 = m.a1 = kTwo53;  // certainly leaves the binade
        } else {
          const double fl = floor(x);
          const double fr = x - fl;
          const long long f = static_cast<long long>(fl);
          if (fr < 0.5) m.a0 = m.a1 = f;
          else if (fr > 0.5) m.a0 = m.a1 = f + 1;
          else {  // tie: round the result to an even integer
            m.a0 = f + (f & 1);
            m.a1 = f + ((1 + f) & 1);
          }
        }
      }
      acc = compose(acc, m);
      loc[i] = acc;  // thread-local inclusive prefix
    }
    // block exclusive scan of the per-thread maps (ordered composition)
    ParityMap incl = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      ParityMap other;
      other.a0 = __shfl_up_sync(0xffffffffu, incl.a0, o);
      other.a1 = __shfl_up_sync(0xffffffffu, incl.a1, o);
      if (lane >= o) incl = compose(other, incl);
    }
    if (lane == 31) sm_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      ParityMap w = sm_warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        ParityMap other;
        other.a0 = __shfl_up_sync(0xffffffffu, w.a0, o);
        other.a1 = __shfl_up_sync(0xffffffffu, w.a1, o);
        if (lane >= o) w = compose(other, w);
      }
      sm_warp[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    ParityMap excl{0, 0};
    {
      ParityMap lane_excl;
      lane_excl.a0 = __shfl_up_sync(0xffffffffu, incl.a0, 1);
      lane_excl.a1 = __shfl_up_sync(0xffffffffu, incl.a1, 1);
      if (lane == 0) lane_excl = ParityMap{0, 0};
      const ParityMap wp = warp > 0 ? sm_warp[warp - 1] : ParityMap{0, 0};
      excl = compose(wp, lane_excl);
    }
    // first term whose running integer reaches 2^53 (binade exit)
    const int p0 = static_cast<int>(ms & 1);
    int first = len;
#pragma unroll
    for (int i = 0; i < kSumItems; ++i) {
      const int j = tid * kSumItems + i;
      if (j < len) {
        const ParityMap t = compose(excl, loc[i]);
        const long long M = ms + (p0 ? t.a1 : t.a0);
        if (M >= kTwo53 && j < first) first = j;
      }
    }
    if (first < len) atomicMin(&sm_event, first);
    __syncthreads();
    const int m = sm_event;
    if (m > 0) {
      // state after m terms: owned by the thread holding term m-1
      const int owner = (m - 1) / kSumItems;
      if (tid == owner) {
        const ParityMap t = compose(excl, loc[(m - 1) % kSumItems]);
        sm_M = ms + (p0 ? t.a1 : t.a0);
      }
      __syncthreads();
      s = ldexp(static_cast<double>(sm_M), e - 52);
    }
    k += m;
    if (m < len) {  // the binade-exit term: plain IEEE add
      s = s + sm_d[m];
      ++k;
    }
    __syncthreads();
  }
  if (tid == 0) {
    const double mean = ntris > 0 ? s / ntris : 1.0;
    const double a = cell_scale * mean;
    out[0] = (a < 1e-9) ? 1e-9 : a;  // std::max(a, 1e-9)
  }
}

constexpr size_t kSumSmem = sizeof(double) * kSumThreads * kSumItems;

static void launch_cell_size(Ctx& c, int n, const double* d, double scale, double* out) {
  WG_CUDA(cudaFuncSetAttribute(k_cell_size, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSumSmem));
  k_cell_size<<<1, kSumThreads, kSumSmem, ls(c)>>>(n, d, scale, out);
}

// Reference serial sum (validation only: weft_gpu_serial_sum).
__global__ void k_serial_sum_naive(int n, const double* __restrict__ d, double* __restrict__ out) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = s + d[i];
  out[0] = s;
}

__global__ void k_lattice(int ntris, const double* __restrict__ lo, const double* __restrict__ hi,
                          const double* __restrict__ cellp, int* __restrict__ lat, int64_t* __restrict__ cnt) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntris) return;
  const double cell = *cellp;
  int b[6];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    b[c] = clamp_lattice(lo[3 * t + c] / cell);
    b[c + 3] = clamp_lattice(hi[3 * t + c] / cell);
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) lat[6 * t + c] = b[c];
  cnt[t] = static_cast<int64_t>(b[3] - b[0] + 1) * (b[4] - b[1] + 1) * (b[5] - b[2] + 1);
}

__global__ void k_emit(int ntris, const int* __restrict__ lat, const int64_t* __restrict__ off,
                       uint64_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntris) return;
  const int* b = lat + 6 * t;
  int64_t o = off[t];
  for (int ix = b[0]; ix <= b[3]; ++ix)
    for (int iy = b[1]; iy <= b[4]; ++iy)
      for (int iz = b[2]; iz <= b[5]; ++iz) {
        keys[o] = pack_cell(ix, iy, iz);
        vals[o] = t;
        ++o;
      }
}

__global__ void k_cell_flags(int64_t n, const uint64_t* __restrict__ keys, int32_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// flag has been exclusive-scanned into idx: cell index of each run start.
__global__ void k_cells(int64_t n, const uint64_t* __restrict__ keys, const int32_t* __restrict__ flag_scan,
                        uint64_t* __restrict__ cell_keys, int64_t* __restrict__ cell_off) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0 || keys[i] != keys[i - 1]) {
    const int c = flag_scan[i];
    cell_keys[c] = keys[i];
    cell_off[c] = i;
  }
}

__global__ void k_pair_counts(int64_t cells, const int64_t* __restrict__ cell_off, int64_t* __restrict__ w) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= cells) return;
  const int64_t s = cell_off[c + 1] - cell_off[c];
  w[c] = s * (s - 1) / 2;
}

void build_grid(Ctx& c, const double* x0, const double* x1, int mode, double thickness, double cell_scale) {
  const int T = c.soup_tris;
  cudaStream_t s = c.stream;
  const bool ccd = mode == WEFT_CONTINUOUS;
  const double inflate = ccd ? 1e-9 : 0.5 * thickness;  // collision.cpp:122
  c.box_lo.resize(3 * static_cast<size_t>(T) + 3);
  c.box_hi.resize(3 * static_cast<size_t>(T) + 3);
  c.diag.resize(static_cast<size_t>(T) + 1);
  c.cell_size.resize(1);
  c.lat.resize(6 * static_cast<size_t>(T) + 6);
  c.ecount.resize(static_cast<size_t>(T) + 1);
  if (T) {
    k_boxes<<<div_up(T, 256), 256, 0, ls(c)>>>(T, c.tris.data(), x0, ccd ? x1 : x0, ccd, inflate, c.box_lo.data(),
                                           c.box_hi.data(), c.diag.data());
  }
  launch_cell_size(c, T, c.diag.data(), cell_scale, c.cell_size.data());
  WG_CUDA(cudaMemsetAsync(c.ecount.data() + T, 0, sizeof(int64_t), s));
  if (T)
    k_lattice<<<div_up(T, 256), 256, 0, ls(c)>>>(T, c.box_lo.data(), c.box_hi.data(), c.cell_size.data(), c.lat.data(),
                                             c.ecount.data());
  WG_CUDA(cudaGetLastError());
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.ecount.data(), c.ecount.data(), T + 1, s);
  void* t = scratch(c, tmp);
  WG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, c.ecount.data(), c.ecount.data(), T + 1, s));
  int64_t K = 0;
  WG_CUDA(cudaMemcpyAsync(&K, c.ecount.data() + T, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  WG_CUDA(cudaMemcpyAsync(&c.grid_cell_size, c.cell_size.data(), sizeof(double), cudaMemcpyDeviceToHost, s));
  WG_CUDA(cudaStreamSynchronize(s));
  if (K > (int64_t(1) << 31) - 1) throw Error(WEFT_ERR_DIMENSION, "build_grid: more than 2^31 cell entries");
  c.keys_a.resize(static_cast<size_t>(K) + 1);
  c.keys_b.resize(static_cast<size_t>(K) + 1);
  c.vals_a.resize(static_cast<size_t>(K) + 1);
  c.vals_b.resize(static_cast<size_t>(K) + 1);
  if (T) k_emit<<<div_up(T, 256), 256, 0, ls(c)>>>(T, c.lat.data(), c.ecount.data(), c.keys_a.data(), c.vals_a.data());
  if (K) {
    tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, c.keys_a.data(), c.keys_b.data(), c.vals_a.data(), c.vals_b.data(),
                                    (int)K, 0, 63, s);
    t = scratch(c, tmp);
    WG_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, c.keys_a.data(), c.keys_b.data(), c.vals_a.data(),
                                            c.vals_b.data(), (int)K, 0, 63, s));
  }
  // run-length cells
  c.cell_flag.resize(static_cast<size_t>(K) + 1);
  if (K) k_cell_flags<<<div_up(K, 256), 256, 0, ls(c)>>>(K, c.keys_b.data(), c.cell_flag.data());
  WG_CUDA(cudaMemsetAsync(c.cell_flag.data() + K, 0, sizeof(int32_t), s));
  tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.cell_flag.data(), c.cell_flag.data(), K + 1, s);
  t = scratch(c, tmp);
  WG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, c.cell_flag.data(), c.cell_flag.data(), K + 1, s));
  int32_t cells32 = 0;
  WG_CUDA(cudaMemcpyAsync(&cells32, c.cell_flag.data() + K, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  WG_CUDA(cudaStreamSynchronize(s));
  const int64_t cells = cells32;
  c.cell_keys.resize(static_cast<size_t>(cells) + 1);
  c.cell_off.resize(static_cast<size_t>(cells) + 1);
  c.wprefix.resize(static_cast<size_t>(cells) + 1);
  if (K) k_cells<<<div_up(K, 256), 256, 0, ls(c)>>>(K, c.keys_b.data(), c.cell_flag.data(), c.cell_keys.data(), c.cell_off.data());
  WG_CUDA(cudaMemcpyAsync(c.cell_off.data() + cells, &K, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  if (cells) k_pair_counts<<<div_up(cells, 256), 256, 0, ls(c)>>>(cells, c.cell_off.data(), c.wprefix.data());
  WG_CUDA(cudaMemsetAsync(c.wprefix.data() + cells, 0, sizeof(int64_t), s));
  tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.wprefix.data(), c.wprefix.data(), cells + 1, s);
  t = scratch(c, tmp);
  WG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, c.wprefix.data(), c.wprefix.data(), cells + 1, s));
  WG_CUDA(cudaMemcpyAsync(&c.grid_total, c.wprefix.data() + cells, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  WG_CUDA(cudaGetLastError());
  WG_CUDA(cudaStreamSynchronize(s));
  c.grid_entries = K;
  c.grid_cells = cells;
  c.has_grid = true;
}

// ---------------------------------------------------------------------------
// candidate walk
// ---------------------------------------------------------------------------
struct WalkArgs {
  int64_t begin, end, chunk, cells;
  const int64_t* __restrict__ prefix;
  const int64_t* __restrict__ cell_off;
  const int32_t* __restrict__ cell_tris;
  const uint64_t* __restrict__ cell_keys;
  const int* __restrict__ lat;
};

// Walks this thread's chunk; calls emit(t1, t2) for each candidate.
template <class F>
__device__ __forceinline__ void walk_chunk(const WalkArgs& w, int64_t g0, int64_t g1, F&& emit) {
  // cell = upper_bound(prefix, g0) - 1
  int64_t lo = 0, hi = w.cells + 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (w.prefix[mid] <= g0) lo = mid + 1;
    else hi = mid;
  }
  int64_t cell = lo - 1;
  int64_t s = w.cell_off[cell + 1] - w.cell_off[cell];
  // decode local pair index k -> (i, j), rows of length s-1-i
  const int64_t k = g0 - w.prefix[cell];
  auto start = [&](int64_t i) { return i * s - i * (i + 1) / 2; };
  const double b = 2.0 * s - 1.0;
  int64_t i = static_cast<int64_t>(floor((b - sqrt(fmax(b * b - 8.0 * (double)k, 0.0))) * 0.5));
  if (i < 0) i = 0;
  while (i > 0 && start(i) > k) --i;
  while (start(i + 1) <= k) ++i;
  int64_t j = i + 1 + (k - start(i));
  int64_t next = w.prefix[cell + 1];
  const int32_t* tl = w.cell_tris + w.cell_off[cell];
  uint64_t key = w.cell_keys[cell];
  for (int64_t g = g0; g < g1; ++g) {
    while (g >= next) {
      ++cell;
      s = w.cell_off[cell + 1] - w.cell_off[cell];
      tl = w.cell_tris + w.cell_off[cell];
      key = w.cell_keys[cell];
      next = w.prefix[cell + 1];
      i = 0;
      j = 1;
    }
    const int t1 = tl[i], t2 = tl[j];
    const int* a = w.lat + 6 * t1;
    const int* bb = w.lat + 6 * t2;
    const uint64_t mc = pack_cell(max(a[0], bb[0]), max(a[1], bb[1]), max(a[2], bb[2]));
    if (mc == key) emit(t1, t2);
    if (++j >= s) {
      ++i;
      j = i + 1;
    }
  }
}

__global__ void k_walk_count(WalkArgs w, int64_t nthreads, int64_t* __restrict__ counts) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= nthreads) return;
  const int64_t g0 = w.begin + tid * w.chunk;
  const int64_t g1 = min(g0 + w.chunk, w.end);
  int64_t n = 0;
  if (g0 < g1) walk_chunk(w, g0, g1, [&](int, int) { ++n; });
  counts[tid] = n;
}

__global__ void k_walk_write(WalkArgs w, int64_t nthreads, const int64_t* __restrict__ offs,
                             int32_t* __restrict__ pairs) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= nthreads) return;
  const int64_t g0 = w.begin + tid * w.chunk;
  const int64_t g1 = min(g0 + w.chunk, w.end);
  int64_t o = offs[tid];
  if (g0 < g1)
    walk_chunk(w, g0, g1, [&](int t1, int t2) {
      pairs[2 * o] = t1;
      pairs[2 * o + 1] = t2;
      ++o;
    });
}

// Returns the candidate count of [begin, end); when pairs_out is non-null
// the pairs are written there (device or host pointer). Device-resident
// pairs stay in c.cand_pairs.
int64_t candidates(Ctx& c, int64_t begin, int64_t end, int32_t* pairs_out) {
  if (!c.has_grid) throw Error(WEFT_ERR_INVALID, "candidates: build_grid first");
  begin = std::max<int64_t>(begin, 0);
  end = std::min<int64_t>(end, c.grid_total);
  if (begin >= end) return 0;
  cudaStream_t s = c.stream;
  const int64_t W = end - begin;
  const int64_t target_threads = 148LL * 1024;
  const int64_t chunk = std::max<int64_t>(32, (W + target_threads - 1) / target_threads);
  const int64_t nthreads = (W + chunk - 1) / chunk;
  WalkArgs w{begin, end, chunk, c.grid_cells, c.wprefix.data(), c.cell_off.data(), c.vals_b.data(),
             c.cell_keys.data(), c.lat.data()};
  c.cand_count.resize(static_cast<size_t>(nthreads) + 1);
  WG_CUDA(cudaMemsetAsync(c.cand_count.data() + nthreads, 0, sizeof(int64_t), s));
  k_walk_count<<<div_up(nthreads, 256), 256, 0, ls(c)>>>(w, nthreads, c.cand_count.data());
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.cand_count.data(), c.cand_count.data(), nthreads + 1, s);
  void* t = scratch(c, tmp);
  WG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, c.cand_count.data(), c.cand_count.data(), nthreads + 1, s));
  int64_t n = 0;
  WG_CUDA(cudaMemcpyAsync(&n, c.cand_count.data() + nthreads, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  WG_CUDA(cudaStreamSynchronize(s));
  c.cand_pairs.resize(2 * static_cast<size_t>(n) + 2);
  k_walk_write<<<div_up(nthreads, 256), 256, 0, ls(c)>>>(w, nthreads, c.cand_count.data(), c.cand_pairs.data());
  WG_CUDA(cudaGetLastError());
  if (pairs_out && n)
    WG_CUDA(cudaMemcpyAsync(pairs_out, c.cand_pairs.data(), 2 * sizeof(int32_t) * n, cudaMemcpyDefault, s));
  WG_CUDA(cudaStreamSynchronize(s));
  return n;
}

// Test hook: exact parallel serial-order sum vs a one-thread serial loop.
void serial_sum(Ctx& c, int n, const double* d_host, double* exact, double* naive) {
  DBuf<double> d, o;
  d.upload(d_host, static_cast<size_t>(n), c.stream);
  o.resize(2);
  launch_cell_size(c, n, d.data(), 1.0, o.data());  // cell = max(sum / n, 1e-9)
  k_serial_sum_naive<<<1, 1, 0, ls(c)>>>(n, d.data(), o.data() + 1);
  WG_CUDA(cudaGetLastError());
  double h[2];
  WG_CUDA(cudaMemcpyAsync(h, o.data(), sizeof(h), cudaMemcpyDeviceToHost, c.stream));
  WG_CUDA(cudaStreamSynchronize(c.stream));
  *exact = h[0];
  *naive = h[1];
}

}  // namespace weft_gpu
