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
#include <climits>
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

__global__ void k_read_small(const unsigned char* a, int na, const unsigned char* b, int nb, const unsigned char* d,
                             int nd, unsigned char* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int i = 0; i < na; ++i) out[i] = a[i];
  for (int i = 0; i < nb; ++i) out[128 + i] = b[i];
  for (int i = 0; i < nd; ++i) out[256 + i] = d[i];
}

void read_small(Ctx& c, cudaStream_t s, SmallRead a, SmallRead b, SmallRead d) {
  if (!c.map_host) {
    WG_CUDA(cudaHostAlloc(&c.map_host, 384, cudaHostAllocMapped));
    WG_CUDA(cudaHostGetDevicePointer(&c.map_dev, c.map_host, 0));
  }
  k_read_small<<<1, 32, 0, s>>>(static_cast<const unsigned char*>(a.src), a.bytes,
                                static_cast<const unsigned char*>(b.src), b.bytes,
                                static_cast<const unsigned char*>(d.src), d.bytes,
                                static_cast<unsigned char*>(c.map_dev));
  ++c.launches;
  WG_CUDA(cudaGetLastError());
  WG_CUDA(cudaStreamSynchronize(s));
  const auto* h = static_cast<const volatile unsigned char*>(c.map_host);
  auto take = [&](const SmallRead& r, int off) {
    auto* o = static_cast<unsigned char*>(r.dst);
    for (int i = 0; i < r.bytes; ++i) o[i] = h[off + i];
  };
  if (a.bytes > 128 || b.bytes > 128 || d.bytes > 128) throw Error(WEFT_ERR_INVALID, "read_small: > 128 bytes");
  take(a, 0);
  take(b, 128);
  take(d, 256);
}

void set_soup(Ctx& c, int verts, int ntris, const int32_t* tris) {
  if (verts < 0 || ntris < 0) throw Error(WEFT_ERR_DIMENSION, "set_soup: negative size");
  std::vector<int32_t> h(3 * static_cast<size_t>(ntris));
  if (ntris) WG_CUDA(cudaMemcpy(h.data(), tris, h.size() * sizeof(int32_t), cudaMemcpyDefault));
  for (int32_t v : h)
    if (v < 0 || v >= verts) throw Error(WEFT_ERR_DIMENSION, "triangle vertex index out of range");
  if (verts != c.soup_verts) c.has_state = c.obstacles_set = false;  // sim_x / sim_v are soup-sized
  c.soup_verts = verts;
  c.soup_tris = ntris;
  c.tris.upload(h.data(), h.size(), c.stream);
  WG_CUDA(cudaStreamSynchronize(c.stream));
  build_soup_edges(c, h);  // CollisionSoup::build's edge table (narrow phase)
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
constexpr int kSumChunk = kSumThreads * kSumItems;
constexpr int kSerialHead = 2048;
constexpr long long kTwo53 = 1LL << 53;

// Parity map of one term d in the binade with 1/u = inv_u.
__device__ __forceinline__ ParityMap term_map(double d, double inv_u, bool& huge) {
  ParityMap m;
  const double x = d * inv_u;  // exact power-of-two scaling
  if (!(x < 0x1p53)) {
    m.a0 = m.a1 = kTwo53;  // certainly leaves the binade
    huge = true;
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
  return m;
}

// Processes terms [k, kend) into the uniform running sum s with the
// window scan (exact). Must be called by all threads of the block.
__device__ void sum_range(const double* __restrict__ diag, int k, const int kend, double& s, double* sm_d,
                          ParityMap* sm_warp, int* sm_event, long long* sm_M) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  while (k < kend) {
    if (s == 0.0) {
      // the start: the running sum crosses a binade every time the term
      // count doubles, so the first kSerialHead terms are added serially by
      // one thread (a window pass per crossing would cost far more)
      const int n = min(kSerialHead, kend - k);
      if (tid == 0) {
        double t = 0.0;
        for (int i = 0; i < n; i += 8) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = i + u < n ? __ldcg(diag + k + i + u) : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (i + u < n) t = t + v[u];
        }
        sm_d[0] = t;
      }
      __syncthreads();
      s = sm_d[0];
      __syncthreads();
      k += n;
      continue;
    }
    if (!(s >= 0x1p-1000) || !isfinite(s)) {
      // start, tiny or non-finite running sums: plain serial adds
      s = s + diag[k];
      ++k;
      if (!isfinite(s)) {
        for (; k < kend; ++k) s = s + diag[k];
      }
      continue;
    }
    const int e = ilogb(s);
    const double inv_u = ldexp(1.0, 52 - e);
    const long long ms = static_cast<long long>(s * inv_u);  // exact: s = ms * u
    const int len = min(kSumChunk, kend - k);
    {
      double r[kSumItems];
#pragma unroll
      for (int i = 0; i < kSumItems; ++i) {
        const int j = tid + i * kSumThreads;
        r[i] = j < len ? __ldcg(diag + k + j) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < kSumItems; ++i) sm_d[tid + i * kSumThreads] = r[i];
    }
    if (tid == 0) *sm_event = len;
    __syncthreads();
    ParityMap loc[kSumItems];
    ParityMap acc{0, 0};
#pragma unroll
    for (int i = 0; i < kSumItems; ++i) {
      const int j = tid * kSumItems + i;
      ParityMap m{0, 0};
      bool huge = false;
      if (j < len) m = term_map(sm_d[j], inv_u, huge);
      acc = compose(acc, m);
      loc[i] = acc;
    }
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
      sm_warp[lane] = w;
    }
    __syncthreads();
    ParityMap lane_excl;
    lane_excl.a0 = __shfl_up_sync(0xffffffffu, incl.a0, 1);
    lane_excl.a1 = __shfl_up_sync(0xffffffffu, incl.a1, 1);
    if (lane == 0) lane_excl = ParityMap{0, 0};
    const ParityMap excl = compose(warp > 0 ? sm_warp[warp - 1] : ParityMap{0, 0}, lane_excl);
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
    if (first < len) atomicMin(sm_event, first);
    __syncthreads();
    const int m = *sm_event;
    if (m > 0) {
      const int owner = (m - 1) / kSumItems;
      if (tid == owner) {
        const ParityMap t = compose(excl, loc[(m - 1) % kSumItems]);
        *sm_M = ms + (p0 ? t.a1 : t.a0);
      }
      __syncthreads();
      s = ldexp(static_cast<double>(*sm_M), e - 52);
    }
    k += m;
    if (m < len) {  // the binade-exit term: plain IEEE add
      s = s + sm_d[m];
      ++k;
    }
    __syncthreads();
  }
}

// Fast path. The running sum crosses a binade ~log2(sum / first term)
// times (config D: 21 times over 1.65 M terms); only those places need the
// exact scan, everything else is a composed parity map per segment.
//  1. an approximate prefix of the terms (any order) predicts where the
//     exact running sum crosses each power of two;
//  2. the terms are cut into segments: up to kSumChunk terms in one
//     predicted binade, and a serial segment of 2 * kCrossPad terms around
//     every predicted crossing (overlapping ones merged: the dense early
//     crossings become one serial head);
//  3. one CTA per segment composes its parity map in the predicted binade;
//  4. one CTA applies the segments in order: map segments in O(1) when the
//     exact sum is in the predicted binade and stays there, serial segments
//     by one thread, and anything mispredicted by the exact window scan
//     (sum_range) — so the result is exact whatever the prediction did.
constexpr int kCrossPad = 32;
constexpr int kMaxCross = 256;

struct SumSeg {
  int k0, k1;
  int serial;   // 1: added term by term by one thread
  int e;        // predicted binade of the running sum at k0 (map segments)
  long long a0, a1;
  int ok;       // map usable
  int pad;
};

// Predicted crossings: term i where the approximate prefix enters a new binade.
__global__ void k_cross_find(int n, const double* __restrict__ pre, int* __restrict__ xs, int* __restrict__ nx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 1 || i >= n) return;
  const double a = pre[i - 1], b = pre[i];
  if (a > 0.0 && isfinite(b) && ilogb(a) != ilogb(b)) {
    const int k = atomicAdd(nx, 1);
    if (k < kMaxCross) xs[k] = i;
  }
}

// Segment list (one thread; a few hundred entries).
__global__ void k_seg_build(int n, const int* __restrict__ xs_in,
                            const int* __restrict__ nx_in, SumSeg* __restrict__ seg, int* __restrict__ nseg) {
  __shared__ int xs[kMaxCross], raw[kMaxCross];
  const int nx = min(*nx_in, kMaxCross);
  for (int i = threadIdx.x; i < nx; i += blockDim.x) raw[i] = xs_in[i];
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int i = 0; i < nx; ++i) {  // insertion sort (atomic order is arbitrary)
    const int v = raw[i];
    int j = i;
    while (j > 0 && xs[j - 1] > v) {
      xs[j] = xs[j - 1];
      --j;
    }
    xs[j] = v;
  }
  int k = 0, xi = 0, ns = 0;
  while (k < n) {
    while (xi < nx && xs[xi] + kCrossPad <= k) ++xi;
    SumSeg sg{};
    sg.k0 = k;
    if (k == 0 || (xi < nx && xs[xi] - kCrossPad <= k)) {
      // serial: the first term (the sum starts at 0) and the crossings near k
      int e = k == 0 ? 1 : k;
      while (xi < nx && xs[xi] - kCrossPad <= e) {
        e = max(e, xs[xi] + kCrossPad);
        ++xi;
      }
      sg.k1 = min(n, e);
      sg.serial = 1;
    } else {
      int r = min(n, k + kSumChunk);
      if (xi < nx) r = min(r, xs[xi] - kCrossPad);
      sg.k1 = r;  // binade and map: k_seg_maps
    }
    seg[ns++] = sg;
    k = sg.k1;
  }
  *nseg = ns;
}

// Parity map of each map segment in its predicted binade.
__global__ void __launch_bounds__(kSumThreads) k_seg_maps(const double* __restrict__ d, const double* __restrict__ pre,
                                                          SumSeg* __restrict__ seg, const int* __restrict__ nseg) {
  __shared__ ParityMap sm_w[32];
  __shared__ int sm_huge;
  const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (c >= *nseg) return;
  SumSeg sg = seg[c];
  if (sg.serial) return;
  const double a = pre[sg.k0 - 1];  // predicted running sum before the segment
  if (!(a > 0x1p-1000 && isfinite(a))) {
    if (tid == 0) seg[c].ok = 0;
    return;
  }
  sg.e = ilogb(a);
  if (tid == 0) sm_huge = 0;
  __syncthreads();
  const double inv_u = ldexp(1.0, 52 - sg.e);
  const int len = sg.k1 - sg.k0;
  ParityMap acc{0, 0};
  bool huge = false;
#pragma unroll
  for (int i = 0; i < kSumItems; ++i) {
    const int j = tid * kSumItems + i;
    if (j < len) acc = compose(acc, term_map(__ldg(d + sg.k0 + j), inv_u, huge));
  }
  if (huge) sm_huge = 1;
  // ordered reduction: lanes, then warps
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    ParityMap other;
    other.a0 = __shfl_down_sync(0xffffffffu, acc.a0, o);
    other.a1 = __shfl_down_sync(0xffffffffu, acc.a1, o);
    if ((lane & (2 * o - 1)) == 0) acc = compose(acc, other);
  }
  if (lane == 0) sm_w[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    ParityMap t{0, 0};
    for (int w = 0; w < 32; ++w) t = compose(t, sm_w[w]);
    seg[c].a0 = t.a0;
    seg[c].a1 = t.a1;
    seg[c].e = sg.e;
    seg[c].ok = sm_huge ? 0 : 1;
  }
}

// cell = max(cell_scale * mean, 1e-9) over the segments, in order.
__global__ void __launch_bounds__(kSumThreads) k_cell_size(int ntris, const double* __restrict__ diag,
                                                           const SumSeg* __restrict__ seg, const int* __restrict__ nsegp,
                                                           double cell_scale, double* __restrict__ out) {
  extern __shared__ double sm_d[];
  __shared__ ParityMap sm_warp[32];
  __shared__ int sm_event;
  __shared__ long long sm_M;
  constexpr int kSegBatch = 256;  // segments staged per batch
  __shared__ SumSeg sm_seg[kSegBatch];
  double s = 0.0;
  if (seg) {
    const int nseg = *nsegp;
    for (int c = 0; c < nseg; ++c) {
      if (c % kSegBatch == 0) {
        __syncthreads();
        for (int i = threadIdx.x; i < kSegBatch && c + i < nseg; i += blockDim.x) sm_seg[i] = seg[c + i];
        __syncthreads();
      }
      const SumSeg sg = sm_seg[c % kSegBatch];
      if (sg.serial) {  // staged by all threads, added in order by one
        for (int b = sg.k0; b < sg.k1; b += kSumChunk) {
          const int len = min(kSumChunk, sg.k1 - b);
          for (int i = threadIdx.x; i < len; i += blockDim.x) sm_d[i] = __ldcg(diag + b + i);
          __syncthreads();
          if (threadIdx.x == 0) {
            double t = s;
            for (int i = 0; i < len; ++i) t = t + sm_d[i];
            sm_M = __double_as_longlong(t);
          }
          __syncthreads();
          s = __longlong_as_double(sm_M);
          __syncthreads();
        }
        continue;
      }
      bool fast = false;
      if (sg.ok && s >= 0x1p-1000 && isfinite(s) && ilogb(s) == sg.e) {
        const double inv_u = ldexp(1.0, 52 - sg.e);
        const long long ms = static_cast<long long>(s * inv_u);
        const long long M = ms + ((ms & 1) ? sg.a1 : sg.a0);
        if (M < kTwo53) {
          s = ldexp(static_cast<double>(M), sg.e - 52);
          fast = true;
        }
      }
      if (!fast) sum_range(diag, sg.k0, sg.k1, s, sm_d, sm_warp, &sm_event, &sm_M);
    }
  } else {
    sum_range(diag, 0, ntris, s, sm_d, sm_warp, &sm_event, &sm_M);
  }
  if (threadIdx.x == 0) {
    const double mean = ntris > 0 ? s / ntris : 1.0;
    const double a = cell_scale * mean;
    out[0] = (a < 1e-9) ? 1e-9 : a;  // std::max(a, 1e-9)
  }
}

// Reference serial sum (validation only: weft_gpu_serial_sum).
__global__ void k_serial_sum_naive(int n, const double* __restrict__ d, double* __restrict__ out) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = s + d[i];
  out[0] = s;
}

constexpr size_t kSumSmem = sizeof(double) * kSumThreads * kSumItems;

static void launch_cell_size(Ctx& c, int n, const double* d, double scale, double* out, bool fast = true) {
  SumSeg* seg = nullptr;
  int* nseg = nullptr;
  if (fast && n > 0) {
    const int max_seg = div_up(n, kSumChunk) + 2 * kMaxCross + 2;
    c.sum_approx.resize(static_cast<size_t>(n));
    c.sum_maps.resize(static_cast<size_t>(max_seg) * sizeof(SumSeg) + (kMaxCross + 4) * sizeof(int));
    seg = reinterpret_cast<SumSeg*>(c.sum_maps.data());
    int* xs = reinterpret_cast<int*>(c.sum_maps.data() + static_cast<size_t>(max_seg) * sizeof(SumSeg));
    int* nx = xs + kMaxCross;
    nseg = nx + 1;
    size_t tmp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp, d, c.sum_approx.data(), n, c.cur);
    void* t = scratch(c, tmp);
    WG_CUDA(cub::DeviceScan::InclusiveSum(t, tmp, d, c.sum_approx.data(), n, c.cur));
    WG_CUDA(cudaMemsetAsync(nx, 0, sizeof(int), c.cur));
    k_cross_find<<<div_up(n, 256), 256, 0, ls(c)>>>(n, c.sum_approx.data(), xs, nx);
    k_seg_build<<<1, 32, 0, ls(c)>>>(n, xs, nx, seg, nseg);
    k_seg_maps<<<max_seg, kSumThreads, 0, ls(c)>>>(d, c.sum_approx.data(), seg, nseg);
  }
  WG_CUDA(cudaFuncSetAttribute(k_cell_size, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSumSmem));
  k_cell_size<<<1, kSumThreads, kSumSmem, ls(c)>>>(n, d, seg, nseg, scale, out);
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

// Lattice bounds (min lo, max hi per axis) so cell keys can be sorted in a
// compact, order-isomorphic form: ((ix-x0)*ey + (iy-y0))*ez + (iz-z0)
// orders cells exactly like the reference's packed 63-bit key.
__global__ void __launch_bounds__(256) k_lat_bounds(int ntris, const int* __restrict__ lat, int* __restrict__ bounds) {
  __shared__ int sm[8][6];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  int v[6] = {INT_MAX, INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MIN};
  if (t < ntris) {
#pragma unroll
    for (int c = 0; c < 6; ++c) v[c] = lat[6 * t + c];
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    for (int o = 16; o > 0; o >>= 1) {
      v[c] = min(v[c], __shfl_xor_sync(0xffffffffu, v[c], o));
      v[c + 3] = max(v[c + 3], __shfl_xor_sync(0xffffffffu, v[c + 3], o));
    }
  }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int c = 0; c < 6; ++c) sm[warp][c] = v[c];
  __syncthreads();
  if (threadIdx.x < 6) {
    const int c = threadIdx.x;
    int r = sm[0][c];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = c < 3 ? min(r, sm[w][c]) : max(r, sm[w][c]);
    if (c < 3) atomicMin(bounds + c, r);
    else atomicMax(bounds + c, r);
  }
}

struct KeyFrame {
  int x0, y0, z0;
  long long ey, ez;
  __device__ __forceinline__ unsigned long long compact(int ix, int iy, int iz) const {
    return (static_cast<unsigned long long>(ix - x0) * ey + static_cast<unsigned long long>(iy - y0)) * ez +
           static_cast<unsigned long long>(iz - z0);
  }
  __device__ __forceinline__ uint64_t packed(unsigned long long k) const {
    const int iz = static_cast<int>(k % ez) + z0;
    k /= ez;
    const int iy = static_cast<int>(k % ey) + y0;
    const int ix = static_cast<int>(k / ey) + x0;
    return pack_cell(ix, iy, iz);
  }
};

template <class K>
__global__ void k_emit(int ntris, const int* __restrict__ lat, const int64_t* __restrict__ off, KeyFrame f,
                       K* __restrict__ keys, int32_t* __restrict__ vals) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntris) return;
  const int* b = lat + 6 * t;
  int64_t o = off[t];
  for (int ix = b[0]; ix <= b[3]; ++ix)
    for (int iy = b[1]; iy <= b[4]; ++iy)
      for (int iz = b[2]; iz <= b[5]; ++iz) {
        keys[o] = static_cast<K>(f.compact(ix, iy, iz));
        vals[o] = t;
        ++o;
      }
}

template <class K>
__global__ void k_cell_flags(int64_t n, const K* __restrict__ keys, int32_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// flag has been exclusive-scanned into idx: cell index of each run start.
template <class K>
__global__ void k_cells(int64_t n, const K* __restrict__ keys, const int32_t* __restrict__ flag_scan, KeyFrame f,
                        uint64_t* __restrict__ cell_keys, int64_t* __restrict__ cell_off) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0 || keys[i] != keys[i - 1]) {
    const int c = flag_scan[i];
    cell_keys[c] = f.packed(keys[i]);
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
  cudaStream_t s = c.cur;
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
  int* bounds = reinterpret_cast<int*>(c.scalars.data() + 16);
  const int init[6] = {INT_MAX, INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MIN};
  WG_CUDA(cudaMemcpyAsync(bounds, init, sizeof(init), cudaMemcpyHostToDevice, s));
  if (T) k_lat_bounds<<<div_up(T, 256), 256, 0, ls(c)>>>(T, c.lat.data(), bounds);
  int64_t K = 0;
  int hb[6];
  read_small(c, s, {c.ecount.data() + T, &K, sizeof(int64_t)}, {bounds, hb, sizeof(hb)},
             {c.cell_size.data(), &c.grid_cell_size, sizeof(double)});
  if (K > (int64_t(1) << 31) - 1) throw Error(WEFT_ERR_DIMENSION, "build_grid: more than 2^31 cell entries");
  KeyFrame f{0, 0, 0, 1, 1};
  int bits = 1;
  if (T) {
    f = KeyFrame{hb[0], hb[1], hb[2], static_cast<long long>(hb[4]) - hb[1] + 1, static_cast<long long>(hb[5]) - hb[2] + 1};
    const unsigned long long ex = static_cast<unsigned long long>(static_cast<long long>(hb[3]) - hb[0] + 1);
    const unsigned long long span = ex * static_cast<unsigned long long>(f.ey) * static_cast<unsigned long long>(f.ez);
    while (bits < 64 && (1ULL << bits) < span) ++bits;
  }
  const bool narrow = bits <= 32;
  c.keys_a.resize(static_cast<size_t>(K) + 1);
  c.keys_b.resize(static_cast<size_t>(K) + 1);
  c.vals_a.resize(static_cast<size_t>(K) + 1);
  c.vals_b.resize(static_cast<size_t>(K) + 1);
  auto* ka32 = reinterpret_cast<uint32_t*>(c.keys_a.data());
  auto* kb32 = reinterpret_cast<uint32_t*>(c.keys_b.data());
  if (T) {
    if (narrow) k_emit<uint32_t><<<div_up(T, 256), 256, 0, ls(c)>>>(T, c.lat.data(), c.ecount.data(), f, ka32, c.vals_a.data());
    else k_emit<uint64_t><<<div_up(T, 256), 256, 0, ls(c)>>>(T, c.lat.data(), c.ecount.data(), f, c.keys_a.data(), c.vals_a.data());
  }
  if (K) {  // stable LSD radix sort: per-cell triangle lists stay ascending
    tmp = 0;
    if (narrow) {
      cub::DeviceRadixSort::SortPairs(nullptr, tmp, ka32, kb32, c.vals_a.data(), c.vals_b.data(), (int)K, 0, bits, s);
      t = scratch(c, tmp);
      WG_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, ka32, kb32, c.vals_a.data(), c.vals_b.data(), (int)K, 0, bits, s));
    } else {
      cub::DeviceRadixSort::SortPairs(nullptr, tmp, c.keys_a.data(), c.keys_b.data(), c.vals_a.data(), c.vals_b.data(),
                                      (int)K, 0, bits, s);
      t = scratch(c, tmp);
      WG_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, c.keys_a.data(), c.keys_b.data(), c.vals_a.data(),
                                              c.vals_b.data(), (int)K, 0, bits, s));
    }
  }
  // run-length cells
  c.cell_flag.resize(static_cast<size_t>(K) + 1);
  if (K) {
    if (narrow) k_cell_flags<uint32_t><<<div_up(K, 256), 256, 0, ls(c)>>>(K, kb32, c.cell_flag.data());
    else k_cell_flags<uint64_t><<<div_up(K, 256), 256, 0, ls(c)>>>(K, c.keys_b.data(), c.cell_flag.data());
  }
  WG_CUDA(cudaMemsetAsync(c.cell_flag.data() + K, 0, sizeof(int32_t), s));
  tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.cell_flag.data(), c.cell_flag.data(), K + 1, s);
  t = scratch(c, tmp);
  WG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, c.cell_flag.data(), c.cell_flag.data(), K + 1, s));
  int32_t cells32 = 0;
  read_small(c, s, {c.cell_flag.data() + K, &cells32, sizeof(int32_t)});
  const int64_t cells = cells32;
  c.cell_keys.resize(static_cast<size_t>(cells) + 1);
  c.cell_off.resize(static_cast<size_t>(cells) + 1);
  c.wprefix.resize(static_cast<size_t>(cells) + 1);
  if (K) {
    if (narrow) k_cells<uint32_t><<<div_up(K, 256), 256, 0, ls(c)>>>(K, kb32, c.cell_flag.data(), f, c.cell_keys.data(), c.cell_off.data());
    else k_cells<uint64_t><<<div_up(K, 256), 256, 0, ls(c)>>>(K, c.keys_b.data(), c.cell_flag.data(), f, c.cell_keys.data(), c.cell_off.data());
  }
  WG_CUDA(cudaMemcpyAsync(c.cell_off.data() + cells, &K, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  if (cells) k_pair_counts<<<div_up(cells, 256), 256, 0, ls(c)>>>(cells, c.cell_off.data(), c.wprefix.data());
  WG_CUDA(cudaMemsetAsync(c.wprefix.data() + cells, 0, sizeof(int64_t), s));
  tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.wprefix.data(), c.wprefix.data(), cells + 1, s);
  t = scratch(c, tmp);
  WG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, c.wprefix.data(), c.wprefix.data(), cells + 1, s));
  WG_CUDA(cudaGetLastError());
  read_small(c, s, {c.wprefix.data() + cells, &c.grid_total, sizeof(int64_t)});
  c.grid_entries = K;
  c.grid_cells = cells;
  c.has_grid = true;
}

// ---------------------------------------------------------------------------
// candidate walk
// ---------------------------------------------------------------------------
// One warp per occupied cell. The cell's pair range intersected with
// [begin, end) is enumerated in the reference's flattened (i, j) order with
// lane l taking local index base + l; a pair is a candidate iff the smallest
// common cell of the two lattice boxes, (max lo_x, max lo_y, max lo_z), is
// this cell (collision.cpp:205-210, 366-369) — only the lo corners are read,
// staged in shared memory. Hits are compacted with a warp ballot, so pass 2
// writes them in exactly the reference's walk order.
constexpr int kWalkWarps = 8;
constexpr int kWalkStage = 320;

struct WalkArgs {
  int64_t begin, end, cells;
  const int64_t* __restrict__ prefix;
  const int64_t* __restrict__ cell_off;
  const int32_t* __restrict__ cell_tris;
  const uint64_t* __restrict__ cell_keys;
  const int* __restrict__ lat;
  // narrow-phase feed (null: every candidate): only pairs whose conservative
  // float boxes are within `margin` are emitted — the whole-pair rejection
  // k_narrow applies first (narrow.cu), so the same hits; the unfiltered
  // candidate count still goes to *all_count
  const float4* __restrict__ tbox;
  double margin;
  unsigned long long* __restrict__ all_count;
  // append mode (kMode 2, the narrow-phase feed): pairs in no particular
  // order, claimed from *cursor; entries at or beyond cap are dropped and the
  // caller re-runs with the exact count
  unsigned long long* __restrict__ cursor;
  int64_t cap;
};

// Append mode: a warp's passing pairs gather in a shared-memory buffer and
// go out with one atomic claim per flush (coalesced copies).
constexpr int kAppendBuf = 480;  // int2 entries: the bitset path's unused sm_lo stage of the warp
__device__ __forceinline__ void append_flush(const WalkArgs& w, int2* buf, int& bn, int lane, int2* __restrict__ out) {
  __syncwarp();
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(w.cursor, static_cast<unsigned long long>(bn));
  base = __shfl_sync(0xffffffffu, base, 0);
  for (int k = lane; k < bn; k += 32)
    if (base + k < static_cast<unsigned long long>(w.cap)) out[base + k] = buf[k];
  __syncwarp();
  bn = 0;
}

__device__ __forceinline__ bool boxes_apart(const float4* __restrict__ tbox, int t1, int t2, double margin) {
  const float4 la = __ldg(tbox + 2 * t1), ha = __ldg(tbox + 2 * t1 + 1);
  const float4 lb = __ldg(tbox + 2 * t2), hb = __ldg(tbox + 2 * t2 + 1);
  return (double)la.x > (double)hb.x + margin || (double)lb.x > (double)ha.x + margin ||
         (double)la.y > (double)hb.y + margin || (double)lb.y > (double)ha.y + margin ||
         (double)la.z > (double)hb.z + margin || (double)lb.z > (double)ha.z + margin;
}

// row i of the upper triangle starts at local index i*s - i(i+1)/2
__device__ __forceinline__ int64_t tri_start(int64_t i, int64_t s) { return i * s - i * (i + 1) / 2; }

// Cells of up to kBitsetMax triangles are walked as bitsets. Every triangle
// of the cell has lo <= cell per axis (its box covers the cell), so
// max(lo_a, lo_b) == cell on an axis iff a or b has lo == cell there: with
// m = (lo.x == cx) | (lo.y == cy) << 1 | (lo.z == cz) << 2, (a, b) is a
// candidate iff m_a | m_b == 7. S[r] = {j : m_j contains r} is built with
// one ballot per (r, 32 triangles); lane l takes rows i = l, l + 32, ... of
// the upper triangle, whose candidates j > i are the set bits of
// S[7 & ~m_i] above i — the same pairs, in the same (i, j) walk order, as
// enumerating every pair, restricted to the local index range [l0, l1) of
// the split. (Config D: 98 triangles per DCD cell on average, 283 M raw
// pairs per build; 178 at most.)
constexpr int kBitsetMax = 256;

// kMode: 0 count, 1 write in walk order at o, 2 append (w.cursor; needs tbox)
template <int kMode>
__device__ __forceinline__ int64_t walk_bitset(const WalkArgs& wa, int s, int lane, int64_t l0, int64_t l1,
                                               const int32_t* __restrict__ tl, const int* __restrict__ lat, int cx,
                                               int cy, int cz, int* sm_id, unsigned* sm_set, int2* sm_buf, int64_t o,
                                               int2* __restrict__ out, const float4* __restrict__ tbox, double margin,
                                               int64_t& nall) {
  constexpr bool kWrite = kMode == 1;
  constexpr int G = kBitsetMax / 32;
  const int ng = (s + 31) >> 5;
  int m[G];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    const int i = lane + 32 * h;
    m[h] = 0;
    if (i < s) {
      const int t = tl[i];
      sm_id[i] = t;
      const int* b = lat + 6 * t;
      m[h] = (b[0] == cx ? 1 : 0) | (b[1] == cy ? 2 : 0) | (b[2] == cz ? 4 : 0);
    }
    if (h < ng) {  // warp-uniform
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const unsigned w = __ballot_sync(0xffffffffu, i < s && (m[h] & r) == r);
        if (lane == 0) sm_set[r * G + h] = w;
      }
    }
  }
  __syncwarp();
  int64_t n = 0;
  if constexpr (kMode == 2) {
    // one pass: every lane steps through its candidates one per round
    // (warp-synchronous), the survivors of the float-box test are compacted
    // into the warp's buffer by ballot
    int bn = 0;
#pragma unroll
    for (int h = 0; h < G; ++h) {
      if (h >= ng) break;  // warp-uniform
      const int i = lane + 32 * h;
      const unsigned* Sr = sm_set + (7 & ~m[h]) * G;
      int64_t jlo = 0, jhi = 0;
      int call = 0, g = ng;
      unsigned bits = 0;
      auto group_bits = [&](int gg) -> unsigned {
        unsigned b = Sr[gg];
        const int64_t b0 = jlo - 32 * gg, b1 = jhi - 32 * gg;  // keep bits in [b0, b1)
        if (b0 > 0) b &= ~0u << b0;
        if (b1 < 32) b &= (1u << b1) - 1u;
        return b;
      };
      if (i < s) {
        const int64_t rs = tri_start(i, s);
        jlo = max(l0 - rs + i + 1, static_cast<int64_t>(i + 1));
        jhi = min(l1 - rs + i + 1, static_cast<int64_t>(s));
        for (int gg = static_cast<int>(jlo >> 5); gg < ng && 32 * gg < jhi; ++gg) call += __popc(group_bits(gg));
        g = static_cast<int>(jlo >> 5);
        while (g < ng && 32 * g < jhi && !(bits = group_bits(g))) ++g;
        if (!(g < ng && 32 * g < jhi)) bits = 0;
      }
      nall += __reduce_add_sync(0xffffffffu, call);
      const int ti = i < s ? sm_id[i] : 0;
      while (__any_sync(0xffffffffu, bits != 0)) {
        bool pass = false;
        int tj = 0;
        if (bits) {
          const int j = 32 * g + __ffs(bits) - 1;
          bits &= bits - 1;
          tj = sm_id[j];
          pass = !boxes_apart(tbox, ti, tj, margin);
          if (!bits) {
            ++g;
            while (g < ng && 32 * g < jhi && !(bits = group_bits(g))) ++g;
          }
        }
        const unsigned pm = __ballot_sync(0xffffffffu, pass);
        if (pass) sm_buf[bn + __popc(pm & ((1u << lane) - 1u))] = make_int2(ti, tj);
        bn += __popc(pm);
        n += __popc(pm);
        if (bn > kAppendBuf - 32) append_flush(wa, sm_buf, bn, lane, out);
      }
    }
    if (bn) append_flush(wa, sm_buf, bn, lane, out);
    __syncwarp();
    return n;
  }
#pragma unroll
  for (int h = 0; h < G; ++h) {
    if (h >= ng) break;  // warp-uniform
    const int i = lane + 32 * h;
    int c = 0;
    int64_t jlo = 0, jhi = 0;
    const unsigned* Sr = sm_set + (7 & ~m[h]) * G;
    int call = 0;
    if (i < s) {
      // the split range: the local index of (i, j) is tri_start(i, s) + j - i - 1
      const int64_t rs = tri_start(i, s);
      jlo = max(l0 - rs + i + 1, static_cast<int64_t>(i + 1));
      jhi = min(l1 - rs + i + 1, static_cast<int64_t>(s));
      const int ti = tbox ? sm_id[i] : 0;
      for (int g = static_cast<int>(jlo >> 5); g < ng && 32 * g < jhi; ++g) {
        unsigned bits = Sr[g];
        const int64_t b0 = jlo - 32 * g, b1 = jhi - 32 * g;  // keep bits in [b0, b1)
        if (b0 > 0) bits &= ~0u << b0;
        if (b1 < 32) bits &= (1u << b1) - 1u;
        call += __popc(bits);
        if (tbox) {
          while (bits) {
            const int j = 32 * g + __ffs(bits) - 1;
            bits &= bits - 1;
            c += boxes_apart(tbox, ti, sm_id[j], margin) ? 0 : 1;
          }
        } else {
          c += __popc(bits);
        }
      }
    }
    nall += __reduce_add_sync(0xffffffffu, call);
    if (kWrite) {
      int x = c;  // inclusive scan of the rows' counts (row order = lane order)
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += v;
      }
      int64_t w = o + n + (x - c);
      if (c) {
        const int ti = sm_id[i];
        for (int g = static_cast<int>(jlo >> 5); g < ng && 32 * g < jhi; ++g) {
          unsigned bits = Sr[g];
          const int64_t b0 = jlo - 32 * g, b1 = jhi - 32 * g;
          if (b0 > 0) bits &= ~0u << b0;
          if (b1 < 32) bits &= (1u << b1) - 1u;
          while (bits) {
            const int j = 32 * g + __ffs(bits) - 1;
            bits &= bits - 1;
            const int tj = sm_id[j];
            if (!tbox || !boxes_apart(tbox, ti, tj, margin)) out[w++] = make_int2(ti, tj);
          }
        }
      }
    }
    n += __reduce_add_sync(0xffffffffu, c);
  }
  __syncwarp();
  return n;
}

template <int kMode>
__global__ void __launch_bounds__(kWalkWarps * 32) k_cell_walk(WalkArgs w, int64_t* __restrict__ counts,
                                                               const int64_t* __restrict__ offs,
                                                               int2* __restrict__ out) {
  constexpr bool kWrite = kMode == 1;
  static_assert(kAppendBuf * sizeof(int2) <= kWalkStage * sizeof(int3), "append buffer aliases sm_lo");
  __shared__ __align__(16) int3 sm_lo[kWalkWarps][kWalkStage];  // (also the append buffer: int2)
  __shared__ int sm_id[kWalkWarps][kWalkStage];
  __shared__ unsigned sm_set[kWalkWarps][8 * (kBitsetMax / 32)];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cell = blockIdx.x * (int64_t)kWalkWarps + warp;
  if (cell >= w.cells) return;  // warp-uniform
  const int64_t p0 = w.prefix[cell], p1 = w.prefix[cell + 1];
  const int64_t lo = max(p0, w.begin), hi = min(p1, w.end);
  int64_t n = 0;
  int64_t o = kWrite ? offs[cell] : 0;
  if (lo < hi) {
    const int64_t cbase = w.cell_off[cell];
    const int64_t s = w.cell_off[cell + 1] - cbase;
    const int32_t* tl = w.cell_tris + cbase;
    const uint64_t key = w.cell_keys[cell];
    const int cx = static_cast<int>(key >> 42) - static_cast<int>(kLatBias);
    const int cy = static_cast<int>((key >> 21) & 0x1FFFFF) - static_cast<int>(kLatBias);
    const int cz = static_cast<int>(key & 0x1FFFFF) - static_cast<int>(kLatBias);
    if (s <= kBitsetMax) {  // bitset walk (above)
      const int64_t l0 = lo - p0, l1 = hi - p0;
      int64_t nall = 0;
      n = walk_bitset<kMode>(w, static_cast<int>(s), lane, l0, l1, tl, w.lat, cx, cy, cz, sm_id[warp], sm_set[warp],
                             reinterpret_cast<int2*>(sm_lo[warp]), o, out, w.tbox, w.margin, nall);
      if (!kWrite && lane == 0) {
        if (kMode == 0) counts[cell] = n;
        if (w.all_count) atomicAdd(w.all_count, static_cast<unsigned long long>(nall));
      }
      return;
    }
    const bool staged = s <= kWalkStage;
    if (staged) {
      for (int i = lane; i < s; i += 32) {
        const int t = tl[i];
        sm_id[warp][i] = t;
        sm_lo[warp][i] = make_int3(w.lat[6 * t], w.lat[6 * t + 1], w.lat[6 * t + 2]);
      }
    }
    __syncwarp();
    auto load = [&](int64_t i, int& t, int3& l) {
      if (staged) {
        t = sm_id[warp][i];
        l = sm_lo[warp][i];
      } else {
        t = tl[i];
        l = make_int3(w.lat[6 * t], w.lat[6 * t + 1], w.lat[6 * t + 2]);
      }
    };
    // decode this lane's first local index
    const int64_t l0 = lo - p0, l1 = hi - p0;
    int64_t k = l0 + lane;
    int64_t i = 0, j = 0;
    if (k < l1) {
      const double b = 2.0 * s - 1.0;
      i = static_cast<int64_t>(floor((b - sqrt(fmax(b * b - 8.0 * static_cast<double>(k), 0.0))) * 0.5));
      if (i < 0) i = 0;
      while (i > 0 && tri_start(i, s) > k) --i;
      while (tri_start(i + 1, s) <= k) ++i;
      j = i + 1 + (k - tri_start(i, s));
    }
    for (int64_t kb = l0; kb < l1; kb += 32) {
      const bool act = k < l1;
      bool hit = false;
      int t1 = 0, t2 = 0;
      if (act) {
        int3 a, c;
        load(i, t1, a);
        load(j, t2, c);
        hit = max(a.x, c.x) == cx && max(a.y, c.y) == cy && max(a.z, c.z) == cz;
      }
      if (w.tbox) {
        const unsigned ma = __ballot_sync(0xffffffffu, hit);
        if (!kWrite && lane == 0 && w.all_count) atomicAdd(w.all_count, static_cast<unsigned long long>(__popc(ma)));
        if (hit && boxes_apart(w.tbox, t1, t2, w.margin)) hit = false;
      }
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (kWrite && hit) out[o + __popc(m & ((1u << lane) - 1u))] = make_int2(t1, t2);
      if (kMode == 2 && m) {  // cells over kBitsetMax (rare): one claim per round
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(w.cursor, static_cast<unsigned long long>(__popc(m)));
        base = __shfl_sync(0xffffffffu, base, 0) + __popc(m & ((1u << lane) - 1u));
        if (hit && base < static_cast<unsigned long long>(w.cap)) out[base] = make_int2(t1, t2);
      }
      o += __popc(m);
      n += __popc(m);
      // advance this lane by 32 local indices
      k += 32;
      if (k < l1) {
        int64_t adv = 32;
        while (adv > 0) {
          const int64_t room = s - j;
          if (adv < room) {
            j += adv;
            adv = 0;
          } else {
            adv -= room;
            ++i;
            j = i + 1;
          }
        }
      }
    }
  }
  if (kMode == 0 && lane == 0) counts[cell] = n;
}

// Returns the candidate count of [begin, end); when pairs_out is non-null
// the pairs are written there (device or host pointer). Device-resident
// pairs stay in c.cand_pairs.
int64_t candidates(Ctx& c, int64_t begin, int64_t end, int32_t* pairs_out, bool count_only, const float4* tbox,
                   double margin, int64_t* all) {
  if (!c.has_grid) throw Error(WEFT_ERR_INVALID, "candidates: build_grid first");
  begin = std::max<int64_t>(begin, 0);
  end = std::min<int64_t>(end, c.grid_total);
  if (begin >= end) return 0;
  cudaStream_t s = c.cur;
  const int64_t cells = c.grid_cells;
  c.cand_all.resize(1);
  if (tbox) WG_CUDA(cudaMemsetAsync(c.cand_all.data(), 0, sizeof(unsigned long long), s));
  WalkArgs w{begin, end, cells, c.wprefix.data(), c.cell_off.data(), c.vals_b.data(), c.cell_keys.data(),
             c.lat.data(), tbox, margin, tbox ? c.cand_all.data() : nullptr, nullptr, 0};
  const int blocks = div_up(cells, kWalkWarps);
  static const bool append_off = std::getenv("WEFT_WALK_APPEND") && std::atoi(std::getenv("WEFT_WALK_APPEND")) == 0;
  if (tbox && !count_only && !pairs_out && !append_off) {
    // the narrow-phase feed: its consumer sorts the hits, so the pairs go
    // out in one order-free pass (append mode) — no count pass, no scan
    c.cand_cursor.resize(1);
    w.cursor = c.cand_cursor.data();
    // the pairs the buffer already holds (never grows it on its own), at least
    // 4 M (WEFT_WALK_CAP: an exact first capacity, tests of the re-run path)
    static const int64_t cap_env = std::getenv("WEFT_WALK_CAP") ? std::atoll(std::getenv("WEFT_WALK_CAP")) : 0;
    int64_t cap = cap_env > 0 ? cap_env
                              : std::max<int64_t>((static_cast<int64_t>(c.cand_pairs.cap) - 2) / 2, int64_t{1} << 22);
    int64_t n = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
      c.cand_pairs.resize(2 * static_cast<size_t>(cap) + 2);
      w.cap = cap;
      WG_CUDA(cudaMemsetAsync(c.cand_cursor.data(), 0, sizeof(unsigned long long), s));
      WG_CUDA(cudaMemsetAsync(c.cand_all.data(), 0, sizeof(unsigned long long), s));
      k_cell_walk<2><<<blocks, kWalkWarps * 32, 0, ls(c)>>>(w, nullptr, nullptr,
                                                            reinterpret_cast<int2*>(c.cand_pairs.data()));
      WG_CUDA(cudaGetLastError());
      unsigned long long nc = 0, na = 0;
      read_small(c, s, {c.cand_cursor.data(), &nc, sizeof(nc)}, {c.cand_all.data(), &na, sizeof(na)});
      n = static_cast<int64_t>(nc);
      if (all) *all = static_cast<int64_t>(na);
      if (n <= cap) break;
      cap = n;  // exact capacity, run once more
    }
    return n;
  }
  c.cand_count.resize(static_cast<size_t>(cells) + 1);
  WG_CUDA(cudaMemsetAsync(c.cand_count.data() + cells, 0, sizeof(int64_t), s));
  k_cell_walk<0><<<blocks, kWalkWarps * 32, 0, ls(c)>>>(w, c.cand_count.data(), nullptr, nullptr);
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.cand_count.data(), c.cand_count.data(), cells + 1, s);
  void* t = scratch(c, tmp);
  WG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, c.cand_count.data(), c.cand_count.data(), cells + 1, s));
  int64_t n = 0;
  if (tbox && all) {
    unsigned long long na = 0;
    read_small(c, s, {c.cand_count.data() + cells, &n, sizeof(int64_t)}, {c.cand_all.data(), &na, sizeof(na)});
    *all = static_cast<int64_t>(na);
  } else {
    read_small(c, s, {c.cand_count.data() + cells, &n, sizeof(int64_t)});
    if (all) *all = n;
  }
  if (count_only) return n;  // the walk's count pass is the whole result
  c.cand_pairs.resize(2 * static_cast<size_t>(n) + 2);
  k_cell_walk<1><<<blocks, kWalkWarps * 32, 0, ls(c)>>>(w, nullptr, c.cand_count.data(),
                                                        reinterpret_cast<int2*>(c.cand_pairs.data()));
  WG_CUDA(cudaGetLastError());
  if (pairs_out && n)
    WG_CUDA(cudaMemcpyAsync(pairs_out, c.cand_pairs.data(), 2 * sizeof(int32_t) * n, cudaMemcpyDefault, s));
  WG_CUDA(cudaStreamSynchronize(s));
  return n;
}

// Test hook: exact parallel serial-order sum vs a one-thread serial loop.
void serial_sum(Ctx& c, int n, const double* d_host, double* exact, double* naive, int fast) {
  DBuf<double> d, o;
  d.upload(d_host, static_cast<size_t>(n), c.stream);
  o.resize(2);
  launch_cell_size(c, n, d.data(), 1.0, o.data(), fast != 0);  // cell = max(sum / n, 1e-9)
  k_serial_sum_naive<<<1, 1, 0, ls(c)>>>(n, d.data(), o.data() + 1);
  WG_CUDA(cudaGetLastError());
  double h[2];
  WG_CUDA(cudaMemcpyAsync(h, o.data(), sizeof(h), cudaMemcpyDeviceToHost, c.stream));
  WG_CUDA(cudaStreamSynchronize(c.stream));
  *exact = h[0];
  *naive = h[1];
}

}  // namespace weft_gpu
