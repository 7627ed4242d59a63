// zones.cu — impact zones: the CCD-and-resolve loop of
// resolve_zones, build_zones and solve_zone on the device.
//
// Reference: proj/src/response.cpp — build_zones (:108-162), distribute_zones
// (:164-182), constraint_gap (:191-195), solve_zone (:199-336),
// resolve_zones (:338-400); ZoneSolveParams / ZoneResolveReport
// (proj/include/weft/response.hpp:46-73).
//
// Device pipeline per outer round:
//   collide(CCD, begin -> candidate)            (narrow.cu, sorted by key)
//   -> accumulate unseen (kind, a, b) keys in first-crossing order
//   -> build_zones: participants, per-vertex first owner (atomicMin), lock-free
//      union-find hooking larger roots under smaller ones (the root of every
//      component is its smallest impact, so zone ids = rank of the root =
//      the reference's numbering by first impact), stable radix sort of
//      impacts by zone (ascending impact index inside a zone), sorted unique
//      movable (zone, vertex) keys, per-vertex incidence lists
//      (zone-vertex slot, zone-impact position, participant) in constraint
//      order
//   -> k_solve_zones: ONE WARP PER ZONE (zones are vertex-disjoint, so warps
//      never touch each other's positions). Per-vertex and per-constraint
//      terms are computed lane-parallel; every sum the reference forms
//      left to right (objective, gradient norm, mean mass) is formed by lane
//      0 over the lane-written terms in the same order, and every gradient
//      component subtracts its constraint forces in ascending constraint
//      order, so positions are bitwise the reference's (-fmad=false, the
//      Eigen shim's left-to-right association).
//   -> trust-region clamp of each zone vertex's move (resolve_zones :372-378).
#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "elements.cuh"

namespace weft_gpu {
namespace {

__device__ __forceinline__ double dmax0(double t) { return 0.0 < t ? t : 0.0; }  // std::max(0.0, t)
__device__ __forceinline__ V3 ld3(const double* __restrict__ x, int v) {
  return V3{x[3 * v], x[3 * v + 1], x[3 * v + 2]};
}
__device__ __forceinline__ void st3(double* __restrict__ x, int v, V3 a) {
  x[3 * v] = a.x;
  x[3 * v + 1] = a.y;
  x[3 * v + 2] = a.z;
}
__device__ __forceinline__ double bcast(double v) { return __shfl_sync(0xffffffffu, v, 0); }

__device__ __forceinline__ int lower_bound_u64(const unsigned long long* __restrict__ a, int64_t n,
                                               unsigned long long key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return static_cast<int>(lo);
}

// ---- accumulation (resolve_zones :349-354: one constraint per feature pair,
// first crossing wins) --------------------------------------------------------
__global__ void k_zone_unseen(int64_t nf, const unsigned long long* __restrict__ fresh, int64_t m,
                              const unsigned long long* __restrict__ sorted, int64_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nf) return;
  const unsigned long long k = fresh[i];
  const int lb = lower_bound_u64(sorted, m, k);
  flag[i] = (lb < m && sorted[lb] == k) ? 0 : 1;
}

__global__ void k_zone_append(int64_t nf, const unsigned long long* __restrict__ fresh,
                              const double* __restrict__ fresh_vals, const int64_t* __restrict__ pos, int64_t m,
                              unsigned long long* __restrict__ keys, double* __restrict__ vals) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nf || pos[i + 1] == pos[i]) return;
  const int64_t o = m + pos[i];
  keys[o] = fresh[i];
#pragma unroll
  for (int q = 0; q < 8; ++q) vals[8 * o + q] = fresh_vals[8 * i + q];
}

// ---- build_zones (:108-162) ------------------------------------------------
// participants (response.cpp:21-39) of impact i; owner[v] = first impact
// touching v (the reference's vertex_owner, :136-145).
__global__ void k_zone_parts(int64_t m, const unsigned long long* __restrict__ keys, const double* __restrict__ vals,
                             const int32_t* __restrict__ tris, const int2* __restrict__ edges,
                             int32_t* __restrict__ part_v, double* __restrict__ part_w, int32_t* __restrict__ owner,
                             int32_t* __restrict__ parent) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const unsigned long long k = keys[i];
  const int kind = static_cast<int>(k >> 62);
  const int a = static_cast<int>((k >> 31) & 0x7FFFFFFFull), b = static_cast<int>(k & 0x7FFFFFFFull);
  const double* hw = vals + 8 * i + 4;
  int v[4];
  double w[4];
  if (kind == 0) {
    v[0] = a;
    w[0] = 1.0;
    for (int q = 0; q < 3; ++q) {
      v[q + 1] = tris[3 * b + q];
      w[q + 1] = -hw[q + 1];
    }
  } else {
    const int2 e1 = edges[a], e2 = edges[b];
    v[0] = e1.x;
    w[0] = hw[0];
    v[1] = e1.y;
    w[1] = hw[1];
    v[2] = e2.x;
    w[2] = -hw[2];
    v[3] = e2.y;
    w[3] = -hw[3];
  }
  for (int q = 0; q < 4; ++q) {
    part_v[4 * i + q] = v[q];
    part_w[4 * i + q] = w[q];
    atomicMin(owner + v[q], static_cast<int32_t>(i));
  }
  parent[i] = static_cast<int32_t>(i);
}

__device__ __forceinline__ int uf_find(int32_t* parent, int x) {
  // path halving; every parent pointer only ever moves to a smaller index
  int p = __ldcg(parent + x);
  while (p != x) {
    const int gp = __ldcg(parent + p);
    if (gp != p) parent[x] = gp;
    x = p;
    p = gp;
  }
  return x;
}

__global__ void k_zone_union(int64_t m, const int32_t* __restrict__ part_v, const int32_t* __restrict__ owner,
                             int32_t* parent) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  for (int q = 0; q < 4; ++q) {
    int a = static_cast<int>(i), b = owner[part_v[4 * i + q]];
    while (true) {
      a = uf_find(parent, a);
      b = uf_find(parent, b);
      if (a == b) break;
      if (a < b) {
        const int t = a;
        a = b;
        b = t;
      }
      // hook the larger root a under the smaller root b
      if (atomicCAS(parent + a, a, b) == a) break;
    }
  }
}

__global__ void k_zone_roots(int64_t m, int32_t* parent, int64_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int r = uf_find(parent, static_cast<int>(i));
  flag[i] = (r == i) ? 1 : 0;
}

__global__ void k_zone_of(int64_t m, int32_t* parent, const int64_t* __restrict__ zid, int32_t* __restrict__ zone_of,
                          int32_t* __restrict__ iota) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  zone_of[i] = static_cast<int32_t>(zid[uf_find(parent, static_cast<int>(i))]);
  iota[i] = static_cast<int32_t>(i);
}

// off[z] = first position of zone z in the zone-sorted impact list
__global__ void k_zone_run_starts(int64_t m, const int32_t* __restrict__ zs, int32_t* __restrict__ off, int32_t nz) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i == 0) off[nz] = static_cast<int32_t>(m);
  if (i >= m) return;
  if (i == 0 || zs[i] != zs[i - 1]) off[zs[i]] = static_cast<int32_t>(i);
}

// (zone << 32 | vertex) for every movable participant (:154-160)
__global__ void k_zone_vkeys(int64_t m, const int32_t* __restrict__ part_v, const int32_t* __restrict__ zone_of,
                             const uint8_t* __restrict__ movable, unsigned long long* __restrict__ vk) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 4 * m) return;
  const int v = part_v[t];
  vk[t] = movable[v] ? ((static_cast<unsigned long long>(zone_of[t >> 2]) << 32) | static_cast<unsigned int>(v))
                     : ~0ull;
}

__global__ void k_unique_u64_flags(int64_t n, const unsigned long long* __restrict__ k, int64_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = (k[i] != ~0ull && (i == 0 || k[i] != k[i - 1])) ? 1 : 0;
}

__global__ void k_compact_u64(int64_t n, const unsigned long long* __restrict__ k, const int64_t* __restrict__ pos,
                              unsigned long long* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || pos[i + 1] == pos[i]) return;
  out[pos[i]] = k[i];
}

// zone-vertex offsets: voff[z] = lower_bound(vkeys, z << 32), z in [0, nz]
__global__ void k_zone_voff(int32_t nz, const unsigned long long* __restrict__ vk, int64_t nzv,
                            int32_t* __restrict__ voff) {
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  if (z > nz) return;
  voff[z] = lower_bound_u64(vk, nzv, static_cast<unsigned long long>(z) << 32);
}

// incidence keys: (slot << 34 | zone-impact position << 2 | participant)
__global__ void k_zone_ikeys(int64_t m, const int32_t* __restrict__ zimp, const int32_t* __restrict__ zs,
                             const int32_t* __restrict__ part_v, const uint8_t* __restrict__ movable,
                             const unsigned long long* __restrict__ vk, int64_t nzv,
                             unsigned long long* __restrict__ ik) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 4 * m) return;
  const int64_t gi = t >> 2;
  const int q = static_cast<int>(t & 3);
  const int v = part_v[4 * static_cast<int64_t>(zimp[gi]) + q];
  if (!movable[v]) {
    ik[t] = ~0ull;
    return;
  }
  const unsigned long long key = (static_cast<unsigned long long>(zs[gi]) << 32) | static_cast<unsigned int>(v);
  const unsigned long long s = static_cast<unsigned long long>(lower_bound_u64(vk, nzv, key));
  ik[t] = (s << 34) | (static_cast<unsigned long long>(gi) << 2) | static_cast<unsigned long long>(q);
}

__global__ void k_zone_ioff(int64_t nzv, const unsigned long long* __restrict__ ik, int64_t ni,
                            int32_t* __restrict__ ioff) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s > nzv) return;
  ioff[s] = lower_bound_u64(ik, ni, static_cast<unsigned long long>(s) << 34);
}

// ---- solve_zone (:199-336) + trust-region clamp (:368-379) ------------------
struct ZoneArgs {
  int32_t nz;
  const int32_t* __restrict__ zoff;   // nz + 1, into zimp
  const int32_t* __restrict__ zimp;   // impact index per zone-impact position
  const double* __restrict__ vals;    // impacts: 8 per impact
  const int32_t* __restrict__ part_v;
  const double* __restrict__ part_w;
  const int32_t* __restrict__ voff;   // nz + 1, into vkeys
  const unsigned long long* __restrict__ vkeys;
  const int32_t* __restrict__ ioff;   // nzv + 1, into ikeys
  const unsigned long long* __restrict__ ikeys;
  const double* __restrict__ mass;
  const double* __restrict__ xb;      // x_begin
  const double* __restrict__ xc;      // the round's proposal (x_candidate of solve_zone)
  double* x;                          // live candidate positions
  double* cn;                         // 3 per zone-impact position: oriented normal
  double* lam;                        // per zone-impact position
  double* force;
  double* tc;                         // per zone-impact position: objective terms
  double* tv;                         // per zone vertex: objective / gradient-norm terms
  double* grad;                       // 3 per zone vertex
  double* saved;                      // 3 per zone vertex
  int32_t* fail;                      // per zone: 1 = inner solver diverged
  double clearance, initial_penalty, inner_tolerance, max_move;
  int al_iterations, inner_iterations, retry_cap;
};

// constraint_gap (:191-195): g = -clearance + sum_p w_p (n . x_p), left to right
__device__ __forceinline__ double cgap(const ZoneArgs& g, int i, V3 n, const double* x, double clearance) {
  double r = -clearance;
#pragma unroll
  for (int q = 0; q < 4; ++q) r = r + g.part_w[4 * i + q] * dot(n, ld3(x, g.part_v[4 * i + q]));
  return r;
}

__device__ __forceinline__ int vslot_vertex(const ZoneArgs& g, int s) {
  return static_cast<int>(g.vkeys[s] & 0xFFFFFFFFull);
}

// objective (:226-240): lane-parallel terms, lane 0 sums them in order
__device__ double zone_objective(const ZoneArgs& g, int c0, int nc, int s0, int nv, double mu, int lane) {
  for (int j = lane; j < nv; j += 32) {
    const int s = s0 + j, v = vslot_vertex(g, s);
    const V3 d = sub(ld3(g.x, v), ld3(g.xc, v));
    g.tv[s] = (0.5 * g.mass[v]) * dot(d, d);
  }
  for (int j = lane; j < nc; j += 32) {
    const int gi = c0 + j;
    const double gg = cgap(g, g.zimp[gi], ld3(g.cn, gi), g.x, g.clearance);
    const double slack = dmax0(g.lam[gi] / mu - gg);
    g.tc[gi] = ((0.5 * mu) * slack) * slack;
  }
  __syncwarp();
  double val = 0.0;
  if (lane == 0) {
    for (int j = 0; j < nv; ++j) val = val + g.tv[s0 + j];
    for (int j = 0; j < nc; ++j) val = val + g.tc[c0 + j];
  }
  return bcast(val);
}

// compute_gradient (:242-266)
__device__ double zone_gradient(const ZoneArgs& g, int c0, int nc, int s0, int nv, double mu, int lane) {
  for (int j = lane; j < nc; j += 32) {
    const int gi = c0 + j;
    const double gg = cgap(g, g.zimp[gi], ld3(g.cn, gi), g.x, g.clearance);
    g.force[gi] = dmax0(g.lam[gi] - mu * gg);
  }
  __syncwarp();
  for (int j = lane; j < nv; j += 32) {
    const int s = s0 + j, v = vslot_vertex(g, s);
    const double m = g.mass[v];
    V3 gr = scl(m, sub(ld3(g.x, v), ld3(g.xc, v)));
    for (int e = g.ioff[s]; e < g.ioff[s + 1]; ++e) {
      const unsigned long long k = g.ikeys[e];
      const int gi = static_cast<int>((k >> 2) & 0xFFFFFFFFull), q = static_cast<int>(k & 3);
      const double f = g.force[gi];
      if (f <= 0.0) continue;
      gr = sub(gr, scl(f * g.part_w[4 * g.zimp[gi] + q], ld3(g.cn, gi)));
    }
    st3(g.grad, s, gr);
    g.tv[s] = dot(gr, gr) / m;
  }
  __syncwarp();
  double n2 = 0.0;
  if (lane == 0)
    for (int j = 0; j < nv; ++j) n2 = n2 + g.tv[s0 + j];
  return sqrt(bcast(n2));
}

__global__ void __launch_bounds__(128) k_solve_zones(ZoneArgs g) {
  const int z = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (z >= g.nz) return;  // warp-uniform
  const int c0 = g.zoff[z], nc = g.zoff[z + 1] - c0;
  const int s0 = g.voff[z], nv = g.voff[z + 1] - s0;
  // frozen constraints, normals oriented at the begin state (:206-213)
  for (int j = lane; j < nc; j += 32) {
    const int gi = c0 + j, i = g.zimp[gi];
    V3 n = ld3(g.vals + 8 * static_cast<int64_t>(i) + 1, 0);
    if (cgap(g, i, n, g.xb, 0.0) < 0.0) n = V3{-n.x, -n.y, -n.z};
    st3(g.cn, gi, n);
    g.lam[gi] = 0.0;
  }
  if (nv == 0) return;
  __syncwarp();
  double mean_mass = 0.0;
  if (lane == 0) {
    for (int j = 0; j < nv; ++j) mean_mass = mean_mass + g.mass[vslot_vertex(g, s0 + j)];
    mean_mass = mean_mass / nv;
  }
  mean_mass = bcast(mean_mass);
  double mu = g.initial_penalty * mean_mass;
  const double cl = g.clearance;
  const double grad_tol = (g.inner_tolerance * sqrt(mean_mass)) * (cl < 1e-9 ? 1e-9 : cl);

  int retries = 0;
  double step = 1.0;
  double last_violation = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  bool failed = false;
  for (int al = 0; al < g.al_iterations && !failed; ++al) {
    double fx = zone_objective(g, c0, nc, s0, nv, mu, lane);
    for (int it = 0; it < g.inner_iterations; ++it) {
      const double gnorm = zone_gradient(g, c0, nc, s0, nv, mu, lane);
      if (gnorm <= grad_tol) break;
      if (!isfinite(fx) || !isfinite(gnorm)) {
        if (++retries > g.retry_cap) {
          failed = true;
          break;
        }
        mu *= 10.0;
        step = 1.0;
        for (int j = lane; j < nv; j += 32) {
          const int v = vslot_vertex(g, s0 + j);
          st3(g.x, v, ld3(g.xc, v));
        }
        for (int j = lane; j < nc; j += 32) g.lam[c0 + j] = 0.0;
        __syncwarp();
        fx = zone_objective(g, c0, nc, s0, nv, mu, lane);
        continue;
      }
      for (int j = lane; j < nv; j += 32) {
        const int s = s0 + j;
        st3(g.saved, s, ld3(g.x, vslot_vertex(g, s)));
      }
      bool accepted = false;
      const double s2 = step * 2.0;
      step = 1.0 < s2 ? 1.0 : s2;  // std::min(step * 2.0, 1.0)
      for (int bt = 0; bt < 40; ++bt) {
        for (int j = lane; j < nv; j += 32) {
          const int s = s0 + j, v = vslot_vertex(g, s);
          st3(g.x, v, sub(ld3(g.saved, s), scl(step / g.mass[v], ld3(g.grad, s))));
        }
        __syncwarp();
        const double fnew = zone_objective(g, c0, nc, s0, nv, mu, lane);
        if (fnew <= fx - ((1e-4 * step) * gnorm) * gnorm) {
          fx = fnew;
          accepted = true;
          break;
        }
        step *= 0.5;
      }
      if (!accepted) {
        for (int j = lane; j < nv; j += 32) {
          const int s = s0 + j;
          st3(g.x, vslot_vertex(g, s), ld3(g.saved, s));
        }
        __syncwarp();
        break;  // no descent possible at this scale
      }
    }
    if (failed) break;
    // multiplier update and feasibility check (:318-332)
    int infeasible = 0;
    double violation = 0.0;
    for (int j = lane; j < nc; j += 32) {
      const int gi = c0 + j;
      const double gg = cgap(g, g.zimp[gi], ld3(g.cn, gi), g.x, cl);
      g.lam[gi] = dmax0(g.lam[gi] - mu * gg);
      if (gg < -1e-10) {
        infeasible = 1;
        violation = violation < -gg ? -gg : violation;
      }
    }
    __syncwarp();
    infeasible = __any_sync(0xffffffffu, infeasible);
    for (int o = 16; o > 0; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, violation, o);
      violation = violation < t ? t : violation;
    }
    if (!infeasible) break;
    if (violation > 0.25 * last_violation) mu *= 10.0;
    last_violation = violation;
  }
  if (failed) {
    if (lane == 0) g.fail[z] = 1;
    return;
  }
  // trust region (:372-378)
  for (int j = lane; j < nv; j += 32) {
    const int v = vslot_vertex(g, s0 + j);
    const V3 p = ld3(g.xc, v);
    const V3 mv = sub(ld3(g.x, v), p);
    const double len = norm(mv);
    if (len > g.max_move) st3(g.x, v, add(p, scl(g.max_move / len, mv)));
  }
}

// commit (driver.cpp:195-204): v += (corrected - candidate) / dt where moved
__global__ void k_zone_commit(int p, const double* __restrict__ corrected, const double* __restrict__ pre, double dt,
                              double* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p) return;
  const V3 a = ld3(corrected, i), b = ld3(pre, i);
  if (a.x != b.x || a.y != b.y || a.z != b.z) {
    const V3 d = sub(a, b);
    st3(v, i, add(ld3(v, i), V3{d.x / dt, d.y / dt, d.z / dt}));
  }
}

template <class T>
void cub_sort_pairs(Ctx& c, const T* kin, T* kout, const int32_t* vin, int32_t* vout, int64_t n, int bits) {
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, n, 0, bits, c.stream);
  WG_CUDA(cub::DeviceRadixSort::SortPairs(scratch(c, tmp), tmp, kin, kout, vin, vout, n, 0, bits, c.stream));
}

void cub_sort_keys(Ctx& c, const unsigned long long* kin, unsigned long long* kout, int64_t n) {
  size_t tmp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp, kin, kout, n, 0, 64, c.stream);
  WG_CUDA(cub::DeviceRadixSort::SortKeys(scratch(c, tmp), tmp, kin, kout, n, 0, 64, c.stream));
}

// exclusive scan of flag[0..n) into flag[0..n]; returns the total
int64_t scan_flags(Ctx& c, DBuf<int64_t>& flag, int64_t n) {
  WG_CUDA(cudaMemsetAsync(flag.data() + n, 0, sizeof(int64_t), c.stream));
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, flag.data(), flag.data(), n + 1, c.stream);
  WG_CUDA(cub::DeviceScan::ExclusiveSum(scratch(c, tmp), tmp, flag.data(), flag.data(), n + 1, c.stream));
  int64_t total = 0;
  WG_CUDA(cudaMemcpyAsync(&total, flag.data() + n, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
  WG_CUDA(cudaStreamSynchronize(c.stream));
  return total;
}

}  // namespace

// build_zones over m impacts (keys/vals on the device). Leaves the zone
// structure in the zn_* buffers; returns the zone count.
int32_t build_zones(Ctx& c, const unsigned long long* keys, const double* vals, int64_t m) {
  if (m >= (int64_t{1} << 31)) throw Error(WEFT_ERR_DIMENSION, "build_zones: more than 2^31 impacts");
  cudaStream_t s = c.stream;
  c.zn_part_v.resize(4 * m + 4);
  c.zn_part_w.resize(4 * m + 4);
  c.zn_owner.resize(static_cast<size_t>(c.soup_verts) + 1);
  c.zn_parent.resize(m + 1);
  c.zn_flag.resize(4 * m + 1);
  c.zn_zone_of.resize(m + 1);
  c.zn_zone_of_sorted.resize(m + 1);
  c.zn_iota.resize(m + 1);
  c.zn_zimp.resize(m + 1);
  c.zn_nz = 0;
  c.zn_nzv = 0;
  if (m == 0) return 0;
  WG_CUDA(cudaMemsetAsync(c.zn_owner.data(), 0x7f, sizeof(int32_t) * c.soup_verts, s));
  const int bs = 256;
  k_zone_parts<<<div_up(m, bs), bs, 0, ls(c)>>>(m, keys, vals, c.tris.data(), c.soup_edges.data(), c.zn_part_v.data(),
                                                c.zn_part_w.data(), c.zn_owner.data(), c.zn_parent.data());
  k_zone_union<<<div_up(m, bs), bs, 0, ls(c)>>>(m, c.zn_part_v.data(), c.zn_owner.data(), c.zn_parent.data());
  k_zone_roots<<<div_up(m, bs), bs, 0, ls(c)>>>(m, c.zn_parent.data(), c.zn_flag.data());
  const int32_t nz = static_cast<int32_t>(scan_flags(c, c.zn_flag, m));
  k_zone_of<<<div_up(m, bs), bs, 0, ls(c)>>>(m, c.zn_parent.data(), c.zn_flag.data(), c.zn_zone_of.data(),
                                             c.zn_iota.data());
  // impacts of each zone in ascending index: stable radix sort by zone id
  int bits = 1;
  while ((int64_t{1} << bits) <= nz) ++bits;
  cub_sort_pairs<int32_t>(c, c.zn_zone_of.data(), c.zn_zone_of_sorted.data(), c.zn_iota.data(), c.zn_zimp.data(), m,
                          bits);
  c.zn_zimp_off.resize(static_cast<size_t>(nz) + 1);
  k_zone_run_starts<<<div_up(m, bs), bs, 0, ls(c)>>>(m, c.zn_zone_of_sorted.data(), c.zn_zimp_off.data(), nz);
  // zone vertices: sorted unique movable (zone, vertex)
  const int64_t np = 4 * m;
  c.zn_vkeys.resize(np + 1);
  c.zn_vkeys_sorted.resize(np + 1);
  k_zone_vkeys<<<div_up(np, bs), bs, 0, ls(c)>>>(m, c.zn_part_v.data(), c.zn_zone_of.data(), c.soup_movable.data(),
                                                 c.zn_vkeys.data());
  cub_sort_keys(c, c.zn_vkeys.data(), c.zn_vkeys_sorted.data(), np);
  k_unique_u64_flags<<<div_up(np, bs), bs, 0, ls(c)>>>(np, c.zn_vkeys_sorted.data(), c.zn_flag.data());
  const int64_t nzv = scan_flags(c, c.zn_flag, np);
  if (nzv >= (int64_t{1} << 30)) throw Error(WEFT_ERR_DIMENSION, "build_zones: more than 2^30 zone vertices");
  k_compact_u64<<<div_up(np, bs), bs, 0, ls(c)>>>(np, c.zn_vkeys_sorted.data(), c.zn_flag.data(), c.zn_vkeys.data());
  c.zn_voff.resize(static_cast<size_t>(nz) + 1);
  k_zone_voff<<<div_up(nz + 1, bs), bs, 0, ls(c)>>>(nz, c.zn_vkeys.data(), nzv, c.zn_voff.data());
  // per zone vertex: its (constraint, participant) incidences in constraint order
  c.zn_ikeys.resize(np + 1);
  c.zn_ikeys_sorted.resize(np + 1);
  k_zone_ikeys<<<div_up(np, bs), bs, 0, ls(c)>>>(m, c.zn_zimp.data(), c.zn_zone_of_sorted.data(), c.zn_part_v.data(),
                                                 c.soup_movable.data(), c.zn_vkeys.data(), nzv, c.zn_ikeys.data());
  cub_sort_keys(c, c.zn_ikeys.data(), c.zn_ikeys_sorted.data(), np);
  c.zn_ioff.resize(static_cast<size_t>(nzv) + 1);
  k_zone_ioff<<<div_up(nzv + 1, bs), bs, 0, ls(c)>>>(nzv, c.zn_ikeys_sorted.data(), np, c.zn_ioff.data());
  WG_CUDA(cudaGetLastError());
  c.zn_nz = nz;
  c.zn_nzv = nzv;
  return nz;
}

// The last build: impact -> zone (m), zone vertex offsets (nz + 1), zone vertices (nzv).
void download_zones(Ctx& c, int64_t m, int32_t* impact_zone, int32_t* vert_off, int32_t* verts) {
  cudaStream_t s = c.stream;
  if (impact_zone && m) c.zn_zone_of.download(impact_zone, static_cast<size_t>(m), s);
  if (vert_off && c.zn_nz) c.zn_voff.download(vert_off, static_cast<size_t>(c.zn_nz) + 1, s);
  if (vert_off && !c.zn_nz) vert_off[0] = 0;
  if (verts && c.zn_nzv) {
    std::vector<unsigned long long> k(static_cast<size_t>(c.zn_nzv));
    c.zn_vkeys.download(k.data(), k.size(), s);
    WG_CUDA(cudaStreamSynchronize(s));
    for (size_t i = 0; i < k.size(); ++i) verts[i] = static_cast<int32_t>(k[i] & 0xFFFFFFFFull);
  }
  WG_CUDA(cudaStreamSynchronize(s));
}

// distribute_zones (response.cpp:164-182): zones in descending vertex count
// (stable) to the least-loaded device (lowest index on ties).
std::vector<std::vector<int>> distribute_zones(const std::vector<int>& sizes, int devices) {
  std::vector<int> order(sizes.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sizes[a] > sizes[b]; });
  std::vector<std::vector<int>> out(static_cast<size_t>(devices));
  std::vector<size_t> load(static_cast<size_t>(devices), 0);
  for (int z : order) {
    int best = 0;
    for (int d = 1; d < devices; ++d)
      if (load[d] < load[best]) best = d;
    out[best].push_back(z);
    load[best] += static_cast<size_t>(sizes[z]);
  }
  return out;
}

// resolve_zones (response.cpp:338-400) on the soup set with set_soup: CCD
// over x_begin -> x_cand (device, 3 * soup_verts), zones built and solved
// until no impacts remain. x_cand is updated in place. The first round's
// collide can be supplied by the caller (have_first: the current
// contact_keys/vals hold collide(CCD, x_begin, x_cand)).
void resolve_zones(Ctx& c, const double* xb, double* xcand, const double* mass, double thickness, double cell_scale,
                   const weft_zone_params& zp, weft_zone_report& rep, bool have_first) {
  // A rank group runs the zone solve replicated (every rank holds all
  // rows of x_begin / x_cand and, after the merged collide, all impacts):
  // identical zones, positions and failures on every rank.
  cudaStream_t s = c.stream;
  rep = weft_zone_report{};
  const int64_t nverts = c.soup_verts;
  c.zn_prop.resize(3 * static_cast<size_t>(nverts) + 3);
  c.zn_m = 0;
  auto collide_ccd = [&]() -> int64_t { return collide(c, xb, xcand, WEFT_CONTINUOUS, thickness, cell_scale); };
  const double max_move = zp.max_correction_factor * (zp.clearance < 1e-9 ? 1e-9 : zp.clearance);
  for (int outer = 0; outer < zp.outer_cap; ++outer) {
    const int64_t nf = (outer == 0 && have_first) ? c.n_contacts_found : collide_ccd();
    if (outer == 0) rep.first_round_impacts = nf;
    if (nf == 0) return;
    // accumulate the unseen feature pairs, in fresh (key) order
    const int64_t m0 = c.zn_m;
    c.zn_flag.resize(static_cast<size_t>(nf) + 1);
    k_zone_unseen<<<div_up(nf, 256), 256, 0, ls(c)>>>(nf, c.contact_keys.data(), m0, c.zn_acc_sorted.data(),
                                                      c.zn_flag.data());
    const int64_t add = scan_flags(c, c.zn_flag, nf);
    const int64_t m = m0 + add;
    if (static_cast<size_t>(m) + 1 > c.zn_acc_keys.cap) {  // grow, keeping the accumulated list
      DBuf<unsigned long long> k2;
      DBuf<double> v2;
      k2.resize(2 * static_cast<size_t>(m) + 1024);
      v2.resize(8 * (2 * static_cast<size_t>(m) + 1024));
      if (m0) {
        WG_CUDA(cudaMemcpyAsync(k2.data(), c.zn_acc_keys.data(), 8 * m0, cudaMemcpyDeviceToDevice, s));
        WG_CUDA(cudaMemcpyAsync(v2.data(), c.zn_acc_vals.data(), 64 * m0, cudaMemcpyDeviceToDevice, s));
      }
      std::swap(k2.ptr, c.zn_acc_keys.ptr);
      std::swap(k2.cap, c.zn_acc_keys.cap);
      std::swap(v2.ptr, c.zn_acc_vals.ptr);
      std::swap(v2.cap, c.zn_acc_vals.cap);
      WG_CUDA(cudaStreamSynchronize(s));
    }
    c.zn_acc_keys.n = static_cast<size_t>(m);
    k_zone_append<<<div_up(nf, 256), 256, 0, ls(c)>>>(nf, c.contact_keys.data(), c.contact_vals.data(),
                                                      c.zn_flag.data(), m0, c.zn_acc_keys.data(),
                                                      c.zn_acc_vals.data());
    c.zn_acc_sorted.resize(static_cast<size_t>(m) + 1);
    cub_sort_keys(c, c.zn_acc_keys.data(), c.zn_acc_sorted.data(), m);
    c.zn_m = m;

    rep.outer_iterations = outer + 1;
    rep.impacts_resolved += nf;
    const int32_t nz = build_zones(c, c.zn_acc_keys.data(), c.zn_acc_vals.data(), m);
    rep.zone_count += nz;
    std::vector<int32_t> voff(static_cast<size_t>(nz) + 1);
    c.zn_voff.download(voff.data(), voff.size(), s);
    // the proposal this round projects from; the live buffer then moves
    WG_CUDA(cudaMemcpyAsync(c.zn_prop.data(), xcand, 24 * nverts, cudaMemcpyDeviceToDevice, s));
    const int64_t nzv = c.zn_nzv;
    c.zn_cn.resize(3 * static_cast<size_t>(m));
    c.zn_lam.resize(static_cast<size_t>(m));
    c.zn_force.resize(static_cast<size_t>(m));
    c.zn_tc.resize(static_cast<size_t>(m));
    c.zn_tv.resize(static_cast<size_t>(nzv) + 1);
    c.zn_grad.resize(3 * static_cast<size_t>(nzv) + 3);
    c.zn_saved.resize(3 * static_cast<size_t>(nzv) + 3);
    c.zn_fail.resize(static_cast<size_t>(nz));
    c.zn_fail.zero(s);
    ZoneArgs a{nz,
               c.zn_zimp_off.data(),
               c.zn_zimp.data(),
               c.zn_acc_vals.data(),
               c.zn_part_v.data(),
               c.zn_part_w.data(),
               c.zn_voff.data(),
               c.zn_vkeys.data(),
               c.zn_ioff.data(),
               c.zn_ikeys_sorted.data(),
               mass,
               xb,
               c.zn_prop.data(),
               xcand,
               c.zn_cn.data(),
               c.zn_lam.data(),
               c.zn_force.data(),
               c.zn_tc.data(),
               c.zn_tv.data(),
               c.zn_grad.data(),
               c.zn_saved.data(),
               c.zn_fail.data(),
               zp.clearance,
               zp.initial_penalty,
               zp.inner_tolerance,
               max_move,
               zp.al_iterations,
               zp.inner_iterations,
               zp.retry_cap};
    k_solve_zones<<<div_up(static_cast<int64_t>(nz) * 32, 128), 128, 0, ls(c)>>>(a);
    WG_CUDA(cudaGetLastError());
    std::vector<int32_t> fail(static_cast<size_t>(nz));
    c.zn_fail.download(fail.data(), fail.size(), s);
    WG_CUDA(cudaStreamSynchronize(s));
    std::vector<int> sizes(static_cast<size_t>(nz));
    for (int32_t z = 0; z < nz; ++z) {
      sizes[z] = voff[z + 1] - voff[z];
      rep.max_zone_vertices = std::max<int32_t>(rep.max_zone_vertices, sizes[z]);
    }
    if (std::any_of(fail.begin(), fail.end(), [](int32_t f) { return f != 0; })) {
      // Engine::parallel rethrows the lowest failing device's error
      // (exec.cpp:96-98); a device stops at its first failing zone.
      const auto asg = distribute_zones(sizes, std::max(1, c.nparts));
      for (const auto& dz : asg)
        for (int z : dz)
          if (fail[z]) throw Error(WEFT_ERR_ZONE, "zone " + std::to_string(z) + ": inner solver diverged");
    }
    log_line(c, "event=zones outer=" + std::to_string(outer + 1) + " zones=" + std::to_string(nz) +
                    " fresh=" + std::to_string(nf) + " accumulated=" + std::to_string(m));  // response.cpp:383-388
  }
  // cap reached: the surviving zones name the failure (:384-399)
  const int64_t nr = collide_ccd();
  if (nr == 0) return;
  const int32_t nz = build_zones(c, c.contact_keys.data(), c.contact_vals.data(), nr);
  std::string msg = "impact zones unresolved after " + std::to_string(zp.outer_cap) + " outer iterations; zone ids:";
  for (int32_t z = 0; z < nz; ++z) msg += " " + std::to_string(z);
  throw Error(WEFT_ERR_ZONE, msg);
}

void zone_commit(Ctx& c, const double* corrected, const double* pre, double dt, double* v) {
  k_zone_commit<<<div_up(c.p, 256), 256, 0, ls(c)>>>(c.p, corrected, pre, dt, v);
  WG_CUDA(cudaGetLastError());
}

}  // namespace weft_gpu
