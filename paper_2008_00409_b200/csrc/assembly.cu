// assembly.cu — per-step dynamic assembly of A = M - (dt^2 + c dt) J (+ dt D)
// and rhs = dt f(x + dt v) into the sliced-ELL matrix.
//
// Reference: distribute_elements (proj/src/assembly.cpp:5-54) and the
// five-step fill_matrix (proj/include/weft/assembly.hpp:74-220).
//
// Design (B200):
//  * The static element list (triangles, hinges, vertices; physics.cpp:5-63)
//    fixes a static row incidence table (row -> (element, stencil slot) in
//    ascending element order) and a static sparsity pattern; both are built
//    once on the device by radix sort (CUB) when the elements are set.
//  * Every step, contact elements (appended after the static list, as in
//    step_system, physics.hpp:50-52) get their own incidence table and
//    (row, col) pattern, merged row by row with the static pattern into a
//    fresh sliced-ELL layout whose slots follow the SpMV accumulation order.
//  * Values: one thread per block row walks its incidences in ascending
//    element order, evaluates the element's row-a force and Jacobian blocks
//    (elements.cuh) and accumulates into per-thread shared-memory slot
//    accumulators — no atomics, the reference's per-slot summation order
//    (mass first, then ascending element instances) is kept exactly, so the
//    matrix is bitwise equal to the CPU reference and independent of the
//    partition count (test_assembly.cpp:263-280).
#include <cub/cub.cuh>

#include <type_traits>

#include <algorithm>
#include <cstring>
#include <vector>

#include "ctx.cuh"
#include "elements.cuh"

namespace weft_gpu {

void* scratch(Ctx& c, size_t bytes) {
  DBuf<unsigned char>& b = c.cur == c.side ? c.scratch_side : c.scratch;
  b.resize(bytes + 256);
  return b.data();
}

// ---------------------------------------------------------------------------
// vertices / elements upload
// ---------------------------------------------------------------------------
void set_vertices(Ctx& c, int p, const double* mass, const uint8_t* pinned) {
  if (p < 0) throw Error(WEFT_ERR_DIMENSION, "negative vertex count");
  if (p >= (1 << 28)) throw Error(WEFT_ERR_DIMENSION, "more than 2^28 vertices");
  if (p < c.nparts) throw Error(WEFT_ERR_DIMENSION, "fewer vertices than partitions");
  if (p != c.p) c.has_state = c.obstacles_set = false;  // the simulation state is sized by p
  c.p = p;
  set_rows(c, p);
  c.mass.upload(mass, static_cast<size_t>(p), c.stream);
  c.pinned.upload(pinned, static_cast<size_t>(p), c.stream);
  c.n_static = c.n_contacts = 0;
  c.static_pay = 0;
  c.inc_ptr.resize(0);
  c.spat_ptr.resize(0);
  c.has_matrix = false;
  c.has_rhs = false;
  WG_CUDA(cudaStreamSynchronize(c.stream));
}

// Per-element result slots of the two-phase SpdProjected fill: the rhs
// contribution dt*f_a of every stencil slot (3 doubles each) followed by the
// element state the slot pass regenerates Jacobian blocks from.
static int state_size(int kind) {
  switch (kind) {
    case WEFT_STRETCH:
      return 18;  // wu_hat, wv_hat, wu, wv, |wu|, |wv|, cu, cv, cs, ok, keep_u2, keep_v2
    case WEFT_BEND:
      return 12;  // dihedral gradient at x_cur
    case WEFT_SPRING:
      return 10;  // K (row-major) and the live flag
    case WEFT_CONTACT:
      return 1;   // active flag (gap < activation at x_cur)
    default:
      return 0;
  }
}

static int payload_size(int kind) {
  switch (kind) {
    case WEFT_STRETCH:
      return 10;
    case WEFT_BEND:
    case WEFT_SPRING:
      return 2;
    case WEFT_EXTERNAL:
      return 4;
    case WEFT_CONTACT:
      return 16;
    default:
      return -1;
  }
}

// Converts flat records into the device SoA (stencil, info, damping,
// payload pool) starting at element index `first` / payload offset `pay0`.
static void upload_elements(Ctx& c, int64_t count, const weft_element* elems, int64_t first, int64_t pay0,
                            int64_t* pay_used, int64_t res0, int64_t* res_used) {
  std::vector<weft_element> host;
  const weft_element* h = elems;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, elems) == cudaSuccess && attr.type == cudaMemoryTypeDevice) {
    host.resize(static_cast<size_t>(count));
    WG_CUDA(cudaMemcpy(host.data(), elems, sizeof(weft_element) * count, cudaMemcpyDeviceToHost));
    h = host.data();
  }
  cudaGetLastError();
  std::vector<int4> st(static_cast<size_t>(count));
  std::vector<int2> info(static_cast<size_t>(count));
  std::vector<double> damp(static_cast<size_t>(count));
  std::vector<double> pay;
  pay.reserve(static_cast<size_t>(count) * 4);
  std::vector<int32_t> roff(static_cast<size_t>(count));
  int64_t rcur = res0;
  for (int64_t i = 0; i < count; ++i) {
    const weft_element& e = h[i];
    const int ps = payload_size(e.kind);
    if (ps < 0) throw Error(WEFT_ERR_INVALID, "element " + std::to_string(first + i) + ": unknown kind");
    if (e.stencil_size < 1 || e.stencil_size > 4)
      throw Error(WEFT_ERR_INVALID, "element " + std::to_string(first + i) + ": bad stencil size");
    int s[4] = {-1, -1, -1, -1};
    for (int a = 0; a < e.stencil_size; ++a) {
      const int v = e.stencil[a];
      if (v < 0 || v >= c.p)  // distribute_elements (assembly.cpp:18-22)
        throw Error(WEFT_ERR_DIMENSION, "element " + std::to_string(first + i) + ": stencil vertex " +
                                            std::to_string(v) + " outside all partitions");
      s[a] = v;
    }
    st[static_cast<size_t>(i)] = make_int4(s[0], s[1], s[2], s[3]);
    const int64_t off = pay0 + static_cast<int64_t>(pay.size());
    if (off > INT32_MAX) throw Error(WEFT_ERR_DIMENSION, "element payload exceeds 2^31 doubles");
    info[static_cast<size_t>(i)] = make_int2(e.kind | (e.stencil_size << 8), static_cast<int>(off));
    damp[static_cast<size_t>(i)] = e.damping;
    pay.insert(pay.end(), e.data, e.data + ps);
    if (rcur > INT32_MAX) throw Error(WEFT_ERR_DIMENSION, "element results exceed 2^31 doubles");
    roff[static_cast<size_t>(i)] = static_cast<int32_t>(rcur);
    rcur += 3 * e.stencil_size + state_size(e.kind);
  }
  const size_t n_total = static_cast<size_t>(first + count);
  const size_t pay_total = static_cast<size_t>(pay0) + pay.size();
  // grow while preserving the static prefix
  auto grow = [&](auto& buf, size_t need, size_t keep) {
    using T = std::remove_reference_t<decltype(*buf.data())>;
    if (need > buf.cap) {
      DBuf<T> tmp;
      tmp.resize(need);
      if (keep) WG_CUDA(cudaMemcpyAsync(tmp.data(), buf.data(), keep * sizeof(T), cudaMemcpyDeviceToDevice, c.stream));
      std::swap(tmp.ptr, buf.ptr);
      std::swap(tmp.cap, buf.cap);
    }
    buf.n = need;
  };
  grow(c.est, n_total, static_cast<size_t>(first));
  grow(c.einfo, n_total, static_cast<size_t>(first));
  grow(c.edamp, n_total, static_cast<size_t>(first));
  grow(c.epay, pay_total, static_cast<size_t>(pay0));
  grow(c.eres_off, n_total, static_cast<size_t>(first));
  c.eres.resize(static_cast<size_t>(rcur) + 1);
  if (count) {
    WG_CUDA(cudaMemcpyAsync(c.est.data() + first, st.data(), sizeof(int4) * count, cudaMemcpyHostToDevice, c.stream));
    WG_CUDA(cudaMemcpyAsync(c.einfo.data() + first, info.data(), sizeof(int2) * count, cudaMemcpyHostToDevice, c.stream));
    WG_CUDA(cudaMemcpyAsync(c.edamp.data() + first, damp.data(), sizeof(double) * count, cudaMemcpyHostToDevice, c.stream));
  }
  if (!pay.empty())
    WG_CUDA(cudaMemcpyAsync(c.epay.data() + pay0, pay.data(), sizeof(double) * pay.size(), cudaMemcpyHostToDevice,
                            c.stream));
  if (count)
    WG_CUDA(cudaMemcpyAsync(c.eres_off.data() + first, roff.data(), sizeof(int32_t) * count, cudaMemcpyHostToDevice,
                            c.stream));
  *res_used = rcur - res0;
  WG_CUDA(cudaStreamSynchronize(c.stream));  // host staging vectors die here
  *pay_used = static_cast<int64_t>(pay.size());
}

// ---------------------------------------------------------------------------
// incidence tables: rows -> (element*4 + a), ascending element
// ---------------------------------------------------------------------------
__global__ void k_inc_emit(int64_t first, int64_t count, const int4* __restrict__ est, const int2* __restrict__ einfo,
                           const uint8_t* __restrict__ pinned, uint32_t* __restrict__ keys, int32_t* __restrict__ vals,
                           int* __restrict__ cnt, int64_t code_base) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int4 s = est[first + i];
  const int ss = (einfo[first + i].x >> 8) & 0xff;
  const int sv[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    uint32_t key = 0xffffffffu;
    if (a < ss && !pinned[sv[a]]) {
      key = static_cast<uint32_t>(sv[a]);
      atomicAdd(cnt + sv[a], 1);
    }
    keys[4 * i + a] = key;
    vals[4 * i + a] = static_cast<int32_t>((code_base + i) * 4 + a);
  }
}

static int bits_for(int64_t v) {
  int b = 1;
  while ((int64_t(1) << b) <= v) ++b;
  return b;
}

// Builds (ptr, list) for elements [first, first+count); codes are
// (code_base + i) * 4 + a.
static void build_incidence(Ctx& c, int64_t first, int64_t count, int64_t code_base, DBuf<int64_t>& ptr,
                            DBuf<int32_t>& list) {
  const int p = c.p;
  cudaStream_t s = c.stream;
  DBuf<int>& cnt = c.sc_inc_cnt;
  cnt.resize(static_cast<size_t>(p) + 1);
  cnt.zero(s);
  ptr.resize(static_cast<size_t>(p) + 1);
  const int64_t m = 4 * count;
  DBuf<uint32_t>& k1 = c.sc_inc_k1;
  DBuf<uint32_t>& k2 = c.sc_inc_k2;
  DBuf<int32_t>& v1 = c.sc_inc_v1;
  k1.resize(static_cast<size_t>(m) + 1);
  k2.resize(static_cast<size_t>(m) + 1);
  v1.resize(static_cast<size_t>(m) + 1);
  list.resize(static_cast<size_t>(m) + 1);
  if (count) {
    if ((code_base + count) * 4 > INT32_MAX) throw Error(WEFT_ERR_DIMENSION, "too many elements (> 2^29)");
    k_inc_emit<<<div_up(count, 256), 256, 0, ls(c)>>>(first, count, c.est.data(), c.einfo.data(), c.pinned.data(),
                                                  k1.data(), v1.data(), cnt.data(), code_base);
    WG_CUDA(cudaGetLastError());
    size_t tmp = 0;
    const int end_bit = 32;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, k1.data(), k2.data(), v1.data(), list.data(), (int)m, 0, end_bit, s);
    void* t = scratch(c, tmp);
    WG_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, k1.data(), k2.data(), v1.data(), list.data(), (int)m, 0,
                                            end_bit, s));
  }
  // exclusive scan of counts -> ptr (int64)
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.data(), ptr.data(), p + 1, s);
  void* t = scratch(c, tmp);
  WG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, cnt.data(), ptr.data(), p + 1, s));
  WG_CUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
// sparsity: sorted unique (row << 32 | col) keys -> CSR
// ---------------------------------------------------------------------------
__global__ void k_pair_count(int64_t first, int64_t count, const int4* __restrict__ est,
                             const int2* __restrict__ einfo, const uint8_t* __restrict__ pinned,
                             int64_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int4 s = est[first + i];
  const int ss = (einfo[first + i].x >> 8) & 0xff;
  const int sv[4] = {s.x, s.y, s.z, s.w};
  int live = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a) live += (a < ss && !pinned[sv[a]]) ? 1 : 0;
  out[i] = live * live;
}

__global__ void k_pair_emit(int64_t first, int64_t count, const int4* __restrict__ est,
                            const int2* __restrict__ einfo, const uint8_t* __restrict__ pinned,
                            const int64_t* __restrict__ off, uint64_t* __restrict__ keys) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int4 s = est[first + i];
  const int ss = (einfo[first + i].x >> 8) & 0xff;
  const int sv[4] = {s.x, s.y, s.z, s.w};
  int64_t o = off[i];
  for (int a = 0; a < ss; ++a) {
    if (pinned[sv[a]]) continue;
    for (int b = 0; b < ss; ++b) {
      if (pinned[sv[b]]) continue;
      keys[o++] = (static_cast<uint64_t>(sv[a]) << 32) | static_cast<uint32_t>(sv[b]);
    }
  }
}

__global__ void k_diag_keys(int p, uint64_t* __restrict__ keys) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < p) keys[r] = (static_cast<uint64_t>(r) << 32) | static_cast<uint32_t>(r);
}

__global__ void k_key_rows(int64_t n, const uint64_t* __restrict__ keys, int* __restrict__ cnt,
                           int32_t* __restrict__ cols) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  atomicAdd(cnt + (k >> 32), 1);
  cols[i] = static_cast<int32_t>(k & 0xffffffffu);
}

// (row, col) pattern of elements [first, first+count) (+ the diagonal of
// every row when with_diag), steps (1)-(3) of fill_matrix
// (assembly.hpp:93-134), as CSR with ascending unique columns.
static void build_pattern(Ctx& c, int64_t first, int64_t count, bool with_diag, DBuf<int64_t>& ptr,
                          DBuf<int32_t>& cols) {
  const int p = c.p;
  cudaStream_t s = c.stream;
  DBuf<int64_t>& pc = c.sc_pat_pc;
  pc.resize(static_cast<size_t>(count) + 1);
  int64_t npairs = 0;
  if (count) {
    k_pair_count<<<div_up(count, 256), 256, 0, ls(c)>>>(first, count, c.est.data(), c.einfo.data(), c.pinned.data(),
                                                    pc.data());
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, pc.data(), pc.data(), count + 1, s);
    void* t = scratch(c, tmp);
    // last element of an exclusive scan over count+1 entries = total
    WG_CUDA(cudaMemsetAsync(pc.data() + count, 0, sizeof(int64_t), s));
    WG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, pc.data(), pc.data(), count + 1, s));
    WG_CUDA(cudaMemcpyAsync(&npairs, pc.data() + count, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
  }
  const int64_t nk = npairs + (with_diag ? p : 0);
  DBuf<uint64_t>& k1 = c.sc_pat_k1;
  DBuf<uint64_t>& k2 = c.sc_pat_k2;
  k1.resize(static_cast<size_t>(nk) + 1);
  k2.resize(static_cast<size_t>(nk) + 1);
  if (count)
    k_pair_emit<<<div_up(count, 256), 256, 0, ls(c)>>>(first, count, c.est.data(), c.einfo.data(), c.pinned.data(),
                                                   pc.data(), k1.data());
  if (with_diag && p) k_diag_keys<<<div_up(p, 256), 256, 0, ls(c)>>>(p, k1.data() + npairs);
  WG_CUDA(cudaGetLastError());
  const int end_bit = 32 + bits_for(p);
  DBuf<int64_t>& nsel = c.sc_pat_nsel;
  nsel.resize(1);
  int64_t nu = 0;
  if (nk) {
    size_t tmp = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmp, k1.data(), k2.data(), nk, 0, end_bit, s);
    size_t tmp2 = 0;
    cub::DeviceSelect::Unique(nullptr, tmp2, k2.data(), k1.data(), nsel.data(), nk, s);
    void* t = scratch(c, std::max(tmp, tmp2));
    WG_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, k1.data(), k2.data(), nk, 0, end_bit, s));
    WG_CUDA(cub::DeviceSelect::Unique(t, tmp2, k2.data(), k1.data(), nsel.data(), nk, s));
    WG_CUDA(cudaMemcpyAsync(&nu, nsel.data(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
  }
  DBuf<int>& cnt = c.sc_pat_cnt;
  cnt.resize(static_cast<size_t>(p) + 1);
  cnt.zero(s);
  cols.resize(static_cast<size_t>(nu) + 1);
  ptr.resize(static_cast<size_t>(p) + 1);
  if (nu) k_key_rows<<<div_up(nu, 256), 256, 0, ls(c)>>>(nu, k1.data(), cnt.data(), cols.data());
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.data(), ptr.data(), p + 1, s);
  void* t = scratch(c, tmp);
  WG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, cnt.data(), ptr.data(), p + 1, s));
  WG_CUDA(cudaStreamSynchronize(s));
}

void set_elements(Ctx& c, int64_t count, const weft_element* elems) {
  if (c.p == 0 && count) throw Error(WEFT_ERR_INVALID, "set_elements: set_vertices first");
  int64_t used = 0;
  int64_t rused = 0;
  upload_elements(c, count, elems, 0, 0, &used, 0, &rused);
  c.n_static = count;
  c.static_pay = used;
  // same-kind runs of the static list (k_elem_eval is compiled per kind)
  c.kind_runs.clear();
  {
    std::vector<weft_element> host;
    const weft_element* h = elems;
    cudaPointerAttributes attr{};
    if (count && cudaPointerGetAttributes(&attr, elems) == cudaSuccess && attr.type == cudaMemoryTypeDevice) {
      host.resize(static_cast<size_t>(count));
      WG_CUDA(cudaMemcpy(host.data(), elems, sizeof(weft_element) * count, cudaMemcpyDeviceToHost));
      h = host.data();
    }
    cudaGetLastError();
    for (int64_t i = 0; i < count;) {
      int64_t j = i + 1;
      while (j < count && h[j].kind == h[i].kind) ++j;
      c.kind_runs.push_back(Ctx::KindRun{h[i].kind, i, j});
      i = j;
    }
    if (c.kind_runs.size() > 16) c.kind_runs.clear();  // unsorted list: one generic launch
  }
  c.static_res = rused;
  c.n_contacts = 0;
  build_incidence(c, 0, count, 0, c.inc_ptr, c.inc);
  build_pattern(c, 0, count, true, c.spat_ptr, c.spat);
  c.cinc_ptr.resize(static_cast<size_t>(c.p) + 1);
  c.cinc_ptr.zero(c.stream);
  c.have_pattern_for_contacts = false;
  c.has_matrix = false;
  WG_CUDA(cudaStreamSynchronize(c.stream));
}

void set_contacts(Ctx& c, int64_t count, const weft_element* elems) {
  if (c.p == 0) throw Error(WEFT_ERR_INVALID, "set_contacts: set_vertices first");
  int64_t used = 0;
  int64_t rused = 0;
  upload_elements(c, count, elems, c.n_static, c.static_pay, &used, c.static_res, &rused);
  c.n_contacts = count;
  // contact incidences: codes are the contact index (element n_static + i).
  build_incidence(c, c.n_static, count, 0, c.cinc_ptr, c.cinc);
  c.have_pattern_for_contacts = false;
}

// Device-generated contacts (proximities_to_elements on the GPU, narrow.cu):
// room for `count` contact elements after the static list — 16 payload
// doubles and 13 result doubles (3 * 4 rhs + 1 state) each — keeping the
// static prefix. The caller's kernel fills the records.
void reserve_contacts(Ctx& c, int64_t count) {
  auto grow = [&](auto& buf, size_t need, size_t keep) {
    using T = std::remove_reference_t<decltype(*buf.data())>;
    if (need > buf.cap) {
      DBuf<T> tmp;
      tmp.resize(need);
      if (keep) WG_CUDA(cudaMemcpyAsync(tmp.data(), buf.data(), keep * sizeof(T), cudaMemcpyDeviceToDevice, c.stream));
      std::swap(tmp.ptr, buf.ptr);
      std::swap(tmp.cap, buf.cap);
    }
    buf.n = need;
  };
  const size_t n_total = static_cast<size_t>(c.n_static + count);
  grow(c.est, n_total + 1, static_cast<size_t>(c.n_static));
  grow(c.einfo, n_total + 1, static_cast<size_t>(c.n_static));
  grow(c.edamp, n_total + 1, static_cast<size_t>(c.n_static));
  grow(c.eres_off, n_total + 1, static_cast<size_t>(c.n_static));
  grow(c.epay, static_cast<size_t>(c.static_pay + kContactPay * count) + 1, static_cast<size_t>(c.static_pay));
  c.eres.resize(static_cast<size_t>(c.static_res + kContactRes * count) + 1);
  WG_CUDA(cudaStreamSynchronize(c.stream));
}

void finish_contacts(Ctx& c, int64_t count) {
  c.n_contacts = count;
  build_incidence(c, c.n_static, count, 0, c.cinc_ptr, c.cinc);
  c.have_pattern_for_contacts = false;
}

// ---------------------------------------------------------------------------
// merged pattern -> sliced-ELL layout in accumulation-group order
// ---------------------------------------------------------------------------
struct MergeIn {
  const int64_t* sptr;
  const int32_t* scol;
  const int64_t* cptr;  // may be null (no contacts)
  const int32_t* ccol;
};

// Walks the union of the static and contact columns of row r in ascending
// order (both inputs sorted, each unique).
template <class F>
__device__ __forceinline__ void for_union(const MergeIn& m, int r, F&& f) {
  int64_t i = m.sptr[r], ie = m.sptr[r + 1];
  int64_t j = 0, je = 0;
  if (m.cptr) {
    j = m.cptr[r];
    je = m.cptr[r + 1];
  }
  while (i < ie || j < je) {
    int col;
    if (j >= je || (i < ie && m.scol[i] <= m.ccol[j])) {
      col = m.scol[i];
      if (j < je && m.ccol[j] == col) ++j;
      ++i;
    } else {
      col = m.ccol[j];
      ++j;
    }
    f(col);
  }
}

__global__ void k_merge_len(int row0, int nloc, MergeIn m, int32_t* __restrict__ len) {
  const int lr = blockIdx.x * blockDim.x + threadIdx.x;
  if (lr >= nloc) return;
  int n = 0;
  for_union(m, row0 + lr, [&](int) { ++n; });
  len[lr] = n;
}

__global__ void k_slice_width(int p, int nslices, const int32_t* __restrict__ len, int64_t* __restrict__ w) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslices) return;
  int m = 0;
  for (int r = s * kSlice; r < min(p, (s + 1) * kSlice); ++r) m = max(m, len[r]);
  w[s] = static_cast<int64_t>(m) * kSlice;
}

// Writes the row's columns grouped by accumulation order: own partition
// first, then the work-queue order (sparse.hpp:89-95); ascending inside a
// group. Padding slots get -1.
__global__ void k_merge_fill(int row0, int nloc, MergeIn m, PartMap pm, GroupOrder go,
                             const int64_t* __restrict__ soff, const int32_t* __restrict__ pos,
                             int32_t* __restrict__ cols) {
  const int lr = blockIdx.x * blockDim.x + threadIdx.x;
  if (lr >= nloc) return;
  const int r = row0 + lr;
  const int mp = pos[lr];  // matrix position of the row (SELL-32-sigma)
  const int s = mp >> 5;
  const int64_t base = soff[s] + (mp & 31);
  const int width = static_cast<int>((soff[s + 1] - soff[s]) / kSlice);
  const int d = pm.owner(r);
  int k = 0;
  for (int g = 0; g < go.n; ++g) {
    for_union(m, r, [&](int col) {
      const int o = pm.owner(col);
      if (go.qpos[d][o] == g) {
        cols[base + (int64_t)k * kSlice] = col | (g << kGroupShift);
        ++k;
      }
    });
  }
  for (; k < width; ++k) cols[base + (int64_t)k * kSlice] = -1;
}

// Pattern of the contact elements (rows/cols among non-pinned vertices).
static void build_layout(Ctx& c) {
  cudaStream_t s = c.stream;
  DBuf<int64_t>& cptr = c.sc_lay_cptr;
  DBuf<int32_t>& ccol = c.sc_lay_ccol;
  MergeIn m{c.spat_ptr.data(), c.spat.data(), nullptr, nullptr};
  if (c.n_contacts) {
    build_pattern(c, c.n_static, c.n_contacts, false, cptr, ccol);
    m.cptr = cptr.data();
    m.ccol = ccol.data();
  }
  SellMatrix& A = c.A;
  const int nloc = c.row1 - c.row0;  // this rank's rows (all rows when world == 1)
  A.rows = nloc;
  A.row0 = c.row0;
  A.nslices = div_up(nloc, kSlice);
  A.slice_off.resize(static_cast<size_t>(A.nslices) + 1);
  DBuf<int32_t>& len_row = c.sc_lay_len;
  len_row.resize(static_cast<size_t>(nloc) + 1);
  if (nloc) k_merge_len<<<div_up(nloc, 256), 256, 0, ls(c)>>>(c.row0, nloc, m, len_row.data());
  build_sigma(c, len_row.data());  // A.perm / A.pos / A.rowlen (by position)
  ++A.layout_id;
  if (nloc)
    k_slice_width<<<div_up(A.nslices, 256), 256, 0, ls(c)>>>(nloc, A.nslices, A.rowlen.data(), A.slice_off.data());
  WG_CUDA(cudaMemsetAsync(A.slice_off.data() + A.nslices, 0, sizeof(int64_t), s));
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, A.slice_off.data(), A.slice_off.data(), A.nslices + 1, s);
  void* t = scratch(c, tmp);
  WG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, A.slice_off.data(), A.slice_off.data(), A.nslices + 1, s));
  // totals: slots, nnzb, max row length
  int64_t total = 0;
  WG_CUDA(cudaMemcpyAsync(&total, A.slice_off.data() + A.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DBuf<int64_t>& red = c.sc_lay_red;
  red.resize(2);
  int* lenp = A.rowlen.data();
  size_t t1 = 0, t2 = 0;
  cub::DeviceReduce::Sum(nullptr, t1, lenp, red.data(), nloc, s);
  cub::DeviceReduce::Max(nullptr, t2, lenp, reinterpret_cast<int*>(red.data() + 1), nloc, s);
  t = scratch(c, std::max(t1, t2));
  int64_t hr[2] = {0, 0};
  if (nloc) {
    WG_CUDA(cub::DeviceReduce::Sum(t, t1, lenp, red.data(), nloc, s));
    WG_CUDA(cudaMemsetAsync(red.data() + 1, 0, sizeof(int64_t), s));
    WG_CUDA(cub::DeviceReduce::Max(t, t2, lenp, reinterpret_cast<int*>(red.data() + 1), nloc, s));
    WG_CUDA(cudaMemcpyAsync(hr, red.data(), sizeof(hr), cudaMemcpyDeviceToHost, s));
  }
  WG_CUDA(cudaStreamSynchronize(s));
  A.total = total;
  A.nnzb = hr[0];
  A.max_len = static_cast<int>(hr[1] & 0xffffffff);
  A.cols.resize(static_cast<size_t>(total) + 1);
  A.vals.resize(9 * static_cast<size_t>(total) + 9);
  if (nloc)
    k_merge_fill<<<div_up(nloc, 256), 256, 0, ls(c)>>>(c.row0, nloc, m, c.pm, c.go, A.slice_off.data(), A.pos.data(),
                                                      A.cols.data());
  WG_CUDA(cudaGetLastError());
  WG_CUDA(cudaStreamSynchronize(s));  // cptr/ccol die here
}

// ---------------------------------------------------------------------------
// value fill
// ---------------------------------------------------------------------------
constexpr int kFillThreadsConst = 64;

struct FillArgs {
  int p;     // held rows (threads walk matrix positions; row = row0 + perm[m])
  int row0;
  const int32_t* __restrict__ perm;
  int64_t n_static;
  double dt;
  bool exact;
  int wcap;  // slots held in shared memory per thread
  const int64_t* __restrict__ slice_off;
  const int32_t* __restrict__ rowlen;
  const int32_t* __restrict__ cols;
  double* __restrict__ vals;
  int64_t total;
  double* __restrict__ rhs;
  float* __restrict__ vals32;  // Precision::Single outputs (T = float)
  float* __restrict__ rhs32;
  const double* __restrict__ mass;
  const uint8_t* __restrict__ pinned;
  const int64_t* __restrict__ inc_ptr;
  const int32_t* __restrict__ inc;
  const int64_t* __restrict__ cinc_ptr;
  const int32_t* __restrict__ cinc;
  const int4* __restrict__ est;
  const int2* __restrict__ einfo;
  const double* __restrict__ edamp;
  const double* __restrict__ epay;
  const double* __restrict__ xc;
  const double* __restrict__ xa;
  const double* __restrict__ vel;
  int* __restrict__ bad_mass;  // min vertex id with non-positive mass
};

// Accumulator access: shared (Wide = false) or the output planes directly.
// T = float: Precision::Single — each contribution cast to float and added
// in float (BellMatrix<float>::add_value, assembly.hpp:212).
template <bool Wide, class T = double>
struct Acc {
  T* sm;   // [wcap][9][blockDim] for this block
  int tid, bs;
  T* gv;   // output planes (Wide)
  int64_t total, base;
  __device__ __forceinline__ T& at(int slot, int q) {
    if (Wide) return gv[vidx(base + (int64_t)slot * kSlice, tid & 31, q)];
    return sm[(slot * 9 + q) * bs + tid];
  }
};

template <bool Wide, bool Exact, class T = double>
__global__ void __launch_bounds__(64) k_fill(FillArgs f) {
  extern __shared__ double smem_d[];
  T* smem = reinterpret_cast<T*>(smem_d);
  T* const vals = std::is_same_v<T, float> ? reinterpret_cast<T*>(f.vals32) : reinterpret_cast<T*>(f.vals);
  T* const rhs = std::is_same_v<T, float> ? reinterpret_cast<T*>(f.rhs32) : reinterpret_cast<T*>(f.rhs);
  const int lr = blockIdx.x * blockDim.x + threadIdx.x;  // matrix position
  const int len = lr < f.p ? f.rowlen[lr] : 0;
  const bool mine = lr < f.p && (Wide ? len > f.wcap : len <= f.wcap);
  if (!mine) return;
  const int r = f.row0 + f.perm[lr];
  const int64_t base = f.slice_off[lr >> 5] + (lr & 31);
  int32_t* colbuf = reinterpret_cast<int32_t*>(smem + (size_t)f.wcap * 9 * blockDim.x);
  Acc<Wide, T> acc{smem, (int)threadIdx.x, (int)blockDim.x, vals, f.total, base};
  static_assert(kFillThreadsConst % 32 == 0, "row lanes must match threadIdx.x % 32");
  auto col_of = [&](int k) -> int {
    if (!Wide) return colbuf[k * blockDim.x + threadIdx.x];
    return f.cols[base + (int64_t)k * kSlice] & kColMask;
  };
  for (int k = 0; k < len; ++k) {
    if (!Wide) colbuf[k * blockDim.x + threadIdx.x] = f.cols[base + (int64_t)k * kSlice] & kColMask;
#pragma unroll
    for (int q = 0; q < 9; ++q) acc.at(k, q) = 0;
  }
  auto find = [&](int col) -> int {
    for (int k = 0; k < len; ++k)
      if (col_of(k) == col) return k;
    return -1;
  };
  // (5) mass diagonal first (assembly.hpp:155-166)
  const bool pin = f.pinned[r] != 0;
  const double m = f.mass[r];
  if (!pin && m <= 0.0) atomicMin(f.bad_mass, r);
  {
    const int ds = find(r);
    const T mv = pin ? T(1) : static_cast<T>(m);
    acc.at(ds, 0) = acc.at(ds, 0) + mv;
    acc.at(ds, 4) = acc.at(ds, 4) + mv;
    acc.at(ds, 8) = acc.at(ds, 8) + mv;
  }
  T r0 = 0, r1 = 0, r2 = 0;
  const double dt = f.dt;
  // then every element instance of this row in ascending element order
  for (int pass = 0; pass < 2; ++pass) {
    const int64_t* ip = pass == 0 ? f.inc_ptr : f.cinc_ptr;
    const int32_t* il = pass == 0 ? f.inc : f.cinc;
    const int64_t i0 = ip[r], i1 = ip[r + 1];
    for (int64_t ii = i0; ii < i1; ++ii) {
      const int code = il[ii];
      const int64_t e = (pass == 0 ? 0 : f.n_static) + (code >> 2);
      const int a = code & 3;
      const int4 s4 = f.est[e];
      const int2 info = f.einfo[e];
      const int kind = info.x & 0xff, ss = (info.x >> 8) & 0xff;
      const double damping = f.edamp[e];
      const int st[4] = {s4.x, s4.y, s4.z, s4.w};
      const double scale = dt * dt + damping * dt;
      const double nscale = -scale;
      double fv[3];
      double mv[4][3];  // J_ab v_b per stencil slot, for the damping term
      eval_row<Exact>(kind, ss, st, f.epay + info.y, a, f.xc, f.xa, f.vel, fv,
               [&](int b, const double* J, const double* D, bool add) {
                 if (damping > 0.0) {
                   const V3 vb = ld3(f.vel, st[b]);
                   mv[b][0] = (J[0] * vb.x + J[1] * vb.y) + J[2] * vb.z;
                   mv[b][1] = (J[3] * vb.x + J[4] * vb.y) + J[5] * vb.z;
                   mv[b][2] = (J[6] * vb.x + J[7] * vb.y) + J[8] * vb.z;
                 }
                 const int col = st[b];
                 if (!add || f.pinned[col]) return;
                 const int slot = find(col);
#pragma unroll
                 for (int q = 0; q < 9; ++q) {
                   double cv = nscale * J[q];
                   if (D) cv = cv + dt * D[q];
                   acc.at(slot, q) = acc.at(slot, q) + static_cast<T>(cv);
                 }
               });
      // rhs (assembly.hpp:185-197): f = force + friction, then the damping
      // products in ascending b, then rhs += dt f.
      double fx = fv[0], fy = fv[1], fz = fv[2];
      if (damping > 0.0) {
        for (int b = 0; b < ss; ++b) {
          fx = fx + damping * mv[b][0];
          fy = fy + damping * mv[b][1];
          fz = fz + damping * mv[b][2];
        }
      }
      r0 = r0 + static_cast<T>(dt * fx);
      r1 = r1 + static_cast<T>(dt * fy);
      r2 = r2 + static_cast<T>(dt * fz);
    }
  }
  rhs[3 * r] = r0;
  rhs[3 * r + 1] = r1;
  rhs[3 * r + 2] = r2;
  if (!Wide) {
    for (int k = 0; k < len; ++k)
#pragma unroll
      for (int q = 0; q < 9; ++q) vals[vidx(base + (int64_t)k * kSlice, lr & 31, q)] = acc.at(k, q);
  }
}

// Padding slots must hold zeros (they are never read by the SpMV, which
// stops at rowlen, but downloads and ncu byte counts stay honest).
template <class T>
__global__ void k_zero_padding(int p, const int64_t* __restrict__ soff, const int32_t* __restrict__ rowlen,
                               T* __restrict__ vals, int64_t total) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= p) return;
  const int s = r >> 5;
  const int width = static_cast<int>((soff[s + 1] - soff[s]) / kSlice);
  const int64_t base = soff[s] + (r & 31);
  for (int k = rowlen[r]; k < width; ++k)
#pragma unroll
    for (int q = 0; q < 9; ++q) vals[vidx(base + (int64_t)k * kSlice, r & 31, q)] = 0;
}

// ---------------------------------------------------------------------------
// Two-phase SpdProjected fill
// ---------------------------------------------------------------------------
// Phase 1, one thread per ELEMENT (no replication): element_force at x_adv,
// friction, all Jacobian blocks at x_cur (for the damping term), and the
// per-stencil-slot rhs contribution dt * f_a, exactly as fill_matrix's
// instance loop computes them (assembly.hpp:170-197); plus a compact state
// from which any block J_ab is regenerated bit-identically.
// Phase 2, one thread per matrix SLOT (row, column): mass first, then every
// incidence of the row in ascending element order that couples to this
// column adds (-scale) J_ab (+ dt D_ab) into register accumulators
// (assembly.hpp:199-215) — no atomics, no shared-memory accumulators, full
// occupancy; the same kernel sums each row's rhs contributions in that order.

// stretch block (i, j) from the stored x_cur state (elements.cpp:209-228,
// keep_s2 = false in SpdProjected mode).
__device__ __forceinline__ void stretch_block_state(const double* __restrict__ S, const double* __restrict__ d,
                                                    int i, int j, double J[9]) {
  if (S[15] == 0.0) {
#pragma unroll
    for (int q = 0; q < 9; ++q) J[q] = 0.0;
    return;
  }
  const V3 wu_hat = v3(S[0], S[1], S[2]), wv_hat = v3(S[3], S[4], S[5]);
  const V3 wu = v3(S[6], S[7], S[8]), wv = v3(S[9], S[10], S[11]);
  const double wu_len = S[12], wv_len = S[13];
  const double a = d[6];
  const double ui = d[i], vi = d[3 + i], uj = d[j], vj = d[3 + j];
  const V3 gui = scl(a * ui, wu_hat), gvi = scl(a * vi, wv_hat);
  const V3 gsi = scl(a, add(scl(ui, wv), scl(vi, wu)));
  const V3 guj = scl(a * uj, wu_hat), gvj = scl(a * vj, wv_hat);
  const V3 gsj = scl(a, add(scl(uj, wv), scl(vj, wu)));
  const double su2 = (d[7] * S[16]) * (((a * ui) * uj) / wu_len);
  const double sv2 = (d[8] * S[17]) * (((a * vi) * vj) / wv_len);
  const bool keep_u2 = S[16] >= 0.0, keep_v2 = S[17] >= 0.0;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double id = r == c ? 1.0 : 0.0;
      double m = 0.0;
      m = m - d[7] * (comp(gui, r) * comp(guj, c));
      m = m - d[8] * (comp(gvi, r) * comp(gvj, c));
      m = m - d[9] * (comp(gsi, r) * comp(gsj, c));
      if (keep_u2) m = m - su2 * (id - comp(wu_hat, r) * comp(wu_hat, c));
      if (keep_v2) m = m - sv2 * (id - comp(wv_hat, r) * comp(wv_hat, c));
      J[r * 3 + c] = 0.0 + m;
    }
}

// Block J_ab (and D_ab) of an element from its phase-1 state. Returns
// whether D is present (velocity damping).
__device__ __forceinline__ bool elem_block(int kind, const double* __restrict__ S, const double* __restrict__ d,
                                           int a, int b, double J[9], double D[9]) {
  switch (kind) {
    case WEFT_STRETCH:
      stretch_block_state(S, d, a, b, J);
      return false;
    case WEFT_BEND: {
      const double nk = -d[1];
      const V3 ga = v3(S[3 * a], S[3 * a + 1], S[3 * a + 2]);
      const V3 gb = v3(S[3 * b], S[3 * b + 1], S[3 * b + 2]);
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) J[r * 3 + c] = 0.0 + nk * (comp(ga, r) * comp(gb, c));
      return false;
    }
    case WEFT_SPRING: {
      const bool live = S[9] != 0.0;
#pragma unroll
      for (int q = 0; q < 9; ++q) J[q] = !live ? 0.0 : (b == a ? 0.0 - S[q] : 0.0 + S[q]);
      return false;
    }
    case WEFT_EXTERNAL: {
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          J[r * 3 + c] = 0.0;
          D[r * 3 + c] = 0.0 + d[3] * (r == c ? 1.0 : 0.0);
        }
      return d[3] > 0.0;
    }
    case WEFT_CONTACT: {
      const V3 n = v3(d[0], d[1], d[2]);
      const bool active = S[0] != 0.0;
      const double k = (d[9] * d[3 + a]) * d[3 + b];
      const double kd = (d[11] * d[3 + a]) * d[3 + b];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double nn = comp(n, r) * comp(n, c);
          J[r * 3 + c] = active ? 0.0 - k * nn : 0.0;
          D[r * 3 + c] = 0.0 + kd * ((r == c ? 1.0 : 0.0) - nn);
        }
      return d[11] > 0.0;
    }
    default:
#pragma unroll
      for (int q = 0; q < 9; ++q) J[q] = 0.0;
      return false;
  }
}

struct ElemArgs {
  int64_t n;
  const int64_t* __restrict__ list;  // element ids to evaluate (null: first .. first+n-1)
  double dt;
  const int4* __restrict__ est;
  const int2* __restrict__ einfo;
  const double* __restrict__ edamp;
  const double* __restrict__ epay;
  const int32_t* __restrict__ eres_off;
  double* __restrict__ eres;
  const double* __restrict__ xc;
  const double* __restrict__ xa;
  const double* __restrict__ vel;
  int64_t first;  // first element id (list == null)
};

#ifndef WEFT_EVAL_MINB
#define WEFT_EVAL_MINB 1
#endif
#ifndef WEFT_SLOT_MINB
#define WEFT_SLOT_MINB 4
#endif
// KIND >= 0: every element of the launch has that kind (runs of the static
// list, which build_elements orders triangles -> hinges -> vertices), so the
// kernel is compiled for one element kind — no divergence, and the register
// allocation of that kind only. KIND < 0: any kind (contacts, rank lists).
template <int KIND>
__global__ void __launch_bounds__(128, WEFT_EVAL_MINB) k_elem_eval(ElemArgs g) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  const int64_t e = g.list ? g.list[i] : g.first + i;
  const int4 s4 = g.est[e];
  const int2 info = g.einfo[e];
  const int kind = KIND >= 0 ? KIND : (info.x & 0xff), ss = (info.x >> 8) & 0xff;
  const int st[4] = {s4.x, s4.y, s4.z, s4.w};
  const double* __restrict__ d = g.epay + info.y;
  const double damping = g.edamp[e];
  double* __restrict__ R = g.eres + g.eres_off[e];
  double* __restrict__ S = R + 3 * ss;
  double f[4][3];
#pragma unroll
  for (int i = 0; i < 4; ++i) f[i][0] = f[i][1] = f[i][2] = 0.0;
  double fr[4][3];
#pragma unroll
  for (int i = 0; i < 4; ++i) fr[i][0] = fr[i][1] = fr[i][2] = 0.0;
  switch (kind) {
    case WEFT_STRETCH: {
      {  // stretch_force (elements.cpp:161-181) at x_adv
        const StretchSt sa = stretch_state(d, ld3(g.xa, st[0]), ld3(g.xa, st[1]), ld3(g.xa, st[2]));
        if (sa.ok) {
          const V3 wu_hat = divs(sa.wu, sa.wu_len), wv_hat = divs(sa.wv, sa.wv_len);
          const double a = d[6];
          const double cu = a * (sa.wu_len - 1.0), cv = a * (sa.wv_len - 1.0), cs = a * dot(sa.wu, sa.wv);
          const double su = -(d[7] * cu), sv = d[8] * cv, sc = d[9] * cs;
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const V3 gu = scl(a * d[i], wu_hat);
            const V3 gv = scl(a * d[3 + i], wv_hat);
            const V3 gs = scl(a, add(scl(d[i], sa.wv), scl(d[3 + i], sa.wu)));
            f[i][0] = 0.0 + ((su * gu.x - sv * gv.x) - sc * gs.x);
            f[i][1] = 0.0 + ((su * gu.y - sv * gv.y) - sc * gs.y);
            f[i][2] = 0.0 + ((su * gu.z - sv * gv.z) - sc * gs.z);
          }
        }
      }
      // x_cur state (elements.cpp:183-205)
      const StretchSt sc = stretch_state(d, ld3(g.xc, st[0]), ld3(g.xc, st[1]), ld3(g.xc, st[2]));
      if (sc.ok) {
        const V3 wu_hat = divs(sc.wu, sc.wu_len), wv_hat = divs(sc.wv, sc.wv_len);
        const double a = d[6];
        S[0] = wu_hat.x; S[1] = wu_hat.y; S[2] = wu_hat.z;
        S[3] = wv_hat.x; S[4] = wv_hat.y; S[5] = wv_hat.z;
        S[6] = sc.wu.x; S[7] = sc.wu.y; S[8] = sc.wu.z;
        S[9] = sc.wv.x; S[10] = sc.wv.y; S[11] = sc.wv.z;
        S[12] = sc.wu_len;
        S[13] = sc.wv_len;
        S[14] = a * dot(sc.wu, sc.wv);  // cs (unused in SpdProjected)
        S[15] = 1.0;
        S[16] = a * (sc.wu_len - 1.0);  // cu: keep_u2 iff cu >= 0
        S[17] = a * (sc.wv_len - 1.0);  // cv: keep_v2 iff cv >= 0
      } else {
#pragma unroll
        for (int q = 0; q < 18; ++q) S[q] = 0.0;
      }
      break;
    }
    case WEFT_BEND: {
      {  // bend_force at x_adv (elements.cpp:232-242)
        const V3 p0 = ld3(g.xa, st[0]), p1 = ld3(g.xa, st[1]), p2 = ld3(g.xa, st[2]), p3 = ld3(g.xa, st[3]);
        const double theta = dihedral_angle(p0, p1, p2, p3);
        V3 gg[4];
        dihedral_gradient(p0, p1, p2, p3, gg);
        const double coeff = -d[1] * (theta - d[0]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          f[i][0] = 0.0 + coeff * gg[i].x;
          f[i][1] = 0.0 + coeff * gg[i].y;
          f[i][2] = 0.0 + coeff * gg[i].z;
        }
      }
      V3 gg[4];
      dihedral_gradient(ld3(g.xc, st[0]), ld3(g.xc, st[1]), ld3(g.xc, st[2]), ld3(g.xc, st[3]), gg);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        S[3 * i] = gg[i].x;
        S[3 * i + 1] = gg[i].y;
        S[3 * i + 2] = gg[i].z;
      }
      break;
    }
    case WEFT_SPRING: {
      {  // spring_force (elements.cpp:269-279)
        const V3 dd = sub(ld3(g.xa, st[1]), ld3(g.xa, st[0]));
        const double len = norm(dd);
        if (len >= 1e-12) {
          const V3 dir = divs(dd, len);
          const V3 fa = scl(d[1] * (len - d[0]), dir);
          f[0][0] = 0.0 + fa.x;
          f[0][1] = 0.0 + fa.y;
          f[0][2] = 0.0 + fa.z;
          f[1][0] = 0.0 - fa.x;
          f[1][1] = 0.0 - fa.y;
          f[1][2] = 0.0 - fa.z;
        }
      }
      const V3 dd = sub(ld3(g.xc, st[1]), ld3(g.xc, st[0]));
      const double len = norm(dd);
      if (len >= 1e-12) {
        const V3 dir = divs(dd, len);
        double lateral = 1.0 - d[0] / len;
        lateral = lateral > 0.0 ? lateral : 0.0;  // SpdProjected
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double oo = comp(dir, r) * comp(dir, c);
            S[r * 3 + c] = d[1] * (oo + lateral * ((r == c ? 1.0 : 0.0) - oo));
          }
        S[9] = 1.0;
      } else {
#pragma unroll
        for (int q = 0; q < 10; ++q) S[q] = 0.0;
      }
      break;
    }
    case WEFT_EXTERNAL: {
      f[0][0] = d[0];
      f[0][1] = d[1];
      f[0][2] = d[2];
      if (d[3] > 0.0) {
        const V3 v = ld3(g.vel, st[0]);
        fr[0][0] = -d[3] * v.x;
        fr[0][1] = -d[3] * v.y;
        fr[0][2] = -d[3] * v.z;
      }
      break;
    }
    case WEFT_CONTACT: {
      const V3 n = v3(d[0], d[1], d[2]);
      double gap = d[7];
      for (int i = 0; i < ss; ++i) gap = gap + d[3 + i] * dot(n, ld3(g.xa, st[i]));
      if (gap < d[8]) {
        const double mag = d[9] * (d[8] - gap);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < ss) {
            const double sv = mag * d[3 + i];
            f[i][0] = 0.0 + sv * n.x;
            f[i][1] = 0.0 + sv * n.y;
            f[i][2] = 0.0 + sv * n.z;
          }
        }
      }
      if (d[11] > 0.0) {
        V3 rel = v3(d[13], d[14], d[15]);
        for (int i = 0; i < ss; ++i) rel = add(rel, scl(d[3 + i], ld3(g.vel, st[i])));
        const double rn = dot(n, rel);
        const V3 tang = sub(rel, scl(rn, n));
        const V3 frv = scl(-d[11], tang);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < ss) {
            fr[i][0] = d[3 + i] * frv.x;
            fr[i][1] = d[3 + i] * frv.y;
            fr[i][2] = d[3 + i] * frv.z;
          }
        }
      }
      double gc = d[7];
      for (int i = 0; i < ss; ++i) gc = gc + d[3 + i] * dot(n, ld3(g.xc, st[i]));
      S[0] = gc < d[8] ? 1.0 : 0.0;
      break;
    }
    default:
      break;
  }
  // rhs contributions (assembly.hpp:185-197): f = force + friction, then
  // + damping * (J_ab v_b) in ascending b, then dt * f.
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i < ss) {
      double fx = f[i][0] + fr[i][0], fy = f[i][1] + fr[i][1], fz = f[i][2] + fr[i][2];
      if (damping > 0.0) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (b < ss) {
            double J[9], D[9];
            elem_block(kind, S, d, i, b, J, D);
            const V3 vb = ld3(g.vel, st[b]);
            fx = fx + damping * ((J[0] * vb.x + J[1] * vb.y) + J[2] * vb.z);
            fy = fy + damping * ((J[3] * vb.x + J[4] * vb.y) + J[5] * vb.z);
            fz = fz + damping * ((J[6] * vb.x + J[7] * vb.y) + J[8] * vb.z);
          }
        }
      }
      R[3 * i] = g.dt * fx;
      R[3 * i + 1] = g.dt * fy;
      R[3 * i + 2] = g.dt * fz;
    }
  }
}

struct SlotArgs {
  int p;     // held rows
  int row0;  // global index of the first
  const int32_t* __restrict__ perm;  // matrix position -> local row
  int64_t n_static;
  double dt;
  const int64_t* __restrict__ slice_off;
  const int32_t* __restrict__ rowlen;
  const int32_t* __restrict__ cols;
  double* __restrict__ vals;
  int64_t total;
  const double* __restrict__ mass;
  const uint8_t* __restrict__ pinned;
  const int64_t* __restrict__ inc_ptr;
  const int32_t* __restrict__ inc;
  const int64_t* __restrict__ cinc_ptr;
  const int32_t* __restrict__ cinc;
  const int4* __restrict__ est;
  const int2* __restrict__ einfo;
  const double* __restrict__ edamp;
  const double* __restrict__ epay;
  const int32_t* __restrict__ eres_off;
  const double* __restrict__ eres;
  double* __restrict__ rhs;
  int* __restrict__ bad_mass;
  float* __restrict__ vals32;  // Precision::Single outputs (T = float)
  float* __restrict__ rhs32;
  int stage_cap;  // k_fill_slots<0>: staged incidences per slice (dynamic shared memory)
};

#ifndef WEFT_SLOT_WARPS
#define WEFT_SLOT_WARPS 4  // 4 warps x 4 CTAs/SM measured best (3, 8, 13 slower)
#endif
constexpr int kSlotWarps = WEFT_SLOT_WARPS;
// staged incidences per slice (static + contact): 1024 for the static list;
// slices of a system with contacts hold up to ~1300 (the longest rows are
// sorted together), and a slice over the cap falls back to global reads
// (config D contacts mode: 9.4 -> 7.2 ms of assembly with the larger cap)
constexpr int kStageCap = 1024;
constexpr int kStageCapContacts = 1300;  // 47 KB of static shared memory

// One staged incidence of the slice (shared memory).
struct StagedInc {
  int4 st;        // stencil
  int kind_ss_a;  // kind | ss << 8 | a << 16
  int pay;        // payload offset
  int res;        // state offset (results + 3 ss)
  double damping;
};

// acc += (-scale) J_ab (+ dt D_ab) for one coupling, block regenerated from
// the element's phase-1 state (bitwise the blocks fill_matrix adds); each
// contribution computed in double and cast to Real before the add.
template <class T = double>
__device__ __forceinline__ void add_block(const StagedInc& si, int b, const double* __restrict__ epay,
                                          const double* __restrict__ eres, double dt, T acc[9]) {
  // acc += (-scale) J_ab (+ dt D_ab), entry by entry with elem_block's exact
  // expressions but no 3x3 temporaries (register pressure of k_fill_slots)
  const int kind = si.kind_ss_a & 0xff, a = (si.kind_ss_a >> 16) & 0xff;
  const double* __restrict__ S = eres + si.res;
  const double* __restrict__ d = epay + si.pay;
  const double nscale = -(dt * dt + si.damping * dt);
  switch (kind) {
    case WEFT_STRETCH: {
      if (S[15] == 0.0) {
#pragma unroll
        for (int q = 0; q < 9; ++q) acc[q] = acc[q] + static_cast<T>(nscale * 0.0);
        return;
      }
      const V3 wu_hat = v3(S[0], S[1], S[2]), wv_hat = v3(S[3], S[4], S[5]);
      const V3 wu = v3(S[6], S[7], S[8]), wv = v3(S[9], S[10], S[11]);
      const double wu_len = S[12], wv_len = S[13];
      const double ar = d[6];
      const double ui = d[a], vi = d[3 + a], uj = d[b], vj = d[3 + b];
      const V3 gui = scl(ar * ui, wu_hat), gvi = scl(ar * vi, wv_hat);
      const V3 gsi = scl(ar, add(scl(ui, wv), scl(vi, wu)));
      const V3 guj = scl(ar * uj, wu_hat), gvj = scl(ar * vj, wv_hat);
      const V3 gsj = scl(ar, add(scl(uj, wv), scl(vj, wu)));
      const double su2 = (d[7] * S[16]) * (((ar * ui) * uj) / wu_len);
      const double sv2 = (d[8] * S[17]) * (((ar * vi) * vj) / wv_len);
      const bool keep_u2 = S[16] >= 0.0, keep_v2 = S[17] >= 0.0;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double id = r == c ? 1.0 : 0.0;
          double m = 0.0;
          m = m - d[7] * (comp(gui, r) * comp(guj, c));
          m = m - d[8] * (comp(gvi, r) * comp(gvj, c));
          m = m - d[9] * (comp(gsi, r) * comp(gsj, c));
          if (keep_u2) m = m - su2 * (id - comp(wu_hat, r) * comp(wu_hat, c));
          if (keep_v2) m = m - sv2 * (id - comp(wv_hat, r) * comp(wv_hat, c));
          acc[r * 3 + c] = acc[r * 3 + c] + static_cast<T>(nscale * (0.0 + m));
        }
      return;
    }
    case WEFT_BEND: {
      const double nk = -d[1];
      const V3 ga = v3(S[3 * a], S[3 * a + 1], S[3 * a + 2]);
      const V3 gb = v3(S[3 * b], S[3 * b + 1], S[3 * b + 2]);
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          acc[r * 3 + c] = acc[r * 3 + c] + static_cast<T>(nscale * (0.0 + nk * (comp(ga, r) * comp(gb, c))));
      return;
    }
    default: {
      double J[9], D[9];
      const bool damped = elem_block(kind, S, d, a, b, J, D);
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        double cv = nscale * J[q];
        if (damped) cv = cv + dt * D[q];
        acc[q] = acc[q] + static_cast<T>(cv);
      }
    }
  }
}

// Phase 2: one CTA per slice of 32 rows. The slice's incidences (static then
// contact, each ascending element per row) are staged in shared memory;
// warp w computes slots w, w+8, ... of its lane's row.
template <int kCap, class T = double>
__global__ void __launch_bounds__(kSlotWarps * 32, WEFT_SLOT_MINB) k_fill_slots(SlotArgs g) {
  T* const out_vals = std::is_same_v<T, float> ? reinterpret_cast<T*>(g.vals32) : reinterpret_cast<T*>(g.vals);
  T* const out_rhs = std::is_same_v<T, float> ? reinterpret_cast<T*>(g.rhs32) : reinterpret_cast<T*>(g.rhs);
  // kCap == 0: the staging arrays live in dynamic shared memory sized
  // g.stage_cap (systems with contacts: room for the heaviest slices)
  constexpr bool kDyn = kCap == 0;
  constexpr int kS = kDyn ? 1 : kCap;
  __shared__ int4 sm_st_s[kS];
  __shared__ int sm_ksa_s[kS], sm_pay_s[kS], sm_res_s[kS];
  __shared__ double sm_damp_s[kS];
  extern __shared__ __align__(16) unsigned char fs_dyn[];
  const int cap = kDyn ? g.stage_cap : kCap;
  int4* const sm_st = kDyn ? reinterpret_cast<int4*>(fs_dyn) : sm_st_s;
  double* const sm_damp = kDyn ? reinterpret_cast<double*>(fs_dyn + 16 * (size_t)cap) : sm_damp_s;
  int* const sm_ksa = kDyn ? reinterpret_cast<int*>(fs_dyn + 24 * (size_t)cap) : sm_ksa_s;
  int* const sm_pay = kDyn ? reinterpret_cast<int*>(fs_dyn + 28 * (size_t)cap) : sm_pay_s;
  int* const sm_res = kDyn ? reinterpret_cast<int*>(fs_dyn + 32 * (size_t)cap) : sm_res_s;
  __shared__ int sm_row[2][kSlice + 1];  // per pass: lane -> first staged entry
  __shared__ int64_t sm_beg[2][kSlice];   // per pass: lane -> first incidence
  __shared__ int sm_rid[kSlice];          // lane -> global row
  const int slice = blockIdx.x;
  const int rows = min(kSlice, g.p - slice * kSlice);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // The slice's rows (SELL-32-sigma positions -> rows, not contiguous):
  // per-lane incidence counts, warp-scanned into staging offsets.
  if (warp == 0) {
    int row = 0, ns = 0, nc = 0;
    if (lane < rows) {
      row = g.row0 + g.perm[slice * kSlice + lane];
      const int64_t a0 = g.inc_ptr[row], c0 = g.cinc_ptr[row];
      ns = static_cast<int>(g.inc_ptr[row + 1] - a0);
      nc = static_cast<int>(g.cinc_ptr[row + 1] - c0);
      sm_beg[0][lane] = a0;
      sm_beg[1][lane] = c0;
      sm_rid[lane] = row;
    }
    int ps = ns, pc = nc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ts = __shfl_up_sync(0xffffffffu, ps, o), tc = __shfl_up_sync(0xffffffffu, pc, o);
      if (lane >= o) {
        ps += ts;
        pc += tc;
      }
    }
    const int tots = __shfl_sync(0xffffffffu, ps, 31);
    sm_row[0][lane] = ps - ns;  // exclusive
    sm_row[1][lane] = tots + pc - nc;
    if (lane == 31) {
      sm_row[0][32] = tots;
      sm_row[1][32] = tots + pc;
    }
  }
  __syncthreads();
  const int nstat = sm_row[0][32], ncont = sm_row[1][32] - nstat;
  const bool staged = nstat + ncont <= cap;
  if (staged) {
    for (int i = threadIdx.x; i < nstat + ncont; i += blockDim.x) {
      const bool cpass = i >= nstat;
      const int* off = sm_row[cpass ? 1 : 0];
      int l = 0;  // lane whose range holds i (ranges of lanes >= rows are empty)
#pragma unroll
      for (int step = 16; step > 0; step >>= 1)
        if (l + step <= 32 && off[l + step] <= i) l += step;
      while (l + 1 < 32 && off[l + 1] <= i) ++l;
      const int64_t at = sm_beg[cpass ? 1 : 0][l] + (i - off[l]);
      const int code = cpass ? g.cinc[at] : g.inc[at];
      const int64_t e = (cpass ? g.n_static : 0) + (code >> 2);
      const int2 info = g.einfo[e];
      const int ss = (info.x >> 8) & 0xff;
      sm_st[i] = g.est[e];
      sm_ksa[i] = info.x | ((code & 3) << 16);
      sm_pay[i] = info.y;
      sm_res[i] = g.eres_off[e] + 3 * ss;
      sm_damp[i] = g.edamp[e];
    }
  }
  __syncthreads();
  if (lane >= rows) return;
  const int r = sm_rid[lane];
  const int len = g.rowlen[slice * kSlice + lane];
  const int64_t base = g.slice_off[slice] + lane;
  const double dt = g.dt;
  for (int k = warp; k < len; k += kSlotWarps) {
    const int64_t at = base + (int64_t)k * kSlice;
    const int col = g.cols[at] & kColMask;
    T acc[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) acc[q] = 0;
    if (col == r) {  // mass diagonal first (assembly.hpp:155-166)
      const T m = g.pinned[r] ? T(1) : static_cast<T>(g.mass[r]);
      acc[0] = acc[0] + m;
      acc[4] = acc[4] + m;
      acc[8] = acc[8] + m;
    }
    if (staged) {
      for (int pass = 0; pass < 2; ++pass) {
        const int i1 = sm_row[pass][lane + 1];
        for (int i = sm_row[pass][lane]; i < i1; ++i) {
          const int4 st4 = sm_st[i];
          const int ss = (sm_ksa[i] >> 8) & 0xff;
          const int stv[4] = {st4.x, st4.y, st4.z, st4.w};
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            if (b < ss && stv[b] == col) {
              StagedInc si{st4, sm_ksa[i], sm_pay[i], sm_res[i], sm_damp[i]};
              add_block<T>(si, b, g.epay, g.eres, dt, acc);
            }
          }
        }
      }
    } else {
      for (int pass = 0; pass < 2; ++pass) {
        const int64_t* ip = pass == 0 ? g.inc_ptr : g.cinc_ptr;
        const int32_t* il = pass == 0 ? g.inc : g.cinc;
        const int64_t i1 = ip[r + 1];
        for (int64_t ii = ip[r]; ii < i1; ++ii) {
          const int code = il[ii];
          const int64_t e = (pass == 0 ? 0 : g.n_static) + (code >> 2);
          const int2 info = g.einfo[e];
          const int ss = (info.x >> 8) & 0xff;
          StagedInc si;
          si.st = g.est[e];
          si.kind_ss_a = info.x | ((code & 3) << 16);
          si.pay = info.y;
          si.res = g.eres_off[e] + 3 * ss;
          si.damping = g.edamp[e];
          const int stv[4] = {si.st.x, si.st.y, si.st.z, si.st.w};
#pragma unroll
          for (int b = 0; b < 4; ++b)
            if (b < ss && stv[b] == col) add_block<T>(si, b, g.epay, g.eres, dt, acc);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) out_vals[vidx(at, lane, q)] = acc[q];
  }
  // rhs of the lane's row (assembly.hpp:182-197): the phase-1 contributions
  // dt f_a of its incidences in ascending element order. Each sits right
  // before the element state the slot loop above just read, so it comes out
  // of L2 (a separate row pass re-read them from DRAM: 1.9 GB per step at D).
  // Done by the last warp, which has the fewest slots.
  if (warp == kSlotWarps - 1) {
    if (!g.pinned[r] && g.mass[r] <= 0.0) atomicMin(g.bad_mass, r);
    T r0 = 0, r1 = 0, r2 = 0;
    for (int pass = 0; pass < 2; ++pass) {
      if (staged) {
        const int i1 = sm_row[pass][lane + 1];
#pragma unroll 4  // the loads of four incidences in flight at once (same summation order)
        for (int i = sm_row[pass][lane]; i < i1; ++i) {
          const int ksa = sm_ksa[i];
          const double* R = g.eres + sm_res[i] - 3 * ((ksa >> 8) & 0xff) + 3 * ((ksa >> 16) & 0xff);
          r0 = r0 + static_cast<T>(R[0]);
          r1 = r1 + static_cast<T>(R[1]);
          r2 = r2 + static_cast<T>(R[2]);
        }
      } else {
        const int64_t* ip = pass == 0 ? g.inc_ptr : g.cinc_ptr;
        const int32_t* il = pass == 0 ? g.inc : g.cinc;
        const int64_t i1 = ip[r + 1];
        for (int64_t ii = ip[r]; ii < i1; ++ii) {
          const int code = il[ii];
          const int64_t e = (pass == 0 ? 0 : g.n_static) + (code >> 2);
          const double* R = g.eres + g.eres_off[e] + 3 * (code & 3);
          r0 = r0 + static_cast<T>(R[0]);
          r1 = r1 + static_cast<T>(R[1]);
          r2 = r2 + static_cast<T>(R[2]);
        }
      }
    }
    out_rhs[3 * r] = r0;
    out_rhs[3 * r + 1] = r1;
    out_rhs[3 * r + 2] = r2;
  }
}

constexpr int kFillThreads = 64;
constexpr int kWideCap = 24;

// 1 for elements with a non-pinned stencil vertex in [row0, row1): the
// element instances distribute_elements hands this rank (assembly.cpp:28-51).
__global__ void k_elem_mine(int64_t n, const int4* __restrict__ est, const int2* __restrict__ einfo,
                            const uint8_t* __restrict__ pinned, int row0, int row1, uint8_t* __restrict__ flag) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int4 s4 = est[e];
  const int ss = (einfo[e].x >> 8) & 0xff;
  const int sv[4] = {s4.x, s4.y, s4.z, s4.w};
  uint8_t mine = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
    if (a < ss && sv[a] >= row0 && sv[a] < row1 && !pinned[sv[a]]) mine = 1;
  flag[e] = mine;
}

// Compacts this rank's element ids (ascending) into c.elist; returns count.
static int64_t select_rank_elements(Ctx& c) {
  const int64_t ne = c.n_static + c.n_contacts;
  cudaStream_t s = c.stream;
  DBuf<uint8_t>& flag = c.sc_sel_flag;
  flag.resize(static_cast<size_t>(ne) + 1);
  c.elist.resize(static_cast<size_t>(ne) + 1);
  DBuf<int64_t>& cnt = c.sc_sel_cnt;
  cnt.resize(1);
  if (!ne) return 0;
  k_elem_mine<<<div_up(ne, 256), 256, 0, ls(c)>>>(ne, c.est.data(), c.einfo.data(), c.pinned.data(), c.row0, c.row1,
                                                   flag.data());
  cub::CountingInputIterator<int64_t> ids(0);
  size_t tmp = 0;
  cub::DeviceSelect::Flagged(nullptr, tmp, ids, flag.data(), c.elist.data(), cnt.data(), ne, s);
  void* t = scratch(c, tmp);
  WG_CUDA(cub::DeviceSelect::Flagged(t, tmp, ids, flag.data(), c.elist.data(), cnt.data(), ne, s));
  int64_t h = 0;
  WG_CUDA(cudaMemcpyAsync(&h, cnt.data(), sizeof(h), cudaMemcpyDeviceToHost, s));
  WG_CUDA(cudaStreamSynchronize(s));
  return h;
}

void fill_matrix(Ctx& c, const double* xc, const double* xa, const double* vel, double dt, int mode, bool finish,
                 bool f32) {
  if (!(dt > 0.0)) throw Error(WEFT_ERR_DIMENSION, "fill_matrix: dt must be positive");
  if (f32 && c.world > 1) throw Error(WEFT_ERR_INVALID, "fill_matrix: Precision::Single runs on one rank");
  if (c.p == 0 && c.n_static == 0) throw Error(WEFT_ERR_INVALID, "fill_matrix: set_vertices/set_elements first");
  if (c.spat_ptr.size() != static_cast<size_t>(c.p) + 1) throw Error(WEFT_ERR_INVALID, "fill_matrix: set_elements first");
  cudaStream_t s = c.stream;
  const bool layout_cached = c.has_matrix && c.n_contacts == 0 && c.have_pattern_for_contacts;
  if (!layout_cached) {
    build_layout(c);
    c.have_pattern_for_contacts = c.n_contacts == 0;
  }
  SellMatrix& A = c.A;
  c.rhs.resize(3 * static_cast<size_t>(c.p) + 3);  // holds 3p floats for Precision::Single
  if (f32) A.vals32.resize(9 * static_cast<size_t>(A.total) + 9);
  c.scalars.resize(64);
  int* bad = reinterpret_cast<int*>(c.scalars.data() + 8);
  const int big = INT32_MAX;
  WG_CUDA(cudaMemcpyAsync(bad, &big, sizeof(int), cudaMemcpyHostToDevice, s));
  const int nloc = c.row1 - c.row0;
  FillArgs f{};
  f.p = nloc;
  f.row0 = c.row0;
  f.perm = A.perm.data();
  f.n_static = c.n_static;
  f.dt = dt;
  f.exact = mode == WEFT_JAC_EXACT;
  f.wcap = std::min(A.max_len, kWideCap);
  f.slice_off = A.slice_off.data();
  f.rowlen = A.rowlen.data();
  f.cols = A.cols.data();
  f.vals = A.vals.data();
  f.total = A.total;
  f.rhs = c.rhs.data();
  f.vals32 = A.vals32.data();
  f.rhs32 = reinterpret_cast<float*>(c.rhs.data());
  f.mass = c.mass.data();
  f.pinned = c.pinned.data();
  f.inc_ptr = c.inc_ptr.data();
  f.inc = c.inc.data();
  f.cinc_ptr = c.cinc_ptr.data();
  f.cinc = c.cinc.data();
  f.est = c.est.data();
  f.einfo = c.einfo.data();
  f.edamp = c.edamp.data();
  f.epay = c.epay.data();
  f.xc = xc;
  f.xa = xa;
  f.vel = vel;
  f.bad_mass = bad;
  auto zero_padding = [&]() {  // the precision's value planes
    if (f32)
      k_zero_padding<float><<<div_up(nloc, 256), 256, 0, ls(c)>>>(nloc, A.slice_off.data(), A.rowlen.data(),
                                                                  A.vals32.data(), A.total);
    else if (!layout_cached)
      k_zero_padding<double><<<div_up(nloc, 256), 256, 0, ls(c)>>>(nloc, A.slice_off.data(), A.rowlen.data(),
                                                                   A.vals.data(), A.total);
  };
  if (nloc && !f.exact) {
    zero_padding();
    // phase 1 over every element (one rank) or over the elements coupled to
    // this rank's rows (distribute_elements, assembly.cpp:28-51)
    int64_t ne = c.n_static + c.n_contacts;
    const int64_t* list = nullptr;
    if (c.world > 1) {
      ne = select_rank_elements(c);
      list = c.elist.data();
    }
    ElemArgs ea{ne, list, dt, c.est.data(), c.einfo.data(), c.edamp.data(), c.epay.data(), c.eres_off.data(),
                c.eres.data(), xc, xa, vel, 0};
    if (list || c.kind_runs.empty()) {
      if (ne) k_elem_eval<-1><<<div_up(ne, 128), 128, 0, ls(c)>>>(ea);
    } else {
      // one launch per same-kind run of the static list, then the contacts
      for (const auto& run : c.kind_runs) {
        ElemArgs er = ea;
        er.first = run.begin;
        er.n = run.end - run.begin;
        if (!er.n) continue;
        const int blocks = div_up(er.n, 128);
        switch (run.kind) {
          case WEFT_STRETCH: k_elem_eval<WEFT_STRETCH><<<blocks, 128, 0, ls(c)>>>(er); break;
          case WEFT_BEND: k_elem_eval<WEFT_BEND><<<blocks, 128, 0, ls(c)>>>(er); break;
          case WEFT_EXTERNAL: k_elem_eval<WEFT_EXTERNAL><<<blocks, 128, 0, ls(c)>>>(er); break;
          default: k_elem_eval<-1><<<blocks, 128, 0, ls(c)>>>(er); break;
        }
      }
      if (c.n_contacts) {
        ElemArgs er = ea;
        er.first = c.n_static;
        er.n = c.n_contacts;
        k_elem_eval<-1><<<div_up(er.n, 128), 128, 0, ls(c)>>>(er);
      }
    }
    SlotArgs sa{nloc, c.row0, A.perm.data(), c.n_static, dt, A.slice_off.data(), A.rowlen.data(), A.cols.data(), A.vals.data(),
                A.total, c.mass.data(), c.pinned.data(), c.inc_ptr.data(), c.inc.data(), c.cinc_ptr.data(),
                c.cinc.data(), c.est.data(), c.einfo.data(), c.edamp.data(), c.epay.data(), c.eres_off.data(),
                c.eres.data(), c.rhs.data(), bad, A.vals32.data(), reinterpret_cast<float*>(c.rhs.data())};
    if (f32) {
      if (c.n_contacts > 0) k_fill_slots<kStageCapContacts, float><<<A.nslices, kSlotWarps * 32, 0, ls(c)>>>(sa);
      else k_fill_slots<kStageCap, float><<<A.nslices, kSlotWarps * 32, 0, ls(c)>>>(sa);
    } else {
      if (c.n_contacts > 0) {
        // 36 bytes per staged incidence; 1536 keeps 4 CTAs per SM (221 KB)
        static const int cap_env = std::getenv("WEFT_FS_CAP") ? std::atoi(std::getenv("WEFT_FS_CAP")) : 1536;
        sa.stage_cap = cap_env;
        const int bytes = 36 * cap_env;
        // per call: the attribute belongs to the current device's module
        WG_CUDA(cudaFuncSetAttribute(k_fill_slots<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        k_fill_slots<0><<<A.nslices, kSlotWarps * 32, bytes, ls(c)>>>(sa);
      }
      else k_fill_slots<kStageCap><<<A.nslices, kSlotWarps * 32, 0, ls(c)>>>(sa);
    }
    WG_CUDA(cudaGetLastError());
  } else if (nloc) {
    zero_padding();
    const size_t smem = static_cast<size_t>(f.wcap) * (9 * sizeof(double) + sizeof(int32_t)) * kFillThreads;
    auto narrow = f32 ? (f.exact ? k_fill<false, true, float> : k_fill<false, false, float>)
                      : (f.exact ? k_fill<false, true> : k_fill<false, false>);
    auto wide = f32 ? (f.exact ? k_fill<true, true, float> : k_fill<true, false, float>)
                    : (f.exact ? k_fill<true, true> : k_fill<true, false>);
    WG_CUDA(cudaFuncSetAttribute(narrow, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    narrow<<<div_up(nloc, kFillThreads), kFillThreads, smem, ls(c)>>>(f);
    if (A.max_len > kWideCap) {
      // rows wider than the shared-memory budget accumulate in place
      wide<<<div_up(nloc, kFillThreads), kFillThreads, 0, ls(c)>>>(f);
    }
    WG_CUDA(cudaGetLastError());
  }
  A.f32 = f32;
  c.has_matrix = true;
  c.has_rhs = true;
  if (finish) fill_matrix_finish(c);
}

void fill_matrix_finish(Ctx& c) {
  const int big = INT32_MAX;
  int hbad = big;
  const int* bad = reinterpret_cast<const int*>(c.scalars.data() + 8);
  read_small(c, c.stream, {bad, &hbad, sizeof(int)});
  if (hbad != big) {
    c.has_matrix = false;
    c.has_rhs = false;
    throw Error(WEFT_ERR_DIMENSION, "fill_matrix: vertex " + std::to_string(hbad) + " has non-positive mass");
  }
}

}  // namespace weft_gpu
