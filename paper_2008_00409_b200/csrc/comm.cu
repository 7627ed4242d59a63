// comm.cu — the rank group: one process per GPU, peer memory over CUDA IPC.
//
// Replaces the reference's in-process "interconnect" — the stage-barrier
// pipelined copies of Engine::run_pipelined (proj/src/exec.cpp:189-307) and
// the ordered all-reduce (exec.cpp:170-174) — by direct loads/stores into
// mapped peer memory (NVLink P2P on a B200 node, NVSwitch-routed). Each rank
// exports ONE window: a header of sequence flags and reduction slots
// (CommHeader) followed by the vectors its peers read: the PCG gather
// vectors z and p, and the simulation state v, x (two buffers, swapped in
// lockstep on every rank). Kernels synchronise through the flags
// (common.cuh); no host round trip and no NCCL call is on the data path.
#include <algorithm>
#include <cstring>

#include "ctx.cuh"

namespace weft_gpu {

namespace {
constexpr size_t kHeaderBytes = 4096;
static_assert(sizeof(CommHeader) <= kHeaderBytes, "comm header too large");
enum WinVec { kWinZ = 0, kWinP, kWinV, kWinX0, kWinX1, kWinVecs };

size_t vec_offset(int p, int which) {
  return kHeaderBytes + static_cast<size_t>(which) * 3 * sizeof(double) * static_cast<size_t>(p);
}
// Narrow-phase hit exchange area after the vectors: keys, then 8 doubles
// per hit. A share's unique hits must fit (config D: 275 K proximities for
// 827 K vertices); more raises ExecError on every rank.
size_t hit_cap(int p) { return std::max<size_t>(size_t(1) << 16, static_cast<size_t>(p)); }
size_t hit_keys_offset(int p) { return vec_offset(p, kWinVecs); }
size_t hit_vals_offset(int p) { return hit_keys_offset(p) + sizeof(unsigned long long) * hit_cap(p); }
size_t win_total(int p) { return hit_vals_offset(p) + 8 * sizeof(double) * hit_cap(p); }
}  // namespace

void comm_need(Ctx& c, const char* what) {
  if (c.world > 1 && !c.attached)
    throw Error(WEFT_ERR_INVALID, std::string(what) +
                                      ": multi-rank context is not attached (weft_gpu_comm_export + "
                                      "weft_gpu_comm_attach first)");
}

void comm_check(Ctx& c) {
  if (c.world <= 1 || !c.attached) return;
  unsigned long long err = 0;
  WG_CUDA(cudaMemcpy(&err, c.seq.data() + 3, sizeof(err), cudaMemcpyDeviceToHost));
  if (err) {
    const unsigned long long zero = 0;
    WG_CUDA(cudaMemcpy(c.seq.data() + 3, &zero, sizeof(zero), cudaMemcpyHostToDevice));
    throw Error(WEFT_ERR_EXEC, "device " + std::to_string(c.device) + " failed: rank " + std::to_string(c.rank) +
                                   " timed out waiting for a peer rank");
  }
}

void comm_export(Ctx& c, void* handle_out) {
  if (c.world <= 1) throw Error(WEFT_ERR_INVALID, "comm_export: single-rank context (partition range covers all)");
  const int p = c.pm.p;
  if (p <= 0) throw Error(WEFT_ERR_INVALID, "comm_export: set_vertices (or set_matrix) first");
  if (c.win) {
    if (c.win_p != p) throw Error(WEFT_ERR_INVALID, "comm_export: vertex count changed after export");
  } else {
    c.win_bytes = win_total(p);
    WG_CUDA(cudaMalloc(&c.win, c.win_bytes));
    WG_CUDA(cudaMemset(c.win, 0, c.win_bytes));
    c.win_p = p;
    char* base = static_cast<char*>(c.win);
    const size_t n = 3 * static_cast<size_t>(p);
    c.z.attach(reinterpret_cast<double*>(base + vec_offset(p, kWinZ)), n);
    c.pv.attach(reinterpret_cast<double*>(base + vec_offset(p, kWinP)), n);
    c.sim_v.attach(reinterpret_cast<double*>(base + vec_offset(p, kWinV)), n);
    c.sim_x.attach(reinterpret_cast<double*>(base + vec_offset(p, kWinX0)), n);
    c.sim_xc.attach(reinterpret_cast<double*>(base + vec_offset(p, kWinX1)), n);
    c.seq.resize(5);
    c.seq.zero(c.stream);
    WG_CUDA(cudaStreamSynchronize(c.stream));
  }
  cudaIpcMemHandle_t h;
  WG_CUDA(cudaIpcGetMemHandle(&h, c.win));
  static_assert(sizeof(h) == WEFT_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
}

void comm_attach(Ctx& c, const void* handles) {
  if (!c.win) throw Error(WEFT_ERR_INVALID, "comm_attach: comm_export first");
  if (c.attached) throw Error(WEFT_ERR_INVALID, "comm_attach: already attached");
  const auto* hb = static_cast<const unsigned char*>(handles);
  CommView& v = c.comm;
  v = CommView();
  v.world = c.world;
  v.rank = c.rank;
  v.ppr = c.part_end - c.part_begin;
  v.seq = c.seq.data();
  for (int q = 0; q < c.world; ++q) {
    if (q == c.rank) {
      c.peer_win[q] = c.win;
    } else {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, hb + static_cast<size_t>(q) * WEFT_IPC_HANDLE_BYTES, sizeof(h));
      void* ptr = nullptr;
      WG_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
      c.peer_win[q] = ptr;
    }
    char* base = static_cast<char*>(c.peer_win[q]);
    v.base[q] = base;
    v.hdr[q] = reinterpret_cast<CommHeader*>(base);
    v.z[q] = reinterpret_cast<const double*>(base + vec_offset(c.win_p, kWinZ));
    v.p[q] = reinterpret_cast<const double*>(base + vec_offset(c.win_p, kWinP));
  }
  c.attached = true;
}

void comm_free(Ctx& c) {
  for (int q = 0; q < kMaxRanks; ++q) {
    if (c.peer_win[q] && c.peer_win[q] != c.win) cudaIpcCloseMemHandle(c.peer_win[q]);
    c.peer_win[q] = nullptr;
  }
  if (c.win) cudaFree(c.win);
  c.win = nullptr;
  c.attached = false;
}

// ---------------------------------------------------------------------------
// Simulation state exchange: after the candidate update each rank owns the
// new v and x_cand of its rows; the replicated broad phase and the next
// assembly need all rows (the reference replicates the grid on every
// device, collision.cpp:397-399).
// ---------------------------------------------------------------------------
__global__ void k_state_publish(CommView cv) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  __threadfence_system();
  const unsigned long long s = cv.seq[2] + 1;
  cv.seq[2] = s;
  for (int q = 0; q < cv.world; ++q) st_release_sys(&cv.hdr[q]->state_ready[cv.rank], s);
}

// Pulls every other rank's rows of v and x_cand (window offsets off_v,
// off_xc, identical on all ranks) into this rank's full copies.
__global__ void k_state_gather(CommView cv, PartMap pm, int64_t off_v, int64_t off_xc, double* __restrict__ v,
                               double* __restrict__ xc) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= pm.p) return;
  const int q = pm.owner(r) / cv.ppr;
  if (q == cv.rank) return;
  if (!wait_flag(&cv.hdr[cv.rank]->state_ready[q], cv.seq[2])) atomicExch(cv.seq + 3, 1ull);
  const double* sv = reinterpret_cast<const double*>(cv.base[q] + off_v);
  const double* sx = reinterpret_cast<const double*>(cv.base[q] + off_xc);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    v[3 * r + k] = __ldcg(sv + 3 * r + k);
    xc[3 * r + k] = __ldcg(sx + 3 * r + k);
  }
}

void exchange_state(Ctx& c) {
  comm_need(c, "sim_step");
  k_state_publish<<<1, 32, 0, ls(c)>>>(c.comm);
  const char* base = static_cast<const char*>(c.win);
  const int64_t off_v = reinterpret_cast<const char*>(c.sim_v.data()) - base;
  const int64_t off_xc = reinterpret_cast<const char*>(c.sim_xc.data()) - base;
  if (c.pm.p)
    k_state_gather<<<div_up(c.pm.p, 256), 256, 0, ls(c)>>>(c.comm, c.pm, off_v, off_xc, c.sim_v.data(),
                                                          c.sim_xc.data());
  WG_CUDA(cudaGetLastError());
  rank_barrier(c);  // peers are done reading this rank's v / x_cand rows
}

// ---------------------------------------------------------------------------
// Narrow-phase hit exchange: the merge of collide (collision.cpp:405-417).
// Every rank narrow-phased its split_workload share of the replicated grid
// into sorted unique (kind, a, b) hits; the union, sorted and deduplicated,
// is the reference's NarrowPhaseResult and becomes every rank's contact
// list (so proximities_to_elements and the zones see all hits).
// ---------------------------------------------------------------------------
__global__ void k_hits_publish(CommView cv, long long nhits, long long npairs) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned long long s = cv.seq[4] + 1;
  cv.seq[4] = s;
  for (int q = 0; q < cv.world; ++q) {
    cv.hdr[q]->hit_count[cv.rank] = nhits;
    cv.hdr[q]->pair_count[cv.rank] = npairs;
  }
  __threadfence_system();
  for (int q = 0; q < cv.world; ++q) st_release_sys(&cv.hdr[q]->hits_ready[cv.rank], s);
}

__global__ void k_hits_wait(CommView cv, long long* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  CommHeader* me = cv.hdr[cv.rank];
  for (int q = 0; q < cv.world; ++q) {
    if (!wait_flag(&me->hits_ready[q], cv.seq[4])) atomicExch(cv.seq + 3, 1ull);
    out[q] = __ldcg(&me->hit_count[q]);
    out[kMaxRanks + q] = __ldcg(&me->pair_count[q]);
  }
}

int64_t merge_hits(Ctx& c) {
  comm_need(c, "collide");
  cudaStream_t s = c.stream;
  const int64_t nu = c.n_contacts_found;
  const size_t cap = hit_cap(c.win_p);
  char* base = static_cast<char*>(c.win);
  const int64_t nput = std::min<int64_t>(nu, static_cast<int64_t>(cap));
  if (nput) {
    WG_CUDA(cudaMemcpyAsync(base + hit_keys_offset(c.win_p), c.contact_keys.data(), 8 * nput,
                            cudaMemcpyDeviceToDevice, s));
    WG_CUDA(cudaMemcpyAsync(base + hit_vals_offset(c.win_p), c.contact_vals.data(), 64 * nput,
                            cudaMemcpyDeviceToDevice, s));
  }
  k_hits_publish<<<1, 32, 0, ls(c)>>>(c.comm, nu, c.narrow_pairs);
  c.hit_counts.resize(2 * kMaxRanks);
  k_hits_wait<<<1, 32, 0, ls(c)>>>(c.comm, c.hit_counts.data());
  WG_CUDA(cudaGetLastError());
  long long cnt[2 * kMaxRanks] = {};
  WG_CUDA(cudaMemcpyAsync(cnt, c.hit_counts.data(), sizeof(cnt), cudaMemcpyDeviceToHost, s));
  WG_CUDA(cudaStreamSynchronize(s));
  comm_check(c);
  int64_t total = 0, pairs = 0;
  for (int q = 0; q < c.world; ++q) {
    if (cnt[q] > static_cast<long long>(cap)) {
      rank_barrier(c);
      WG_CUDA(cudaStreamSynchronize(s));
      throw Error(WEFT_ERR_EXEC, "device " + std::to_string(c.device) + " failed: rank " + std::to_string(q) +
                                     " found " + std::to_string(cnt[q]) + " narrow-phase hits, more than the " +
                                     std::to_string(cap) + " the rank window holds");
    }
    total += cnt[q];
    pairs += cnt[kMaxRanks + q];
  }
  c.hit_keys.resize(static_cast<size_t>(total) + 1);
  c.hit_vals.resize(8 * static_cast<size_t>(total) + 8);
  int64_t off = 0;
  for (int q = 0; q < c.world; ++q) {
    if (!cnt[q]) continue;
    const char* pb = static_cast<const char*>(c.peer_win[q]);
    WG_CUDA(cudaMemcpyAsync(c.hit_keys.data() + off, pb + hit_keys_offset(c.win_p), 8 * cnt[q], cudaMemcpyDefault, s));
    WG_CUDA(cudaMemcpyAsync(c.hit_vals.data() + 8 * off, pb + hit_vals_offset(c.win_p), 64 * cnt[q],
                            cudaMemcpyDefault, s));
    off += cnt[q];
  }
  rank_barrier(c);  // no rank refills its hit area while a peer still reads it
  const int64_t n = dedup_hits(c, total);
  c.narrow_pairs = pairs;
  comm_check(c);
  return n;
}

}  // namespace weft_gpu
