// ctx.cuh — the device-resident session behind weft_gpu_ctx.
#pragma once

#include "common.cuh"

namespace weft_gpu {

// Sliced-ELL (SELL-32) 3x3-block matrix. Slot k of row r lives at
// slice_off[r/32] + 32*k + r%32 (column words); its nine block components
// sit at vidx(at, r%32, q): per (slice, slot) nine 256-byte component
// chunks, i.e. the reference's nine SoA value planes
// (proj/include/weft/bell.hpp:61-79) re-laid slot-major per warp of rows so
// each load instruction moves 256 contiguous bytes and a slice is one
// sequential stream. Per row, slots are
// ordered by accumulation group (own partition first, then the work-queue
// order) and by ascending column within a group; the group position is
// packed in bits 28..30 of the column word.
struct SellMatrix {
  int rows = 0;       // block rows held (the rank's rows)
  int row0 = 0;       // global index of the first held row
  int nslices = 0;
  int64_t total = 0;  // slots incl. padding
  int64_t nnzb = 0;
  int max_len = 0;
  DBuf<int64_t> slice_off;  // nslices + 1
  DBuf<int32_t> rowlen;     // rows, by matrix position
  // SELL-32-sigma: matrix position m holds local row perm[m]; rows are
  // sorted by descending length inside windows of kSigma rows (aligned to
  // partition starts), so a slice's rows have (nearly) equal lengths and
  // no padding is streamed. Per-row slot order is untouched.
  DBuf<int32_t> perm;       // rows
  DBuf<int32_t> pos;        // rows: local row -> matrix position
  DBuf<int32_t> colp;       // total: column words as positions (one-partition persistent PCG)
  int64_t layout_id = 0;    // bumped whenever the layout changes
  int64_t colp_id = -1;     // layout colp was built for
  DBuf<int16_t> colp16;     // total: colp as offsets from the row position (when all fit 16 bits)
  bool colp16_ok = false;   // ... for the layout colp_id
  DBuf<int32_t> pair_at;    // total: slot of each lower block's transposed twin, -1 none (layout pair_id)
  int64_t pair_id = -1;
  DBuf<uint32_t> mwords;    // total: column offset | twin slot delta of blocks bitwise equal to it (per solve)
  DBuf<int32_t> cols;       // total (packed col | group << 28; -1 padding)
  DBuf<double> vals;        // 9 * total
  DBuf<float> vals32;       // 9 * total: the values of a Precision::Single system
  bool f32 = false;         // the system is single precision (vals32 holds the values)
};

constexpr int kColMask = 0x0FFFFFFF;
constexpr int kSigma = 256;         // sorting window of the SELL-32-sigma layout
constexpr int kSigmaContacts = 512; // ... of a system with contact elements (longer rows to group)

// Value index of component q (row-major 3x3) of the slot at column-index
// position `at` of a row with lane = row % 32: the nine components of one
// slot of a 32-row slice are nine consecutive 256-byte chunks, so a warp
// walking its rows' slot k streams one contiguous 2304-byte record.
__host__ __device__ __forceinline__ int64_t vidx(int64_t at, int lane, int q) {
  return 9 * (at - lane) + 32 * q + lane;
}
constexpr int kGroupShift = 28;

struct PcgState;  // device scalars, see pcg.cu

struct Ctx {
  int device = 0;
  int nparts = 1;
  int part_begin = 0, part_end = 1;
  // Rank group (one process per GPU): this context owns partitions
  // [part_begin, part_end) = global rows [row0, row1); world ranks own
  // equal contiguous partition ranges. world == 1: everything local.
  int world = 1, rank = 0;
  int row0 = 0, row1 = 0;
  void* win = nullptr;          // own peer-visible window (cudaMalloc, IPC-exported)
  size_t win_bytes = 0;
  int win_p = 0;                // vertex count the window was sized for
  void* peer_win[kMaxRanks] = {};  // mapped peer windows (own = win)
  bool attached = false;
  DBuf<unsigned long long> seq;    // [0] vec, [1] red, [2] state, [3] error
  CommView comm;                   // kernel view (valid once attached)
  cudaStream_t stream = nullptr;
  // side stream: the DCD broad phase runs on it concurrently with the
  // assembly (independent work, both latency-bound); `cur` is the stream
  // library launches currently go to (ls()).
  cudaStream_t side = nullptr;
  cudaStream_t cur = nullptr;
  cudaEvent_t ev[8] = {};
  cudaEvent_t ev_side[4] = {};

  // ---- vertices / partitions
  int p = 0;
  PartMap pm;
  GroupOrder go;
  std::vector<int> queue_vec;  // n*(n-1)
  DBuf<double> mass;
  DBuf<uint8_t> pinned;

  // ---- elements (static list followed by per-step contacts)
  int64_t n_static = 0, n_contacts = 0;
  DBuf<int4> est;         // stencil per element (-1 padded)
  DBuf<int2> einfo;       // (kind | stencil_size << 8, payload offset)
  DBuf<double> edamp;     // element damping
  DBuf<double> epay;      // payload pool
  int64_t static_pay = 0;  // payload doubles used by static elements
  DBuf<int32_t> eres_off;  // per element: offset of its results in eres
  DBuf<double> eres;       // phase-1 results (rhs contributions + state)
  DBuf<int64_t> elist;     // rank group: ids of the elements coupled to held rows
  struct KindRun {
    int kind;
    int64_t begin, end;
  };
  std::vector<KindRun> kind_runs;  // same-kind runs of the static list
  int64_t static_res = 0;
  // static row incidences: per row, (element*4 + a) ascending element
  DBuf<int64_t> inc_ptr;  // p + 1
  DBuf<int32_t> inc;
  // static pattern: per row ascending columns (CSR)
  DBuf<int64_t> spat_ptr;  // p + 1
  DBuf<int32_t> spat;
  int static_max_len = 0;
  // contact incidences (rebuilt per step)
  DBuf<int64_t> cinc_ptr;  // p + 1
  DBuf<int32_t> cinc;      // (contact index * 4 + a), ascending contact
  bool have_pattern_for_contacts = false;

  // ---- assembled / loaded system
  SellMatrix A;
  DBuf<double> rhs;
  bool has_matrix = false;
  bool has_rhs = false;

  // ---- vectors of the current step (3p doubles)
  DBuf<double> x_cur, x_adv, vel;

  // ---- PCG work
  DBuf<double> r, z, pv, q, xs, dinv, bvec;
  DBuf<double> xp;  // persistent PCG: solution in position space
  DBuf<double> dinv6;  // persistent PCG: packed symmetric block-Jacobi inverses
  DBuf<unsigned long long> timing;  // dev instrumentation of the persistent PCG
  DBuf<double> partials;
  DBuf<double> hist, phist;
  PcgState* pcg = nullptr;       // device
  void* pcg_host = nullptr;      // pinned mirror
  DBuf<unsigned char> pcg_args;  // device PcgArgs
  bool use_graphs = true;        // whole-solve CUDA graph (conditional WHILE)
  cudaGraphExec_t pcg_exec = nullptr;
  int pcg_exec_blocks = 0;
  bool pcg_exec_single = false;
  bool pcg_exec_pair = false;
  bool spmv_pair = false;  // two threads per row SpMV variant (WEFT_SPMV_PAIR=1)
  bool use_persistent = true;  // one-partition solves: one cooperative kernel (WEFT_PCG_PERSISTENT=0: graph)
  DBuf<double> p2;             // its second search-direction buffer
  DBuf<double> z4, p4a, p4b;   // its z / p at 32 bytes per row (WEFT_PK_V4)

  // ---- broad phase
  int soup_verts = 0, soup_tris = 0;
  DBuf<int32_t> tris;          // 3 per triangle
  DBuf<double> box_lo, box_hi; // 3 per triangle
  DBuf<double> diag;           // per triangle
  DBuf<double> cell_size;      // 1
  DBuf<int32_t> lat;           // 6 per triangle
  DBuf<int64_t> ecount;        // per triangle entries (+1 for scan)
  DBuf<uint64_t> keys_a, keys_b;
  DBuf<int32_t> vals_a, vals_b;
  DBuf<uint64_t> cell_keys;
  DBuf<int64_t> cell_off;      // cells + 1
  DBuf<int64_t> wprefix;       // cells + 1
  DBuf<int32_t> cell_flag;
  DBuf<double> sum_approx;
  DBuf<unsigned char> sum_maps;
  int64_t grid_entries = 0, grid_cells = 0, grid_total = 0;
  double grid_cell_size = 0.0;
  DBuf<int64_t> cand_count;
  DBuf<unsigned long long> cand_all;  // unfiltered candidates of a filtered walk
  DBuf<int32_t> cand_pairs;
  bool has_grid = false;

  // ---- narrow phase (narrow.cu)
  DBuf<int2> soup_edges;          // CollisionSoup::edges (sorted vertex pairs)
  DBuf<int32_t> soup_tri_edges;   // 3 edge ids per triangle
  DBuf<uint8_t> soup_movable;     // per soup vertex
  DBuf<unsigned long long> hit_count, hit_keys, hit_keys_sorted, contact_keys;
  DBuf<double> hit_vals, contact_vals;  // 8 per hit: gap | toi, normal, weights
  DBuf<long long> hit_counts;           // rank group: every rank's hit / pair counts
  DBuf<int64_t> hit_idx, hit_idx_sorted, hit_flag;
  int64_t n_contacts_found = 0, narrow_pairs = 0, narrow_raw_hits = 0;
  DBuf<int> contact_active;      // proximities_to_elements: active count per vertex
  DBuf<int64_t> contact_flag;    // per proximity: element flag, then position

  // ---- persistent scratch of the pattern / layout builds (they run every
  // step in contacts mode: no cudaMalloc / cudaFree per step)
  DBuf<int> sc_inc_cnt, sc_pat_cnt;
  DBuf<uint32_t> sc_inc_k1, sc_inc_k2;
  DBuf<int32_t> sc_inc_v1, sc_lay_ccol, sc_lay_len, sc_sigma_w;
  DBuf<int64_t> sc_pat_pc, sc_pat_nsel, sc_lay_cptr, sc_lay_red, sc_sel_cnt;
  DBuf<uint64_t> sc_pat_k1, sc_pat_k2;
  DBuf<uint8_t> sc_sel_flag;

  // ---- small device->host reads through mapped pinned memory (read_small)
  void* map_host = nullptr;
  void* map_dev = nullptr;

  // ---- CUB scratch (one per stream)
  DBuf<unsigned char> scratch;
  DBuf<unsigned char> scratch_side;
  DBuf<int64_t> scalars;  // small device scratch

  // ---- instrumentation
  bool instrument = false;        // record the reference's solver event lines
  std::string log;                // ... here (weft_gpu_take_log)
  int64_t launches = 0;           // kernels of this library launched so far
  bool profile = false;           // time every PCG SpMV launch with events
  int64_t spmv_launches = 0;      // PCG SpMV launches timed
  double spmv_ms = 0.0;           // their summed device time
  int64_t pcg_solves = 0;         // persistent solves timed while profiling
  int64_t pcg_iterations = 0;     // their iterations
  double pcg_ms = 0.0;            // their summed device time
  double pcg_bytes = 0.0;         // their summed algorithmic bytes
  int64_t pcg_mirrored = 0;       // blocks the last mirrored persistent solve read from their twins
  std::vector<cudaEvent_t> prof_ev;

  // ---- resident simulation state
  DBuf<double> sim_x, sim_v, sim_xc;  // soup-sized: the cloth's 3p, then obstacle vertices
  DBuf<double> sim_vbak;              // v at the step's start: restored when a step fails after v += dv
  DBuf<double> soup_mass;             // cloth masses, 1.0 for obstacle vertices
  bool has_state = false;
  bool obstacles_set = false;         // obstacle positions of this step given
  // weft_gpu_sim_step_io: the step's host buffers (null outside that call)
  const double* io_vin = nullptr;
  double* io_xout = nullptr;
  double* io_vout = nullptr;

  // impact zones (zones.cu): accumulated impacts, zone structure, solver scratch
  DBuf<unsigned long long> zn_acc_keys, zn_acc_sorted, zn_tmp_keys;
  DBuf<double> zn_acc_vals;
  DBuf<int64_t> zn_flag;
  DBuf<int32_t> zn_part_v, zn_owner, zn_parent, zn_zone_of, zn_zone_of_sorted, zn_iota, zn_zimp, zn_zimp_off;
  DBuf<double> zn_part_w;
  DBuf<unsigned long long> zn_vkeys, zn_vkeys_sorted, zn_ikeys, zn_ikeys_sorted;
  DBuf<int32_t> zn_voff, zn_ioff;
  DBuf<double> zn_cn, zn_lam, zn_force, zn_tc, zn_tv, zn_grad, zn_saved, zn_prop, zn_pre;
  DBuf<int32_t> zn_fail;
  DBuf<float4> zn_tbox;  // narrow phase: conservative float triangle boxes
  DBuf<double> zn_dbox;  // narrow phase: exact triangle boxes (6 per triangle)
  DBuf<double> zn_vbox;  // narrow phase: exact vertex boxes (6 per vertex)
  DBuf<unsigned long long> cand_cursor;  // append-mode candidate walk: pairs claimed
  DBuf<int4> zn_feats;                  // two-pass narrow phase: surviving features (2 int4 each)
  DBuf<unsigned long long> zn_feat_count;
  int64_t zn_m = 0;      // accumulated impacts
  int32_t zn_nz = 0;     // zones of the last build
  int64_t zn_nzv = 0;    // zone vertices of the last build
};

// Engine::log_line (exec.cpp:176-180) while instrumentation is on.
inline void log_line(Ctx& c, const std::string& line) {
  if (c.instrument) c.log += line + "\n";
}
// ostream << double with the default format (precision 6, %g).
inline std::string fmt_g(double v) {
  char b[64];
  std::snprintf(b, sizeof(b), "%g", v);
  return b;
}

// Launch-site stream accessor: counts the launch (gpu_launches in bench.py).
inline cudaStream_t ls(Ctx& c) {
  ++c.launches;
  return c.cur;
}

// ---- entry points implemented across the .cu files
void set_matrix_csr(Ctx& c, int rows, const int64_t* row_ptr, const int32_t* cols, const double* vals);
// Window starts (local rows) of the sigma sort: partition-aligned chunks.
std::vector<int32_t> sigma_windows(const Ctx& c, int win = kSigma);
// Device sigma layout from per-row lengths (local row order): fills A.perm,
// A.pos and A.rowlen (by position).
void build_sigma(Ctx& c, const int32_t* len_row);
void spmv(Ctx& c, const double* x_dev, double* y_dev);
// Precision::Single (driver.hpp:13): float systems on one rank
void spmv_f32(Ctx& c, const float* x_dev, float* y_dev);
void set_matrix_csr_f32(Ctx& c, int rows, const int64_t* row_ptr, const int32_t* cols, const float* vals);
void narrow_to_f32(Ctx& c);  // the current double values -> vals32 (exact when they came from floats)
void download_csr(Ctx& c, int64_t* row_ptr, int32_t* cols, double* vals);
void download_csr_f32(Ctx& c, int64_t* row_ptr, int32_t* cols, float* vals);
struct PcgResult {
  int iterations = 0;
  int converged = 0;
  double rel_residual = 0.0;
};
PcgResult pcg_solve(Ctx& c, const double* b_dev, const weft_pcg_config& cfg, double* hist_host,
                    double* phist_host);
void pcg_free(Ctx& c);
PcgResult pcg_solve_f32(Ctx& c, const float* b_dev, const weft_pcg_config& cfg, double* hist_host,
                        double* phist_host);

void set_vertices(Ctx& c, int p, const double* mass, const uint8_t* pinned);
void set_elements(Ctx& c, int64_t count, const weft_element* elems);
void set_contacts(Ctx& c, int64_t count, const weft_element* elems);
// finish = false leaves the final host check (non-positive mass) to
// fill_matrix_finish, so other streams can be fed while the kernels run.
// f32: Precision::Single — AssembledSystem<float> (each contribution cast to
// float and added in float, assembly.hpp:163,196,212), one rank.
void fill_matrix(Ctx& c, const double* xc, const double* xa, const double* vel, double dt, int mode,
                 bool finish = true, bool f32 = false);
void fill_matrix_finish(Ctx& c);

void set_soup(Ctx& c, int verts, int ntris, const int32_t* tris);
void build_grid(Ctx& c, const double* x0_dev, const double* x1_dev, int mode, double thickness, double cell_scale);
// tbox (narrow phase): emit only the candidates whose conservative float
// boxes are within margin (k_narrow's whole-pair rejection); *all gets the
// unfiltered candidate count.
int64_t candidates(Ctx& c, int64_t begin, int64_t end, int32_t* pairs_dev_or_null, bool count_only = false,
                   const float4* tbox = nullptr, double margin = 0.0, int64_t* all = nullptr);

void serial_sum(Ctx& c, int n, const double* d_host, double* exact, double* naive, int fast);

// narrow phase (narrow.cu)
void build_soup_edges(Ctx& c, const std::vector<int32_t>& tris);
void set_soup_movable(Ctx& c, const uint8_t* movable);
int64_t narrow_phase(Ctx& c, const double* x0, const double* x1, int mode, double thickness, int64_t begin,
                     int64_t end);
void download_contacts(Ctx& c, int32_t* kab, double* vals);
// proximities_to_elements on the device (response.cpp:43-106): contact
// elements from the last DCD narrow phase, written after the static list.
constexpr int kContactPay = 16, kContactRes = 13;
struct ContactParamsDev {
  double thickness, stiffness_scale, friction, damping;
};
int64_t contacts_from_proximities(Ctx& c, const double* x, const double* v, double dt, const ContactParamsDev& kp);
void reserve_contacts(Ctx& c, int64_t count);
int32_t build_zones(Ctx& c, const unsigned long long* keys, const double* vals, int64_t m);
void download_zones(Ctx& c, int64_t m, int32_t* impact_zone, int32_t* vert_off, int32_t* verts);
std::vector<std::vector<int>> distribute_zones(const std::vector<int>& sizes, int devices);
void resolve_zones(Ctx& c, const double* xb, double* xcand, const double* mass, double thickness, double cell_scale,
                   const weft_zone_params& zp, weft_zone_report& rep, bool have_first);
void zone_commit(Ctx& c, const double* corrected, const double* pre, double dt, double* v);
void finish_contacts(Ctx& c, int64_t count);

// rank group (comm.cu, sparse.cu)
void set_rows(Ctx& c, int p);  // partition map + this rank's row window
void comm_need(Ctx& c, const char* what);
void comm_check(Ctx& c);
void comm_export(Ctx& c, void* handle_out);
void comm_attach(Ctx& c, const void* handles);
void comm_free(Ctx& c);
void publish_vectors(Ctx& c);  // z/p rows of this rank are final
void rank_barrier(Ctx& c);
void exchange_state(Ctx& c);   // sim: publish own v/x_cand rows, pull the peers'
// collide's merge over ranks: the union of every rank's unique hits
// (contact_keys / contact_vals), sorted and deduplicated, on every rank
int64_t merge_hits(Ctx& c);
// sort + dedup of n raw hits in hit_keys / hit_vals -> contact_keys / vals
int64_t dedup_hits(Ctx& c, int64_t n);
// collide (collision.cpp:391-417): build_grid + the narrow phase of this
// rank's split_workload share, merged over the rank group
int64_t collide(Ctx& c, const double* x0, const double* x1, int mode, double thickness, double cell_scale);

// CUB scratch helper
void* scratch(Ctx& c, size_t bytes);
// Reads up to three small device values (bytes each <= 128) on stream s and
// waits: a one-thread kernel stores them into mapped pinned host memory, so
// the read never queues on a copy engine behind a large transfer (the e2e
// step's 40 MB read-back runs concurrently with the CCD broad phase).
struct SmallRead {
  const void* src;
  void* dst;
  int bytes;
};
void read_small(Ctx& c, cudaStream_t s, SmallRead a, SmallRead b = {}, SmallRead d = {});

}  // namespace weft_gpu

// The opaque handle of the C-ABI.
struct weft_gpu_ctx {
  weft_gpu::Ctx c;
};
