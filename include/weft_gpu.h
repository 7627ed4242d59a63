/*
 * weft_gpu.h — the C-ABI drop-in boundary of the B200-native implicit-
 * integration hot path of P-Cloth (arXiv 2008.00409).
 *
 * The reference engine ("weft", /root/reference/proj) is C++20; its hot path
 * is called from exactly one place per step, Simulator::step_impl
 * (proj/src/driver.cpp:136-161). This header exports plain-C entry points,
 * plain pointers and sizes only, one per reference interface the GPU path
 * replaces (each cited below as file:line of the reference). A C++ caller of
 * the reference keeps its types and calls these through the thin wrapper in
 * paper_2008_00409_b200/host/weft_dropin.hpp.
 *
 * Conventions
 *  - Every entry point returns a weft_status; on failure the message of the
 *    reference's exception (same wording) is available from
 *    weft_gpu_last_error() (thread-local).
 *  - Array arguments may be host or device pointers (cudaMemcpyDefault/UVA);
 *    they are borrowed for the duration of the call. All device state is
 *    owned by the context. Output buffers are caller-allocated; passing NULL
 *    where a size query is documented returns only the size.
 *  - Vectors of vertices are flat doubles, 3 per vertex (x0,y0,z0,x1,...),
 *    the layout of std::vector<Vec3>/DistVector<double> gathered.
 *  - Every call is synchronous on return (Engine::parallel fork-join
 *    semantics, proj/include/weft/exec.hpp:99-101).
 */
#ifndef WEFT_GPU_H
#define WEFT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror the reference's error hierarchy
 * (proj/include/weft/common.hpp:16-47, proj/include/weft/solver.hpp:10-13). */
typedef enum weft_status {
  WEFT_OK = 0,
  WEFT_ERR_DIMENSION = 1, /* weft::DimensionError */
  WEFT_ERR_SOLVER = 2,    /* weft::SolverError    */
  WEFT_ERR_EXEC = 3,      /* weft::ExecError: CUDA/NCCL failure, names the GPU */
  WEFT_ERR_TOPOLOGY = 4,  /* weft::TopologyError  */
  WEFT_ERR_SCHEDULE = 5,  /* weft::ScheduleError  */
  WEFT_ERR_INVALID = 6,   /* invalid argument or call order */
  WEFT_ERR_ZONE = 7       /* weft::ZoneFailure (response.hpp:8-11) */
} weft_status;

/* Message of the last failed call on this thread ("" if none). */
const char* weft_gpu_last_error(void);

/* ---------------------------------------------------------------------- */
/* Element records (proj/include/weft/elements.hpp:11-81)                  */
/* ---------------------------------------------------------------------- */

/* ElementKind, same order as the reference enum (elements.hpp:11). */
enum { WEFT_STRETCH = 0, WEFT_BEND = 1, WEFT_SPRING = 2, WEFT_EXTERNAL = 3, WEFT_CONTACT = 4 };
/* JacobianMode (elements.hpp:13-16). */
enum { WEFT_JAC_EXACT = 0, WEFT_JAC_SPD_PROJECTED = 1 };

/* Flat AssemblyElement (elements.hpp:71-77); `data` holds the variant
 * payload of the element's kind:
 *   STRETCH  (StretchData, :20-27): pwu[0..2] pwv[3..5] area[6] k_warp[7]
 *                                   k_weft[8] k_shear[9]
 *   BEND     (BendData, :30-33):    rest_angle[0] stiffness[1]
 *   SPRING   (SpringData, :35-38):  rest_length[0] stiffness[1]
 *   EXTERNAL (ExternalData, :40-43): force[0..2] drag[3]
 *   CONTACT  (ContactData, :51-62): normal[0..2] w[3..6] bias[7]
 *             activation[8] stiffness[9] friction[10] tangential_damping[11]
 *             frozen_normal_force[12] rel_vel_bias[13..15]
 */
typedef struct weft_element {
  int32_t kind;
  int32_t stencil_size;
  int32_t stencil[4];
  double damping;
  double data[18];
} weft_element;

/* ---------------------------------------------------------------------- */
/* Context                                                                */
/* ---------------------------------------------------------------------- */

typedef struct weft_gpu_ctx weft_gpu_ctx;

typedef struct weft_gpu_options {
  int32_t cuda_device; /* CUDA ordinal this context runs on */
  /* Logical row partitions n: the reference's Engine(n)/make_partitions
   * (proj/src/exec.cpp:10-23). Fixes the SpMV accumulation order
   * (proj/include/weft/sparse.hpp:72-101) and the dot-product reduction
   * order (proj/src/exec.cpp:170-174). n must be a power of two when > 1
   * (proj/src/topology.cpp:7-11). */
  int32_t partitions;
  /* Partitions [part_begin, part_end) are resident on this GPU; the rest
   * live on peer ranks (multi-process). Single-process: 0 and partitions. */
  int32_t part_begin;
  int32_t part_end;
} weft_gpu_options;

/* Creates a context (replaces Engine construction, exec.cpp:145-148). */
weft_status weft_gpu_create(const weft_gpu_options* opts, weft_gpu_ctx** out);
weft_status weft_gpu_destroy(weft_gpu_ctx* ctx);

/* ---------------------------------------------------------------------- */
/* Rank group: one process per GPU (replaces the in-process interconnect  */
/* of Engine::run_pipelined / all_reduce_sum, proj/src/exec.cpp:170-307)   */
/* ---------------------------------------------------------------------- */

/* A context whose partition range [part_begin, part_end) is a proper subset
 * of [0, partitions) is one rank of a group: ranks own equal contiguous
 * partition ranges (rank = part_begin / (part_end - part_begin)), hold only
 * their rows of the matrix, assemble only their rows, and exchange halo
 * vectors, reduction partials and state rows through peer memory.
 * Protocol: every rank calls weft_gpu_set_vertices (or weft_gpu_set_matrix),
 * then weft_gpu_comm_export, shares the handle bytes with all ranks (any
 * transport, e.g. torch.distributed.all_gather_object), then
 * weft_gpu_comm_attach with all handles in rank order. Afterwards every
 * collective entry point (spmv, pcg, sim_step) must be called by all ranks
 * in the same order. Destroy only after a host barrier. */
enum { WEFT_IPC_HANDLE_BYTES = 64 };
weft_status weft_gpu_comm_export(weft_gpu_ctx* ctx, void* handle_out /* WEFT_IPC_HANDLE_BYTES */);
weft_status weft_gpu_comm_attach(weft_gpu_ctx* ctx, const void* handles /* world * WEFT_IPC_HANDLE_BYTES */);
typedef struct weft_rank_info {
  int32_t world, rank;
  int32_t first_row, rows; /* global block rows [first_row, first_row + rows) held here */
  int32_t global_rows;
} weft_rank_info;
weft_status weft_gpu_rank_info(weft_gpu_ctx* ctx, weft_rank_info* info);

/* ---------------------------------------------------------------------- */
/* Partitions and schedule (proj/src/exec.cpp:10-27, proj/src/topology.cpp)*/
/* ---------------------------------------------------------------------- */

/* Hinge angle probes (tests and tools). The reference's hinge angle is
 * std::atan2(s, c) (proj/src/elements.cpp:116); the library evaluates it as
 * a correctly rounded double atan2 (csrc/cr_atan2.cuh). _host runs the same
 * code compiled for the CPU; the _gpu variant runs it on the context's
 * device (x, y, out host or device pointers). */
weft_status weft_hinge_atan2_host(int64_t n, const double* y, const double* x, double* out);
weft_status weft_gpu_hinge_atan2(weft_gpu_ctx* ctx, int64_t n, const double* y, const double* x, double* out);
/* make_partitions (exec.cpp:10-23): begin/end arrays of length `devices`. */
weft_status weft_make_partitions(int32_t vertex_count, int32_t devices, int32_t* begin, int32_t* end);
/* generate_work_queues(FatTree::make(n)) (topology.cpp:79-89): for device
 * d, node k: peer[d*(n-1)+k], vec[d*(n-1)+k]. */
weft_status weft_work_queues(int32_t devices, int32_t* peer, int32_t* vec);

/* ---------------------------------------------------------------------- */
/* Sparse matrix + SpMV (proj/include/weft/bell.hpp, sparse.hpp)          */
/* ---------------------------------------------------------------------- */

/* Loads a global 3x3-block matrix given as block CSR with ascending columns
 * per row, values row-major per block (9 doubles). Equivalent of
 * partition_matrix(global, make_partitions(rows, n)) (sparse.hpp:103-147). */
weft_status weft_gpu_set_matrix(weft_gpu_ctx* ctx, int32_t block_rows, const int64_t* row_ptr,
                                const int32_t* cols, const double* vals);

/* y = A x with the pipelined order of spmv_pipelined (sparse.hpp:72-101):
 * per row the own-partition sub-block sum first, then the other sub-blocks
 * in work-queue order. x, y: 3*global_rows doubles. Bitwise equal to
 * oracle::spmv_partitioned_serial (src/oracle/sparse_oracle.hpp:12-42).
 * In a rank group only this rank's rows of x are read (the others are
 * gathered from their owners) and only its rows of y are written. */
weft_status weft_gpu_spmv(weft_gpu_ctx* ctx, const double* x, double* y);

/* Matrix shape of the context's current system (assembled or loaded). */
typedef struct weft_matrix_info {
  int32_t block_rows;
  int32_t max_row_blocks; /* widest compacted row */
  int64_t nnzb;           /* live blocks */
  int64_t padded_slots;   /* device storage slots (sliced-ELL) */
} weft_matrix_info;
weft_status weft_gpu_matrix_info(weft_gpu_ctx* ctx, weft_matrix_info* info);

/* Downloads the current system as block CSR, ascending columns
 * (gather_matrix, sparse.hpp:149-173): all rows, or this rank's rows in a
 * rank group (weft_gpu_rank_info). Any pointer may be NULL. */
weft_status weft_gpu_download_matrix(weft_gpu_ctx* ctx, int64_t* row_ptr, int32_t* cols, double* vals);
/* Downloads the assembled right-hand side of the held rows
 * (3*block_rows doubles). */
weft_status weft_gpu_download_rhs(weft_gpu_ctx* ctx, double* rhs);

/* ---------------------------------------------------------------------- */
/* PCG (proj/include/weft/solver.hpp:15-178)                              */
/* ---------------------------------------------------------------------- */

enum { WEFT_PRECOND_NONE = 0, WEFT_PRECOND_BLOCK_JACOBI = 1 }; /* solver.hpp:15 */

typedef struct weft_pcg_config { /* PcgConfig, solver.hpp:17-21 */
  double rel_tolerance;          /* default 1e-4 */
  int32_t max_iterations;        /* default 400 */
  int32_t preconditioner;        /* default WEFT_PRECOND_BLOCK_JACOBI */
} weft_pcg_config;

typedef struct weft_pcg_report { /* PcgReport, solver.hpp:23-29 */
  int32_t iterations;
  int32_t converged;
  double rel_residual;
  /* Optional histories (length >= max_iterations, may be NULL): */
  double* residual_history;
  double* precond_norm_history;
} weft_pcg_report;

/* Solves A x = b for the context's current matrix (pcg_solve,
 * solver.hpp:36-178). b may be NULL to use the assembled rhs. x receives the
 * solution (3*global_rows doubles; NULL keeps it on the device). In a rank
 * group b and x are full-length, only this rank's rows are read/written,
 * and the result is bitwise that of one context with the same partitions. Returns
 * WEFT_ERR_SOLVER with the reference's message on non-finite/non-positive
 * curvature or divergence; non-convergence is only flagged. */
weft_status weft_gpu_pcg(weft_gpu_ctx* ctx, const double* b, double* x, const weft_pcg_config* config,
                         weft_pcg_report* report);

/* Precision::Single (driver.hpp:13, Real = float; one rank): the same entry
 * points over float values — BellMatrix<float> and spmv_serial /
 * spmv_pipelined<float> (bell.cpp:87-129, float products and sums in the
 * same order), pcg_solve<float> (solver.hpp:36-178: float vectors, double
 * dot products and block-Jacobi inverses, alpha / beta cast to float). */
weft_status weft_gpu_set_matrix_f32(weft_gpu_ctx* ctx, int32_t block_rows, const int64_t* row_ptr,
                                    const int32_t* cols, const float* vals);
weft_status weft_gpu_spmv_f32(weft_gpu_ctx* ctx, const float* x, float* y);
weft_status weft_gpu_pcg_f32(weft_gpu_ctx* ctx, const float* b, float* x, const weft_pcg_config* config,
                             weft_pcg_report* report);
weft_status weft_gpu_download_matrix_f32(weft_gpu_ctx* ctx, int64_t* row_ptr, int32_t* cols, float* vals);
/* fill_matrix<float> / step_system<float> (assembly.hpp:74-220 and
 * physics.hpp:44-69 with Real = float: each contribution computed in double,
 * cast to float, added in float) and the float rhs. */
weft_status weft_gpu_fill_matrix_f32(weft_gpu_ctx* ctx, const double* x_cur, const double* x_adv,
                                     const double* velocity, double dt, int32_t jac_mode);
weft_status weft_gpu_step_system_f32(weft_gpu_ctx* ctx, const double* x, const double* v, double dt,
                                     int32_t jac_mode);
weft_status weft_gpu_download_rhs_f32(weft_gpu_ctx* ctx, float* rhs);

/* ---------------------------------------------------------------------- */
/* Assembly (proj/include/weft/assembly.hpp:48-220, physics.hpp:44-69)    */
/* ---------------------------------------------------------------------- */

/* Per-vertex data of SystemInputs (assembly.hpp:51-60): mass, pinned. */
weft_status weft_gpu_set_vertices(weft_gpu_ctx* ctx, int32_t vertex_count, const double* mass,
                                  const uint8_t* pinned);
/* The static element list (build_elements order: triangles, hinges,
 * vertices; physics.cpp:5-63). Precomputes its sparsity contribution. */
weft_status weft_gpu_set_elements(weft_gpu_ctx* ctx, int64_t count, const weft_element* elements);
/* Per-step elements appended after the static list (contacts,
 * physics.hpp:50-52). count may be 0. */
weft_status weft_gpu_set_contacts(weft_gpu_ctx* ctx, int64_t count, const weft_element* contacts);

/* fill_matrix<double> (assembly.hpp:74-220) over static + contact
 * elements: rebuilds the sparsity pattern and values of
 * A = M - (dt^2 + c dt) J (+ dt D) and rhs = dt f(x_adv) on the device.
 * x_cur, x_adv, velocity: 3*p doubles. jac_mode: WEFT_JAC_*. */
weft_status weft_gpu_fill_matrix(weft_gpu_ctx* ctx, const double* x_cur, const double* x_adv,
                                 const double* velocity, double dt, int32_t jac_mode);

/* step_system<double> (physics.hpp:44-69): x_adv = x + dt v computed on
 * the device, then fill_matrix. */
weft_status weft_gpu_step_system(weft_gpu_ctx* ctx, const double* x, const double* v, double dt,
                                 int32_t jac_mode);

/* ---------------------------------------------------------------------- */
/* Spatial-hash broad phase (proj/src/collision.cpp:77-192,205-210,329-378)*/
/* ---------------------------------------------------------------------- */

enum { WEFT_DISCRETE = 0, WEFT_CONTINUOUS = 1 }; /* CollisionMode, collision.hpp:18 */

/* Static soup topology (CollisionSoup::build, collision.cpp:95-116). */
weft_status weft_gpu_set_soup(weft_gpu_ctx* ctx, int32_t vertex_count, int32_t tri_count,
                              const int32_t* tris);

/* build_grid (collision.cpp:118-179) on the device. x_end is ignored in
 * Discrete mode. Bit-exact with the reference: cell size from the serial
 * diagonal sum, lattice boxes, cell keys, per-cell triangle lists and
 * workload prefix. */
weft_status weft_gpu_build_grid(weft_gpu_ctx* ctx, const double* x_begin, const double* x_end,
                                int32_t mode, double thickness, double cell_scale);

typedef struct weft_grid_info {
  double cell_size;
  int64_t cells;   /* occupied cells */
  int64_t entries; /* (cell, triangle) memberships */
  int64_t total;   /* WorkloadTable::total, sum of c(c-1)/2 */
} weft_grid_info;
weft_status weft_gpu_grid_info(weft_gpu_ctx* ctx, weft_grid_info* info);

/* HashGrid + WorkloadTable (collision.hpp:59-70) as flat arrays; any may be
 * NULL. cell_offsets/prefix have cells+1 entries; tri_boxes 6 per triangle
 * (lo xyz, hi xyz inclusive). */
weft_status weft_gpu_download_grid(weft_gpu_ctx* ctx, uint64_t* cell_keys, int64_t* cell_offsets,
                                   int32_t* cell_tris, int64_t* prefix, int64_t* tri_boxes);

/* Candidate triangle pairs of the flattened pair range [begin, end)
 * (narrow_phase_range's walk + min-common-cell rule, collision.cpp:
 * 329-378): each lattice-overlapping pair t1 < t2 exactly once across all
 * ranges. pairs: 2 int32 per candidate, in walk order. pairs == NULL ->
 * count only. */
weft_status weft_gpu_candidates(weft_gpu_ctx* ctx, int64_t begin, int64_t end, int64_t* count,
                                int32_t* pairs);

/* Narrow phase (collision.cpp:214-309, collision_geom.cpp:35-317). The soup
 * edge table (CollisionSoup::build, collision.cpp:95-116) is built by
 * weft_gpu_set_soup; movable flags default to all movable (NULL resets). */
weft_status weft_gpu_set_soup_movable(weft_gpu_ctx* ctx, const uint8_t* movable);

/* collide (collision.cpp:391-417): build_grid, the candidate walk and the
 * elementary DCD (vertex-face / edge-edge proximity within `thickness`) or
 * CCD (coplanarity cubic + bisection, earliest contact) tests of every
 * candidate pair, merged, sorted and deduplicated by (kind, a, b) like
 * sync_shared_cells. VertexFace: a = vertex, b = triangle, weights = (1,
 * bary0..2); EdgeEdge: a < b edge ids, weights = (1-s, s, 1-t, t). The
 * result stays on the device; *count = number of hits. In a rank group each
 * rank returns the hits of its split_workload share. */
weft_status weft_gpu_collide(weft_gpu_ctx* ctx, const double* x_begin, const double* x_end, int32_t mode,
                             double thickness, double cell_scale, int64_t* count);
/* The last collide result: kind_ab = 3 int32 per hit (kind 0 = VertexFace,
 * 1 = EdgeEdge, a, b); vals = 8 doubles per hit (gap or toi, normal xyz,
 * weights 0..3). Either pointer may be NULL. */
weft_status weft_gpu_download_contacts(weft_gpu_ctx* ctx, int32_t* kind_ab, double* vals);

/* ---------------------------------------------------------------------- */
/* Impact zones (proj/src/response.cpp:108-400)                           */
/* ---------------------------------------------------------------------- */

typedef struct weft_zone_params { /* ZoneSolveParams, response.hpp:46-60 */
  double clearance;               /* h' (Simulator: clearance_fraction * thickness) */
  double initial_penalty;         /* mu, in units of the mean zone vertex mass */
  double inner_tolerance;
  int32_t al_iterations;
  int32_t inner_iterations;
  int32_t outer_cap;
  int32_t retry_cap;
  double max_correction_factor;
} weft_zone_params;

typedef struct weft_zone_report { /* ZoneResolveReport, response.hpp:62-68 */
  int32_t outer_iterations;
  int32_t zone_count;
  int32_t max_zone_vertices;
  int64_t impacts_resolved;
  int64_t first_round_impacts;
} weft_zone_report;

/* build_zones (response.cpp:108-162) over n impacts given as (kind, a, b)
 * triples on the soup set with weft_gpu_set_soup (+ set_soup_movable):
 * connected components of the impact graph (impacts adjacent iff they share
 * a participant vertex), zones numbered by their first impact.
 * impact_zone: n int32 (may be NULL); *zone_count; *vertex_total = movable
 * zone vertices over all zones. Fetch the vertex lists with
 * weft_gpu_zone_vertices. */
weft_status weft_gpu_build_zones(weft_gpu_ctx* ctx, int64_t n, const int32_t* kind_ab, int32_t* impact_zone,
                                 int32_t* zone_count, int64_t* vertex_total);
/* The last build_zones: vert_off = zone_count + 1 offsets into verts
 * (each zone's movable vertices, ascending). */
weft_status weft_gpu_zone_vertices(weft_gpu_ctx* ctx, int32_t* vert_off, int32_t* verts);
/* distribute_zones (response.cpp:164-182): device_of[z] for zones of the
 * given vertex counts (greedy, descending size, least-loaded device). */
weft_status weft_distribute_zones(int32_t zone_count, const int32_t* sizes, int32_t devices, int32_t* device_of);
/* resolve_zones (response.cpp:338-400) on the soup set with set_soup (+
 * set_soup_movable): CCD over x_begin -> x_candidate, impact zones built and
 * solved (augmented Lagrangian, Armijo gradient descent) until clean.
 * x_candidate (3 * soup vertices, host or device) is updated in place;
 * vertex_mass has one entry per soup vertex. WEFT_ERR_ZONE with the
 * reference's message when the outer cap is reached or a zone diverges. */
weft_status weft_gpu_resolve_zones(weft_gpu_ctx* ctx, const double* x_begin, double* x_candidate,
                                   const double* vertex_mass, double thickness, double cell_scale,
                                   const weft_zone_params* params, weft_zone_report* report);

/* split_workload (collision.cpp:181-192). */
weft_status weft_split_workload(int64_t total, int32_t devices, int64_t* begin, int64_t* end);

/* ---------------------------------------------------------------------- */
/* Device-resident hot-path step (Simulator::step_impl stages 1-4 + CCD   */
/* broad phase, proj/src/driver.cpp:96-215, without narrow phase/zones)   */
/* ---------------------------------------------------------------------- */

typedef struct weft_sim_params {
  double dt;
  double thickness;  /* CollisionParams::thickness */
  double cell_scale; /* CollisionParams::cell_scale */
  weft_pcg_config pcg;
  int32_t jac_mode;
  /* 1: Simulator::step_impl stages 1-2 in full (driver.cpp:132-149): the DCD
   * narrow phase, proximities_to_elements (response.cpp:43-106) on the
   * device and the contact elements assembled with the static ones; the CCD
   * narrow phase counts impacts (impact zones are not resolved). A rank group
   * narrow-phases its split_workload shares and merges the hits over peer
   * memory (collision.cpp:405-417). 0: the hot-path step (candidate pairs
   * counted, no contacts). */
  int32_t contacts;
  double stiffness_scale; /* ContactParams (response.hpp:13-21); contact thickness = thickness */
  double friction;
  double contact_damping;
  /* contacts mode only — 1: resolve_zones after the CCD (driver.cpp:181-191)
   * and the commit's velocity correction (:195-204): the full step_impl. */
  int32_t zones;
  weft_zone_params zone;
  /* SimConfig::precision (driver.hpp:13,35): 0 = Precision::Double, 1 =
   * Precision::Single — step_impl<float> (driver.cpp:92-94): the system
   * assembled as AssembledSystem<float>, pcg_solve<float>, v += double(dv).
   * One rank. */
  int32_t precision;
} weft_sim_params;

typedef struct weft_step_report {
  int32_t pcg_iterations;
  int32_t pcg_converged;
  double pcg_residual;
  int64_t dcd_candidates;
  int64_t ccd_candidates;
  double ms_broad;    /* device time of both broad phases (the DCD one runs on a
                         side stream, overlapped with the assembly) */
  double ms_assemble; /* device time of fill_matrix */
  double ms_solve;    /* device time of the PCG */
  int64_t proximities;      /* contacts mode: DCD hits */
  int64_t contact_elements; /* contacts mode: elements built from them */
  int64_t impacts;          /* contacts mode: CCD hits (first round) */
  int32_t zone_count;       /* zones mode: zones over all outer rounds */
  int32_t zone_outer;       /* zones mode: outer rounds */
  double ms_zones;          /* zones mode: device time of resolve_zones */
  int32_t stages;           /* stages of Simulator::step_impl run, in canonical_stage_order
                               (driver.cpp:49-53): proximity_dcd, assemble, solve, candidate,
                               ccd, zones, commit — 7 for a committed zones-mode step */
} weft_step_report;

/* Uploads the state (x, v: 3*p doubles each; the soup positions of the
 * cloth are x). Requires vertices, elements and soup to be set. */
weft_status weft_gpu_sim_set_state(weft_gpu_ctx* ctx, const double* x, const double* v);
/* Kinematic obstacles (driver.cpp:113-131): when the soup holds vertices
 * beyond the cloth's p (obstacle triangles appended after the cloth's, ids
 * offset by p, set_soup_movable 0 for them), their positions at the step's
 * start and end (Obstacle::positions_at(t), positions_at(t + dt); 3 doubles
 * per obstacle vertex) must be given before every weft_gpu_sim_step; their
 * velocities are (end - begin) / dt and their masses 1.0. */
weft_status weft_gpu_sim_set_obstacles(weft_gpu_ctx* ctx, double dt, const double* x_begin, const double* x_end);
/* One step on device-resident state: DCD grid + candidates on x, assembly
 * of step_system at x, PCG, v += dv, x_cand = x + dt v, CCD grid +
 * candidates on (x, x_cand), commit x = x_cand. */
weft_status weft_gpu_sim_step(weft_gpu_ctx* ctx, const weft_sim_params* params, weft_step_report* report);
/* One step with the state in host buffers (the e2e path of a caller that
 * keeps x, v on the host): uploads x_in, v_in, steps, and writes x_out, v_out
 * — equivalent to sim_set_state + sim_step + sim_get_state (same results),
 * with the v upload hidden behind the DCD broad phase and the read-back behind
 * the CCD broad phase (one rank, no obstacles; otherwise exactly that
 * sequence). Requires a prior weft_gpu_sim_set_state. */
weft_status weft_gpu_sim_step_io(weft_gpu_ctx* ctx, const double* x_in, const double* v_in,
                                 const weft_sim_params* params, double* x_out, double* v_out,
                                 weft_step_report* report);
/* Reads the state back (either pointer may be NULL). */
weft_status weft_gpu_sim_get_state(weft_gpu_ctx* ctx, double* x, double* v);

/* ---------------------------------------------------------------------- */
/* Instrumentation (bench.py)                                             */
/* ---------------------------------------------------------------------- */

typedef struct weft_gpu_stats_t {
  int64_t launches;       /* kernels of this library launched by the context */
  int64_t spmv_launches;  /* SpMV launches timed while profiling (PCG graph/launch path, weft_gpu_spmv) */
  double spmv_ms;         /* their summed device time (CUDA events) */
  int64_t pcg_solves;     /* persistent PCG kernels timed while profiling */
  int64_t pcg_iterations; /* their iterations */
  double pcg_ms;          /* their summed device time (CUDA events) */
  double pcg_bytes;       /* their summed algorithmic HBM bytes */
} weft_gpu_stats_t;

/* Enables CUDA-event timing of the PCG kernels (resets the counters):
 * each SpMV launch on the multi-kernel path, each whole-solve persistent
 * kernel on the one-partition path. */
weft_status weft_gpu_profile(weft_gpu_ctx* ctx, int32_t enable);
weft_status weft_gpu_stats(weft_gpu_ctx* ctx, weft_gpu_stats_t* out);

/* Engine instrumentation (EngineOptions::instrument, exec.hpp; Engine::log_line
 * exec.cpp:176-180): while on, the library records the event lines the
 * reference writes from inside its solvers, in its format —
 *   "event=pcg iterations=N rel_residual=R converged=C"   (solver.hpp:171-175)
 *   "event=zones outer=K zones=Z fresh=F accumulated=A"   (response.cpp:383-388)
 * weft_gpu_take_log copies the recorded lines (newline-terminated, NUL-ended)
 * into buf and clears them; buf = NULL (or cap too small) only reports the
 * byte count (without the NUL) in *len. Stage lines ("event=stage frame=..")
 * belong to the driver (driver.cpp:104-111): weft_step_report.stages. */
weft_status weft_gpu_set_instrument(weft_gpu_ctx* ctx, int32_t on);
weft_status weft_gpu_take_log(weft_gpu_ctx* ctx, char* buf, int64_t cap, int64_t* len);
/* Test hook for the exact serial-order sum behind build_grid's cell size
 * (collision.cpp:124-133): mean_exact = max(sum/n, 1e-9) from the parallel
 * exact kernel (fast = 1: chunk-map fast path, 0: window scan only),
 * sum_naive = the same sum by one GPU thread, left to right. */
weft_status weft_gpu_test_serial_sum(weft_gpu_ctx* ctx, int32_t n, const double* d, int32_t fast,
                                     double* mean_exact, double* sum_naive);
/* The cudaStream_t all of the context's work is issued on. */
weft_status weft_gpu_get_stream(weft_gpu_ctx* ctx, void** stream);

#ifdef __cplusplus
}
#endif

#endif /* WEFT_GPU_H */
