/*
 * weft_oracle.h — CPU restatement of the reference's hot-path algorithms.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the B200 path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it, and only to check or time the reference algorithm — never as the
 * thing measured or shipped. The product (paper_2008_00409_b200) never links
 * it and fails loudly when its CUDA library is missing.
 *
 * Every function cites the reference file:line it restates. Floating-point
 * association follows the reference compiled against oracle/shim/Eigen/Dense
 * (strict left-to-right 3-term reductions, no FMA: build with
 * -ffp-contract=off). The restatement is pinned bit-for-bit against the
 * reference itself (oracle/_ref/libweft_ref.so, built from the unmodified
 * sources by `make -C oracle ref`) in tests/test_oracle_vs_ref.py, and the
 * reference passes its own 96 doctest cases against the same shim.
 */
#ifndef WEFT_ORACLE_H
#define WEFT_ORACLE_H

#include <stdint.h>

#include "../include/weft_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- partitions / schedule (exec.cpp:10-27, topology.cpp:34-89) ---- */
void orc_make_partitions(int32_t p, int32_t n, int32_t* begin, int32_t* end);
int32_t orc_owner(int32_t p, int32_t n, int32_t v); /* PartitionMap::owner, assembly.hpp:27-31 */
/* peer/vec: n*(n-1) entries, queue of device d at d*(n-1). Returns 0 or -1
 * (n not a power of two). */
int32_t orc_work_queues(int32_t n, int32_t* peer, int32_t* vec);

/* ---- SpMV (bell.cpp:87-129, sparse_oracle.hpp:12-42) ---- */
/* Global block CSR with ascending columns; y = A x in the order of
 * spmv_partitioned_serial for n partitions (n = 1: spmv_serial). */
void orc_spmv(int32_t rows, const int64_t* row_ptr, const int32_t* cols, const double* vals,
              int32_t n, const double* x, double* y);

/* ---- PCG (solver.hpp:36-178) ---- */
/* Returns 0 ok, 2 solver error (message in err[256]). report histories
 * may be NULL. */
int32_t orc_pcg(int32_t rows, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                int32_t n, const double* b, double* x, const weft_pcg_config* cfg, weft_pcg_report* rep,
                char* err);

/* ---- elements (elements.cpp:94-403) ---- */
/* force: 12 doubles (4 x Vec3); jac: 144 doubles, block (a,b) row-major at
 * (a*4+b)*9; fric: 12 doubles; vdamp: 144 doubles. */
void orc_element_force(const weft_element* e, const double* x, double* force);
void orc_element_jacobian(const weft_element* e, const double* x, int32_t mode, double* jac);
void orc_element_friction(const weft_element* e, const double* v, double* force);
int32_t orc_element_has_damping(const weft_element* e);
void orc_element_velocity_damping(const weft_element* e, double* jac);
double orc_dihedral_angle(const double* x0, const double* x1, const double* x2, const double* x3);

/* ---- assembly (assembly.hpp:74-220, assembly.cpp:5-54) ---- */
typedef struct orc_system {
  int32_t rows;
  int64_t nnzb;
  int64_t* row_ptr; /* rows+1 */
  int32_t* cols;    /* nnzb, ascending per row */
  double* vals;     /* 9*nnzb, row-major blocks */
  double* rhs;      /* 3*rows */
} orc_system;
/* Global fill (partition-independent by the reference's own contract,
 * test_assembly.cpp:263-280). Returns 0 ok, 1 DimensionError (err). */
int32_t orc_fill_matrix(int32_t p, int64_t n_elem, const weft_element* elems, const double* x_cur,
                        const double* x_adv, const double* vel, const double* mass, const uint8_t* pinned,
                        double dt, int32_t mode, orc_system* out, char* err);
void orc_free_system(orc_system* s);

/* ---- broad phase (collision.cpp:77-192,205-210,329-378) ---- */
typedef struct orc_grid {
  int32_t tri_count;
  double cell_size;
  int64_t* tri_boxes; /* 6 per triangle */
  int64_t cells;
  uint64_t* cell_keys;   /* cells, sorted */
  int64_t* cell_offsets; /* cells+1 into cell_tris */
  int32_t* cell_tris;    /* ascending per cell */
  int64_t* prefix;       /* cells+1 workload prefix */
  int64_t total;
} orc_grid;
void orc_build_grid(int32_t tri_count, const int32_t* tris, const double* x0, const double* x1,
                    int32_t mode, double thickness, double cell_scale, orc_grid* out);
/* Candidate pairs of [begin,end); pairs may be NULL (count only). */
int64_t orc_candidates(const orc_grid* g, int64_t begin, int64_t end, int32_t* pairs);
void orc_free_grid(orc_grid* g);

/* ---- oracle::Rng (src/oracle/oracle.hpp:19-43): mt19937_64 ---- */
typedef struct orc_rng {
  uint64_t mt[312];
  int32_t idx;
} orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_raw(orc_rng* r);
double orc_rng_uniform(orc_rng* r, double lo, double hi);
int32_t orc_rng_uniform_int(orc_rng* r, int32_t lo, int32_t hi);

#ifdef __cplusplus
}
#endif

#endif
