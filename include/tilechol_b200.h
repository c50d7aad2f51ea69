/*
 * tilechol_b200 — C ABI of the B200-native arrowhead tile-Cholesky path.
 *
 * Drop-in boundary for the reference plugin seam `tilechol.backend.impl`
 * (reference pkg/src/tilechol/backend.py:1-26), whose two implementations
 * (_backend_numba.py, _backend_numpy.py) export exactly eight functions.
 * Each entry below names the reference function it replaces.  Conventions:
 *
 *   - plain pointers and sizes only, no C++ exceptions cross the ABI;
 *   - every function returns TC_OK (0) or a negative TC_ERR_* status;
 *     tc_last_error() returns a thread-local message for the last failure;
 *   - tiles are nt x nt float64 column-major (element (i, j) at j*nt + i),
 *     slot s of a storage array starts at s*nt*nt (reference ctsf.py:87-98);
 *   - "dev" pointers are CUDA device pointers, `stream` is a cudaStream_t
 *     (NULL = legacy default stream); integer op/index arrays are host arrays;
 *   - no CPU fallback: device entry points fail with TC_ERR_CUDA when no
 *     device is present.
 */
#ifndef TILECHOL_B200_H
#define TILECHOL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TC_OK 0
#define TC_ERR_ARG (-1)
#define TC_ERR_CUDA (-2)
#define TC_ERR_NOMEM (-3)
#define TC_ERR_STATE (-4)
#define TC_ERR_FORMAT (-5)

/* task / op codes: reference symbolic.py:19-21, _backend_numba.py:13 */
#define TC_POTRF 1
#define TC_SYRK 2
#define TC_TRSM 3
#define TC_GEMM 4
#define TC_GEADD 5
#define TC_ZERO 6

const char* tc_last_error(void);
int32_t tc_abi_version(void);
/* number of visible CUDA devices (0 when none); never fails */
int32_t tc_device_count(void);

/* ======================================================================
 * Host-side integer analysis (bit-exact with the reference; no GPU used)
 * ====================================================================== */

/* reference _backend_numba.py:188-215 etree_fill_count(n, row_ptr, row_cols):
 * strict-lower nnz(L) from the strict-lower CSR of a symmetric pattern. */
int tc_etree_fill_count(int64_t n, const int64_t* row_ptr, const int64_t* row_cols,
                        int64_t* out_count);

/* reference ordering.py:239-263 symbolic_fill_count(m, p): nnz(L) incl. the
 * diagonal of P A P^T (forward may be NULL for the identity). */
/* Zero-fill test of the identity ordering (parallel perfect-elimination
 * check); *perfect = 1 iff nnz(L) = nnz(lower A), *offdiag = strictly lower
 * entries.  Shortcut in front of tc_symbolic_fill_count for select_ordering
 * (reference ordering.py:266-275: identity wins unless strictly beaten). */
int tc_zero_fill(int64_t n, const int64_t* col_ptr, const int32_t* row_idx, int32_t* perfect, int64_t* offdiag);
int tc_symbolic_fill_count(int64_t n, const int64_t* col_ptr, const int32_t* row_idx,
                           const int64_t* forward, int64_t* out_nnz_factor);

/* Column counts of L (incl. diagonal) of P A P^T, counts[n]; sum c_j^2 is the
 * tile-size independent "useful" flop count of survey 8(d). */
int tc_factor_column_counts(int64_t n, const int64_t* col_ptr, const int32_t* row_idx,
                            const int64_t* forward, int64_t* counts);

/* reference matcore.py:320-348 structure_stats (bandwidth, thickness). */
int tc_structure_stats(int64_t n, const int64_t* col_ptr, const int32_t* row_idx,
                       double dense_row_threshold, int64_t* out_bandwidth,
                       int64_t* out_thickness);

/* reference matcore.py:269-317 generate_arrowhead, pattern part: col_ptr[n+1]
 * always written, row_idx[nnz] when non-NULL (memory-light, no temporaries). */
int tc_arrowhead_pattern(int64_t n, int64_t b, int64_t t, int32_t block_diagonal,
                         int64_t* col_ptr, int32_t* row_idx);
/* Variable-bandwidth arrowhead pattern (BASELINE config 2 / survey App. A2):
 * head column j < n-t holds rows j..j+band[j] and the t arrow rows, tail
 * columns are dense.  Same two-call convention as tc_arrowhead_pattern. */
int tc_band_arrow_pattern(int64_t n, int64_t t, const int64_t* band, int64_t* col_ptr,
                          int32_t* row_idx);
/* reference matcore.py:309-316: diagonal = 1 + |row| sums, accumulated in CSC
 * order exactly like the two np.bincount passes (bit-identical). */
int tc_arrowhead_diag(int64_t n, const int64_t* col_ptr, const int32_t* row_idx,
                      double* values);

/* reference ordering.py:134-170 rcm(m, pinned_tail) -> forward[n]. */
int tc_rcm(int64_t n, const int64_t* col_ptr, const int32_t* row_idx,
           int64_t pinned_tail, int64_t* forward_out);

/* reference ordering.py:209-236 adaptable_nd(m, stats, max_levels) -> forward[n]. */
int tc_adaptable_nd(int64_t n, int64_t bandwidth, int64_t thickness, int32_t max_levels,
                    int64_t* forward_out);

/* Tile symbolic analysis handle: reference ctsf.py:57-84 (grid_from_tiles,
 * build_tile_grid), symbolic.py:98-123 (tile_symbolic_factorize),
 * symbolic.py:126-164 (enumerate_tasks), symbolic.py:218-269
 * (plan_tree_reduction), symbolic.py:287-331 (dag_stats) and the op compiler
 * of the reference's missing scheduler. */
typedef struct tc_symbolic* tc_symbolic_t;

int tc_symbolic_from_csc(int64_t n, int32_t nt, const int64_t* col_ptr,
                         const int32_t* row_idx, tc_symbolic_t* out);
int tc_symbolic_from_tiles(int64_t n, int32_t nt, int64_t count, const int64_t* rows,
                           const int64_t* cols, tc_symbolic_t* out);
int tc_symbolic_info(tc_symbolic_t h, int64_t* T, int64_t* S_in, int64_t* S, int64_t* P);
int tc_symbolic_grid(tc_symbolic_t h, int32_t* tile_rows, int32_t* tile_cols);
int tc_symbolic_factor(tc_symbolic_t h, int32_t* f_rows, int32_t* f_cols, int64_t* accum);
int tc_symbolic_tasks(tc_symbolic_t h, int8_t* type, int32_t* m, int32_t* k, int32_t* n,
                      int32_t* target);
/* chains with accum >= 2*workers: slots[n_chains], ranges[n_chains*workers*2]
 * (call with NULL arrays to get n_chains). */
int tc_symbolic_tree_plan(tc_symbolic_t h, int32_t workers, int64_t* n_chains,
                          int64_t* slots, int64_t* ranges);
/* op stream (sequential when workers < 2): call with NULL arrays for sizes. */
int tc_symbolic_compile_ops(tc_symbolic_t h, int32_t workers, int64_t* n_ops,
                            int64_t* n_scratch, int8_t* op, int64_t* dst, int64_t* src1,
                            int64_t* src2);
int tc_symbolic_dag_stats(tc_symbolic_t h, int64_t* critical_path, int64_t* max_width);
void tc_symbolic_destroy(tc_symbolic_t h);

/* ======================================================================
 * Device tile kernels (single-tile launches; KAT / plugin parity)
 * ====================================================================== */

/* reference _backend_numba.py:16-38 potrf_tile(a) -> -1 | first pivot j with
 * a[j,j] <= 0 (NaN passes).  Synchronises `stream` to return *info. */
int tc_potrf_tile(double* a_dev, int32_t nt, void* stream, int32_t* info);
/* reference _backend_numba.py:41-59 trsm_tile(l, x): X L^T = B in place;
 * *info = -1 | first k with l[k,k] == 0.  Synchronises. */
int tc_trsm_tile(const double* l_dev, double* x_dev, int32_t nt, void* stream,
                 int32_t* info);
/* reference _backend_numba.py:62-69 syrk_tile(a, c): c -= a a^T (full tile). */
int tc_syrk_tile(const double* a_dev, double* c_dev, int32_t nt, void* stream);
/* reference _backend_numba.py:72-79 gemm_tile(a, b, c): c -= b a^T. */
int tc_gemm_tile(const double* a_dev, const double* b_dev, double* c_dev, int32_t nt,
                 void* stream);
/* reference _backend_numba.py:82-88 geadd_tile(t, c): c += t. */
int tc_geadd_tile(const double* t_dev, double* c_dev, int32_t nt, void* stream);

/* reference _backend_numba.py:98-133 run_ops(storage, scratch, op_type, dst,
 * src1, src2, start, stop) -> (p, info): executes ops [start, stop) in order;
 * slot ids >= S address scratch[s - S].  On the first POTRF/TRSM failure the
 * remaining ops are skipped on device and (*out_p, *out_info) = (p, local
 * index); on success (stop, -1).  Synchronises `stream`. */
int tc_run_ops(double* storage_dev, int64_t S, double* scratch_dev, int64_t R, int32_t nt,
               const int8_t* op_type, const int64_t* dst, const int64_t* src1,
               const int64_t* src2, int64_t n_ops, int64_t start, int64_t stop,
               void* stream, int64_t* out_p, int32_t* out_info);

/* reference _backend_numba.py:136-185 replay_residual(storage, template, op_type,
 * dst, src1, src2, diag_slot) -> sum of squared errors (symmetric weights). */
int tc_replay_residual(const double* storage_dev, const double* template_dev, int64_t S,
                       int32_t nt, const int8_t* op_type, const int64_t* dst,
                       const int64_t* src1, const int64_t* src2, int64_t n_ops,
                       const uint8_t* diag_slot, void* stream, double* out_err2);

/* ======================================================================
 * Optimised path: device launch plan (api.factorize / logdet / solve,
 * SPEC.md:477-519; replaces the missing scheduler SPEC.md:412-475)
 * ====================================================================== */

typedef struct tc_plan* tc_plan_t;

typedef struct tc_plan_opts {
    int32_t tree_workers;   /* W partial accumulators per long chain; 0 = 8 */
    int32_t tree_threshold; /* chains with accum >= threshold are split; 0 = 2*W, <0 = off */
    int32_t chunk;          /* columns per split-K chunk launch; 0 = auto */
    int32_t lookahead;      /* D >= 1: last D contributing columns split off the bulk update; 0 = off; < 0 = auto (3 / 4) */
    int32_t use_graph;      /* 2 = persistent (default), 1 = CUDA graph, 0 = direct launches */
    int32_t reserved[3];    /* [0] 1 = no POTRF->TRSM streaming, [1] persistent CTAs/SM (0 auto),
                               [2] concurrent factorisations sharing the GPU (grid share) */
} tc_plan_opts;

/* Build a plan from the factor tile pattern (slots in (col,row) order, all
 * diagonals present), e.g. tc_symbolic_factor output. */
int tc_plan_create(int64_t n, int32_t nt, int64_t S, const int32_t* f_rows,
                   const int32_t* f_cols, const tc_plan_opts* opts, tc_plan_t* out);
int tc_plan_info(tc_plan_t p, int64_t* n_launches, int64_t* n_items, int64_t* n_pairs,
                 int64_t* scratch_tiles, double* tile_flops);
/* In-place numeric factorisation of storage_dev[S,nt,nt]; *fail_index = -1 or
 * the global permuted scalar index k*nt+info of the first non-positive pivot.
 * Also computes the log-determinant (read with tc_plan_last_logdet).
 * Synchronises `stream`. */
int tc_plan_factorize(tc_plan_t p, double* storage_dev, void* stream, int64_t* fail_index);
/* Asynchronous variant: enqueue only (no sync); results via tc_plan_collect. */
int tc_plan_factorize_async(tc_plan_t p, int32_t lane, double* storage_dev, void* stream);
int tc_plan_collect(tc_plan_t p, int32_t lane, void* stream, int64_t* fail_index,
                    double* logdet);
/* End-to-end host staging: page-lock a host array in place (cudaHostRegister)
 * / release it; async H2D copy on `stream`. */
int tc_host_register(void* ptr, size_t bytes);
int tc_host_unregister(void* ptr);
int tc_memcpy_h2d_async(void* dst_dev, const void* src_host, size_t bytes, void* stream);
/* Debug: the current ticket of a lane's persistent kernel (read while it runs). */
int tc_plan_debug_ticket(tc_plan_t p, int32_t lane, int32_t* ticket, int32_t* ntasks);
/* Streaming batches: enqueue on `stream` device copies of the lane's failure
 * word (INT64_MAX = success, else k*nt+info) and log-determinant. */
int tc_plan_copy_result(tc_plan_t p, int32_t lane, void* stream, int64_t* fail_dev,
                        double* logdet_dev);
/* 2 * sum log diag(L) over non-padding diagonal positions. */
int tc_plan_logdet(tc_plan_t p, const double* storage_dev, void* stream, double* out);
/* In-place tile forward/back substitution of rhs_dev[nrhs][T*nt] (column of
 * length T*nt per right-hand side, padded entries must be 0) against the
 * factor: rhs <- L^-T L^-1 rhs.  Asynchronous on `stream`:
 * a batched TRSM forms L_kk^-T for every diagonal tile, then ONE persistent
 * launch runs both sweeps (per-column done flags, fixed summation order, so
 * the result does not depend on timing).  nt <= 480. */
int tc_plan_solve(tc_plan_t p, const double* storage_dev, double* rhs_dev, int32_t nrhs,
                  void* stream);
/* Scatter CSC values (already on device) into zeroed tile storage with unit
 * padding (reference ctsf.py:118-139); offsets_dev from tc_plan_pack_offsets. */
int tc_plan_pack_offsets(tc_plan_t p, int64_t n, const int64_t* col_ptr,
                         const int32_t* row_idx, int64_t* offsets_out);
int tc_plan_pack(tc_plan_t p, const double* values_dev, const int64_t* offsets_dev,
                 int64_t nnz, double* storage_dev, void* stream);
/* Device value assembly for a family of matrices sharing the pattern
 * (INLA batch): storage <- scatter of sum_i coef[i] *
 * basis_dev[i][0:nnz] (nbasis <= 16, evaluated left to right, products and
 * sums separately rounded: bitwise the host evaluation of the same sum). */
int tc_plan_pack_lincomb(tc_plan_t p, const double* basis_dev, int32_t nbasis, const double* coef,
                         const int64_t* offsets_dev, int64_t nnz, double* storage_dev, void* stream);
void tc_plan_destroy(tc_plan_t p);

/* Profiling: serialised single-stream pass of the plan with CUDA events around
 * every launch.  Per class c (0 bulk update, 1 last update, 2 POTRF, 3 TRSM,
 * 4 tree combine, 5 logdet, 6 split-K chunk; n_cls >= 7): summed ms, launch
 * count and algorithmic flops.  Factorises storage_dev in place. */
int tc_plan_profile(tc_plan_t p, double* storage_dev, void* stream, int32_t n_cls, double* ms,
                    int64_t* counts, double* flops);
/* Persistent-executor task trace (diagnostics): factorises storage_dev once
 * and returns per task [ticket_ns, start_ns, end_ns, sm_id] (tasks_out[cap][4])
 * and its launch id, per launch [kind, column, class] (launch_meta[NL][3]).
 * With cap < n_tasks or launch_cap < n_launches only the sizes are returned. */
int tc_plan_trace(tc_plan_t p, double* storage_dev, void* stream, int64_t cap, int64_t* tasks_out,
                  int32_t* task_launch, int64_t launch_cap, int32_t* launch_meta, int64_t* n_tasks,
                  int64_t* n_launches);
/* FP64 tensor-pipe (DMMA m8n8k4) throughput microbenchmark, TFLOP/s. */
int tc_bench_dmma_peak(int64_t iters, int32_t blocks_per_sm, int32_t warps_per_block,
                       double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* TILECHOL_B200_H */
