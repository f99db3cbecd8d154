/*
 * amg.h -- C ABI of libamg_b200.so: the solve-phase hot path of J. Brannick,
 * "Aggregation-based aggressive coarsening with polynomial smoothing"
 * (arXiv:1307.6305), on NVIDIA B200 (sm_100a).
 *
 *   amg_setup  -- builds the unsmoothed-aggregation hierarchy of the problem of
 *                 PAPER.md Eq. (prob) (l.26-30): aggregates by repeated pairwise
 *                 matching (l.62-73), coarse operators A_H = P^T A P (l.112,
 *                 l.401-402), lambda_1 = ||A||_inf (l.146, l.326-327), the degree-m
 *                 best-uniform-approximation polynomial smoother (l.138-154) and a
 *                 dense coarsest solve (l.112, l.115).
 *   amg_solve  -- flexible CG (restart 5, l.322-323) preconditioned by the
 *                 nonlinear AMLI / k-cycle (l.319-321), W(1,1) (l.394).
 *   amg_free   -- releases everything.
 *
 * Citation keys: PAPER.md line numbers (l.N); readings of passages the paper
 * leaves silent or garbled are SURVEY.md 8(c) A1-A22, restated in DESIGN.md.
 *
 * Pointers.  Every array argument may be a HOST pointer (pageable or pinned)
 * or a DEVICE pointer of the current CUDA device; the library detects which
 * with cudaPointerGetAttributes and copies host data itself (the copies are
 * part of the call).  All computation runs in the library's CUDA kernels; no
 * step of setup or solve runs on the CPU.
 *
 * Threading.  A handle is used by one host thread at a time; different handles
 * may be used concurrently from different threads (each handle owns its own
 * library stream).  Calls block until their GPU work is complete (setup and
 * solve synchronise their stream).
 *
 * Errors.  Every call returns an int status (table below); no C++ exception
 * crosses the ABI.  amg_last_error() returns a thread-local message for the
 * last non-zero status.  On a setup error *out is NULL and nothing leaks.
 */
#ifndef AMG_B200_H
#define AMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---- */
#define AMG_OK              0   /* success */
#define AMG_NOT_CONVERGED   1   /* max_iter reached; x holds the last iterate */
#define AMG_E_ARG          (-1) /* bad argument: NULL where required, m < 1, passes < 1, nu < 1, tol <= 0,
                                   user kappa with E_m(kappa) >= 1 (reading A9), sizes out of range */
#define AMG_E_INPUT        (-2) /* CSR invalid: unsorted/duplicate columns, column out of range,
                                   positive off-diagonal, asymmetric pattern or values, stored diagonal
                                   != sum of off-diagonal weights (rel. 1e-10), d_i < 0 (Eq. (prob)) */
#define AMG_E_CUDA         (-3) /* CUDA runtime error */
#define AMG_E_NCCL         (-4) /* NCCL error (multi-GPU) */
#define AMG_E_OOM          (-5) /* device out of memory */
#define AMG_E_BREAKDOWN    (-6) /* FCG breakdown: d.q <= 0 or not finite */
#define AMG_E_SETUP        (-7) /* coarsening stagnated (n_{l+1} = n_l) above the coarsest size */

typedef struct amg_hierarchy* amg_handle; /* opaque, library-owned */
typedef struct amg_comm_s* amg_comm;       /* opaque communicator of the row-partitioned path */

#define AMG_COMM_ID_BYTES 128              /* size of an NCCL unique id */

typedef struct {
    int64_t  coarsest_size; /* stop coarsening once n_l <= this ("< 100"); default 100 */
    double   kappa;         /* lambda1/lambda0; 0 => rule R1 (reading A8): 10 (l.327) if E_m(10) < 1,
                               else the kappa with E_m = 1/2; default 0 */
    int32_t  restart;       /* outer FCG restart length (l.322-323); default 5 */
    int32_t  max_iter;      /* outer FCG iteration cap; default 500 */
    uint64_t seed;          /* matching-key salt seed (docs/keys.md); default 0 */
    void*    stream;        /* cudaStream_t the caller orders against; NULL = legacy default stream */
    int32_t  use_graphs;    /* 1 = replay each outer iteration as a captured CUDA graph; default 1 */
    int32_t  compress;      /* 1 = store each level's SELL streams losslessly compressed when possible:
                               <= 256 distinct values -> 1-byte codes into an fp64 dictionary, column
                               offsets col-row -> 1-byte codes (<= 256 distinct) or int16; default 1 */
    int64_t  tail_nnz;      /* the first level l >= 1 with nnz(A_l) <= tail_nnz and every level below it
                               run inside one single-CTA kernel per visit (coarse-tail megakernel);
                               0 disables; default 8192 */
    int64_t  gather_rows;   /* amg_setup_dist only: the first level with fewer than gather_rows rows
                               (and always the coarsest) is gathered onto every rank, which runs the
                               rest of the hierarchy redundantly; default 50000 */
    int32_t  tail_smem;     /* coarse-tail kernel's shared memory (200 KB): 0 = none; 1 = every vector of its
                               levels when they all fit; 2 = greedy by access frequency -- each level's
                               matrix (copied in per call), the smoother / transfer vectors, the aggregate
                               maps, then the inner-FCG vectors, the rest global; default 2 */
    int32_t  cycle;         /* coarse-level correction: 0 = N-AMLI / k-cycle, nu inner
                               FCG iterations (the paper's NPCG column; default); 2 = stationary AMLI:
                               e = q(B A) B rho with q the degree-(nu-1) best uniform approximation to
                               1/t on [1/amli_kappa, 1] (reading A23), a linear SPD preconditioner */
    double   amli_kappa;    /* cycle 2: 1/theta of the AMLI polynomial interval; 0 => rule R1 (A8) for
                               degree nu-1 (4 for nu = 2); default 0 */
    int32_t  lanczos_steps; /* 0 = lambda_1 = ||A_l||_inf (default); k > 0 = reading A24
                               (SURVEY 8(f) item 3): lambda_1 = min(||A_l||_inf, 1.1 theta_k), theta_k the
                               largest Ritz value of k Lanczos steps (smoothed levels; amg_setup only) */
    int32_t  mis_k;         /* 0 = p passes of pairwise matching (default); k >= 1 = reading A25 (SURVEY
                               8(f) item 2): each level is aggregated once by the MIS of
                               the graph of A^k grown into neighbourhood aggregates, p is ignored; k <= 8,
                               amg_setup only */
    int32_t  dense_b_rows;  /* the k-cycle operator B_{L-2} of the level above the coarsest is linear (exact
                               coarse solve, reading A12): when n_{L-2} <= dense_b_rows (and the level is
                               not row-partitioned) it is formed once at setup as a dense n x n matrix and
                               each application is one GEMV; 0 disables; default 4096 */
    int32_t  global_agg;    /* amg_setup_dist only: 0 = decoupled aggregation (reading A20: the matching passes
                               of a row-partitioned level see the edges inside each block; default); 1 = global
                               aggregation: the passes see every edge, matching by halo
                               rounds across the blocks, aggregates owned by their leader's rank -- the
                               single-GPU hierarchy for any number of ranks */
} amg_options;

typedef struct {
    int32_t  levels;            /* L: number of levels including the dense coarsest */
    int32_t  poly_degree;       /* m */
    int32_t  n_match_passes;    /* p */
    int32_t  singular;          /* 1 if d == NULL or d == 0: pure graph Laplacian, kernel = constants */
    int64_t  n[32];             /* n_l, l < min(levels, 32) */
    int64_t  nnz[32];           /* nnz(A_l) */
    double   lambda1[32];       /* ||A_l||_inf */
    double   kappa[32];         /* lambda1/lambda0 used on level l */
    double   grid_complexity;   /* sum n_l / n_0 (l.343) */
    double   operator_complexity; /* sum nnz_l / nnz_0 (l.344) */
    double   setup_ms;          /* device time of the last amg_setup (CUDA events) */
    double   solve_ms;          /* device time of the last amg_solve */
    int32_t  last_iters;        /* iterations of the last amg_solve */
    int32_t  reserved0;
    double   last_relres;       /* recursive ||r||/||b|| at exit */
    double   last_true_relres;  /* ||b - A x||/||b|| recomputed at exit */
    int64_t  launches_last_solve; /* kernels launched (incl. graph nodes) by the last amg_solve */
    int64_t  launches_per_iter; /* kernels per outer iteration */
    int64_t  launches_last_setup; /* library kernels launched by the last amg_setup (excl. CUB sort/scan) */
    int64_t  device_bytes;      /* device memory held by the handle */
    /* live profile of the dominant kernel inside the last amg_solve: CUDA events (on the launching
     * stream, recorded inside the replayed graph) around the level-0 post-smoothing steps k=1..m,
     * i.e. m launches of the fused three-term smoother step per outer iteration */
    double   prof_smoother_ms;        /* summed device time of the timed launches */
    int64_t  prof_smoother_launches;  /* number of timed launches */
    int64_t  prof_smoother_bytes;     /* algorithmic bytes per launch in the level-0 storage format: per entry
                                         value+column stream bytes (12 uncompressed; 2 for paired 1-byte
                                         codes), plus 32 n_0 for the four vectors */
    int32_t  level0_format;           /* 0 CSR tiles, 1 SELL-32 fp64/int32, 2 SELL-32 compressed */
    int32_t  nranks;                  /* ranks of the communicator (1 for amg_setup) */
    int32_t  dist_levels;             /* number of row-partitioned levels g (levels >= g are replicated) */
    int32_t  level0_path;             /* bit 0: level 0's SpMV-class passes (its interior view when split) take the
                                         TMA-staged kernel; bit 1: halo/compute overlap split (row-partitioned) */
} amg_info;

/* Fills *o with the defaults listed above.  Returns AMG_E_ARG if o == NULL. */
int amg_options_default(amg_options* o);

/*
 * amg_setup -- build the hierarchy.
 *   n        number of rows/unknowns (1 <= n < 2^31)
 *   row_ptr  int64[n+1], row_ptr[0] = 0, non-decreasing
 *   col      int32[nnz], strictly increasing within each row, 0 <= col < n
 *   val      fp64[nnz]: the weighted graph Laplacian part sum_e w_e (d_e u)(d_e v) of Eq. (prob):
 *            symmetric, off-diagonals -w_e < 0; diagonal entries optional (if present they must
 *            equal sum_{j != i} w_ij; if absent they are inserted)
 *   d        fp64[n] lower-order terms d_i >= 0 (Eq. (prob), l.34-35), or NULL.  The operator
 *            solved is A = L + diag(d).  d == NULL or all zero => singular mode (l.36-38): the
 *            graph must be connected; b is projected to mean zero.
 *   n_match_passes  p >= 1 pairwise-matching passes per level (aggregates ~2^p; readings A1-A5)
 *   poly_degree     m >= 1 smoother degree (l.149-152)
 *   opt      options or NULL for defaults
 * Arrays are borrowed for the duration of the call and copied; *out owns all device memory.
 */
int amg_setup(amg_handle* out, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
              const double* d, int32_t n_match_passes, int32_t poly_degree, const amg_options* opt);

/*
 * amg_solve -- outer flexible CG preconditioned by the k-cycle.
 *   b        fp64[n] right-hand side (host or device)
 *   x        fp64[n] in: initial guess x_0; out: solution (host or device; overwritten)
 *   tol      stop when ||r_k||_2 <= tol ||b||_2 on the recursive residual (reading A14)
 *   k_inner  1 <= nu <= 16 inner FCG iterations per coarse-level visit (k-cycle, l.321; BASELINE uses 2;
 *            16 = the inner direction window)
 *   iters    out (nullable): outer iterations performed
 *   relres   out (nullable): ||r||/||b|| at exit
 * Returns AMG_OK, AMG_NOT_CONVERGED, AMG_E_BREAKDOWN or an error.
 */
int amg_solve(amg_handle h, const double* b, double* x, double tol, int32_t k_inner, int32_t* iters,
              double* relres);

/* ---------------------------------------------------------------------------------------------
 * Row-partitioned multi-GPU path.  One process (or, for testing,
 * one host thread) per rank.  Levels are row-partitioned with DECOUPLED aggregation (reading A20:
 * the matching passes of a partitioned level use only the edges inside each block, so aggregates,
 * restriction and prolongation are rank-local and the coarse blocks are the fine blocks'
 * aggregates).  Every SpMV-class pass exchanges a halo (grouped point-to-point messages), every FCG
 * dot batch is allgathered and summed in rank order (identical scalars on every rank), and the
 * first level below opt->gather_rows (at the latest the coarsest) is gathered once at setup and
 * then run redundantly on every rank.  All calls on a distributed handle are collective.
 * ------------------------------------------------------------------------------------------- */
/* NCCL unique id (rank 0 creates it and sends the AMG_COMM_ID_BYTES bytes to the other ranks,
 * e.g. with torch.distributed).  Returns AMG_E_NCCL if libnccl.so.2 cannot be loaded. */
int amg_comm_unique_id(uint8_t* id);
/* NCCL communicator over the current CUDA device (collective over the nranks processes). */
int amg_comm_init_nccl(amg_comm* out, const uint8_t* id, int32_t nranks, int32_t rank);
/* nranks communicators out[0..nranks) for nranks host threads of THIS process sharing the current
 * device (single-GPU emulation of the multi-rank path for tests: each exchange synchronises the
 * caller's stream and meets the other threads at a host barrier; CUDA graphs are not used). */
int amg_comm_init_threads(amg_comm* out, int32_t nranks);
int amg_comm_rank(amg_comm c, int32_t* rank, int32_t* size);
/* Releases a communicator (after every handle that uses it).  NULL is a no-op. */
int amg_comm_free(amg_comm c);

/*
 * amg_setup_dist -- collective amg_setup over the ranks of `comm`.
 *   n_global    rows of the whole problem
 *   row_begin   first global row of this rank; the ranks' blocks [row_begin, row_begin + n_local)
 *               must tile [0, n_global) in rank order (AMG_E_ARG on every rank otherwise)
 *   n_local     rows of this rank (>= 1)
 *   row_ptr     int64[n_local+1] of this rank's rows; col int32 GLOBAL column ids; val, d as in
 *               amg_setup (d: this rank's n_local entries, or NULL on every rank)
 * Cross-block symmetry of the values is the caller's contract (the pattern is checked through the
 * halo requests).  amg_solve on the handle takes this rank's blocks of b and x (n_local each).
 */
int amg_setup_dist(amg_handle* out, amg_comm comm, int64_t n_global, int64_t row_begin, int64_t n_local,
                   const int64_t* row_ptr, const int32_t* col_global, const double* val, const double* d,
                   int32_t n_match_passes, int32_t poly_degree, const amg_options* opt);

/* Releases the handle and all its device memory.  NULL is a no-op returning AMG_OK. */
int amg_free(amg_handle h);

/* Hierarchy / last-call statistics. */
int amg_get_info(amg_handle h, amg_info* info);

/* Thread-local message for the last non-zero status ("" if none). */
const char* amg_last_error(void);

/* ---------------------------------------------------------------------------------------------
 * Parity hooks (test-only, not part of the product API): export the hierarchy and apply single
 * pieces of the path so tests can compare them with the CPU oracle.  Output arrays may be host or
 * device pointers sized by amg_level_sizes.
 * ------------------------------------------------------------------------------------------- */
/* n, nnz of A_l, coarse size nc (0 on the coarsest), lambda1, kappa, alpha/beta (m+1 each, nullable). */
int amg_level_sizes(amg_handle h, int32_t level, int64_t* n, int64_t* nnz, int64_t* nc, double* lambda1,
                    double* kappa, double* alpha, double* beta);
/* CSR of A_l (row_ptr int64[n+1], col int32[nnz], val fp64[nnz]) and agg int32[n] (NULL to skip). */
int amg_level_export(amg_handle h, int32_t level, int64_t* row_ptr, int32_t* col, double* val, int32_t* agg);
/* x = S_l(f, x0) = x0 + q_m(A_l)(f - A_l x0), one whole smoother application. */
int amg_level_smooth(amg_handle h, int32_t level, const double* f, const double* x0, double* x);
/* z = B_l(r), one k-cycle application from level l with nu inner iterations. */
int amg_level_precond(amg_handle h, int32_t level, int32_t k_inner, const double* r, double* z);
/* e = A_L^{-1} r (or A_L^dagger r if singular) on the coarsest level. */
int amg_coarse_solve(amg_handle h, const double* r, double* e);
/* Partition of level l: *dist = 1 if row-partitioned (then amg_level_sizes reports this rank's rows,
 * amg_level_export exports them with GLOBAL column ids and global coarse aggregate ids, and
 * amg_level_smooth / amg_level_precond take this rank's blocks), 0 if every rank holds it whole. */
int amg_level_dist(amg_handle h, int32_t level, int32_t* dist, int64_t* row_begin, int64_t* n_global);
/* Host-only (no CUDA): the halo receive plan of one block -- for the sorted unique global ids of the
 * columns outside [row_begin, row_begin + n_local), the runs owned by one rank (owner offs[q] <= id <
 * offs[q+1]): seg_peer/seg_off (relative column of the run's first id: negative below the block,
 * >= n_local above)/seg_cnt, *n_seg runs, *n_lo ids below the block.  Output arrays hold >= n_halo. */
int amg_halo_plan(int64_t row_begin, int32_t n_local, const int64_t* offs, int32_t nranks, int32_t rank,
                  const int32_t* halo_ids, int32_t n_halo, int32_t* seg_peer, int32_t* seg_off, int32_t* seg_cnt,
                  int32_t* n_seg, int32_t* n_lo);

#ifdef __cplusplus
}
#endif

#endif /* AMG_B200_H */
