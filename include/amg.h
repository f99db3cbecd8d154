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
 * Threading.  A handle is used by one host thread at a time.  Calls block until
 * their GPU work is complete (setup and solve synchronise their stream).
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
    int64_t  reserved[5];
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
    int32_t  reserved1;
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
 *   k_inner  nu >= 1 inner FCG iterations per coarse-level visit (k-cycle, l.321; BASELINE uses 2)
 *   iters    out (nullable): outer iterations performed
 *   relres   out (nullable): ||r||/||b|| at exit
 * Returns AMG_OK, AMG_NOT_CONVERGED, AMG_E_BREAKDOWN or an error.
 */
int amg_solve(amg_handle h, const double* b, double* x, double tol, int32_t k_inner, int32_t* iters,
              double* relres);

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

#ifdef __cplusplus
}
#endif

#endif /* AMG_B200_H */
