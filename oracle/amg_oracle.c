/*
 * oracle/amg_oracle.c -- plain, slow, obviously-correct CPU oracle of the solve
 * path of J. Brannick, "Aggregation-based aggressive coarsening with polynomial
 * smoothing" (arXiv:1307.6305), as scoped by SURVEY.md 8(a)-(c).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product
 * (paper_1307_6305_b200/, libamg_b200.so) never links, imports or calls it, and
 * shares no source, header, table or constant generator with it.
 *
 * Citation keys: P:n = PAPER.md line n; S:n = SPEC.md line n; SURVEY 8(c) On / An
 * = the oracle step / reading of SURVEY.md section 8(c) (readings restated in
 * DESIGN.md "Readings").  Everything is fp64, sequential, in the order the cited
 * passage states; no blocking, fusion or reordering.  Build with
 * -ffp-contract=off so no multiply-add is fused.
 *
 * Pins: every function here is pinned by a -m "not gpu" test in tests/ against
 * something other than itself (closed forms, dense linear algebra, brute force,
 * the paper's golden example); see DESIGN.md "Oracle pins".  The multilevel
 * nonlinear k-cycle (ocycle with cycle=0 at > 2 levels) is pinned in its two
 * closed-form regimes (nu large: the P:136 two-level formula with the exact
 * A_1^{-1}, L = 3 and 4; nu = 1: one optimal inner step along B_1 rho) and by
 * homogeneity; for nu = 2 at L >= 3 only those general pins apply.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_NOT_CONVERGED 1
#define ORC_E_ARG (-1)
#define ORC_E_INPUT (-2)
#define ORC_E_OOM (-5)
#define ORC_E_BREAKDOWN (-6)
#define ORC_E_SETUP (-7)

#define ORC_MAXLEV 64
#define ORC_MAXDEG 32
#define ORC_MAXLANCZOS 64

/* ========================================================== sparse matrix */
typedef struct {
    int64_t n, nnz;
    int64_t *rp;  /* [n+1] */
    int32_t *ci;  /* [nnz], strictly increasing within a row */
    double *v;    /* [nnz] values (matrices), or NULL */
    int64_t *w;   /* [nnz] integer multiplicities (matching pass graphs), or NULL */
} ocsr;

static void ocsr_free(ocsr *a) {
    if (!a) return;
    free(a->rp); free(a->ci); free(a->v); free(a->w);
    memset(a, 0, sizeof(*a));
}

/* y = A x, each row summed left to right in CSR order. */
static void ospmv(const ocsr *A, const double *x, double *y) {
    for (int64_t i = 0; i < A->n; ++i) {
        double s = 0.0;
        for (int64_t p = A->rp[i]; p < A->rp[i + 1]; ++p) s += A->v[p] * x[A->ci[p]];
        y[i] = s;
    }
}

/* lambda_1 = ||A||_inf = max_i sum_j |a_ij|. */
static double oinf_norm(const ocsr *A) {
    double m = 0.0;
    for (int64_t i = 0; i < A->n; ++i) {
        double s = 0.0;
        for (int64_t p = A->rp[i]; p < A->rp[i + 1]; ++p) s += fabs(A->v[p]);
        if (s > m) m = s;
    }
    return m;
}

static double odot(int64_t n, const double *a, const double *b) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* =================================================== polynomial smoother */
/* delta = (sqrt(kappa)-1)/(sqrt(kappa)+1). */
static double odelta(double kappa) { return (sqrt(kappa) - 1.0) / (sqrt(kappa) + 1.0); }

/* E_m = delta^m (kappa-1)/2. */
double orc_Em(int m, double kappa) { return pow(odelta(kappa), (double)m) * (kappa - 1.0) / 2.0; }

/* Reading A8 (rule R1): kappa = 10 if E_m(10) < 1, else the kappa* with
 * E_m(kappa*) = 1/2, i.e. t = sqrt(kappa*) the root > 1 of
 * (t-1)^(m+1) = (t+1)^(m-1)  (SURVEY Appendix A "Closed form for R1").
 * Solved by plain bisection on [1, 1+2^(1+2/m)...] down to adjacent doubles. */
double orc_kappa_rule(int m) {
    if (m >= 1 && orc_Em(m, 10.0) < 1.0) return 10.0;
    double lo = 1.0, hi = 16.0; /* g(lo) < 0 < g(hi) for m <= 2 */
    for (int it = 0; it < 2000; ++it) {
        double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        double g = pow(mid - 1.0, (double)(m + 1)) - pow(mid + 1.0, (double)(m - 1));
        if (g < 0.0) lo = mid; else hi = mid;
    }
    double t = 0.5 * (lo + hi);
    return t * t;
}

/* Three-term recurrence of the best uniform approximation q_m to 1/x on
 * [lambda0, lambda1] (the recurrence P:153-154 defers to [KVZ_09];
 * its closed form is derived in SURVEY Appendix A):
 *   x_{k+1} = alpha_k x_k + (1-alpha_k) x_{k-1} + beta_k (f - A x_k), k = 0..m,
 *   alpha_0 = 1,                                   beta_0 = (l0+l1)/(2 l0 l1),
 *   alpha_1 = 1 + 2 d^2 (1-d^2)/(1+d^2)^2,         beta_1 = 2/(l0+l1),
 *   alpha_k = 1 + d^2 (k >= 2),                    beta_k = 4 d/(l1-l0),
 * with d = delta(kappa), l0 = l1/kappa. */
void orc_poly_coeffs(double lambda1, double kappa, int m, double *alpha, double *beta) {
    double l1 = lambda1, l0 = lambda1 / kappa, d = odelta(kappa), d2 = d * d;
    for (int k = 0; k <= m; ++k) {
        if (k == 0) { alpha[k] = 1.0; beta[k] = (l0 + l1) / (2.0 * l0 * l1); }
        else if (k == 1) { alpha[k] = 1.0 + 2.0 * d2 * (1.0 - d2) / ((1.0 + d2) * (1.0 + d2)); beta[k] = 2.0 / (l0 + l1); }
        else { alpha[k] = 1.0 + d2; beta[k] = 4.0 * d / (l1 - l0); }
    }
}

/* S(f, x0) = x0 + q_m(A)(f - A x0) by m+1 recurrence steps with x_{-1} = x_0
 * (SURVEY 8(c) O5).  x may alias x0. */
static void osmooth(const ocsr *A, int m, const double *alpha, const double *beta,
                    const double *f, const double *x0, double *x) {
    int64_t n = A->n;
    double *xm1 = malloc(sizeof(double) * n), *xk = malloc(sizeof(double) * n);
    double *xn = malloc(sizeof(double) * n), *t = malloc(sizeof(double) * n);
    memcpy(xm1, x0, sizeof(double) * n);
    memcpy(xk, x0, sizeof(double) * n);
    for (int k = 0; k <= m; ++k) {
        ospmv(A, xk, t);
        for (int64_t i = 0; i < n; ++i)
            xn[i] = alpha[k] * xk[i] + (1.0 - alpha[k]) * xm1[i] + beta[k] * (f[i] - t[i]);
        double *tmp = xm1; xm1 = xk; xk = xn; xn = tmp;
    }
    memcpy(x, xk, sizeof(double) * n);
    free(xm1); free(xk); free(xn); free(t);
}

/* ===================================================== matching */
/* SplitMix64 output for state z (docs/keys.md). */
static uint64_t osm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Largest eigenvalue of the symmetric tridiagonal T (diagonal a[0..k), off-diagonal b[1..k)) by
 * bisection on the Sturm count (number of eigenvalues < x), to adjacent doubles. */
static double otridiag_max(int k, const double *a, const double *b) {
    double lo = a[0], hi = a[0];
    for (int j = 0; j < k; ++j) { /* Gershgorin interval */
        double r = (j > 0 ? fabs(b[j]) : 0.0) + (j + 1 < k ? fabs(b[j + 1]) : 0.0);
        if (a[j] - r < lo) lo = a[j] - r;
        if (a[j] + r > hi) hi = a[j] + r;
    }
    for (int it = 0; it < 200; ++it) {
        double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        int cnt = 0; /* eigenvalues < mid: negative pivots of T - mid I */
        double d = 1.0;
        for (int j = 0; j < k; ++j) {
            d = a[j] - mid - (j > 0 ? b[j] * b[j] / d : 0.0);
            if (d == 0.0) d = -1e-300;
            if (d < 0.0) cnt++;
        }
        if (cnt == k) hi = mid; else lo = mid;
    }
    return 0.5 * (lo + hi);
}

/* Reading A24 ("tighter lambda_max"; opt-in, the paper's setting is
 * lambda_1 = ||A||_inf): lambda_1 = min(||A||_inf, 1.1 theta_k) with theta_k the largest Ritz
 * value of k plain Lanczos steps on A from v_0 = u/||u||, u_i = 2 U(z ^ i) - 1,
 * U(y) = (splitmix64(y) >> 11) 2^-53, z = splitmix64(seed ^ 0x4C414E435A4F5300 ^ level):
 *   w = A v_j - beta_j v_{j-1}; alpha_j = v_j.A v_j; w -= alpha_j v_j; beta_{j+1} = ||w||; v_{j+1} = w/beta_{j+1}
 * (w formed as A v_j - alpha_j v_j - beta_j v_{j-1}; stops early if beta_{j+1} = 0). */
static uint64_t osm64(uint64_t z);
double orc_lanczos_max(const int64_t n, const int64_t *rp, const int32_t *ci, const double *v, int k, uint64_t seed,
                       int level) {
    ocsr A = {n, rp[n], (int64_t *)rp, (int32_t *)ci, (double *)v, NULL};
    double *vj = malloc(sizeof(double) * n), *vm = calloc((size_t)n, sizeof(double));
    double *w = malloc(sizeof(double) * n);
    double al[ORC_MAXLANCZOS], be[ORC_MAXLANCZOS + 1];
    uint64_t z = osm64(seed ^ 0x4C414E435A4F5300ULL ^ (uint64_t)level);
    for (int64_t i = 0; i < n; ++i) vj[i] = 2.0 * ((double)(osm64(z ^ (uint64_t)i) >> 11) * 0x1.0p-53) - 1.0;
    double nr = sqrt(odot(n, vj, vj));
    for (int64_t i = 0; i < n; ++i) vj[i] /= nr;
    be[0] = 0.0;
    int steps = 0;
    if (k > ORC_MAXLANCZOS) k = ORC_MAXLANCZOS;
    for (int j = 0; j < k; ++j) {
        ospmv(&A, vj, w);
        al[j] = odot(n, vj, w);
        for (int64_t i = 0; i < n; ++i) w[i] = w[i] - al[j] * vj[i] - be[j] * vm[i];
        steps = j + 1;
        be[j + 1] = sqrt(odot(n, w, w));
        if (!(be[j + 1] > 0.0)) break;
        for (int64_t i = 0; i < n; ++i) {
            vm[i] = vj[i];
            vj[i] = w[i] / be[j + 1];
        }
    }
    double t = otridiag_max(steps, al, be);
    free(vj); free(vm); free(w);
    return t;
}

/* salt(seed, level, pass) = splitmix64(seed ^ ((level << 8) ^ pass))  (A2). */
static uint64_t osalt(uint64_t seed, int level, int pass) {
    return osm64(seed ^ (((uint64_t)level << 8) ^ (uint64_t)pass));
}

/* Edge key (w, h, lo, hi), compared lexicographically, larger wins (A2). */
typedef struct { int64_t w; uint64_t h; int64_t lo, hi; } okey;

static okey omkkey(int64_t w, int64_t a, int64_t b, uint64_t salt) {
    okey k;
    k.w = w;
    k.lo = a < b ? a : b;
    k.hi = a < b ? b : a;
    k.h = osm64((((uint64_t)k.lo) << 32 | (uint64_t)(uint32_t)k.hi) ^ salt);
    return k;
}

static int okey_gt(okey a, okey b) {
    if (a.w != b.w) return a.w > b.w;
    if (a.h != b.h) return a.h > b.h;
    if (a.lo != b.lo) return a.lo > b.lo;
    return a.hi > b.hi;
}

typedef struct { okey k; } oedge;

static int oedge_cmp_desc(const void *pa, const void *pb) {
    const oedge *a = pa, *b = pb;
    if (okey_gt(a->k, b->k)) return -1;
    if (okey_gt(b->k, a->k)) return 1;
    return 0;
}

/* Sequential rule ("edge-greedy"): scan edges in decreasing key order, take an
 * edge if both ends are free (A1; "a matching ... no two edges incident"). */
static void omatch_greedy(const ocsr *G, uint64_t salt, int32_t *mate) {
    int64_t n = G->n, ne = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = G->rp[i]; p < G->rp[i + 1]; ++p) if (G->ci[p] > i) ne++;
    oedge *E = malloc(sizeof(oedge) * (ne ? ne : 1));
    ne = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = G->rp[i]; p < G->rp[i + 1]; ++p)
            if (G->ci[p] > i) E[ne++].k = omkkey(G->w[p], i, G->ci[p], salt);
    qsort(E, (size_t)ne, sizeof(oedge), oedge_cmp_desc);
    for (int64_t i = 0; i < n; ++i) mate[i] = -1;
    for (int64_t e = 0; e < ne; ++e) {
        int64_t a = E[e].k.lo, b = E[e].k.hi;
        if (mate[a] < 0 && mate[b] < 0) { mate[a] = (int32_t)b; mate[b] = (int32_t)a; }
    }
    free(E);
}

/* Parallel rule ("handshake"): repeat {every free vertex points to its max-key
 * free neighbour; mutual pairs match} until no free vertex has a free
 * neighbour (A1).  Returns the number of rounds. */
static int omatch_handshake(const ocsr *G, uint64_t salt, int32_t *mate) {
    int64_t n = G->n;
    int32_t *prop = malloc(sizeof(int32_t) * (n ? n : 1));
    for (int64_t i = 0; i < n; ++i) mate[i] = -1;
    int rounds = 0;
    for (;;) {
        int any = 0;
        for (int64_t v = 0; v < n; ++v) {
            prop[v] = -1;
            if (mate[v] >= 0) continue;
            okey best;
            for (int64_t p = G->rp[v]; p < G->rp[v + 1]; ++p) {
                int64_t u = G->ci[p];
                if (mate[u] >= 0) continue;
                okey k = omkkey(G->w[p], v, u, salt);
                if (prop[v] < 0 || okey_gt(k, best)) { best = k; prop[v] = (int32_t)u; }
            }
            if (prop[v] >= 0) any = 1;
        }
        if (!any) break;
        rounds++;
        for (int64_t v = 0; v < n; ++v)
            if (mate[v] < 0 && prop[v] >= 0 && prop[prop[v]] == v) mate[v] = prop[v];
    }
    free(prop);
    return rounds;
}

/* One aggregation pass on pass graph G: matching, attach
 * (A3), numbering by leader rank (A4).  agg[v] in [0, *nc). */
static int oaggregate_pass(const ocsr *G, uint64_t salt, int rule, int32_t *agg, int64_t *nc) {
    int64_t n = G->n;
    int32_t *mate = malloc(sizeof(int32_t) * (n ? n : 1));
    int32_t *leader = malloc(sizeof(int32_t) * (n ? n : 1));
    int rounds = 0;
    if (rule == 0) omatch_greedy(G, salt, mate); else rounds = omatch_handshake(G, salt, mate);
    for (int64_t v = 0; v < n; ++v) {
        if (mate[v] >= 0) {
            leader[v] = (int32_t)(v < mate[v] ? v : mate[v]);
        } else if (G->rp[v + 1] > G->rp[v]) {
            /* attach to the pair of the max-key neighbour; all neighbours are matched (maximality) */
            okey best; int64_t bu = -1;
            for (int64_t p = G->rp[v]; p < G->rp[v + 1]; ++p) {
                okey k = omkkey(G->w[p], v, G->ci[p], salt);
                if (bu < 0 || okey_gt(k, best)) { best = k; bu = G->ci[p]; }
            }
            leader[v] = (int32_t)(bu < mate[bu] ? bu : mate[bu]);
        } else {
            leader[v] = (int32_t)v; /* isolated: singleton */
        }
    }
    /* id = rank of the leader among leaders in increasing vertex order;
     * attached vertices are never leaders (their leader is their pair's min). */
    int32_t *id = malloc(sizeof(int32_t) * (n ? n : 1));
    int64_t c = 0;
    for (int64_t v = 0; v < n; ++v) {
        int is_leader = (mate[v] >= 0) ? (v < mate[v]) : (G->rp[v + 1] == G->rp[v]);
        id[v] = is_leader ? (int32_t)c++ : -1;
    }
    for (int64_t v = 0; v < n; ++v) agg[v] = id[leader[v]];
    *nc = c;
    free(mate); free(leader); free(id);
    return rounds;
}

/* Members of each aggregate in increasing vertex order (stable counting sort). */
static void omembers(int64_t n, const int32_t *agg, int64_t nc, int64_t **ptr_out, int32_t **mem_out) {
    int64_t *ptr = calloc((size_t)nc + 1, sizeof(int64_t));
    int32_t *mem = malloc(sizeof(int32_t) * (n ? n : 1));
    for (int64_t i = 0; i < n; ++i) ptr[agg[i] + 1]++;
    for (int64_t I = 0; I < nc; ++I) ptr[I + 1] += ptr[I];
    int64_t *fill = malloc(sizeof(int64_t) * (nc ? nc : 1));
    memcpy(fill, ptr, sizeof(int64_t) * nc);
    for (int64_t i = 0; i < n; ++i) mem[fill[agg[i]]++] = (int32_t)i;
    free(fill);
    *ptr_out = ptr;
    *mem_out = mem;
}

typedef struct { int32_t j; double v; int64_t w; } oent;
static int oent_cmp(const void *a, const void *b) {
    int32_t x = ((const oent *)a)->j, y = ((const oent *)b)->j;
    return (x > y) - (x < y);
}

/* Quotient of A (values) or of a pass graph (multiplicities) under agg
 * (P:88-95 coarse graph; "simple summations").
 * Entry (I,J) = sum over i in I increasing, then CSR position increasing, of
 * the entries (i,j) with agg(j) = J.  drop_diag: omit I == J (pass graphs). */
static void oquotient(const ocsr *A, const int32_t *agg, int64_t nc, int drop_diag, ocsr *H) {
    int64_t *ptr; int32_t *mem;
    omembers(A->n, agg, nc, &ptr, &mem);
    int64_t *marker = malloc(sizeof(int64_t) * (nc ? nc : 1));
    int64_t *pos = malloc(sizeof(int64_t) * (nc ? nc : 1));
    for (int64_t J = 0; J < nc; ++J) marker[J] = -1;
    int64_t cap = A->nnz + 1, nnz = 0;
    oent *buf = malloc(sizeof(oent) * (size_t)cap);
    int64_t *rp = malloc(sizeof(int64_t) * ((size_t)nc + 1));
    for (int64_t I = 0; I < nc; ++I) {
        rp[I] = nnz;
        for (int64_t t = ptr[I]; t < ptr[I + 1]; ++t) {
            int64_t i = mem[t];
            for (int64_t p = A->rp[i]; p < A->rp[i + 1]; ++p) {
                int32_t J = agg[A->ci[p]];
                if (drop_diag && J == I) continue;
                if (marker[J] != I) {
                    marker[J] = I;
                    pos[J] = nnz;
                    buf[nnz].j = J;
                    buf[nnz].v = A->v ? A->v[p] : 0.0;
                    buf[nnz].w = A->w ? A->w[p] : 0;
                    nnz++;
                } else {
                    if (A->v) buf[pos[J]].v += A->v[p];
                    if (A->w) buf[pos[J]].w += A->w[p];
                }
            }
        }
        qsort(buf + rp[I], (size_t)(nnz - rp[I]), sizeof(oent), oent_cmp);
    }
    rp[nc] = nnz;
    H->n = nc;
    H->nnz = nnz;
    H->rp = rp;
    H->ci = malloc(sizeof(int32_t) * (nnz ? nnz : 1));
    H->v = A->v ? malloc(sizeof(double) * (nnz ? nnz : 1)) : NULL;
    H->w = A->w ? malloc(sizeof(int64_t) * (nnz ? nnz : 1)) : NULL;
    for (int64_t p = 0; p < nnz; ++p) {
        H->ci[p] = buf[p].j;
        if (H->v) H->v[p] = buf[p].v;
        if (H->w) H->w[p] = buf[p].w;
    }
    free(buf); free(marker); free(pos); free(ptr); free(mem);
}

/* Pass graph G_0 of a level: off-diagonal pattern of A with multiplicity 1
 * (A5), minus edges between different blocks when the level is partitioned (A20). */
static void opass_graph0(const ocsr *A, const int32_t *blk, ocsr *G) {
    int64_t n = A->n, nnz = 0;
    G->n = n;
    G->rp = malloc(sizeof(int64_t) * (n + 1));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = A->rp[i]; p < A->rp[i + 1]; ++p)
            if (A->ci[p] != i && blk[A->ci[p]] == blk[i]) nnz++;
    G->nnz = nnz;
    G->ci = malloc(sizeof(int32_t) * (nnz ? nnz : 1));
    G->w = malloc(sizeof(int64_t) * (nnz ? nnz : 1));
    G->v = NULL;
    nnz = 0;
    for (int64_t i = 0; i < n; ++i) {
        G->rp[i] = nnz;
        for (int64_t p = A->rp[i]; p < A->rp[i + 1]; ++p)
            if (A->ci[p] != i && blk[A->ci[p]] == blk[i]) { G->ci[nnz] = A->ci[p]; G->w[nnz] = 1; nnz++; }
    }
    G->rp[n] = nnz;
}

/* ===================================================== MIS-k aggregation (A25) */
/* The paper's own partitioner, reading A25:
 *  (A) S = the maximal independent set of the graph of A^k (vertices at graph distance <= k are
 *      adjacent) chosen greedily by decreasing key: v joins S iff no vertex of S with a larger key is
 *      within distance k.  key(v) = (hi32(splitmix64(v ^ misalt)) << 32) | v, misalt =
 *      splitmix64(seed ^ 0x4D49530000000000 ^ level) (distinct keys: v breaks ties).
 *  (B) "collecting vertices and edges of the neighbors of vertices in S", layer by layer: every S
 *      vertex roots its aggregate (layer 0); in layer d = 1..k every vertex not yet assigned takes,
 *      among its neighbours assigned in layers < d, the root with the largest key.  By maximality of S
 *      every vertex is assigned after k layers; aggregates are connected (each vertex joins through
 *      a neighbour of its own aggregate).  Aggregate id = rank of its root in increasing vertex order.
 * G is the level's pass graph G_0 (off-diagonal pattern). */
static uint64_t omis_key(int64_t v, uint64_t misalt) {
    return ((osm64((uint64_t)v ^ misalt) >> 32) << 32) | (uint64_t)(uint32_t)v;
}

static int64_t omis_aggregate(const ocsr *G, int k, uint64_t seed, int level, int32_t *agg, int8_t *roots_out);
int64_t orc_mis_aggregate(const ocsr *G, int k, uint64_t seed, int level, int32_t *agg) {
    return omis_aggregate(G, k, seed, level, agg, NULL);
}
static int64_t omis_aggregate(const ocsr *G, int k, uint64_t seed, int level, int32_t *agg, int8_t *roots_out) {
    int64_t n = G->n;
    uint64_t misalt = osm64(seed ^ 0x4D49530000000000ULL ^ (uint64_t)level);
    uint64_t *key = malloc(sizeof(uint64_t) * (n ? n : 1));
    int64_t *order = malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t v = 0; v < n; ++v) { key[v] = omis_key(v, misalt); order[v] = v; }
    /* sort vertices by decreasing key (insertion into a heap-free merge: plain qsort with keys) */
    for (int64_t w = 1; w < n; w *= 2) { /* bottom-up merge sort, descending key */
        int64_t *tmp = malloc(sizeof(int64_t) * n);
        for (int64_t lo = 0; lo < n; lo += 2 * w) {
            int64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n, a = lo, b = mid, o = lo;
            while (a < mid && b < hi) tmp[o++] = key[order[a]] > key[order[b]] ? order[a++] : order[b++];
            while (a < mid) tmp[o++] = order[a++];
            while (b < hi) tmp[o++] = order[b++];
        }
        memcpy(order, tmp, sizeof(int64_t) * n);
        free(tmp);
    }
    char *inS = calloc((size_t)n + 1, 1);
    int64_t *dist = malloc(sizeof(int64_t) * (n ? n : 1)), *queue = malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t v = 0; v < n; ++v) dist[v] = -1;
    for (int64_t t = 0; t < n; ++t) { /* (A): greedy by decreasing key; BFS of depth k from v */
        int64_t v = order[t], qh = 0, qt = 0;
        int blocked = 0;
        queue[qt++] = v;
        dist[v] = 0;
        while (qh < qt && !blocked) {
            int64_t u = queue[qh++];
            if (inS[u]) { blocked = 1; break; }
            if (dist[u] == k) continue;
            for (int64_t p = G->rp[u]; p < G->rp[u + 1]; ++p) {
                int64_t x = G->ci[p];
                if (dist[x] < 0) { dist[x] = dist[u] + 1; queue[qt++] = x; }
            }
        }
        for (int64_t q = 0; q < qt; ++q) dist[queue[q]] = -1;
        if (!blocked) inS[v] = 1;
    }
    /* (B): layered growth */
    int64_t *root = malloc(sizeof(int64_t) * (n ? n : 1)), *nroot = malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t v = 0; v < n; ++v) root[v] = inS[v] ? v : -1;
    for (int d = 1; d <= k; ++d) {
        for (int64_t v = 0; v < n; ++v) {
            nroot[v] = root[v];
            if (root[v] >= 0) continue;
            int64_t best = -1;
            for (int64_t p = G->rp[v]; p < G->rp[v + 1]; ++p) {
                int64_t r = root[G->ci[p]];
                if (r >= 0 && (best < 0 || key[r] > key[best])) best = r;
            }
            nroot[v] = best;
        }
        memcpy(root, nroot, sizeof(int64_t) * n);
    }
    if (roots_out) for (int64_t v = 0; v < n; ++v) roots_out[v] = inS[v];
    int64_t nc = 0;
    int32_t *id = malloc(sizeof(int32_t) * (n ? n : 1));
    for (int64_t v = 0; v < n; ++v) id[v] = inS[v] ? (int32_t)nc++ : -1;
    int64_t ok = nc;
    for (int64_t v = 0; v < n; ++v) {
        if (root[v] < 0) { ok = -1; agg[v] = -1; continue; } /* unreachable by maximality */
        agg[v] = id[root[v]];
    }
    free(key); free(order); free(inS); free(dist); free(queue); free(root); free(nroot); free(id);
    return ok;
}

/* test hook: MIS-k aggregation of a CSR pattern (off-diagonals) */
int64_t orc_mis_aggregate_csr(int64_t n, const int64_t *rp, const int32_t *ci, int k, uint64_t seed, int level,
                              int32_t *agg, int8_t *roots) {
    ocsr A = {n, rp[n], (int64_t *)rp, (int32_t *)ci, NULL, NULL}, G;
    int32_t *blk = calloc((size_t)n + 1, sizeof(int32_t));
    opass_graph0(&A, blk, &G);
    int64_t nc = omis_aggregate(&G, k, seed, level, agg, roots);
    ocsr_free(&G);
    free(blk);
    return nc;
}

/* ================================================================ hierarchy */
typedef struct {
    ocsr A;
    double lambda1, kappa;
    double alpha[ORC_MAXDEG + 1], beta[ORC_MAXDEG + 1];
    int32_t *agg;   /* fine -> coarse map to level l+1 (NULL on the coarsest) */
    int64_t nc;
    int32_t *blk;   /* block id of each row (decoupled aggregation, A20) */
    int nparts;
    int match_rounds[ORC_MAXDEG];
} olevel;

typedef struct {
    int nlev, m, singular;
    int64_t coarsest_size;
    double kappa_opt;
    int restart, max_iter, rule, cycle, nparts;
    double amli_kappa; /* cycle 2: 1/theta of the AMLI polynomial interval; 0 = reading A23 */
    int lanczos;       /* reading A24: k Lanczos steps for lambda_1 (0 = ||A||_inf, the paper's) */
    int mis_k;         /* reading A25: 0 = repeated pairwise matching (A1-A5); k > 0 = MIS of A^k */
    int64_t gather_rows;
    uint64_t seed;
    olevel lev[ORC_MAXLEV];
    /* coarsest level: dense Cholesky factor (lower, row-major) of A_L (SPD) or
     * of A_L + (s/n_L) 1 1^T with s = ||A_L||_inf (singular), SURVEY 8(c) O4 / S:84. */
    double *chol;
    double shift;
} orc_h;

/* Dense Cholesky A = L L^T in place (lower triangle), A row-major n x n. */
static int ochol(int64_t n, double *a) {
    for (int64_t j = 0; j < n; ++j) {
        double s = a[j * n + j];
        for (int64_t k = 0; k < j; ++k) s -= a[j * n + k] * a[j * n + k];
        if (!(s > 0.0)) return -1;
        a[j * n + j] = sqrt(s);
        for (int64_t i = j + 1; i < n; ++i) {
            double t = a[i * n + j];
            for (int64_t k = 0; k < j; ++k) t -= a[i * n + k] * a[j * n + k];
            a[i * n + j] = t / a[j * n + j];
        }
    }
    return 0;
}

/* e = A_L^{-1} r, or A_L^dagger r for the singular case: project r to mean
 * zero, solve with (A_L + (s/n) 1 1^T), project the result. */
static void ocoarse_solve(const orc_h *h, const double *r, double *e) {
    const olevel *L = &h->lev[h->nlev - 1];
    int64_t n = L->A.n;
    double *y = malloc(sizeof(double) * n);
    memcpy(y, r, sizeof(double) * n);
    if (h->singular) {
        double mu = 0.0;
        for (int64_t i = 0; i < n; ++i) mu += y[i];
        mu /= (double)n;
        for (int64_t i = 0; i < n; ++i) y[i] -= mu;
    }
    for (int64_t i = 0; i < n; ++i) { /* forward: L y = r */
        double s = y[i];
        for (int64_t k = 0; k < i; ++k) s -= h->chol[i * n + k] * y[k];
        y[i] = s / h->chol[i * n + i];
    }
    for (int64_t i = n - 1; i >= 0; --i) { /* backward: L^T e = y */
        double s = y[i];
        for (int64_t k = i + 1; k < n; ++k) s -= h->chol[k * n + i] * y[k];
        y[i] = s / h->chol[i * n + i];
    }
    if (h->singular) {
        double mu = 0.0;
        for (int64_t i = 0; i < n; ++i) mu += y[i];
        mu /= (double)n;
        for (int64_t i = 0; i < n; ++i) y[i] -= mu;
    }
    memcpy(e, y, sizeof(double) * n);
    free(y);
}

/* Validates the input (reading A17) and forms A_0 = L + diag(d)
 * (Eq. (prob)).  Missing diagonals are inserted as sum_{j!=i} w_ij. */
static int oform_A0(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                    const double *d, ocsr *A) {
    if (n <= 0 || rp[0] != 0) return ORC_E_INPUT;
    for (int64_t i = 0; i < n; ++i) {
        if (rp[i + 1] < rp[i]) return ORC_E_INPUT;
        double off = 0.0; int has_diag = 0; double dv = 0.0;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            if (ci[p] < 0 || ci[p] >= n) return ORC_E_INPUT;
            if (p > rp[i] && ci[p] <= ci[p - 1]) return ORC_E_INPUT;
            if (ci[p] == i) { has_diag = 1; dv = val[p]; continue; }
            if (!(val[p] <= 0.0)) return ORC_E_INPUT; /* weights w_e >= 0: structural zeros allowed (A17) */
            off += -val[p];
            /* symmetry: (j,i) stored with equal value */
            int64_t j = ci[p], lo = rp[j], hi = rp[j + 1], f = -1;
            while (lo < hi) { int64_t mid = (lo + hi) / 2; if (ci[mid] < i) lo = mid + 1; else hi = mid; }
            if (lo < rp[j + 1] && ci[lo] == i) f = lo;
            if (f < 0 || val[f] != val[p]) return ORC_E_INPUT;
        }
        if (has_diag && fabs(dv - off) > 1e-10 * (fabs(dv) + off)) return ORC_E_INPUT;
        if (d && !(d[i] >= 0.0)) return ORC_E_INPUT;
    }
    int64_t nnz = 0;
    for (int64_t i = 0; i < n; ++i) {
        int has = 0;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) has |= (ci[p] == i);
        nnz += rp[i + 1] - rp[i] + (has ? 0 : 1);
    }
    A->n = n; A->nnz = nnz;
    A->rp = malloc(sizeof(int64_t) * (n + 1));
    A->ci = malloc(sizeof(int32_t) * nnz);
    A->v = malloc(sizeof(double) * nnz);
    A->w = NULL;
    int64_t q = 0;
    for (int64_t i = 0; i < n; ++i) {
        A->rp[i] = q;
        int has = 0; double off = 0.0;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) { has |= (ci[p] == i); if (ci[p] != i) off += -val[p]; }
        int done = has;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            if (!done && ci[p] > i) { A->ci[q] = (int32_t)i; A->v[q] = off + (d ? d[i] : 0.0); q++; done = 1; }
            A->ci[q] = ci[p];
            A->v[q] = (ci[p] == i) ? val[p] + (d ? d[i] : 0.0) : val[p];
            q++;
        }
        if (!done) { A->ci[q] = (int32_t)i; A->v[q] = off + (d ? d[i] : 0.0); q++; }
    }
    A->rp[n] = q;
    return ORC_OK;
}

void orc_free(orc_h *h) {
    if (!h) return;
    for (int l = 0; l < h->nlev; ++l) {
        ocsr_free(&h->lev[l].A);
        free(h->lev[l].agg);
        free(h->lev[l].blk);
    }
    free(h->chol);
    free(h);
}

static int orc_get_lanczos(void);
static int orc_get_mis_k(void);

/* Setup: level loop while n_l > coarsest_size:
 * lambda_1, kappa rule (A8), coefficients, p matching passes composed
 * into agg_l, Galerkin A_{l+1} = P^T A_l P, then the dense coarsest. */
int orc_setup(int64_t n, const int64_t *rp, const int32_t *ci, const double *val, const double *d,
              int passes, int degree, int64_t coarsest_size, double kappa, int restart, int max_iter,
              uint64_t seed, int nparts, int64_t gather_rows, int rule, int cycle, orc_h **out) {
    *out = NULL;
    if (passes < 1 || degree < 1 || degree > ORC_MAXDEG || coarsest_size < 1 || restart < 1 ||
        max_iter < 0 || nparts < 1 || (kappa != 0.0 && !(kappa > 1.0)))
        return ORC_E_ARG;
    if (kappa > 1.0 && !(orc_Em(degree, kappa) < 1.0)) return ORC_E_ARG; /* A9 */
    orc_h *h = calloc(1, sizeof(orc_h));
    h->m = degree; h->coarsest_size = coarsest_size; h->kappa_opt = kappa;
    h->restart = restart; h->max_iter = max_iter; h->seed = seed; h->nparts = nparts;
    h->gather_rows = gather_rows; h->rule = rule; h->cycle = cycle;
    h->lanczos = orc_get_lanczos();
    h->mis_k = orc_get_mis_k();
    int st = oform_A0(n, rp, ci, val, d, &h->lev[0].A);
    if (st) { free(h); return st; }
    h->singular = 1;
    if (d) for (int64_t i = 0; i < n; ++i) if (d[i] != 0.0) { h->singular = 0; break; }
    /* level-0 blocks: block b owns rows [floor(b n/P), floor((b+1) n/P)) (O1) */
    h->lev[0].blk = malloc(sizeof(int32_t) * n);
    for (int b = 0; b < nparts; ++b)
        for (int64_t i = (int64_t)b * n / nparts; i < (int64_t)(b + 1) * n / nparts; ++i) h->lev[0].blk[i] = b;
    int distributed = nparts > 1;
    int l = 0;
    for (;;) {
        olevel *L = &h->lev[l];
        L->lambda1 = oinf_norm(&L->A);
        if (h->lanczos > 0 && L->A.n > coarsest_size) { /* reading A24 (smoothed levels only) */
            double t = 1.1 * orc_lanczos_max(L->A.n, L->A.rp, L->A.ci, L->A.v, h->lanczos, seed, l);
            if (t < L->lambda1) L->lambda1 = t;
        }
        L->kappa = kappa > 1.0 ? kappa : orc_kappa_rule(degree);
        orc_poly_coeffs(L->lambda1, L->kappa, degree, L->alpha, L->beta);
        if (L->A.n <= coarsest_size) break;
        if (l + 1 >= ORC_MAXLEV) { orc_free(h); h = NULL; return ORC_E_SETUP; }
        /* nparts_l = P while n_l >= gather_rows, else 1 (and stays 1) (O1) */
        if (distributed && L->A.n < gather_rows) distributed = 0;
        L->nparts = distributed ? nparts : 1;
        if (!distributed) for (int64_t i = 0; i < L->A.n; ++i) L->blk[i] = 0;
        ocsr G;
        opass_graph0(&L->A, L->blk, &G);
        int32_t *agg = malloc(sizeof(int32_t) * L->A.n);
        int32_t *gblk = malloc(sizeof(int32_t) * L->A.n);
        for (int64_t i = 0; i < L->A.n; ++i) { agg[i] = (int32_t)i; gblk[i] = L->blk[i]; }
        int64_t nc = L->A.n;
        if (h->mis_k > 0) { /* reading A25: one MIS-k aggregation replaces the matching passes */
            int64_t ncm = orc_mis_aggregate(&G, h->mis_k, seed, l, agg);
            if (ncm < 0) { ocsr_free(&G); free(agg); free(gblk); orc_free(h); return ORC_E_SETUP; }
            int32_t *nblk = malloc(sizeof(int32_t) * (ncm ? ncm : 1));
            for (int64_t v = 0; v < L->A.n; ++v) nblk[agg[v]] = gblk[v];
            free(gblk); gblk = nblk;
            nc = ncm;
        }
        for (int t = 0; t < (h->mis_k > 0 ? 0 : passes); ++t) {
            int32_t *aggt = malloc(sizeof(int32_t) * (G.n ? G.n : 1));
            int64_t nct;
            uint64_t salt = osalt(seed, l, t);
            L->match_rounds[t] = oaggregate_pass(&G, salt, rule, aggt, &nct);
            int32_t *nblk = malloc(sizeof(int32_t) * (nct ? nct : 1));
            for (int64_t v = 0; v < G.n; ++v) nblk[aggt[v]] = gblk[v];
            free(gblk); gblk = nblk;
            for (int64_t i = 0; i < L->A.n; ++i) agg[i] = aggt[agg[i]]; /* compose (O3d) */
            if (t + 1 < passes) {
                ocsr G2;
                oquotient(&G, aggt, nct, 1, &G2);
                ocsr_free(&G);
                G = G2;
            }
            nc = nct;
            free(aggt);
        }
        ocsr_free(&G);
        if (nc >= L->A.n) { free(agg); free(gblk); orc_free(h); return ORC_E_SETUP; } /* stagnation */
        L->agg = agg;
        L->nc = nc;
        olevel *C = &h->lev[l + 1];
        oquotient(&L->A, agg, nc, 0, &C->A); /* Galerkin (O3e) */
        C->blk = gblk;
        l++;
    }
    h->nlev = l + 1;
    /* coarsest (O4) */
    {
        olevel *L = &h->lev[l];
        int64_t nL = L->A.n;
        h->chol = calloc((size_t)(nL * nL), sizeof(double));
        for (int64_t i = 0; i < nL; ++i)
            for (int64_t p = L->A.rp[i]; p < L->A.rp[i + 1]; ++p) h->chol[i * nL + L->A.ci[p]] = L->A.v[p];
        if (h->singular) {
            double s = L->lambda1 > 0.0 ? L->lambda1 : 1.0;
            h->shift = s;
            for (int64_t i = 0; i < nL * nL; ++i) h->chol[i] += s / (double)nL;
        }
        if (ochol(nL, h->chol)) { orc_free(h); return ORC_E_SETUP; }
    }
    *out = h;
    return ORC_OK;
}

/* ================================================================ cycles */
static void oB(const orc_h *h, int l, int nu, const double *r, double *x);

/* FCG_inner(l, b, nu) ("NPCG applied recursively"):
 * e = 0, rho = b; for i < nu: z = B_l(rho); d_i = z - sum_{j<i} (z.q_j)/(d_j.q_j) d_j;
 * q_i = A d_i; alpha = (d_i.rho)/(d_i.q_i); e += alpha d_i; rho -= alpha q_i. */
static void ofcg_inner(const orc_h *h, int l, int nu, const double *b, double *e) {
    const ocsr *A = &h->lev[l].A;
    int64_t n = A->n;
    double *rho = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n);
    double *D = malloc(sizeof(double) * n * nu), *Q = malloc(sizeof(double) * n * nu);
    double *dq = malloc(sizeof(double) * nu);
    memcpy(rho, b, sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i) e[i] = 0.0;
    for (int i = 0; i < nu; ++i) {
        double *d = D + (int64_t)i * n, *q = Q + (int64_t)i * n;
        oB(h, l, nu, rho, z);
        memcpy(d, z, sizeof(double) * n);
        for (int j = 0; j < i; ++j) {
            /* d_j = 0 (only when rho was 0, reading A13) gives d_j.q_j = 0: that direction adds nothing */
            double beta = dq[j] != 0.0 ? odot(n, z, Q + (int64_t)j * n) / dq[j] : 0.0;
            for (int64_t k = 0; k < n; ++k) d[k] -= beta * D[(int64_t)j * n + k];
        }
        ospmv(A, d, q);
        dq[i] = odot(n, d, q);
        double alpha = dq[i] != 0.0 ? odot(n, d, rho) / dq[i] : 0.0; /* rho = 0 => d = 0 */
        for (int64_t k = 0; k < n; ++k) e[k] += alpha * d[k];
        for (int64_t k = 0; k < n; ++k) rho[k] -= alpha * q[k];
    }
    free(rho); free(z); free(D); free(Q); free(dq);
}

/* k-cycle B_l(r) (P:108-114 two-level step, W(1,1) P:394,
 * readings A10-A12):  x = S_l(r, 0); rho_H = P^T(r - A x);
 * e = A_L^{-1/dagger} rho_H if l+1 is the coarsest, else FCG_inner(l+1, rho_H, nu)
 * (cycle=1: B_{l+1}(rho_H), the linear test-only V-cycle); x += P e; x = S_l(r, x). */
/* Stationary AMLI coarse correction (cycle 2; "we use the polynomial based on the best
 * approximation to x^{-1} in the uniform norm to form the preconditioner between any two successive
 * levels"; reading A23):  e = q(B_l A_l) B_l rho, q = the degree-(nu-1) best uniform
 * approximation to 1/t on [1/kappa_A, 1] (the smoother's family, on the preconditioned
 * operator), evaluated by the smoother's three-term recurrence applied to B_l A_l y = B_l rho:
 *   y_0 = 0,  y_{k+1} = alpha_k y_k + (1 - alpha_k) y_{k-1} + beta_k B_l(rho - A_l y_k),  k = 0..nu-1,
 * i.e. nu applications of B_l and nu-1 SpMVs; kappa_A = rule R1 (A8) for degree nu-1 unless set.
 * nu = 1: e = B_l rho (no polynomial: the V-cycle). */
static void oamli(const orc_h *h, int l, int nu, const double *rho, double *e) {
    const ocsr *A = &h->lev[l].A;
    int64_t n = A->n;
    if (nu == 1) { oB(h, l, nu, rho, e); return; }
    int m = nu - 1;
    double kap = h->amli_kappa > 1.0 ? h->amli_kappa : orc_kappa_rule(m);
    double alpha[ORC_MAXDEG + 1], beta[ORC_MAXDEG + 1];
    orc_poly_coeffs(1.0, kap, m, alpha, beta);
    double *ym1 = calloc((size_t)n, sizeof(double)), *yk = calloc((size_t)n, sizeof(double));
    double *t = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n);
    for (int k = 0; k <= m; ++k) {
        ospmv(A, yk, t);
        for (int64_t i = 0; i < n; ++i) t[i] = rho[i] - t[i];
        oB(h, l, nu, t, z);
        for (int64_t i = 0; i < n; ++i) {
            double yn = alpha[k] * yk[i] + (1.0 - alpha[k]) * ym1[i] + beta[k] * z[i];
            ym1[i] = yk[i];
            yk[i] = yn;
        }
    }
    memcpy(e, yk, sizeof(double) * n);
    free(ym1); free(yk); free(t); free(z);
}

static void oB(const orc_h *h, int l, int nu, const double *r, double *x) {
    if (l == h->nlev - 1) { ocoarse_solve(h, r, x); return; }
    const olevel *L = &h->lev[l];
    int64_t n = L->A.n, nc = L->nc;
    double *zero = calloc((size_t)n, sizeof(double)), *t = malloc(sizeof(double) * n);
    double *rH = calloc((size_t)nc, sizeof(double)), *eH = malloc(sizeof(double) * nc);
    osmooth(&L->A, h->m, L->alpha, L->beta, r, zero, x);
    ospmv(&L->A, x, t);
    for (int64_t i = 0; i < n; ++i) rH[L->agg[i]] += r[i] - t[i]; /* P^T, i increasing */
    if (l + 1 == h->nlev - 1) ocoarse_solve(h, rH, eH);
    else if (h->cycle == 1) oB(h, l + 1, nu, rH, eH);
    else if (h->cycle == 2) oamli(h, l + 1, nu, rH, eH);
    else ofcg_inner(h, l + 1, nu, rH, eH);
    for (int64_t i = 0; i < n; ++i) x[i] += eH[L->agg[i]];
    osmooth(&L->A, h->m, L->alpha, L->beta, r, x, x);
    free(zero); free(t); free(rH); free(eH);
}

static const double *orc_get_xstar(void);
/* ||x - x*||_A = sqrt((x - x*)^T A (x - x*)) */
static double oanorm_err(const ocsr *A, const double *x, const double *xs) {
    int64_t n = A->n;
    double *e = malloc(sizeof(double) * n), *t = malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i) e[i] = x[i] - xs[i];
    ospmv(A, e, t);
    double v = odot(n, e, t);
    free(e); free(t);
    return sqrt(v > 0.0 ? v : 0.0);
}

/* Outer flexible CG (P:322-323 restart every 5; stopping
 * reading A14: ||r|| <= tol ||b|| on the recursive residual; or, when an exact solution x* is set
 * (orc_set_xstar), the paper's rule: ||x - x*||_A <= tol ||x_0 - x*||_A). */
int orc_solve(const orc_h *h, const double *b_in, double *x, double tol, int nu,
              int *iters_out, double *relres_out, double *true_relres_out) {
    if (!h || !(tol > 0.0) || nu < 1) return ORC_E_ARG;
    const ocsr *A = &h->lev[0].A;
    int64_t n = A->n;
    int W = h->restart;
    double *b = malloc(sizeof(double) * n), *r = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n);
    double *D = malloc(sizeof(double) * n * W), *Q = malloc(sizeof(double) * n * W);
    double *dq = malloc(sizeof(double) * W), *t = malloc(sizeof(double) * n);
    memcpy(b, b_in, sizeof(double) * n);
    if (h->singular) { /* b <- b - mean(b) (A16) */
        double mu = 0.0;
        for (int64_t i = 0; i < n; ++i) mu += b[i];
        mu /= (double)n;
        for (int64_t i = 0; i < n; ++i) b[i] -= mu;
    }
    double bnorm = sqrt(odot(n, b, b));
    const double *xstar = orc_get_xstar();
    double e0A = xstar ? oanorm_err(A, x, xstar) : 0.0;
    int status = ORC_NOT_CONVERGED, k = 0, w = 0;
    if (bnorm == 0.0) {
        for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
        status = ORC_OK;
    } else {
        ospmv(A, x, t);
        for (int64_t i = 0; i < n; ++i) r[i] = b[i] - t[i];
        for (k = 0;; ++k) {
            if (xstar ? oanorm_err(A, x, xstar) <= tol * e0A : sqrt(odot(n, r, r)) <= tol * bnorm) {
                status = ORC_OK;
                break;
            }
            if (k >= h->max_iter) break;
            oB(h, 0, nu, r, z);
            if (h->singular) {
                double mu = 0.0;
                for (int64_t i = 0; i < n; ++i) mu += z[i];
                mu /= (double)n;
                for (int64_t i = 0; i < n; ++i) z[i] -= mu;
            }
            double *d = D + (int64_t)w * n, *q = Q + (int64_t)w * n;
            memcpy(d, z, sizeof(double) * n);
            for (int j = 0; j < w; ++j) {
                double beta = odot(n, z, Q + (int64_t)j * n) / dq[j];
                for (int64_t i = 0; i < n; ++i) d[i] -= beta * D[(int64_t)j * n + i];
            }
            ospmv(A, d, q);
            dq[w] = odot(n, d, q);
            if (!(dq[w] > 0.0)) { status = ORC_E_BREAKDOWN; break; }
            double alpha = odot(n, d, r) / dq[w];
            for (int64_t i = 0; i < n; ++i) x[i] += alpha * d[i];
            for (int64_t i = 0; i < n; ++i) r[i] -= alpha * q[i];
            w++;
            if (w == W) w = 0; /* restart: window emptied, x and r kept */
        }
    }
    if (iters_out) *iters_out = k;
    if (relres_out) *relres_out = bnorm > 0.0 ? sqrt(odot(n, r, r)) / bnorm : 0.0;
    if (true_relres_out) {
        ospmv(A, x, t);
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += (b[i] - t[i]) * (b[i] - t[i]);
        *true_relres_out = bnorm > 0.0 ? sqrt(s) / bnorm : 0.0;
    }
    free(b); free(r); free(z); free(D); free(Q); free(dq); free(t);
    return status;
}

/* ================================================= exported accessors / pieces */
int orc_num_levels(const orc_h *h) { return h->nlev; }
/* reading A24: k Lanczos steps for lambda_1 in subsequent orc_setup calls of this thread (0 = off) */
static _Thread_local int g_lanczos = 0;
void orc_set_lanczos(int k) { g_lanczos = k; }
/* reading A25: MIS-k aggregation in subsequent orc_setup calls of this thread (0 = matching) */
static _Thread_local int g_mis_k = 0;
void orc_set_mis_k(int k) { g_mis_k = k; }
/* A-norm stopping (the paper's protocol): when set, orc_solve stops on
 * ||x - x*||_A <= tol ||x_0 - x*||_A instead of the residual (reading A14) */
static _Thread_local const double *g_xstar = NULL;
void orc_set_xstar(const double *xs) { g_xstar = xs; }
/* cycle 2 (stationary AMLI): 1/theta of the coarse polynomial interval (0 = reading A23) */
void orc_set_amli_kappa(orc_h *h, double kappa) { h->amli_kappa = kappa; }
int orc_is_singular(const orc_h *h) { return h->singular; }

void orc_level_info(const orc_h *h, int l, int64_t *n, int64_t *nnz, double *lambda1, double *kappa, int64_t *nc,
                    int *nparts) {
    const olevel *L = &h->lev[l];
    *n = L->A.n; *nnz = L->A.nnz; *lambda1 = L->lambda1; *kappa = L->kappa;
    *nc = (l < h->nlev - 1) ? L->nc : 0;
    *nparts = L->nparts ? L->nparts : 1;
}

void orc_level_csr(const orc_h *h, int l, int64_t *rp, int32_t *ci, double *v) {
    const ocsr *A = &h->lev[l].A;
    memcpy(rp, A->rp, sizeof(int64_t) * (A->n + 1));
    memcpy(ci, A->ci, sizeof(int32_t) * A->nnz);
    memcpy(v, A->v, sizeof(double) * A->nnz);
}

void orc_level_agg(const orc_h *h, int l, int32_t *agg) {
    memcpy(agg, h->lev[l].agg, sizeof(int32_t) * h->lev[l].A.n);
}

void orc_level_coeffs(const orc_h *h, int l, double *alpha, double *beta) {
    memcpy(alpha, h->lev[l].alpha, sizeof(double) * (h->m + 1));
    memcpy(beta, h->lev[l].beta, sizeof(double) * (h->m + 1));
}

void orc_level_rounds(const orc_h *h, int l, int *rounds, int passes) {
    for (int t = 0; t < passes && t < ORC_MAXDEG; ++t) rounds[t] = h->lev[l].match_rounds[t];
}

/* S_l(f, x0) on a level of a hierarchy. */
void orc_level_smooth(const orc_h *h, int l, const double *f, const double *x0, double *x) {
    const olevel *L = &h->lev[l];
    osmooth(&L->A, h->m, L->alpha, L->beta, f, x0, x);
}

/* One preconditioner application z = B_l(r) (test hook for SURVEY T3). */
void orc_level_precond(const orc_h *h, int l, int nu, const double *r, double *z) { oB(h, l, nu, r, z); }

void orc_coarse_solve(const orc_h *h, const double *r, double *e) { ocoarse_solve(h, r, e); }

/* ---- standalone building blocks on caller CSR (for the pins) ---- */
static ocsr owrap(int64_t n, int64_t nnz, const int64_t *rp, const int32_t *ci, const double *v, const int64_t *w) {
    ocsr a;
    a.n = n; a.nnz = nnz; a.rp = (int64_t *)rp; a.ci = (int32_t *)ci; a.v = (double *)v; a.w = (int64_t *)w;
    return a;
}

double orc_inf_norm(int64_t n, const int64_t *rp, const int32_t *ci, const double *v) {
    ocsr a = owrap(n, rp[n], rp, ci, v, NULL);
    return oinf_norm(&a);
}

void orc_spmv(int64_t n, const int64_t *rp, const int32_t *ci, const double *v, const double *x, double *y) {
    ocsr a = owrap(n, rp[n], rp, ci, v, NULL);
    ospmv(&a, x, y);
}

void orc_smooth(int64_t n, const int64_t *rp, const int32_t *ci, const double *v, int m, const double *alpha,
                const double *beta, const double *f, const double *x0, double *x) {
    ocsr a = owrap(n, rp[n], rp, ci, v, NULL);
    osmooth(&a, m, alpha, beta, f, x0, x);
}

/* Matching on a pass graph with multiplicities w; rule 0 edge-greedy, 1 handshake. */
int orc_match(int64_t n, const int64_t *rp, const int32_t *ci, const int64_t *w, uint64_t seed, int level, int pass,
              int rule, int32_t *mate) {
    ocsr g = owrap(n, rp[n], rp, ci, NULL, w);
    uint64_t s = osalt(seed, level, pass);
    if (rule == 0) { omatch_greedy(&g, s, mate); return 0; }
    return omatch_handshake(&g, s, mate);
}

int64_t orc_aggregate_pass(int64_t n, const int64_t *rp, const int32_t *ci, const int64_t *w, uint64_t seed,
                           int level, int pass, int rule, int32_t *agg) {
    ocsr g = owrap(n, rp[n], rp, ci, NULL, w);
    int64_t nc;
    oaggregate_pass(&g, osalt(seed, level, pass), rule, agg, &nc);
    return nc;
}

uint64_t orc_edge_hash(uint64_t seed, int level, int pass, int64_t a, int64_t b) {
    return omkkey(0, a, b, osalt(seed, level, pass)).h;
}

/* Quotient / Galerkin of a caller CSR under agg; result via orc_csr_* getters. */
void *orc_quotient(int64_t n, const int64_t *rp, const int32_t *ci, const double *v, const int64_t *w,
                   const int32_t *agg, int64_t nc, int drop_diag) {
    ocsr a = owrap(n, rp[n], rp, ci, v, w);
    ocsr *H = calloc(1, sizeof(ocsr));
    oquotient(&a, agg, nc, drop_diag, H);
    return H;
}

void orc_csr_sizes(const void *H, int64_t *n, int64_t *nnz) {
    *n = ((const ocsr *)H)->n;
    *nnz = ((const ocsr *)H)->nnz;
}

void orc_csr_fetch(const void *Hv, int64_t *rp, int32_t *ci, double *v, int64_t *w) {
    const ocsr *H = Hv;
    memcpy(rp, H->rp, sizeof(int64_t) * (H->n + 1));
    memcpy(ci, H->ci, sizeof(int32_t) * H->nnz);
    if (v && H->v) memcpy(v, H->v, sizeof(double) * H->nnz);
    if (w && H->w) memcpy(w, H->w, sizeof(int64_t) * H->nnz);
}

void orc_csr_free(void *H) {
    ocsr_free((ocsr *)H);
    free(H);
}

static int orc_get_lanczos(void) { return g_lanczos; }
static int orc_get_mis_k(void) { return g_mis_k; }
static const double *orc_get_xstar(void) { return g_xstar; }
