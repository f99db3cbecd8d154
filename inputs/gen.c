/*
 * inputs/gen.c -- seeded synthetic workload generators (BASELINE.json configs C1-C5).
 *
 * This module is shared by the oracle tests, the GPU parity tests and bench.py.
 * It holds NONE of the method's arithmetic: it only builds the problem of
 * PAPER.md Eq. (prob) (lines 26-30): the weighted graph Laplacian L of a graph
 * (stored as CSR with its diagonal, sorted columns) and the lower-order terms
 * d_i (Dirichlet boundary contributions), plus the seeded
 * right-hand side.  The solver (oracle or CUDA) forms A = L + diag(d) itself.
 *
 * Recipes:
 *   grid2d(n):  n x n interior nodes of the unit square, natural order (x fastest).
 *               P1 FE on the uniform right-triangle mesh = 5-point stencil (4,-1);
 *               L = interior grid-graph Laplacian (diag = #interior neighbours),
 *               d_i = #Dirichlet neighbours (1 on edges, 2 at corners).
 *   grid3d(n):  n^3 interior nodes of the unit cube, Kuhn 6-tet P1 FE = 7-point
 *               stencil times h, h = 1/(n+1): off-diagonal fl(-h),
 *               diag fl(h*deg), d_i = fl(h*#Dirichlet neighbours) (single roundings).
 *   rgg(N):     N points uniform in the unit square from the counter RNG below,
 *               edge iff squared distance < r^2, r = sqrt(8/(pi N)), unit weights,
 *               vertices ordered by cell (cy*nc+cx, cell side 1/nc >= r) stable by
 *               point index, largest connected component kept (in that order).
 *   rhs(n):     b_i = 2*u(seed ^ (offset+i)) - 1, u(z) = (splitmix64(z) >> 11) * 2^-53.
 *
 * splitmix64(z): the standard SplitMix64 output for state z:
 *   z += 0x9E3779B97F4A7C15; z = (z^(z>>30))*0xBF58476D1CE4E5B9;
 *   z = (z^(z>>27))*0x94D049BB133111EB; return z^(z>>31).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

static uint64_t gen_sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static double gen_u01(uint64_t z) { return (double)(gen_sm64(z) >> 11) * 0x1.0p-53; }

/* ---------------------------------------------------------------- rhs */
void gen_rhs(int64_t n, uint64_t seed, int64_t offset, double *b) {
    for (int64_t i = 0; i < n; ++i) b[i] = 2.0 * gen_u01(seed ^ (uint64_t)(offset + i)) - 1.0;
}

/* ---------------------------------------------------------------- 2D grid */
int64_t gen_grid2d_nnz(int64_t n) { return n * n + 4 * n * (n - 1); }

/* rp[n*n+1], ci[nnz], val[nnz], d[n*n] caller-allocated. */
void gen_grid2d(int64_t n, int64_t *rp, int32_t *ci, double *val, double *d) {
    int64_t p = 0;
    for (int64_t iy = 0; iy < n; ++iy)
        for (int64_t ix = 0; ix < n; ++ix) {
            int64_t i = iy * n + ix;
            int deg = (iy > 0) + (ix > 0) + (ix < n - 1) + (iy < n - 1);
            rp[i] = p;
            if (iy > 0)     { ci[p] = (int32_t)(i - n); val[p++] = -1.0; }
            if (ix > 0)     { ci[p] = (int32_t)(i - 1); val[p++] = -1.0; }
            ci[p] = (int32_t)i; val[p++] = (double)deg;
            if (ix < n - 1) { ci[p] = (int32_t)(i + 1); val[p++] = -1.0; }
            if (iy < n - 1) { ci[p] = (int32_t)(i + n); val[p++] = -1.0; }
            d[i] = (double)(4 - deg);
        }
    rp[n * n] = p;
}

/* ---------------------------------------------------------------- 3D grid */
int64_t gen_grid3d_nnz(int64_t n) { return n * n * n + 6 * n * n * (n - 1); }

void gen_grid3d(int64_t n, int64_t *rp, int32_t *ci, double *val, double *d) {
    const double h = 1.0 / (double)(n + 1);
    const int64_t n2 = n * n;
    int64_t p = 0;
    for (int64_t iz = 0; iz < n; ++iz)
        for (int64_t iy = 0; iy < n; ++iy)
            for (int64_t ix = 0; ix < n; ++ix) {
                int64_t i = iz * n2 + iy * n + ix;
                int deg = (iz > 0) + (iy > 0) + (ix > 0) + (ix < n - 1) + (iy < n - 1) + (iz < n - 1);
                rp[i] = p;
                if (iz > 0)     { ci[p] = (int32_t)(i - n2); val[p++] = -h; }
                if (iy > 0)     { ci[p] = (int32_t)(i - n);  val[p++] = -h; }
                if (ix > 0)     { ci[p] = (int32_t)(i - 1);  val[p++] = -h; }
                ci[p] = (int32_t)i; val[p++] = h * (double)deg;
                if (ix < n - 1) { ci[p] = (int32_t)(i + 1);  val[p++] = -h; }
                if (iy < n - 1) { ci[p] = (int32_t)(i + n);  val[p++] = -h; }
                if (iz < n - 1) { ci[p] = (int32_t)(i + n2); val[p++] = -h; }
                d[i] = h * (double)(6 - deg);
            }
    rp[n2 * n] = p;
}

/* ---------------------------------------------------------------- random geometric graph */
typedef struct {
    int64_t n, nnz;
    int64_t *rp;
    int32_t *ci;
} gen_rgg_t;

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

static int64_t uf_find(int64_t *par, int64_t x) {
    while (par[x] != x) { par[x] = par[par[x]]; x = par[x]; }
    return x;
}

/* Builds the RGG; returns an opaque handle (NULL on allocation failure).
 * Sizes via gen_rgg_sizes, arrays via gen_rgg_fetch, release via gen_rgg_free. */
void *gen_rgg_build(int64_t N, uint64_t seed) {
    const double r = sqrt(8.0 / (M_PI * (double)N));
    const double r2 = r * r;
    int64_t nc = (int64_t)floor(1.0 / r);
    if (nc < 1) nc = 1;
    const uint64_t gseed = gen_sm64(seed ^ 0x5247470000000000ULL);
    double *px = malloc(sizeof(double) * N), *py = malloc(sizeof(double) * N);
    int64_t *cell_cnt = calloc((size_t)(nc * nc + 1), sizeof(int64_t));
    int64_t *order = malloc(sizeof(int64_t) * N);   /* new position -> point index */
    int64_t *cellof = malloc(sizeof(int64_t) * N);
    if (!px || !py || !cell_cnt || !order || !cellof) return NULL;
    for (int64_t k = 0; k < N; ++k) {
        px[k] = gen_u01(gseed ^ (uint64_t)(2 * k));
        py[k] = gen_u01(gseed ^ (uint64_t)(2 * k + 1));
        int64_t cx = (int64_t)(px[k] * (double)nc), cy = (int64_t)(py[k] * (double)nc);
        if (cx >= nc) cx = nc - 1;
        if (cy >= nc) cy = nc - 1;
        cellof[k] = cy * nc + cx;
        cell_cnt[cellof[k] + 1]++;
    }
    for (int64_t c = 0; c < nc * nc; ++c) cell_cnt[c + 1] += cell_cnt[c];
    {
        int64_t *fill = malloc(sizeof(int64_t) * (size_t)(nc * nc));
        memcpy(fill, cell_cnt, sizeof(int64_t) * (size_t)(nc * nc));
        for (int64_t k = 0; k < N; ++k) order[fill[cellof[k]]++] = k; /* stable by point index */
        free(fill);
    }
    /* adjacency in cell order (positions 0..N-1) */
    int64_t *deg = calloc((size_t)N + 1, sizeof(int64_t));
    for (int pass = 0; pass < 2; ++pass) {
        int64_t *nb_pos = NULL;
        int32_t *adj = NULL;
        if (pass == 1) {
            for (int64_t a = 0; a < N; ++a) deg[a + 1] += deg[a];
            adj = malloc(sizeof(int32_t) * (size_t)deg[N]);
            nb_pos = malloc(sizeof(int64_t) * (size_t)N);
            memcpy(nb_pos, deg, sizeof(int64_t) * (size_t)N);
        }
        for (int64_t a = 0; a < N; ++a) {
            int64_t k = order[a];
            int64_t c = cellof[k], cx = c % nc, cy = c / nc;
            for (int64_t dy = -1; dy <= 1; ++dy)
                for (int64_t dx = -1; dx <= 1; ++dx) {
                    int64_t ux = cx + dx, uy = cy + dy;
                    if (ux < 0 || uy < 0 || ux >= nc || uy >= nc) continue;
                    int64_t cc = uy * nc + ux;
                    for (int64_t b = cell_cnt[cc]; b < cell_cnt[cc + 1]; ++b) {
                        if (b == a) continue;
                        int64_t q = order[b];
                        double ddx = px[k] - px[q], ddy = py[k] - py[q];
                        if (ddx * ddx + ddy * ddy < r2) {
                            if (pass == 0) deg[a + 1]++;
                            else adj[nb_pos[a]++] = (int32_t)b;
                        }
                    }
                }
        }
        if (pass == 1) {
            free(nb_pos);
            /* largest connected component via union-find */
            int64_t *par = malloc(sizeof(int64_t) * (size_t)N);
            for (int64_t a = 0; a < N; ++a) par[a] = a;
            for (int64_t a = 0; a < N; ++a)
                for (int64_t e = deg[a]; e < deg[a + 1]; ++e) {
                    int64_t x = uf_find(par, a), y = uf_find(par, adj[e]);
                    if (x != y) { if (x < y) par[y] = x; else par[x] = y; }
                }
            int64_t *csize = calloc((size_t)N, sizeof(int64_t));
            int64_t best = 0;
            for (int64_t a = 0; a < N; ++a) csize[uf_find(par, a)]++;
            for (int64_t a = 0; a < N; ++a) if (csize[a] > csize[best]) best = a;
            int64_t *newid = malloc(sizeof(int64_t) * (size_t)N);
            int64_t n = 0;
            for (int64_t a = 0; a < N; ++a) newid[a] = (uf_find(par, a) == best) ? n++ : -1;
            gen_rgg_t *g = malloc(sizeof(gen_rgg_t));
            g->n = n;
            g->rp = malloc(sizeof(int64_t) * (size_t)(n + 1));
            int64_t nnz = 0;
            for (int64_t a = 0; a < N; ++a) if (newid[a] >= 0) nnz += deg[a + 1] - deg[a] + 1;
            g->nnz = nnz;
            g->ci = malloc(sizeof(int32_t) * (size_t)nnz);
            int64_t p = 0;
            for (int64_t a = 0; a < N; ++a) {
                if (newid[a] < 0) continue;
                int64_t i = newid[a];
                g->rp[i] = p;
                int64_t p0 = p;
                g->ci[p++] = (int32_t)i;
                for (int64_t e = deg[a]; e < deg[a + 1]; ++e) g->ci[p++] = (int32_t)newid[adj[e]];
                qsort(g->ci + p0, (size_t)(p - p0), sizeof(int32_t), cmp_i32);
            }
            g->rp[n] = p;
            free(newid); free(csize); free(par); free(adj); free(deg);
            free(px); free(py); free(cell_cnt); free(order); free(cellof);
            return g;
        }
    }
    return NULL;
}

void gen_rgg_sizes(void *h, int64_t *n, int64_t *nnz) {
    gen_rgg_t *g = (gen_rgg_t *)h;
    *n = g->n;
    *nnz = g->nnz;
}

/* Unit-weight pure graph Laplacian: off-diagonal -1, diagonal = degree. */
void gen_rgg_fetch(void *h, int64_t *rp, int32_t *ci, double *val) {
    gen_rgg_t *g = (gen_rgg_t *)h;
    memcpy(rp, g->rp, sizeof(int64_t) * (size_t)(g->n + 1));
    memcpy(ci, g->ci, sizeof(int32_t) * (size_t)g->nnz);
    for (int64_t i = 0; i < g->n; ++i)
        for (int64_t p = g->rp[i]; p < g->rp[i + 1]; ++p)
            val[p] = (g->ci[p] == i) ? (double)(g->rp[i + 1] - g->rp[i] - 1) : -1.0;
}

void gen_rgg_free(void *h) {
    gen_rgg_t *g = (gen_rgg_t *)h;
    if (!g) return;
    free(g->rp); free(g->ci); free(g);
}
