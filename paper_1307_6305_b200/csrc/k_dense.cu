// k_dense.cu -- the k-cycle operator of the level above the coarsest as a dense matrix (sm_100a).
//
// At level l = L-2 the coarse correction is the exact coarsest solve (reading A12: no inner FCG), so
// B_l (the two-level step of l.136) is a LINEAR operator:
//   B_l r = S_l(r, x),  x = S_l(r, 0) + P A_{L-1}^{-1/dagger} P^T (r - A_l S_l(r, 0)).
// On the small L2-resident levels where it is formed (n_l <= amg_options.dense_b_rows) one B_l
// application as 2m+3 dependent sparse launches costs ~35 us of launch and L2-round-trip latency;
// the same map as one dense GEMV from L2 costs ~3 us.  Each B_l is formed once at setup by running
// exactly those steps on all n_l unit vectors at once (column-batched: column j of every n x n
// work matrix is the vector of input e_j), then transposed so row i of Bd is (B_l)_{i,:}.  The
// arithmetic per column is the sparse path's (same recurrence, residual, member-order restriction,
// coarsest GEMV, prolongation), so Bd e_j equals B_l e_j up to rounding; the solve applies Bd r with
// a CTA-per-row GEMV (k_solve.cu k_gemv_rows), whose summation order differs from the sparse path's
// (within the 1e-10 preconditioner tolerance; tests/test_gpu_parity.py compares every level).
#include <cuda_runtime.h>

#include "amg_internal.h"

namespace amg {

// out[j][i] = a X[j][i] + (1 - a) Xp[j][i] + b (delta_ij - (A X[j])_i)  (Xp null: 0; X null: X = 0)
// resid (a = 0, b = 1, Xp null): out = delta - A X.  Column stride n.
__global__ void k_bat_step(int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                           const double* __restrict__ X, const double* __restrict__ Xp, double a, double b,
                           double* __restrict__ out) {
    const int64_t total = (int64_t)n * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(t / n), i = (int)(t - (int64_t)j * n);
        const double* xj = X ? X + (size_t)j * n : nullptr;
        double s = 0.0;
        if (xj)
            for (int p = rp[i]; p < rp[i + 1]; ++p) s = fma(v[p], xj[ci[p]], s);
        const double fi = (i == j) ? 1.0 : 0.0;
        const double xi = xj ? xj[i] : 0.0;
        const double pi = Xp ? Xp[(size_t)j * n + i] : 0.0;
        out[(size_t)j * n + i] = a * xi + (1.0 - a) * pi + b * (fi - s);
    }
}

// RHO[j][I] = sum_{t in I} RES[j][perm[t]] (members in increasing order, as k_restrict)
__global__ void k_bat_restrict(int n, int nc, const int* __restrict__ aptr, const int* __restrict__ perm,
                               const double* __restrict__ R, double* __restrict__ RHO) {
    const int64_t total = (int64_t)n * nc;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(t / nc), I = (int)(t - (int64_t)j * nc);
        const double* rj = R + (size_t)j * n;
        double s = 0.0;
        for (int q = aptr[I]; q < aptr[I + 1]; ++q) s += rj[perm[q]];
        RHO[(size_t)j * nc + I] = s;
    }
}

// X[j][i] += sum_K M[agg_i][K] RHO[j][K]  (coarsest (pseudo-)inverse applied, then prolongated)
__global__ void k_bat_coarse_prolong(int n, int nc, const int* __restrict__ agg, const double* __restrict__ M,
                                     const double* __restrict__ RHO, double* __restrict__ X) {
    const int64_t total = (int64_t)n * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(t / n), i = (int)(t - (int64_t)j * n);
        const int I = agg[i];
        const double* rj = RHO + (size_t)j * nc;
        double s = 0.0;
        for (int K = 0; K < nc; ++K) s = fma(M[(size_t)I * nc + K], rj[K], s);
        X[(size_t)j * n + i] += s;
    }
}

// Bd[i][j] = X[j][i]  (32 x 32 tiles through shared memory)
__global__ void k_transpose(int n, const double* __restrict__ X, double* __restrict__ Bd) {
    __shared__ double tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int j = by + k, i = bx + threadIdx.x;
        if (j < n && i < n) tile[k][threadIdx.x] = X[(size_t)j * n + i];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int i = bx + k, j = by + threadIdx.x;
        if (j < n && i < n) Bd[(size_t)i * n + j] = tile[threadIdx.x][k];
    }
}

static int bgrid(int64_t total) {
    int64_t g = (total + kBlock - 1) / kBlock;
    if (g > 148 * 16) g = 148 * 16;
    return g < 1 ? 1 : (int)g;
}

void dense_level_operator(const Csr& A, int m, const double* alpha, const double* beta, int nc, const int* agg,
                          const int* perm, const int* aptr, const double* Minv, double* Bd, cudaStream_t s) {
    const int n = A.n;
    const size_t nn = (size_t)n * n;
    double* X0 = dalloc<double>(nn, s);
    double* X1 = dalloc<double>(nn, s);
    double* X2 = dalloc<double>(nn, s);
    double* RHO = dalloc<double>((size_t)n * nc, s);
    const int g = bgrid((int64_t)nn);
    auto step = [&](const double* X, const double* Xp, double a, double b, double* out) {
        k_bat_step<<<g, kBlock, 0, s>>>(n, A.rp, A.ci, A.v, X, Xp, a, b, out);
        ++g_launches;
    };
    // pre-smoothing S(F, 0), F = I: x_1 = beta_0 F, then k = 1..m (x_0 = 0); a step may write over
    // x_{k-1} (each element is read and written by the same thread), never over x_k
    step(nullptr, nullptr, 0.0, beta[0], X1);  // x_1 = b0 (F - A 0)
    double *cur = X1, *prev = nullptr;
    for (int k = 1; k <= m; ++k) {
        double* out = prev ? prev : X0;
        step(cur, prev, alpha[k], beta[k], out);
        prev = cur;
        cur = out;
    }
    // residual F - A x (into the third buffer), restriction, coarsest solve + prolongation into x
    double* res = (cur != X2 && prev != X2) ? X2 : ((cur != X1 && prev != X1) ? X1 : X0);
    step(cur, nullptr, 0.0, 1.0, res);
    k_bat_restrict<<<bgrid((int64_t)n * nc), kBlock, 0, s>>>(n, nc, aptr, perm, res, RHO);
    k_bat_coarse_prolong<<<g, kBlock, 0, s>>>(n, nc, agg, Minv, RHO, cur);
    g_launches += 2;
    // post-smoothing S(F, x): x_{-1} = x_0 = cur; k = 0 (alpha_0 = 1) into a fresh buffer, then in place
    double* xk = cur;
    double* xprev = cur;
    for (int k = 0; k <= m; ++k) {
        double* out = (k == 0) ? res : xprev;
        step(xk, xprev, k == 0 ? 1.0 : alpha[k], beta[k], out);
        xprev = xk;
        xk = out;
    }
    dim3 tb(32, 8), tg((n + 31) / 32, (n + 31) / 32);
    k_transpose<<<tg, tb, 0, s>>>(n, xk, Bd);
    ++g_launches;
    CK(cudaGetLastError());
    dfree(X0, s);
    dfree(X1, s);
    dfree(X2, s);
    dfree(RHO, s);
}

}  // namespace amg
