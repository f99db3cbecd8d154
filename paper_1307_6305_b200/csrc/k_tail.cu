// k_tail.cu -- coarse-tail megakernel (sm_100a, one CTA of 1024 threads).
//
// The W-shaped k-cycle visits level l 2^l times per outer iteration (
// SURVEY.md 8(d) "latency floor"), so below a few thousand rows the cost is launch latency, not
// bandwidth: C4's 7-level hierarchy issues ~850 dependent launches per outer iteration without it.
// This kernel runs the whole recursion B_l -- and the inner FCG that calls it
// (O7) -- for every level l >= l_tail inside ONE CTA:
//   * rows of every pass are spread over the CTA's threads; dependent phases are separated by
//     __syncthreads() (the data stays in this SM's L1 / shared memory);
//   * FCG dots are deterministic: fixed-order warp and block reductions;
//   * in shared-memory mode (amg_options.tail_smem) the tail levels' matrices and vectors are
//     placed in the CTA's shared memory by access frequency (driver.cu upload_tail_levels).
// The arithmetic is the same three-term recurrence / residual / restriction / FCG as k_solve.cu.
// (A thread-block-cluster variant with DSMEM reductions was measured slower -- ~4 us per phase of
// cluster barriers -- and removed.)
#include <cuda_runtime.h>

#include <cstdlib>

#include "amg_internal.h"

namespace amg {

constexpr int kTailBlock = 1024;

struct TCtx {
    int t;  // thread id
    int T;  // thread count
};

__device__ __forceinline__ void csync() { __syncthreads(); }

__device__ __forceinline__ double t_warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// CTA-wide sums of k values (k <= kMaxWin); every thread returns the same totals.
// Deterministic: fixed warp and block order.
__device__ void cta_sums(double* v, int k) {
    __shared__ double wred[kMaxWin][32];
    __shared__ double part[kMaxWin];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = 0; j < k; ++j) {
        double x = t_warp_sum(v[j]);
        if (lane == 0) wred[j][wid] = x;
    }
    __syncthreads();
    if (wid == 0) {
        for (int j = 0; j < k; ++j) {
            double x = lane < nw ? wred[j][lane] : 0.0;
            x = t_warp_sum(x);
            if (lane == 0) part[j] = x;
        }
    }
    __syncthreads();
    for (int j = 0; j < k; ++j) v[j] = part[j];
    __syncthreads();
}

// one three-term recurrence step on level L:
// out_i = a*cg*xg_i + (1-a)*prev_i + b*(f_i - cg*(A xg)_i), prev_i = xprev ? xprev_i : cp*f_i
__device__ void t_step(const TLevel& L, const double* xg, double cgs, const double* f, const double* xprev, double cp,
                       double a, double b, double* out, TCtx c) {
    for (int i = c.t; i < L.n; i += c.T) {
        double s = 0.0;
        for (int p = L.rp[i]; p < L.rp[i + 1]; ++p) s = fma(L.v[p], xg[L.ci[p]], s);
        const double fi = f[i];
        const double prev = xprev ? xprev[i] : cp * fi;
        out[i] = a * (cgs * xg[i]) + (1.0 - a) * prev + b * (fi - cgs * s);
    }
    csync();
}

// dense coarsest apply, one warp per row (lanes stride the columns, a fixed-order warp sum): a
// thread per row left 32x fewer loads in flight on the coarsest levels' few rows
__device__ void t_gemv(int n, const double* M, const double* r, double* e, TCtx c) {
    const int lane = c.t & 31, w = c.t >> 5, nw = c.T >> 5;
    for (int i = w; i < n; i += nw) {
        double s = 0.0;
        for (int j = lane; j < n; j += 32) s = fma(M[(size_t)i * n + j], r[j], s);
        s = t_warp_sum(s);
        if (lane == 0) e[i] = s;
    }
    csync();
}

__device__ __noinline__ void t_fcg(const TailArgs& A, int l, TCtx c);

// z = B_l(r) -- same schedule as driver.cu apply_B
__device__ __noinline__ void t_B(const TailArgs& A, int l, const double* r, double* out, TCtx c) {
    if (l == A.L - 1) {
        t_gemv(A.lev[l - A.lbase].n, A.Minv, r, out, c);
        return;
    }
    if (l == A.dense_l && A.Bd) {  // the linear B_{L-2} as its dense matrix (k_dense.cu)
        t_gemv(A.lev[l - A.lbase].n, A.Bd, r, out, c);
        return;
    }
    const TLevel& L = A.lev[l - A.lbase];
    const int m = A.m;
    double* cur = L.X;
    double* prev = L.XA;
    t_step(L, r, L.beta[0], r, nullptr, 0.0, L.alpha[1], L.beta[1], L.X, c);  // k = 1 (x_0 = 0)
    if (m >= 2) {
        t_step(L, L.X, 1.0, r, nullptr, L.beta[0], L.alpha[2], L.beta[2], L.XA, c);  // k = 2
        cur = L.XA;
        prev = L.X;
        for (int k = 3; k <= m; ++k) {
            t_step(L, cur, 1.0, r, prev, 0.0, L.alpha[k], L.beta[k], prev, c);
            double* t = cur;
            cur = prev;
            prev = t;
        }
    }
    // residual
    for (int i = c.t; i < L.n; i += c.T) {
        double s = 0.0;
        for (int p = L.rp[i]; p < L.rp[i + 1]; ++p) s = fma(L.v[p], cur[L.ci[p]], s);
        L.RES[i] = r[i] - s;
    }
    csync();
    // restriction
    const TLevel& C = A.lev[l + 1 - A.lbase];
    for (int I = c.t; I < L.nc; I += c.T) {
        double s = 0.0;
        for (int t = L.aptr[I]; t < L.aptr[I + 1]; ++t) s += L.RES[L.perm[t]];
        C.RHO[I] = s;
    }
    csync();
    if (l + 1 == A.L - 1)
        t_gemv(C.n, A.Minv, C.RHO, C.E, c);
    else
        t_fcg(A, l + 1, c);
    // prolongation + axpy
    for (int i = c.t; i < L.n; i += c.T) cur[i] += C.E[L.agg[i]];
    csync();
    // post-smoothing S(r, x), x_{-1} = x_0
    double* other = (cur == L.X) ? L.XA : L.X;
    t_step(L, cur, 1.0, r, cur, 0.0, 1.0, L.beta[0], other, c);  // k = 0
    prev = cur;
    cur = other;
    for (int k = 1; k <= m; ++k) {
        double* target = (k == m) ? out : prev;
        t_step(L, cur, 1.0, r, prev, 0.0, L.alpha[k], L.beta[k], target, c);
        prev = cur;
        cur = target;
    }
}

// FCG_inner(l): RHO_l -> E_l with nu iterations
__device__ __noinline__ void t_fcg(const TailArgs& A, int l, TCtx c) {
    const TLevel& L = A.lev[l - A.lbase];
    const int n = L.n, nu = A.nu;
    double dq[kTailMaxNu];
    for (int i = 0; i < nu; ++i) {
        double* Di = L.D + (size_t)i * L.ld;
        double* Qi = L.Q + (size_t)i * L.ld;
        if (i == 0) {
            t_B(A, l, L.RHO, Di, c);
        } else {
            t_B(A, l, L.RHO, L.Z, c);
            double cj[kTailMaxNu];
            for (int j = 0; j < i; ++j) cj[j] = 0.0;
            for (int r = c.t; r < n; r += c.T) {
                const double z = L.Z[r];
                for (int j = 0; j < i; ++j) cj[j] += z * L.Q[(size_t)j * L.ld + r];
            }
            cta_sums(cj, i);
            for (int r = c.t; r < n; r += c.T) {
                double v = L.Z[r];
                for (int j = 0; j < i; ++j) v -= (dq[j] != 0.0 ? cj[j] / dq[j] : 0.0) * L.D[(size_t)j * L.ld + r];
                Di[r] = v;
            }
            csync();
        }
        double acc[2] = {0.0, 0.0};
        for (int r = c.t; r < n; r += c.T) {
            double s = 0.0;
            for (int p = L.rp[r]; p < L.rp[r + 1]; ++p) s = fma(L.v[p], Di[L.ci[p]], s);
            Qi[r] = s;
            acc[0] += Di[r] * s;
            acc[1] += Di[r] * L.RHO[r];
        }
        cta_sums(acc, 2);
        dq[i] = acc[0];
        const double alpha = acc[0] != 0.0 ? acc[1] / acc[0] : 0.0;  // rho = 0 => d = 0 (A13)
        for (int r = c.t; r < n; r += c.T) {
            if (i == 0) L.E[r] = alpha * Di[r]; else L.E[r] += alpha * Di[r];
            if (i < nu - 1) L.RHO[r] -= alpha * Qi[r];
        }
        csync();
    }
}

__global__ void __launch_bounds__(kTailBlock, 1) k_tail(TailArgs a) {
    extern __shared__ __align__(16) double tsv[];
    __shared__ TLevel slev[kTailMaxLev];
    const TCtx c{(int)threadIdx.x, (int)blockDim.x};
    if (a.smem) {
        // shared-memory mode: every vector of the tail levels lives in this CTA's shared memory
        // for the whole call (the matrices are read-only and stay in L1/L2); only the call's
        // input (rin, or RHO_l0) and output (out, or E_l0) are global
        const int nl = a.L - a.l0;
        for (int k = threadIdx.x; k < nl; k += blockDim.x) {
            TLevel t = a.lev[a.l0 - a.lbase + k];
            double** ptr[8] = {&t.X, &t.XA, &t.RES, &t.RHO, &t.E, &t.Z, &t.D, &t.Q};
            for (int j = 0; j < 8; ++j)
                if (t.off[j] >= 0) *ptr[j] = tsv + t.off[j];
            // tail_smem = 2: read-only level data placed in shared memory too (copied below)
            const int** iptr[5] = {&t.rp, &t.ci, &t.agg, &t.perm, &t.aptr};
            const int imap[5] = {0, 1, 3, 4, 5};
            for (int j = 0; j < 5; ++j)
                if (t.moff[imap[j]] >= 0) *iptr[j] = reinterpret_cast<const int*>(tsv + t.moff[imap[j]]);
            if (t.moff[2] >= 0) t.v = tsv + t.moff[2];
            slev[k] = t;
        }
        __syncthreads();
        for (int k = 0; k < nl; ++k) {
            const TLevel& g = a.lev[a.l0 - a.lbase + k];
            const TLevel& sl = slev[k];
            if (sl.moff[0] >= 0 || sl.moff[1] >= 0 || sl.moff[2] >= 0) {
                const int nnz = g.rp[g.n];
                auto cp_i = [&](const int* src, const int* dst, int len) {
                    int* d = const_cast<int*>(dst);
                    for (int i = threadIdx.x; i < len; i += blockDim.x) d[i] = src[i];
                };
                if (sl.moff[0] >= 0) cp_i(g.rp, sl.rp, g.n + 1);
                if (sl.moff[1] >= 0) cp_i(g.ci, sl.ci, nnz);
                if (sl.moff[2] >= 0) {
                    double* d = const_cast<double*>(sl.v);
                    for (int i = threadIdx.x; i < nnz; i += blockDim.x) d[i] = g.v[i];
                }
            }
            if (sl.moff[3] >= 0)
                for (int i = threadIdx.x; i < g.n; i += blockDim.x) const_cast<int*>(sl.agg)[i] = g.agg[i];
            if (sl.moff[4] >= 0)
                for (int i = threadIdx.x; i < g.n; i += blockDim.x) const_cast<int*>(sl.perm)[i] = g.perm[i];
            if (sl.moff[5] >= 0)
                for (int i = threadIdx.x; i <= g.nc; i += blockDim.x) const_cast<int*>(sl.aptr)[i] = g.aptr[i];
        }
        const TLevel& g0 = a.lev[a.l0 - a.lbase];
        if (a.mode == 1 && slev[0].RHO != g0.RHO)
            for (int i = threadIdx.x; i < g0.n; i += blockDim.x) slev[0].RHO[i] = g0.RHO[i];
        a.lev = slev;
        a.lbase = a.l0;
        __syncthreads();
        if (a.mode == 0) {
            t_B(a, a.l0, a.rin, a.out, c);
        } else {
            t_fcg(a, a.l0, c);
            if (slev[0].E != g0.E)
                for (int i = threadIdx.x; i < g0.n; i += blockDim.x) g0.E[i] = slev[0].E[i];
        }
        return;
    }
    if (a.mode == 0)
        t_B(a, a.l0, a.rin, a.out, c);
    else
        t_fcg(a, a.l0, c);
}

void launch_tail(const TailArgs& a, cudaStream_t s) {
    static int cfg_bytes = 0;
    const int bytes = a.smem * (int)sizeof(double);
    if (bytes > cfg_bytes) {
        CK(cudaFuncSetAttribute(k_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        cfg_bytes = bytes;
    }
    launch_k(k_tail, dim3(1), dim3(kTailBlock), (size_t)bytes, s, a);
    CK(cudaGetLastError());
    ++g_launches;
}

}  // namespace amg
