// tools/vec_micro.cu -- microbenchmark of the level-0 FCG vector and transfer kernel designs on the
// C3 sizes (n = 4096^2 fp64 vectors; aggregates = 4x4 blocks of the grid, 16 members, perm-ordered
// the way the library stores them), to choose the library's kernels.  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/vec_micro tools/vec_micro.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CKM(x)                                                                                   \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) {                                                                 \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);      \
            exit(1);                                                                             \
        }                                                                                        \
    } while (0)

static int g_sms = 148;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ double block_sum(double v) {
    __shared__ double red[32];
    __shared__ double tot;
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double t = lane < nw ? red[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) tot = t;
    }
    __syncthreads();
    return tot;
}

// ---------------------------------------------------------------- references
__global__ void k_copy2(long n2, const double2* __restrict__ a, double2* __restrict__ b) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void k_read4(long n2, const double2* __restrict__ a, const double2* __restrict__ b,
                        const double2* __restrict__ c, const double2* __restrict__ d, double* out) {
    double s = 0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
        double2 x = a[i], y = b[i], z = c[i], w = d[i];
        s += x.x + x.y + y.x + y.y + z.x + z.y + w.x + w.y;
    }
    if (s == 12345.0) out[0] = s;
}

// ---------------------------------------------------------------- fcg_update: x += a d; r -= a q; rr += r^2
__global__ void upd_v0(int n, double a, const double* __restrict__ d, const double* __restrict__ q, double* __restrict__ x,
                       double* __restrict__ r, double* part) {
    double acc = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        x[i] += a * d[i];
        double ri = r[i] - a * q[i];
        r[i] = ri;
        acc += ri * ri;
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}
template <int U>
__global__ void upd_v2(int n, double a, const double* __restrict__ d, const double* __restrict__ q, double* __restrict__ x,
                       double* __restrict__ r, double* part) {
    const long n2 = n >> 1, st = (long)gridDim.x * blockDim.x;
    const double2* D = (const double2*)d;
    const double2* Q = (const double2*)q;
    double2* X = (double2*)x;
    double2* R = (double2*)r;
    double acc = 0;
    long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    for (; i + (U - 1) * st < n2; i += U * st) {
        double2 dd[U], qq[U], xx[U], rr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) { dd[u] = D[i + u * st]; qq[u] = Q[i + u * st]; xx[u] = X[i + u * st]; rr[u] = R[i + u * st]; }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            xx[u].x += a * dd[u].x; xx[u].y += a * dd[u].y;
            rr[u].x -= a * qq[u].x; rr[u].y -= a * qq[u].y;
            X[i + u * st] = xx[u];
            R[i + u * st] = rr[u];
            acc += rr[u].x * rr[u].x;
            acc += rr[u].y * rr[u].y;
        }
    }
    for (; i < n2; i += st) {
        double2 dd = D[i], qq = Q[i], xx = X[i], rr = R[i];
        xx.x += a * dd.x; xx.y += a * dd.y; rr.x -= a * qq.x; rr.y -= a * qq.y;
        X[i] = xx; R[i] = rr; acc += rr.x * rr.x; acc += rr.y * rr.y;
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// ---------------------------------------------------------------- multidot c_j = z.Q_j, j < W
struct P4 { const double* p[4]; };
template <int W>
__global__ void md_v0(int n, const double* __restrict__ z, P4 Q, double* part) {
    double acc[W] = {};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double zi = z[i];
#pragma unroll
        for (int j = 0; j < W; ++j) acc[j] += zi * Q.p[j][i];
    }
#pragma unroll
    for (int j = 0; j < W; ++j) {
        double b = block_sum(acc[j]);
        if (threadIdx.x == 0) part[j * gridDim.x + blockIdx.x] = b;
    }
}
template <int W, int U>
__global__ void md_v2(int n, const double* __restrict__ z, P4 Q, double* part) {
    const long n2 = n >> 1, st = (long)gridDim.x * blockDim.x;
    double acc[W] = {};
    long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    for (; i + (U - 1) * st < n2; i += U * st) {
        double2 zz[U], qq[U][W];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            zz[u] = ((const double2*)z)[i + u * st];
#pragma unroll
            for (int j = 0; j < W; ++j) qq[u][j] = ((const double2*)Q.p[j])[i + u * st];
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < W; ++j) { acc[j] += zz[u].x * qq[u][j].x; acc[j] += zz[u].y * qq[u][j].y; }
    }
    for (; i < n2; i += st) {
        double2 zz = ((const double2*)z)[i];
#pragma unroll
        for (int j = 0; j < W; ++j) { double2 q = ((const double2*)Q.p[j])[i]; acc[j] += zz.x * q.x; acc[j] += zz.y * q.y; }
    }
#pragma unroll
    for (int j = 0; j < W; ++j) {
        double b = block_sum(acc[j]);
        if (threadIdx.x == 0) part[j * gridDim.x + blockIdx.x] = b;
    }
}

// ---------------------------------------------------------------- direction d = z - sum beta_j D_j
template <int W>
__global__ void dir_v0(int n, const double* __restrict__ z, P4 D, double* __restrict__ d) {
    const double beta[4] = {0.1, 0.2, 0.3, 0.4};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double v = z[i];
#pragma unroll
        for (int j = 0; j < W; ++j) v -= beta[j] * D.p[j][i];
        d[i] = v;
    }
}
template <int W, int U>
__global__ void dir_v2(int n, const double* __restrict__ z, P4 D, double* __restrict__ d) {
    const double beta[4] = {0.1, 0.2, 0.3, 0.4};
    const long n2 = n >> 1, st = (long)gridDim.x * blockDim.x;
    long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    for (; i + (U - 1) * st < n2; i += U * st) {
        double2 zz[U], dd[U][W];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            zz[u] = ((const double2*)z)[i + u * st];
#pragma unroll
            for (int j = 0; j < W; ++j) dd[u][j] = ((const double2*)D.p[j])[i + u * st];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double2 v = zz[u];
#pragma unroll
            for (int j = 0; j < W; ++j) { v.x -= beta[j] * dd[u][j].x; v.y -= beta[j] * dd[u][j].y; }
            ((double2*)d)[i + u * st] = v;
        }
    }
    for (; i < n2; i += st) {
        double2 v = ((const double2*)z)[i];
#pragma unroll
        for (int j = 0; j < W; ++j) { double2 q = ((const double2*)D.p[j])[i]; v.x -= beta[j] * q.x; v.y -= beta[j] * q.y; }
        ((double2*)d)[i] = v;
    }
}

// ---------------------------------------------------------------- prolongation x += eH[agg]
__global__ void pro_v0(int n, const int* __restrict__ agg, const double* __restrict__ eH, double* __restrict__ x) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] += __ldg(eH + agg[i]);
}
template <int U>
__global__ void pro_v2(int n, const int* __restrict__ agg, const double* __restrict__ eH, double* __restrict__ x) {
    const long n4 = n >> 2, st = (long)gridDim.x * blockDim.x;
    long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    for (; i + (U - 1) * st < n4; i += U * st) {
        int4 a[U];
        double2 x0[U], x1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            a[u] = ((const int4*)agg)[i + u * st];
            x0[u] = ((const double2*)x)[2 * (i + u * st)];
            x1[u] = ((const double2*)x)[2 * (i + u * st) + 1];
        }
        double e[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            e[u][0] = __ldg(eH + a[u].x); e[u][1] = __ldg(eH + a[u].y);
            e[u][2] = __ldg(eH + a[u].z); e[u][3] = __ldg(eH + a[u].w);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            x0[u].x += e[u][0]; x0[u].y += e[u][1]; x1[u].x += e[u][2]; x1[u].y += e[u][3];
            ((double2*)x)[2 * (i + u * st)] = x0[u];
            ((double2*)x)[2 * (i + u * st) + 1] = x1[u];
        }
    }
    for (; i < n4; i += st) {
        int4 a = ((const int4*)agg)[i];
        double2 x0 = ((const double2*)x)[2 * i], x1 = ((const double2*)x)[2 * i + 1];
        x0.x += __ldg(eH + a.x); x0.y += __ldg(eH + a.y); x1.x += __ldg(eH + a.z); x1.y += __ldg(eH + a.w);
        ((double2*)x)[2 * i] = x0;
        ((double2*)x)[2 * i + 1] = x1;
    }
}

// ---------------------------------------------------------------- restriction rH[I] = sum_{t in I} r[perm[t]]
__global__ void res_v0(int nc, const int* __restrict__ aptr, const int* __restrict__ perm, const double* __restrict__ r,
                       double* __restrict__ rH) {
    for (int I = blockIdx.x * blockDim.x + threadIdx.x; I < nc; I += gridDim.x * blockDim.x) {
        const int t0 = aptr[I], t1 = aptr[I + 1];
        double s = 0.0;
        for (int t = t0; t < t1; ++t) s += __ldg(r + perm[t]);
        rH[I] = s;
    }
}
// unrolled thread-per-aggregate: perm loads of 4 issued before the gathers
__global__ void res_v1(int nc, const int* __restrict__ aptr, const int* __restrict__ perm, const double* __restrict__ r,
                       double* __restrict__ rH) {
    for (int I = blockIdx.x * blockDim.x + threadIdx.x; I < nc; I += gridDim.x * blockDim.x) {
        const int t0 = aptr[I], t1 = aptr[I + 1];
        double s = 0.0;
        int t = t0;
        for (; t + 4 <= t1; t += 4) {
            int p0 = perm[t], p1 = perm[t + 1], p2 = perm[t + 2], p3 = perm[t + 3];
            double a0 = __ldg(r + p0), a1 = __ldg(r + p1), a2 = __ldg(r + p2), a3 = __ldg(r + p3);
            s += a0; s += a1; s += a2; s += a3;
        }
        for (; t < t1; ++t) s += __ldg(r + perm[t]);
        rH[I] = s;
    }
}
// CTA stages the members of AG consecutive aggregates: perm read coalesced, r gathered into shared
// memory by all threads, then one thread per aggregate sums its members in order (same order as v0)
template <int AG, int CAP>
__global__ void __launch_bounds__(256) res_v2(int nc, const int* __restrict__ aptr, const int* __restrict__ perm,
                                              const double* __restrict__ r, double* __restrict__ rH) {
    __shared__ double sv[CAP];
    __shared__ int sp[AG + 1];
    for (int I0 = blockIdx.x * AG; I0 < nc; I0 += gridDim.x * AG) {
        const int na = min(AG, nc - I0);
        for (int k = threadIdx.x; k <= na; k += blockDim.x) sp[k] = aptr[I0 + k];
        __syncthreads();
        const int t0 = sp[0], cnt = sp[na] - t0;
        if (cnt <= CAP) {
            for (int k = threadIdx.x; k < cnt; k += blockDim.x) sv[k] = __ldg(r + __ldg(perm + t0 + k));
            __syncthreads();
            for (int a = threadIdx.x; a < na; a += blockDim.x) {
                double s = 0.0;
                for (int k = sp[a] - t0; k < sp[a + 1] - t0; ++k) s += sv[k];
                rH[I0 + a] = s;
            }
        } else {
            for (int a = threadIdx.x; a < na; a += blockDim.x) {
                double s = 0.0;
                for (int t = sp[a]; t < sp[a + 1]; ++t) s += __ldg(r + perm[t]);
                rH[I0 + a] = s;
            }
        }
        __syncthreads();
    }
}

// warp window: 32 consecutive aggregates per warp; their members' perm entries are read coalesced
// and r gathered (consecutive members are grid neighbours) into a per-warp shared buffer (padded one
// slot per 32), then lane k sums aggregate k's members in member order (the v0 order, bitwise)
template <int CAP>
__global__ void __launch_bounds__(256) res_v3(int nc, const int* __restrict__ aptr, const int* __restrict__ perm,
                                              const double* __restrict__ r, double* __restrict__ rH) {
    extern __shared__ double sbuf[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* sb = sbuf + wib * (CAP + CAP / 32);
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int I0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; I0 < nc; I0 += nwarps * 32) {
        const int I = I0 + lane;
        const int a0 = I < nc ? aptr[I] : 0;
        const int a1 = I < nc ? aptr[I + 1] : 0;
        const int base = __shfl_sync(0xffffffffu, a0, 0);
        const int last = min(nc, I0 + 32) - 1 - I0;
        const int end = __shfl_sync(0xffffffffu, a1, last);
        const int M = end - base;
        if (M <= CAP) {
            int c = 0;
            for (; c + 128 <= M; c += 128) {
                int p[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) p[u] = __ldg(perm + base + c + 32 * u + lane);
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldg(r + p[u]);
#pragma unroll
                for (int u = 0; u < 4; ++u) { const int j = c + 32 * u + lane; sb[j + (j >> 5)] = v[u]; }
            }
            for (; c < M; c += 32)
                if (c + lane < M) { const int j = c + lane; sb[j + (j >> 5)] = __ldg(r + __ldg(perm + base + j)); }
            __syncwarp();
            if (I < nc) {
                double s = 0.0;
                for (int j = a0 - base; j < a1 - base; ++j) s += sb[j + (j >> 5)];
                rH[I] = s;
            }
            __syncwarp();
        } else if (I < nc) {
            double s = 0.0;
            for (int t = a0; t < a1; ++t) s += __ldg(r + perm[t]);
            rH[I] = s;
        }
    }
}

// ---------------------------------------------------------------- timing
template <class F>
static float timeit(F f, int reps = 20) {
    cudaEvent_t a, b;
    CKM(cudaEventCreate(&a));
    CKM(cudaEventCreate(&b));
    f();
    f();
    CKM(cudaDeviceSynchronize());
    CKM(cudaEventRecord(a));
    for (int i = 0; i < reps; ++i) f();
    CKM(cudaEventRecord(b));
    CKM(cudaEventSynchronize(b));
    float ms;
    CKM(cudaEventElapsedTime(&ms, a, b));
    return 1e3f * ms / reps;
}
static void report(const char* name, float us, double bytes) {
    printf("%-40s %8.1f us  %7.0f GB/s\n", name, us, bytes / (us * 1e-6) / 1e9);
}

template <class K>
static int occ_grid(K k, int block = 256, int cap = 64) {
    int b = 0;
    CKM(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, block, 0));
    if (b > cap) b = cap;
    return g_sms * b;
}

int main() {
    CKM(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
    const int N = 4096, n = N * N;
    const size_t vb = (size_t)n * 8;
    double* v[12];
    for (auto& p : v) {
        CKM(cudaMalloc(&p, vb));
        CKM(cudaMemset(p, 0, vb));
    }
    double* part;
    CKM(cudaMalloc(&part, 64 * 4096 * 8));
    // aggregates: 4x4 blocks
    const int nb = N / 4, nc = nb * nb;
    std::vector<int> agg(n), perm(n), aptr(nc + 1);
    for (int y = 0; y < N; ++y)
        for (int x = 0; x < N; ++x) agg[y * N + x] = (y / 4) * nb + x / 4;
    {
        std::vector<int> cnt(nc + 1, 0);
        for (int i = 0; i < n; ++i) cnt[agg[i] + 1]++;
        for (int I = 0; I < nc; ++I) cnt[I + 1] += cnt[I];
        aptr = cnt;
        std::vector<int> fill(cnt.begin(), cnt.end() - 1);
        for (int i = 0; i < n; ++i) perm[fill[agg[i]]++] = i;
    }
    int *dagg, *dperm, *daptr;
    CKM(cudaMalloc(&dagg, n * 4));
    CKM(cudaMalloc(&dperm, n * 4));
    CKM(cudaMalloc(&daptr, (nc + 1) * 4));
    CKM(cudaMemcpy(dagg, agg.data(), n * 4, cudaMemcpyHostToDevice));
    CKM(cudaMemcpy(dperm, perm.data(), n * 4, cudaMemcpyHostToDevice));
    CKM(cudaMemcpy(daptr, aptr.data(), (nc + 1) * 4, cudaMemcpyHostToDevice));
    double* eH = v[11];
    const long n2 = n / 2;
    printf("n = %d, %d SMs\n", n, g_sms);
    for (int cps : {4, 8, 16}) {
        int g = g_sms * cps;
        char nm[64];
        snprintf(nm, 64, "copy double2 (%d CTA/SM)", cps);
        report(nm, timeit([&] { k_copy2<<<g, 256>>>(n2, (double2*)v[0], (double2*)v[1]); }), 2.0 * vb);
        snprintf(nm, 64, "read 4 streams double2 (%d CTA/SM)", cps);
        report(nm, timeit([&] { k_read4<<<g, 256>>>(n2, (double2*)v[0], (double2*)v[1], (double2*)v[2], (double2*)v[3], part); }),
               4.0 * vb);
    }
    // fcg update: 4 reads + 2 writes
    for (int cps : {4, 8}) {
        int g = g_sms * cps;
        char nm[64];
        snprintf(nm, 64, "fcg_update v0 scalar (%d/SM)", cps);
        report(nm, timeit([&] { upd_v0<<<g, 256>>>(n, 0.5, v[0], v[1], v[2], v[3], part); }), 6.0 * vb);
        snprintf(nm, 64, "fcg_update v2 double2 U1 (%d/SM)", cps);
        report(nm, timeit([&] { upd_v2<1><<<g, 256>>>(n, 0.5, v[0], v[1], v[2], v[3], part); }), 6.0 * vb);
        snprintf(nm, 64, "fcg_update v2 double2 U2 (%d/SM)", cps);
        report(nm, timeit([&] { upd_v2<2><<<g, 256>>>(n, 0.5, v[0], v[1], v[2], v[3], part); }), 6.0 * vb);
        snprintf(nm, 64, "fcg_update v2 double2 U4 (%d/SM)", cps);
        report(nm, timeit([&] { upd_v2<4><<<g, 256>>>(n, 0.5, v[0], v[1], v[2], v[3], part); }), 6.0 * vb);
    }
    P4 q4{{v[4], v[5], v[6], v[7]}};
    for (int cps : {4, 8}) {
        int g = g_sms * cps;
        char nm[64];
        snprintf(nm, 64, "multidot w4 v0 (%d/SM)", cps);
        report(nm, timeit([&] { md_v0<4><<<g, 256>>>(n, v[0], q4, part); }), 5.0 * vb);
        snprintf(nm, 64, "multidot w4 v2 U1 (%d/SM)", cps);
        report(nm, timeit([&] { md_v2<4, 1><<<g, 256>>>(n, v[0], q4, part); }), 5.0 * vb);
        snprintf(nm, 64, "multidot w4 v2 U2 (%d/SM)", cps);
        report(nm, timeit([&] { md_v2<4, 2><<<g, 256>>>(n, v[0], q4, part); }), 5.0 * vb);
        snprintf(nm, 64, "multidot w1 v0 (%d/SM)", cps);
        report(nm, timeit([&] { md_v0<1><<<g, 256>>>(n, v[0], q4, part); }), 2.0 * vb);
        snprintf(nm, 64, "multidot w1 v2 U2 (%d/SM)", cps);
        report(nm, timeit([&] { md_v2<1, 2><<<g, 256>>>(n, v[0], q4, part); }), 2.0 * vb);
        snprintf(nm, 64, "multidot w1 v2 U4 (%d/SM)", cps);
        report(nm, timeit([&] { md_v2<1, 4><<<g, 256>>>(n, v[0], q4, part); }), 2.0 * vb);
        snprintf(nm, 64, "direction w4 v0 (%d/SM)", cps);
        report(nm, timeit([&] { dir_v0<4><<<g, 256>>>(n, v[0], q4, v[8]); }), 6.0 * vb);
        snprintf(nm, 64, "direction w4 v2 U1 (%d/SM)", cps);
        report(nm, timeit([&] { dir_v2<4, 1><<<g, 256>>>(n, v[0], q4, v[8]); }), 6.0 * vb);
        snprintf(nm, 64, "direction w4 v2 U2 (%d/SM)", cps);
        report(nm, timeit([&] { dir_v2<4, 2><<<g, 256>>>(n, v[0], q4, v[8]); }), 6.0 * vb);
        snprintf(nm, 64, "direction w1 v2 U2 (%d/SM)", cps);
        report(nm, timeit([&] { dir_v2<1, 2><<<g, 256>>>(n, v[0], q4, v[8]); }), 3.0 * vb);
        snprintf(nm, 64, "direction w1 v2 U4 (%d/SM)", cps);
        report(nm, timeit([&] { dir_v2<1, 4><<<g, 256>>>(n, v[0], q4, v[8]); }), 3.0 * vb);
    }
    const double pbytes = 20.0 * n + 8.0 * nc, rbytes = 12.0 * n + 12.0 * nc;
    for (int cps : {4, 8, 16}) {
        int g = g_sms * cps;
        char nm[64];
        snprintf(nm, 64, "prolong v0 (%d/SM)", cps);
        report(nm, timeit([&] { pro_v0<<<g, 256>>>(n, dagg, eH, v[9]); }), pbytes);
        snprintf(nm, 64, "prolong v2 U1 (%d/SM)", cps);
        report(nm, timeit([&] { pro_v2<1><<<g, 256>>>(n, dagg, eH, v[9]); }), pbytes);
        snprintf(nm, 64, "prolong v2 U2 (%d/SM)", cps);
        report(nm, timeit([&] { pro_v2<2><<<g, 256>>>(n, dagg, eH, v[9]); }), pbytes);
        int gr = (nc + 255) / 256;
        snprintf(nm, 64, "restrict v0 (%d/SM)", cps);
        report(nm, timeit([&] { res_v0<<<std::min(gr, g), 256>>>(nc, daptr, dperm, v[10], eH); }), rbytes);
        snprintf(nm, 64, "restrict v1 unroll4 (%d/SM)", cps);
        report(nm, timeit([&] { res_v1<<<std::min(gr, g), 256>>>(nc, daptr, dperm, v[10], eH); }), rbytes);
    }
    for (int g : {g_sms * 2, g_sms * 4, g_sms * 8}) {
        char nm[64];
        snprintf(nm, 64, "restrict v2 smem AG128 (%d CTAs)", g);
        report(nm, timeit([&] { res_v2<128, 4096><<<g, 256>>>(nc, daptr, dperm, v[10], eH); }), rbytes);
        snprintf(nm, 64, "restrict v2 smem AG256 (%d CTAs)", g);
        report(nm, timeit([&] { res_v2<256, 5120><<<g, 256>>>(nc, daptr, dperm, v[10], eH); }), rbytes);
    }
    for (int cps : {2, 3, 4}) {
        constexpr int CAP = 1024;
        const size_t sm = 8 * (CAP + CAP / 32) * sizeof(double);
        CKM(cudaFuncSetAttribute(res_v3<CAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        int g = g_sms * cps;
        char nm[64];
        snprintf(nm, 64, "restrict v3 warp window (%d/SM)", cps);
        report(nm, timeit([&] { res_v3<CAP><<<g, 256, sm>>>(nc, daptr, dperm, v[10], eH); }), rbytes);
    }
    {
        // check v3 == v0 bitwise
        std::vector<double> hr(n);
        for (int i = 0; i < n; ++i) hr[i] = (double)((i * 2654435761u) % 1000003) / 1000003.0 - 0.5;
        CKM(cudaMemcpy(v[10], hr.data(), vb, cudaMemcpyHostToDevice));
        res_v0<<<4096, 256>>>(nc, daptr, dperm, v[10], v[0]);
        constexpr int CAP = 1024;
        const size_t sm = 8 * (CAP + CAP / 32) * sizeof(double);
        res_v3<CAP><<<g_sms * 3, 256, sm>>>(nc, daptr, dperm, v[10], v[1]);
        std::vector<double> a(nc), b(nc);
        CKM(cudaMemcpy(a.data(), v[0], nc * 8, cudaMemcpyDeviceToHost));
        CKM(cudaMemcpy(b.data(), v[1], nc * 8, cudaMemcpyDeviceToHost));
        int bad = 0;
        for (int I = 0; I < nc; ++I) bad += a[I] != b[I];
        printf("restrict v3 vs v0: %d of %d differ\n", bad, nc);
    }
    CKM(cudaDeviceSynchronize());
    return 0;
}
