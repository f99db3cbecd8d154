// tools/spmv_micro.cu -- microbenchmark of SELL-32 three-term smoother-step kernel variants on the
// C3 level-0 operator (4096^2 5-point stencil, natural order), to choose the hot kernel design.
// Not part of the library.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o spmv_micro tools/spmv_micro.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CKM(x)                                                                         \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

__device__ __forceinline__ int ldi(const int* p) {
    int r;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ double ldd(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

struct Args {
    int n, nslices;
    const int* sptr;
    const int* col;
    const double* val;
    const double* xg;
    const double* f;
    const double* xprev;
    double* out;
    double alpha, beta;
};

// V0: as in the library (U=8, epilogue after the gathers)
template <int U>
__global__ void __launch_bounds__(256) v0(Args a) {
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < a.nslices; sl += nw) {
        const int b = __ldg(a.sptr + sl), e = __ldg(a.sptr + sl + 1);
        const int* cp = a.col + (size_t)b * 32 + lane;
        const double* vp = a.val + (size_t)b * 32 + lane;
        const int i = sl * 32 + lane, w = e - b;
        double sum = 0.0;
        for (int j0 = 0; j0 < w; j0 += U) {
            int c[U];
            double v[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j0 + u < w) { c[u] = ldi(cp + (size_t)(j0 + u) * 32); v[u] = ldd(vp + (size_t)(j0 + u) * 32); }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j0 + u < w) xv[u] = __ldg(a.xg + c[u]);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j0 + u < w) sum = fma(v[u], xv[u], sum);
        }
        if (i < a.n) {
            double fi = a.f[i];
            a.out[i] = a.alpha * __ldg(a.xg + i) + (1.0 - a.alpha) * a.xprev[i] + a.beta * (fi - sum);
        }
    }
}

// V1: epilogue operands loaded first (independent of the matrix), optional min blocks
template <int U, int MINB>
__global__ void __launch_bounds__(256, MINB) v1(Args a) {
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < a.nslices; sl += nw) {
        const int b = __ldg(a.sptr + sl), e = __ldg(a.sptr + sl + 1);
        const int* cp = a.col + (size_t)b * 32 + lane;
        const double* vp = a.val + (size_t)b * 32 + lane;
        const int i = sl * 32 + lane, w = e - b;
        const bool act = i < a.n;
        double fi = 0, xp = 0, xi = 0;
        if (act) { fi = ldd(a.f + i); xp = ldd(a.xprev + i); xi = __ldg(a.xg + i); }
        double sum = 0.0;
        for (int j0 = 0; j0 < w; j0 += U) {
            int c[U];
            double v[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j0 + u < w) { c[u] = ldi(cp + (size_t)(j0 + u) * 32); v[u] = ldd(vp + (size_t)(j0 + u) * 32); }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j0 + u < w) xv[u] = __ldg(a.xg + c[u]);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j0 + u < w) sum = fma(v[u], xv[u], sum);
        }
        if (act) a.out[i] = a.alpha * xi + (1.0 - a.alpha) * xp + a.beta * (fi - sum);
    }
}

// V1b: like V1 but plain (coherent) loads for f / xprev
template <int U>
__global__ void __launch_bounds__(256) v1b(Args a) {
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < a.nslices; sl += nw) {
        const int b = __ldg(a.sptr + sl), e = __ldg(a.sptr + sl + 1);
        const int* cp = a.col + (size_t)b * 32 + lane;
        const double* vp = a.val + (size_t)b * 32 + lane;
        const int i = sl * 32 + lane, w = e - b;
        const bool act = i < a.n;
        double fi = 0, xp = 0, xi = 0;
        if (act) { fi = a.f[i]; xp = a.xprev[i]; xi = __ldg(a.xg + i); }
        double sum = 0.0;
        for (int j0 = 0; j0 < w; j0 += U) {
            int c[U];
            double v[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j0 + u < w) { c[u] = ldi(cp + (size_t)(j0 + u) * 32); v[u] = ldd(vp + (size_t)(j0 + u) * 32); }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j0 + u < w) xv[u] = __ldg(a.xg + c[u]);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j0 + u < w) sum = fma(v[u], xv[u], sum);
        }
        if (act) a.out[i] = a.alpha * xi + (1.0 - a.alpha) * xp + a.beta * (fi - sum);
    }
}

// V2: two slices per warp iteration (slices sl and sl + nw), all independent loads first
template <int U>
__global__ void __launch_bounds__(256) v2(Args a) {
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int s0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s0 < a.nslices; s0 += 2 * nw) {
        int sl[2] = {s0, s0 + nw};
        int b[2], w[2], ii[2];
        double fi[2], xp[2], xi[2], sum[2] = {0.0, 0.0};
        int c[2][U];
        double v[2][U], xv[2][U];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            bool ok = sl[k] < a.nslices;
            b[k] = ok ? __ldg(a.sptr + sl[k]) : 0;
            w[k] = ok ? __ldg(a.sptr + sl[k] + 1) - b[k] : 0;
            ii[k] = sl[k] * 32 + lane;
            bool act = ok && ii[k] < a.n;
            fi[k] = act ? ldd(a.f + ii[k]) : 0;
            xp[k] = act ? ldd(a.xprev + ii[k]) : 0;
            xi[k] = act ? __ldg(a.xg + ii[k]) : 0;
        }
        // assumes w <= U (true for the 5-point stencil); general widths fall back to a loop
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u < w[k]) {
                    c[k][u] = ldi(a.col + ((size_t)b[k] + u) * 32 + lane);
                    v[k][u] = ldd(a.val + ((size_t)b[k] + u) * 32 + lane);
                }
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u < w[k]) xv[k][u] = __ldg(a.xg + c[k][u]);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u < w[k]) sum[k] = fma(v[k][u], xv[k][u], sum[k]);
            if (sl[k] < a.nslices && ii[k] < a.n)
                a.out[ii[k]] = a.alpha * xi[k] + (1.0 - a.alpha) * xp[k] + a.beta * (fi[k] - sum[k]);
        }
    }
}

// V3: block-contiguous slice ranges (each block owns a contiguous chunk of slices), V1 body
template <int U>
__global__ void __launch_bounds__(256) v3(Args a, int per_block) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int s_begin = blockIdx.x * per_block;
    const int s_end = min(a.nslices, s_begin + per_block);
    for (int sl = s_begin + wid; sl < s_end; sl += 8) {
        const int b = __ldg(a.sptr + sl), e = __ldg(a.sptr + sl + 1);
        const int* cp = a.col + (size_t)b * 32 + lane;
        const double* vp = a.val + (size_t)b * 32 + lane;
        const int i = sl * 32 + lane, w = e - b;
        const bool act = i < a.n;
        double fi = 0, xp = 0, xi = 0;
        if (act) { fi = ldd(a.f + i); xp = ldd(a.xprev + i); xi = __ldg(a.xg + i); }
        double sum = 0.0;
        for (int j0 = 0; j0 < w; j0 += U) {
            int c[U];
            double v[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j0 + u < w) { c[u] = ldi(cp + (size_t)(j0 + u) * 32); v[u] = ldd(vp + (size_t)(j0 + u) * 32); }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j0 + u < w) xv[u] = __ldg(a.xg + c[u]);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j0 + u < w) sum = fma(v[u], xv[u], sum);
        }
        if (act) a.out[i] = a.alpha * xi + (1.0 - a.alpha) * xp + a.beta * (fi - sum);
    }
}

// ---- compressed variants: uint8 value codes + uint8 offset codes (dictionaries in shared memory)
__device__ __forceinline__ int ldu8(const unsigned char* p) {
    int r;
    asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ double ldg_nc(const double* p) {
    double r;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}
struct CArgs {
    int n, nslices;
    const int* sptr;
    const unsigned char* vc;
    const unsigned char* cc;
    const double* vdict;
    const int* cdict;
    const double* xg;
    const double* f;
    const double* xprev;
    double* out;
    double alpha, beta;
};

// NS slices per warp iteration (slices sl, sl + nw, ...), fixed width W = 5 fast path
template <int NS, int MINB>
__global__ void __launch_bounds__(256, MINB) vc_k(CArgs a) {
    __shared__ double sv[256];
    __shared__ int sc[256];
    for (int k = threadIdx.x; k < 256; k += blockDim.x) { sv[k] = a.vdict[k]; sc[k] = a.cdict[k]; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    constexpr int W = 5;
    for (int s0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s0 < a.nslices; s0 += NS * nw) {
        int i[NS];
        double fi[NS], xp[NS], xi[NS];
        int cr[NS][W], vr[NS][W];
        bool ok[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            int sl = s0 + k * nw;
            ok[k] = sl < a.nslices;
            i[k] = sl * 32 + lane;
            bool act = ok[k] && i[k] < a.n;
            fi[k] = act ? ldd(a.f + i[k]) : 0;
            xp[k] = act ? ldd(a.xprev + i[k]) : 0;
            xi[k] = act ? ldg_nc(a.xg + i[k]) : 0;
        }
#pragma unroll
        for (int k = 0; k < NS; ++k)
#pragma unroll
            for (int u = 0; u < W; ++u) {
                size_t e = ((size_t)(s0 + k * nw) * W + u) * 32 + lane;
                vr[k][u] = ok[k] ? ldu8(a.vc + e) : 0;
                cr[k][u] = ok[k] ? ldu8(a.cc + e) : 2;
            }
        int all = 0;
        int col[NS][W];
#pragma unroll
        for (int k = 0; k < NS; ++k)
#pragma unroll
            for (int u = 0; u < W; ++u) {
                int c = i[k] + sc[cr[k][u]];
                c = c < a.n ? c : a.n - 1;
                c = c < 0 ? 0 : c;
                col[k][u] = c;
                all |= c | vr[k][u];
            }
        const int z = all < 0 ? 1 : 0;
        double x[NS][W];
#pragma unroll
        for (int k = 0; k < NS; ++k)
#pragma unroll
            for (int u = 0; u < W; ++u) x[k][u] = ldg_nc(a.xg + (col[k][u] | z));
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            double s = 0.0;
#pragma unroll
            for (int u = 0; u < W; ++u) s = fma(sv[vr[k][u]], x[k][u], s);
            if (ok[k] && i[k] < a.n) a.out[i[k]] = a.alpha * xi[k] + (1.0 - a.alpha) * xp[k] + a.beta * (fi[k] - s);
        }
    }
}

// uncompressed with the same NS structure
template <int NS, int MINB>
__global__ void __launch_bounds__(256, MINB) vu_k(Args a) {
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    constexpr int W = 5;
    for (int s0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s0 < a.nslices; s0 += NS * nw) {
        int i[NS];
        double fi[NS], xp[NS], xi[NS];
        int c[NS][W];
        double v[NS][W];
        bool ok[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            int sl = s0 + k * nw;
            ok[k] = sl < a.nslices;
            i[k] = sl * 32 + lane;
            bool act = ok[k] && i[k] < a.n;
            fi[k] = act ? ldd(a.f + i[k]) : 0;
            xp[k] = act ? ldd(a.xprev + i[k]) : 0;
            xi[k] = act ? ldg_nc(a.xg + i[k]) : 0;
        }
#pragma unroll
        for (int k = 0; k < NS; ++k)
#pragma unroll
            for (int u = 0; u < W; ++u) {
                size_t e = ((size_t)(s0 + k * nw) * W + u) * 32 + lane;
                v[k][u] = ok[k] ? ldd(a.val + e) : 0;
                c[k][u] = ok[k] ? ldi(a.col + e) : 0;
            }
        int all = 0;
#pragma unroll
        for (int k = 0; k < NS; ++k)
#pragma unroll
            for (int u = 0; u < W; ++u) all |= c[k][u];
        const int z = all < 0 ? 1 : 0;
        double x[NS][W];
#pragma unroll
        for (int k = 0; k < NS; ++k)
#pragma unroll
            for (int u = 0; u < W; ++u) x[k][u] = ldg_nc(a.xg + (c[k][u] | z));
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            double s = 0.0;
#pragma unroll
            for (int u = 0; u < W; ++u) s = fma(v[k][u], x[k][u], s);
            if (ok[k] && i[k] < a.n) a.out[i[k]] = a.alpha * xi[k] + (1.0 - a.alpha) * xp[k] + a.beta * (fi[k] - s);
        }
    }
}

__global__ void build5c(int N, unsigned char* vc, unsigned char* cc) {
    // codes: values {-1 -> 0, 4 -> 1, 0 -> 2}; offsets {-N -> 0, -1 -> 1, 0 -> 2, 1 -> 3, N -> 4}
    const int n = N * N, nsl = (n + 31) / 32;
    for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < (long)nsl * 32; t += (long)gridDim.x * blockDim.x) {
        int sl = (int)(t >> 5), lane = (int)(t & 31), i = sl * 32 + lane;
        int iy = i / N, ix = i % N;
        int cs[5], vs[5], m = 0;
        if (i < n) {
            if (iy > 0) { cs[m] = 0; vs[m++] = 0; }
            if (ix > 0) { cs[m] = 1; vs[m++] = 0; }
            cs[m] = 2; vs[m++] = 1;
            if (ix < N - 1) { cs[m] = 3; vs[m++] = 0; }
            if (iy < N - 1) { cs[m] = 4; vs[m++] = 0; }
        }
        for (int j = 0; j < 5; ++j) {
            vc[((size_t)sl * 5 + j) * 32 + lane] = (unsigned char)(j < m ? vs[j] : 2);
            cc[((size_t)sl * 5 + j) * 32 + lane] = (unsigned char)(j < m ? cs[j] : 2);
        }
    }
}

// stream copy reference (read 2 arrays, write 1) to calibrate the achievable bandwidth
__global__ void copy3(const double2* a, const double2* b, double2* c, size_t n2) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n2; k += (size_t)gridDim.x * blockDim.x) {
        double2 x = a[k], y = b[k];
        c[k] = make_double2(x.x + y.x, x.y + y.y);
    }
}

__global__ void build5(int N, int* sptr, int* col, double* val) {
    const int n = N * N, nsl = (n + 31) / 32;
    for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < (long)nsl * 32; t += (long)gridDim.x * blockDim.x) {
        int sl = (int)(t >> 5), lane = (int)(t & 31), i = sl * 32 + lane;
        if (lane == 0) sptr[sl] = sl * 5;
        if (t == 0) sptr[nsl] = nsl * 5;
        int iy = i / N, ix = i % N;
        int cs[5];
        double vs[5];
        int m = 0;
        if (i < n) {
            if (iy > 0) { cs[m] = i - N; vs[m++] = -1; }
            if (ix > 0) { cs[m] = i - 1; vs[m++] = -1; }
            cs[m] = i; vs[m++] = 4;
            if (ix < N - 1) { cs[m] = i + 1; vs[m++] = -1; }
            if (iy < N - 1) { cs[m] = i + N; vs[m++] = -1; }
        }
        for (int j = 0; j < 5; ++j) {
            col[((size_t)sl * 5 + j) * 32 + lane] = j < m ? cs[j] : (i < n ? i : 0);
            val[((size_t)sl * 5 + j) * 32 + lane] = j < m ? vs[j] : 0.0;
        }
    }
}

__global__ void fill(double* x, size_t n, double s) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x)
        x[k] = s * (double)((k * 2654435761u) % 1000) / 1000.0;
}

int main(int argc, char** argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 4096;
    const int n = N * N, nsl = (n + 31) / 32;
    const long nnz = (long)n + 4L * N * (N - 1);
    int *sptr, *col;
    double *val, *xg, *f, *xp, *out;
    CKM(cudaMalloc(&sptr, sizeof(int) * (nsl + 1)));
    CKM(cudaMalloc(&col, sizeof(int) * (size_t)nsl * 160 + 256));
    CKM(cudaMalloc(&val, sizeof(double) * (size_t)nsl * 160 + 256));
    for (double** p : {&xg, &f, &xp, &out}) CKM(cudaMalloc(p, sizeof(double) * (size_t)n + 256));
    build5<<<4096, 256>>>(N, sptr, col, val);
    fill<<<4096, 256>>>(xg, n, 1.0);
    fill<<<4096, 256>>>(f, n, 2.0);
    fill<<<4096, 256>>>(xp, n, 3.0);
    CKM(cudaDeviceSynchronize());
    int nsm = 0;
    CKM(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    Args a{n, nsl, sptr, col, val, xg, f, xp, out, 1.2698738636122384, 0.2886};
    const double model = 12.0 * nnz + 36.0 * n;
    const double actual = 12.0 * nsl * 160 + 4.0 * (nsl + 1) + 32.0 * n;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        for (int r = 0; r < 3; ++r) launch();
        CKM(cudaDeviceSynchronize());
        const int R = 20;
        cudaEventRecord(e0);
        for (int r = 0; r < R; ++r) launch();
        cudaEventRecord(e1);
        CKM(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double us = 1e3 * ms / R;
        printf("%-34s %8.1f us  model %6.0f GB/s  actual %6.0f GB/s\n", name, us, model / us / 1e3, actual / us / 1e3);
    };
    auto occ = [&](auto k) {
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, 256, 0);
        return b * nsm;
    };
    {
        size_t n2 = (size_t)n / 2 * 3;  // ~ same bytes as a smoother pass: 3 arrays of 1.5 n doubles
        double *A, *B, *Cc;
        CKM(cudaMalloc(&A, n2 * 16));
        CKM(cudaMalloc(&B, n2 * 16));
        CKM(cudaMalloc(&Cc, n2 * 16));
        for (int r = 0; r < 3; ++r) copy3<<<nsm * 8, 256>>>((double2*)A, (double2*)B, (double2*)Cc, n2);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 20; ++r) copy3<<<nsm * 8, 256>>>((double2*)A, (double2*)B, (double2*)Cc, n2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-34s %8.1f us  %6.0f GB/s (3 x %.0f MB)\n", "stream a+b->c", 1e3 * ms / 20, 3.0 * n2 * 16 / (1e3 * ms / 20) / 1e3, n2 * 16 / 1e6);
        cudaFree(A); cudaFree(B); cudaFree(Cc);
    }
    printf("n=%d nnz=%ld model bytes %.3f GB actual %.3f GB\n", n, nnz, model / 1e9, actual / 1e9);
    run("v0<8> resident grid", [&] { v0<8><<<occ(v0<8>), 256>>>(a); });
    run("v0<4> resident grid", [&] { v0<4><<<occ(v0<4>), 256>>>(a); });
    run("v0<8> grid = all slices", [&] { v0<8><<<(nsl + 7) / 8, 256>>>(a); });
    run("v1<8,1>", [&] { v1<8, 1><<<occ(v1<8, 1>), 256>>>(a); });
    {
        Args ai = a;
        ai.out = const_cast<double*>(ai.xprev);  // in place: out aliases xprev
        run("v1<8,1> in-place (nc)", [&] { v1<8, 1><<<occ(v1<8, 1>), 256>>>(ai); });
        run("v1b<8> in-place (plain)", [&] { v1b<8><<<occ(v1b<8>), 256>>>(ai); });
        run("v1b<8> separate out (plain)", [&] { v1b<8><<<occ(v1b<8>), 256>>>(a); });
    }
    run("v1<8,4>", [&] { v1<8, 4><<<occ(v1<8, 4>), 256>>>(a); });
    run("v1<4,4>", [&] { v1<4, 4><<<occ(v1<4, 4>), 256>>>(a); });
    run("v1<8,4> grid = all slices", [&] { v1<8, 4><<<(nsl + 7) / 8, 256>>>(a); });
    run("v1<4,6>", [&] { v1<4, 6><<<occ(v1<4, 6>), 256>>>(a); });
    run("v1<8,8> (32 regs)", [&] { v1<8, 8><<<occ(v1<8, 8>), 256>>>(a); });
    run("v2<5>", [&] { v2<5><<<occ(v2<5>), 256>>>(a); });
    run("v2<8>", [&] { v2<8><<<occ(v2<8>), 256>>>(a); });
    {
        int g = occ(v3<8>);
        int per = (nsl + g - 1) / g;
        run("v3<8> contiguous chunks", [&] { v3<8><<<g, 256>>>(a, per); });
    }
    {
        unsigned char *vc, *cc;
        double* vd;
        int* cd;
        CKM(cudaMalloc(&vc, (size_t)nsl * 160 + 256));
        CKM(cudaMalloc(&cc, (size_t)nsl * 160 + 256));
        CKM(cudaMalloc(&vd, 256 * 8));
        CKM(cudaMalloc(&cd, 256 * 4));
        double hv[256] = {-1.0, 4.0, 0.0};
        int hc[256] = {-N, -1, 0, 1, N};
        CKM(cudaMemcpy(vd, hv, sizeof(hv), cudaMemcpyHostToDevice));
        CKM(cudaMemcpy(cd, hc, sizeof(hc), cudaMemcpyHostToDevice));
        build5c<<<4096, 256>>>(N, vc, cc);
        CKM(cudaDeviceSynchronize());
        CArgs c{n, nsl, sptr, vc, cc, vd, cd, xg, f, xp, out, a.alpha, a.beta};
        const double cbytes = 2.0 * nsl * 160 + 32.0 * n;
        auto runc = [&](const char* name, auto k) {
            int g = occ(k);
            for (int r = 0; r < 3; ++r) k<<<g, 256>>>(c);
            CKM(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            for (int r = 0; r < 20; ++r) k<<<g, 256>>>(c);
            cudaEventRecord(e1);
            CKM(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double us = 1e3 * ms / 20;
            printf("%-34s %8.1f us  actual %6.0f GB/s  (grid %d)\n", name, us, cbytes / us / 1e3, g);
        };
        runc("vc NS=1", vc_k<1, 1>);
        runc("vc NS=2", vc_k<2, 1>);
        runc("vc NS=4", vc_k<4, 1>);
        runc("vc NS=1 minb4", vc_k<1, 4>);
        runc("vc NS=2 minb3", vc_k<2, 3>);
        auto runu = [&](const char* name, auto k) {
            int g = occ(k);
            run(name, [&] { k<<<g, 256>>>(a); });
        };
        runu("vu NS=1", vu_k<1, 1>);
        runu("vu NS=2", vu_k<2, 1>);
        runu("vu NS=1 minb4", vu_k<1, 4>);
    }
    printf("occupancy (blocks/GPU): v0<8> %d v1<8,1> %d v1<8,4> %d v2<5> %d v2<8> %d\n", occ(v0<8>), occ(v1<8, 1>),
           occ(v1<8, 4>), occ(v2<5>), occ(v2<8>));
    return 0;
}
