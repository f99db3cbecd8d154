// k_setup.cu -- setup-phase kernels of libamg_b200.so (sm_100a): SURVEY.md 8(a) rows a1-a8.
//
//  * lambda_1 = ||A||_inf: per-row |a| sums in CSR order, max by an
//    ordered-integer atomicMax (exact, order independent).
//  * Aggregation by repeated pairwise matching (l.62-73; readings A1-A5 in DESIGN.md): the
//    integer-keyed handshake (propose / accept rounds) -- equal to the sequential edge-greedy
//    matching for the strict key order of docs/keys.md -- then attach, leader numbering by an
//    exclusive scan, and the quotient pass graph (l.88-95) by radix sort + segmented sums.
//  * Galerkin A_H = P^T A P (l.112, "simple summations", l.401-402): keys (agg(i), agg(j)) for
//    every stored entry, stable radix sort of the entry indices, then one sequential sum per
//    coarse entry in (row, CSR position) order.
//  * Dense coarsest (pseudo-)inverse by Gauss-Jordan steps (SPD, no pivoting).
// CUB (header-only, CUDA 12.9) supplies the radix sorts and scans.
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "amg_internal.h"

namespace amg {

void dfree(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

static int grid_for(int64_t n) {
    int64_t g = (n + kBlock - 1) / kBlock;
    if (g < 1) g = 1;
    if (g > 65535 * 8) g = 65535 * 8;
    return (int)g;
}

// grids of kernels that end in one global atomic per warp: a few waves of grid-stride blocks, so
// the atomics do not serialise at one L2 slice (n / 256 blocks made them the kernels' cost)
static int grid_red(int64_t n) { return std::min(grid_for(n), 148 * 8); }

__device__ __forceinline__ int warp_max_i(int m) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    return m;
}

// persistent pinned host scratch (one per host thread) for the few scalars setup reads back
static void* pinned_scratch() {
    static thread_local void* p = nullptr;
    if (!p) CK(cudaMallocHost(&p, 256));
    return p;
}

template <class T>
static T read_scalar(const T* dptr, cudaStream_t s) {
    T* h = static_cast<T*>(pinned_scratch());
    CK(cudaMemcpyAsync(h, dptr, sizeof(T), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return *h;
}

static int bits_for(int64_t x) {  // smallest b >= 1 with 2^b >= x
    int b = 1;
    while ((int64_t(1) << b) < x) ++b;
    return b;
}

// exclusive scan of int32 flags/counts into out (n+1 entries: out[n] = total); returns total
// the same without reading the total back (callers that know it: no host synchronisation)
static void exclusive_scan(const int* in, int* out, int n, cudaStream_t s) {
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n + 1, s));
    void* tmp = dalloc<char>(tb, s);
    CK(cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, n + 1, s));
    dfree(tmp, s);
}

static int64_t exclusive_scan_total(const int* in, int* out, int n, cudaStream_t s) {
    exclusive_scan(in, out, n, s);
    int total = read_scalar(out + n, s);
    return total;
}

template <class K, class V>
static void sort_pairs(const K* kin, K* kout, const V* vin, V* vout, int n, int end_bit, cudaStream_t s) {
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, 0, end_bit, s));
    void* tmp = dalloc<char>(tb, s);
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, n, 0, end_bit, s));
    dfree(tmp, s);
}

void free_csr(Csr& A, cudaStream_t s) {
    dfree(A.rp, s);
    dfree(A.ci, s);
    dfree(A.v, s);
    A = Csr{};
}

void free_graph(PassGraph& g, cudaStream_t s) {
    dfree(g.rp, s);
    dfree(g.ci, s);
    dfree(g.w, s);
    g = PassGraph{};
}

// ------------------------------------------------------------------ validation (A17)
enum : int {
    VF_RANGE = 1, VF_UNSORTED = 2, VF_POSOFF = 4, VF_ASYM = 8, VF_DIAG = 16, VF_D = 32, VF_RP = 64
};

// Columns must lie in [cmin, cmax): [0, n) on one GPU; [-nlo, n + nhi) on a row-partitioned level
// (columns relative to the first own row, halo outside [0, n)).  Symmetry is checked for pairs of
// own rows (a cross-block pair is split between two ranks: the caller's contract).
// Every row range is checked against [0, nnz] before it is read (a non-monotone row_ptr must give
// AMG_E_INPUT, not an out-of-bounds read); so is the neighbour row searched for the symmetric entry.
__device__ __forceinline__ bool row_ok(int64_t p0, int64_t p1, int64_t nnz) { return 0 <= p0 && p0 <= p1 && p1 <= nnz; }

__global__ void k_validate(int n, int64_t nnz, int cmin, int cmax, const int64_t* __restrict__ rp,
                           const int32_t* __restrict__ ci, const double* __restrict__ v, const double* __restrict__ d,
                           int* flags) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int f = 0;
        const int64_t p0 = rp[i], p1 = rp[i + 1];
        if (!row_ok(p0, p1, nnz) || (i == 0 && p0 != 0) || (i == n - 1 && p1 != nnz)) { atomicOr(flags, VF_RP); continue; }
        double off = 0.0, dv = 0.0;
        bool has = false;
        for (int64_t p = p0; p < p1; ++p) {
            const int c = ci[p];
            if (c < cmin || c >= cmax) { f |= VF_RANGE; continue; }
            if (p > p0 && c <= ci[p - 1]) f |= VF_UNSORTED;
            if (c == i) { has = true; dv = v[p]; continue; }
            if (!(v[p] <= 0.0)) f |= VF_POSOFF;  // weights w_e >= 0 (structural zeros allowed, A17)
            off += -v[p];
            if (c < 0 || c >= n) continue;
            int64_t lo = rp[c], hi = rp[c + 1];
            const int64_t end = hi;
            if (!row_ok(lo, hi, nnz)) { f |= VF_RP; continue; }
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                if (ci[mid] < i) lo = mid + 1; else hi = mid;
            }
            if (!(lo < end && ci[lo] == i && v[lo] == v[p])) f |= VF_ASYM;
        }
        if (has && fabs(dv - off) > 1e-10 * (fabs(dv) + off)) f |= VF_DIAG;
        if (d && !(d[i] >= 0.0)) f |= VF_D;
        if (f) atomicOr(flags, f);
    }
}

// The pattern part of the checks (row_ptr monotone, columns in [0, n) and strictly increasing,
// pattern symmetry) and the int32 row pointers of the pattern: enough to run the value-free matching passes of level 0
// safely while the values are still being copied in (e2e path).
__global__ void k_pattern_rp32(int n, int64_t nnz, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                               int* __restrict__ rp32, int* flags) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
        rp32[i] = (int)rp[i];
        if (i == n) continue;
        const int64_t p0 = rp[i], p1 = rp[i + 1];
        if (!row_ok(p0, p1, nnz) || (i == 0 && p0 != 0) || (i == n - 1 && p1 != nnz)) { atomicOr(flags, VF_RP); continue; }
        int f = 0;
        for (int64_t p = p0; p < p1; ++p) {
            const int c = ci[p];
            if (c < 0 || c >= n) { f |= VF_RANGE; continue; }
            if (p > p0 && c <= ci[p - 1]) f |= VF_UNSORTED;
            if (c == i) continue;
            int64_t lo = rp[c], hi = rp[c + 1];  // the pattern must be symmetric (the matching relies on it)
            const int64_t end = hi;
            if (!row_ok(lo, hi, nnz)) { f |= VF_RP; continue; }
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (ci[mid] < i) lo = mid + 1; else hi = mid;
            }
            if (!(lo < end && ci[lo] == i)) f |= VF_ASYM;
        }
        if (f) atomicOr(flags, f);
    }
}

int pattern_rp32(int n, int64_t nnz, const int64_t* rp, const int32_t* ci, int* rp32, cudaStream_t s) {
    int* fl = dalloc<int>(1, s);
    CK(cudaMemsetAsync(fl, 0, sizeof(int), s));
    k_pattern_rp32<<<grid_for((int64_t)n + 1), kBlock, 0, s>>>(n, nnz, rp, ci, rp32, fl);
    ++g_launches;
    CK(cudaGetLastError());
    int f = read_scalar(fl, s);
    dfree(fl, s);
    return f;
}

int validate_input(int n, int64_t nnz, int cmin, int cmax, const int64_t* rp, const int32_t* ci, const double* v,
                   const double* d, cudaStream_t s) {
    int* fl = dalloc<int>(1, s);
    CK(cudaMemsetAsync(fl, 0, sizeof(int), s));
    k_validate<<<grid_for(n), kBlock, 0, s>>>(n, nnz, cmin, cmax, rp, ci, v, d, fl);
    ++g_launches;
    CK(cudaGetLastError());
    int f = read_scalar(fl, s);
    dfree(fl, s);
    return f;
}

// ------------------------------------------------------------------ A_0 = L + diag(d) (Eq. (prob))
__global__ void k_a0_count(int n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int* cnt) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        bool has = false;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) has |= (ci[p] == i);
        cnt[i] = (int)(rp[i + 1] - rp[i]) + (has ? 0 : 1);
    }
}

__global__ void k_a0_fill(int n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ v, const double* __restrict__ d, const int* __restrict__ orp,
                          int* __restrict__ oci, double* __restrict__ ov) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        bool has = false;
        double off = 0.0;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            has |= (ci[p] == i);
            if (ci[p] != i) off += -v[p];
        }
        const double di = d ? d[i] : 0.0;
        int q = orp[i];
        bool done = has;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            if (!done && ci[p] > i) { oci[q] = i; ov[q] = off + di; ++q; done = true; }
            oci[q] = ci[p];
            ov[q] = (ci[p] == i) ? v[p] + di : v[p];
            ++q;
        }
        if (!done) { oci[q] = i; ov[q] = off + di; }
    }
}

Csr form_A0(int n, const int64_t* rp, const int32_t* ci, const double* v, const double* d, cudaStream_t s) {
    int* cnt = dalloc<int>((size_t)n + 1, s);
    CK(cudaMemsetAsync(cnt + n, 0, sizeof(int), s));
    k_a0_count<<<grid_for(n), kBlock, 0, s>>>(n, rp, ci, cnt);
    ++g_launches;
    CK(cudaGetLastError());
    Csr A;
    A.n = n;
    A.rp = dalloc<int>((size_t)n + 1, s);
    // nnz must fit int32 (checked by the caller on the input nnz + n)
    A.nnz = exclusive_scan_total(cnt, A.rp, n, s);
    dfree(cnt, s);
    A.ci = dalloc<int>((size_t)A.nnz + 8, s);
    A.v = dalloc<double>((size_t)A.nnz + 8, s);
    CK(cudaMemsetAsync(A.ci + A.nnz, 0, 8 * sizeof(int), s));
    CK(cudaMemsetAsync(A.v + A.nnz, 0, 8 * sizeof(double), s));
    k_a0_fill<<<grid_for(n), kBlock, 0, s>>>(n, rp, ci, v, d, A.rp, A.ci, A.v);
    ++g_launches;
    CK(cudaGetLastError());
    return A;
}

__global__ void k_any_nonzero(int n, const double* __restrict__ d, int* flag) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (d[i] != 0.0) *flag = 1;
}

bool any_nonzero(int n, const double* d, cudaStream_t s) {
    int* fl = dalloc<int>(1, s);
    CK(cudaMemsetAsync(fl, 0, sizeof(int), s));
    k_any_nonzero<<<grid_for(n), kBlock, 0, s>>>(n, d, fl);
    ++g_launches;
    CK(cudaGetLastError());
    int f = read_scalar(fl, s);
    dfree(fl, s);
    return f != 0;
}

// ------------------------------------------------------------------ Lanczos start vector (A24)
__device__ __forceinline__ uint64_t sm64(uint64_t z);
__global__ void k_lanczos_start(int n, uint64_t z, double* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = 2.0 * ((double)(sm64(z ^ (uint64_t)i) >> 11) * 0x1.0p-53) - 1.0;
}

void launch_lanczos_start(int n, uint64_t z, double* out, cudaStream_t s) {
    k_lanczos_start<<<grid_for(n), kBlock, 0, s>>>(n, z, out);
    ++g_launches;
    CK(cudaGetLastError());
}

// ------------------------------------------------------------------ lambda_1 (a1)
__global__ void k_rowabs_max(int n, const int* __restrict__ rp, const double* __restrict__ v,
                             unsigned long long* out) {
    double m = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int p = rp[i]; p < rp[i + 1]; ++p) s += fabs(v[p]);
        m = fmax(m, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// lambda_1 into a device slot (zeroed by the caller; the bit pattern of a double >= 0 orders as an
// unsigned integer), read back later together with the other levels' (no host synchronisation)
void inf_norm_launch(const Csr& A, unsigned long long* o, cudaStream_t s) {
    k_rowabs_max<<<grid_red(A.n), kBlock, 0, s>>>(A.n, A.rp, A.v, o);
    ++g_launches;
    CK(cudaGetLastError());
}

double inf_norm(const Csr& A, cudaStream_t s) {
    unsigned long long* o = dalloc<unsigned long long>(1, s);
    CK(cudaMemsetAsync(o, 0, sizeof(unsigned long long), s));
    k_rowabs_max<<<grid_red(A.n), kBlock, 0, s>>>(A.n, A.rp, A.v, o);
    ++g_launches;
    CK(cudaGetLastError());
    unsigned long long h = read_scalar(o, s);
    dfree(o, s);
    double r;
    memcpy(&r, &h, sizeof(double));
    return r;
}

// ------------------------------------------------------------------ pass graph G_0 (A5)
__global__ void k_g0_count(int n, const int* __restrict__ rp, const int* __restrict__ ci, int* cnt) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int c = 0;
        for (int p = rp[i]; p < rp[i + 1]; ++p) c += (ci[p] != i && ci[p] >= 0 && ci[p] < n);
        cnt[i] = c;
    }
}

__global__ void k_g0_fill(int n, const int* __restrict__ rp, const int* __restrict__ ci, const int* __restrict__ grp,
                          int* __restrict__ gci, uint32_t* __restrict__ gw) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int q = grp[i];
        for (int p = rp[i]; p < rp[i + 1]; ++p)
            if (ci[p] != i && ci[p] >= 0 && ci[p] < n) { gci[q] = ci[p]; gw[q] = 1u; ++q; }
    }
}

PassGraph pass_graph0(const Csr& A, cudaStream_t s) {
    PassGraph G;
    G.n = A.n;
    int* cnt = dalloc<int>((size_t)A.n + 1, s);
    CK(cudaMemsetAsync(cnt + A.n, 0, sizeof(int), s));
    k_g0_count<<<grid_for(A.n), kBlock, 0, s>>>(A.n, A.rp, A.ci, cnt);
    ++g_launches;
    CK(cudaGetLastError());
    G.rp = dalloc<int>((size_t)A.n + 1, s);
    G.nnz = exclusive_scan_total(cnt, G.rp, A.n, s);
    dfree(cnt, s);
    G.ci = dalloc<int>((size_t)G.nnz, s);
    G.w = dalloc<uint32_t>((size_t)G.nnz, s);
    k_g0_fill<<<grid_for(A.n), kBlock, 0, s>>>(A.n, A.rp, A.ci, G.rp, G.ci, G.w);
    ++g_launches;
    CK(cudaGetLastError());
    G.unit = true;  // multiplicities start at 1 on every level (A5)
    return G;
}

// ------------------------------------------------------------------ matching keys (docs/keys.md)
__device__ __forceinline__ uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

struct EKey {
    uint32_t w;
    uint64_t h;
    int lo, hi;
};

// a, b: local vertex ids of G_t; `off` = global id of local vertex 0 (row-partitioned levels:
// docs/keys.md uses global ids; 0 on one GPU).  The order of keys is offset invariant except
// through the hash, which must see the global ids.
__device__ __forceinline__ EKey make_key(uint32_t w, int a, int b, uint64_t salt, int off) {
    a += off;
    b += off;
    EKey k;
    k.w = w;
    k.lo = a < b ? a : b;
    k.hi = a < b ? b : a;
    k.h = sm64((((uint64_t)(uint32_t)k.lo) << 32 | (uint64_t)(uint32_t)k.hi) ^ salt);
    return k;
}

__device__ __forceinline__ bool key_gt(const EKey& a, const EKey& b) {
    if (a.w != b.w) return a.w > b.w;
    if (a.h != b.h) return a.h > b.h;
    if (a.lo != b.lo) return a.lo > b.lo;
    return a.hi > b.hi;
}

// handshake round, step 1: every free vertex (mate -1) proposes to its max-key free neighbour.  A
// free vertex with no free neighbour can never be matched (matches are never undone): it is marked
// settled (mate -2, unmatched) so later rounds skip it.  Within one round only settled marks are
// written, and a vertex is settled only if no neighbour is free, so no free vertex reads one.
// G lanes per vertex (G a power of two <= 32, picked from the mean degree): lane t scans entries
// t, t+G, ... and the group takes the max key by a shuffle butterfly.  Keys are distinct per
// neighbour (they end in (lo, hi)), so the max does not depend on the scan order.  `list` (or
// nullptr = all vertices 0..nv) holds the vertices still free when the batch started.
__device__ __forceinline__ bool prop_gt(uint32_t w1, uint64_t h1, int u1, uint32_t w2, uint64_t h2, int u2, int v) {
    if (w1 != w2) return w1 > w2;
    if (h1 != h2) return h1 > h2;
    const int lo1 = min(u1, v), hi1 = max(u1, v), lo2 = min(u2, v), hi2 = max(u2, v);
    if (lo1 != lo2) return lo1 > lo2;
    return hi1 > hi2;
}

template <int G>
__global__ void __launch_bounds__(kBlock) k_propose(int nv, const int* __restrict__ nvp, const int* __restrict__ list,
                                                    const int* __restrict__ rp, const int* __restrict__ ci,
                                                    const uint32_t* __restrict__ w, int* __restrict__ mate,
                                                    int* __restrict__ prop, uint64_t salt, int off, int* any) {
    if (nvp) nv = *nvp;  // list length produced on the device (no host read-back)
    __shared__ int bany;
    if (threadIdx.x == 0) bany = 0;
    __syncthreads();
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31, t = lane & (G - 1), gi = lane / G;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    bool found = false;
    for (int base = wid * GPW; base < nv; base += nw * GPW) {  // trip count uniform per warp
        const int idx = base + gi;
        const int v = idx < nv ? (list ? list[idx] : idx) : -1;
        const bool act = v >= 0 && mate[v] == -1;
        uint32_t bw = 0;
        uint64_t bh = 0;
        int bu = -1;
        if (act) {
            // the lane's entries in batches of 4: columns and weights, then the mate gathers, are each
            // in flight together (the max over distinct keys does not depend on the visiting order)
            const int p1 = rp[v + 1];
            for (int p = rp[v] + t; p < p1; p += 4 * G) {
                int uu[4];
                uint32_t ww[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int q = p + k * G;
                    uu[k] = q < p1 ? ci[q] : -1;
                    ww[k] = q < p1 ? (w ? w[q] : 1u) : 0u;
                }
                bool fr[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) fr[k] = uu[k] >= 0 && mate[uu[k]] == -1;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (!fr[k]) continue;
                    const int u = uu[k];
                    const EKey key = make_key(ww[k], v, u, salt, off);
                    if (bu < 0 || prop_gt(key.w, key.h, u, bw, bh, bu, v)) { bw = key.w; bh = key.h; bu = u; }
                }
            }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            const uint32_t ow = __shfl_xor_sync(0xffffffffu, bw, o, G);
            const uint64_t oh = __shfl_xor_sync(0xffffffffu, bh, o, G);
            const int ou = __shfl_xor_sync(0xffffffffu, bu, o, G);
            if (ou >= 0 && (bu < 0 || prop_gt(ow, oh, ou, bw, bh, bu, v))) { bw = ow; bh = oh; bu = ou; }
        }
        if (act && t == 0) {
            if (bu < 0) mate[v] = -2;
            prop[v] = bu;
            found |= bu >= 0;
        }
    }
    if (found) bany = 1;
    __syncthreads();
    if (threadIdx.x == 0 && bany) *any = 1;
}

// handshake round, step 2: mutual proposals match.  A free vertex's proposal target u was free when
// the batch started, so u is on the list and prop[u] is this round's.
__global__ void k_accept(int nv, const int* __restrict__ nvp, const int* __restrict__ list, int* __restrict__ mate,
                         const int* __restrict__ prop) {
    if (nvp) nv = *nvp;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nv; idx += gridDim.x * blockDim.x) {
        const int v = list ? list[idx] : idx;
        if (mate[v] != -1) continue;
        const int u = prop[v];
        if (u >= 0 && prop[u] == v) mate[v] = u;
    }
}

// free-list compaction: the vertices of list (or of 0..n-1) still free, appended tile by tile (tiles of
// kBlock * 16 entries, one atomic per tile, so the atomics never serialise at one L2 slice).  The
// order of the list changes no result: every round's proposal and acceptance is a function of the
// vertex and of mate[] alone.
__global__ void __launch_bounds__(kBlock) k_compact_free(int n, const int* __restrict__ nvp, const int* __restrict__ list,
                                                         const int* __restrict__ mate, int* __restrict__ out,
                                                         int* __restrict__ cnt) {
    constexpr int IT = 16, TILE = kBlock * IT, NW = kBlock / 32;
    const int nv = nvp ? *nvp : n;
    __shared__ int wsum[NW];
    __shared__ int base;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t t0 = (int64_t)blockIdx.x * TILE; t0 < nv; t0 += (int64_t)gridDim.x * TILE) {
        int v[IT];
        int c = 0;
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            const int64_t idx = t0 + k * kBlock + threadIdx.x;
            v[k] = idx < nv ? (list ? list[idx] : (int)idx) : -1;
        }
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            if (v[k] >= 0 && mate[v[k]] != -1) v[k] = -1;
            c += v[k] >= 0;
        }
        int inc = c;  // inclusive warp scan of the per-thread counts
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wsum[wid] = inc;
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int k = 0; k < NW; ++k) { const int x = wsum[k]; wsum[k] = t; t += x; }
            base = t ? atomicAdd(cnt, t) : 0;
        }
        __syncthreads();
        int pos = base + wsum[wid] + inc - c;
#pragma unroll
        for (int k = 0; k < IT; ++k)
            if (v[k] >= 0) out[pos++] = v[k];
        __syncthreads();  // wsum / base are rewritten by the next tile
    }
}

// attach (A3) + leader (A4)
__global__ void k_leader(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                         const uint32_t* __restrict__ w, const int* __restrict__ mate, uint64_t salt, int off,
                         int* __restrict__ leader, int* __restrict__ isl) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int m = mate[v];
        if (m >= 0) {
            leader[v] = v < m ? v : m;
            isl[v] = v < m;
        } else if (rp[v + 1] > rp[v]) {
            EKey bk{};
            int bu = -1;
            for (int p = rp[v]; p < rp[v + 1]; ++p) {
                EKey k = make_key(w ? w[p] : 1u, v, ci[p], salt, off);
                if (bu < 0 || key_gt(k, bk)) { bk = k; bu = ci[p]; }
            }
            const int mu = mate[bu];  // matched by maximality
            leader[v] = bu < mu ? bu : mu;
            isl[v] = 0;
        } else {
            leader[v] = v;
            isl[v] = 1;
        }
    }
}

__global__ void k_assign(int n, const int* __restrict__ leader, const int* __restrict__ id, int* __restrict__ agg) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) agg[v] = id[leader[v]];
}

// One matching pass of a small pass graph in ONE cooperative launch (a2 + a3): the handshake rounds
// of k_propose / k_accept, the attach and leader rule of k_leader, the leader numbering (exclusive
// scan in vertex order) and k_assign, with grid barriers in place of kernel boundaries and of the
// host's per-batch read-backs.  The rounds stop after the first round in which no free vertex found
// a free neighbour: that round settles every vertex still free, and any later round is a no-op, so
// the matching is the launch path's.  mate / prop / leader are written inside the launch, so they are
// read with ld.global.cg (L2), never through the incoherent L1.  ctl: [0..1] round flags (double
// buffered), [2] n_c, [3] rounds.
template <int G>
__global__ void __launch_bounds__(kBlock) k_match_coop(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                       const uint32_t* __restrict__ w, int* mate, int* prop,
                                                       int* leader, int* bcnt, int* ctl, uint64_t salt, int off,
                                                       int* __restrict__ agg_t) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ int wsh[kBlock / 32];
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31, t = lane & (G - 1), gi = lane / G, wl = threadIdx.x >> 5;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gth = gridDim.x * blockDim.x;
    auto block_sum = [&](int x) {  // every thread gets the block's sum
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) wsh[wl] = x;
        __syncthreads();
        int tot = 0;
#pragma unroll
        for (int k = 0; k < kBlock / 32; ++k) tot += wsh[k];
        __syncthreads();
        return tot;
    };
    for (int v = gtid; v < n; v += gth) mate[v] = -1;
    if (gtid == 0) { ctl[0] = 0; ctl[1] = 0; }
    grid.sync();
    int r = 0;
    for (;; ++r) {
        bool found = false;
        for (int base = wid * GPW; base < n; base += nw * GPW) {  // k_propose's body, list = all vertices
            const int v = base + gi < n ? base + gi : -1;
            const bool act = v >= 0 && __ldcg(&mate[v]) == -1;
            uint32_t bw = 0;
            uint64_t bh = 0;
            int bu = -1;
            if (act) {
                const int p1 = rp[v + 1];
                for (int p = rp[v] + t; p < p1; p += 4 * G) {
                    int uu[4];
                    uint32_t ww[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int q = p + k * G;
                        uu[k] = q < p1 ? ci[q] : -1;
                        ww[k] = q < p1 ? (w ? w[q] : 1u) : 0u;
                    }
                    bool fr[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) fr[k] = uu[k] >= 0 && __ldcg(&mate[uu[k]]) == -1;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (!fr[k]) continue;
                        const int u = uu[k];
                        const EKey key = make_key(ww[k], v, u, salt, off);
                        if (bu < 0 || prop_gt(key.w, key.h, u, bw, bh, bu, v)) { bw = key.w; bh = key.h; bu = u; }
                    }
                }
            }
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) {
                const uint32_t ow = __shfl_xor_sync(0xffffffffu, bw, o, G);
                const uint64_t oh = __shfl_xor_sync(0xffffffffu, bh, o, G);
                const int ou = __shfl_xor_sync(0xffffffffu, bu, o, G);
                if (ou >= 0 && (bu < 0 || prop_gt(ow, oh, ou, bw, bh, bu, v))) { bw = ow; bh = oh; bu = ou; }
            }
            if (act && t == 0) {
                if (bu < 0) mate[v] = -2;
                prop[v] = bu;
                found |= bu >= 0;
            }
        }
        if (__syncthreads_or(found) && threadIdx.x == 0) atomicExch(&ctl[r & 1], 1);
        grid.sync();
        const bool go = __ldcg(&ctl[r & 1]) != 0;
        if (!go) break;  // uniform: every thread read the flag after the barrier
        if (gtid == 0) ctl[(r + 1) & 1] = 0;  // next round's flag (its writers start after the next barrier)
        for (int v = gtid; v < n; v += gth) {  // k_accept
            if (__ldcg(&mate[v]) != -1) continue;
            const int u = __ldcg(&prop[v]);
            if (u >= 0 && __ldcg(&prop[u]) == v) mate[v] = u;
        }
        grid.sync();
    }
    // attach (A3) + leader (A4) over a contiguous chunk per block, so ids can be numbered in vertex order
    const int chunk = (n + gridDim.x - 1) / gridDim.x;
    const int v0 = min(n, blockIdx.x * chunk), v1 = min(n, v0 + chunk);
    int cnt = 0;
    for (int v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
        const int m = __ldcg(&mate[v]);
        int ld;
        if (m >= 0) {
            ld = v < m ? v : m;
        } else if (rp[v + 1] > rp[v]) {
            EKey bk{};
            int bu = -1;
            for (int p = rp[v]; p < rp[v + 1]; ++p) {
                EKey k = make_key(w ? w[p] : 1u, v, ci[p], salt, off);
                if (bu < 0 || key_gt(k, bk)) { bk = k; bu = ci[p]; }
            }
            const int mu = __ldcg(&mate[bu]);  // matched by maximality
            ld = bu < mu ? bu : mu;
        } else {
            ld = v;
        }
        leader[v] = ld;
        cnt += ld == v;  // leader flag: the smaller end of a pair, or an isolated vertex
    }
    cnt = block_sum(cnt);
    if (threadIdx.x == 0) bcnt[blockIdx.x] = cnt;
    grid.sync();
    int pre = 0;
    for (int k = threadIdx.x; k < (int)blockIdx.x; k += blockDim.x) pre += __ldcg(&bcnt[k]);
    pre = block_sum(pre);
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        ctl[2] = pre + cnt;
        ctl[3] = r + 1;
    }
    // ids: exclusive scan of the leader flags in vertex order (prop reused as the id array)
    for (int b0 = v0; b0 < v1; b0 += blockDim.x) {
        const int v = b0 + threadIdx.x;
        const bool fl = v < v1 && __ldcg(&leader[v]) == v;
        const unsigned bal = __ballot_sync(0xffffffffu, fl);
        if (lane == 0) wsh[wl] = __popc(bal);
        __syncthreads();
        int wpre = 0, tot = 0;
        for (int k = 0; k < kBlock / 32; ++k) {
            const int x = wsh[k];
            if (k < wl) wpre += x;
            tot += x;
        }
        if (fl) prop[v] = pre + wpre + __popc(bal & ((1u << lane) - 1u));
        pre += tot;
        __syncthreads();
    }
    grid.sync();
    for (int v = v0 + threadIdx.x; v < v1; v += blockDim.x) agg_t[v] = __ldcg(&prop[__ldcg(&leader[v])]);
}

int aggregate_pass(const PassGraph& G, uint64_t salt, int id_off, int* agg_t, int* nc, int* rounds, cudaStream_t s) {
    const int n = G.n;
    const uint32_t* Gw = G.unit ? nullptr : G.w;  // unit multiplicities: not read
    int* mate = dalloc<int>(n, s);
    int* prop = dalloc<int>(n, s);
    int* any = dalloc<int>(4, s);
    int r = 0;
    const int g = grid_for(n);
    // Rounds are issued in batches of 3, each batch followed by the compaction of the free list; the
    // matching is maximal once no vertex is left free (a vertex with no free neighbour settles at
    // mate -2 in its next proposal), and further rounds are no-ops, so the result does not depend
    // on the batch size.
    constexpr int kBatch = 3;
    static int gsel = -1;
    if (gsel < 0) gsel = getenv("AMG_PROPOSE_G") ? atoi(getenv("AMG_PROPOSE_G")) : 0;
    int Gl = gsel;
    if (Gl <= 0) {  // about four entries per lane
        const double dg = n > 0 ? (double)G.nnz / (double)n : 0.0;
        Gl = 2;
        while (Gl < 16 && 4.0 * Gl < dg) Gl <<= 1;
    }
    // small pass graphs: the whole pass in one cooperative launch (AMG_COOP_MATCH = largest n; 0 = off)
    static int coop_max = -1;
    if (coop_max < 0) coop_max = getenv("AMG_COOP_MATCH") ? atoi(getenv("AMG_COOP_MATCH")) : (1 << 20);
    if (n > 0 && n <= coop_max) {
        void (*fn)(int, const int*, const int*, const uint32_t*, int*, int*, int*, int*, int*, uint64_t, int, int*);
        switch (Gl) {
            case 1: fn = k_match_coop<1>; break;
            case 2: fn = k_match_coop<2>; break;
            case 4: fn = k_match_coop<4>; break;
            case 8: fn = k_match_coop<8>; break;
            default: fn = k_match_coop<16>; break;
        }
        int bpsm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm, fn, kBlock, 0));
        int dev = 0, nsm = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        const int want = (int)std::max<int64_t>(1, ((int64_t)n * Gl + kBlock - 1) / kBlock);
        const int nb = std::min(want, bpsm * nsm);
        if (nb >= 1 && bpsm >= 1) {
            int* leader = dalloc<int>((size_t)n + 1, s);
            int* bcnt = dalloc<int>((size_t)nb + 1, s);
            int* ctl = dalloc<int>(4, s);
            int n_ = n, off_ = id_off;
            uint64_t salt_ = salt;
            const int* rp_ = G.rp;
            const int* ci_ = G.ci;
            const uint32_t* w_ = Gw;
            void* args[] = {&n_, &rp_, &ci_, &w_, &mate, &prop, &leader, &bcnt, &ctl, &salt_, &off_, &agg_t};
            CK(cudaLaunchCooperativeKernel((const void*)fn, dim3(nb), dim3(kBlock), args, 0, s));
            ++g_launches;
            int* h = static_cast<int*>(pinned_scratch()) + 28;
            CK(cudaMemcpyAsync(h, ctl + 2, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            *nc = h[0];
            *rounds = h[1];
            dfree(leader, s);
            dfree(bcnt, s);
            dfree(ctl, s);
            dfree(mate, s);
            dfree(prop, s);
            dfree(any, s);
            return 0;
        }
    }
    CK(cudaMemsetAsync(mate, 0xff, sizeof(int) * (size_t)n, s));
    // After the first batch the rounds run over the vertices still free (a shrinking list).  The list
    // and its length stay on the device: batch b+1 is issued before batch b's length is known on the
    // host (its kernels read the length from device memory), so the host's read-back of batch b
    // overlaps batch b+1 and the GPU never waits on it.  When batch b leaves no free vertex the
    // matching is maximal and batch b+1 runs on an empty list (a no-op); the result does not depend
    // on the batching.
    int* lists = dalloc<int>(2 * ((size_t)n + 8), s);
    constexpr int R = 4;  // ring of device counts / pinned mirrors / events
    int* dcnt = dalloc<int>(R, s);
    volatile int* hcnt = static_cast<int*>(pinned_scratch()) + 20;
    cudaEvent_t ev[R];
    for (int k = 0; k < R; ++k) CK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
    static int first = -1;  // rounds before the first free-list compaction (AMG_MATCH_FIRST; 2 measured best)
    if (first < 0) first = getenv("AMG_MATCH_FIRST") ? std::max(1, atoi(getenv("AMG_MATCH_FIRST"))) : 2;
    // small graphs (coarse levels): rounds cost ~5 us, so the batches are longer there
    const bool small = n <= 200000;
    auto issue = [&](int b, int nv_ub) {  // batch b: rounds over list b, then list b+1 and its length
        const int* list = b ? lists + (size_t)(b & 1) * (n + 8) : nullptr;
        const int* nvp = b ? dcnt + (b - 1) % R : nullptr;
        int* out = lists + (size_t)((b + 1) & 1) * (n + 8);
        const int nb = b ? (small ? 4 : kBatch) : (small ? 6 : first);
        const int gp = std::max(1, std::min((int)(((int64_t)nv_ub * Gl + kBlock - 1) / kBlock), 148 * 8));
        const int ga = std::max(1, std::min(grid_for(nv_ub), 148 * 8));
        for (int k = 0; k < nb; ++k) {
            switch (Gl) {
                case 1: k_propose<1><<<gp, kBlock, 0, s>>>(nv_ub, nvp, list, G.rp, G.ci, Gw, mate, prop, salt, id_off, any); break;
                case 2: k_propose<2><<<gp, kBlock, 0, s>>>(nv_ub, nvp, list, G.rp, G.ci, Gw, mate, prop, salt, id_off, any); break;
                case 4: k_propose<4><<<gp, kBlock, 0, s>>>(nv_ub, nvp, list, G.rp, G.ci, Gw, mate, prop, salt, id_off, any); break;
                case 8: k_propose<8><<<gp, kBlock, 0, s>>>(nv_ub, nvp, list, G.rp, G.ci, Gw, mate, prop, salt, id_off, any); break;
                default: k_propose<16><<<gp, kBlock, 0, s>>>(nv_ub, nvp, list, G.rp, G.ci, Gw, mate, prop, salt, id_off, any); break;
            }
            k_accept<<<ga, kBlock, 0, s>>>(nv_ub, nvp, list, mate, prop);
            g_launches += 2;
        }
        CK(cudaMemsetAsync(dcnt + b % R, 0, sizeof(int), s));
        const int gc = std::max(1, std::min((int)((nv_ub + kBlock * 16 - 1) / (kBlock * 16)), 148 * 8));
        k_compact_free<<<gc, kBlock, 0, s>>>(nv_ub, nvp, list, mate, out, dcnt + b % R);
        ++g_launches;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync((void*)(hcnt + b % R), dcnt + b % R, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(ev[b % R], s));
        return nb;
    };
    int nv_ub = n;
    int nb = issue(0, nv_ub);
    for (int b = 0;; ++b) {
        const int nb_next = issue(b + 1, nv_ub);  // speculative: a no-op if batch b ends the matching
        CK(cudaEventSynchronize(ev[b % R]));
        r += nb;
        const int left = hcnt[b % R];
        if (left == 0) break;
        nv_ub = left;
        nb = nb_next;
        if (r > 30000) {
            CK(cudaStreamSynchronize(s));
            for (int k = 0; k < R; ++k) cudaEventDestroy(ev[k]);
            throw Error(-7, "matching did not terminate");
        }
    }
    for (int k = 0; k < R; ++k) CK(cudaEventDestroy(ev[k]));
    dfree(lists, s);
    dfree(dcnt, s);
    int* leader = prop;  // reuse
    int* isl = dalloc<int>((size_t)n + 1, s);
    CK(cudaMemsetAsync(isl + n, 0, sizeof(int), s));
    k_leader<<<g, kBlock, 0, s>>>(n, G.rp, G.ci, Gw, mate, salt, id_off, leader, isl);
    ++g_launches;
    CK(cudaGetLastError());
    int* id = dalloc<int>((size_t)n + 1, s);
    *nc = (int)exclusive_scan_total(isl, id, n, s);
    k_assign<<<g, kBlock, 0, s>>>(n, leader, id, agg_t);
    ++g_launches;
    CK(cudaGetLastError());
    dfree(id, s);
    dfree(isl, s);
    dfree(mate, s);
    dfree(prop, s);
    dfree(any, s);
    *rounds = r;
    return 0;
}

// ------------------------------------------------------------------ MIS-k aggregation (reading A25)
// The paper's own partitioner, opt-in (mis_k > 0).
// (A) S = the greedy MIS of the graph of A^k in decreasing key order, key(v) = (hi32(splitmix64(v ^
// misalt)) << 32) | v.  Computed by rounds with fixed priorities: an undecided vertex joins S iff its
// key is the largest among the undecided vertices within distance k (k max-propagation sweeps);
// then every undecided vertex within distance k of S is excluded (k OR sweeps).  A vertex joins only
// once every larger-key vertex of its k-ball is decided, and it is decided out only by an S member
// within distance k, so the rounds reproduce the sequential greedy set exactly.
// (B) layered growth: in layer d = 1..k every unassigned vertex takes, among its neighbours assigned
// in layers < d, the root of largest key.  Aggregate id = rank of the root in vertex order.
__device__ __forceinline__ uint64_t mis_key(int v, uint64_t misalt) {
    return ((sm64((uint64_t)v ^ misalt) >> 32) << 32) | (uint64_t)(uint32_t)v;
}

// state: 0 undecided, 1 in S, 2 excluded
__global__ void k_mis_seed(int n, const uint8_t* __restrict__ state, uint64_t misalt, uint64_t* __restrict__ M) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        M[v] = state[v] == 0 ? mis_key(v, misalt) : 0ull;
}

__global__ void k_mis_max(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                          const uint64_t* __restrict__ Min, uint64_t* __restrict__ Mout) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        uint64_t m = Min[v];
        for (int p = rp[v]; p < rp[v + 1]; ++p) m = max(m, Min[ci[p]]);
        Mout[v] = m;
    }
}

__global__ void k_mis_join(int n, uint8_t* __restrict__ state, const uint64_t* __restrict__ M, uint64_t misalt,
                           uint8_t* __restrict__ E) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        uint8_t st = state[v];
        if (st == 0 && M[v] == mis_key(v, misalt)) {
            st = 1;
            state[v] = 1;
        }
        E[v] = st == 1;
    }
}

__global__ void k_mis_or(int n, const int* __restrict__ rp, const int* __restrict__ ci, const uint8_t* __restrict__ Ein,
                         uint8_t* __restrict__ Eout) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        uint8_t e = Ein[v];
        for (int p = rp[v]; p < rp[v + 1] && !e; ++p) e = Ein[ci[p]];
        Eout[v] = e;
    }
}

__global__ void k_mis_exclude(int n, uint8_t* __restrict__ state, const uint8_t* __restrict__ E, int* any) {
    bool und = false;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        if (state[v] == 0) {
            if (E[v]) state[v] = 2;
            else und = true;
        }
    }
    if (__any_sync(0xffffffffu, und) && (threadIdx.x & 31) == 0) *any = 1;
}

__global__ void k_mis_root0(int n, const uint8_t* __restrict__ state, int* __restrict__ root, int* __restrict__ isl) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        root[v] = state[v] == 1 ? v : -1;
        isl[v] = state[v] == 1;
    }
}

__global__ void k_mis_grow(int n, const int* __restrict__ rp, const int* __restrict__ ci, const int* __restrict__ rin,
                           int* __restrict__ rout, uint64_t misalt) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        int r = rin[v];
        if (r < 0) {
            uint64_t bk = 0;
            for (int p = rp[v]; p < rp[v + 1]; ++p) {
                const int c = rin[ci[p]];
                if (c >= 0) {
                    const uint64_t k = mis_key(c, misalt);
                    if (r < 0 || k > bk) { r = c; bk = k; }
                }
            }
        }
        rout[v] = r;
    }
}

__global__ void k_mis_assign(int n, const int* __restrict__ root, const int* __restrict__ id, int* __restrict__ agg,
                             int* bad) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int r = root[v];
        if (r < 0) { *bad = 1; agg[v] = -1; }
        else agg[v] = id[r];
    }
}

int mis_aggregate(const PassGraph& G, int k, uint64_t seed, int level, int* agg, int* nc, int* rounds, cudaStream_t s) {
    const int n = G.n;
    const uint64_t misalt = host_sm64(seed ^ 0x4D49530000000000ULL ^ (uint64_t)level);
    uint8_t* state = dalloc<uint8_t>((size_t)n + 16, s);
    uint8_t* E0 = dalloc<uint8_t>((size_t)n + 16, s);
    uint8_t* E1 = dalloc<uint8_t>((size_t)n + 16, s);
    uint64_t* M0 = dalloc<uint64_t>((size_t)n + 1, s);
    uint64_t* M1 = dalloc<uint64_t>((size_t)n + 1, s);
    int* flag = dalloc<int>(2, s);
    int* hflag = static_cast<int*>(pinned_scratch()) + 48;
    CK(cudaMemsetAsync(state, 0, (size_t)n, s));
    const int g = grid_for(n);
    int r = 0;
    for (;;) {
        ++r;
        if (r > 100000) throw Error(-7, "MIS did not terminate");
        k_mis_seed<<<g, kBlock, 0, s>>>(n, state, misalt, M0);
        for (int d = 0; d < k; ++d) {
            k_mis_max<<<g, kBlock, 0, s>>>(n, G.rp, G.ci, M0, M1);
            std::swap(M0, M1);
        }
        k_mis_join<<<g, kBlock, 0, s>>>(n, state, M0, misalt, E0);
        for (int d = 0; d < k; ++d) {
            k_mis_or<<<g, kBlock, 0, s>>>(n, G.rp, G.ci, E0, E1);
            std::swap(E0, E1);
        }
        CK(cudaMemsetAsync(flag, 0, sizeof(int), s));
        k_mis_exclude<<<grid_red(n), kBlock, 0, s>>>(n, state, E0, flag);
        g_launches += 2 * k + 3;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (!*hflag) break;
    }
    dfree(M0, s);
    dfree(M1, s);
    dfree(E0, s);
    dfree(E1, s);
    int* root = dalloc<int>((size_t)n + 1, s);
    int* root2 = dalloc<int>((size_t)n + 1, s);
    int* isl = dalloc<int>((size_t)n + 1, s);
    int* id = dalloc<int>((size_t)n + 1, s);
    CK(cudaMemsetAsync(isl + n, 0, sizeof(int), s));
    k_mis_root0<<<g, kBlock, 0, s>>>(n, state, root, isl);
    for (int d = 1; d <= k; ++d) {
        k_mis_grow<<<g, kBlock, 0, s>>>(n, G.rp, G.ci, root, root2, misalt);
        std::swap(root, root2);
    }
    *nc = (int)exclusive_scan_total(isl, id, n, s);
    CK(cudaMemsetAsync(flag + 1, 0, sizeof(int), s));
    k_mis_assign<<<g, kBlock, 0, s>>>(n, root, id, agg, flag + 1);
    g_launches += k + 2;
    CK(cudaGetLastError());
    const int bad = read_scalar(flag + 1, s);
    dfree(root, s);
    dfree(root2, s);
    dfree(isl, s);
    dfree(id, s);
    dfree(state, s);
    dfree(flag, s);
    *rounds = r;
    if (bad) throw Error(-7, "MIS-k growth left a vertex unassigned");
    return 0;
}

// ------------------------------------------------------------------ segmented reductions
// keys for every stored entry of a CSR: (agg(i) << b) | agg(j); `drop` => self entries get the
// sentinel (all ones in the low 2b bits) which sorts last.
__global__ void k_pair_keys(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                            const int* __restrict__ agg, const int* __restrict__ cmap, int b, bool drop,
                            uint64_t* __restrict__ keys, int* __restrict__ idx) {
    const uint64_t sentinel = (b >= 32) ? ~0ULL : ((1ULL << (2 * b)) - 1ULL);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t I = (uint64_t)agg[i];
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            const uint64_t J = (uint64_t)cmap[ci[p]];
            keys[p] = (drop && I == J) ? sentinel : ((I << b) | J);
            idx[p] = p;
        }
    }
}

__global__ void k_heads(int64_t m, const uint64_t* __restrict__ keys, uint64_t sentinel, bool drop, int* head) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[t];
        head[t] = (t == 0 || k != keys[t - 1]) && !(drop && k == sentinel);
    }
}

__global__ void k_seg_start(int64_t m, const int* __restrict__ head, const int* __restrict__ pos,
                            int* __restrict__ start) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
        if (head[t]) start[pos[t]] = (int)t;
}

// per segment: coarse column and the sequential sum of the segment's values
template <class VAL>
__global__ void k_seg_sum(int S, const int* __restrict__ start, int64_t m_valid, const uint64_t* __restrict__ keys,
                          const int* __restrict__ idx, const VAL* __restrict__ src, int b, int* __restrict__ ocol,
                          int* __restrict__ orow, VAL* __restrict__ oval) {
    const uint64_t mask = (1ULL << b) - 1ULL;
    for (int sg = blockIdx.x * blockDim.x + threadIdx.x; sg < S; sg += gridDim.x * blockDim.x) {
        const int t0 = start[sg];
        const int t1 = (sg + 1 < S) ? start[sg + 1] : (int)m_valid;
        VAL acc = src[idx[t0]];
        for (int t = t0 + 1; t < t1; ++t) acc += src[idx[t]];
        const uint64_t k = keys[t0];
        ocol[sg] = (int)(k & mask);
        orow[sg] = (int)(k >> b);
        oval[sg] = acc;
    }
}

__global__ void k_rowptr_from_rows(int nrows, int S, const int* __restrict__ orow, int* __restrict__ rp) {
    for (int I = blockIdx.x * blockDim.x + threadIdx.x; I <= nrows; I += gridDim.x * blockDim.x) {
        int lo = 0, hi = S;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (orow[mid] < I) lo = mid + 1; else hi = mid;
        }
        rp[I] = lo;
    }
}

__global__ void k_lower_bound_u64(int64_t m, const uint64_t* keys, uint64_t x, int* out) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < x) lo = mid + 1; else hi = mid;
    }
    *out = (int)lo;
}

// Quotient of a CSR under agg: returns (rp, ci, val) of the nc x nc result.  VAL = uint32
// multiplicities (pass graphs, drop self entries) or double values (Galerkin, keep all).
template <class VAL>
static void quotient_impl(int n, int64_t nnz, const int* rp, const int* ci, const VAL* src, const int* agg,
                          const int* cmap, int nc, int ncols, bool drop, int** orp, int** oci, VAL** oval,
                          int64_t* onnz, cudaStream_t s) {
    const int b = bits_for(std::max(nc, ncols));
    const uint64_t sentinel = (b >= 32) ? ~0ULL : ((1ULL << (2 * b)) - 1ULL);
    const int m = (int)nnz;
    uint64_t* k0 = dalloc<uint64_t>(m, s);
    uint64_t* k1 = dalloc<uint64_t>(m, s);
    int* i0 = dalloc<int>(m, s);
    int* i1 = dalloc<int>(m, s);
    k_pair_keys<<<grid_for(n), kBlock, 0, s>>>(n, rp, ci, agg, cmap, b, drop, k0, i0);
    ++g_launches;
    CK(cudaGetLastError());
    sort_pairs(k0, k1, i0, i1, m, 2 * b, s);  // stable: equal keys keep (row, position) order
    dfree(k0, s);
    dfree(i0, s);
    int* head = dalloc<int>((size_t)m + 1, s);
    int* pos = dalloc<int>((size_t)m + 1, s);
    CK(cudaMemsetAsync(head + m, 0, sizeof(int), s));
    k_heads<<<grid_for(m), kBlock, 0, s>>>(m, k1, sentinel, drop, head);
    ++g_launches;
    CK(cudaGetLastError());
    const int S = (int)exclusive_scan_total(head, pos, m, s);
    int* start = dalloc<int>((size_t)S + 1, s);
    k_seg_start<<<grid_for(m), kBlock, 0, s>>>(m, head, pos, start);
    ++g_launches;
    CK(cudaGetLastError());
    int64_t m_valid = m;  // number of non-sentinel sorted entries (sentinels sort last)
    dfree(head, s);
    dfree(pos, s);
    int* ocol = dalloc<int>((size_t)S + 8, s);
    int* orow = dalloc<int>((size_t)S + 1, s);
    VAL* ov = dalloc<VAL>((size_t)S + 8, s);
    CK(cudaMemsetAsync(ocol, 0, sizeof(int) * ((size_t)S + 8), s));
    CK(cudaMemsetAsync(ov, 0, sizeof(VAL) * ((size_t)S + 8), s));
    if (drop) {
        // m_valid = index of the first sentinel = number of non-sentinel keys
        int* cnt = dalloc<int>(1, s);
        k_lower_bound_u64<<<1, 1, 0, s>>>(m, k1, sentinel, cnt);
        ++g_launches;
        CK(cudaGetLastError());
        m_valid = read_scalar(cnt, s);
        dfree(cnt, s);
    }
    if (S > 0) {
        k_seg_sum<VAL><<<grid_for(S), kBlock, 0, s>>>(S, start, m_valid, k1, i1, src, b, ocol, orow, ov);
        ++g_launches;
        CK(cudaGetLastError());
    }
    int* nrp = dalloc<int>((size_t)nc + 1, s);
    k_rowptr_from_rows<<<grid_for(nc + 1), kBlock, 0, s>>>(nc, S, orow, nrp);
    ++g_launches;
    CK(cudaGetLastError());
    dfree(orow, s);
    dfree(start, s);
    dfree(k1, s);
    dfree(i1, s);
    *orp = nrp;
    *oci = ocol;
    *oval = ov;
    *onnz = S;
}

// ------------------------------------------------------------------ row-merge quotient / Galerkin
void aggregate_order(int n, const int* agg, int nc, int* perm, int* aptr, cudaStream_t s);
void aggregate_order_counting(int n, const int* agg, int nc, int* perm, int* aptr, bool sorted, cudaStream_t s);
// Coarse row I is the merge of its members' rows (members = perm[aptr[I] .. aptr[I+1]), increasing
// vertex order).  Two steps:
//  1. staging: every fine row's entries, mapped (J = agg(col), value), are copied in perm order into
//     one array, so coarse row I's E entries are the contiguous segment [S[aptr[I]], S[aptr[I+1]])
//     in (member, CSR position) order -- the order k of the sequential definition;
//  2. merge: each segment is reduced to its distinct J in place, by a kernel chosen by the row's
//     size class (sub-warp shuffle/match merges, a warp bitonic or hash merge, one CTA for the
//     widest).  Every run of equal J is summed sequentially in k order, so fp64 Galerkin values
//     are bit-exact with the definition; fp64 rows come out sorted by J.  Pass-graph rows (uint32
//     weights, integer sums) may come out in first-occurrence order: the matching is order free.
// Rows with E > kRMB make the level fall back to the radix-sort path.
constexpr int kRM = 256;          // entries per warp buffer
constexpr int kRMWarps = 8;       // warps per block
constexpr int kRMB = 4096;        // entries per CTA buffer (widest rows)
constexpr int kRMClasses = 5;     // E <= 8 | <= 16 | <= 32 | <= kRM | <= kRMB

// lenp[t] = row length of fine vertex perm[t]
__global__ void k_stage_len(int n, const int* __restrict__ rp, const int* __restrict__ perm, int* __restrict__ lenp) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int v = perm[t];
        lenp[t] = rp[v + 1] - rp[v];
    }
}

// One warp per 32 consecutive t: their entries are the contiguous range [S[t0], S[t0 + 32]); lane
// writes position e (coalesced), its row found by a shuffle binary search over the 32 S values.
template <class VAL>
__global__ void k_stage_fill(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                             const VAL* __restrict__ src, const int* __restrict__ agg, const int* __restrict__ perm,
                             const int* __restrict__ S, unsigned* __restrict__ stJ, VAL* __restrict__ stv) {
    const int lane = threadIdx.x & 31;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int t0 = wid * 32; t0 < n; t0 += nw * 32) {
        const int t = t0 + lane;
        const int st = t < n ? S[t] : S[n];
        const int p0 = t < n ? rp[perm[t]] : 0;
        const int sb = __shfl_sync(0xffffffffu, st, 0);
        const int se = S[min(t0 + 32, n)];
        const int nr = min(32, n - t0);
        for (int eb = sb; eb < se; eb += 32) {  // warp-uniform bounds: every lane shuffles
            const int e = eb + lane;
            int m = 0;
#pragma unroll
            for (int w = 16; w > 0; w >>= 1) {
                const int sm = __shfl_sync(0xffffffffu, st, (m + w) & 31);
                if (m + w < nr && sm <= e) m += w;
            }
            const int ps = __shfl_sync(0xffffffffu, p0, m) + (e - __shfl_sync(0xffffffffu, st, m));
            if (e < se) {
                stJ[e] = (unsigned)agg[ci[ps]];
                stv[e] = src[ps];
            }
        }
    }
}

// eoff[I] = segment start, E = its length; rows sorted into size classes by warp-aggregated appends
// to lists[c * nc ..] (a row's output position comes from eoff, so the list order changes nothing)
__device__ __forceinline__ int rm_class(int e) { return e <= 8 ? 0 : e <= 16 ? 1 : e <= 32 ? 2 : e <= kRM ? 3 : 4; }

__global__ void __launch_bounds__(256) k_rm_classify(int nc, int n, const int* __restrict__ aptr,
                                                     const int* __restrict__ S, int* __restrict__ eoff,
                                                     int* __restrict__ emax, int* __restrict__ lists,
                                                     int* __restrict__ counts) {
    // one tile of 256 rows per iteration; per-class offsets: warp ballots -> block prefix in shared
    // memory -> one global atomic per class per tile (a global atomic per warp serialised)
    __shared__ int wc[8][kRMClasses];
    __shared__ int gb[kRMClasses];
    int mx = 0;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int tile = blockIdx.x; tile * 256 < nc; tile += gridDim.x) {
        const int I = tile * 256 + threadIdx.x;
        int c = -1;
        if (I < nc) {
            const int e0 = S[aptr[I]], e = S[aptr[I + 1]] - e0;
            eoff[I] = e0;
            if (I == nc - 1) eoff[nc] = S[n];
            mx = max(mx, e);
            c = e > kRMB ? -1 : rm_class(e);
        }
        unsigned mk[kRMClasses];
#pragma unroll
        for (int k = 0; k < kRMClasses; ++k) {
            mk[k] = __ballot_sync(0xffffffffu, c == k);
            if (lane == 0) wc[wib][k] = __popc(mk[k]);
        }
        __syncthreads();
        if (threadIdx.x < kRMClasses) {
            const int k = threadIdx.x;
            int acc = 0;
            for (int w = 0; w < 8; ++w) { const int t = wc[w][k]; wc[w][k] = acc; acc += t; }
            gb[k] = acc ? atomicAdd(counts + k, acc) : 0;
        }
        __syncthreads();
        if (c >= 0) {
            unsigned m = 0;
#pragma unroll
            for (int k = 0; k < kRMClasses; ++k) if (c == k) m = mk[k];
            lists[(size_t)c * nc + gb[c] + wc[wib][c] + __popc(m & ((1u << lane) - 1u))] = I;
        }
        __syncthreads();
    }
    mx = warp_max_i(mx);
    if (lane == 0) atomicMax(emax, mx);
}

// Class kernels.  In place: a row's segment [eoff[I], eoff[I+1]) is read whole before its distinct
// entries are written to its first U slots; uc[I] = U.  `drop`: J == I (a self loop) is skipped.

// E <= G, G lanes per row: lane t holds entry k = t.  An entry heads its run if no earlier entry has
// the same J (found with __match_any_sync on (row slot, J)); the head sums its run in increasing k.
// SORTED: output slot = number of heads with a smaller J (fp64 levels); else the number of heads
// before it (first-occurrence order, pass graphs).
template <class VAL, int G, bool SORTED>
__global__ void __launch_bounds__(256) k_rm_small(int nl, const int* __restrict__ list, const int* __restrict__ eoff,
                                                  bool drop, unsigned* __restrict__ stJ, VAL* __restrict__ stv,
                                                  int* __restrict__ ucount) {
    __shared__ VAL sv[256];
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31, t = lane & (G - 1), gi = lane / G;
    const unsigned NONE = 0xFFFFFFFFu;
    const unsigned gm = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gi * G));
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    VAL* ws = sv + (threadIdx.x & ~31);
    // list == nullptr: the class holds most rows, so walk all nl = nc rows in order (coalesced eoff,
    // no list indirection) and skip the rows of other classes
    const int elo = G == 8 ? -1 : G / 2;
    for (int base = wid * GPW; base < nl; base += nw * GPW) {  // uniform trip count per warp
        const int idx = base + gi;
        bool mine = idx < nl;
        const int I = mine ? (list ? list[idx] : idx) : 0;
        const int e0 = mine ? eoff[I] : 0;
        int E = mine ? eoff[I + 1] - e0 : 0;
        if (!list && (E <= elo || E > G)) {
            mine = false;
            E = 0;
        }
        unsigned J = NONE;
        VAL v = VAL(0);
        if (t < E) {
            const unsigned j = stJ[e0 + t];
            v = stv[e0 + t];
            J = (drop && j == (unsigned)I) ? NONE : j;
        }
        ws[lane] = v;
        const unsigned long long key = ((unsigned long long)gi << 32) | J;
        const unsigned grp = __match_any_sync(0xffffffffu, key);
        const bool head = J != NONE && __ffs(grp) - 1 == lane;
        const unsigned hb = __ballot_sync(0xffffffffu, head) & gm;
        __syncwarp();
        VAL acc = v;
        if (head)
            for (unsigned b = grp & (grp - 1); b; b &= b - 1) acc += ws[__ffs(b) - 1];
        int slot;
        if constexpr (SORTED) {
            slot = 0;
#pragma unroll
            for (int r = 0; r < G; ++r) {
                const unsigned Jr = __shfl_sync(0xffffffffu, J, r, G);
                if (((hb >> (gi * G + r)) & 1u) && Jr < J) ++slot;
            }
        } else {
            slot = __popc(hb & ((1u << lane) - 1u));
        }
        if (head) {
            stJ[e0 + slot] = J;
            stv[e0 + slot] = acc;
        }
        if (mine && t == 0) ucount[I] = __popc(hb);
        __syncwarp();
    }
}

// Pass-graph rows of E <= K, one thread each (registers only: the warp versions above are bound by
// the shuffle/match pipe at these sizes).  First-occurrence order, integer sums.  list == nullptr:
// all nl = nc rows in order, rows of other classes skipped.
template <int K>
__global__ void __launch_bounds__(256) k_qg_thread(int nl, const int* __restrict__ list, const int* __restrict__ eoff,
                                                   unsigned* __restrict__ stJ, uint32_t* __restrict__ stv,
                                                   int* __restrict__ ucount) {
    const unsigned NONE = 0xFFFFFFFFu;
    const int elo = K == 8 ? -1 : K / 2;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nl; idx += gridDim.x * blockDim.x) {
        const int I = list ? list[idx] : idx;
        const int e0 = eoff[I], E = eoff[I + 1] - e0;
        if (!list && (E <= elo || E > K)) continue;
        unsigned J[K];
        uint32_t w[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            J[k] = NONE;
            w[k] = 0;
            if (k < E) {
                const unsigned j = stJ[e0 + k];
                w[k] = stv[e0 + k];
                J[k] = j == (unsigned)I ? NONE : j;
            }
        }
        int u = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            bool head = J[k] != NONE;
            uint32_t acc = w[k];
#pragma unroll
            for (int r = 0; r < K; ++r) {
                if (r < k && J[r] == J[k]) head = false;
                if (r > k && J[r] == J[k]) acc += w[r];
            }
            if (head) {
                stJ[e0 + u] = J[k];
                stv[e0 + u] = acc;
                ++u;
            }
        }
        ucount[I] = u;
    }
}

// kRM-entry rows, one warp each: keys (J, k) bitonic-sorted in shared memory, runs of equal J
// summed in k order (sorted output)
template <class VAL>
__global__ void __launch_bounds__(32 * kRMWarps) k_rm_merge(int nl, const int* __restrict__ list,
                                                            const int* __restrict__ eoff, bool drop,
                                                            unsigned* __restrict__ stJ, VAL* __restrict__ stv,
                                                            int* __restrict__ ucount) {
    __shared__ unsigned long long skey[kRMWarps][kRM];
    __shared__ VAL sval[kRMWarps][kRM];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned long long* key = skey[wib];
    VAL* val = sval[wib];
    const int nwarp = gridDim.x * kRMWarps;
    for (int r = blockIdx.x * kRMWarps + wib; r < nl; r += nwarp) {
        const int I = list[r];
        const int e0 = eoff[I], E = eoff[I + 1] - e0;
        for (int q = lane; q < E; q += 32) {
            const unsigned J = stJ[e0 + q];
            const unsigned long long hi = (drop && J == (unsigned)I) ? 0xFFFFFFFFull : (unsigned long long)J;
            key[q] = (hi << 32) | (unsigned)q;
            val[q] = stv[e0 + q];
        }
        int P = 1;
        while (P < E) P <<= 1;
        for (int q = E + lane; q < P; q += 32) key[q] = ~0ull;
        __syncwarp();
        for (int size = 2; size <= P; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int q = lane; q < P; q += 32) {
                    const int partner = q ^ stride;
                    if (partner > q) {
                        const bool up = (q & size) == 0;
                        const unsigned long long a = key[q], b = key[partner];
                        if ((a > b) == up) { key[q] = b; key[partner] = a; }
                    }
                }
                __syncwarp();
            }
        }
        int base = 0;
        for (int q0 = 0; q0 < E; q0 += 32) {
            const int q = q0 + lane;
            bool head = false;
            unsigned J = 0xFFFFFFFFu;
            if (q < E) {
                J = (unsigned)(key[q] >> 32);
                head = J != 0xFFFFFFFFu && (q == 0 || (unsigned)(key[q - 1] >> 32) != J);
            }
            const unsigned hm = __ballot_sync(0xffffffffu, head);
            if (head) {
                const int slot = e0 + base + __popc(hm & ((1u << lane) - 1));
                VAL acc = val[(unsigned)(key[q] & 0xFFFFFFFFull)];
                for (int r2 = q + 1; r2 < E && (unsigned)(key[r2] >> 32) == J; ++r2)
                    acc += val[(unsigned)(key[r2] & 0xFFFFFFFFull)];
                stJ[slot] = J;
                stv[slot] = acc;
            }
            base += __popc(hm);
        }
        if (lane == 0) ucount[I] = base;
        __syncwarp();
    }
}

// Sort-free warp merge for E <= kRM, in two sweeps.  (1) The row's entries are staged in shared
// memory in k order while the distinct J are collected: __match_any_sync groups a 32-entry chunk's
// equal J and the group's first lane inserts J into a per-warp hash set (open addressing, 2 kRM
// slots), appending it to the distinct list when new.  (2) The U distinct J are ranked by counting
// (sorted output); lane u then owns the u-th one and walks all E staged entries in k order, adding
// those equal to it -- every sum in the sequential order (the first entry initialises it, so -0.0
// survives), and the walk is warp-uniform: no per-group serial loops.
constexpr int kRHWarps = 8;
constexpr int kRHSlots = 2 * kRM;
template <class VAL>
struct alignas(16) RhEnt {  // one staged entry: a single 16-byte (8-byte for uint32) shared load
    VAL v;
    unsigned J;
};
template <class VAL>
struct RhWarp {
    RhEnt<VAL> se[kRM];
    unsigned hk[kRHSlots];
    unsigned lj[kRM];
    short ls[kRM];
    int cnt;
};

template <class VAL>
__global__ void __launch_bounds__(32 * kRHWarps) k_rm_hash(int nl, const int* __restrict__ list,
                                                           const int* __restrict__ eoff, bool drop,
                                                           unsigned* __restrict__ stJ, VAL* __restrict__ stv,
                                                           int* __restrict__ ucount) {
    extern __shared__ __align__(16) unsigned char rh_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    RhWarp<VAL>& W = reinterpret_cast<RhWarp<VAL>*>(rh_raw)[wib];
    const unsigned NONE = 0xFFFFFFFFu;
    for (int q = lane; q < kRHSlots; q += 32) W.hk[q] = NONE;
    if (lane == 0) W.cnt = 0;
    __syncwarp();
    const int nwarp = gridDim.x * kRHWarps;
    for (int r = blockIdx.x * kRHWarps + wib; r < nl; r += nwarp) {
        const int I = list[r];
        const int e0 = eoff[I], E = eoff[I + 1] - e0;
        for (int c = 0; c < E; c += 32) {
            const int k = c + lane;
            unsigned J = NONE;
            if (k < E) {
                const unsigned j = stJ[e0 + k];
                J = (drop && j == (unsigned)I) ? NONE : j;
                W.se[k].J = J;
                W.se[k].v = stv[e0 + k];
            }
            const unsigned grp = __match_any_sync(0xffffffffu, J);
            if (J != NONE && __ffs(grp) - 1 == lane) {
                unsigned h = (J * 2654435761u) >> (32 - 9);
                for (;;) {
                    const unsigned old = atomicCAS(&W.hk[h], NONE, J);
                    if (old == NONE) {
                        const int u = atomicAdd(&W.cnt, 1);
                        W.lj[u] = J;
                        W.ls[u] = (short)h;
                        break;
                    }
                    if (old == J) break;
                    h = (h + 1) & (kRHSlots - 1);
                }
            }
        }
        __syncwarp();
        const int U = W.cnt;
        for (int ub = 0; ub < U; ub += 32) {
            const int u = ub + lane;
            const unsigned Ju = u < U ? W.lj[u] : NONE;
            int rank = 0;
            for (int q = 0; q < U; ++q) rank += W.lj[q] < Ju;
            // -0.0 + v == v exactly for every v, so starting from -0.0 the first term initialises the
            // sum and the additions are those of the sequential definition
            VAL acc = std::is_same<VAL, double>::value ? VAL(-0.0) : VAL(0);
#pragma unroll 4
            for (int k = 0; k < E; ++k) {
                const RhEnt<VAL> e = W.se[k];
                if (e.J == Ju) acc += e.v;
            }
            if (u < U) {
                stJ[e0 + rank] = Ju;
                stv[e0 + rank] = acc;
                W.hk[W.ls[u]] = NONE;
            }
        }
        if (lane == 0) {
            ucount[I] = U;
            W.cnt = 0;
        }
        __syncwarp();
    }
}

// the widest rows (kRM < E <= kRMB), one 256-thread CTA each: the bitonic merge in dynamic shared
// memory
template <class VAL>
__global__ void __launch_bounds__(256) k_rm_merge_block(int nl, const int* __restrict__ list,
                                                        const int* __restrict__ eoff, bool drop,
                                                        unsigned* __restrict__ stJ, VAL* __restrict__ stv,
                                                        int* __restrict__ ucount) {
    extern __shared__ __align__(16) unsigned char rmb_raw[];
    unsigned long long* key = reinterpret_cast<unsigned long long*>(rmb_raw);
    VAL* val = reinterpret_cast<VAL*>(key + kRMB);
    __shared__ int wsum[9];
    for (int wi = blockIdx.x; wi < nl; wi += gridDim.x) {
        const int I = list[wi];
        const int e0 = eoff[I], E = eoff[I + 1] - e0;
        for (int q = threadIdx.x; q < E; q += blockDim.x) {
            const unsigned J = stJ[e0 + q];
            const unsigned long long hi = (drop && J == (unsigned)I) ? 0xFFFFFFFFull : (unsigned long long)J;
            key[q] = (hi << 32) | (unsigned)q;
            val[q] = stv[e0 + q];
        }
        int P = 1;
        while (P < E) P <<= 1;
        for (int q = E + threadIdx.x; q < P; q += blockDim.x) key[q] = ~0ull;
        __syncthreads();
        for (int size = 2; size <= P; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int q = threadIdx.x; q < P; q += blockDim.x) {
                    const int partner = q ^ stride;
                    if (partner > q) {
                        const bool up = (q & size) == 0;
                        const unsigned long long a = key[q], b = key[partner];
                        if ((a > b) == up) { key[q] = b; key[partner] = a; }
                    }
                }
                __syncthreads();
            }
        int base = 0;
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        for (int q0 = 0; q0 < E; q0 += blockDim.x) {
            const int q = q0 + threadIdx.x;
            bool head = false;
            unsigned J = 0xFFFFFFFFu;
            if (q < E) {
                J = (unsigned)(key[q] >> 32);
                head = J != 0xFFFFFFFFu && (q == 0 || (unsigned)(key[q - 1] >> 32) != J);
            }
            const unsigned hm = __ballot_sync(0xffffffffu, head);
            if (lane == 0) wsum[wid] = __popc(hm);
            __syncthreads();
            if (threadIdx.x == 0) {
                int acc = 0;
                for (int w = 0; w < 8; ++w) { int t = wsum[w]; wsum[w] = acc; acc += t; }
                wsum[8] = acc;
            }
            __syncthreads();
            if (head) {
                const int slot = e0 + base + wsum[wid] + __popc(hm & ((1u << lane) - 1));
                VAL acc = val[(unsigned)(key[q] & 0xFFFFFFFFull)];
                for (int r = q + 1; r < E && (unsigned)(key[r] >> 32) == J; ++r) acc += val[(unsigned)(key[r] & 0xFFFFFFFFull)];
                stJ[slot] = J;
                stv[slot] = acc;
            }
            base += wsum[8];
            __syncthreads();
        }
        if (threadIdx.x == 0) ucount[I] = base;
        __syncthreads();
    }
}

template <class VAL>
__global__ void k_rm_compact(int nc, const int* __restrict__ eoff, const int* __restrict__ orp,
                             const unsigned* __restrict__ tcol, const VAL* __restrict__ tval, int* __restrict__ ocol,
                             VAL* __restrict__ oval) {
    for (int I = blockIdx.x * blockDim.x + threadIdx.x; I < nc; I += gridDim.x * blockDim.x) {
        const int src = eoff[I], dst = orp[I], u = orp[I + 1] - orp[I];
        for (int r = 0; r < u; ++r) {
            ocol[dst + r] = (int)tcol[src + r];
            oval[dst + r] = tval[src + r];
        }
    }
}

// returns false (nothing allocated) if some coarse row has more than kRMB entries
template <class VAL>
static bool quotient_rowmerge(int n, int64_t nnz, const int* rp, const int* ci, const VAL* src, const int* agg, int nc,
                              bool drop, const int* perm, const int* aptr, int** orp, int** oci, VAL** oval,
                              int64_t* onnz, cudaStream_t s) {
    // 1. staging offsets S (perm order) and the staged entries
    int* S = dalloc<int>((size_t)n + 1, s);
    {
        int* lenp = dalloc<int>((size_t)n + 1, s);
        CK(cudaMemsetAsync(lenp + n, 0, sizeof(int), s));
        k_stage_len<<<grid_for(n), kBlock, 0, s>>>(n, rp, perm, lenp);
        ++g_launches;
        exclusive_scan(lenp, S, n, s);  // S[n] = nnz: no read back
        dfree(lenp, s);
    }
    int* cnt = dalloc<int>(8, s);  // emax, counts[5]
    int* lists = dalloc<int>((size_t)kRMClasses * nc + 1, s);
    int* eoff = dalloc<int>((size_t)nc + 1, s);
    CK(cudaMemsetAsync(cnt, 0, 8 * sizeof(int), s));
    k_rm_classify<<<std::max(1, std::min((nc + 255) / 256, 148 * 8)), 256, 0, s>>>(nc, n, aptr, S, eoff, cnt, lists, cnt + 1);
    ++g_launches;
    CK(cudaGetLastError());
    int* hc = static_cast<int*>(pinned_scratch()) + 40;
    CK(cudaMemcpyAsync(hc, cnt, 6 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int mx = hc[0];
    int ncl[kRMClasses];
    for (int k = 0; k < kRMClasses; ++k) ncl[k] = hc[1 + k];
    dfree(cnt, s);
    if (mx > kRMB) {
        dfree(S, s);
        dfree(lists, s);
        dfree(eoff, s);
        return false;
    }
    const int64_t tot = nnz;  // = S[n] = eoff[nc]: every stored entry is staged once
    unsigned* stJ = dalloc<unsigned>((size_t)tot + 8, s);
    VAL* stv = dalloc<VAL>((size_t)tot + 8, s);
    {
        const int g = std::max(1, std::min((n + 255) / 256, 148 * 16));
        k_stage_fill<VAL><<<g, 256, 0, s>>>(n, rp, ci, src, agg, perm, S, stJ, stv);
        ++g_launches;
        CK(cudaGetLastError());
    }
    dfree(S, s);
    auto L = [&](int k) { return lists + (size_t)k * nc; };
    int* uc = dalloc<int>((size_t)nc + 1, s);
    CK(cudaMemsetAsync(uc + nc, 0, sizeof(int), s));
    auto grid_rows = [](int nrows, int rows_per_block, int cap) {
        return (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)nrows + rows_per_block - 1) / rows_per_block, cap));
    };
    // 2. class kernels.  Pass graphs: unsorted sub-warp merges up to 32 entries.  fp64: sorted
    // sub-warp merge up to 8, the bitonic warp merge up to 32 (AMG_RM_SPLIT=8|16 moves the rows
    // above it to the hash merge); the hash warp merge up to kRM; one CTA above.
    static int split = -1;
    if (split < 0) split = getenv("AMG_RM_SPLIT") ? atoi(getenv("AMG_RM_SPLIT")) : 32;
    bool pass_graph = false;
    if constexpr (std::is_same<VAL, uint32_t>::value) pass_graph = drop;
    int hash_from = 3;
    // a class with more than half the rows walks all rows in order (list == nullptr)
    auto LL = [&](int k, int* nrows) -> const int* {
        if (2 * (int64_t)ncl[k] > nc) { *nrows = nc; return nullptr; }
        *nrows = ncl[k];
        return L(k);
    };
    if (pass_graph) {
        int nr;
        const int* l;
        static int qthr = -1;
        if (qthr < 0) qthr = getenv("AMG_QG_WARP") ? 0 : 1;
        if (qthr) {
            if constexpr (std::is_same<VAL, uint32_t>::value) {
                if (ncl[0]) { l = LL(0, &nr); k_qg_thread<8><<<grid_rows(nr, 256, 148 * 16), 256, 0, s>>>(nr, l, eoff, stJ, stv, uc); }
                if (ncl[1]) { l = LL(1, &nr); k_qg_thread<16><<<grid_rows(nr, 256, 148 * 16), 256, 0, s>>>(nr, l, eoff, stJ, stv, uc); }
            }
        } else {
            if (ncl[0]) { l = LL(0, &nr); k_rm_small<VAL, 8, false><<<grid_rows(nr, 32, 148 * 32), 256, 0, s>>>(nr, l, eoff, drop, stJ, stv, uc); }
            if (ncl[1]) { l = LL(1, &nr); k_rm_small<VAL, 16, false><<<grid_rows(nr, 16, 148 * 32), 256, 0, s>>>(nr, l, eoff, drop, stJ, stv, uc); }
        }
        if (ncl[2]) { l = LL(2, &nr); k_rm_small<VAL, 32, false><<<grid_rows(nr, 8, 148 * 32), 256, 0, s>>>(nr, l, eoff, drop, stJ, stv, uc); }
        g_launches += 3;
    } else {
        if (split <= 16) hash_from = 2;
        if (split <= 8) hash_from = 1;
        if (ncl[0]) {
            int nr;
            const int* l = LL(0, &nr);
            k_rm_small<VAL, 8, true><<<grid_rows(nr, 32, 148 * 32), 256, 0, s>>>(nr, l, eoff, drop, stJ, stv, uc);
        }
        ++g_launches;
        for (int k = 1; k < hash_from; ++k)
            if (ncl[k]) {
                k_rm_merge<VAL><<<grid_rows(ncl[k], kRMWarps, 148 * 16), 32 * kRMWarps, 0, s>>>(ncl[k], L(k), eoff, drop,
                                                                                                 stJ, stv, uc);
                ++g_launches;
            }
    }
    CK(cudaGetLastError());
    {
        const size_t sm = sizeof(RhWarp<VAL>) * kRHWarps;
        static bool cfg = false;
        if (!cfg) {
            CK(cudaFuncSetAttribute(k_rm_hash<VAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            cfg = true;
        }
        for (int k = hash_from; k <= 3; ++k)
            if (ncl[k]) {
                k_rm_hash<VAL><<<grid_rows(ncl[k], kRHWarps, 148 * 3), 32 * kRHWarps, sm, s>>>(ncl[k], L(k), eoff, drop,
                                                                                               stJ, stv, uc);
                ++g_launches;
            }
    }
    CK(cudaGetLastError());
    if (ncl[4]) {
        const size_t sm = (size_t)kRMB * (sizeof(unsigned long long) + sizeof(VAL));
        static bool cfg = false;
        if (!cfg) {
            CK(cudaFuncSetAttribute(k_rm_merge_block<VAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            cfg = true;
        }
        k_rm_merge_block<VAL><<<std::min(ncl[4], 148 * 2), 256, sm, s>>>(ncl[4], L(4), eoff, drop, stJ, stv, uc);
        ++g_launches;
        CK(cudaGetLastError());
    }
    dfree(lists, s);
    // 3. compact the merged segments into the coarse CSR
    int* nrp = dalloc<int>((size_t)nc + 1, s);
    const int64_t Sn = exclusive_scan_total(uc, nrp, nc, s);
    int* ocol = dalloc<int>((size_t)Sn + 8, s);
    VAL* ov = dalloc<VAL>((size_t)Sn + 8, s);
    CK(cudaMemsetAsync(ocol + Sn, 0, 8 * sizeof(int), s));
    CK(cudaMemsetAsync(ov + Sn, 0, 8 * sizeof(VAL), s));
    k_rm_compact<VAL><<<grid_for(nc), kBlock, 0, s>>>(nc, eoff, nrp, stJ, stv, ocol, ov);
    ++g_launches;
    CK(cudaGetLastError());
    dfree(stJ, s);
    dfree(stv, s);
    dfree(eoff, s);
    dfree(uc, s);
    *orp = nrp;
    *oci = ocol;
    *oval = ov;
    *onnz = Sn;
    return true;
}

PassGraph quotient_graph(const PassGraph& G, const int* agg_t, int nc, cudaStream_t s) {
    PassGraph H;
    H.n = nc;
    if (!getenv("AMG_RADIX_QUOTIENT")) {
        int* perm = dalloc<int>((size_t)G.n + 8, s);
        int* aptr = dalloc<int>((size_t)nc + 8, s);
        aggregate_order_counting(G.n, agg_t, nc, perm, aptr, false, s);  // pass graphs: any member order
        const bool ok = quotient_rowmerge<uint32_t>(G.n, G.nnz, G.rp, G.ci, G.w, agg_t, nc, true, perm, aptr, &H.rp,
                                                    &H.ci, &H.w, &H.nnz, s);
        dfree(perm, s);
        dfree(aptr, s);
        if (ok) return H;
    }
    quotient_impl<uint32_t>(G.n, G.nnz, G.rp, G.ci, G.w, agg_t, agg_t, nc, nc, true, &H.rp, &H.ci, &H.w, &H.nnz, s);
    return H;
}

Csr galerkin(const Csr& A, const int* agg, const int* cmap, int nc, int ncols, const int* perm, const int* aptr,
             cudaStream_t s) {
    Csr H;
    H.n = nc;
    if (!cmap) cmap = agg;
    // the row merge reads the coarse column of every entry through `cmap` (rows come from perm/aptr)
    if (!getenv("AMG_RADIX_QUOTIENT") &&
        quotient_rowmerge<double>(A.n, A.nnz, A.rp, A.ci, A.v, cmap, nc, false, perm, aptr, &H.rp, &H.ci, &H.v, &H.nnz,
                                  s))
        return H;
    quotient_impl<double>(A.n, A.nnz, A.rp, A.ci, A.v, agg, cmap, nc, ncols, false, &H.rp, &H.ci, &H.v, &H.nnz, s);
    return H;
}

__global__ void k_compose(int n, int* __restrict__ agg, const int* __restrict__ agg_t) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) agg[i] = agg_t[agg[i]];
}

void compose(int n, int* agg, const int* agg_t, cudaStream_t s) {
    k_compose<<<grid_for(n), kBlock, 0, s>>>(n, agg, agg_t);
    ++g_launches;
    CK(cudaGetLastError());
}

__global__ void k_iota(int n, int* a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

// aptr[I] = first position of aggregate I in the sorted order: every id in [0, nc) has a member (its
// leader), so the heads of the sorted runs write every entry; aptr[nc] = n
__global__ void k_aptr(int nc, int n, const int* __restrict__ sorted_agg, int* __restrict__ aptr) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int a = sorted_agg[t];
        if (t == 0 || sorted_agg[t - 1] != a) aptr[a] = t;
        if (t == n - 1) aptr[nc] = n;
    }
}

// Counting-sort aggregate order: members counted per aggregate (atomics), aptr by a scan, members
// placed by atomic cursors, then (sorted) each aggregate's members sorted in increasing vertex order
// by one thread (insertion sort; heap sort for the rare aggregates of > 32 members).  sorted == false
// (the pass graphs, whose merges are order free) skips the last step.
__global__ void k_agg_count(int n, const int* __restrict__ agg, int* __restrict__ cnt) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) atomicAdd(cnt + agg[v], 1);
}

__global__ void k_agg_place(int n, const int* __restrict__ agg, const int* __restrict__ aptr, int* __restrict__ cur,
                            int* __restrict__ perm) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int I = agg[v];
        perm[aptr[I] + atomicAdd(cur + I, 1)] = v;
    }
}

__device__ void heap_sift(int* a, int i, int m) {
    for (;;) {
        int c = 2 * i + 1;
        if (c >= m) return;
        if (c + 1 < m && a[c + 1] > a[c]) ++c;
        if (a[i] >= a[c]) return;
        const int t = a[i]; a[i] = a[c]; a[c] = t;
        i = c;
    }
}

__global__ void k_agg_sortseg(int nc, const int* __restrict__ aptr, int* __restrict__ perm) {
    for (int I = blockIdx.x * blockDim.x + threadIdx.x; I < nc; I += gridDim.x * blockDim.x) {
        int* a = perm + aptr[I];
        const int m = aptr[I + 1] - aptr[I];
        if (m <= 32) {
            for (int k = 1; k < m; ++k) {
                const int x = a[k];
                int j = k - 1;
                while (j >= 0 && a[j] > x) { a[j + 1] = a[j]; --j; }
                a[j + 1] = x;
            }
        } else {
            for (int k = m / 2 - 1; k >= 0; --k) heap_sift(a, k, m);
            for (int e = m - 1; e > 0; --e) {
                const int t = a[0]; a[0] = a[e]; a[e] = t;
                heap_sift(a, 0, e);
            }
        }
    }
}

void aggregate_order_counting(int n, const int* agg, int nc, int* perm, int* aptr, bool sorted, cudaStream_t s) {
    int* cnt = dalloc<int>((size_t)nc + 1, s);
    CK(cudaMemsetAsync(cnt, 0, sizeof(int) * ((size_t)nc + 1), s));
    k_agg_count<<<grid_for(n), kBlock, 0, s>>>(n, agg, cnt);
    exclusive_scan(cnt, aptr, nc, s);  // aptr[nc] = n
    CK(cudaMemsetAsync(cnt, 0, sizeof(int) * (size_t)nc, s));
    k_agg_place<<<grid_for(n), kBlock, 0, s>>>(n, agg, aptr, cnt, perm);
    g_launches += 2;
    if (sorted) {
        k_agg_sortseg<<<grid_for(nc), kBlock, 0, s>>>(nc, aptr, perm);
        ++g_launches;
    }
    CK(cudaGetLastError());
    dfree(cnt, s);
}

void aggregate_order(int n, const int* agg, int nc, int* perm, int* aptr, cudaStream_t s) {
    // the level order (members sorted) stays on the radix sort: the counting version's per-aggregate
    // sort measured slower there (C3 setup 19.2 vs 20.0 ms); AMG_AGG_COUNTING=1 selects it
    static int radix = -1;
    if (radix < 0) radix = getenv("AMG_AGG_COUNTING") ? 0 : 1;
    if (!radix) {
        aggregate_order_counting(n, agg, nc, perm, aptr, true, s);
        return;
    }
    int* iota = dalloc<int>(n, s);
    int* sk = dalloc<int>(n, s);
    k_iota<<<grid_for(n), kBlock, 0, s>>>(n, iota);
    ++g_launches;
    CK(cudaGetLastError());
    sort_pairs(agg, sk, iota, perm, n, bits_for(nc), s);
    k_aptr<<<grid_for(n), kBlock, 0, s>>>(nc, n, sk, aptr);
    ++g_launches;
    CK(cudaGetLastError());
    dfree(iota, s);
    dfree(sk, s);
}

// ------------------------------------------------------------------ tiles
// Tile boundary at row r iff the bucket floor(rp[r]/H) changes, or r or r-1 is longer than H.
// Then every tile holds <= 2H - 1 entries, or is a single long row (long path if > 2H).
__global__ void k_tile_flags(int n, const int* __restrict__ rp, int H, int* __restrict__ flag) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        int f = (r == 0);
        if (r > 0) {
            const int a = rp[r - 1], b = rp[r], c = rp[r + 1];
            f = (a / H != b / H) || (c - b > H) || (b - a > H);
        }
        flag[r] = f;
    }
}

__global__ void k_tile_rows(int n, const int* __restrict__ flag, const int* __restrict__ pos, int* __restrict__ row,
                            int ntiles) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
        if (flag[r]) row[pos[r]] = r;
    if (blockIdx.x == 0 && threadIdx.x == 0) row[ntiles] = n;
}

int tiled_grid(int cap, int ntiles);  // k_solve.cu

Tiles build_tiles(const Csr& A, int grid_per_sm, cudaStream_t s) {
    (void)grid_per_sm;
    Tiles T;
    const double avg = A.n > 0 ? (double)A.nnz / (double)A.n : 1.0;
    int H = (int)std::ceil(256.0 * avg);
    H = (H + 3) & ~3;
    if (H < 256) H = 256;
    if (H > 2048) H = 2048;
    T.cap = 2 * H;
    int* flag = dalloc<int>((size_t)A.n + 1, s);
    int* pos = dalloc<int>((size_t)A.n + 1, s);
    CK(cudaMemsetAsync(flag + A.n, 0, sizeof(int), s));
    k_tile_flags<<<grid_for(A.n), kBlock, 0, s>>>(A.n, A.rp, H, flag);
    ++g_launches;
    CK(cudaGetLastError());
    T.ntiles = (int)exclusive_scan_total(flag, pos, A.n, s);
    T.row = dalloc<int>((size_t)T.ntiles + 1, s);
    k_tile_rows<<<grid_for(A.n), kBlock, 0, s>>>(A.n, flag, pos, T.row, T.ntiles);
    ++g_launches;
    CK(cudaGetLastError());
    dfree(flag, s);
    dfree(pos, s);
    T.grid = tiled_grid(T.cap, T.ntiles);
    return T;
}

// ------------------------------------------------------------------ SELL-32
__global__ void k_sell_width(int n, int nslices, const int* __restrict__ rp, int* __restrict__ width) {
    for (int sl = blockIdx.x * blockDim.x + threadIdx.x; sl < nslices; sl += gridDim.x * blockDim.x) {
        int w = 0;
        const int i1 = min(n, sl * 32 + 32);
        for (int i = sl * 32; i < i1; ++i) w = max(w, rp[i + 1] - rp[i]);
        width[sl] = w;
    }
}

__global__ void k_sell_fill(int n, int nslices, const int* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ v, const int* __restrict__ sptr, int* __restrict__ scol,
                            double* __restrict__ sval) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)nslices * 32;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int sl = (int)(t >> 5), lane = (int)(t & 31);
        const int i = sl * 32 + lane;
        const int w = sptr[sl + 1] - sptr[sl];
        const int64_t base = (int64_t)sptr[sl] * 32 + lane;
        const int p0 = i < n ? rp[i] : 0;
        const int len = i < n ? rp[i + 1] - p0 : 0;
        for (int j = 0; j < w; ++j) {
            const bool real = j < len;
            scol[base + (int64_t)j * 32] = real ? ci[p0 + j] : (i < n ? i : 0);
            sval[base + (int64_t)j * 32] = real ? v[p0 + j] : 0.0;
        }
    }
}

__global__ void k_max_int(int n, const int* __restrict__ a, int* out) {
    int m = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m = max(m, a[i]);
    m = warp_max_i(m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

Sell build_sell(const Csr& A, double max_pad_ratio, cudaStream_t s) {
    Sell S;
    S.n = A.n;
    S.chi = A.n - 1;  // raised by the caller on a level with an upper halo
    S.nslices = (A.n + 31) / 32;
    int* width = dalloc<int>((size_t)S.nslices + 1, s);
    CK(cudaMemsetAsync(width + S.nslices, 0, sizeof(int), s));
    k_sell_width<<<grid_for(S.nslices), kBlock, 0, s>>>(A.n, S.nslices, A.rp, width);
    CK(cudaGetLastError());
    ++g_launches;
    int* sptr = dalloc<int>((size_t)S.nslices + 1, s);
    const int64_t units = exclusive_scan_total(width, sptr, S.nslices, s);
    {
        int* wm = dalloc<int>(1, s);
        CK(cudaMemsetAsync(wm, 0, sizeof(int), s));
        k_max_int<<<grid_red(S.nslices), kBlock, 0, s>>>(S.nslices, width, wm);
        ++g_launches;
        CK(cudaGetLastError());
        S.wmax = read_scalar(wm, s);
        dfree(wm, s);
    }
    dfree(width, s);
    S.padded = units * 32;
    if ((double)S.padded > max_pad_ratio * (double)A.nnz + 64.0) {  // too irregular: keep CSR tiles
        dfree(sptr, s);
        return Sell{};
    }
    S.sptr = sptr;
    S.col = dalloc<int>((size_t)S.padded + 32, s);
    S.val = dalloc<double>((size_t)S.padded + 32, s);
    k_sell_fill<<<grid_for((int64_t)S.nslices * 32), kBlock, 0, s>>>(A.n, S.nslices, A.rp, A.ci, A.v, sptr, S.col,
                                                                      S.val);
    CK(cudaGetLastError());
    ++g_launches;
    return S;
}

// ------------------------------------------------------------------ lossless SELL compression
// Distinct fp64 values and distinct column offsets (col - row) of a level are collected with
// per-block shared-memory hash sets (warp-deduplicated with __match_any_sync) flushed into global
// hash sets; if <= 256 values (offsets) occur they become sorted dictionaries and each stored entry
// keeps only a 1-byte code (int16 offsets when the offsets fit but are too many).  The SpMV kernels
// expand codes through shared-memory copies of the dictionaries: bit-identical operands, 2-3 bytes
// per entry instead of 12.
constexpr int kGHT = 4096;  // global hash-set capacity (power of 2)
constexpr int kBHT = 1024;  // per-block hash-set capacity
constexpr unsigned long long kEmptyKey = 0xFFFFFFFFFFFFFFFFULL;

__device__ __forceinline__ uint32_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return (uint32_t)x;
}

// returns true on overflow (a full or crowded set: more than kMaxProbe probes)
constexpr int kMaxProbe = 32;
__device__ bool set_insert(unsigned long long* tab, int cap, unsigned long long key, int* count) {
    uint32_t h = mix64(key) & (uint32_t)(cap - 1);
    for (int probe = 0; probe < kMaxProbe; ++probe) {
        unsigned long long old = atomicCAS(&tab[h], kEmptyKey, key);
        if (old == kEmptyKey) {
            if (count) atomicAdd(count, 1);
            return false;
        }
        if (old == key) return false;
        h = (h + 1) & (uint32_t)(cap - 1);
    }
    return true;
}

__device__ __forceinline__ unsigned long long off_key(int off) { return (unsigned long long)(uint32_t)off; }

// warp per SELL slice: insert every stored entry's value bits and offset (padding included: 0.0
// and offset 0; lanes past n use offset 0) into the block sets, then flush into the global sets.
__global__ void __launch_bounds__(kBlock) k_distinct(Sell S, unsigned long long* gv, unsigned long long* gc,
                                                     int* counts, int* flags) {
    __shared__ unsigned long long bv[kBHT], bc[kBHT];
    __shared__ int bflag;
    for (int k = threadIdx.x; k < kBHT; k += blockDim.x) { bv[k] = kEmptyKey; bc[k] = kEmptyKey; }
    if (threadIdx.x == 0) bflag = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < S.nslices; sl += nw) {
        const int b = S.sptr[sl], w = S.sptr[sl + 1] - b;
        const int i = sl * 32 + lane;
        const int fl = *((volatile int*)&bflag);
        if (fl == 3) break;  // both sets overflowed: nothing left to learn
        for (int j = 0; j < w; ++j) {
            const size_t e = ((size_t)b + j) * 32 + lane;
            if (!(fl & 1)) {
                const unsigned long long vk = (unsigned long long)__double_as_longlong(S.val[e]);
                unsigned mv = __match_any_sync(0xffffffffu, vk);
                if (lane == __ffs(mv) - 1 && set_insert(bv, kBHT, vk, nullptr)) atomicOr(&bflag, 1);
            }
            if (!(fl & 2)) {
                const unsigned long long ck = off_key(i < S.n ? S.col[e] - i : 0);
                unsigned mc = __match_any_sync(0xffffffffu, ck);
                if (lane == __ffs(mc) - 1 && set_insert(bc, kBHT, ck, nullptr)) atomicOr(&bflag, 2);
            }
        }
    }
    __syncthreads();
    int f = bflag;
    for (int k = threadIdx.x; k < kBHT; k += blockDim.x) {
        if (!(f & 1) && bv[k] != kEmptyKey && set_insert(gv, kGHT, bv[k], counts + 0)) f |= 1;
        if (!(f & 2) && bc[k] != kEmptyKey && set_insert(gc, kGHT, bc[k], counts + 1)) f |= 2;
    }
    if (f) atomicOr(flags, f);
}

// one block: compact a global set and rank-sort it into a dictionary (values as doubles, offsets as int)
__global__ void k_dict_build(const unsigned long long* gv, const unsigned long long* gc, double* vdict, int* cdict,
                             int nvmax, int ncmax) {
    __shared__ unsigned long long kv[256], kc[256];
    __shared__ int nv, nc;
    if (threadIdx.x == 0) { nv = 0; nc = 0; }
    __syncthreads();
    for (int k = threadIdx.x; k < kGHT; k += blockDim.x) {
        if (gv[k] != kEmptyKey) { int t = atomicAdd(&nv, 1); if (t < 256) kv[t] = gv[k]; }
        if (gc[k] != kEmptyKey) { int t = atomicAdd(&nc, 1); if (t < 256) kc[t] = gc[k]; }
    }
    __syncthreads();
    if (threadIdx.x < nv && nv <= nvmax) {
        const double x = __longlong_as_double((long long)kv[threadIdx.x]);
        int r = 0;
        for (int k = 0; k < nv; ++k) {
            const double y = __longlong_as_double((long long)kv[k]);
            r += (y < x) || (y == x && kv[k] < kv[threadIdx.x]);  // total order (also splits +0 / -0)
        }
        vdict[r] = x;
    }
    if (threadIdx.x < nc && nc <= ncmax) {
        const int x = (int)(uint32_t)kc[threadIdx.x];
        int r = 0;
        for (int k = 0; k < nc; ++k) r += ((int)(uint32_t)kc[k] < x);
        cdict[r] = x;
    }
}

__global__ void __launch_bounds__(kBlock) k_sell_encode(Sell S, int vmode, int cmode, const double* __restrict__ vdict,
                                                        int nvd, const int* __restrict__ cdict, int ncd,
                                                        uint8_t* vcode, uint8_t* ccode, int16_t* coff,
                                                        uint16_t* pcode) {
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < S.nslices; sl += nw) {
        const int b = S.sptr[sl], w = S.sptr[sl + 1] - b;
        const int i = sl * 32 + lane;
        for (int j = 0; j < w; ++j) {
            const size_t e = ((size_t)b + j) * 32 + lane;
            int vc = 0;
            if (vmode == 1) {
                const double x = S.val[e];
                const unsigned long long xb = (unsigned long long)__double_as_longlong(x);
                for (int k = 0; k < nvd; ++k)  // <= 256 entries, exact bit match
                    if ((unsigned long long)__double_as_longlong(vdict[k]) == xb) { vc = k; break; }
                if (cmode != 3) vcode[e] = (uint8_t)vc;
            }
            const int off = i < S.n ? S.col[e] - i : 0;
            if (cmode == 1 || cmode == 3) {
                int lo = 0, hi = ncd;
                while (lo < hi) {
                    int mid = (lo + hi) >> 1;
                    if (cdict[mid] < off) lo = mid + 1; else hi = mid;
                }
                if (cmode == 1) ccode[e] = (uint8_t)lo;
                else pcode[e] = (uint16_t)(vc | (lo << 8));
            } else if (cmode == 2) {
                coff[e] = (int16_t)off;
            }
        }
    }
}

__global__ void k_pair_codes(int64_t m, const uint8_t* __restrict__ vc, const uint8_t* __restrict__ cc,
                             uint16_t* __restrict__ pc) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
        pc[e] = (uint16_t)(vc[e] | (cc[e] << 8));
}

__global__ void k_minmax_off(Sell S, int* mm) {
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    int mn = 0, mx = 0;
    for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < S.nslices; sl += nw) {
        const int b = S.sptr[sl], w = S.sptr[sl + 1] - b;
        const int i = sl * 32 + lane;
        if (i >= S.n) continue;
        for (int j = 0; j < w; ++j) {
            const int off = S.col[((size_t)b + j) * 32 + lane] - i;
            mn = min(mn, off);
            mx = max(mx, off);
        }
    }
    __syncwarp();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
        atomicMin(mm, mn);
        atomicMax(mm + 1, mx);
    }
}

void free_sell(Sell& S, cudaStream_t s) {
    dfree(S.sptr, s); dfree(S.col, s); dfree(S.val, s); dfree(S.vcode, s); dfree(S.ccode, s);
    dfree(S.coff, s); dfree(S.pcode, s); dfree(S.vdict, s); dfree(S.cdict, s);
    S = Sell{};
}

void compress_sell(Sell& S, const Csr& A, cudaStream_t s) {
    (void)A;
    // only levels large enough to be HBM-bound (smaller ones are L2-resident and latency-bound)
    if (!S.col || S.padded < (int64_t(1) << 22)) return;
    unsigned long long* gv = dalloc<unsigned long long>(kGHT, s);
    unsigned long long* gc = dalloc<unsigned long long>(kGHT, s);
    int* aux = dalloc<int>(8, s);  // counts[2], flags, minmax[2]
    CK(cudaMemsetAsync(gv, 0xff, sizeof(unsigned long long) * kGHT, s));
    CK(cudaMemsetAsync(gc, 0xff, sizeof(unsigned long long) * kGHT, s));
    CK(cudaMemsetAsync(aux, 0, sizeof(int) * 8, s));
    const int g = grid_red((int64_t)S.nslices * 32);
    k_distinct<<<g, kBlock, 0, s>>>(S, gv, gc, aux, aux + 2);
    ++g_launches;
    k_minmax_off<<<g, kBlock, 0, s>>>(S, aux + 3);
    ++g_launches;
    CK(cudaGetLastError());
    int* h = static_cast<int*>(pinned_scratch()) + 32;
    CK(cudaMemcpyAsync(h, aux, sizeof(int) * 5, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int nv = h[0], nc = h[1], fl = h[2], omin = h[3], omax = h[4];
    S.vmode = (!(fl & 1) && nv <= 256) ? 1 : 0;
    S.cmode = (!(fl & 2) && nc <= 256) ? 1 : ((omin >= -32768 && omax <= 32767) ? 2 : 0);
    if (S.vmode || S.cmode) {
        S.vdict = dalloc<double>(256, s);
        S.cdict = dalloc<int>(256, s);
        S.nvdict = S.vmode ? nv : 0;
        S.ncdict = S.cmode == 1 ? nc : 0;
        k_dict_build<<<1, 1024, 0, s>>>(gv, gc, S.vdict, S.cdict, S.vmode ? 256 : 0, S.cmode == 1 ? 256 : 0);
        S.ncdict = S.cmode == 1 ? nc : 0;
        ++g_launches;
        if (S.vmode == 1 && S.cmode == 1) S.cmode = 3;  // one 2-byte code pair load per entry
        if (S.vmode && S.cmode != 3) S.vcode = dalloc<uint8_t>((size_t)S.padded + 64, s);
        if (S.cmode == 1) S.ccode = dalloc<uint8_t>((size_t)S.padded + 64, s);
        if (S.cmode == 2) S.coff = dalloc<int16_t>((size_t)S.padded + 64, s);
        if (S.cmode == 3) S.pcode = dalloc<uint16_t>((size_t)S.padded + 64, s);
        k_sell_encode<<<g, kBlock, 0, s>>>(S, S.vmode, S.cmode, S.vdict, S.nvdict, S.cdict, S.ncdict, S.vcode,
                                           S.ccode, S.coff, S.pcode);
        ++g_launches;
        CK(cudaGetLastError());
        // the replaced full-width streams are no longer needed by the solve
        if (S.vmode) { dfree(S.val, s); S.val = nullptr; }
        if (S.cmode) { dfree(S.col, s); S.col = nullptr; }
    }
    dfree(gv, s);
    dfree(gc, s);
    dfree(aux, s);
}

// ------------------------------------------------------------------ coarsest (a7)
__global__ void k_densify(int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                          double shift_per_entry, double* __restrict__ M) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        for (int j = 0; j < n; ++j) M[(size_t)i * n + j] = shift_per_entry;
        for (int p = rp[i]; p < rp[i + 1]; ++p) M[(size_t)i * n + ci[p]] += v[p];
    }
}

// one Gauss-Jordan step k (in-place inverse of an SPD matrix, no pivoting): B' from B
__global__ void k_gj_step(int n, int k, const double* __restrict__ B, double* __restrict__ Bn) {
    const double piv = B[(size_t)k * n + k];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(e / n), j = (int)(e % n);
        double r;
        if (i == k && j == k) r = 1.0 / piv;
        else if (i == k) r = B[(size_t)k * n + j] / piv;
        else if (j == k) r = -B[(size_t)i * n + k] / piv;
        else r = B[e] - B[(size_t)i * n + k] * B[(size_t)k * n + j] / piv;
        Bn[e] = r;
    }
}

__global__ void k_add_const(int64_t m, double c, double* a) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
        a[e] += c;
}

double* coarse_inverse(const Csr& A, bool singular, double shift, cudaStream_t s) {
    const int n = A.n;
    const size_t m = (size_t)n * n;
    double* M0 = dalloc<double>(m, s);
    double* M1 = dalloc<double>(m, s);
    // singular: factor A + (s/n) 1 1^T; A^dagger = (A + s J)^{-1} - J/s, J = 1 1^T / n  (reading A16)
    k_densify<<<grid_for(n), kBlock, 0, s>>>(n, A.rp, A.ci, A.v, singular ? shift / (double)n : 0.0, M0);
    ++g_launches;
    CK(cudaGetLastError());
    for (int k = 0; k < n; ++k) {
        k_gj_step<<<grid_for((int64_t)m), kBlock, 0, s>>>(n, k, M0, M1);
        ++g_launches;
        std::swap(M0, M1);
    }
    CK(cudaGetLastError());
    if (singular) {
        k_add_const<<<grid_for((int64_t)m), kBlock, 0, s>>>((int64_t)m, -1.0 / (shift * (double)n), M0);
        ++g_launches;
        CK(cudaGetLastError());
    }
    dfree(M1, s);
    return M0;
}

}  // namespace amg
