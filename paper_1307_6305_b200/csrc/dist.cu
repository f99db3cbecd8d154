// dist.cu -- the row-partitioned (multi-GPU) path of libamg_b200.so: SURVEY.md 8(a) row a17 and 8(e).
//
// Partition.  Rank r owns the contiguous block [offs[r], offs[r+1]) of level-0 rows (the caller's
// blocks, in rank order).  Aggregation is DECOUPLED (reading A20): the matching passes of a
// row-partitioned level see only the edges inside the block, so every aggregate lies inside one
// block and level l+1's block r is exactly the aggregates of level l's block r (leader numbering
// preserves block order: coarse block offsets are the prefix sums of the per-rank aggregate
// counts).  Restriction and prolongation therefore stay local.  The matching keys hash GLOBAL
// vertex ids (docs/keys.md), so the aggregates equal those of the sequential definition with the
// same blocks (oracle/amg_oracle.c, nparts = P) bit for bit.
//
// Levels with n_l < gather_rows (and always the coarsest) are REPLICATED: the first such level g is
// allgathered once at setup, and every rank builds and runs the rest of the hierarchy redundantly on
// identical data (deterministic kernels => identical results, no broadcast).  In the solve, level
// g-1 restricts into its own block of level g's residual and the blocks are allgathered (C-gather);
// the prolongation reads the same block of the correction.
//
// Exchange steps per solve (C-halo, C-dot, C-gather of SURVEY 8(e)):
//   * halo: before every SpMV-class pass on a row-partitioned level, the rows other ranks reference
//     are packed (one gather kernel) and exchanged with grouped point-to-point messages straight into
//     the receivers' halo slots (each peer's halo is one contiguous run: blocks are contiguous);
//   * dots: every batch of FCG dot partials is allgathered (P x k doubles) and summed in rank order
//     by one tiny kernel, so every rank holds bit-identical scalars whatever the collective does;
//   * gather: the level-g residual blocks, by grouped point-to-point messages.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <vector>

#include "hierarchy.h"

namespace amg {

static int gridn(int64_t n) {
    int64_t g = (n + kBlock - 1) / kBlock;
    if (g < 1) g = 1;
    if (g > 148 * 16) g = 148 * 16;
    return (int)g;
}

// ------------------------------------------------------------------ kernels
// global column ids outside the own block [gbeg, gend) (halo candidates; duplicates allowed)
// (row ranges outside [0, nnz] set *bad = VF_RP (64) and are skipped; bad columns set VF_RANGE (1))
__global__ void k_halo_collect(int n, int64_t nnz, const int64_t* __restrict__ rp, const int* __restrict__ ci,
                               int64_t gbeg, int64_t gend, int64_t nglob, int* __restrict__ out, int* __restrict__ cnt,
                               int* __restrict__ bad) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int64_t p0 = rp[i], p1 = rp[i + 1];
        if (p0 < 0 || p1 < p0 || p1 > nnz || (i == 0 && p0 != 0) || (i == n - 1 && p1 != nnz)) {
            atomicOr(bad, 64);
            continue;
        }
        for (int64_t p = p0; p < p1; ++p) {
            const int c = ci[p];
            if (c < 0 || (int64_t)c >= nglob) { atomicOr(bad, 1); continue; }
            if ((int64_t)c < gbeg || (int64_t)c >= gend) out[atomicAdd(cnt, 1)] = c;
        }
    }
}

__device__ __forceinline__ int lower_bound_i(const int* a, int n, int x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// global column -> relative column (own: c - gbeg; halo: position in hid, below or above the block)
__global__ void k_to_rel(int n, const int64_t* __restrict__ rp, const int* __restrict__ ci, int64_t gbeg,
                         int64_t gend, const int* __restrict__ hid, int nh, int nlo, int* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            const int c = ci[p];
            int r;
            if ((int64_t)c >= gbeg && (int64_t)c < gend) {
                r = (int)(c - gbeg);
            } else {
                const int k = lower_bound_i(hid, nh, c);
                r = k < nlo ? k - nlo : n + (k - nlo);
            }
            out[p] = r;
        }
}

// relative column -> global id
__global__ void k_rel_to_glob(int64_t m, const int* __restrict__ ci, int64_t gbeg, int n,
                              const int* __restrict__ hid, int nlo, int* __restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        const int c = ci[p];
        out[p] = c < 0 ? hid[nlo + c] : (c < n ? (int)(gbeg + c) : hid[nlo + (c - n)]);
    }
}

template <class T>
__global__ void k_pack(int m, const int* __restrict__ sidx, const T* __restrict__ x, T* __restrict__ buf) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) buf[k] = x[sidx[k]];
}

__global__ void k_agg_glob(int n, const int* __restrict__ agg, int cbeg, int* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = cbeg + agg[i];
}

// coarse column map of every fine column j in [-nlo, n + nhi): the coarse level's relative column of
// the aggregate holding j, shifted by the coarse nlo so it is >= 0 (the Galerkin key)
__global__ void k_colmap(int jlo, int jhi, const int* __restrict__ aggg, int cbeg, int nc, const int* __restrict__ hidc,
                         int nhc, int nloc, int* __restrict__ cmap) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < jhi - jlo; t += gridDim.x * blockDim.x) {
        const int j = jlo + t;
        const int G = aggg[j];
        int r;
        if (G >= cbeg && G < cbeg + nc) {
            r = G - cbeg;
        } else {
            const int k = lower_bound_i(hidc, nhc, G);
            r = k < nloc ? k - nloc : nc + (k - nloc);
        }
        cmap[j] = r + nloc;
    }
}

__global__ void k_shift_cols(int64_t m, int* __restrict__ ci, int d) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x)
        ci[p] += d;
}

__global__ void k_row_len(int n, const int* __restrict__ rp, int* __restrict__ len) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) len[i] = rp[i + 1] - rp[i];
}

struct ScalarPtrs {
    double* p[kArMax];
    int k;
};
// local partial = main (+ the boundary views' partials of a split pass, added in this fixed order)
__global__ void k_ar_pack(ScalarPtrs sp, ScalarPtrs e1, ScalarPtrs e2, double* __restrict__ buf) {
    for (int j = threadIdx.x; j < sp.k; j += blockDim.x) {
        double v = *sp.p[j];
        if (j < e1.k) v += *e1.p[j];
        if (j < e2.k) v += *e2.p[j];
        buf[j] = v;
    }
}
// rank-order sum of the gathered partials: identical bits on every rank
__global__ void k_ar_sum(ScalarPtrs sp, const double* __restrict__ g, int P) {
    for (int j = threadIdx.x; j < sp.k; j += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < P; ++r) s += g[(size_t)r * sp.k + j];
        *sp.p[j] = s;
    }
}

// ------------------------------------------------------------------ host exchange helpers
template <class T>
static std::vector<T> allgather_host(Comm* c, const T& v, cudaStream_t s) {
    T* d = dalloc<T>(1 + (size_t)c->size, s);
    CK(cudaMemcpyAsync(d, &v, sizeof(T), cudaMemcpyHostToDevice, s));
    c->allgather(d, d + 1, sizeof(T), s);
    std::vector<T> out(c->size);
    CK(cudaMemcpyAsync(out.data(), d + 1, sizeof(T) * c->size, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(d, s);
    return out;
}

template <class T>
static std::vector<T> allgather_vec_host(Comm* c, const std::vector<T>& v, cudaStream_t s) {
    const size_t k = v.size();
    T* d = dalloc<T>(k * (1 + (size_t)c->size), s);
    CK(cudaMemcpyAsync(d, v.data(), sizeof(T) * k, cudaMemcpyHostToDevice, s));
    c->allgather(d, d + k, sizeof(T) * k, s);
    std::vector<T> out(k * c->size);
    CK(cudaMemcpyAsync(out.data(), d + k, sizeof(T) * out.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(d, s);
    return out;
}

// every rank's int list for every peer -> the lists every peer addressed to this rank
static std::vector<std::vector<int>> alltoallv_int(Comm* c, const std::vector<std::vector<int>>& send,
                                                   cudaStream_t s) {
    const int P = c->size, me = c->rank;
    std::vector<int> cnt(P);
    for (int q = 0; q < P; ++q) cnt[q] = (int)send[q].size();
    const std::vector<int> M = allgather_vec_host(c, cnt, s);  // M[r * P + q]: r sends q
    std::vector<int> soff(P + 1, 0), roff(P + 1, 0);
    for (int q = 0; q < P; ++q) {
        soff[q + 1] = soff[q] + (q == me ? 0 : cnt[q]);
        roff[q + 1] = roff[q] + (q == me ? 0 : M[(size_t)q * P + me]);
    }
    int* sb = dalloc<int>((size_t)soff[P] + 1, s);
    int* rb = dalloc<int>((size_t)roff[P] + 1, s);
    std::vector<int> hs((size_t)soff[P] + 1);
    for (int q = 0; q < P; ++q)
        if (q != me) std::copy(send[q].begin(), send[q].end(), hs.begin() + soff[q]);
    CK(cudaMemcpyAsync(sb, hs.data(), sizeof(int) * soff[P], cudaMemcpyHostToDevice, s));
    std::vector<P2P> ss, rr;
    for (int q = 0; q < P; ++q) {
        if (q == me) continue;
        if (cnt[q]) ss.push_back({q, sb + soff[q], sizeof(int) * (size_t)cnt[q]});
        const int rc = M[(size_t)q * P + me];
        if (rc) rr.push_back({q, rb + roff[q], sizeof(int) * (size_t)rc});
    }
    c->sendrecv(ss, rr, s);
    std::vector<int> hr((size_t)roff[P] + 1);
    CK(cudaMemcpyAsync(hr.data(), rb, sizeof(int) * roff[P], cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(sb, s);
    dfree(rb, s);
    std::vector<std::vector<int>> out(P);
    for (int q = 0; q < P; ++q) {
        if (q == me) out[q] = send[q];
        else out[q].assign(hr.begin() + roff[q], hr.begin() + roff[q + 1]);
    }
    return out;
}

// grouped point-to-point allgatherv: chunk r = bytes [displ[r], displ[r+1]) of `full`; the own chunk
// is already in place
static void allgatherv_bytes(Comm* c, void* full, const std::vector<int64_t>& displ, cudaStream_t s) {
    const int P = c->size, me = c->rank;
    char* f = static_cast<char*>(full);
    std::vector<P2P> ss, rr;
    const size_t own = (size_t)(displ[me + 1] - displ[me]);
    for (int q = 0; q < P; ++q) {
        if (q == me) continue;
        if (own) ss.push_back({q, f + displ[me], own});
        const size_t b = (size_t)(displ[q + 1] - displ[q]);
        if (b) rr.push_back({q, f + displ[q], b});
    }
    c->sendrecv(ss, rr, s);
}

void allgatherv_d(amg_hierarchy* h, double* full, const std::vector<int64_t>& offs) {
    std::vector<int64_t> displ(offs.size());
    for (size_t r = 0; r < offs.size(); ++r) displ[r] = offs[r] * (int64_t)sizeof(double);
    allgatherv_bytes(h->comm, full, displ, h->s);
}

// ------------------------------------------------------------------ halo plan (host bookkeeping)
// From the sorted halo ids of a block: the receive segments (one contiguous run per owner, below
// then above the own rows) and, per owner, the list of requested global ids.
static void plan_halo(int64_t gbeg, int n, const std::vector<int64_t>& offs, int rank, const std::vector<int>& hid,
                      Halo& H, std::vector<std::vector<int>>& req) {
    const int P = (int)offs.size() - 1;
    H.hid = hid;
    H.nlo = (int)(std::lower_bound(hid.begin(), hid.end(), (int)gbeg) - hid.begin());
    H.nhi = (int)hid.size() - H.nlo;
    H.recv.clear();
    req.assign(P, {});
    for (size_t k = 0; k < hid.size();) {
        const int q = (int)(std::upper_bound(offs.begin(), offs.end(), (int64_t)hid[k]) - offs.begin()) - 1;
        if (q < 0 || q >= P || q == rank) throw Error(AMG_E_INPUT, "halo column outside every other rank's block");
        size_t e = k;
        while (e < hid.size() && hid[e] < offs[q + 1]) ++e;
        const int off = (int)k < H.nlo ? (int)k - H.nlo : n + ((int)k - H.nlo);
        H.recv.push_back({q, off, (int)(e - k)});
        req[q].insert(req[q].end(), hid.begin() + k, hid.begin() + e);
        k = e;
    }
}

// exchange the requests; build the send lists (device sidx) and the send buffer
static void finish_halo(amg_hierarchy* h, Level& Lv, const std::vector<std::vector<int>>& req) {
    cudaStream_t s = h->s;
    const std::vector<std::vector<int>> got = alltoallv_int(h->comm, req, s);
    Halo& H = Lv.H;
    H.send.clear();
    std::vector<int> sidx;
    int bad = 0;
    for (int q = 0; q < (int)got.size(); ++q) {
        if (q == h->comm->rank || got[q].empty()) continue;
        H.send.push_back({q, (int)sidx.size(), (int)got[q].size()});
        for (int G : got[q]) {
            if ((int64_t)G < Lv.gbeg || (int64_t)G >= Lv.gbeg + Lv.A.n) bad = 1;
            sidx.push_back((int)(G - Lv.gbeg));
        }
    }
    // collective decision: every rank fails together (no rank is left waiting in a later exchange)
    const std::vector<int> bads = allgather_host<int>(h->comm, bad, s);
    if (std::accumulate(bads.begin(), bads.end(), 0))
        throw Error(AMG_E_INPUT, "halo request outside the owner's block (asymmetric pattern across blocks)");
    H.nsend = (int)sidx.size();
    H.sidx = halloc<int>(h, sidx.size());
    H.sbuf = halloc<double>(h, sidx.size());
    H.d_hid = halloc<int>(h, H.hid.size());
    if (!sidx.empty()) CK(cudaMemcpyAsync(H.sidx, sidx.data(), sizeof(int) * sidx.size(), cudaMemcpyHostToDevice, s));
    if (!H.hid.empty())
        CK(cudaMemcpyAsync(H.d_hid, H.hid.data(), sizeof(int) * H.hid.size(), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
}

template <class T>
static void halo_exchange_t(amg_hierarchy* h, Level& Lv, T* x) {
    const Halo& H = Lv.H;
    T* buf = reinterpret_cast<T*>(H.sbuf);
    if (H.nsend) {
        launch_k(k_pack<T>, dim3(gridn(H.nsend)), dim3(kBlock), 0, h->s, H.nsend, (const int*)H.sidx, (const T*)x, buf);
        CK(cudaGetLastError());
        ++g_launches;
    }
    std::vector<P2P> ss, rr;
    for (const Seg& g : H.send) ss.push_back({g.peer, buf + g.off, sizeof(T) * (size_t)g.cnt});
    for (const Seg& g : H.recv) rr.push_back({g.peer, x + g.off, sizeof(T) * (size_t)g.cnt});
    h->comm->sendrecv(ss, rr, h->s);
}

void halo_exchange(amg_hierarchy* h, int l, double* x) {
    Level& Lv = h->lev[l];
    if (!Lv.dist) return;
    halo_exchange_t<double>(h, Lv, x);
}

void halo_start(amg_hierarchy* h, int l, double* x) {
    Level& Lv = h->lev[l];
    if (!Lv.dist) return;
    const Halo& H = Lv.H;
    double* buf = H.sbuf;
    if (H.nsend) {
        launch_k(k_pack<double>, dim3(gridn(H.nsend)), dim3(kBlock), 0, h->s, H.nsend, (const int*)H.sidx,
                 (const double*)x, buf);
        CK(cudaGetLastError());
        ++g_launches;
    }
    CK(cudaEventRecord(h->ev_pack, h->s));
    CK(cudaStreamWaitEvent(h->cs, h->ev_pack, 0));
    std::vector<P2P> ss, rr;
    for (const Seg& g : H.send) ss.push_back({g.peer, buf + g.off, sizeof(double) * (size_t)g.cnt});
    for (const Seg& g : H.recv) rr.push_back({g.peer, x + g.off, sizeof(double) * (size_t)g.cnt});
    h->comm->sendrecv(ss, rr, h->cs);
    CK(cudaEventRecord(h->ev_halo, h->cs));
}

void halo_finish(amg_hierarchy* h, int l) {
    if (!h->lev[l].dist) return;
    CK(cudaStreamWaitEvent(h->s, h->ev_halo, 0));
}

__global__ void k_slice_flags(int n, const int* __restrict__ rp, const int* __restrict__ ci, unsigned char* flag) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        bool b = false;
        for (int p = rp[i]; p < rp[i + 1]; ++p) b |= (ci[p] < 0 || ci[p] >= n);
        if (b) flag[i >> 5] = 1;
    }
}

// The interior range is the longest run of slices without a halo column; the boundary ranges are
// the slices before and after it (2D strips / 3D slabs: the first and last grid lines of the block).
void build_split(amg_hierarchy* h, int l) {
    Level& Lv = h->lev[l];
    Lv.split = false;
    if (!Lv.dist || !Lv.op.sell || getenv("AMG_NO_OVERLAP")) return;
    const int ns = Lv.S.nslices;
    unsigned char* f = dalloc<unsigned char>((size_t)ns + 1, h->s);
    CK(cudaMemsetAsync(f, 0, (size_t)ns + 1, h->s));
    k_slice_flags<<<gridn(Lv.A.n), kBlock, 0, h->s>>>(Lv.A.n, Lv.A.rp, Lv.A.ci, f);
    ++g_launches;
    CK(cudaGetLastError());
    std::vector<unsigned char> hf((size_t)ns);
    CK(cudaMemcpyAsync(hf.data(), f, (size_t)ns, cudaMemcpyDeviceToHost, h->s));
    CK(cudaStreamSynchronize(h->s));
    dfree(f, h->s);
    int best_b = 0, best_e = 0;
    for (int s = 0; s < ns;) {
        if (hf[s]) { ++s; continue; }
        int e = s;
        while (e < ns && !hf[e]) ++e;
        if (e - s > best_e - best_b) { best_b = s; best_e = e; }
        s = e;
    }
    if (best_b == 0 && best_e == ns) return;  // no boundary slice (no halo): nothing to overlap
    if (best_e - best_b < ns / 4) return;     // too little interior to hide the messages behind
    auto view = [&](int a, int b) {
        SpOp v = Lv.op;
        v.S.sptr = Lv.S.sptr + a;
        v.S.nslices = b - a;
        v.S.srow0 = 32 * a;
        return v;
    };
    Lv.op_int = view(best_b, best_e);
    Lv.op_lo = view(0, best_b);
    Lv.op_hi = view(best_e, ns);
    Lv.split = true;
}

void dot_allreduce(amg_hierarchy* h, const std::vector<double*>& ptrs, const std::vector<double*>& extra1,
                   const std::vector<double*>& extra2) {
    if (!h->comm || ptrs.empty()) return;
    if ((int)ptrs.size() > kArMax) throw Error(AMG_E_ARG, "too many scalars in one allreduce");
    ScalarPtrs sp{}, e1{}, e2{};
    sp.k = (int)ptrs.size();
    e1.k = (int)extra1.size();
    e2.k = (int)extra2.size();
    for (int j = 0; j < sp.k; ++j) sp.p[j] = ptrs[j];
    for (int j = 0; j < e1.k; ++j) e1.p[j] = extra1[j];
    for (int j = 0; j < e2.k; ++j) e2.p[j] = extra2[j];
    launch_k(k_ar_pack, dim3(1), dim3(64), 0, h->s, sp, e1, e2, h->ar_send);
    CK(cudaGetLastError());
    h->comm->allgather(h->ar_send, h->ar_recv, sizeof(double) * (size_t)sp.k, h->s);
    launch_k(k_ar_sum, dim3(1), dim3(64), 0, h->s, sp, (const double*)h->ar_recv, h->comm->size);
    CK(cudaGetLastError());
    g_launches += 2;
}

// ------------------------------------------------------------------ sorted unique ids (device)
static std::vector<int> sorted_unique(const int* d_in, int m, cudaStream_t s) {
    std::vector<int> out;
    if (m <= 0) return out;
    int* k1 = dalloc<int>(m, s);
    int* k2 = dalloc<int>(m, s);
    int* nu = dalloc<int>(1, s);
    size_t tb = 0, tb2 = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, d_in, k1, m, 0, 32, s));
    CK(cub::DeviceSelect::Unique(nullptr, tb2, k1, k2, nu, m, s));
    void* tmp = dalloc<char>(std::max(tb, tb2), s);
    CK(cub::DeviceRadixSort::SortKeys(tmp, tb, d_in, k1, m, 0, 32, s));
    CK(cub::DeviceSelect::Unique(tmp, tb2, k1, k2, nu, m, s));
    int hn = 0;
    CK(cudaMemcpyAsync(&hn, nu, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    out.resize(hn);
    if (hn) CK(cudaMemcpyAsync(out.data(), k2, sizeof(int) * hn, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(tmp, s);
    dfree(k1, s);
    dfree(k2, s);
    dfree(nu, s);
    return out;  // non-negative ids: the unsigned-radix order is the signed order
}

static int64_t scan_counts(const int* in, int* out, int n, cudaStream_t s) {  // exclusive, out[n] = total
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n + 1, s));
    void* tmp = dalloc<char>(tb, s);
    CK(cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, n + 1, s));
    dfree(tmp, s);
    int tot = 0;
    CK(cudaMemcpyAsync(&tot, out + n, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return tot;
}

// ------------------------------------------------------------------ gather a level (replicate it)
static void gather_level(amg_hierarchy* h, int l) {
    Comm* c = h->comm;
    cudaStream_t s = h->s;
    Level& Lv = h->lev[l];
    const int P = c->size, me = c->rank;
    const int n = Lv.A.n;
    const std::vector<int64_t> nnzs = allgather_host<int64_t>(c, Lv.A.nnz, s);
    std::vector<int64_t> eoff(P + 1, 0);
    for (int r = 0; r < P; ++r) eoff[r + 1] = eoff[r] + nnzs[r];
    const int64_t N = Lv.nglob, NNZ = eoff[P];
    if (N + NNZ >= (int64_t(1) << 31) - 64) throw Error(AMG_E_ARG, "gathered level too large");
    int* len = dalloc<int>((size_t)N + 1, s);
    int* ci = dalloc<int>((size_t)NNZ + 8, s);
    double* v = dalloc<double>((size_t)NNZ + 8, s);
    CK(cudaMemsetAsync(ci + NNZ, 0, 8 * sizeof(int), s));
    CK(cudaMemsetAsync(v + NNZ, 0, 8 * sizeof(double), s));
    k_row_len<<<gridn(n), kBlock, 0, s>>>(n, Lv.A.rp, len + Lv.offs[me]);
    k_rel_to_glob<<<gridn(Lv.A.nnz), kBlock, 0, s>>>(Lv.A.nnz, Lv.A.ci, Lv.gbeg, n, Lv.H.d_hid, Lv.H.nlo,
                                                       ci + eoff[me]);
    g_launches += 2;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(v + eoff[me], Lv.A.v, sizeof(double) * Lv.A.nnz, cudaMemcpyDeviceToDevice, s));
    std::vector<int64_t> d(P + 1);
    for (int r = 0; r <= P; ++r) d[r] = Lv.offs[r] * (int64_t)sizeof(int);
    allgatherv_bytes(c, len, d, s);
    for (int r = 0; r <= P; ++r) d[r] = eoff[r] * (int64_t)sizeof(int);
    allgatherv_bytes(c, ci, d, s);
    for (int r = 0; r <= P; ++r) d[r] = eoff[r] * (int64_t)sizeof(double);
    allgatherv_bytes(c, v, d, s);
    int* rp = dalloc<int>((size_t)N + 1, s);
    CK(cudaMemsetAsync(len + N, 0, sizeof(int), s));
    scan_counts(len, rp, (int)N, s);
    dfree(len, s);
    free_csr(Lv.A, s);
    Lv.A.n = (int)N;
    Lv.A.nnz = NNZ;
    Lv.A.rp = rp;
    Lv.A.ci = ci;
    Lv.A.v = v;
    Lv.dist = false;
    Lv.H = Halo{};
    CK(cudaStreamSynchronize(s));
}

// global aggregation (below): one level, the prolongation indices, the export-plan warm-up
static void gx_build_level(amg_hierarchy* h, int l);
static void gx_finish(amg_hierarchy* h);
static void gx_warm(amg_hierarchy* h);

// ------------------------------------------------------------------ distributed setup
void build_dist(amg_hierarchy* h, int64_t n_global, int64_t row_begin, int n_local_in, const int64_t* rp_in,
                const int32_t* ci_in, const double* v_in, const double* d_in) {
    Comm* c = h->comm;
    cudaStream_t s = h->s;
    const int P = c->size, me = c->rank;
    // collective argument check (every rank takes the same decision)
    struct Args {
        int64_t n_global, row_begin, n_local, nnz, rp0;
    } a{n_global, row_begin, n_local_in, 0, 0};
    const bool local_ok = n_local_in >= 1 && n_local_in < (1 << 30) && rp_in && ci_in && v_in;
    void* t_rp = nullptr;
    const int64_t* rp = nullptr;
    if (local_ok) {
        int64_t* drp = dalloc<int64_t>((size_t)n_local_in + 1, s);
        CK(cudaMemcpyAsync(drp, rp_in, sizeof(int64_t) * ((size_t)n_local_in + 1), cudaMemcpyDefault, s));
        CK(cudaMemcpyAsync(&a.nnz, drp + n_local_in, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&a.rp0, drp, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        t_rp = drp;
        rp = drp;
    } else {
        a.n_local = -1;
    }
    const std::vector<Args> all = allgather_host(c, a, s);
    std::vector<int64_t> offs(P + 1, 0);
    bool ok = true;
    for (int r = 0; r < P; ++r) {
        const Args& x = all[r];
        ok = ok && x.n_local >= 1 && x.n_global == all[0].n_global && x.row_begin == offs[r] && x.rp0 == 0 &&
             x.nnz >= 0 && x.nnz + x.n_local < (int64_t(1) << 31) - 64;
        offs[r + 1] = offs[r] + (x.n_local > 0 ? x.n_local : 0);
    }
    ok = ok && offs[P] == n_global && n_global < (int64_t(1) << 31) - 8;
    if (!ok) {
        dfree(t_rp, s);
        throw Error(AMG_E_ARG, "amg_setup_dist: the ranks' row blocks must tile [0, n_global) in rank order "
                               "(row_begin, n_local >= 1, row_ptr[0] = 0)");
    }
    const int n = n_local_in;
    const int64_t gbeg = row_begin, gend = row_begin + n, nnz_in = a.nnz;
    {   // pool pre-reservation (as on one GPU)
        const size_t want = (size_t)(nnz_in + n) * 64 + ((size_t)256 << 20);
        void* r = nullptr;
        if (cudaMallocAsync(&r, want, s) == cudaSuccess) dfree(r, s); else cudaGetLastError();
    }
    int* ci_g = dalloc<int>((size_t)nnz_in + 8, s);
    double* v = dalloc<double>((size_t)nnz_in + 8, s);
    double* d = d_in ? dalloc<double>((size_t)n + 8, s) : nullptr;
    CK(cudaMemcpyAsync(ci_g, ci_in, sizeof(int) * nnz_in, cudaMemcpyDefault, s));
    CK(cudaMemcpyAsync(v, v_in, sizeof(double) * nnz_in, cudaMemcpyDefault, s));
    if (d) CK(cudaMemcpyAsync(d, d_in, sizeof(double) * n, cudaMemcpyDefault, s));
    // halo ids and relative columns
    int* cand = dalloc<int>((size_t)nnz_in + 1, s);
    int* cnt = dalloc<int>(2, s);
    CK(cudaMemsetAsync(cnt, 0, 2 * sizeof(int), s));
    k_halo_collect<<<gridn(n), kBlock, 0, s>>>(n, nnz_in, rp, ci_g, gbeg, gend, n_global, cand, cnt, cnt + 1);
    ++g_launches;
    CK(cudaGetLastError());
    int hc[2] = {0, 0};
    CK(cudaMemcpyAsync(hc, cnt, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const std::vector<int> hid = sorted_unique(cand, hc[0], s);
    dfree(cand, s);
    dfree(cnt, s);
    Level& L0 = h->lev[0];
    L0.dist = true;
    L0.gbeg = gbeg;
    L0.nglob = n_global;
    L0.offs = offs;
    std::vector<std::vector<int>> req;
    int vf = hc[1];  // VF_RANGE / VF_RP
    int* ci_r = dalloc<int>((size_t)nnz_in + 8, s);
    if (!vf) {
        plan_halo(gbeg, n, offs, me, hid, L0.H, req);
        if (L0.H.nlo >= (1 << 30) || L0.H.nhi >= (1 << 30) || (int64_t)n + L0.H.nhi >= (int64_t(1) << 31) - 8)
            vf |= 1;
    }
    if (!vf) {
        int* dh = dalloc<int>(hid.size() + 1, s);
        if (!hid.empty()) CK(cudaMemcpyAsync(dh, hid.data(), sizeof(int) * hid.size(), cudaMemcpyHostToDevice, s));
        k_to_rel<<<gridn(n), kBlock, 0, s>>>(n, rp, ci_g, gbeg, gend, dh, (int)hid.size(), L0.H.nlo, ci_r);
        ++g_launches;
        CK(cudaGetLastError());
        dfree(dh, s);
        vf |= validate_input(n, nnz_in, -L0.H.nlo, n + L0.H.nhi, rp, ci_r, v, d, s);
    }
    const int nonzero_d = (d && any_nonzero(n, d, s)) ? 1 : 0;
    const std::vector<int> flags = allgather_vec_host(c, std::vector<int>{vf, nonzero_d}, s);
    int vall = 0, dall = 0;
    for (int r = 0; r < P; ++r) {
        vall |= flags[2 * r];
        dall |= flags[2 * r + 1];
    }
    if (vall) {
        dfree(t_rp, s); dfree(ci_g, s); dfree(ci_r, s); dfree(v, s); dfree(d, s);
        throw Error(AMG_E_INPUT, validation_message(vall) + (vf ? "" : " (on another rank)"));
    }
    h->singular = !dall;
    L0.A = form_A0(n, rp, ci_r, v, d, s);
    dfree(t_rp, s); dfree(ci_g, s); dfree(ci_r, s); dfree(v, s); dfree(d, s);
    h->L = 1;
    h->row_begin = gbeg;
    h->n_global = n_global;
    h->n_local = n;
    finish_halo(h, L0, req);

    // row-partitioned level loop (a1-a6 with decoupled aggregation, A20)
    const int m = h->m, p = h->p;
    int l = 0;
    for (;;) {
        Level& Lv = h->lev[l];
        const std::vector<int64_t> nz = allgather_host<int64_t>(c, Lv.A.nnz, s);
        Lv.nnz_glob = std::accumulate(nz.begin(), nz.end(), (int64_t)0);
        const std::vector<double> l1 = allgather_host<double>(c, inf_norm(Lv.A, s), s);
        Lv.lambda1 = *std::max_element(l1.begin(), l1.end());
        Lv.kappa = h->opt.kappa > 1.0 ? h->opt.kappa : kappa_rule(m);
        poly_coeffs(Lv.lambda1, Lv.kappa, m, Lv.alpha, Lv.beta);
        if (Lv.nglob <= h->opt.coarsest_size || Lv.nglob < h->opt.gather_rows) break;  // replicate from here
        if (l + 1 >= kMaxLevels) throw Error(AMG_E_SETUP, "too many levels");
        if (h->opt.global_agg) {  // aggregates across the blocks
            gx_build_level(h, l);
            ++l;
            continue;
        }
        PassGraph G = pass_graph0(Lv.A, s);  // in-block edges only
        int* agg = nullptr;
        int nc = Lv.A.n;
        for (int t = 0; t < p; ++t) {
            const std::vector<int> gn = allgather_host<int>(c, G.n, s);
            const int id_off = std::accumulate(gn.begin(), gn.begin() + me, 0);
            const uint64_t salt = host_sm64(h->opt.seed ^ (((uint64_t)l << 8) ^ (uint64_t)t));
            int* agg_t = dalloc<int>((size_t)G.n + 8, s);
            int nct = 0;
            aggregate_pass(G, salt, id_off, agg_t, &nct, &Lv.rounds[t], s);
            if (t + 1 < p) {
                PassGraph G2 = quotient_graph(G, agg_t, nct, s);
                free_graph(G, s);
                G = G2;
            }
            if (t == 0) {
                agg = agg_t;
            } else {
                compose(Lv.A.n, agg, agg_t, s);
                dfree(agg_t, s);
            }
            nc = nct;
        }
        free_graph(G, s);
        const std::vector<int> ncs = allgather_host<int>(c, nc, s);
        std::vector<int64_t> coffs(P + 1, 0);
        for (int r = 0; r < P; ++r) coffs[r + 1] = coffs[r] + ncs[r];
        if (coffs[P] >= Lv.nglob) {
            dfree(agg, s);
            throw Error(AMG_E_SETUP, "coarsening stagnated (n_{l+1} = n_l)");
        }
        Lv.nc = nc;
        Lv.agg = agg;
        h->allocs.push_back(agg);
        Lv.perm = halloc<int>(h, Lv.A.n);
        Lv.aptr = halloc<int>(h, (size_t)nc + 1);
        aggregate_order(Lv.A.n, agg, nc, Lv.perm, Lv.aptr, s);
        // global coarse id of every own and halo column
        const int nlo = Lv.H.nlo, nhi = Lv.H.nhi;
        int* aggg_b = dalloc<int>((size_t)nlo + n + nhi + 8, s);
        int* aggg = aggg_b + nlo;
        const int cbeg = (int)coffs[me];
        k_agg_glob<<<gridn(Lv.A.n), kBlock, 0, s>>>(Lv.A.n, agg, cbeg, aggg);
        ++g_launches;
        CK(cudaGetLastError());
        halo_exchange_t<int>(h, Lv, aggg);
        std::vector<int> hh((size_t)nlo + nhi);
        if (nlo) CK(cudaMemcpyAsync(hh.data(), aggg_b, sizeof(int) * nlo, cudaMemcpyDeviceToHost, s));
        if (nhi) CK(cudaMemcpyAsync(hh.data() + nlo, aggg + Lv.A.n, sizeof(int) * nhi, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::sort(hh.begin(), hh.end());
        hh.erase(std::unique(hh.begin(), hh.end()), hh.end());
        Level& Cn = h->lev[l + 1];
        Cn.dist = true;
        Cn.gbeg = cbeg;
        Cn.nglob = coffs[P];
        Cn.offs = coffs;
        std::vector<std::vector<int>> creq;
        plan_halo(cbeg, nc, coffs, me, hh, Cn.H, creq);
        // Galerkin with the coarse relative columns (shifted by the coarse nlo to be >= 0)
        const int nloc = Cn.H.nlo;
        int* dhc = dalloc<int>(hh.size() + 1, s);
        if (!hh.empty()) CK(cudaMemcpyAsync(dhc, hh.data(), sizeof(int) * hh.size(), cudaMemcpyHostToDevice, s));
        int* cmap_b = dalloc<int>((size_t)nlo + n + nhi + 8, s);
        k_colmap<<<gridn((int64_t)nlo + Lv.A.n + nhi), kBlock, 0, s>>>(-nlo, Lv.A.n + nhi, aggg, cbeg, nc, dhc,
                                                                        (int)hh.size(), nloc, cmap_b + nlo);
        ++g_launches;
        CK(cudaGetLastError());
        Cn.A = galerkin(Lv.A, agg, cmap_b + nlo, nc, nc + (int)hh.size(), Lv.perm, Lv.aptr, s);
        k_shift_cols<<<gridn(Cn.A.nnz), kBlock, 0, s>>>(Cn.A.nnz, Cn.A.ci, -nloc);
        ++g_launches;
        CK(cudaGetLastError());
        dfree(aggg_b, s);
        dfree(cmap_b, s);
        dfree(dhc, s);
        h->L = l + 2;
        finish_halo(h, Cn, creq);
        ++l;
    }
    h->g = l;
    gather_level(h, l);  // every rank now holds level g whole
    build_levels(h, l);
    gx_finish(h);
    finish_build(h);
    warm_comm(h);
}

void warm_comm(amg_hierarchy* h) {
    for (int l = 0; l < h->g; ++l)
        if (h->lev[l].X) halo_exchange(h, l, h->lev[l].X);
    gx_warm(h);
    dot_allreduce(h, {h->osc + 2 * kMaxWin + 4});
    // the split passes' message pattern (same messages, other stream) -- on every rank: whether a
    // level is split is a local decision, and the number of exchanges must match across the ranks
    for (int l = 0; l < h->g; ++l)
        if (h->lev[l].X) {
            halo_start(h, l, h->lev[l].X);
            halo_finish(h, l);
        }
    if (h->g >= 1) allgatherv_d(h, h->lev[h->g].RHO, h->lev[h->g].offs);
    else allgatherv_d(h, h->b, h->lev[0].offs);
    CK(cudaStreamSynchronize(h->s));
}

void export_dist_cols(amg_hierarchy* h, int l, int* out) {
    const Level& Lv = h->lev[l];
    k_rel_to_glob<<<gridn(Lv.A.nnz), kBlock, 0, h->s>>>(Lv.A.nnz, Lv.A.ci, Lv.gbeg, Lv.A.n, Lv.H.d_hid, Lv.H.nlo, out);
    CK(cudaGetLastError());
}

void export_dist_agg(amg_hierarchy* h, int l, int* out) {
    const Level& Lv = h->lev[l];
    if (Lv.gx) {  // global coarse ids already
        CK(cudaMemcpyAsync(out, Lv.aggG, sizeof(int) * Lv.A.n, cudaMemcpyDeviceToDevice, h->s));
        return;
    }
    const Level& C = h->lev[l + 1];
    k_agg_glob<<<gridn(Lv.A.n), kBlock, 0, h->s>>>(Lv.A.n, Lv.agg, (int)C.offs[h->comm->rank], out);
    CK(cudaGetLastError());
}

}  // namespace amg

// ------------------------------------------------------------------ host-only hook (CPU tests)
extern "C" int amg_halo_plan(int64_t row_begin, int32_t n_local, const int64_t* offs, int32_t nranks, int32_t rank,
                             const int32_t* halo_ids, int32_t n_halo, int32_t* seg_peer, int32_t* seg_off,
                             int32_t* seg_cnt, int32_t* n_seg, int32_t* n_lo) {
    if (!offs || nranks < 1 || rank < 0 || rank >= nranks || n_halo < 0 || (n_halo && !halo_ids) || !n_seg)
        return AMG_E_ARG;
    try {
        std::vector<int64_t> o(offs, offs + nranks + 1);
        std::vector<int> hid(halo_ids, halo_ids + n_halo);
        if (!std::is_sorted(hid.begin(), hid.end()) || std::adjacent_find(hid.begin(), hid.end()) != hid.end())
            return AMG_E_ARG;
        amg::Halo H;
        std::vector<std::vector<int>> req;
        amg::plan_halo(row_begin, n_local, o, rank, hid, H, req);
        *n_seg = (int)H.recv.size();
        if (n_lo) *n_lo = H.nlo;
        for (size_t k = 0; k < H.recv.size(); ++k) {
            if (seg_peer) seg_peer[k] = H.recv[k].peer;
            if (seg_off) seg_off[k] = H.recv[k].off;
            if (seg_cnt) seg_cnt[k] = H.recv[k].cnt;
        }
    } catch (const amg::Error& e) {
        amg::set_last_error(e.what());
        return e.code;
    }
    return AMG_OK;
}

namespace amg {

// ================================================================== global aggregation (f4)
// amg_options.global_agg = 1: the matching passes of a row-partitioned level
// see every edge, including the edges between blocks, so the aggregates are those of the
// single-GPU rule (the oracle's nparts = 1) bit for bit.  Matching: handshake rounds in which every
// rank proposes for its own free vertices over own and halo neighbours (keys of global ids, docs/
// keys.md), and the proposals and mates of the boundary vertices are exchanged over the pass
// graph's halo plan after every step ("halo rounds").  An aggregate is owned by the rank of its
// leader (the min vertex of its pair): coarse ids are leader ranks, so every rank's coarse block is
// contiguous.  The quotient pass graphs and the Galerkin product are formed from (I, J, value)
// triples routed to the owner of I (members' rows cross ranks), merged by a stable sort, so each
// coarse entry is summed in increasing (fine row, CSR position) order: the oracle's order.  In the
// solve the restriction receives the remote members' residuals through an export plan and sums
// every aggregate's members in increasing global row order; the prolongation reads the correction
// of remote aggregates from the coarse level's halo (their ids are added to it).

struct DistG {                 // distributed pass graph G_t: own vertices [gbeg, gbeg + n)
    int n = 0;
    int64_t gbeg = 0;
    std::vector<int64_t> offs;  // vertex blocks of all ranks
    int64_t nnz = 0;
    int* rp = nullptr;
    int* ci = nullptr;          // relative columns (halo outside [0, n))
    uint32_t* w = nullptr;
    Halo H;                     // exchange plan of per-vertex values (own -> halo slots)
    bool own_plan = false;      // H's device arrays belong to this graph (else to the level)
    int* gid_b = nullptr;       // global id of every relative index, base = -nlo
    const int* gid() const { return gid_b + H.nlo; }
};

template <class T>
static void plan_xchg(amg_hierarchy* h, const Halo& H, const T* src, T* dst) {
    T* buf = reinterpret_cast<T*>(H.sbuf);
    if (H.nsend) {
        launch_k(k_pack<T>, dim3(gridn(H.nsend)), dim3(kBlock), 0, h->s, H.nsend, (const int*)H.sidx, src, buf);
        CK(cudaGetLastError());
        ++g_launches;
    }
    std::vector<P2P> ss, rr;
    for (const Seg& g : H.send) ss.push_back({g.peer, buf + g.off, sizeof(T) * (size_t)g.cnt});
    for (const Seg& g : H.recv) rr.push_back({g.peer, dst + g.off, sizeof(T) * (size_t)g.cnt});
    h->comm->sendrecv(ss, rr, h->s);
}

// send lists from the requests (temporary plan: device arrays from dalloc, freed with the graph)
static void finish_plan_tmp(amg_hierarchy* h, Halo& H, int64_t gbeg, int n, const std::vector<std::vector<int>>& req) {
    cudaStream_t s = h->s;
    const std::vector<std::vector<int>> got = alltoallv_int(h->comm, req, s);
    H.send.clear();
    std::vector<int> sidx;
    for (int q = 0; q < (int)got.size(); ++q) {
        if (q == h->comm->rank || got[q].empty()) continue;
        H.send.push_back({q, (int)sidx.size(), (int)got[q].size()});
        for (int G : got[q]) {
            if ((int64_t)G < gbeg || (int64_t)G >= gbeg + n) throw Error(AMG_E_SETUP, "global aggregation: bad request");
            sidx.push_back((int)(G - gbeg));
        }
    }
    H.nsend = (int)sidx.size();
    H.sidx = dalloc<int>(sidx.size() + 1, s);
    H.sbuf = dalloc<double>(sidx.size() + 1, s);
    H.d_hid = dalloc<int>(H.hid.size() + 1, s);
    if (!sidx.empty()) CK(cudaMemcpyAsync(H.sidx, sidx.data(), sizeof(int) * sidx.size(), cudaMemcpyHostToDevice, s));
    if (!H.hid.empty())
        CK(cudaMemcpyAsync(H.d_hid, H.hid.data(), sizeof(int) * H.hid.size(), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
}

static void free_distg(DistG& g, cudaStream_t s) {
    dfree(g.rp, s);
    dfree(g.ci, s);
    dfree(g.w, s);
    dfree(g.gid_b, s);
    if (g.own_plan) {
        dfree(g.H.sidx, s);
        dfree(g.H.sbuf, s);
        dfree(g.H.d_hid, s);
    }
    g = DistG{};
}

__global__ void k_gid(int nlo, int n, int nhi, int64_t gbeg, const int* __restrict__ hid, int* __restrict__ gid_b) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nlo + n + nhi; t += gridDim.x * blockDim.x) {
        const int rel = t - nlo;
        gid_b[t] = rel < 0 ? hid[t] : (rel < n ? (int)(gbeg + rel) : hid[t - n]);
    }
}

static void make_gid(DistG& g, cudaStream_t s) {
    const int tot = g.H.nlo + g.n + g.H.nhi;
    g.gid_b = dalloc<int>((size_t)tot + 1, s);
    k_gid<<<gridn(tot), kBlock, 0, s>>>(g.H.nlo, g.n, g.H.nhi, g.gbeg, g.H.d_hid, g.gid_b);
    ++g_launches;
    CK(cudaGetLastError());
}

// G_0: every off-diagonal entry of the level (halo columns included), multiplicity 1 (A5)
__global__ void k_gx0_count(int n, const int* __restrict__ rp, const int* __restrict__ ci, int* cnt) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int c = 0;
        for (int p = rp[i]; p < rp[i + 1]; ++p) c += (ci[p] != i);
        cnt[i] = c;
    }
}
__global__ void k_gx0_fill(int n, const int* __restrict__ rp, const int* __restrict__ ci, const int* __restrict__ grp,
                           int* __restrict__ gci, uint32_t* __restrict__ gw) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int q = grp[i];
        for (int p = rp[i]; p < rp[i + 1]; ++p)
            if (ci[p] != i) { gci[q] = ci[p]; gw[q] = 1u; ++q; }
    }
}

// ---- matching keys (docs/keys.md), on global ids
__device__ __forceinline__ uint64_t gx_sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
struct GKey {
    uint32_t w;
    uint64_t h;
    int lo, hi;
};
__device__ __forceinline__ GKey gx_key(uint32_t w, int a, int b, uint64_t salt) {
    GKey k;
    k.w = w;
    k.lo = a < b ? a : b;
    k.hi = a < b ? b : a;
    k.h = gx_sm64((((uint64_t)(uint32_t)k.lo) << 32 | (uint64_t)(uint32_t)k.hi) ^ salt);
    return k;
}
__device__ __forceinline__ bool gx_gt(const GKey& a, const GKey& b) {
    if (a.w != b.w) return a.w > b.w;
    if (a.h != b.h) return a.h > b.h;
    if (a.lo != b.lo) return a.lo > b.lo;
    return a.hi > b.hi;
}

// handshake step 1 (own free vertices): propose to the max-key free neighbour (own or halo); a free
// vertex without a free neighbour is settled (-2).  mate: -1 free, -2 settled, >= 0 global id.
__global__ void k_gx_propose(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                             const uint32_t* __restrict__ w, const int* __restrict__ gid, int* __restrict__ mate,
                             int* __restrict__ prop_g, int* __restrict__ prop_r, uint64_t salt, int* any) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        prop_g[v] = -1;
        if (mate[v] != -1) continue;
        const int gv = gid[v];
        GKey best{};
        int bu = 0;
        bool found = false;  // (relative indices of the halo below the block are negative)
        for (int p = rp[v]; p < rp[v + 1]; ++p) {
            const int u = ci[p];
            if (mate[u] != -1) continue;
            const GKey k = gx_key(w[p], gv, gid[u], salt);
            if (!found || gx_gt(k, best)) { best = k; bu = u; found = true; }
        }
        if (!found) {
            mate[v] = -2;
        } else {
            prop_g[v] = gid[bu];
            prop_r[v] = bu;
            *any = 1;
        }
    }
}

// handshake step 2: mutual proposals match (the halo's proposals were exchanged after step 1)
__global__ void k_gx_accept(int n, const int* __restrict__ gid, int* __restrict__ mate, int* __restrict__ mate_r,
                            const int* __restrict__ prop_g, const int* __restrict__ prop_r) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        if (mate[v] != -1 || prop_g[v] < 0) continue;
        const int u = prop_r[v];
        if (prop_g[u] == gid[v]) {
            mate[v] = prop_g[v];
            mate_r[v] = u;
        }
    }
}

// attach (A3) + leader (A4): leader global id, leader flag, attach target (relative)
__global__ void k_gx_leader(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                            const uint32_t* __restrict__ w, const int* __restrict__ gid, const int* __restrict__ mate,
                            uint64_t salt, int* __restrict__ isl, int* __restrict__ att_r) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int gv = gid[v], m = mate[v];
        att_r[v] = -1;
        if (m >= 0) {
            isl[v] = gv < m;
        } else if (rp[v + 1] > rp[v]) {
            GKey best{};
            int bu = 0;
            bool found = false;
            for (int p = rp[v]; p < rp[v + 1]; ++p) {
                const GKey k = gx_key(w[p], gv, gid[ci[p]], salt);
                if (!found || gx_gt(k, best)) { best = k; bu = ci[p]; found = true; }
            }
            isl[v] = 0;
            att_r[v] = bu;  // matched by maximality; its pair's aggregate (assign step 2)
        } else {
            isl[v] = 1;     // isolated: singleton
        }
    }
}

__global__ void k_gx_lid(int n, const int* __restrict__ isl, const int* __restrict__ rank, int off, int* __restrict__ lid) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        lid[v] = isl[v] ? off + rank[v] : -1;
}

// assign step 1: leaders, and matched vertices whose leader is the mate (its id was exchanged)
__global__ void k_gx_assign1(int n, const int* __restrict__ isl, const int* __restrict__ mate,
                             const int* __restrict__ mate_r, const int* __restrict__ lid, int* __restrict__ agg) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        agg[v] = isl[v] ? lid[v] : (mate[v] >= 0 ? lid[mate_r[v]] : -1);
}
// assign step 2: attached vertices take the aggregate of their (matched) attach target
__global__ void k_gx_assign2(int n, const int* __restrict__ att_r, int* __restrict__ agg) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        if (agg[v] < 0) agg[v] = agg[att_r[v]];
}

// one aggregation pass on a distributed pass graph: agg_b (base -nlo, own + halo filled) = global
// coarse ids; returns the coarse vertex blocks of all ranks (leader counts, prefix summed)
static std::vector<int64_t> gx_aggregate_pass(amg_hierarchy* h, const DistG& g, uint64_t salt, int* agg_b,
                                              int* rounds) {
    cudaStream_t s = h->s;
    Comm* c = h->comm;
    const int P = c->size, me = c->rank;
    const int n = g.n, nlo = g.H.nlo, tot = nlo + n + g.H.nhi;
    int* mate_b = dalloc<int>((size_t)tot + 1, s);
    int* propg_b = dalloc<int>((size_t)tot + 1, s);
    int* prop_r = dalloc<int>((size_t)n + 1, s);
    int* mate_r = dalloc<int>((size_t)n + 1, s);
    int* any = dalloc<int>(1, s);
    int* mate = mate_b + nlo;
    int* propg = propg_b + nlo;
    int* agg = agg_b + nlo;
    const int* gid = g.gid();
    CK(cudaMemsetAsync(mate_b, 0xff, sizeof(int) * (size_t)tot, s));
    const int gr = gridn(n);
    int r = 0;
    for (;;) {
        CK(cudaMemsetAsync(any, 0, sizeof(int), s));
        k_gx_propose<<<gr, kBlock, 0, s>>>(n, g.rp, g.ci, g.w, gid, mate, propg, prop_r, salt, any);
        ++g_launches;
        CK(cudaGetLastError());
        plan_xchg<int>(h, g.H, propg, propg);
        k_gx_accept<<<gr, kBlock, 0, s>>>(n, gid, mate, mate_r, propg, prop_r);
        ++g_launches;
        CK(cudaGetLastError());
        plan_xchg<int>(h, g.H, mate, mate);
        int ha = 0;
        CK(cudaMemcpyAsync(&ha, any, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const std::vector<int> anys = allgather_host<int>(c, ha, s);
        if (std::accumulate(anys.begin(), anys.end(), 0) == 0) break;
        if (++r > 30000) throw Error(AMG_E_SETUP, "matching did not terminate");
    }
    *rounds = r + 1;
    // attach + leaders, numbering by leader rank (own leaders in vertex order after the lower ranks')
    int* isl = dalloc<int>((size_t)n + 1, s);
    int* att_r = dalloc<int>((size_t)n + 1, s);
    int* lrank = dalloc<int>((size_t)n + 1, s);
    k_gx_leader<<<gr, kBlock, 0, s>>>(n, g.rp, g.ci, g.w, gid, mate, salt, isl, att_r);
    ++g_launches;
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(isl + n, 0, sizeof(int), s));
    const int nlead = (int)scan_counts(isl, lrank, n, s);
    const std::vector<int> nl = allgather_host<int>(c, nlead, s);
    std::vector<int64_t> coffs(P + 1, 0);
    for (int q = 0; q < P; ++q) coffs[q + 1] = coffs[q] + nl[q];
    int* lid_b = propg_b;  // reuse: leader ids with halo slots
    k_gx_lid<<<gr, kBlock, 0, s>>>(n, isl, lrank, (int)coffs[me], lid_b + nlo);
    ++g_launches;
    CK(cudaGetLastError());
    plan_xchg<int>(h, g.H, lid_b + nlo, lid_b + nlo);
    k_gx_assign1<<<gr, kBlock, 0, s>>>(n, isl, mate, mate_r, lid_b + nlo, agg);
    ++g_launches;
    CK(cudaGetLastError());
    plan_xchg<int>(h, g.H, agg, agg);
    k_gx_assign2<<<gr, kBlock, 0, s>>>(n, att_r, agg);
    ++g_launches;
    CK(cudaGetLastError());
    plan_xchg<int>(h, g.H, agg, agg);  // halo slots hold the final ids too
    dfree(mate_b, s); dfree(propg_b, s); dfree(prop_r, s); dfree(mate_r, s); dfree(any, s);
    dfree(isl, s); dfree(att_r, s); dfree(lrank, s);
    return coffs;
}

// ---- (I, J, value) triples routed to the owner of I, merged in order
struct Triples {
    int64_t m = 0;
    int* I = nullptr;
    int* J = nullptr;
    double* V = nullptr;
};
static void free_triples(Triples& t, cudaStream_t s) {
    dfree(t.I, s); dfree(t.J, s); dfree(t.V, s);
    t = Triples{};
}

__device__ __forceinline__ int owner_of(const int64_t* offs, int P, int64_t x) {
    int lo = 0, hi = P;  // largest q with offs[q] <= x
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (offs[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}
__global__ void k_tr_dest(int64_t m, const int* __restrict__ I, const int64_t* __restrict__ offs, int P,
                          int* __restrict__ dest, int* __restrict__ cnt) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const int q = owner_of(offs, P, I[t]);
        dest[t] = q;
        atomicAdd(cnt + q, 1);
    }
}
__global__ void k_iota64(int64_t m, int* __restrict__ o) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) o[t] = (int)t;
}
__global__ void k_tr_gather(int64_t m, const int* __restrict__ idx, const int* __restrict__ I, const int* __restrict__ J,
                            const double* __restrict__ V, int* __restrict__ I2, int* __restrict__ J2,
                            double* __restrict__ V2) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const int k = idx[t];
        I2[t] = I[k];
        J2[t] = J[k];
        V2[t] = V[k];
    }
}

// route every triple to the owner of I (stable: each source's triples keep their order); the result
// holds the triples of the own rows, sources in rank order (= increasing fine row order)
static Triples route_triples(amg_hierarchy* h, Triples& T, const std::vector<int64_t>& offs) {
    cudaStream_t s = h->s;
    Comm* c = h->comm;
    const int P = c->size, me = c->rank;
    const int64_t m = T.m;
    int64_t* doffs = dalloc<int64_t>(P + 1, s);
    CK(cudaMemcpyAsync(doffs, offs.data(), sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice, s));
    int* dest = dalloc<int>((size_t)m + 1, s);
    int* cnt = dalloc<int>((size_t)P + 1, s);
    CK(cudaMemsetAsync(cnt, 0, sizeof(int) * (P + 1), s));
    if (m) k_tr_dest<<<gridn(m), kBlock, 0, s>>>(m, T.I, doffs, P, dest, cnt);
    ++g_launches;
    CK(cudaGetLastError());
    // stable sort by destination
    int* idx = dalloc<int>((size_t)m + 1, s);
    int* idx2 = dalloc<int>((size_t)m + 1, s);
    int* dest2 = dalloc<int>((size_t)m + 1, s);
    if (m) {
        k_iota64<<<gridn(m), kBlock, 0, s>>>(m, idx);
        ++g_launches;
        size_t tb = 0;
        int bits = 1;
        while ((1 << bits) < P) ++bits;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dest, dest2, idx, idx2, (int)m, 0, bits, s));
        void* tmp = dalloc<char>(tb, s);
        CK(cub::DeviceRadixSort::SortPairs(tmp, tb, dest, dest2, idx, idx2, (int)m, 0, bits, s));
        dfree(tmp, s);
    }
    Triples S;
    S.m = m;
    S.I = dalloc<int>((size_t)m + 1, s);
    S.J = dalloc<int>((size_t)m + 1, s);
    S.V = dalloc<double>((size_t)m + 1, s);
    if (m) k_tr_gather<<<gridn(m), kBlock, 0, s>>>(m, idx2, T.I, T.J, T.V, S.I, S.J, S.V);
    ++g_launches;
    CK(cudaGetLastError());
    std::vector<int> hc(P + 1);
    CK(cudaMemcpyAsync(hc.data(), cnt, sizeof(int) * (P + 1), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(doffs, s); dfree(dest, s); dfree(cnt, s); dfree(idx, s); dfree(idx2, s); dfree(dest2, s);
    std::vector<int> cntv(hc.begin(), hc.begin() + P);
    const std::vector<int> M = allgather_vec_host(c, cntv, s);  // M[r * P + q]: r sends q
    std::vector<int64_t> soff(P + 1, 0), roff(P + 1, 0);
    for (int q = 0; q < P; ++q) {
        soff[q + 1] = soff[q] + cntv[q];
        roff[q + 1] = roff[q] + M[(size_t)q * P + me];
    }
    Triples R;
    R.m = roff[P];
    R.I = dalloc<int>((size_t)R.m + 1, s);
    R.J = dalloc<int>((size_t)R.m + 1, s);
    R.V = dalloc<double>((size_t)R.m + 1, s);
    const int64_t own = cntv[me];
    if (own) {
        CK(cudaMemcpyAsync(R.I + roff[me], S.I + soff[me], sizeof(int) * own, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(R.J + roff[me], S.J + soff[me], sizeof(int) * own, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(R.V + roff[me], S.V + soff[me], sizeof(double) * own, cudaMemcpyDeviceToDevice, s));
    }
    std::vector<P2P> ss, rr;
    for (int q = 0; q < P; ++q) {
        if (q == me) continue;
        const int64_t sc = cntv[q], rc = M[(size_t)q * P + me];
        if (sc) {
            ss.push_back({q, S.I + soff[q], sizeof(int) * (size_t)sc});
            ss.push_back({q, S.J + soff[q], sizeof(int) * (size_t)sc});
            ss.push_back({q, S.V + soff[q], sizeof(double) * (size_t)sc});
        }
        if (rc) {
            rr.push_back({q, R.I + roff[q], sizeof(int) * (size_t)rc});
            rr.push_back({q, R.J + roff[q], sizeof(int) * (size_t)rc});
            rr.push_back({q, R.V + roff[q], sizeof(double) * (size_t)rc});
        }
    }
    c->sendrecv(ss, rr, s);
    CK(cudaStreamSynchronize(s));
    free_triples(S, s);
    return R;
}

__global__ void k_tr_key(int64_t m, const int* __restrict__ I, const int* __restrict__ J, int64_t cbeg,
                         unsigned long long* __restrict__ key) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
        key[t] = ((unsigned long long)(uint32_t)(I[t] - cbeg) << 32) | (unsigned long long)(uint32_t)J[t];
}
__global__ void k_tr_heads(int64_t m, const unsigned long long* __restrict__ key, int* __restrict__ head) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
        head[t] = (t == 0 || key[t] != key[t - 1]) ? 1 : 0;
}
// one thread per distinct (I, J): its triples in their (stable) order, summed sequentially from 0
__global__ void k_tr_sum(int64_t m, const unsigned long long* __restrict__ key, const int* __restrict__ idx,
                         const int* __restrict__ head, const int* __restrict__ pos, const double* __restrict__ V,
                         int* __restrict__ row, int* __restrict__ col, double* __restrict__ val) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        if (!head[t]) continue;
        const unsigned long long k = key[t];
        double acc = 0.0;
        for (int64_t u = t; u < m && key[u] == k; ++u) acc += V[idx[u]];
        const int e = pos[t];
        row[e] = (int)(k >> 32);
        col[e] = (int)(uint32_t)(k & 0xffffffffu);
        val[e] = acc;
    }
}
__global__ void k_row_count(int64_t e, const int* __restrict__ row, int* __restrict__ cnt) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < e; t += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + row[t], 1);
}

// merged CSR of the own coarse rows [cbeg, cbeg + nrows): rp (device), global columns, values
struct MergedRows {
    int64_t nnz = 0;
    int* rp = nullptr;
    int* colg = nullptr;
    double* val = nullptr;
};
static MergedRows merge_triples(amg_hierarchy* h, const Triples& R, int64_t cbeg, int nrows) {
    cudaStream_t s = h->s;
    const int64_t m = R.m;
    unsigned long long* key = dalloc<unsigned long long>((size_t)m + 1, s);
    unsigned long long* key2 = dalloc<unsigned long long>((size_t)m + 1, s);
    int* idx = dalloc<int>((size_t)m + 1, s);
    int* idx2 = dalloc<int>((size_t)m + 1, s);
    int* head = dalloc<int>((size_t)m + 1, s);
    int* pos = dalloc<int>((size_t)m + 1, s);
    MergedRows out;
    out.rp = dalloc<int>((size_t)nrows + 1, s);
    int* cnt = dalloc<int>((size_t)nrows + 1, s);
    CK(cudaMemsetAsync(cnt, 0, sizeof(int) * ((size_t)nrows + 1), s));
    int64_t e = 0;
    if (m) {
        k_tr_key<<<gridn(m), kBlock, 0, s>>>(m, R.I, R.J, cbeg, key);
        k_iota64<<<gridn(m), kBlock, 0, s>>>(m, idx);
        g_launches += 2;
        size_t tb = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, idx, idx2, (int)m, 0, 64, s));
        void* tmp = dalloc<char>(tb, s);
        CK(cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, idx, idx2, (int)m, 0, 64, s));  // stable
        dfree(tmp, s);
        k_tr_heads<<<gridn(m), kBlock, 0, s>>>(m, key2, head);
        ++g_launches;
        CK(cudaMemsetAsync(head + m, 0, sizeof(int), s));
        e = scan_counts(head, pos, (int)m, s);
    }
    out.nnz = e;
    out.colg = dalloc<int>((size_t)e + 8, s);
    out.val = dalloc<double>((size_t)e + 8, s);
    int* row = dalloc<int>((size_t)e + 1, s);
    if (m) {
        k_tr_sum<<<gridn(m), kBlock, 0, s>>>(m, key2, idx2, head, pos, R.V, row, out.colg, out.val);
        k_row_count<<<gridn(e), kBlock, 0, s>>>(e, row, cnt);
        g_launches += 2;
    }
    scan_counts(cnt, out.rp, nrows, s);
    CK(cudaGetLastError());
    dfree(key, s); dfree(key2, s); dfree(idx, s); dfree(idx2, s); dfree(head, s); dfree(pos, s);
    dfree(row, s); dfree(cnt, s);
    return out;
}

// global column -> relative (own: c - cbeg; halo: position in the sorted halo ids hid)
__global__ void k_glob_to_rel(int64_t m, const int* __restrict__ cg, int64_t cbeg, int n, const int* __restrict__ hid,
                              int nh, int nlo, int* __restrict__ out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const int c = cg[t];
        int r;
        if ((int64_t)c >= cbeg && (int64_t)c < cbeg + n) {
            r = (int)(c - cbeg);
        } else {
            const int k = lower_bound_i(hid, nh, c);
            r = k < nlo ? k - nlo : n + (k - nlo);
        }
        out[t] = r;
    }
}
__global__ void k_not_own(int64_t m, const int* __restrict__ cg, int64_t cbeg, int n, int* __restrict__ out,
                          int* __restrict__ cnt) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const int c = cg[t];
        if ((int64_t)c < cbeg || (int64_t)c >= cbeg + n) out[atomicAdd(cnt, 1)] = c;
    }
}

// the halo ids (sorted, unique) of merged rows' global columns plus `extra` (device, global ids)
static std::vector<int> halo_ids_of(amg_hierarchy* h, const int* colg, int64_t m, const int* extra, int64_t me_,
                                    int64_t cbeg, int n) {
    cudaStream_t s = h->s;
    int* cand = dalloc<int>((size_t)(m + me_) + 1, s);
    int* cnt = dalloc<int>(1, s);
    CK(cudaMemsetAsync(cnt, 0, sizeof(int), s));
    if (m) k_not_own<<<gridn(m), kBlock, 0, s>>>(m, colg, cbeg, n, cand, cnt);
    if (me_) k_not_own<<<gridn(me_), kBlock, 0, s>>>(me_, extra, cbeg, n, cand, cnt);
    g_launches += 2;
    CK(cudaGetLastError());
    int hc = 0;
    CK(cudaMemcpyAsync(&hc, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<int> out = sorted_unique(cand, hc, s);
    dfree(cand, s);
    dfree(cnt, s);
    return out;
}

// triples of a distributed pass graph's quotient: (agg v, agg u, w) for every edge v-u between
// different aggregates (the diagonal of the quotient is dropped, A5)
__global__ void k_tr_graph(int n, const int* __restrict__ rp, const int* __restrict__ ci, const uint32_t* __restrict__ w,
                           const int* __restrict__ agg, int* __restrict__ cnt, int* __restrict__ I,
                           int* __restrict__ J, double* __restrict__ V, int pass) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int a = agg[v];
        if (pass == 0) {
            int c = 0;
            for (int p = rp[v]; p < rp[v + 1]; ++p) c += (agg[ci[p]] != a);
            cnt[v] = c;
        } else {
            int q = cnt[v];
            for (int p = rp[v]; p < rp[v + 1]; ++p) {
                const int b = agg[ci[p]];
                if (b == a) continue;
                I[q] = a;
                J[q] = b;
                V[q] = (double)w[p];
                ++q;
            }
        }
    }
}
// Galerkin triples: (agg i, agg j, a_ij) for every stored entry, in (row, CSR position) order
__global__ void k_tr_galerkin(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                              const double* __restrict__ v, const int* __restrict__ agg, int* __restrict__ I,
                              int* __restrict__ J, double* __restrict__ V) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int a = agg[i];
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            I[p] = a;
            J[p] = agg[ci[p]];
            V[p] = v[p];
        }
    }
}
__global__ void k_to_u32(int64_t m, const double* __restrict__ a, uint32_t* __restrict__ b) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
        b[t] = (uint32_t)a[t];
}

// quotient of a distributed pass graph by its aggregation (global ids in agg_b, base -nlo)
static DistG gx_quotient(amg_hierarchy* h, const DistG& g, const int* agg_b, const std::vector<int64_t>& coffs) {
    cudaStream_t s = h->s;
    const int me = h->comm->rank;
    const int n = g.n;
    const int* agg = agg_b + g.H.nlo;
    int* cnt = dalloc<int>((size_t)n + 1, s);
    int* off = dalloc<int>((size_t)n + 1, s);
    k_tr_graph<<<gridn(n), kBlock, 0, s>>>(n, g.rp, g.ci, g.w, agg, cnt, nullptr, nullptr, nullptr, 0);
    ++g_launches;
    CK(cudaMemsetAsync(cnt + n, 0, sizeof(int), s));
    Triples T;
    T.m = scan_counts(cnt, off, n, s);
    T.I = dalloc<int>((size_t)T.m + 1, s);
    T.J = dalloc<int>((size_t)T.m + 1, s);
    T.V = dalloc<double>((size_t)T.m + 1, s);
    k_tr_graph<<<gridn(n), kBlock, 0, s>>>(n, g.rp, g.ci, g.w, agg, off, T.I, T.J, T.V, 1);
    ++g_launches;
    CK(cudaGetLastError());
    dfree(cnt, s);
    dfree(off, s);
    Triples R = route_triples(h, T, coffs);
    free_triples(T, s);
    DistG q;
    q.gbeg = coffs[me];
    q.n = (int)(coffs[me + 1] - coffs[me]);
    q.offs = coffs;
    MergedRows M = merge_triples(h, R, q.gbeg, q.n);
    free_triples(R, s);
    const std::vector<int> hid = halo_ids_of(h, M.colg, M.nnz, nullptr, 0, q.gbeg, q.n);
    std::vector<std::vector<int>> req;
    plan_halo(q.gbeg, q.n, coffs, me, hid, q.H, req);
    finish_plan_tmp(h, q.H, q.gbeg, q.n, req);
    q.own_plan = true;
    q.nnz = M.nnz;
    q.rp = M.rp;
    q.ci = dalloc<int>((size_t)M.nnz + 8, s);
    q.w = dalloc<uint32_t>((size_t)M.nnz + 8, s);
    if (M.nnz) {
        k_glob_to_rel<<<gridn(M.nnz), kBlock, 0, s>>>(M.nnz, M.colg, q.gbeg, q.n, q.H.d_hid, (int)hid.size(), q.H.nlo, q.ci);
        k_to_u32<<<gridn(M.nnz), kBlock, 0, s>>>(M.nnz, M.val, q.w);
        g_launches += 2;
    }
    CK(cudaGetLastError());
    dfree(M.colg, s);
    dfree(M.val, s);
    make_gid(q, s);
    return q;
}

// host lookup of the next pass's aggregate of every own fine vertex's current coarse vertex
static void gx_compose(amg_hierarchy* h, std::vector<int>& cur, const std::vector<int64_t>& offs_t,
                       const int* agg_t_dev, int n_t) {
    cudaStream_t s = h->s;
    Comm* c = h->comm;
    const int P = c->size, me = c->rank;
    std::vector<int> at((size_t)n_t + 1);
    if (n_t) CK(cudaMemcpyAsync(at.data(), agg_t_dev, sizeof(int) * n_t, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    auto owner = [&](int64_t x) { return (int)(std::upper_bound(offs_t.begin(), offs_t.end(), x) - offs_t.begin()) - 1; };
    std::vector<std::vector<int>> req(P);
    for (int x : cur) {
        const int q = owner(x);
        if (q != me) req[q].push_back(x);
    }
    for (auto& r : req) {
        std::sort(r.begin(), r.end());
        r.erase(std::unique(r.begin(), r.end()), r.end());
    }
    const std::vector<std::vector<int>> got = alltoallv_int(c, req, s);
    std::vector<std::vector<int>> ans(P);
    for (int q = 0; q < P; ++q) {
        if (q == me) continue;
        for (int x : got[q]) ans[q].push_back(at[(size_t)(x - offs_t[me])]);
    }
    const std::vector<std::vector<int>> back = alltoallv_int(c, ans, s);
    for (int& x : cur) {
        const int q = owner(x);
        if (q == me) {
            x = at[(size_t)(x - offs_t[me])];
        } else {
            const auto& r = req[q];
            const size_t k = (size_t)(std::lower_bound(r.begin(), r.end(), x) - r.begin());
            x = back[q][k];
        }
    }
}

__global__ void k_restrict_x(int nc, const int* __restrict__ aptr, const int* __restrict__ perm, int n,
                             const double* __restrict__ r, const double* __restrict__ rb, double* __restrict__ rH) {
    for (int I = blockIdx.x * blockDim.x + threadIdx.x; I < nc; I += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int t = aptr[I]; t < aptr[I + 1]; ++t) {
            const int e = perm[t];
            s += e < n ? r[e] : rb[e - n];
        }
        rH[I] = s;
    }
}

void restrict_global(amg_hierarchy* h, int l, const double* r, double* rH) {
    Level& Lv = h->lev[l];
    plan_xchg<double>(h, Lv.XP, r, Lv.RB);
    launch_k(k_restrict_x, dim3(gridn(Lv.nc)), dim3(kBlock), 0, h->s, Lv.nc, (const int*)Lv.aptr_x,
             (const int*)Lv.perm_x, Lv.A.n, r, (const double*)Lv.RB, rH);
    CK(cudaGetLastError());
    ++g_launches;
}

__global__ void k_tr_ext(int m, const int* __restrict__ aggI, int64_t cbeg, const int* __restrict__ ext,
                         int* __restrict__ key, int* __restrict__ val) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
        key[t] = (int)(aggI[t] - cbeg);
        val[t] = ext[t];
    }
}
__global__ void k_aptr_from_sorted(int m, int nc, const int* __restrict__ key, int* __restrict__ aptr) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= m; t += gridDim.x * blockDim.x) {
        const int a = t == 0 ? -1 : key[t - 1];
        const int b = t == m ? nc : key[t];
        for (int I = a + 1; I <= b; ++I) aptr[I] = t;
    }
}

// Level l (row-partitioned) aggregated globally: p matching passes with halo rounds, the coarse
// level's rows (Galerkin triples routed to the owners), the restriction export plan.
static void gx_build_level(amg_hierarchy* h, int l) {
    cudaStream_t s = h->s;
    Comm* c = h->comm;
    const int P = c->size, me = c->rank;
    Level& Lv = h->lev[l];
    const int n = Lv.A.n, nlo = Lv.H.nlo, nhi = Lv.H.nhi;
    // G_0 on the level's own rows (halo columns kept), the level's halo plan
    DistG g;
    g.n = n;
    g.gbeg = Lv.gbeg;
    g.offs = Lv.offs;
    g.H = Lv.H;
    g.own_plan = false;
    {
        int* cnt = dalloc<int>((size_t)n + 1, s);
        CK(cudaMemsetAsync(cnt + n, 0, sizeof(int), s));
        k_gx0_count<<<gridn(n), kBlock, 0, s>>>(n, Lv.A.rp, Lv.A.ci, cnt);
        g.rp = dalloc<int>((size_t)n + 1, s);
        g.nnz = scan_counts(cnt, g.rp, n, s);
        dfree(cnt, s);
        g.ci = dalloc<int>((size_t)g.nnz + 1, s);
        g.w = dalloc<uint32_t>((size_t)g.nnz + 1, s);
        k_gx0_fill<<<gridn(n), kBlock, 0, s>>>(n, Lv.A.rp, Lv.A.ci, g.rp, g.ci, g.w);
        g_launches += 2;
        CK(cudaGetLastError());
        make_gid(g, s);
    }
    std::vector<int> cur(n);
    for (int v = 0; v < n; ++v) cur[v] = (int)(Lv.gbeg + v);
    std::vector<int64_t> coffs;
    for (int t = 0; t < h->p; ++t) {
        const uint64_t salt = host_sm64(h->opt.seed ^ (((uint64_t)l << 8) ^ (uint64_t)t));
        int* agg_b = dalloc<int>((size_t)g.H.nlo + g.n + g.H.nhi + 1, s);
        coffs = gx_aggregate_pass(h, g, salt, agg_b, &Lv.rounds[t]);
        gx_compose(h, cur, g.offs, agg_b + g.H.nlo, g.n);
        if (t + 1 < h->p) {
            DistG q = gx_quotient(h, g, agg_b, coffs);
            free_distg(g, s);
            g = q;
        }
        dfree(agg_b, s);
    }
    free_distg(g, s);
    if (coffs[P] >= Lv.nglob) throw Error(AMG_E_SETUP, "coarsening stagnated (n_{l+1} = n_l)");
    const int64_t cbeg = coffs[me];
    const int nc = (int)(coffs[me + 1] - coffs[me]);
    Lv.gx = true;
    Lv.nc = nc;
    // global coarse id of every own and halo fine row
    int* aggg_b = dalloc<int>((size_t)nlo + n + nhi + 8, s);
    int* aggg = aggg_b + nlo;
    CK(cudaMemcpyAsync(aggg, cur.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    halo_exchange_t<int>(h, Lv, aggg);
    Lv.aggG = halloc<int>(h, (size_t)n + 1);
    CK(cudaMemcpyAsync(Lv.aggG, aggg, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
    // Galerkin: triples of every stored entry, routed to the owner of the row's aggregate
    Triples T;
    T.m = Lv.A.nnz;
    T.I = dalloc<int>((size_t)T.m + 1, s);
    T.J = dalloc<int>((size_t)T.m + 1, s);
    T.V = dalloc<double>((size_t)T.m + 1, s);
    k_tr_galerkin<<<gridn(n), kBlock, 0, s>>>(n, Lv.A.rp, Lv.A.ci, Lv.A.v, aggg, T.I, T.J, T.V);
    ++g_launches;
    CK(cudaGetLastError());
    Triples R = route_triples(h, T, coffs);
    free_triples(T, s);
    MergedRows M = merge_triples(h, R, cbeg, nc);
    free_triples(R, s);
    // coarse halo: the merged rows' remote columns + the remote aggregates of own fine rows (read by
    // the prolongation)
    const std::vector<int> hid = halo_ids_of(h, M.colg, M.nnz, Lv.aggG, n, cbeg, nc);
    Level& Cn = h->lev[l + 1];
    Cn.dist = true;
    Cn.gbeg = cbeg;
    Cn.nglob = coffs[P];
    Cn.offs = coffs;
    std::vector<std::vector<int>> creq;
    plan_halo(cbeg, nc, coffs, me, hid, Cn.H, creq);
    Cn.A.n = nc;
    Cn.A.nnz = M.nnz;
    Cn.A.rp = M.rp;
    Cn.A.v = M.val;
    Cn.A.ci = dalloc<int>((size_t)M.nnz + 8, s);
    h->L = l + 2;
    finish_halo(h, Cn, creq);
    if (M.nnz)
        k_glob_to_rel<<<gridn(M.nnz), kBlock, 0, s>>>(M.nnz, M.colg, cbeg, nc, Cn.H.d_hid, (int)hid.size(), Cn.H.nlo,
                                                      Cn.A.ci);
    ++g_launches;
    CK(cudaGetLastError());
    dfree(M.colg, s);
    // restriction export plan: own fine rows of remote aggregates go to the owners (increasing row)
    std::vector<int> hagg(n);
    CK(cudaMemcpyAsync(hagg.data(), Lv.aggG, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    auto owner = [&](int64_t x) { return (int)(std::upper_bound(coffs.begin(), coffs.end(), x) - coffs.begin()) - 1; };
    std::vector<std::vector<int>> out_rows(P), out_ids(P);
    for (int i = 0; i < n; ++i) {
        const int q = owner(hagg[i]);
        if (q != me) {
            out_rows[q].push_back(i);
            out_ids[q].push_back(hagg[i]);
        }
    }
    const std::vector<std::vector<int>> in_ids = alltoallv_int(c, out_ids, s);  // aggregate of each received member
    Halo& X = Lv.XP;
    std::vector<int> sidx;
    for (int q = 0; q < P; ++q) {
        if (q == me || out_rows[q].empty()) continue;
        X.send.push_back({q, (int)sidx.size(), (int)out_rows[q].size()});
        sidx.insert(sidx.end(), out_rows[q].begin(), out_rows[q].end());
    }
    X.nsend = (int)sidx.size();
    X.sidx = halloc<int>(h, sidx.size() + 1);
    X.sbuf = halloc<double>(h, sidx.size() + 1);
    if (!sidx.empty()) CK(cudaMemcpyAsync(X.sidx, sidx.data(), sizeof(int) * sidx.size(), cudaMemcpyHostToDevice, s));
    // extended member list in increasing global row order: received from lower ranks, own rows of own
    // aggregates, received from higher ranks; ext index < n: own row, >= n: RB slot
    std::vector<int> ext_agg, ext_idx;
    int nrb = 0;
    auto take_recv = [&](int q) {
        if (in_ids[q].empty()) return;
        X.recv.push_back({q, nrb, (int)in_ids[q].size()});
        for (int a : in_ids[q]) {
            ext_agg.push_back(a);
            ext_idx.push_back(n + nrb++);
        }
    };
    for (int q = 0; q < me; ++q) take_recv(q);
    for (int i = 0; i < n; ++i)
        if (owner(hagg[i]) == me) {
            ext_agg.push_back(hagg[i]);
            ext_idx.push_back(i);
        }
    for (int q = me + 1; q < P; ++q) take_recv(q);
    Lv.RB = halloc<double>(h, (size_t)nrb + 1);
    const int me_ = (int)ext_agg.size();
    int* dA = dalloc<int>((size_t)me_ + 1, s);
    int* dE = dalloc<int>((size_t)me_ + 1, s);
    CK(cudaMemcpyAsync(dA, ext_agg.data(), sizeof(int) * me_, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dE, ext_idx.data(), sizeof(int) * me_, cudaMemcpyHostToDevice, s));
    int* k1 = dalloc<int>((size_t)me_ + 1, s);
    int* v1 = dalloc<int>((size_t)me_ + 1, s);
    int* k2 = dalloc<int>((size_t)me_ + 1, s);
    Lv.perm_x = halloc<int>(h, (size_t)me_ + 1);
    Lv.aptr_x = halloc<int>(h, (size_t)nc + 1);
    if (me_) {
        k_tr_ext<<<gridn(me_), kBlock, 0, s>>>(me_, dA, cbeg, dE, k1, v1);
        size_t tb = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k1, k2, v1, Lv.perm_x, me_, 0, 32, s));
        void* tmp = dalloc<char>(tb, s);
        CK(cub::DeviceRadixSort::SortPairs(tmp, tb, k1, k2, v1, Lv.perm_x, me_, 0, 32, s));  // stable
        dfree(tmp, s);
    }
    k_aptr_from_sorted<<<gridn(me_ + 1), kBlock, 0, s>>>(me_, nc, k2, Lv.aptr_x);
    g_launches += 2;
    CK(cudaGetLastError());
    dfree(dA, s); dfree(dE, s); dfree(k1, s); dfree(v1, s); dfree(k2, s); dfree(aggg_b, s);
    CK(cudaStreamSynchronize(s));
}

// prolongation indices of the globally aggregated levels, once the partition of every level is
// known: the coarse relative index (the coarse level is row-partitioned: own rows, or the halo slot
// of a remote aggregate) or the global id (the coarse level is replicated)
__global__ void k_gx_prolong_index(int n, const int* __restrict__ aggG, int64_t cbeg, int nc, const int* __restrict__ hid,
                                   int nh, int nlo, int rel, int* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int G = aggG[i];
        if (!rel) { out[i] = G; continue; }
        int r;
        if ((int64_t)G >= cbeg && (int64_t)G < cbeg + nc) {
            r = (int)(G - cbeg);
        } else {
            const int k = lower_bound_i(hid, nh, G);
            r = k < nlo ? k - nlo : nc + (k - nlo);
        }
        out[i] = r;
    }
}

static void gx_finish(amg_hierarchy* h) {
    cudaStream_t s = h->s;
    for (int l = 0; l + 1 < h->L; ++l) {
        Level& Lv = h->lev[l];
        if (!Lv.gx) continue;
        const Level& C = h->lev[l + 1];
        Lv.agg = halloc<int>(h, (size_t)Lv.A.n + 1);
        k_gx_prolong_index<<<gridn(Lv.A.n), kBlock, 0, s>>>(Lv.A.n, Lv.aggG, C.gbeg, C.A.n, C.H.d_hid,
                                                            (int)C.H.hid.size(), C.H.nlo, C.dist ? 1 : 0, Lv.agg);
        ++g_launches;
        CK(cudaGetLastError());
    }
}

static void gx_warm(amg_hierarchy* h) {
    for (int l = 0; l < h->g; ++l) {
        Level& Lv = h->lev[l];
        if (Lv.gx && Lv.RES) plan_xchg<double>(h, Lv.XP, Lv.RES, Lv.RB);
    }
}

}  // namespace amg
