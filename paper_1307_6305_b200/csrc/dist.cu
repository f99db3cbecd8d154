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
    finish_build(h);
    warm_comm(h);
}

void warm_comm(amg_hierarchy* h) {
    for (int l = 0; l < h->g; ++l)
        if (h->lev[l].X) halo_exchange(h, l, h->lev[l].X);
    dot_allreduce(h, {h->osc + 2 * kMaxWin + 4});
    for (int l = 0; l < h->g; ++l)  // the split passes' message pattern (same messages, other stream)
        if (h->lev[l].X && h->lev[l].split) {
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
