// hierarchy.h -- the handle behind amg_handle (include/amg.h): levels, workspaces, the row partition
// of the distributed levels, and the host-side entry points shared by driver.cu (single GPU, the
// replicated levels, the solve schedule) and dist.cu (row-partitioned setup, halo exchange, the
// batched dot allreduce).  Internal; not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "../../include/amg.h"
#include "amg_internal.h"

namespace amg {

// ------------------------------------------------------------------ row partition
// A row-partitioned level stores its own rows [gbeg, gbeg + n) of nglob.  Columns are RELATIVE to
// the first own row: own columns in [0, n), the halo below in [-nlo, 0) and above in [n, n + nhi),
// both in increasing global order (blocks are contiguous in rank order, so the map global ->
// relative is monotone: CSR rows stay sorted and the Galerkin summation order is the global one).
// Every vector of the level is laid out [pad | lower halo | own | upper halo] so an SpMV input x
// (pointer to its first own element) is read as x[col] for any column.
struct Seg {
    int peer, off, cnt;  // recv: off = relative column of the first element; send: offset into sidx
};
struct Halo {
    int nlo = 0, nhi = 0;
    std::vector<int> hid;        // sorted global ids of the halo columns (nlo below, then nhi above)
    int* d_hid = nullptr;        // device copy of hid
    std::vector<Seg> recv, send;
    int nsend = 0;
    int* sidx = nullptr;         // device [nsend]: own row of each element sent (send segments concatenated)
    double* sbuf = nullptr;      // device [nsend] doubles (also carries int payloads at setup)
};

struct Level {
    Csr A;
    Tiles T;
    Sell S;
    SpOp op;  // the format the SpMV-class kernels use on this level
    double lambda1 = 0, kappa = 0;
    double alpha[kMaxDeg + 1] = {}, beta[kMaxDeg + 1] = {};
    int nc = 0;
    int* agg = nullptr;
    int* perm = nullptr;
    int* aptr = nullptr;
    int rounds[kMaxDeg] = {};
    // workspaces (pointers to the first own element)
    double *X = nullptr, *XA = nullptr, *RES = nullptr;  // B_l
    double *RHO = nullptr, *E = nullptr;                  // written / read by the parent level
    double *Z = nullptr, *D = nullptr, *Q = nullptr;      // inner FCG (nu slots, stride ld)
    double* sc = nullptr;                                 // dq[kMaxWin], dr[kMaxWin], c[kMaxWin]
    // partition
    bool dist = false;           // row-partitioned (levels < g of a distributed handle)
    int64_t gbeg = 0, nglob = 0; // own rows [gbeg, gbeg + A.n) of nglob (nglob = A.n when not partitioned)
    int64_t nnz_glob = 0;        // nnz of the whole level (sum over ranks)
    std::vector<int64_t> offs;   // block offsets of all ranks (P+1): the partition this level's rows came in
    Halo H;
    int lo_pad = 0;              // own element offset inside a vector allocation (>= H.nlo, multiple of 4)
    // global (non-decoupled) aggregation on a row-partitioned level (amg_options.global_agg, SURVEY
    // 8(f) item 4): aggregates may span ranks and are owned by the rank of their leader
    bool gx = false;
    int* aggG = nullptr;         // own rows: global coarse id (export); agg holds the prolongation index
    Halo XP;                     // restriction export plan: own rows of remote aggregates -> their owners
    double* RB = nullptr;        // received fine residual values of remote members of own aggregates
    int* perm_x = nullptr;       // own aggregates' members in increasing global row order: < n own row,
    int* aptr_x = nullptr;       //   >= n: RB[perm - n]
    // halo overlap: the SELL slices that read no halo column (interior, one range) run while the halo
    // is in flight; the boundary slices (the ranges around it) after it has arrived
    bool split = false;
    SpOp op_int, op_lo, op_hi;   // slice views: interior, boundary before it, boundary after it
    int ld = 0;                  // vector slot stride (lo_pad + n + nhi, rounded up to 4)
};

}  // namespace amg

struct amg_hierarchy {
    cudaStream_t s = nullptr;     // this handle's library stream (stream_acquire / stream_release)
    int dev = 0;                  // device the handle was created on
    cudaStream_t user = nullptr;
    int L = 0, m = 0, p = 0;
    bool singular = false;
    amg_options opt{};
    amg::Level lev[amg::kMaxLevels];
    double* Minv = nullptr;
    double* Bd = nullptr;   // dense B_{L-2} (k_dense.cu) when n_{L-2} <= opt.dense_b_rows
    int dense_l = -1;       // its level (-1: none)
    // outer FCG (level 0 own rows)
    int n = 0, W = 5;
    double *b = nullptr, *x = nullptr, *r = nullptr, *Z = nullptr, *D = nullptr, *Q = nullptr;
    double* osc = nullptr;  // dq[kMaxWin], c[kMaxWin], dr, rr, bb, tmp, rr_true
    double* alph = nullptr;  // alpha_j of the window positions whose x update is still pending (deferred)
    int* xold = nullptr;     // device flag: the last window slot's x update is pending (fused flush)
    bool xf = false;         // x updates flushed inside the last position's direction kernel
    int* flag = nullptr;
    double* hsc = nullptr;  // pinned host mirror: rr, flag
    amg::DotScratch ds;
    int nu_ws = 0;          // nu the inner workspaces are sized for
    int l_tail = 0;         // first level run by the coarse-tail kernel (L = none)
    int tail_smem = 0;      // doubles of shared memory the tail kernel keeps its vectors in (0 = global)
    amg::TLevel* d_tlev = nullptr;
    std::vector<cudaGraphExec_t> graphs;
    std::vector<cudaGraphExec_t> graphs_head;  // first part of each window position's graph (split capture)
    bool no_zform = false;                     // AMG_NO_ZFORM: nu = 2 inner FCG in the direct form (A/B)
    bool cap_split = false;                    // capture in progress, split point not reached yet
    cudaGraph_t cap_head = nullptr;
    int graph_nu = 0;
    long long graph_launches = 0;
    std::vector<long long> graph_launches_pos;  // per restart-window position
    std::vector<void*> allocs;
    std::vector<void*> ws_allocs;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaEvent_t pe0 = nullptr, pe1 = nullptr;  // live profile of the level-0 smoother steps
    bool prof_on = false;
    int64_t prof_win_bytes = 0;      // algorithmic bytes / launches inside the live-profile window
    int64_t prof_win_launches = 0;
    int64_t bytes = 0;
    amg_info info{};
    // distributed handle (amg_setup_dist); comm == nullptr on one GPU
    amg::Comm* comm = nullptr;
    int g = 0;                       // first replicated level: levels < g are row-partitioned
    int64_t n_global = 0, row_begin = 0;  // the caller's level-0 block
    int n_local = 0;
    double* ar_send = nullptr;       // batched dot allreduce scratch: [kArMax] and [kArMax * P]
    double* ar_recv = nullptr;
    double *bfull = nullptr, *xfull = nullptr;  // g == 0: gathered b and x
    cudaStream_t cs = nullptr;       // communication stream (halo messages overlap the interior rows)
    cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
    double* dsplit = nullptr;        // boundary-view partial dots of a split pass [4]: lo (dq, dr), hi (dq, dr)
};

namespace amg {

constexpr int kArMax = 40;  // scalars per batched allreduce

// driver.cu
template <class T>
T* halloc(amg_hierarchy* h, size_t n, bool ws = false) {
    T* p = dalloc<T>(n + 8, h->s);  // +8: padding for the 16-byte vector loads
    (ws ? h->ws_allocs : h->allocs).push_back(p);
    h->bytes += (int64_t)((n + 8) * sizeof(T));
    return p;
}
uint64_t host_sm64(uint64_t z);
double kappa_rule(int m);
void poly_coeffs(double l1, double kappa, int m, double* a, double* b);
// level loop (a1-a6) from h->lev[l0].A, which every rank holds whole (replicated); sets h->L
void build_levels(amg_hierarchy* h, int l0, int* agg0 = nullptr, int nc0 = 0);
int* aggregate_level(amg_hierarchy* h, int l, PassGraph& G, int* nc);
// coarsest inverse, SpMV formats, workspaces, tail (after all levels exist)
void finish_build(amg_hierarchy* h);
// vector of level l laid out for halo exchange: returns the pointer to its first own element
double* valloc(amg_hierarchy* h, Level& Lv, int slots, bool ws);

// dist.cu
void build_dist(amg_hierarchy* h, int64_t n_global, int64_t row_begin, int n_local, const int64_t* rp,
                const int32_t* ci_global, const double* v, const double* d);
void halo_exchange(amg_hierarchy* h, int l, double* x);  // no-op unless level l is row-partitioned
// sum the scalars at ptrs over the ranks (each rank's local partial; rank-order sum, identical on
// every rank); no-op on one GPU
// (extra1/extra2: partials of the boundary views of a split pass, added to ptrs[j] in this order)
void dot_allreduce(amg_hierarchy* h, const std::vector<double*>& ptrs, const std::vector<double*>& extra1 = {},
                   const std::vector<double*>& extra2 = {});
// split halo exchange: pack + messages on the communication stream (halo_start), then make the
// compute stream wait for them (halo_finish); no-op pair unless level l is row-partitioned
void halo_start(amg_hierarchy* h, int l, double* x);
void halo_finish(amg_hierarchy* h, int l);
// interior/boundary slice views of a row-partitioned SELL level (sets Lv.split, op_int, op_lo, op_hi)
void build_split(amg_hierarchy* h, int l);
// own block (count_r elements at displ_r of `full`) of every rank gathered into `full` (device)
void allgatherv_d(amg_hierarchy* h, double* full, const std::vector<int64_t>& offs);
// warm every exchange pattern once outside graph capture (NCCL connects peers lazily)
void warm_comm(amg_hierarchy* h);
// export helpers for the parity hooks: relative columns -> global ids, own agg -> global coarse ids
void export_dist_cols(amg_hierarchy* h, int l, int* out_dev);
void export_dist_agg(amg_hierarchy* h, int l, int* out_dev);
// global aggregation (Lv.gx): rH (own aggregates of level l+1) = P^T r over every member, the remote
// members' values received through the export plan, summed in increasing global row order
void restrict_global(amg_hierarchy* h, int l, const double* r, double* rH);

}  // namespace amg
