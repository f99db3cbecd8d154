// amg_internal.h -- internal declarations of libamg_b200.so (host launchers of the sm_100a
// kernels in k_setup.cu / k_solve.cu, used by driver.cu).  Not part of the ABI (include/amg.h).
// Shares nothing with oracle/ (the CPU oracle is test infrastructure only).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace amg {

constexpr int kMaxDeg = 16;      // poly_degree m <= kMaxDeg
constexpr int kMaxLevels = 48;
constexpr int kFuseRestrictRows = 40000;  // levels below this fuse residual + restriction (k_resid_restrict; C2 -4%)
constexpr int kMaxWin = 16;      // restart window / inner nu <= kMaxWin
constexpr int kBlock = 256;      // threads per block of the tile / vector kernels

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what, const char* file, int line);
void set_last_error(const std::string& msg);  // amg_last_error() text of the calling thread
std::string validation_message(int flags);    // text of validate_input's flags
#define CK(call) ::amg::cuda_check((call), #call, __FILE__, __LINE__)

// NVTX ranges (tracing): ABI calls, setup phases per level, outer FCG iterations.  Header-only
// NVTX v3: without a tool attached (nsys, ncu --nvtx) every push/pop is a no-op call.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---------------------------------------------------------------- device views
struct Csr {           // A_l: int32 row_ptr / col, fp64 values; arrays padded by >= 4 elements
    int n = 0;
    int64_t nnz = 0;
    int* rp = nullptr;
    int* ci = nullptr;
    double* v = nullptr;
};

struct Tiles {         // row tiles of the SpMV-class kernels: tile t = rows [row[t], row[t+1])
    int ntiles = 0;
    int cap = 0;       // shared-memory entry capacity; tiles with more nnz (single long rows) use the long path
    int grid = 0;      // resident grid used by the grid-stride launch
    int* row = nullptr;
};

struct Sell {          // SELL-32: 32-row slices, entries column-major inside a slice (lane = row % 32)
    int n = 0;
    int nslices = 0;
    int* sptr = nullptr;   // [nslices+1] slice offsets in units of 32 entries; width_s = sptr[s+1]-sptr[s]
    int* col = nullptr;    // [32 * sptr[nslices]]; padding: col = a valid row, val = 0
    double* val = nullptr;
    int64_t padded = 0;    // 32 * sptr[nslices]
    int wmax = 0;          // maximum slice width (selects the kernel's width bucket)
    int chi = 0;           // largest valid column index (n-1; n+nhi-1 with an upper halo) -- decode clamp
    // a VIEW of a contiguous slice range (halo overlap on a row-partitioned level runs the interior
    // slices while the halo is in flight, then the boundary slices): sptr/nslices describe the
    // view's slices and srow0 is the absolute first row of its first slice (0 for the whole level)
    int srow0 = 0;
    // lossless compressed streams (same slice layout), chosen per level at setup:
    int vmode = 0;         // 0: val (fp64); 1: vcode (uint8) into vdict (<= 256 distinct values)
    int cmode = 0;         // 0: col (int32); 1: ccode (uint8) into cdict of offsets col-row; 2: coff (int16 col-row);
                           // 3: pcode = vcode | ccode << 8 (uint16, one load per entry; requires vmode 1)
    uint8_t* vcode = nullptr;
    uint8_t* ccode = nullptr;
    int16_t* coff = nullptr;
    uint16_t* pcode = nullptr;
    double* vdict = nullptr;
    int* cdict = nullptr;
    int nvdict = 0, ncdict = 0;
};

struct SpOp {          // the operator of one level as the SpMV-class kernels see it
    Csr A;
    Tiles T;
    Sell S;
    bool sell = false;     // true: SELL-32 warp-per-slice kernel; false: CSR row-tile kernel
    int vg = 0;            // > 0: vector-CSR kernel with vg lanes per row (wide-row coarse levels; k_vcsr)
};

bool tma_eligible(const SpOp& op);  // format/size part of the TMA-staged kernel's eligibility

struct DotScratch {    // deterministic two-stage reductions (per-block partials + last-block sum)
    double* partials = nullptr;  // [kMaxWin+2][max grid]
    unsigned* ticket = nullptr;  // zero-initialised counter, reset by the last block
};

// ---------------------------------------------------------------- setup launchers (k_setup.cu)
// Allocation helpers use cudaMallocAsync on `s`.
template <class T>
T* dalloc(size_t n, cudaStream_t s) {
    void* p = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMallocAsync(&p, n * sizeof(T), s);
    if (e == cudaErrorMemoryAllocation) { cudaGetLastError(); throw Error(-5, "device out of memory"); }
    CK(e);
    return static_cast<T*>(p);
}
void dfree(void* p, cudaStream_t s);

// validation of the user CSR (reading A17).  Returns bit flags (0 = valid).
// Columns must lie in [cmin, cmax) ([0, n) on one GPU; [-nlo, n+nhi) relative on a row-partitioned level).
int pattern_rp32(int n, int64_t nnz, const int64_t* rp, const int32_t* ci, int* rp32, cudaStream_t s);
int validate_input(int n, int64_t nnz, int cmin, int cmax, const int64_t* rp, const int32_t* ci, const double* v, const double* d,
                   cudaStream_t s);
// A_0 = L + diag(d) with inserted missing diagonals; returns a fresh Csr.
Csr form_A0(int n, const int64_t* rp, const int32_t* ci, const double* v, const double* d, cudaStream_t s);
// lambda_1 = max_i sum_j |a_ij|  (exact: per-row sums in CSR order, max by ordered-int atomicMax)
double inf_norm(const Csr& A, cudaStream_t s);
void inf_norm_launch(const Csr& A, unsigned long long* o, cudaStream_t s);
// true if some d_i != 0
bool any_nonzero(int n, const double* d, cudaStream_t s);
// max |col - row| over the stored entries (0 if only a diagonal)
// Lanczos start vector of reading A24: out_i = 2 U(z ^ i) - 1, U(y) = (splitmix64(y) >> 11) 2^-53
void launch_lanczos_start(int n, uint64_t z, double* out, cudaStream_t s);

struct PassGraph {     // matching pass graph G_t: CSR with integer multiplicities, no diagonal
    int n = 0;
    int64_t nnz = 0;
    int* rp = nullptr;
    int* ci = nullptr;
    uint32_t* w = nullptr;
    bool unit = false;  // every multiplicity is 1 (G_0 of a level, reading A5): the matching kernels skip w
};
// off-diagonal entries with 0 <= col < n only (a row-partitioned level keeps its in-block edges: A20)
PassGraph pass_graph0(const Csr& A, cudaStream_t s);
void free_graph(PassGraph& g, cudaStream_t s);
// one aggregation pass: handshake matching + attach + leader numbering.  agg_t[v] in [0, *nc).
// id_off = global id of local vertex 0 (hash keys use global ids, docs/keys.md); 0 on one GPU.
int aggregate_pass(const PassGraph& G, uint64_t salt, int id_off, int* agg_t, int* nc, int* rounds, cudaStream_t s);
// reading A25 (opt-in mis_k > 0): MIS of the graph of A^k + layered growth, one aggregation per level
int mis_aggregate(const PassGraph& G, int k, uint64_t seed, int level, int* agg, int* nc, int* rounds, cudaStream_t s);
uint64_t host_sm64(uint64_t z);
// G_{t+1} = quotient of G_t under agg_t (multiplicities summed, self-loops dropped)
PassGraph quotient_graph(const PassGraph& G, const int* agg_t, int nc, cudaStream_t s);
// agg[i] = agg_t[agg[i]]
void compose(int n, int* agg, const int* agg_t, cudaStream_t s);
// A_H = P^T A P as entry sums in (row, CSR position) order per coarse entry (bit-exact with a
// sequential left-to-right summation).  Rows map through agg (perm/aptr), columns through cmap
// (nullptr = agg); coarse columns lie in [0, ncols) (ncols = nc on one GPU; on a row-partitioned
// level cmap is the shifted coarse column of every local/halo column, see dist.cu).
Csr galerkin(const Csr& A, const int* agg, const int* cmap, int nc, int ncols, const int* perm, const int* aptr,
             cudaStream_t s);
// perm = vertices sorted stably by aggregate, aptr[I] = first position of aggregate I
void aggregate_order(int n, const int* agg, int nc, int* perm, int* aptr, cudaStream_t s);
// row tiles for the CSR SpMV-class kernels
Tiles build_tiles(const Csr& A, int grid_per_sm, cudaStream_t s);
// SELL-32 copy of A (built when its padding is acceptable); returns S with S.col == nullptr otherwise
Sell build_sell(const Csr& A, double max_pad_ratio, cudaStream_t s);
// Lossless compression of a SELL level: value dictionary (<= 256 distinct fp64 values) and column
// offsets (<= 256 distinct col-row -> uint8 codes, else int16 if they fit).  Sets S.vmode/S.cmode.
void compress_sell(Sell& S, const Csr& A, cudaStream_t s);
void free_sell(Sell& S, cudaStream_t s);
// dense (pseudo-)inverse of the coarsest operator, row-major n x n
double* coarse_inverse(const Csr& A, bool singular, double shift, cudaStream_t s);
// dense B_l (n_l x n_l, row-major) of the level above the coarsest (k_dense.cu)
void dense_level_operator(const Csr& A, int m, const double* alpha, const double* beta, int nc, const int* agg,
                          const int* perm, const int* aptr, const double* Minv, double* Bd, cudaStream_t s);
void free_csr(Csr& A, cudaStream_t s);

// ---------------------------------------------------------------- solve launchers (k_solve.cu)
// Count of kernels launched through these launchers (for the gpu_launches report).
extern thread_local long long g_launches;

// SpMV-class fused kernels (one pass over A_l):
//  smooth: out_i = alpha*cg*xg_i + (1-alpha)*prev_i + beta*(f_i - cg*(A xg)_i),
//          prev_i = xprev ? xprev_i : cp*f_i          (three-term recurrence step)
void launch_smooth(const SpOp& op, const double* xg, double cg, const double* f, const double* xprev,
                   double cp, double alpha, double beta, double* out, cudaStream_t s);
//  two consecutive general steps in one launch (x_{k+1} into out1, x_{k+2} into out2; out2 may alias xk,
//  out1 may alias xkm1); flags [>= slices/8 + 1] and sync [3] are zero-initialised level scratch.
//  Returns false (nothing launched) when the level is not eligible.
//  resid: out = f - A xg; optional dot r.r into dots[0]
void launch_resid(const SpOp& op, const double* xg, const double* f, double* out, double* dot_rr,
                  const DotScratch& ds, cudaStream_t s);
//  spmv with dots: q = A d; *dot_dq = d.q, *dot_dr = d.rho
void launch_spmv_dots(const SpOp& op, const double* d, const double* rho, double* q, double* dot_dq,
                      double* dot_dr, const DotScratch& ds, cudaStream_t s);

// restriction rH[I] = sum_{t in [aptr[I], aptr[I+1])} r[perm[t]]  (sequential per aggregate)
void launch_restrict(int nc, const int* aptr, const int* perm, const double* r, double* rH, cudaStream_t s);
// prolongation + axpy: x[i] += eH[agg[i]]
void launch_prolong(int n, const int* agg, const double* eH, double* x, cudaStream_t s);
// nu = 2 inner FCG without d_1: the z-dots pass (out3 = z.Az, z.q0, z.rho) and the prolongation of
// E = c0 d0 + c1 z with the coefficients formed from sc (k_solve.cu k_prolong_fcg2)
void launch_spmv_zdots(const SpOp& op, const double* z, const double* q0, const double* rho, double* out3,
                       const DotScratch& ds, cudaStream_t s);
void launch_prolong_fcg2(int n, const int* agg, const double* d0, const double* z, const double* sc, double* x,
                         cudaStream_t s);
// x_i += E'[agg_i] with E' the last inner-FCG update (E' = alpha dH + eH, or alpha dH when assign;
// alpha = *dr / *dq, 0 when *dq = 0) -- fcg_update of the coarse level fused into the prolongation
void launch_prolong_fcg(int n, const int* agg, const double* eH, const double* dH, const double* dr, const double* dq,
                        bool assign, double* x, cudaStream_t s);
// dense coarse apply e = M r (M row-major n x n)
void launch_resid_restrict(int nc, const int* aptr, const int* perm, const Csr& A, const double* x, const double* f,
                           double* rho, cudaStream_t s);
void launch_gemv_prolong(int nf, const int* agg, int cb, int nL, const double* M, const double* r, double* x,
                         cudaStream_t s);
void launch_gemv_dense(int n, const double* M, const double* r, double* e, cudaStream_t s);
void launch_gemv(int n, const double* M, const double* r, double* e, cudaStream_t s);
// c[j] = z . Q_j for j < w  (Q_j = Q[j], pointers in a device array)
void launch_multidot(int n, const double* z, const double* const* Q, int w, double* c, const DotScratch& ds,
                     cudaStream_t s);
// d = z - sum_{j<w} (c[j]/dq[j]) D_j
void launch_direction(int n, const double* z, const double* const* D, const double* c, const double* dq, int w,
                      double* d, cudaStream_t s);
// FCG update: alpha = dr/dq (alpha = 0 if dq == 0 and inner);  x (+)= alpha d;  r -= alpha q (if r);
// optional rr = r.r; outer: breakdown flag if !(dq > 0).
// x = nullptr: the x update is deferred (alpha is stored to alpha_out, *set_old = 1 if set_old;
// launch_x_flush / launch_direction_xf apply it later)
void launch_fcg_update(int n, const double* dr, const double* dq, const double* d, const double* q, double* x,
                       bool assign_x, double* r, double* rr, int* breakdown, const DotScratch& ds, cudaStream_t s,
                       double* alpha_out = nullptr, int* set_old = nullptr);
struct Slots {
    int j[kMaxWin];
};
// x = (((x + a[j0] d_{j0}) + a[j1] d_{j1}) + ...) over the slots sl.j[0..cnt), d_j = D + j*ld: the same
// fma sequence as cnt successive launch_fcg_update x updates, so x is bitwise the same
void launch_x_flush(int n, double* x, const double* D, size_t ld, const double* a, const Slots& sl, int cnt,
                    cudaStream_t s);
// direction d = z - sum_{j<w} beta_j D[j] fused with x += a[W] d_old (if *has_old) + sum_{j<w} a[j] D[j]
bool direction_xf_ok(int w, const double* z, const double* const* D, const double* d, const double* x);
void launch_direction_xf(int n, const double* z, const double* const* D, const double* c, const double* dq, int w,
                         double* d, double* x, const double* alph, const int* has_old, cudaStream_t s);
// v -= mean(v) (two kernels: sum then subtract); tmp = one device double
void launch_mean_project(int n, double* v, double* tmp, const DotScratch& ds, cudaStream_t s);
// v -= (*sum) / ntot  (the second half of a mean projection whose sum was allreduced)
void launch_sub_mean(int n, double ntot, double* v, const double* sum, cudaStream_t s);
// out = a x + b y + c z  (y, z nullable; out may alias any input: elementwise)
void launch_lincomb3(int n, double a, const double* x, double b, const double* y, double c, const double* z,
                     double* out, cudaStream_t s);
// y = x (device copy kernel)
void launch_copy(int n, const double* x, double* y, cudaStream_t s);
// dot = x.y (deterministic)
void launch_dot(int n, const double* x, const double* y, double* out, const DotScratch& ds, cudaStream_t s);
// ---------------------------------------------------------------- coarse-tail megakernel (k_tail.cu)
// Every level l >= l_tail (small levels) is run entirely inside ONE thread-block cluster: the whole
// recursion B_l (smoothing, residual, restriction, inner FCG, coarsest GEMV, prolongation) with
// cluster barriers between dependent phases and cluster-wide (DSMEM) deterministic reductions.
struct TLevel {
    int n = 0, nc = 0;
    int ld = 0;  // slot stride of the inner-FCG D / Q arrays (global or shared)
    const int* rp = nullptr;
    const int* ci = nullptr;
    const double* v = nullptr;
    const int* agg = nullptr;
    const int* perm = nullptr;
    const int* aptr = nullptr;
    double alpha[kMaxDeg + 1] = {};
    double beta[kMaxDeg + 1] = {};
    double *X = nullptr, *XA = nullptr, *RES = nullptr, *RHO = nullptr, *E = nullptr;
    double *Z = nullptr, *D = nullptr, *Q = nullptr;
    // shared-memory mode: offsets (in doubles) of X, XA, RES, RHO, E, Z, D, Q inside the kernel's
    // dynamic shared memory; -1 = the global vector above
    int off[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
    // tail_smem = 2: the same for the read-only level data rp, ci, v, agg, perm, aptr (copied into
    // shared memory at kernel start); -1 = global
    int moff[6] = {-1, -1, -1, -1, -1, -1};
};
struct TailArgs {
    int l0 = 0;       // level the call starts at
    int L = 0;        // number of levels (L-1 = coarsest)
    int m = 0, nu = 0;
    int mode = 0;     // 0: out = B_l0(rin);  1: FCG_inner(l0): lev[l0].RHO -> lev[l0].E
    int smem = 0;     // doubles of dynamic shared memory holding the tail levels' vectors (0 = global)
    int lbase = 0;    // lev[k] describes level lbase + k
    const double* Minv = nullptr;
    const double* Bd = nullptr;   // dense B of level dense_l (k_dense.cu), or null
    int dense_l = -1;
    const double* rin = nullptr;
    double* out = nullptr;
    const TLevel* lev = nullptr;  // device array
};
constexpr int kTailMaxLev = 12;   // shared-memory mode: at most this many tail levels
constexpr int kTailSmemBytes = 200 * 1024;  // shared-memory mode budget for the tail vectors
constexpr int kTailMaxNu = 4;
constexpr int64_t kTailDenseEntries = 100000;  // dense B_{L-2} inside the tail only up to this many entries  // the tail kernel supports nu <= 4
// cluster size actually used (16 if the device allows non-portable clusters, else 8)
void launch_tail(const TailArgs& a, cudaStream_t s);

// Kernel launch through cudaLaunchKernelEx (stream-ordered, capturable into the CUDA graphs).
template <class... KArgs, class... Args>
void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.numAttrs = 0;
    CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// grid size used by the vector kernels
int vector_grid();
void init_device_props();

// ---------------------------------------------------------------- communicator (comm.cu)
// The three exchange steps of the row-partitioned path: a grouped point-to-point
// exchange (halo, allgatherv) and an equal-size allgather (batched dot partials).  Both are
// stream-ordered.  Two backends:
//   * NCCL (one process per GPU, over NVLink / NVSwitch), capturable into CUDA graphs;
//   * in-process host threads sharing one device (test emulation of P ranks on one GPU): each
//     call synchronises the caller's stream, meets the other ranks at a host barrier, copies
//     peer buffers with device-to-device cudaMemcpyAsync, and meets them again.  No kernel ever
//     waits on another rank's kernel; not capturable.
struct P2P {
    int peer;
    void* ptr;
    size_t bytes;
};
struct Comm {
    int rank = 0, size = 1;
    virtual ~Comm() {}
    // sends[k] goes to sends[k].peer; recvs[k] arrives from recvs[k].peer.  Messages between one
    // pair of ranks are matched in order.  A peer may not be the caller itself.
    virtual void sendrecv(const std::vector<P2P>& sends, const std::vector<P2P>& recvs, cudaStream_t s) = 0;
    // out[r * bytes .. (r+1) * bytes) = rank r's in[0 .. bytes) (device buffers, out != in)
    virtual void allgather(const void* in, void* out, size_t bytes, cudaStream_t s) = 0;
    virtual bool capturable() const = 0;
    virtual const char* kind() const = 0;
    virtual void abort() {}  // wake and fail the other ranks after a local error (thread backend)
};

}  // namespace amg

// opaque C-ABI communicator object (include/amg.h amg_comm)
struct amg_comm_s {
    amg::Comm* c = nullptr;
};

