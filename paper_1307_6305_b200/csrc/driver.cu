// driver.cu -- host driver and C ABI of libamg_b200.so (include/amg.h).
//
// Builds the hierarchy with the setup kernels (k_setup.cu) and runs the solve schedule with the
// solve kernels (k_solve.cu).  The k-cycle recursion (SURVEY.md
// 8(c) O6-O8) is a static schedule of kernel launches with all FCG scalars resident on the device,
// so one outer FCG iteration is captured once per restart-window position as a CUDA graph and
// replayed; the host only reads ||r||^2 and the breakdown flag once per outer iteration.
// Host code computes scalars only (the polynomial coefficients of SURVEY App. A, launch
// configurations); every vector/matrix operation runs in the library's kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <cstdlib>
#include <string>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/amg.h"
#include "amg_internal.h"
#include "hierarchy.h"

namespace amg {

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    char buf[512];
    snprintf(buf, sizeof(buf), "%s failed: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
    throw Error(e == cudaErrorMemoryAllocation ? AMG_E_OOM : AMG_E_CUDA, buf);
}

int tiled_grid(int cap, int ntiles);

}  // namespace amg

using namespace amg;

static thread_local std::string g_last_error;

void amg::set_last_error(const std::string& msg) { g_last_error = msg; }

static int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

// ------------------------------------------------------------------ host scalar math
// SplitMix64 (docs/keys.md) -- the salt of the matching keys.
uint64_t amg::host_sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static double delta_of(double kappa) { return (std::sqrt(kappa) - 1.0) / (std::sqrt(kappa) + 1.0); }
static double Em_of(int m, double kappa) { return std::pow(delta_of(kappa), m) * (kappa - 1.0) * 0.5; }

// Reading A8 (rule R1): kappa = 10 if E_m(10) < 1, else the kappa with E_m = 1/2:
// t = sqrt(kappa) solves (t-1)^(m+1) = (t+1)^(m-1) (Newton from t = 3, then stop at a fixed point).
double amg::kappa_rule(int m) {
    if (Em_of(m, 10.0) < 1.0) return 10.0;
    double t = 3.0;
    for (int it = 0; it < 200; ++it) {
        double f = std::pow(t - 1.0, m + 1) - std::pow(t + 1.0, m - 1);
        double df = (m + 1) * std::pow(t - 1.0, m) - (m - 1) * std::pow(t + 1.0, m - 2);
        double tn = t - f / df;
        if (tn == t) break;
        t = tn;
    }
    return t * t;
}

// Three-term recurrence coefficients: x_{k+1} = a_k x_k + (1-a_k) x_{k-1} + b_k (f - A x_k)
void amg::poly_coeffs(double l1, double kappa, int m, double* a, double* b) {
    const double l0 = l1 / kappa, d = delta_of(kappa), d2 = d * d;
    for (int k = 0; k <= m; ++k) {
        if (k == 0) { a[k] = 1.0; b[k] = (l0 + l1) / (2.0 * l0 * l1); }
        else if (k == 1) { a[k] = 1.0 + 2.0 * d2 * (1.0 - d2) / ((1.0 + d2) * (1.0 + d2)); b[k] = 2.0 / (l0 + l1); }
        else { a[k] = 1.0 + d2; b[k] = 4.0 * d / (l1 - l0); }
    }
}

static bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Stage a caller array on the device (copy if host). Returns device pointer; *tmp set if allocated.
template <class T>
static const T* stage_in(const T* p, size_t n, cudaStream_t s, void** tmp) {
    *tmp = nullptr;
    if (!p) return nullptr;
    if (is_device_ptr(p)) return p;
    T* d = dalloc<T>(n + 8, s);
    CK(cudaMemcpyAsync(d, p, n * sizeof(T), cudaMemcpyHostToDevice, s));
    *tmp = d;
    return d;
}

static void copy_out(void* dst, const void* src_dev, size_t bytes, cudaStream_t s) {
    CK(cudaMemcpyAsync(dst, src_dev, bytes, is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
}

// event record that is a real event node when the stream is being captured into a graph
static void record_event(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(s, &cs));
    if (cs == cudaStreamCaptureStatusActive)
        CK(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
    else
        CK(cudaEventRecord(e, s));
}

// cudaGraphExecDestroy of a handle's 5 graphs costs ~1.2 ms of host time; amg_free hands them to a
// process-wide worker thread instead (joined, and the rest destroyed, at exit).
namespace {
struct GraphReaper {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<std::pair<int, cudaGraphExec_t>> q;
    bool stop = false;
    std::thread th;
    GraphReaper() : th([this] { run(); }) {}
    void run() {
        std::unique_lock<std::mutex> lk(mu);
        for (;;) {
            cv.wait(lk, [this] { return stop || !q.empty(); });
            auto items = std::move(q);
            q.clear();
            const bool last = stop;
            lk.unlock();
            for (auto& it : items) {
                cudaSetDevice(it.first);
                cudaGraphExecDestroy(it.second);
            }
            lk.lock();
            if (last && q.empty()) return;
        }
    }
    void push(int dev, cudaGraphExec_t g) {
        {
            std::lock_guard<std::mutex> lk(mu);
            q.emplace_back(dev, g);
        }
        cv.notify_one();
    }
    void shutdown() {
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
        cv.notify_one();
        if (th.joinable()) th.join();
    }
};
GraphReaper* g_reaper = nullptr;
std::mutex g_reaper_mu;
GraphReaper* reaper() {
    std::lock_guard<std::mutex> lk(g_reaper_mu);
    if (!g_reaper) {
        g_reaper = new GraphReaper();
        std::atexit([] { if (g_reaper) g_reaper->shutdown(); });
    }
    return g_reaper;
}

}  // namespace

static void destroy_graphs(amg_hierarchy* h, bool deferred = false) {
    int dev = 0;
    if (deferred) cudaGetDevice(&dev);
    for (auto* v : {&h->graphs, &h->graphs_head})
        for (auto g : *v)
            if (g) {
                if (deferred) reaper()->push(dev, g);
                else cudaGraphExecDestroy(g);
            }
    h->graphs.clear();
    h->graphs_head.clear();
    h->graph_nu = 0;
    h->graph_launches = 0;
}

static double now_ms() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

// Pinned 64-byte host mirrors of the handles' scalars, recycled through a process-wide free list:
// cudaMallocHost / cudaFreeHost cost ~0.5 ms each, once per amg_setup / amg_free otherwise.
static std::mutex g_pin_mu;
static std::vector<double*> g_pin_free;
static double* pinned_take() {
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        if (!g_pin_free.empty()) {
            double* p = g_pin_free.back();
            g_pin_free.pop_back();
            return p;
        }
    }
    void* p = nullptr;
    CK(cudaMallocHost(&p, 8 * sizeof(double)));
    return static_cast<double*>(p);
}
static void pinned_give(double* p) {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back(p);
}

// Library streams: every live handle owns one (two handles may be used concurrently from different
// host threads), checked out of a per-device free list at setup and returned at amg_free after the
// handle's work has drained.  Reusing the stream (LIFO) keeps the memory a handle freed
// (stream-ordered) immediately reusable by the next setup without growing the pool.
static std::mutex g_stream_mu;
static std::vector<cudaStream_t> g_stream_free[64];

static cudaStream_t stream_acquire(int dev) {
    {
        std::lock_guard<std::mutex> lk(g_stream_mu);
        if (!g_stream_free[dev].empty()) {
            cudaStream_t s = g_stream_free[dev].back();
            g_stream_free[dev].pop_back();
            return s;
        }
    }
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    return s;
}

static void stream_release(int dev, cudaStream_t s) {
    if (!s) return;
    std::lock_guard<std::mutex> lk(g_stream_mu);
    g_stream_free[dev].push_back(s);
}

static void release(amg_hierarchy* h) {
    if (!h) return;
    static const bool trace = getenv("AMG_FREE_TRACE") != nullptr;
    const double t0 = trace ? now_ms() : 0.0;
    destroy_graphs(h, true);
    const double t1 = trace ? now_ms() : 0.0;
    if (h->s) {
        for (int l = 0; l < h->L; ++l) {
            dfree(h->lev[l].A.rp, h->s);
            dfree(h->lev[l].A.ci, h->s);
            dfree(h->lev[l].A.v, h->s);
            dfree(h->lev[l].T.row, h->s);
            free_sell(h->lev[l].S, h->s);
        }
        for (void* p : h->allocs) dfree(p, h->s);
        for (void* p : h->ws_allocs) dfree(p, h->s);
    }
    const double t2 = trace ? now_ms() : 0.0;
    if (h->s) cudaStreamSynchronize(h->s);  // drained: the stream goes back to the free list below
    const double t3 = trace ? now_ms() : 0.0;
    if (trace) fprintf(stderr, "[amg free] graphs %.3f ms, frees %.3f ms, sync %.3f ms\n", t1 - t0, t2 - t1, t3 - t2);
    if (h->hsc) pinned_give(h->hsc);
    if (h->e0) cudaEventDestroy(h->e0);
    if (h->e1) cudaEventDestroy(h->e1);
    if (h->pe0) cudaEventDestroy(h->pe0);
    if (h->pe1) cudaEventDestroy(h->pe1);
    if (h->ev_pack) cudaEventDestroy(h->ev_pack);
    if (h->ev_halo) cudaEventDestroy(h->ev_halo);
    if (h->cs) cudaStreamDestroy(h->cs);
    if (h->s) stream_release(h->dev, h->s);
    delete h;
}

// ------------------------------------------------------------------ setup
// AMG_SETUP_TRACE=1 prints a wall-clock phase breakdown (each phase ends in a stream sync).
struct PhaseTimer {
    bool on;
    cudaStream_t s;
    double t0;
    PhaseTimer(cudaStream_t st) : on(getenv("AMG_SETUP_TRACE") != nullptr), s(st), t0(now()) {}
    static double now() {
        timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
    }
    void mark(const char* what, int l = -1) {
        nvtxMarkA(what);  // phase boundary on the NVTX timeline (no-op without a tool)
        if (!on) return;
        cudaStreamSynchronize(s);
        double t = now();
        fprintf(stderr, "[amg setup] %-22s level %2d  %8.3f ms\n", what, l, t - t0);
        t0 = t;
    }
};
// Single GPU: stage and validate the caller's CSR (reading A17), A_0 = L + diag(d) (Eq. (prob)).
static void build(amg_hierarchy* h, int64_t n64, const int64_t* rp_in, const int32_t* ci_in, const double* v_in,
                  const double* d_in) {
    cudaStream_t s = h->s;
    PhaseTimer pt(s);
    if (n64 < 1 || n64 >= (int64_t(1) << 31) - 8) throw Error(AMG_E_ARG, "n out of range");
    const int n = (int)n64;
    // row_ptr first (to learn nnz)
    void* t_rp;
    const int64_t* rp = stage_in(rp_in, (size_t)n + 1, s, &t_rp);
    int64_t nnz_in = 0, rp0 = 0;
    CK(cudaMemcpyAsync(&nnz_in, rp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&rp0, rp, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (rp0 != 0 || nnz_in < 0 || nnz_in + n64 >= (int64_t(1) << 31) - 64) {
        dfree(t_rp, s);
        throw Error(rp0 != 0 || nnz_in < 0 ? AMG_E_INPUT : AMG_E_ARG, "row_ptr[0] != 0 or nnz out of range");
    }
    {   // grow the stream-ordered pool once to the estimated setup peak (freed blocks stay reserved:
        // release threshold = max), so the setup's many allocations never map memory mid-setup
        const size_t want = (size_t)(nnz_in + n) * 64 + ((size_t)256 << 20);
        void* r = nullptr;
        if (cudaMallocAsync(&r, want, s) == cudaSuccess) dfree(r, s); else cudaGetLastError();
    }
    void *t_ci, *t_v = nullptr, *t_d = nullptr;
    const int32_t* ci = stage_in(ci_in, (size_t)nnz_in, s, &t_ci);
    // Host inputs: the values (and d) are copied on a side stream while level 0's value-free
    // matching passes run on the pattern (row_ptr, col), which is checked first (ranges, order).
    const bool host_vals = (v_in && !is_device_ptr(v_in)) || (d_in && !is_device_ptr(d_in));
    cudaStream_t cs = nullptr;
    cudaEvent_t ev_vals = nullptr;
    struct SideStream {  // released on every exit path (an exception while staging included)
        cudaStream_t& cs;
        cudaEvent_t& ev;
        ~SideStream() {
            if (cs) { cudaStreamSynchronize(cs); cudaStreamDestroy(cs); }
            if (ev) cudaEventDestroy(ev);
        }
    } side_guard{cs, ev_vals};
    const double *v, *d;
    if (host_vals) {
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ev_vals, cudaEventDisableTiming));
        cudaEvent_t ev0;  // cs allocates from the pool after the row_ptr/col staging on s
        CK(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming));
        CK(cudaEventRecord(ev0, s));
        CK(cudaStreamWaitEvent(cs, ev0, 0));
        CK(cudaEventDestroy(ev0));
        v = stage_in(v_in, (size_t)nnz_in, cs, &t_v);
        d = stage_in(d_in, (size_t)n, cs, &t_d);
        CK(cudaEventRecord(ev_vals, cs));
    } else {
        v = stage_in(v_in, (size_t)nnz_in, s, &t_v);
        d = stage_in(d_in, (size_t)n, s, &t_d);
    }
    auto join_vals = [&]() {
        if (!cs) return;
        CK(cudaStreamWaitEvent(s, ev_vals, 0));
        CK(cudaStreamSynchronize(cs));
        CK(cudaEventDestroy(ev_vals));
        ev_vals = nullptr;
        CK(cudaStreamDestroy(cs));
        cs = nullptr;
    };
    auto free_inputs = [&]() { dfree(t_rp, s); dfree(t_ci, s); dfree(t_v, s); dfree(t_d, s); };
    pt.mark("stage inputs");
    int* agg0 = nullptr;
    int nc0 = 0;
    if (host_vals && n > h->opt.coarsest_size) {
        int* rp32 = dalloc<int>((size_t)n + 8, s);
        const int pf = pattern_rp32(n, nnz_in, rp, ci, rp32, s);
        if (pf) {
            dfree(rp32, s);
            join_vals();
            free_inputs();
            throw Error(AMG_E_INPUT, validation_message(pf));
        }
        try {
            Csr P;  // the input pattern: G_0's off-diagonal entries are the same as A_0's
            P.n = n;
            P.nnz = nnz_in;
            P.rp = rp32;
            P.ci = const_cast<int*>(ci);
            PassGraph G = pass_graph0(P, s);
            pt.mark("pass graph 0 (overlapped)", 0);
            agg0 = aggregate_level(h, 0, G, &nc0);
        } catch (...) {
            dfree(rp32, s);
            join_vals();
            free_inputs();
            throw;
        }
        dfree(rp32, s);
    }
    join_vals();
    int vf = validate_input(n, nnz_in, 0, n, rp, ci, v, d, s);
    pt.mark("validate");
    if (vf) {
        dfree(agg0, s);
        free_inputs();
        throw Error(AMG_E_INPUT, validation_message(vf));
    }
    h->singular = !(d && any_nonzero(n, d, s));
    h->lev[0].A = form_A0(n, rp, ci, v, d, s);
    free_inputs();
    h->L = 1;
    pt.mark("form A0");
    build_levels(h, 0, agg0, nc0);
    finish_build(h);
}

std::string amg::validation_message(int vf) {
    char buf[160];
    snprintf(buf, sizeof(buf), "invalid CSR input (flags 0x%x: 1 range, 2 unsorted, 4 positive off-diagonal, "
             "8 asymmetric, 16 diagonal, 32 d<0, 64 row_ptr)", vf);
    return buf;
}

// Level loop from level l0, whose operator every rank holds whole: lambda_1,
// kappa and coefficients, p matching passes composed into agg_l, the aggregate order and the
// Galerkin product, until n_l <= coarsest_size.
// p matching passes (or one MIS-k aggregation, reading A25) on level l's pass graph G (consumed);
// returns agg_l (device, caller-owned) and n_{l+1}
int* amg::aggregate_level(amg_hierarchy* h, int l, PassGraph& G, int* nc_out) {
    cudaStream_t s = h->s;
    PhaseTimer pt(s);
    Level& Lv = h->lev[l];
    const int n = G.n, p = h->p;
    int* agg = nullptr;
    int nc = n;
    if (h->opt.mis_k > 0) {
        agg = dalloc<int>((size_t)G.n + 8, s);
        mis_aggregate(G, h->opt.mis_k, h->opt.seed, l, agg, &nc, &Lv.rounds[0], s);
        pt.mark("MIS-k aggregation", l);
    }
    for (int t = 0; t < (h->opt.mis_k > 0 ? 0 : p); ++t) {
        const uint64_t salt = host_sm64(h->opt.seed ^ (((uint64_t)l << 8) ^ (uint64_t)t));
        int* agg_t = dalloc<int>((size_t)G.n + 8, s);
        int nct = 0;
        aggregate_pass(G, salt, 0, agg_t, &nct, &Lv.rounds[t], s);
        pt.mark("matching pass", l);
        if (t + 1 < p) {
            PassGraph G2 = quotient_graph(G, agg_t, nct, s);
            free_graph(G, s);
            G = G2;
            pt.mark("quotient graph", l);
        }
        if (t == 0) {
            agg = agg_t;
        } else {
            compose(n, agg, agg_t, s);
            dfree(agg_t, s);
        }
        nc = nct;
    }
    free_graph(G, s);
    *nc_out = nc;
    return agg;
}

void amg::build_levels(amg_hierarchy* h, int l0, int* agg0, int nc0) {
    cudaStream_t s = h->s;
    PhaseTimer pt(s);
    const int m = h->m;
    int l = l0;
    // lambda_1 of every level goes to a device slot; one read-back after the loop (a8 needs it only
    // for the solve and finish_build)
    unsigned long long* lam = dalloc<unsigned long long>(kMaxLevels, s);
    CK(cudaMemsetAsync(lam, 0, sizeof(unsigned long long) * kMaxLevels, s));
    struct LamGuard {
        unsigned long long* p;
        cudaStream_t s;
        ~LamGuard() { dfree(p, s); }
    } lam_guard{lam, s};
    for (;;) {
        char nvname[32];
        snprintf(nvname, sizeof(nvname), "amg setup level %d", l);
        NvtxRange nv(nvname);
        Level& Lv = h->lev[l];
        Lv.nglob = Lv.A.n;
        Lv.nnz_glob = Lv.A.nnz;
        inf_norm_launch(Lv.A, lam + l, s);
        pt.mark("lambda1", l);
        if (Lv.A.n <= h->opt.coarsest_size) break;
        if (l + 1 >= kMaxLevels) throw Error(AMG_E_SETUP, "too many levels");
        int* agg = nullptr;
        int nc = Lv.A.n;
        if (l == l0 && agg0) {  // level 0's aggregation already ran (overlapped with the value copies)
            agg = agg0;
            nc = nc0;
            agg0 = nullptr;
        } else {
            PassGraph G = pass_graph0(Lv.A, s);
            pt.mark("pass graph 0", l);
            agg = aggregate_level(h, l, G, &nc);
        }
        if (nc >= Lv.A.n) {
            dfree(agg, s);
            throw Error(AMG_E_SETUP, "coarsening stagnated (n_{l+1} = n_l)");
        }
        Lv.nc = nc;
        Lv.agg = agg;
        h->allocs.push_back(agg);
        Lv.perm = halloc<int>(h, Lv.A.n);
        Lv.aptr = halloc<int>(h, (size_t)nc + 1);
        aggregate_order(Lv.A.n, agg, nc, Lv.perm, Lv.aptr, s);
        pt.mark("aggregate order", l);
        h->lev[l + 1].A = galerkin(Lv.A, agg, nullptr, nc, nc, Lv.perm, Lv.aptr, s);
        h->L = l + 2;
        pt.mark("galerkin", l);
        ++l;
    }
    h->L = l + 1;
    std::vector<unsigned long long> lh((size_t)(l - l0 + 1));
    CK(cudaMemcpyAsync(lh.data(), lam + l0, sizeof(unsigned long long) * lh.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int k = l0; k <= l; ++k) {
        Level& Lv = h->lev[k];
        memcpy(&Lv.lambda1, &lh[k - l0], sizeof(double));
        Lv.kappa = h->opt.kappa > 1.0 ? h->opt.kappa : kappa_rule(m);
        poly_coeffs(Lv.lambda1, Lv.kappa, m, Lv.alpha, Lv.beta);
    }
}

double* amg::valloc(amg_hierarchy* h, Level& Lv, int slots, bool ws) {
    double* base = halloc<double>(h, (size_t)Lv.ld * slots, ws);
    return base + Lv.lo_pad;
}

// Largest eigenvalue of the symmetric tridiagonal (a[0..k), b[1..k)) by Sturm-count bisection.
static double tridiag_max(int k, const double* a, const double* b) {
    double lo = a[0], hi = a[0];
    for (int j = 0; j < k; ++j) {
        const double r = (j > 0 ? std::fabs(b[j]) : 0.0) + (j + 1 < k ? std::fabs(b[j + 1]) : 0.0);
        lo = std::min(lo, a[j] - r);
        hi = std::max(hi, a[j] + r);
    }
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        int cnt = 0;
        double d = 1.0;
        for (int j = 0; j < k; ++j) {
            d = a[j] - mid - (j > 0 ? b[j] * b[j] / d : 0.0);
            if (d == 0.0) d = -1e-300;
            if (d < 0.0) ++cnt;
        }
        if (cnt == k) hi = mid; else lo = mid;
    }
    return 0.5 * (lo + hi);
}

// Reading A24 (opt-in): largest Ritz value of k plain Lanczos steps on A_l from
// the counter-based start vector, every vector operation in the library's kernels (SpMV + dots,
// linear combinations), the k x k tridiagonal on the host.
static double lanczos_max(amg_hierarchy* h, int l, int k) {
    Level& Lv = h->lev[l];
    cudaStream_t s = h->s;
    const int n = Lv.A.n;
    double* buf = dalloc<double>(3 * ((size_t)n + 8), s);
    double* vj = buf;
    double* vm = buf + n + 8;
    double* w = buf + 2 * (n + 8);
    double* sc = dalloc<double>(4, s);
    const uint64_t z = host_sm64(h->opt.seed ^ 0x4C414E435A4F5300ULL ^ (uint64_t)l);
    launch_lanczos_start(n, z, vj, s);
    CK(cudaMemsetAsync(vm, 0, sizeof(double) * n, s));
    auto read = [&](const double* p) {
        double v = 0.0;
        CK(cudaMemcpyAsync(&v, p, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return v;
    };
    launch_dot(n, vj, vj, sc, h->ds, s);
    launch_lincomb3(n, 1.0 / std::sqrt(read(sc)), vj, 0.0, nullptr, 0.0, nullptr, vj, s);
    if (k > 64) k = 64;
    double al[64] = {}, be[65] = {};
    be[0] = 0.0;
    int steps = 0;
    for (int j = 0; j < k; ++j) {
        launch_spmv_dots(Lv.op, vj, vj, w, sc, sc + 1, h->ds, s);  // w = A v_j, alpha_j = v_j.w
        al[j] = read(sc);
        launch_lincomb3(n, 1.0, w, -al[j], vj, -be[j], vm, w, s);
        launch_dot(n, w, w, sc + 2, h->ds, s);
        steps = j + 1;
        be[j + 1] = std::sqrt(read(sc + 2));
        if (!(be[j + 1] > 0.0)) break;
        launch_lincomb3(n, 1.0 / be[j + 1], w, 0.0, nullptr, 0.0, nullptr, vm, s);  // v_{j+1} into v_{j-1}'s slot
        std::swap(vj, vm);
    }
    dfree(buf, s);
    dfree(sc, s);
    return tridiag_max(steps, al, be);
}

void amg::finish_build(amg_hierarchy* h) {
    cudaStream_t s = h->s;
    PhaseTimer pt(s);
    // coarsest (a7): every rank holds it whole
    Level& C = h->lev[h->L - 1];
    const double shift = C.lambda1 > 0.0 ? C.lambda1 : 1.0;
    h->Minv = coarse_inverse(C.A, h->singular, shift, s);
    h->allocs.push_back(h->Minv);
    pt.mark("coarse inverse", h->L - 1);
    // SpMV formats of every level the SpMV-class kernels run on (all but the coarsest; level 0 always)
    for (int k = 0; k < h->L; ++k) {
        Level& Lv = h->lev[k];
        if (k < h->L - 1 || k == 0) {
            if (!getenv("AMG_NO_SELL")) Lv.S = build_sell(Lv.A, 1.6, s);
            if (Lv.S.sptr) Lv.S.chi = Lv.A.n + Lv.H.nhi - 1;
            pt.mark("sell", k);
            if (!Lv.S.sptr) {  // CSR row tiles: only the levels too irregular for SELL use them
                Lv.T = build_tiles(Lv.A, 0, s);
                pt.mark("tiles", k);
            }
            if (Lv.S.sptr && h->opt.compress) compress_sell(Lv.S, Lv.A, s);
            pt.mark("compress", k);
        }
        Lv.op.A = Lv.A;
        Lv.op.T = Lv.T;
        Lv.op.S = Lv.S;
        Lv.op.sell = Lv.S.sptr != nullptr;
        if (Lv.dist) build_split(h, k);
        // wide-row levels (generic SELL width) that the TMA kernel does not take, small enough for the
        // fp64/int32 CSR to stay L2-resident (<= 6M entries): vector-CSR kernel with G lanes per row,
        // G ~ mean row length / 5.  C4 levels 2-4 (18-21 entries per row): solve 94.3 -> 83.9 ms
        // (3 entries per lane: 85.8, 8: 87.0); on C4's level 1 (24.7M entries) the CSR lost to the
        // compressed SELL, with fp64 values (121.7 ms) and with 1-byte value codes (100.5 ms).
        if (k < h->L - 1 && !Lv.dist && Lv.op.sell && Lv.S.wmax > 16 && !tma_eligible(Lv.op)) {
            static const double min_avg = getenv("AMG_VCSR_MIN_AVG") ? atof(getenv("AMG_VCSR_MIN_AVG")) : 12.0;
            const double avg = (double)Lv.A.nnz / std::max(1, Lv.A.n);
            if (min_avg > 0.0 && avg >= min_avg && Lv.A.nnz <= 6000000) {
                int g = 4;
                while (g < 32 && 5.0 * g < avg) g <<= 1;
                Lv.op.vg = g;
            }
        }
        // vector layout [pad | lower halo | own | upper halo]
        Lv.lo_pad = (Lv.H.nlo + 3) & ~3;
        Lv.ld = Lv.dist ? ((Lv.lo_pad + Lv.A.n + Lv.H.nhi + 3) & ~3) : ((Lv.A.n + 3) & ~3);  // 32-byte aligned slots
    }
    pt.mark("formats");
    // level workspaces
    for (int k = 0; k < h->L; ++k) {
        Level& Lv = h->lev[k];
        if (k < h->L - 1) {
            Lv.X = valloc(h, Lv, 1, false);
            Lv.XA = valloc(h, Lv, 1, false);
            Lv.RES = valloc(h, Lv, 1, false);
        }
        if (k >= 1) {
            Lv.RHO = valloc(h, Lv, 1, false);
            Lv.E = valloc(h, Lv, 1, false);
        }
        Lv.sc = halloc<double>(h, 3 * kMaxWin);
    }
    // outer FCG on level 0's own rows
    Level& L0 = h->lev[0];
    const int n = L0.A.n;
    h->n = n;
    h->W = h->opt.restart;
    h->b = valloc(h, L0, 1, false);
    h->x = valloc(h, L0, 1, false);
    h->r = valloc(h, L0, 1, false);
    h->Z = valloc(h, L0, 1, false);
    h->D = valloc(h, L0, h->W, false);
    h->Q = valloc(h, L0, h->W, false);
    h->osc = halloc<double>(h, 2 * kMaxWin + 8);
    h->alph = halloc<double>(h, kMaxWin);
    h->xold = halloc<int>(h, 4);
    h->flag = reinterpret_cast<int*>(h->osc + 2 * kMaxWin + 4);  // next to rr: one read-back per outer iteration
    h->ds.partials = halloc<double>(h, (size_t)(kMaxWin + 2) * 4096);
    h->ds.ticket = halloc<unsigned>(h, 4);
    CK(cudaMemsetAsync(h->ds.ticket, 0, 4 * sizeof(unsigned), s));
    h->hsc = pinned_take();
    if (h->comm) {
        h->ar_send = halloc<double>(h, kArMax);
        h->ar_recv = halloc<double>(h, (size_t)kArMax * h->comm->size);
        h->dsplit = halloc<double>(h, kArMax);
        CK(cudaStreamCreateWithFlags(&h->cs, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&h->ev_pack, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming));
    }
    // coarse tail: first replicated level l >= 1 with nnz(A_l) <= tail_nnz (one SM runs it from L1/L2)
    h->l_tail = h->L;
    if (h->opt.tail_nnz > 0)
        for (int k = std::max(1, h->g); k < h->L; ++k)
            if (h->lev[k].A.nnz <= h->opt.tail_nnz) { h->l_tail = k; break; }
    // When the tail would only hold the level above the coarsest (and the coarsest), the dense B_{L-2}
    // applied by full-GPU launches is faster than the one-CTA tail (C4 99.8 -> 94.2 ms, C5 203 -> 190 ms)
    if (h->l_tail >= h->L - 2 && h->L >= 2 && h->opt.dense_b_rows > 0 && !h->lev[h->L - 2].dist &&
        h->lev[h->L - 2].A.n <= h->opt.dense_b_rows)
        h->l_tail = h->L;
    if (h->l_tail < h->L) {
        size_t cur = 0;
        CK(cudaDeviceGetLimit(&cur, cudaLimitStackSize));
        if (cur < 4096) CK(cudaDeviceSetLimit(cudaLimitStackSize, 4096));  // t_B/t_fcg recursion
        h->d_tlev = halloc<TLevel>(h, kMaxLevels);
    }
    // reading A24 (opt-in): tighter lambda_1 on the smoothed levels (needs the SpMV formats and the
    // dot scratch above), coefficients recomputed
    if (h->opt.lanczos_steps > 0) {
        for (int k = 0; k < h->L - 1; ++k) {
            Level& Lv = h->lev[k];
            const double t = 1.1 * lanczos_max(h, k, h->opt.lanczos_steps);
            if (t < Lv.lambda1) Lv.lambda1 = t;
            poly_coeffs(Lv.lambda1, Lv.kappa, h->m, Lv.alpha, Lv.beta);
        }
    }
    // the level above the coarsest: B_{L-2} is linear (exact coarse solve, reading A12); formed
    // densely on small replicated levels and applied as one GEMV per visit (k_dense.cu)
    // Inside the one-CTA coarse tail a GEMV streams all n^2 entries through one SM, so there it is
    // formed only when small (C4's 267 rows: faster; C5's 591: slower than the sparse phases).
    h->dense_l = -1;
    if (h->L >= 2 && h->opt.dense_b_rows > 0) {
        Level& Lv = h->lev[h->L - 2];
        const bool in_tail = h->L - 2 >= h->l_tail;
        if (!Lv.dist && Lv.A.n <= h->opt.dense_b_rows &&
            (!in_tail || (int64_t)Lv.A.n * Lv.A.n <= kTailDenseEntries)) {
            h->Bd = halloc<double>(h, (size_t)Lv.A.n * Lv.A.n);
            dense_level_operator(Lv.A, h->m, Lv.alpha, Lv.beta, Lv.nc, Lv.agg, Lv.perm, Lv.aptr, h->Minv, h->Bd, s);
            h->dense_l = h->L - 2;
            pt.mark("dense B", h->L - 2);
        }
    }
    CK(cudaStreamSynchronize(s));
    pt.mark("workspaces");
}

// device descriptors of the tail levels (refreshed whenever the inner workspaces change)
static void upload_tail_levels(amg_hierarchy* h) {
    if (!h->d_tlev) return;
    std::vector<TLevel> t(h->L);
    for (int k = 0; k < h->L; ++k) {
        const Level& Lv = h->lev[k];
        TLevel& d = t[k];
        d.n = Lv.A.n;
        d.ld = Lv.ld;
        d.nc = Lv.nc;
        d.rp = Lv.A.rp;
        d.ci = Lv.A.ci;
        d.v = Lv.A.v;
        d.agg = Lv.agg;
        d.perm = Lv.perm;
        d.aptr = Lv.aptr;
        for (int j = 0; j <= h->m; ++j) { d.alpha[j] = Lv.alpha[j]; d.beta[j] = Lv.beta[j]; }
        d.X = Lv.X; d.XA = Lv.XA; d.RES = Lv.RES; d.RHO = Lv.RHO; d.E = Lv.E;
        d.Z = Lv.Z; d.D = Lv.D; d.Q = Lv.Q;
    }
    // shared-memory mode of the tail (k_tail.cu): every vector of the tail levels in the CTA's shared
    // memory when they fit (nu inner slots), so each phase of the recursion costs L1/shared-memory
    // latencies instead of L2 round trips
    h->tail_smem = 0;
    if (h->l_tail < h->L && h->opt.tail_smem && h->L - h->l_tail <= kTailMaxLev &&
        h->nu_ws >= 1) {
        int64_t off = 0;
        auto take = [&](int64_t len) {
            const int64_t o = off;
            off += (len + 1) & ~int64_t(1);  // 16-byte aligned slots
            return (int)o;
        };
        for (int k = h->l_tail; k < h->L; ++k) {
            TLevel& d = t[k];
            const int64_t n = d.n;
            if (k < h->L - 1) {
                d.off[0] = take(n);
                d.off[1] = take(n);
                d.off[2] = take(n);
                d.off[5] = take(n);
                d.off[6] = take((int64_t)d.ld * h->nu_ws);
                d.off[7] = take((int64_t)d.ld * h->nu_ws);
            }
            d.off[3] = take(n);
            d.off[4] = take(n);
        }
        if (h->opt.tail_smem == 1 && off * (int64_t)sizeof(double) <= kTailSmemBytes) {
            h->tail_smem = (int)off;
        } else if (h->opt.tail_smem == 1) {
            for (int k = h->l_tail; k < h->L; ++k)
                for (int j = 0; j < 8; ++j) t[k].off[j] = -1;
        } else {
            // tail_smem = 2: greedy placement by access frequency until the budget is spent -- each
            // level's matrix (read by every SpMV phase), then the smoother / residual / transfer
            // vectors, the aggregate maps, and last the inner-FCG vectors; the rest stays global
            for (int k = h->l_tail; k < h->L; ++k) {
                for (int j = 0; j < 8; ++j) t[k].off[j] = -1;
                for (int j = 0; j < 6; ++j) t[k].moff[j] = -1;
            }
            off = 0;
            const int64_t cap = kTailSmemBytes / (int64_t)sizeof(double);
            auto place = [&](int64_t len) -> int {  // len in doubles; -1 if it does not fit
                const int64_t a = (len + 1) & ~int64_t(1);
                if (off + a > cap) return -1;
                const int64_t o = off;
                off += a;
                return (int)o;
            };
            auto ints = [](int64_t n) { return (n + 1) / 2; };  // ints -> doubles
            for (int k = h->l_tail; k < h->L - 1; ++k) {  // tier 1: matrices (not the dense coarsest)
                TLevel& d = t[k];
                const int64_t nnz = h->lev[k].A.nnz;
                const int64_t need = ints(d.n + 1) + ints(nnz) + nnz + 6;
                if (off + need > cap) break;
                d.moff[0] = place(ints(d.n + 1));
                d.moff[1] = place(ints(nnz));
                d.moff[2] = place(nnz);
            }
            for (int k = h->l_tail; k < h->L; ++k) {  // tier 2: hot vectors
                TLevel& d = t[k];
                if (k < h->L - 1) {
                    d.off[0] = place(d.n);
                    d.off[1] = place(d.n);
                    d.off[2] = place(d.n);
                }
                d.off[3] = place(d.n);
                d.off[4] = place(d.n);
            }
            for (int k = h->l_tail; k < h->L - 1; ++k) {  // tier 3: aggregate maps
                TLevel& d = t[k];
                d.moff[3] = place(ints(d.n));
                d.moff[4] = place(ints(d.n));
                d.moff[5] = place(ints(d.nc + 1));
            }
            for (int k = h->l_tail; k < h->L - 1; ++k) {  // tier 4: inner FCG vectors
                TLevel& d = t[k];
                d.off[5] = place(d.n);
                d.off[6] = place((int64_t)d.ld * h->nu_ws);
                d.off[7] = place((int64_t)d.ld * h->nu_ws);
            }
            h->tail_smem = (int)off;
        }
    }
    CK(cudaMemcpyAsync(h->d_tlev, t.data(), sizeof(TLevel) * t.size(), cudaMemcpyHostToDevice, h->s));
    CK(cudaStreamSynchronize(h->s));
}

// Algorithmic bytes of one general three-term smoother step on a level in the storage format the
// kernel actually streams: per stored entry the value stream (fp64 8 B or 1-byte code)
// plus the column stream (int32 4 B, 1-byte code, int16 2 B; a value/column code pair = 2 B total),
// per row the four vectors x_k (gathered, counted once), x_{k-1}, f and the output (32 B), and the
// row pointer (4 B) for the CSR row-tile fallback.  Uncompressed SELL: 12 nnz + 32 n.
static int64_t smoother_bytes(const Level& Lv) {
    const int64_t nnz = Lv.A.nnz, n = Lv.A.n;
    if (!Lv.op.sell) return 12 * nnz + 36 * n;
    const Sell& S = Lv.S;
    int64_t per = 0;
    if (S.cmode == 3) per = 2;
    else per = (S.vmode ? 1 : 8) + (S.cmode == 0 ? 4 : S.cmode == 1 ? 1 : 2);
    return per * nnz + 32 * n;
}

// the coarse-tail kernel implements the k-cycle only
static bool use_tail(const amg_hierarchy* h, int l, int nu) {
    return l >= h->l_tail && nu <= kTailMaxNu && h->opt.cycle == 0;
}

static void tail_call(amg_hierarchy* h, int mode, int l, int nu, const double* rin, double* out) {
    TailArgs a;
    a.l0 = l;
    a.L = h->L;
    a.m = h->m;
    a.nu = nu;
    a.mode = mode;
    a.Minv = h->Minv;
    a.Bd = h->Bd;
    a.dense_l = h->dense_l;
    a.rin = rin;
    a.out = out;
    a.lev = h->d_tlev;
    a.smem = h->tail_smem;
    a.lbase = 0;
    launch_tail(a, h->s);
}

static void ensure_inner_ws(amg_hierarchy* h, int nu) {
    if (nu <= h->nu_ws) return;
    for (void* p : h->ws_allocs) dfree(p, h->s);
    h->ws_allocs.clear();
    for (int k = 1; k < h->L - 1; ++k) {
        Level& Lv = h->lev[k];
        Lv.Z = valloc(h, Lv, 1, true);
        Lv.D = valloc(h, Lv, nu, true);
        Lv.Q = valloc(h, Lv, nu, true);
    }
    h->nu_ws = nu;
    destroy_graphs(h);
    upload_tail_levels(h);
}

// ------------------------------------------------------------------ solve schedule
static void apply_B(amg_hierarchy* h, int l, int nu, const double* rin, double* out);

// One SpMV-class pass on level l that reads x at the halo columns: `run(op, part)` launches the pass
// over the slices of `op`.  On a row-partitioned level with an interior/boundary split the interior
// slices (part 0) run while the halo messages are in flight, then the boundary slices
// before (part 1) and after (part 2) them; a dot-producing pass writes parts 1/2 into split slots.
template <class F>
static void spmv_pass(amg_hierarchy* h, int l, double* x, F&& run) {
    Level& Lv = h->lev[l];
    if (!Lv.dist) {
        run(Lv.op, 0);
        return;
    }
    if (!Lv.split) {
        halo_exchange(h, l, x);
        run(Lv.op, 0);
        return;
    }
    halo_start(h, l, x);
    run(Lv.op_int, 0);
    halo_finish(h, l);
    run(Lv.op_lo, 1);
    run(Lv.op_hi, 2);
}

// q = A d with d.q and d.rho into dq, dr (allreduced over the ranks on a row-partitioned level)
static void spmv_dots_pass(amg_hierarchy* h, int l, double* d, const double* rho, double* q, double* dq,
                           double* dr) {
    Level& Lv = h->lev[l];
    spmv_pass(h, l, d, [&](const SpOp& op, int part) {
        double* o0 = part == 0 ? dq : h->dsplit + 2 * (part - 1);
        double* o1 = part == 0 ? dr : h->dsplit + 2 * (part - 1) + 1;
        launch_spmv_dots(op, d, rho, q, o0, o1, h->ds, h->s);
    });
    if (Lv.dist) {
        if (Lv.split) dot_allreduce(h, {dq, dr}, {h->dsplit, h->dsplit + 1}, {h->dsplit + 2, h->dsplit + 3});
        else dot_allreduce(h, {dq, dr});
    }
}

// FCG_inner(l, RHO_l, nu) -> E_l.  On a row-partitioned level every SpMV
// input is halo-exchanged first and every batch of dot partials is summed over the ranks before the
// kernels that consume it.
// defer_last: the last update E (+)= alpha D_{nu-1} is left to the caller's fused prolongation.
// Returns kFcgDone (E written), kFcgDeferred (launch_prolong_fcg with D_{nu-1} and its dots), or, for
// nu = 2, kFcgZ: the second direction d_1 = z - beta_0 d_0 and q_1 = A d_1 are never formed -- one
// pass over z gives z.Az, z.q_0, z.rho_1, from which beta_0, d_1.q_1 and alpha_1 follow (symmetric A;
// see k_prolong_fcg2), and the caller prolongs E = (alpha_0 - alpha_1 beta_0) d_0 + alpha_1 z.  Two
// launches (the multidot and the direction) and the d_1 / q_1 vectors less per visit; the same
// iterate as the direct form up to rounding.
enum { kFcgDone = 0, kFcgDeferred = 1, kFcgZ = 2 };
static int fcg_inner(amg_hierarchy* h, int l, int nu, bool defer_last = false) {
    if (use_tail(h, l, nu)) {
        tail_call(h, 1, l, nu, nullptr, nullptr);
        return kFcgDone;
    }
    Level& Lv = h->lev[l];
    cudaStream_t s = h->s;
    const int n = Lv.A.n;
    double* rho = Lv.RHO;
    double* dq = Lv.sc;
    double* dr = Lv.sc + kMaxWin;
    double* c = Lv.sc + 2 * kMaxWin;
    const double* Dp[kMaxWin];
    const double* Qp[kMaxWin];
    for (int i = 0; i < nu; ++i) {
        double* Di = Lv.D + (size_t)i * Lv.ld;
        double* Qi = Lv.Q + (size_t)i * Lv.ld;
        Dp[i] = Di;
        Qp[i] = Qi;
        if (i == 0) {
            apply_B(h, l, nu, rho, Di);
        } else if (defer_last && nu == 2 && !Lv.dist && !h->no_zform) {
            apply_B(h, l, nu, rho, Lv.Z);
            launch_spmv_zdots(Lv.op, Lv.Z, Qp[0], rho, c, h->ds, s);
            return kFcgZ;
        } else {
            apply_B(h, l, nu, rho, Lv.Z);
            launch_multidot(n, Lv.Z, Qp, i, c, h->ds, s);
            if (Lv.dist) {
                std::vector<double*> cs;
                for (int j = 0; j < i; ++j) cs.push_back(c + j);
                dot_allreduce(h, cs);
            }
            launch_direction(n, Lv.Z, Dp, c, dq, i, Di, s);
        }
        spmv_dots_pass(h, l, Di, rho, Qi, dq + i, dr + i);  // q = A d, d.q, d.rho
        if (defer_last && i == nu - 1) return kFcgDeferred;
        launch_fcg_update(n, dr + i, dq + i, Di, Qi, Lv.E, i == 0, (i < nu - 1) ? rho : nullptr, nullptr, nullptr,
                          h->ds, s);
    }
    return kFcgDone;
}

// Stationary AMLI coarse correction at level l (cycle 2; reading A23):
// E_l = q(B_l A_l) B_l RHO_l, q the degree-(nu-1) best uniform approximation to 1/t on [1/kappa_A, 1]
// by the smoother's three-term recurrence on the preconditioned operator:
//   y_0 = 0, y_{k+1} = a_k y_k + (1 - a_k) y_{k-1} + b_k B_l(RHO - A_l y_k), k = 0..nu-1.
// nu applications of B_l, nu-1 residual passes; nu = 1: E = B_l RHO.
static void amli_correction(amg_hierarchy* h, int l, int nu) {
    Level& Lv = h->lev[l];
    cudaStream_t s = h->s;
    if (nu == 1) {
        apply_B(h, l, nu, Lv.RHO, Lv.E);
        return;
    }
    const int m = nu - 1, n = Lv.A.n;
    const double kap = h->opt.amli_kappa > 1.0 ? h->opt.amli_kappa : kappa_rule(m);
    double a[kMaxDeg + 1], b[kMaxDeg + 1];
    poly_coeffs(1.0, kap, m, a, b);
    double* T = Lv.Q;   // residual RHO - A y_k (vector layout of the level: its halo is exchanged by B)
    double* cur = Lv.E;
    double* prev = Lv.D;
    apply_B(h, l, nu, Lv.RHO, Lv.Z);
    launch_lincomb3(n, b[0], Lv.Z, 0.0, nullptr, 0.0, nullptr, cur, s);  // y_1 = b_0 B rho
    for (int k = 1; k <= m; ++k) {
        spmv_pass(h, l, cur, [&](const SpOp& op, int) { launch_resid(op, cur, Lv.RHO, T, nullptr, h->ds, s); });
        apply_B(h, l, nu, T, Lv.Z);
        // y_{k+1} = a_k y_k + (1 - a_k) y_{k-1} + b_k z  (y_0 = 0) into the y_{k-1} buffer
        launch_lincomb3(n, a[k], cur, 1.0 - a[k], k >= 2 ? prev : nullptr, b[k], Lv.Z, prev, s);
        std::swap(cur, prev);
    }
    if (cur != Lv.E) launch_copy(n, cur, Lv.E, s);
}

// A chain of general smoothing steps x_out = a x_g + (1 - a) x_prev + b (f - A x_g) on level l, each the
// next one's x_prev / x_g, one launch per step.  When `prof`, the algorithmic bytes and launches are
// added to the live-profile window counters.
struct SmStep {
    const double* xg;
    const double* xprev;
    double a, b;
    double* out;
};
static int64_t smoother_bytes(const Level& Lv);
static void run_steps(amg_hierarchy* h, int l, const double* f, const std::vector<SmStep>& st, bool prof) {
    for (const SmStep& s1 : st) {
        spmv_pass(h, l, const_cast<double*>(s1.xg), [&](const SpOp& op, int) {
            launch_smooth(op, s1.xg, 1.0, f, s1.xprev, 0.0, s1.a, s1.b, s1.out, h->s);
        });
        if (prof) {
            h->prof_win_bytes += smoother_bytes(h->lev[l]);
            h->prof_win_launches += 1;
        }
    }
}

// Each outer iteration's graph is captured in two parts, split after level 0's residual and
// restriction: the head (the m pre-smoothing steps, the residual, the restriction: ~0.5 ms of GPU
// work on C3/C4) and the rest.  cudaGraphLaunch of the whole 134-node (C3) / 508-node (C4) graph kept
// the GPU idle for ~0.09 / ~0.43 ms after every convergence check (tools/timeline.py); the head is
// submitted in a few microseconds and the rest is submitted while the head runs.
static void capture_split_point(amg_hierarchy* h) {
    if (!h->cap_split) return;
    h->cap_split = false;
    CK(cudaStreamEndCapture(h->s, &h->cap_head));
    CK(cudaStreamBeginCapture(h->s, cudaStreamCaptureModeThreadLocal));
}

// z = B_l(r): pre-smoothing from 0, residual, restriction, coarse correction,
// prolongation, post-smoothing; the last smoothing step writes `out` (distinct from rin and the
// level buffers).  `rin` must be a vector of level l's layout (it is the first step's SpMV input).
static void apply_B(amg_hierarchy* h, int l, int nu, const double* rin, double* out) {
    cudaStream_t s = h->s;
    if (l == h->L - 1) {
        launch_gemv(h->lev[l].A.n, h->Minv, rin, out, s);
        return;
    }
    if (l == h->dense_l) {  // the linear B_{L-2} as one dense GEMV (k_dense.cu)
        launch_gemv_dense(h->lev[l].A.n, h->Bd, rin, out, s);
        return;
    }
    if (use_tail(h, l, nu)) {
        tail_call(h, 0, l, nu, rin, out);
        return;
    }
    Level& Lv = h->lev[l];
    const int m = h->m;
    const double* a = Lv.alpha;
    const double* b = Lv.beta;
    // pre-smoothing S(r, 0): step 0 is free (x_1 = b0 r implicit)
    double* cur = Lv.X;
    double* prev = Lv.XA;
    spmv_pass(h, l, const_cast<double*>(rin), [&](const SpOp& op, int) {
        launch_smooth(op, rin, b[0], rin, nullptr, 0.0, a[1], b[1], Lv.X, s);  // k = 1 (x_0 = 0)
    });
    if (m >= 2) {
        spmv_pass(h, l, Lv.X, [&](const SpOp& op, int) {
            launch_smooth(op, Lv.X, 1.0, rin, nullptr, b[0], a[2], b[2], Lv.XA, s);  // k = 2 (x_1 = b0 r)
        });
        cur = Lv.XA;
        prev = Lv.X;
        std::vector<SmStep> st;
        for (int k = 3; k <= m; ++k) {
            st.push_back({cur, prev, a[k], b[k], prev});
            std::swap(cur, prev);
        }
        run_steps(h, l, rin, st, false);
    }
    // residual + restriction
    Level& C = h->lev[l + 1];
    // the level below the last row-partitioned one is replicated: restrict into this rank's block of
    // it and allgather the blocks (C-gather); prolong from the same block
    const bool gather = Lv.dist && !C.dist;
    const int64_t cb = gather ? C.offs[h->comm->rank] : 0;
    static const int rr_rows = getenv("AMG_FUSE_RR_ROWS") ? atoi(getenv("AMG_FUSE_RR_ROWS")) : kFuseRestrictRows;
    if (!Lv.dist && Lv.A.n < rr_rows) {  // small level: one fused launch
        launch_resid_restrict(Lv.nc, Lv.aptr, Lv.perm, Lv.A, cur, rin, C.RHO, s);
    } else {
        spmv_pass(h, l, cur, [&](const SpOp& op, int) { launch_resid(op, cur, rin, Lv.RES, nullptr, h->ds, s); });
        if (Lv.gx) restrict_global(h, l, Lv.RES, C.RHO + cb);  // members on other ranks included
        else launch_restrict(Lv.nc, Lv.aptr, Lv.perm, Lv.RES, C.RHO + cb, s);
    }
    if (gather) allgatherv_d(h, C.RHO, C.offs);
    if (l == 0) capture_split_point(h);
    // coarse correction (A12: exact solve when the next level is the coarsest)
    // (global aggregation: agg holds global ids of a replicated coarse level, or coarse relative
    // indices -- remote aggregates in the coarse halo -- of a row-partitioned one)
    if (l + 1 == h->L - 1) {  // exact coarsest solve fused with the prolongation
        launch_gemv_prolong(Lv.A.n, Lv.agg, Lv.gx ? 0 : (int)cb, C.A.n, h->Minv, C.RHO, cur, s);
    } else {
        // single-GPU levels: the inner FCG's last E update is fused into the prolongation
        const bool fuse = h->opt.cycle != 2 && !Lv.dist && !C.dist && !Lv.gx;
        int fr = kFcgDone;
        if (h->opt.cycle == 2)
            amli_correction(h, l + 1, nu);
        else
            fr = fcg_inner(h, l + 1, nu, fuse);
        if (fr == kFcgZ) {
            launch_prolong_fcg2(Lv.A.n, Lv.agg, C.D, C.Z, C.sc, cur, s);
        } else if (fr == kFcgDeferred) {
            const int i = nu - 1;
            launch_prolong_fcg(Lv.A.n, Lv.agg, C.E, C.D + (size_t)i * C.ld, C.sc + kMaxWin + i, C.sc + i, i == 0, cur,
                               s);
        } else if (Lv.gx) {
            if (C.dist) halo_exchange(h, l + 1, C.E);
            launch_prolong(Lv.A.n, Lv.agg, C.E, cur, s);
        } else {
            launch_prolong(Lv.A.n, Lv.agg, C.E + cb, cur, s);
        }
    }
    // post-smoothing S(r, x): x_{-1} = x_0 = cur
    double* other = (cur == Lv.X) ? Lv.XA : Lv.X;
    std::vector<SmStep> st;
    st.push_back({cur, cur, 1.0, b[0], other});  // k = 0
    prev = cur;
    cur = other;
    for (int k = 1; k <= m; ++k) {
        double* target = (k == m) ? out : prev;
        st.push_back({cur, prev, a[k], b[k], target});
        prev = cur;
        cur = target;
    }
    // live profile of the dominant kernel: the level-0 post-smoothing launches (all m+1 steps)
    const bool prof = (l == 0 && h->prof_on);
    if (prof) {
        h->prof_win_bytes = 0;
        h->prof_win_launches = 0;
        record_event(h->pe0, s);
    }
    run_steps(h, l, rin, st, prof);
    if (prof) record_event(h->pe1, s);
}

// v -= mean(v) over the whole level-0 vector (A16); the sum is allreduced when partitioned
static void mean_project(amg_hierarchy* h, double* v) {
    double* tmp = h->osc + 2 * kMaxWin + 3;
    if (!h->lev[0].dist) {
        launch_mean_project(h->n, v, tmp, h->ds, h->s);
        return;
    }
    launch_dot(h->n, v, nullptr, tmp, h->ds, h->s);
    dot_allreduce(h, {tmp});
    launch_sub_mean(h->n, (double)h->lev[0].nglob, v, tmp, h->s);
}

// one outer FCG iteration at window position p
static void outer_iteration(amg_hierarchy* h, int pos, int nu) {
    cudaStream_t s = h->s;
    const int n = h->n;
    const size_t ld = h->lev[0].ld;
    const bool dist = h->lev[0].dist;
    double* dq = h->osc;
    double* c = h->osc + kMaxWin;
    double* dr = h->osc + 2 * kMaxWin;
    double* rr = h->osc + 2 * kMaxWin + 1;
    double* Dp = h->D + (size_t)pos * ld;
    double* Qp = h->Q + (size_t)pos * ld;
    double* zdst = (pos == 0) ? Dp : h->Z;
    h->prof_on = true;
    apply_B(h, 0, nu, h->r, zdst);
    h->prof_on = false;
    if (h->singular) mean_project(h, zdst);
    if (pos > 0) {
        const double* Ds[kMaxWin];
        const double* Qs[kMaxWin];
        for (int j = 0; j < pos; ++j) {
            Ds[j] = h->D + (size_t)j * ld;
            Qs[j] = h->Q + (size_t)j * ld;
        }
        launch_multidot(n, h->Z, Qs, pos, c, h->ds, s);
        if (dist) {
            std::vector<double*> cs;
            for (int j = 0; j < pos; ++j) cs.push_back(c + j);
            dot_allreduce(h, cs);
        }
        if (h->xf && pos == h->W - 1)  // the window's deferred x updates ride along (k_direction_xf)
            launch_direction_xf(n, h->Z, Ds, c, dq, pos, Dp, h->x, h->alph, h->xold, s);
        else
            launch_direction(n, h->Z, Ds, c, dq, pos, Dp, s);
    }
    spmv_dots_pass(h, 0, Dp, h->r, Qp, dq + pos, dr);
    // x += alpha d is deferred: the window keeps every d_j, and nothing reads x before the solve ends.
    // With xf the last position's direction applies positions 0..W-2 and the previous window's W-1;
    // otherwise one flush at the end of every window.
    const bool last = pos == h->W - 1;
    launch_fcg_update(n, dr, dq + pos, Dp, Qp, nullptr, false, h->r, rr, h->flag, h->ds, s, h->alph + pos,
                      h->xf && last ? h->xold : nullptr);
    if (!h->xf && last) {
        Slots sl{};
        for (int j = 0; j < h->W; ++j) sl.j[j] = j;
        launch_x_flush(n, h->x, h->D, ld, h->alph, sl, h->W, s);
    }
    if (dist) dot_allreduce(h, {rr});
}

// One graph per restart-window position, captured lazily: position p+1's graph is captured on the
// host while position p's graph runs on the device (capture only records; the stream's pending work
// keeps executing), so the ~0.5 ms per capture + instantiation hides behind the solve.
static void capture_graph(amg_hierarchy* h, int pos, int nu) {
    if (h->graph_nu != nu) {
        destroy_graphs(h);
        h->graphs.assign(h->W, nullptr);
        h->graphs_head.assign(h->W, nullptr);
        h->graph_launches_pos.assign(h->W, 0);
        h->graph_nu = nu;
    }
    if (h->graphs[pos]) return;
    cudaGraph_t g;
    long long before = g_launches;
    CK(cudaStreamBeginCapture(h->s, cudaStreamCaptureModeThreadLocal));
    h->cap_head = nullptr;
    static const bool no_split = getenv("AMG_NO_GRAPH_SPLIT") != nullptr;  // A/B experiments
    h->cap_split = !h->comm && !no_split;  // (row-partitioned levels fork onto the communication stream)
    try {
        outer_iteration(h, pos, nu);
    } catch (...) {
        h->cap_split = false;
        cudaStreamEndCapture(h->s, &g);
        if (h->cap_head) cudaGraphDestroy(h->cap_head);
        h->cap_head = nullptr;
        throw;
    }
    h->cap_split = false;
    CK(cudaStreamEndCapture(h->s, &g));
    h->graph_launches_pos[pos] = g_launches - before;
    h->graph_launches = std::max(h->graph_launches, g_launches - before);  // the fullest window position
    g_launches = before;
    if (h->cap_head) {
        CK(cudaGraphInstantiate(&h->graphs_head[pos], h->cap_head, 0));
        CK(cudaGraphDestroy(h->cap_head));
        h->cap_head = nullptr;
    }
    CK(cudaGraphInstantiate(&h->graphs[pos], g, 0));
    CK(cudaGraphDestroy(g));
}

static int solve(amg_hierarchy* h, const double* b_in, double* x_out, double tol, int nu, int* iters_out,
                 double* relres_out) {
    cudaStream_t s = h->s;
    const int n = h->n;
    if (h->user) {
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CK(cudaEventRecord(ev, h->user));
        CK(cudaStreamWaitEvent(s, ev, 0));
        CK(cudaEventDestroy(ev));
    }
    // graphs need a capturable communicator (NCCL); the thread-emulated ranks run eagerly
    const bool graphs = h->opt.use_graphs && (!h->comm || h->comm->capturable());
    const bool dist = h->lev[0].dist;
    // distributed handle whose whole hierarchy is replicated (g = 0): gather the caller's blocks
    const bool gather_in = h->comm && !dist;
    ensure_inner_ws(h, nu);
    {   // deferred outer x updates: fused into the last window position's direction when it can be
        const double* Ds[kMaxWin];
        for (int j = 0; j < h->W; ++j) Ds[j] = h->D + (size_t)j * h->lev[0].ld;
        const bool xf = h->W >= 2 && direction_xf_ok(h->W - 1, h->Z, Ds, Ds[h->W - 1], h->x);
        if (xf != h->xf) {  // the captured graphs depend on it
            destroy_graphs(h);
            h->xf = xf;
        }
        CK(cudaMemsetAsync(h->xold, 0, sizeof(int), s));
    }
    long long launches0 = g_launches;
    CK(cudaEventRecord(h->e0, s));
    // inputs
    const int64_t own0 = gather_in ? h->row_begin : 0;
    const int nown = gather_in ? h->n_local : n;
    CK(cudaMemcpyAsync(h->b + own0, b_in, sizeof(double) * nown,
                       is_device_ptr(b_in) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(h->x + own0, x_out, sizeof(double) * nown,
                       is_device_ptr(x_out) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    if (gather_in) {
        allgatherv_d(h, h->b, h->lev[0].offs);
        allgatherv_d(h, h->x, h->lev[0].offs);
    }
    double* bb = h->osc + 2 * kMaxWin + 2;
    double* rr = h->osc + 2 * kMaxWin + 1;
    if (h->singular) mean_project(h, h->b);  // S:449, A16
    launch_dot(n, h->b, h->b, bb, h->ds, s);
    halo_exchange(h, 0, h->x);
    launch_resid(h->lev[0].op, h->x, h->b, h->r, rr, h->ds, s);
    if (dist) dot_allreduce(h, {rr, bb});
    CK(cudaMemsetAsync(h->flag, 0, sizeof(double), s));
    CK(cudaMemcpyAsync(h->hsc, rr, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const double bnorm = std::sqrt(h->hsc[1]);
    double rnorm = std::sqrt(h->hsc[0]);
    int status = AMG_NOT_CONVERGED, k = 0;
    long long graph_kernels = 0;  // launches replayed from graphs
    double prof_ms = 0.0;
    int64_t prof_n = 0, prof_bytes = 0;
    if (bnorm == 0.0) {
        CK(cudaMemsetAsync(h->x, 0, sizeof(double) * n, s));
        status = AMG_OK;
        rnorm = 0.0;
    } else {
        // deferred x updates (outer_iteration): pending = this window's positions not yet applied,
        // oldp = the previous window's last position not yet applied (xf mode)
        int pos = 0, pending = 0;
        bool oldp = false;
        for (k = 0;; ++k) {
            if (rnorm <= tol * bnorm) { status = AMG_OK; break; }
            if (k >= h->opt.max_iter) break;
            NvtxRange nv_it("amg outer FCG iteration");
            if (graphs) {
                // A position with no graph yet (the first iteration of a handle's first solve) is
                // launched directly: the device starts at once instead of idling through a capture +
                // instantiation (0.4 ms on C3, 1.6 ms on C4), and the host, which runs ahead of the
                // level-0 kernels, captures the next position's graph behind it.
                static const bool eager_first = getenv("AMG_NO_EAGER_FIRST") == nullptr;  // A/B experiments
                if (h->graph_nu != nu) destroy_graphs(h);
                if (!eager_first && (h->graphs.empty() || !h->graphs[pos])) capture_graph(h, pos, nu);
                if (!h->graphs.empty() && h->graphs[pos]) {
                    if (h->graphs_head[pos]) CK(cudaGraphLaunch(h->graphs_head[pos], s));
                    CK(cudaGraphLaunch(h->graphs[pos], s));
                    graph_kernels += h->graph_launches_pos[pos];
                } else {
                    outer_iteration(h, pos, nu);
                }
                const int nxt = (pos + 1) % h->W;
                if (h->graphs.empty() || !h->graphs[nxt]) capture_graph(h, nxt, nu);  // overlaps this iteration
            } else {
                outer_iteration(h, pos, nu);
            }
            // rr and the breakdown flag in one 32-byte copy: osc slots +1..+4 = rr, bb, (mean scratch), flag
            CK(cudaMemcpyAsync(h->hsc, rr, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (pos == h->W - 1) { pending = 0; oldp = h->xf; } else { pending = pos + 1; }
            int fl;
            memcpy(&fl, h->hsc + 3, sizeof(int));
            if (h->L > 1) {
                float pm = 0.f;
                CK(cudaEventElapsedTime(&pm, h->pe0, h->pe1));
                prof_ms += pm;
                prof_n += h->prof_win_launches;
                prof_bytes += h->prof_win_bytes;
            }
            if (fl) { status = AMG_E_BREAKDOWN; ++k; break; }
            rnorm = std::sqrt(h->hsc[0]);
            pos = (pos + 1) % h->W;
        }
        Slots sl{};
        int cnt = 0;
        if (oldp) sl.j[cnt++] = h->W - 1;  // in iteration order: the previous window's last, then this one's
        for (int j = 0; j < pending; ++j) sl.j[cnt++] = j;
        launch_x_flush(n, h->x, h->D, h->lev[0].ld, h->alph, sl, cnt, s);
    }
    // true residual ||b - A x|| (reported) and the solution back to the caller
    double* rt = h->osc + 2 * kMaxWin + 6;
    halo_exchange(h, 0, h->x);
    launch_resid(h->lev[0].op, h->x, h->b, h->Z, rt, h->ds, s);
    if (dist) dot_allreduce(h, {rt});
    copy_out(x_out, h->x + own0, sizeof(double) * nown, s);
    CK(cudaEventRecord(h->e1, s));
    CK(cudaMemcpyAsync(h->hsc + 3, rt, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->e0, h->e1));
    h->info.solve_ms = ms;
    h->info.last_iters = k;
    h->info.last_relres = bnorm > 0 ? rnorm / bnorm : 0.0;
    h->info.last_true_relres = bnorm > 0 ? std::sqrt(h->hsc[3]) / bnorm : 0.0;
    h->info.launches_last_solve = (g_launches - launches0) + graph_kernels;
    h->info.launches_per_iter = h->graph_launches;
    h->info.prof_smoother_ms = prof_ms;
    h->info.prof_smoother_launches = prof_n;
    h->info.prof_smoother_bytes = prof_n ? prof_bytes / prof_n : smoother_bytes(h->lev[0]);
    if (h->user) {  // order the caller's stream after this call's work
        CK(cudaEventRecord(h->e1, s));
        CK(cudaStreamWaitEvent(h->user, h->e1, 0));
    }
    if (iters_out) *iters_out = k;
    if (relres_out) *relres_out = h->info.last_relres;
    if (status == AMG_E_BREAKDOWN) g_last_error = "FCG breakdown: d.q <= 0 or not finite";
    return status;
}

// ------------------------------------------------------------------ C ABI
extern "C" {

int amg_options_default(amg_options* o) {
    if (!o) return fail(AMG_E_ARG, "amg_options_default: NULL");
    memset(o, 0, sizeof(*o));
    o->coarsest_size = 100;
    o->kappa = 0.0;
    o->restart = 5;
    o->max_iter = 500;
    o->seed = 0;
    o->stream = nullptr;
    o->use_graphs = 1;
    o->tail_nnz = 8192;
    o->dense_b_rows = 4096;
    o->global_agg = 0;
    o->tail_smem = 2;  // greedy placement, matrices first: C4 -5%, C1/C2 -2%, C3/C5 neutral
    o->compress = 1;
    o->gather_rows = 50000;
    return AMG_OK;
}

const char* amg_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"

// amg_setup / amg_setup_dist: comm == nullptr is the single-GPU path (n_global = n_local, row_begin 0)
static int setup_impl(amg_handle* out, amg_comm comm, int64_t n_global, int64_t row_begin, int64_t n,
                      const int64_t* row_ptr, const int32_t* col, const double* val, const double* d,
                      int32_t n_match_passes, int32_t poly_degree, const amg_options* opt) {
    if (!out) return fail(AMG_E_ARG, "amg_setup: out is NULL");
    *out = nullptr;
    if (!row_ptr || !val || !col) return fail(AMG_E_ARG, "amg_setup: NULL array");
    if (n_match_passes < 1 || n_match_passes > kMaxDeg) return fail(AMG_E_ARG, "amg_setup: n_match_passes out of range");
    if (poly_degree < 1 || poly_degree > kMaxDeg) return fail(AMG_E_ARG, "amg_setup: poly_degree out of range");
    amg_options o;
    amg_options_default(&o);
    if (opt) o = *opt;
    if (o.coarsest_size < 1 || o.restart < 1 || o.restart > kMaxWin || o.max_iter < 0 || o.gather_rows < 0)
        return fail(AMG_E_ARG, "amg_setup: bad options");
    if (o.cycle != 0 && o.cycle != 2) return fail(AMG_E_ARG, "amg_setup: cycle must be 0 (k-cycle) or 2 (AMLI)");
    if (o.tail_smem < 0 || o.tail_smem > 2) return fail(AMG_E_ARG, "amg_setup: tail_smem must be 0, 1 or 2");
    if (o.amli_kappa != 0.0 && !(o.amli_kappa > 1.0)) return fail(AMG_E_ARG, "amg_setup: amli_kappa must be 0 or > 1");
    if (comm && !comm->c) return fail(AMG_E_ARG, "amg_setup_dist: invalid communicator");
    if (o.lanczos_steps < 0 || o.lanczos_steps > 64 || (comm && o.lanczos_steps > 0))
        return fail(AMG_E_ARG, "amg_setup: lanczos_steps must be in [0, 64] (single GPU only)");
    if (o.mis_k < 0 || o.mis_k > 8 || (comm && o.mis_k > 0))
        return fail(AMG_E_ARG, "amg_setup: mis_k must be in [0, 8] (single GPU only)");
    if (o.kappa != 0.0 && !(o.kappa > 1.0)) return fail(AMG_E_ARG, "amg_setup: kappa must be 0 or > 1");
    if (o.kappa > 1.0 && !(Em_of(poly_degree, o.kappa) < 1.0))
        return fail(AMG_E_ARG, "amg_setup: E_m(kappa) >= 1: the smoother would not converge (reading A9)");
    NvtxRange nv(comm ? "amg_setup_dist" : "amg_setup");
    amg_hierarchy* h = new amg_hierarchy();
    try {
        init_device_props();
        {   // keep freed stream-ordered memory in the pool (default threshold 0 unmaps it at every sync)
            int dev = 0;
            cudaMemPool_t pool;
            CK(cudaGetDevice(&dev));
            CK(cudaDeviceGetDefaultMemPool(&pool, dev));
            uint64_t thr = UINT64_MAX;
            CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        }
        h->opt = o;
        h->m = poly_degree;
        h->p = n_match_passes;
        h->user = (cudaStream_t)o.stream;
        {   // the handle's own non-blocking library stream (recycled, see stream_acquire)
            int dev = 0;
            CK(cudaGetDevice(&dev));
            if (dev < 0 || dev >= 64) throw Error(AMG_E_ARG, "device ordinal out of range");
            h->dev = dev;
            h->s = stream_acquire(dev);
        }
        h->no_zform = getenv("AMG_NO_ZFORM") != nullptr;
        CK(cudaEventCreate(&h->e0));
        CK(cudaEventCreate(&h->e1));
        CK(cudaEventCreate(&h->pe0));
        CK(cudaEventCreate(&h->pe1));
        if (h->user) {
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, h->user));
            CK(cudaStreamWaitEvent(h->s, ev, 0));
            CK(cudaEventDestroy(ev));
        }
        CK(cudaEventRecord(h->e0, h->s));
        long long l0 = g_launches;
        if (comm) {
            h->comm = comm->c;
            build_dist(h, n_global, row_begin, (int)n, row_ptr, col, val, d);
        } else {
            build(h, n, row_ptr, col, val, d);
        }
        h->info.launches_last_setup = g_launches - l0;
        CK(cudaEventRecord(h->e1, h->s));
        CK(cudaEventSynchronize(h->e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->e0, h->e1));
        h->info.setup_ms = ms;
        if (h->user) CK(cudaStreamWaitEvent(h->user, h->e1, 0));
    } catch (const Error& e) {
        g_last_error = e.what();
        cudaGetLastError();
        // argument, input and stagnation errors are collective decisions (every rank throws them);
        // any other error is local: wake and fail the other ranks instead of leaving them waiting
        if (h->comm && e.code != AMG_E_NCCL && e.code != AMG_E_ARG && e.code != AMG_E_INPUT && e.code != AMG_E_SETUP)
            h->comm->abort();
        release(h);
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        if (h->comm) h->comm->abort();
        release(h);
        return AMG_E_CUDA;
    }
    *out = h;
    return AMG_OK;
}

extern "C" {

int amg_setup(amg_handle* out, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
              const double* d, int32_t n_match_passes, int32_t poly_degree, const amg_options* opt) {
    return setup_impl(out, nullptr, n, 0, n, row_ptr, col, val, d, n_match_passes, poly_degree, opt);
}

int amg_setup_dist(amg_handle* out, amg_comm comm, int64_t n_global, int64_t row_begin, int64_t n_local,
                   const int64_t* row_ptr, const int32_t* col_global, const double* val, const double* d,
                   int32_t n_match_passes, int32_t poly_degree, const amg_options* opt) {
    if (!comm) return fail(AMG_E_ARG, "amg_setup_dist: comm is NULL");
    return setup_impl(out, comm, n_global, row_begin, n_local, row_ptr, col_global, val, d, n_match_passes,
                      poly_degree, opt);
}

int amg_solve(amg_handle h, const double* b, double* x, double tol, int32_t k_inner, int32_t* iters, double* relres) {
    if (!h || !b || !x) return fail(AMG_E_ARG, "amg_solve: NULL argument");
    if (!(tol > 0.0) || k_inner < 1 || k_inner > kMaxWin) return fail(AMG_E_ARG, "amg_solve: bad tol or k_inner");
    NvtxRange nv("amg_solve");
    try {
        int it = 0;
        int st = solve(h, b, x, tol, k_inner, &it, relres);
        if (iters) *iters = it;
        return st;
    } catch (const Error& e) {
        g_last_error = e.what();
        cudaGetLastError();
        if (h->comm && e.code != AMG_E_NCCL) h->comm->abort();
        return e.code;
    }
}

int amg_free(amg_handle h) {
    if (!h) return AMG_OK;
    NvtxRange nv("amg_free");
    release(h);
    return AMG_OK;
}

int amg_get_info(amg_handle h, amg_info* info) {
    if (!h || !info) return fail(AMG_E_ARG, "amg_get_info: NULL argument");
    amg_info r = h->info;
    r.levels = h->L;
    r.poly_degree = h->m;
    r.n_match_passes = h->p;
    r.singular = h->singular;
    double sn = 0, snz = 0;  // whole-level sizes (summed over the ranks on a row-partitioned level)
    for (int l = 0; l < h->L; ++l) {
        sn += (double)h->lev[l].nglob;
        snz += (double)h->lev[l].nnz_glob;
        if (l < 32) {
            r.n[l] = h->lev[l].nglob;
            r.nnz[l] = h->lev[l].nnz_glob;
            r.lambda1[l] = h->lev[l].lambda1;
            r.kappa[l] = h->lev[l].kappa;
        }
    }
    r.grid_complexity = sn / (double)h->lev[0].nglob;
    r.operator_complexity = snz / (double)h->lev[0].nnz_glob;
    r.nranks = h->comm ? h->comm->size : 1;
    r.dist_levels = h->comm ? h->g : 0;
    r.device_bytes = h->bytes;
    {
        const Level& L0 = h->lev[0];
        r.level0_format = !L0.op.sell ? 0 : ((L0.S.vmode || L0.S.cmode) ? 2 : 1);
        r.level0_path = (tma_eligible(L0.split ? L0.op_int : L0.op) ? 1 : 0) | (L0.split ? 2 : 0);
    }
    *info = r;
    return AMG_OK;
}

// ---- parity hooks ----
int amg_level_sizes(amg_handle h, int32_t level, int64_t* n, int64_t* nnz, int64_t* nc, double* lambda1,
                    double* kappa, double* alpha, double* beta) {
    if (!h || level < 0 || level >= h->L) return fail(AMG_E_ARG, "amg_level_sizes: bad level");
    const Level& Lv = h->lev[level];
    if (n) *n = Lv.A.n;
    if (nnz) *nnz = Lv.A.nnz;
    if (nc) *nc = (level < h->L - 1) ? Lv.nc : 0;
    if (lambda1) *lambda1 = Lv.lambda1;
    if (kappa) *kappa = Lv.kappa;
    if (alpha) memcpy(alpha, Lv.alpha, sizeof(double) * (h->m + 1));
    if (beta) memcpy(beta, Lv.beta, sizeof(double) * (h->m + 1));
    return AMG_OK;
}

int amg_level_export(amg_handle h, int32_t level, int64_t* row_ptr, int32_t* col, double* val, int32_t* agg) {
    if (!h || level < 0 || level >= h->L) return fail(AMG_E_ARG, "amg_level_export: bad level");
    try {
        const Level& Lv = h->lev[level];
        cudaStream_t s = h->s;
        if (row_ptr) {
            std::vector<int> tmp((size_t)Lv.A.n + 1);
            CK(cudaMemcpyAsync(tmp.data(), Lv.A.rp, sizeof(int) * tmp.size(), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            std::vector<int64_t> w(tmp.begin(), tmp.end());
            CK(cudaMemcpy(row_ptr, w.data(), sizeof(int64_t) * w.size(),
                          is_device_ptr(row_ptr) ? cudaMemcpyHostToDevice : cudaMemcpyHostToHost));
        }
        if (Lv.dist) {  // global column ids and global coarse ids
            int* tmp = dalloc<int>((size_t)std::max<int64_t>(Lv.A.nnz, Lv.A.n) + 8, s);
            if (col) {
                export_dist_cols(h, level, tmp);
                copy_out(col, tmp, sizeof(int) * Lv.A.nnz, s);
            }
            if (agg && level < h->L - 1) {
                export_dist_agg(h, level, tmp);
                copy_out(agg, tmp, sizeof(int) * Lv.A.n, s);
            }
            CK(cudaStreamSynchronize(s));
            dfree(tmp, s);
        } else {
            if (col) copy_out(col, Lv.A.ci, sizeof(int) * Lv.A.nnz, s);
            if (agg && level < h->L - 1) copy_out(agg, Lv.agg, sizeof(int) * Lv.A.n, s);
        }
        if (val) copy_out(val, Lv.A.v, sizeof(double) * Lv.A.nnz, s);
        CK(cudaStreamSynchronize(s));
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    }
    return AMG_OK;
}

int amg_level_smooth(amg_handle h, int32_t level, const double* f, const double* x0, double* x) {
    if (!h || level < 0 || level >= h->L - 1 || !f || !x0 || !x) return fail(AMG_E_ARG, "amg_level_smooth: bad args");
    try {
        Level& Lv = h->lev[level];
        cudaStream_t s = h->s;
        const int n = Lv.A.n;
        double* F = dalloc<double>((size_t)n + 8, s);
        double* O = dalloc<double>((size_t)n + 8, s);
        CK(cudaMemcpyAsync(F, f, sizeof(double) * n, cudaMemcpyDefault, s));
        CK(cudaMemcpyAsync(Lv.X, x0, sizeof(double) * n, cudaMemcpyDefault, s));
        // S(f, x0): x_{-1} = x_0
        double* cur = Lv.X;
        double* other = Lv.XA;
        halo_exchange(h, level, cur);
        launch_smooth(Lv.op, cur, 1.0, F, cur, 0.0, 1.0, Lv.beta[0], other, s);
        double* prev = cur;
        cur = other;
        for (int k = 1; k <= h->m; ++k) {
            double* target = (k == h->m) ? O : prev;
            halo_exchange(h, level, cur);
            launch_smooth(Lv.op, cur, 1.0, F, prev, 0.0, Lv.alpha[k], Lv.beta[k], target, s);
            prev = cur;
            cur = target;
        }
        copy_out(x, cur, sizeof(double) * n, s);
        CK(cudaStreamSynchronize(s));
        dfree(F, s);
        dfree(O, s);
        CK(cudaStreamSynchronize(s));
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    }
    return AMG_OK;
}

int amg_level_precond(amg_handle h, int32_t level, int32_t k_inner, const double* r, double* z) {
    if (!h || level < 0 || level >= h->L || !r || !z || k_inner < 1 || k_inner > kMaxWin)
        return fail(AMG_E_ARG, "amg_level_precond: bad args");
    try {
        cudaStream_t s = h->s;
        ensure_inner_ws(h, k_inner);
        Level& Lv = h->lev[level];
        const int n = Lv.A.n;
        // R in the level's vector layout (its halo is exchanged by the first smoothing step)
        double* Rb = dalloc<double>((size_t)std::max(Lv.ld, n) + 8, s);
        double* R = Rb + Lv.lo_pad;
        double* O = dalloc<double>((size_t)n + 8, s);
        CK(cudaMemcpyAsync(R, r, sizeof(double) * n, cudaMemcpyDefault, s));
        apply_B(h, level, k_inner, R, O);
        copy_out(z, O, sizeof(double) * n, s);
        CK(cudaStreamSynchronize(s));
        dfree(Rb, s);
        dfree(O, s);
        CK(cudaStreamSynchronize(s));
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    }
    return AMG_OK;
}

int amg_level_dist(amg_handle h, int32_t level, int32_t* dist, int64_t* row_begin, int64_t* n_global) {
    if (!h || level < 0 || level >= h->L) return fail(AMG_E_ARG, "amg_level_dist: bad level");
    const Level& Lv = h->lev[level];
    if (dist) *dist = Lv.dist ? 1 : 0;
    if (row_begin) *row_begin = Lv.dist ? Lv.gbeg : 0;
    if (n_global) *n_global = Lv.nglob;
    return AMG_OK;
}

int amg_coarse_solve(amg_handle h, const double* r, double* e) {
    if (!h || !r || !e) return fail(AMG_E_ARG, "amg_coarse_solve: bad args");
    try {
        cudaStream_t s = h->s;
        const int n = h->lev[h->L - 1].A.n;
        double* R = dalloc<double>((size_t)n + 8, s);
        double* O = dalloc<double>((size_t)n + 8, s);
        CK(cudaMemcpyAsync(R, r, sizeof(double) * n, cudaMemcpyDefault, s));
        launch_gemv(n, h->Minv, R, O, s);
        copy_out(e, O, sizeof(double) * n, s);
        CK(cudaStreamSynchronize(s));
        dfree(R, s);
        dfree(O, s);
    } catch (const Error& e2) {
        g_last_error = e2.what();
        return e2.code;
    }
    return AMG_OK;
}

}  // extern "C"
