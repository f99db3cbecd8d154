// k_solve.cu -- solve-phase kernels of libamg_b200.so (sm_100a): the hot path of SURVEY.md 8(a)
// rows a9-a16.  HBM-bound fp64 CSR work; no tensor cores (nothing here is a dense contraction).
//
//  * SpMV-class kernels (smoother step a9, residual a10, SpMV+dots a15) share one tiled,
//    grid-stride kernel: each tile's contiguous col/val run is streamed into shared memory with
//    16-byte non-allocating loads (coalesced), then one thread per row reduces its row from shared
//    memory, gathers x through the read-only path, and runs the fused epilogue (three-term update,
//    residual, dots).  One pass over A per smoother degree step.
//  * Reductions are deterministic: per-block partials in a fixed order, the last block to finish
//    (atomic ticket) sums them in a fixed order and resets the ticket.
//  * Restriction (a11) is a per-aggregate sequential sum over the aggregate-sorted order; the
//    prolongation (a12) is fused with its axpy.
#include <cuda_runtime.h>

#include <cstdlib>

#include "amg_internal.h"

namespace amg {

thread_local long long g_launches = 0;
static int g_num_sms = 148;

void init_device_props() {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
}

int vector_grid() { return g_num_sms * 4; }

// grid of a grid-stride vector kernel over n work units (elements, double2 pairs, int4 quads, or
// aggregates): one unit per thread while that fits in 8 CTAs of 256 threads per SM, grid-stride
// beyond.  Small (coarse-level) vectors are latency-bound: spreading them over every SM is what
// helps; large ones want the full 2048 threads per SM in flight (tools/vec_micro.cu: 4 CTAs/SM left
// too few loads in flight on C3's level 0 -- fcg_update 160 -> 125 us, multidot(4) 219 -> 97 us).
static int vgrid(int64_t n) {
    int64_t g = (n + kBlock - 1) / kBlock;
    if (g > 2 * vector_grid()) g = 2 * vector_grid();
    return g < 1 ? 1 : (int)g;
}

static bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ double2 ld_stream(const double2* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ int4 ld_stream(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum (fixed order => deterministic).  All threads get the result.
__device__ double block_sum(double v) {
    __shared__ double red[32];
    __shared__ double total;
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double t = lane < nw ? red[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) total = t;
    }
    __syncthreads();
    return total;
}

struct DotOut {
    double* p[4];
};

// Two-stage deterministic reduction of ND per-thread accumulators into *out.p[k], k < ND.
template <int ND>
__device__ void finalize_dots(double (&acc)[ND], double* partials, unsigned* ticket, DotOut out) {
    __shared__ bool amlast;
    const int G = gridDim.x;
#pragma unroll
    for (int k = 0; k < ND; ++k) {
        double b = block_sum(acc[k]);
        if (threadIdx.x == 0) partials[k * G + blockIdx.x] = b;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) amlast = (atomicAdd(ticket, 1u) == (unsigned)(G - 1));
    __syncthreads();
    if (amlast) {
        __threadfence();
#pragma unroll
        for (int k = 0; k < ND; ++k) {
            double v = 0.0;
            for (int b = threadIdx.x; b < G; b += blockDim.x) v += __ldcg(partials + k * G + b);
            v = block_sum(v);
            if (threadIdx.x == 0) *out.p[k] = v;
        }
        if (threadIdx.x == 0) *ticket = 0u;
    }
}

// ------------------------------------------------------------------ epilogues
// Each epilogue splits into load(i) -- the row's vector operands, issued BEFORE the matrix stream
// and the dependent x gathers so their DRAM latency overlaps -- and store(i, s, x_i, pre, acc).
// The read-only streaming loads (.nc, no L1 allocate) are safe even when `out` aliases `xprev`:
// every element is read and then written by the same thread only.
__device__ __forceinline__ double ld_nc(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

struct EpiSmooth {  // three-term recurrence step, optional implicit x_{k-1} = cp*f
    const double* f;
    const double* xprev;
    double* out;
    double alpha, beta, cg, cp;
    static constexpr int ND = 0;
    struct Pre { double fi, prev; };
    __device__ __forceinline__ Pre load(int i) const {
        Pre p;
        p.fi = ld_nc(f + i);
        p.prev = xprev ? ld_nc(xprev + i) : cp * p.fi;
        return p;
    }
    __device__ __forceinline__ void store(int i, double s, double xgi, const Pre& p, double*) const {
        out[i] = alpha * (cg * xgi) + (1.0 - alpha) * p.prev + beta * (p.fi - cg * s);
    }
};

struct EpiResid {  // out = f - A x; acc[0] += out^2 (reduced only when a dot pointer is given)
    const double* f;
    double* out;
    static constexpr int ND = 1;
    struct Pre { double fi; };
    __device__ __forceinline__ Pre load(int i) const { return Pre{ld_nc(f + i)}; }
    __device__ __forceinline__ void store(int i, double s, double, const Pre& p, double* acc) const {
        double r = p.fi - s;
        out[i] = r;
        acc[0] += r * r;
    }
};

struct EpiSpmvDots {  // q = A d; acc = (d.q, d.rho)
    const double* rho;
    double* q;
    static constexpr int ND = 2;
    struct Pre { double ri; };
    __device__ __forceinline__ Pre load(int i) const { return Pre{ld_nc(rho + i)}; }
    __device__ __forceinline__ void store(int i, double s, double di, const Pre& p, double* acc) const {
        q[i] = s;
        acc[0] += di * s;
        acc[1] += di * p.ri;
    }
};

// The last inner-FCG iteration for nu = 2 without materialising d_1 = z - beta_0 d_0 (driver.cu
// fcg_inner): (A z)_i is formed and consumed, never stored; acc = (z.Az, z.q_0, z.rho_1)
struct EpiZDots {
    const double* q0;
    const double* rho;
    static constexpr int ND = 3;
    struct Pre { double q, r; };
    __device__ __forceinline__ Pre load(int i) const { return Pre{ld_nc(q0 + i), ld_nc(rho + i)}; }
    __device__ __forceinline__ void store(int, double s, double zi, const Pre& p, double* acc) const {
        acc[0] += zi * s;
        acc[1] += zi * p.q;
        acc[2] += zi * p.r;
    }
};

// ------------------------------------------------------------------ tiled SpMV-class kernel
// Shared memory per block: cap+2 doubles and cap+4 ints (16-byte aligned staging of the tile's
// col/val run from the 16-byte-aligned chunk containing its first entry).
template <class Epi, bool DOTS>
__global__ void __launch_bounds__(kBlock) k_tiled(Csr A, const double* __restrict__ xg,
                                                  const int* __restrict__ tile_row, int ntiles, int cap, Epi epi,
                                                  double* partials, unsigned* ticket, DotOut dot_out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* sv = reinterpret_cast<double*>(smem_raw);
    int* sc = reinterpret_cast<int*>(sv + cap + 2);
    double acc[Epi::ND > 0 ? Epi::ND : 1];
#pragma unroll
    for (int k = 0; k < (Epi::ND > 0 ? Epi::ND : 1); ++k) acc[k] = 0.0;
    const int* __restrict__ rp = A.rp;
    const int* __restrict__ ci = A.ci;
    const double* __restrict__ va = A.v;

    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int r0 = tile_row[t], r1 = tile_row[t + 1];
        const int p0 = rp[r0], p1 = rp[r1];
        if (p1 - p0 <= cap) {
            const int a0 = p0 & ~1;
            const int nv2 = (p1 - a0 + 1) >> 1;
            const double2* gv = reinterpret_cast<const double2*>(va + a0);
            double2* sv2 = reinterpret_cast<double2*>(sv);
            const int c0 = p0 & ~3;
            const int nc4 = (p1 - c0 + 3) >> 2;
            const int4* gc = reinterpret_cast<const int4*>(ci + c0);
            int4* sc4 = reinterpret_cast<int4*>(sc);
            for (int k = threadIdx.x; k < nv2; k += kBlock) sv2[k] = ld_stream(gv + k);
            for (int k = threadIdx.x; k < nc4; k += kBlock) sc4[k] = ld_stream(gc + k);
            __syncthreads();
            for (int i = r0 + threadIdx.x; i < r1; i += kBlock) {
                const typename Epi::Pre pre = epi.load(i);
                const double xi = __ldg(xg + i);
                const int q0 = rp[i], q1 = rp[i + 1];
                double s = 0.0;
                for (int q = q0; q < q1; ++q) s = fma(sv[q - a0], __ldg(xg + sc[q - c0]), s);
                epi.store(i, s, xi, pre, acc);
            }
            __syncthreads();
        } else {  // single long row: block-wide reduction straight from global memory
            double s = 0.0;
            for (int q = p0 + threadIdx.x; q < p1; q += kBlock) s = fma(va[q], __ldg(xg + ci[q]), s);
            s = block_sum(s);
            if (threadIdx.x == 0) epi.store(r0, s, __ldg(xg + r0), epi.load(r0), acc);
            __syncthreads();
        }
    }
    if constexpr (DOTS) finalize_dots<Epi::ND>(acc, partials, ticket, dot_out);
}

// ------------------------------------------------------------------ SELL-32 kernel
// Warp per 32-row slice, grid-stride over slices.  Lane l owns row 32 s + l; entry j of the slice
// lives at 32 (sptr[s] + j) + l, so every load instruction of the warp is one contiguous 256-byte
// (values) or 128-byte (columns) run: fully coalesced, no shared memory, no block barriers.  All
// column/value loads of an 8-entry chunk are issued before the dependent x gathers.
__device__ __forceinline__ int ld_stream_i(const int* p) {
    int r;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ double ld_stream_d(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}
// read-only gather through L1 (x of the SpMV: neighbours share lines); volatile so that the
// source order -- all column/value loads of a chunk, then all gathers -- is the issue order
__device__ __forceinline__ double ld_gather(const double* p) {
    double r;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

__device__ __forceinline__ int ld_stream_u8(const uint8_t* p) {
    int r;
    asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ int ld_stream_u16(const uint16_t* p) {
    int r;
    asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ int ld_stream_s16(const int16_t* p) {
    int r;
    asm volatile("ld.global.nc.L1::no_allocate.s16 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

// Operand streams of one SELL level in one of its storage formats:
//   VM = 0: fp64 values;  VM = 1: uint8 codes into the value dictionary (shared memory)
//   CM = 0: int32 columns; CM = 1: uint8 codes into the offset dictionary; CM = 2: int16 offsets
template <int VM, int CM>
struct SellOps {
    const double* __restrict__ val;     // VM = 0
    const uint8_t* __restrict__ vcode;  // VM = 1
    const int* __restrict__ col;        // CM = 0
    const uint8_t* __restrict__ ccode;  // CM = 1
    const int16_t* __restrict__ coff;   // CM = 2
    const uint16_t* __restrict__ pcode; // CM = 3: (value code | column code << 8), one load per entry
    const double* sv;  // shared-memory value dictionary (VM = 1)
    const int* sc;     // shared-memory offset dictionary (CM = 1)
    int i;             // the lane's row
    int chi;           // last valid column: n - 1, or n + nhi - 1 on a row-partitioned level (halo above)
    __device__ __forceinline__ void load_val(size_t e, double& v, int& vraw) const {
        if constexpr (CM == 3) vraw = ld_stream_u16(pcode + e);
        else if constexpr (VM == 0) v = ld_stream_d(val + e);
        else vraw = ld_stream_u8(vcode + e);
    }
    // CM = 3 takes the column code from the pair already loaded by load_val
    __device__ __forceinline__ int load_col(size_t e, int vraw) const {
        if constexpr (CM == 0) return ld_stream_i(col + e);
        else if constexpr (CM == 1) return ld_stream_u8(ccode + e);
        else if constexpr (CM == 2) return ld_stream_s16(coff + e);
        else return vraw >> 8;
    }
    __device__ __forceinline__ int column(int craw) const {
        if constexpr (CM == 0) return craw;
        else {
            const int c = i + ((CM == 1 || CM == 3) ? sc[craw] : craw);
            return c < chi ? c : chi;  // lanes past n (last slice) read a valid element
        }
    }
    __device__ __forceinline__ double value(double v, int vraw) const {
        if constexpr (VM == 0) return v;
        else if constexpr (CM == 3) return sv[vraw & 0xff];
        else return sv[vraw];
    }
};

// Straight-line row reduction for a fixed slice width W, scheduled as: all W value loads, all W
// column loads, then (after every stream load has arrived) all W gathers, then the FMA chain in CSR
// order.  `z` is an always-zero term that depends on every stream load, so ptxas cannot hoist a
// gather between them and stall the warp before all streams of the slice are in flight.
template <int W, int VM, int CM>
__device__ __forceinline__ double sell_row(const SellOps<VM, CM>& ops, size_t e0, const double* __restrict__ xg) {
    int c[W], vr[W];
    double v[W], x[W];
#pragma unroll
    for (int u = 0; u < W; ++u) ops.load_val(e0 + (size_t)u * 32, v[u], vr[u]);
#pragma unroll
    for (int u = 0; u < W; ++u) c[u] = ops.load_col(e0 + (size_t)u * 32, vr[u]);
    // columns are >= -2^30 (halo below the own rows of a row-partitioned level; setup checks
    // nlo < 2^30), so the OR of any set of them (and of the non-negative codes) is >= -2^30
    int all = 0, vdep = -1;
#pragma unroll
    for (int u = 0; u < W; ++u) {
        c[u] = ops.column(c[u]);
        all |= c[u];
        if constexpr (VM == 0) vdep &= __double2hiint(v[u]); else all |= vr[u];
    }
    // z == 0 always (the OR of columns and codes is >= -2^30; no stored value has the NaN high word 0x7ff80001),
    // but it depends on every column and value load, so every stream load is issued before any gather
    const int z = (all < -(1 << 30) || vdep == 0x7ff80001) ? 1 : 0;
#pragma unroll
    for (int u = 0; u < W; ++u) x[u] = ld_gather(xg + (c[u] | z));
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < W; ++u) s = fma(ops.value(v[u], vr[u]), x[u], s);
    return s;
}

// generic width: straight-line chunks of 8 entries, then a straight-line remainder (0..7)
template <int VM, int CM>
__device__ __noinline__ double sell_row_any(const SellOps<VM, CM> ops, size_t e0, const double* __restrict__ xg,
                                            int w) {
    double s = 0.0;
    int j = 0;
    for (; j + 8 <= w; j += 8) s += sell_row<8, VM, CM>(ops, e0 + (size_t)j * 32, xg);
    const size_t er = e0 + (size_t)j * 32;
    switch (w - j) {
        case 1: s += sell_row<1, VM, CM>(ops, er, xg); break;
        case 2: s += sell_row<2, VM, CM>(ops, er, xg); break;
        case 3: s += sell_row<3, VM, CM>(ops, er, xg); break;
        case 4: s += sell_row<4, VM, CM>(ops, er, xg); break;
        case 5: s += sell_row<5, VM, CM>(ops, er, xg); break;
        case 6: s += sell_row<6, VM, CM>(ops, er, xg); break;
        case 7: s += sell_row<7, VM, CM>(ops, er, xg); break;
        default: break;
    }
    return s;
}

// Width dispatch limited to the level's maximum slice width bucket WMAX (5, 8, 12, 16, or 0 = generic):
// ptxas sizes the register file for the largest straight-line case compiled in, so a level whose
// slices are all <= 5 wide must not carry the 12-wide case (80 vs ~48 registers, 3 vs 5 CTAs/SM).
template <int WMAX, int VM, int CM>
__device__ __forceinline__ double sell_row_w(const SellOps<VM, CM>& ops, size_t e0, const double* __restrict__ xg,
                                             int w) {
    if constexpr (WMAX == 0) {
        return sell_row_any<VM, CM>(ops, e0, xg, w);
    } else {
        switch (w) {
            case 0: return 0.0;
            case 1: return sell_row<1>(ops, e0, xg);
            case 2: return sell_row<2>(ops, e0, xg);
            case 3: return sell_row<3>(ops, e0, xg);
            case 4: return sell_row<4>(ops, e0, xg);
            case 5: return sell_row<5>(ops, e0, xg);
            default: break;
        }
        if constexpr (WMAX >= 8) {
            switch (w) {
                case 6: return sell_row<6>(ops, e0, xg);
                case 7: return sell_row<7>(ops, e0, xg);
                case 8: return sell_row<8>(ops, e0, xg);
                default: break;
            }
        }
        if constexpr (WMAX >= 12) {
            switch (w) {
                case 9: return sell_row<9>(ops, e0, xg);
                case 10: return sell_row<10>(ops, e0, xg);
                case 11: return sell_row<11>(ops, e0, xg);
                case 12: return sell_row<12>(ops, e0, xg);
                default: break;
            }
        }
        if constexpr (WMAX >= 16) {
            switch (w) {
                case 13: return sell_row<13>(ops, e0, xg);
                case 14: return sell_row<14>(ops, e0, xg);
                case 15: return sell_row<15>(ops, e0, xg);
                case 16: return sell_row<16>(ops, e0, xg);
                default: break;
            }
        }
        return 0.0;  // unreachable: every slice of the level is at most WMAX wide (S.wmax, setup)
    }
}

// (the generic-width instance, C4's level 1, is latency-bound on its gathers -- ncu: L1/TEX 81% busy,
// 29% issue, 64 registers = 4 CTAs/SM -- but capping it at 48 / 40 registers for 5 / 6 CTAs/SM
// spilled and was slower: 64.0 / 69.3 us per step against 61.9)
template <class Epi, bool DOTS, int VM, int CM, int WMAX>
__global__ void __launch_bounds__(kBlock) k_sell(Sell S, const double* __restrict__ xg, Epi epi, double* partials,
                                                 unsigned* ticket, DotOut dot_out) {
    __shared__ double sv[VM ? 256 : 1];
    __shared__ int sc[(CM == 1 || CM == 3) ? 256 : 1];  // the dictionaries are constant: load them before waiting on the predecessor
    if constexpr (VM == 1)
        for (int k = threadIdx.x; k < S.nvdict; k += blockDim.x) sv[k] = S.vdict[k];
    if constexpr (CM == 1 || CM == 3)
        for (int k = threadIdx.x; k < S.ncdict; k += blockDim.x) sc[k] = S.cdict[k];
    if constexpr (VM == 1 || CM == 1 || CM == 3) __syncthreads();
    double acc[Epi::ND > 0 ? Epi::ND : 1];
#pragma unroll
    for (int k = 0; k < (Epi::ND > 0 ? Epi::ND : 1); ++k) acc[k] = 0.0;
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    int sl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    // slice bounds are software-pipelined: the next slice's sptr pair is fetched while this slice
    // streams, so every slice costs two dependent memory round trips (streams, then gathers)
    int b = 0, e = 0;
    if (sl < S.nslices) { b = __ldg(S.sptr + sl); e = __ldg(S.sptr + sl + 1); }
    for (; sl < S.nslices; sl += nwarps) {
        const int sn = sl + nwarps;
        int bn = 0, en = 0;
        if (sn < S.nslices) { bn = __ldg(S.sptr + sn); en = __ldg(S.sptr + sn + 1); }
        const int i = S.srow0 + sl * 32 + lane;
        const bool act = i < S.n;
        const SellOps<VM, CM> ops{S.val, S.vcode, S.col, S.ccode, S.coff, S.pcode, sv, sc, i, S.chi};
        typename Epi::Pre pre{};
        double xi = 0.0;
        if (act) {  // independent row operands first (their latency overlaps the matrix stream)
            pre = epi.load(i);
            xi = ld_gather(xg + i);
        }
        const double sum = sell_row_w<WMAX>(ops, (size_t)b * 32 + lane, xg, e - b);  // width is warp-uniform
        if (act) epi.store(i, sum, xi, pre, acc);
        b = bn;
        e = en;
    }
    if constexpr (DOTS) finalize_dots<Epi::ND>(acc, partials, ticket, dot_out);
}

// ------------------------------------------------------------------ TMA-staged smoother step
// The fused three-term step on a SELL level whose slices are all <= W wide, with every STREAM (the
// slice's value/column code runs, f, x_{k-1} and the x_k tile of the chunk's own rows) moved by the
// bulk-copy engine (cp.async.bulk global -> shared, completion on an mbarrier) through an NS-stage
// ring in shared memory.  A chunk is 8 slices = 256 rows; warp w of the 8 consumer warps owns slice
// 8c + w; a 9th warp (one lane) is the producer, NS - 1 chunks ahead.  The consumer warps only issue
// the dependent x gathers (L1/L2), so the DRAM streams stay in flight without costing registers.
// Same arithmetic as k_sell (fma chain in slice-entry order): bitwise-equal results.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// the same address held in an ordinary register: opaque to the compiler, so it is not
// rematerialised from the CTA id before every shared load of an unrolled body (4 uniform ops each)
__device__ __forceinline__ uint32_t smem_reg(const void* p) {
    uint32_t r;
    asm("mov.b32 %0, %1;" : "=r"(r) : "r"(smem_u32(p)));
    return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "MBW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra MBW_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ int lds_s32(uint32_t a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_u16(uint32_t a) {
    int v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_s16(uint32_t a) {
    int v;
    asm volatile("ld.shared.s16 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_u8(uint32_t a) {
    int v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

constexpr int kTmaWarps = 8;  // consumer warps per CTA (+1 producer warp)
constexpr int kBndAhead = 4;  // producer fetches slice offsets this many chunks early
constexpr int kBndRing = 8;   // ring of fetched offsets (> kBndAhead)

template <int VM, int CM>
struct TmaStreams {
    static constexpr int ESA = CM == 3 ? 2 : (VM == 0 ? 8 : 1);              // value / pair stream
    static constexpr int ESB = CM == 3 ? 0 : (CM == 0 ? 4 : (CM == 1 ? 1 : 2)); // column stream
};

__host__ __device__ constexpr int tma_align16(int x) { return (x + 15) & ~15; }

// chunk = kTmaWarps * SPW slices (each consumer warp owns SPW slices of it); NS-stage ring
template <int VM, int CM, int W, int SPW, int NS>
struct TmaLayout {
    static constexpr int CS = kTmaWarps * SPW;  // slices per chunk
    static constexpr int ROWS = 32 * CS;
    static constexpr int HDR = tma_align16(4 * (CS + 1));
    static constexpr int A = tma_align16(CS * W * 32 * TmaStreams<VM, CM>::ESA);
    static constexpr int B = tma_align16(CS * W * 32 * TmaStreams<VM, CM>::ESB);
    static constexpr int V = ROWS * 8;
    static constexpr int STAGE = HDR + A + B + 3 * V;
    static constexpr int BYTES = NS * STAGE + 2 * NS * 8 + 16;
};

// Epilogues of the TMA path: NV row vectors are staged besides the x tile (vec(k) = their global
// pointers, null = not staged), store() combines them with the row sum.
struct TEpiSmooth {  // three-term recurrence step; prev = xprev ? xprev_i : cp * f_i
    const double* f;
    const double* xprev;
    double* out;
    double alpha, beta, cg, cp;
    static constexpr int ND = 0;
    __device__ __forceinline__ const double* vec(int k) const { return k == 0 ? f : xprev; }
    __device__ __forceinline__ void store(int i, double s, double xi, double v0, double v1, double*) const {
        const double prev = xprev ? v1 : cp * v0;
        out[i] = alpha * (cg * xi) + (1.0 - alpha) * prev + beta * (v0 - cg * s);
    }
};
struct TEpiResid {  // out = f - A x; acc[0] += out^2
    const double* f;
    double* out;
    static constexpr int ND = 1;
    __device__ __forceinline__ const double* vec(int k) const { return k == 0 ? f : nullptr; }
    __device__ __forceinline__ void store(int i, double s, double, double v0, double, double* acc) const {
        const double r = v0 - s;
        out[i] = r;
        acc[0] += r * r;
    }
};
struct TEpiSpmvDots {  // q = A d; acc = (d.q, d.rho)
    const double* rho;
    double* q;
    static constexpr int ND = 2;
    __device__ __forceinline__ const double* vec(int k) const { return k == 0 ? rho : nullptr; }
    __device__ __forceinline__ void store(int i, double s, double di, double v0, double, double* acc) const {
        q[i] = s;
        acc[0] += di * s;
        acc[1] += di * v0;
    }
};

// One slice of exact width K (straight-line): decode the K codes of this lane's row from the stage,
// issue the K gathers, run the fma chain in entry order, apply the epilogue (variable-width levels).
template <class Epi, int VM, int CM, int K, int ESA, int ESB, int LA, int LB, int LV, int ROWS>
__device__ __forceinline__ void tma_slice(const Epi& epi, uint32_t sb, int q, uint32_t off, int i, int lane, int n,
                                          int chi, uint32_t sv_a, uint32_t sc_a, const double* __restrict__ xg,
                                          bool v0, bool v1, double* acc) {
    constexpr int HDR = 0;
    const uint32_t A = sb + LA + off * 32 * ESA + lane * ESA;
    const uint32_t Bc = sb + LB + off * 32 * ESB + lane * ESB;
    int craw[K], col[K];
#pragma unroll
    for (int u = 0; u < K; ++u) {
        int cr;
        if constexpr (CM == 3) {
            craw[u] = lds_u16(A + u * 64);
            cr = (int)__byte_perm((uint32_t)craw[u], 0u, 0x4441u);  // byte 1 (PRMT + LEA address)
        } else {
            if constexpr (VM == 1) craw[u] = lds_u8(A + u * 32);
            if constexpr (CM == 0) cr = lds_s32(Bc + u * 128);
            else if constexpr (CM == 1) cr = lds_u8(Bc + u * 32);
            else cr = lds_s16(Bc + u * 64);
        }
        int cc;
        if constexpr (CM == 0) cc = cr;
        else {
            cc = i + ((CM == 1 || CM == 3) ? lds_s32(sc_a + 4 * cr) : cr);
            cc = cc < chi ? cc : chi;
        }
        col[u] = cc;
    }
    double x[K];
#pragma unroll
    for (int u = 0; u < K; ++u) x[u] = ld_gather(xg + col[u]);
    double sum = 0.0;
#pragma unroll
    for (int u = 0; u < K; ++u) {
        double v;
        if constexpr (VM == 0) v = lds_f64(A + u * 256);
        else v = lds_f64(sv_a + 8 * (CM == 3 ? (int)__byte_perm((uint32_t)craw[u], 0u, 0x4440u) : craw[u]));
        sum = fma(v, x[u], sum);
    }
    (void)HDR;
    if (i < n) {
        const uint32_t r8 = 8 * (q * 32 + lane);
        const uint32_t vt = sb + LV;
        const double xi = lds_f64(vt + r8);
        const double a0 = v0 ? lds_f64(vt + 8 * ROWS + r8) : 0.0;
        const double a1 = v1 ? lds_f64(vt + 16 * ROWS + r8) : 0.0;
        epi.store(i, sum, xi, a0, a1, acc);
    }
}

template <class Epi, int VM, int CM, int W, class Lay, int K = W>
__device__ __forceinline__ void tma_slice_dispatch(int w, const Epi& epi, uint32_t sb, int q, uint32_t off, int i,
                                                   int lane, int n, int chi, uint32_t sv_a, uint32_t sc_a,
                                                   const double* __restrict__ xg, bool v0, bool v1, double* acc) {
    if constexpr (K >= 1) {
        if (w == K)
            tma_slice<Epi, VM, CM, K, TmaStreams<VM, CM>::ESA, TmaStreams<VM, CM>::ESB, Lay::HDR, Lay::HDR + Lay::A,
                      Lay::HDR + Lay::A + Lay::B, Lay::ROWS>(epi, sb, q, off, i, lane, n, chi, sv_a, sc_a, xg, v0, v1,
                                                             acc);
        else
            tma_slice_dispatch<Epi, VM, CM, W, Lay, K - 1>(w, epi, sb, q, off, i, lane, n, chi, sv_a, sc_a, xg, v0,
                                                          v1, acc);
    }
}

template <class Epi, bool DOTS, int VM, int CM, int W, int SPW, int NS>
__global__ void __launch_bounds__(32 * (kTmaWarps + 1)) k_sell_tma(Sell S, const double* __restrict__ xg, Epi epi,
                                                                   double* partials, unsigned* ticket,
                                                                   DotOut dot_out) {
    using Lay = TmaLayout<VM, CM, W, SPW, NS>;
    using St = TmaStreams<VM, CM>;
    constexpr int CS = Lay::CS;
    extern __shared__ __align__(128) unsigned char tsm[];
    __shared__ double sv[VM ? 256 : 1];
    __shared__ int sc[(CM == 1 || CM == 3) ? 256 : 1];
    __shared__ int bnd[kBndRing * (CS + 1)];
    uint64_t* full = reinterpret_cast<uint64_t*>(tsm + NS * Lay::STAGE);
    uint64_t* empty = full + NS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double acc[Epi::ND > 0 ? Epi::ND : 1];
#pragma unroll
    for (int k = 0; k < (Epi::ND > 0 ? Epi::ND : 1); ++k) acc[k] = 0.0;
    if (threadIdx.x == 0) {
        for (int k = 0; k < NS; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], kTmaWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if constexpr (VM == 1)
        for (int k = threadIdx.x; k < S.nvdict; k += blockDim.x) sv[k] = S.vdict[k];
    if constexpr (CM == 1 || CM == 3)
        for (int k = threadIdx.x; k < S.ncdict; k += blockDim.x) sc[k] = S.cdict[k];
    __syncthreads();
    const int nchunks = (S.nslices + CS - 1) / CS;
    const int K = blockIdx.x < nchunks ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const double* v0g = epi.vec(0);
    const double* v1g = epi.vec(1);
    if (warp == kTmaWarps) {  // producer: one lane
        if (lane == 0) {
            const unsigned char* gA = CM == 3 ? reinterpret_cast<const unsigned char*>(S.pcode)
                                              : (VM == 0 ? reinterpret_cast<const unsigned char*>(S.val) : S.vcode);
            const unsigned char* gB = CM == 0 ? reinterpret_cast<const unsigned char*>(S.col)
                                              : (CM == 1 ? S.ccode : reinterpret_cast<const unsigned char*>(S.coff));
            // The chunk's slice offsets (sptr) are fetched kBndAhead chunks early with 4-byte cp.async into a
            // shared ring, so the copy issue never waits on a dependent global load.
            auto fetch_bounds = [&](int k) {
                if (k < K) {
                    const int s0 = (blockIdx.x + k * gridDim.x) * CS, s1 = min(s0 + CS, S.nslices);
                    int* dst = bnd + (k % kBndRing) * (CS + 1);
                    for (int q = 0; q <= CS; ++q)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst + q)),
                                     "l"(S.sptr + min(s0 + q, s1))
                                     : "memory");
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            for (int k = 0; k < kBndAhead; ++k) fetch_bounds(k);
            for (int k = 0; k < K; ++k) {
                fetch_bounds(k + kBndAhead);
                asm volatile("cp.async.wait_group %0;" ::"n"(kBndAhead) : "memory");
                const int* hb = bnd + (k % kBndRing) * (CS + 1);
                const int st = k % NS, j = k / NS;
                if (j > 0) mbar_wait(&empty[st], (j - 1) & 1);
                unsigned char* sb = tsm + st * Lay::STAGE;
                int* hdr = reinterpret_cast<int*>(sb);
                const int c = blockIdx.x + k * gridDim.x;
                const int s0 = c * CS, s1 = min(s0 + CS, S.nslices);
                for (int q = 0; q <= CS; ++q) hdr[q] = hb[q];
                const int b0 = hdr[0], b1 = hdr[CS];
                const int r0 = S.srow0 + s0 * 32, r1 = min(S.srow0 + s1 * 32, S.n);
                const uint32_t vb = (uint32_t)tma_align16((r1 - r0) * 8);
                const uint32_t ab = (uint32_t)(b1 - b0) * 32u * St::ESA;
                const uint32_t bb = (uint32_t)(b1 - b0) * 32u * St::ESB;
                mbar_expect_tx(&full[st], ab + bb + vb * (1u + (v0g ? 1u : 0u) + (v1g ? 1u : 0u)));
                if (ab) bulk_g2s(sb + Lay::HDR, gA + (size_t)b0 * 32 * St::ESA, ab, &full[st]);
                if (bb) bulk_g2s(sb + Lay::HDR + Lay::A, gB + (size_t)b0 * 32 * St::ESB, bb, &full[st]);
                bulk_g2s(sb + Lay::HDR + Lay::A + Lay::B, xg + r0, vb, &full[st]);
                if (v0g) bulk_g2s(sb + Lay::HDR + Lay::A + Lay::B + Lay::V, v0g + r0, vb, &full[st]);
                if (v1g) bulk_g2s(sb + Lay::HDR + Lay::A + Lay::B + 2 * Lay::V, v1g + r0, vb, &full[st]);
            }
        }
    } else {
        // consumers: shared-window addresses are formed once (32-bit ld.shared below)
        const uint32_t tsm_a = smem_reg(tsm), sv_a = smem_reg(sv), sc_a = smem_reg(sc);
        const double* __restrict__ xgr = xg;
        for (int k = 0; k < K; ++k) {
            const int st = k % NS, j = k / NS;
            mbar_wait(&full[st], j & 1);
            const uint32_t sb = tsm_a + st * Lay::STAGE;
            const int c = blockIdx.x + k * gridDim.x;
            const int h0 = lds_s32(sb);
            if constexpr (W > 8 && SPW == 1) {  // variable slice widths: exact-width straight-line bodies
                const int s = c * CS + warp;
                if (s < S.nslices) {
                    const int hq = lds_s32(sb + 4 * warp), wq = lds_s32(sb + 4 * (warp + 1)) - hq;
                    tma_slice_dispatch<Epi, VM, CM, W, Lay>(wq, epi, sb, warp, (uint32_t)(hq - h0),
                                                            S.srow0 + s * 32 + lane,
                                                            lane, S.n, S.chi, sv_a, sc_a, xgr, v0g != nullptr,
                                                            v1g != nullptr, acc);
                }
            } else {
            // this warp's SPW slices of the chunk: codes -> columns, then every gather, then the fma chains
            int craw[SPW][W], w[SPW], col[SPW][W];
            uint32_t aoff[SPW];
#pragma unroll
            for (int h = 0; h < SPW; ++h) {
                const int q = warp + h * kTmaWarps;
                const int s = c * CS + q;
                const int hq = lds_s32(sb + 4 * q), hq1 = lds_s32(sb + 4 * (q + 1));
                w[h] = s < S.nslices ? hq1 - hq : 0;
                const uint32_t off = (uint32_t)(hq - h0);
                aoff[h] = off;
                const uint32_t A = sb + Lay::HDR + off * 32 * St::ESA + lane * St::ESA;
                const uint32_t Bc = sb + Lay::HDR + Lay::A + off * 32 * St::ESB + lane * St::ESB;
                const int i = S.srow0 + s * 32 + lane;
                auto entry = [&](int u) {
                    int cr;
                    if constexpr (CM == 3) {
                        craw[h][u] = lds_u16(A + u * 64);
                        cr = (int)__byte_perm((uint32_t)craw[h][u], 0u, 0x4441u);
                    } else {
                        if constexpr (VM == 1) craw[h][u] = lds_u8(A + u * 32);
                        if constexpr (CM == 0) cr = lds_s32(Bc + u * 128);
                        else if constexpr (CM == 1) cr = lds_u8(Bc + u * 32);
                        else cr = lds_s16(Bc + u * 64);
                    }
                    int cc;
                    if constexpr (CM == 0) cc = cr;
                    else {
                        cc = i + ((CM == 1 || CM == 3) ? lds_s32(sc_a + 4 * cr) : cr);
                        cc = cc < S.chi ? cc : S.chi;
                    }
                    col[h][u] = cc;
                };
                if (w[h] == W) {  // full-width slice (the common case): straight-line
#pragma unroll
                    for (int u = 0; u < W; ++u) entry(u);
                } else {
#pragma unroll
                    for (int u = 0; u < W; ++u)
                        if (u < w[h]) entry(u);
                }
            }
            double x[SPW][W];
#pragma unroll
            for (int h = 0; h < SPW; ++h) {
                if (w[h] == W) {
#pragma unroll
                    for (int u = 0; u < W; ++u) x[h][u] = ld_gather(xgr + col[h][u]);
                } else {
#pragma unroll
                    for (int u = 0; u < W; ++u)
                        if (u < w[h]) x[h][u] = ld_gather(xgr + col[h][u]);
                }
            }
            const uint32_t vt = sb + Lay::HDR + Lay::A + Lay::B;
#pragma unroll
            for (int h = 0; h < SPW; ++h) {
                const int q = warp + h * kTmaWarps;
                const uint32_t A = sb + Lay::HDR + aoff[h] * 32 * St::ESA + lane * St::ESA;
                double sum = 0.0;
                auto term = [&](int u) {
                    double v;
                    if constexpr (VM == 0) v = lds_f64(A + u * 256);
                    else v = lds_f64(sv_a + 8 * (CM == 3 ? (int)__byte_perm((uint32_t)craw[h][u], 0u, 0x4440u) : craw[h][u]));
                    sum = fma(v, x[h][u], sum);
                };
                if (w[h] == W) {
#pragma unroll
                    for (int u = 0; u < W; ++u) term(u);
                } else {
#pragma unroll
                    for (int u = 0; u < W; ++u)
                        if (u < w[h]) term(u);
                }
                const int i = S.srow0 + (c * CS + q) * 32 + lane;
                const uint32_t r8 = 8 * (q * 32 + lane);
                if (w[h] > 0 && i < S.n) {
                    const double xi = lds_f64(vt + r8);
                    const double a0 = v0g ? lds_f64(vt + Lay::V + r8) : 0.0;
                    const double a1 = v1g ? lds_f64(vt + 2 * Lay::V + r8) : 0.0;
                    epi.store(i, sum, xi, a0, a1, acc);
                }
            }
            }  // fixed-width path
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
    }
    if constexpr (DOTS) finalize_dots<Epi::ND>(acc, partials, ticket, dot_out);
}

// resident grid of one kernel instance (cached per instance and dynamic smem size)
template <class K>
static int resident_grid(K kernel, size_t smem) {
    int bps = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kernel, kBlock, smem));
    return g_num_sms * (bps < 1 ? 1 : bps);
}

static size_t tile_smem(const Tiles& T) { return (size_t)(T.cap + 2) * sizeof(double) + (size_t)(T.cap + 4) * sizeof(int); }

template <class Epi, bool DOTS>
static int tiled_resident(int cap) {
    static bool configured = false;  // per template instance
    static int cached_cap = -1, cached = 0;
    if (!configured) {
        CK(cudaFuncSetAttribute(k_tiled<Epi, DOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = true;
    }
    if (cap != cached_cap) {
        cached = resident_grid(k_tiled<Epi, DOTS>, (size_t)(cap + 2) * sizeof(double) + (size_t)(cap + 4) * sizeof(int));
        cached_cap = cap;
    }
    return cached;
}

int tiled_grid(int cap, int ntiles) {
    int g = tiled_resident<EpiSmooth, false>(cap);
    if (g > ntiles) g = ntiles;
    return g < 1 ? 1 : g;
}

template <class Epi, bool DOTS, int VM, int CM, int WMAX>
static void launch_sell_w(const SpOp& op, const double* xg, const Epi& epi, double* part, unsigned* tk,
                          DotOut dot_out, cudaStream_t s) {
    const int need = (op.S.nslices + (kBlock / 32) - 1) / (kBlock / 32);
    static int res = 0;  // per instance
    if (!res) res = resident_grid(k_sell<Epi, DOTS, VM, CM, WMAX>, 0);
    int g = need < res ? need : res;
    if (g < 1) g = 1;
    launch_k(k_sell<Epi, DOTS, VM, CM, WMAX>, dim3(g), dim3(kBlock), 0, s, op.S, xg, epi, part, tk, dot_out);
}

template <class Epi, bool DOTS, int VM, int CM>
static void launch_sell(const SpOp& op, const double* xg, const Epi& epi, double* part, unsigned* tk, DotOut dot_out,
                        cudaStream_t s) {
    const int w = op.S.wmax;
    if (w <= 5) launch_sell_w<Epi, DOTS, VM, CM, 5>(op, xg, epi, part, tk, dot_out, s);
    else if (w <= 8) launch_sell_w<Epi, DOTS, VM, CM, 8>(op, xg, epi, part, tk, dot_out, s);
    else if (w <= 12) launch_sell_w<Epi, DOTS, VM, CM, 12>(op, xg, epi, part, tk, dot_out, s);
    else if (w <= 16) launch_sell_w<Epi, DOTS, VM, CM, 16>(op, xg, epi, part, tk, dot_out, s);
    else launch_sell_w<Epi, DOTS, VM, CM, 0>(op, xg, epi, part, tk, dot_out, s);
}

// ------------------------------------------------------------------ vector-CSR kernel
// The wide-row coarse levels (3D Galerkin levels: 18-21 entries per row, slices up to 38 wide) are
// latency-bound in the SELL kernel, whose lane-per-row chain walks a wide slice in dependent 8-entry
// chunks.  Here G lanes share a row of the CSR: the row's entries are read contiguously (coalesced),
// all gathers of the row are in flight at once, and the G partial sums are combined by a fixed
// shuffle tree (deterministic; a different summation order than the CSR chain, within the parity
// tolerance).  The loop over rows is warp-uniform so every lane takes part in the shuffles.
template <class Epi, bool DOTS, int G>
__global__ void __launch_bounds__(kBlock) k_vcsr(Csr A, const double* __restrict__ xg, Epi epi, double* partials,
                                                 unsigned* ticket, DotOut dot_out) {
    double acc[Epi::ND > 0 ? Epi::ND : 1];
#pragma unroll
    for (int k = 0; k < (Epi::ND > 0 ? Epi::ND : 1); ++k) acc[k] = 0.0;
    constexpr int RPW = 32 / G;  // rows per warp
    const int lane = threadIdx.x & 31, sub = lane % G, grp = lane / G;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int* __restrict__ rp = A.rp;
    const int* __restrict__ ci = A.ci;
    const double* __restrict__ va = A.v;
    for (int r0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * RPW; r0 < A.n; r0 += nwarps * RPW) {
        const int i = r0 + grp;
        const bool act = i < A.n;
        typename Epi::Pre pre{};
        double xi = 0.0, s = 0.0;
        if (act) {
            if (sub == 0) {
                pre = epi.load(i);
                xi = ld_gather(xg + i);
            }
            // the lane's entries p = rp[i] + sub + G*u in batches of 8: the batch's column and value
            // loads, then its 8 gathers, are each in flight together (one dependent round trip per
            // batch instead of per entry); the fma chain keeps the entry order
            const int p1 = rp[i + 1];
            for (int p = rp[i] + sub; p < p1; p += 8 * G) {
                int c[8];
                double a[8], xv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int q = p + u * G;
                    c[u] = q < p1 ? __ldg(ci + q) : -1;
                    a[u] = q < p1 ? __ldg(va + q) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) xv[u] = c[u] >= 0 ? ld_gather(xg + c[u]) : 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (c[u] >= 0) s = fma(a[u], xv[u], s);
            }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, G);
        if (act && sub == 0) epi.store(i, s, xi, pre, acc);
    }
    if constexpr (DOTS) finalize_dots<Epi::ND>(acc, partials, ticket, dot_out);
}

template <class Epi, bool DOTS>
static void launch_vcsr(const SpOp& op, const double* xg, const Epi& epi, double* part, unsigned* tk, DotOut dot_out,
                        cudaStream_t s) {
    const int64_t threads = (int64_t)op.A.n * op.vg;
    int g = (int)std::min<int64_t>((threads + kBlock - 1) / kBlock, 148 * 8);
    if constexpr (DOTS) g = std::min(g, 4096);
    if (g < 1) g = 1;
    switch (op.vg) {
        case 4: launch_k(k_vcsr<Epi, DOTS, 4>, dim3(g), dim3(kBlock), 0, s, op.A, xg, epi, part, tk, dot_out); break;
        case 8: launch_k(k_vcsr<Epi, DOTS, 8>, dim3(g), dim3(kBlock), 0, s, op.A, xg, epi, part, tk, dot_out); break;
        case 16: launch_k(k_vcsr<Epi, DOTS, 16>, dim3(g), dim3(kBlock), 0, s, op.A, xg, epi, part, tk, dot_out); break;
        default: launch_k(k_vcsr<Epi, DOTS, 32>, dim3(g), dim3(kBlock), 0, s, op.A, xg, epi, part, tk, dot_out); break;
    }
}

template <class Epi, bool DOTS>
static void launch_op(const SpOp& op, const double* xg, const Epi& epi, const DotScratch* ds, DotOut dot_out,
                      cudaStream_t s) {
    double* part = ds ? ds->partials : nullptr;
    unsigned* tk = ds ? ds->ticket : nullptr;
    if (op.vg > 0) {
        launch_vcsr<Epi, DOTS>(op, xg, epi, part, tk, dot_out, s);
    } else if (op.sell) {
        const int fmt = op.S.vmode * 4 + op.S.cmode;
        switch (fmt) {
            case 0: launch_sell<Epi, DOTS, 0, 0>(op, xg, epi, part, tk, dot_out, s); break;
            case 1: launch_sell<Epi, DOTS, 0, 1>(op, xg, epi, part, tk, dot_out, s); break;
            case 2: launch_sell<Epi, DOTS, 0, 2>(op, xg, epi, part, tk, dot_out, s); break;
            case 4: launch_sell<Epi, DOTS, 1, 0>(op, xg, epi, part, tk, dot_out, s); break;
            case 5: launch_sell<Epi, DOTS, 1, 1>(op, xg, epi, part, tk, dot_out, s); break;
            case 6: launch_sell<Epi, DOTS, 1, 2>(op, xg, epi, part, tk, dot_out, s); break;
            default: launch_sell<Epi, DOTS, 1, 3>(op, xg, epi, part, tk, dot_out, s); break;
        }
    } else {
        int g = tiled_resident<Epi, DOTS>(op.T.cap);
        if (g > op.T.ntiles) g = op.T.ntiles;
        if (g < 1) g = 1;
        launch_k(k_tiled<Epi, DOTS>, dim3(g), dim3(kBlock), tile_smem(op.T), s, op.A, xg, (const int*)op.T.row,
                 op.T.ntiles, op.T.cap, epi, part, tk, dot_out);
    }
    CK(cudaGetLastError());
    ++g_launches;
}


static bool tma_enabled() {
    static int on = -1;
    if (on < 0) on = getenv("AMG_NO_TMA") ? 0 : 1;
    return on == 1;
}

// formats that get W = 32 instances (variable-width levels wider than 16, e.g. the RGG's level 0:
// 1-byte value codes + int16 column offsets); the others stop at 16 to bound compile time
// (C4's level 1 -- 1-byte value codes + int32 columns, offsets +-53k -- measured no faster on a W = 32
// TMA instance than on the register SELL: 61.9 us per pass either way; its scattered gathers bound it)
__host__ __device__ constexpr bool tma_wide_fmt(int vm, int cm) { return (vm == 1 && cm == 2) || (vm == 0 && cm == 2); }

template <class Epi, bool DOTS, int VM, int CM, int W, int SPW, int NS>
static void launch_tma_w(const SpOp& op, const double* xg, const Epi& e, double* part, unsigned* tk, DotOut dot_out,
                         cudaStream_t s) {
    using Lay = TmaLayout<VM, CM, W, SPW, NS>;
    static_assert(Lay::BYTES <= 227 * 1024, "TMA stage ring exceeds the 227 KB of shared memory per CTA");
    static int res = 0;  // resident grid per instance
    if (!res) {
        CK(cudaFuncSetAttribute(k_sell_tma<Epi, DOTS, VM, CM, W, SPW, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                Lay::BYTES));
        int bps = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_sell_tma<Epi, DOTS, VM, CM, W, SPW, NS>,
                                                         32 * (kTmaWarps + 1), Lay::BYTES));
        res = g_num_sms * (bps < 1 ? 1 : bps);
    }
    const int nchunks = (op.S.nslices + Lay::CS - 1) / Lay::CS;
    int g = nchunks < res ? nchunks : res;
    if (g < 1) g = 1;
    if constexpr (DOTS) g = g < 4096 ? g : 4096;  // partials buffer (DotScratch) holds 4096 blocks per dot
    launch_k(k_sell_tma<Epi, DOTS, VM, CM, W, SPW, NS>, dim3(g), dim3(32 * (kTmaWarps + 1)), (size_t)Lay::BYTES, s,
             op.S, xg, e, part, tk, dot_out);
}

// compressed streams (few bytes per row): 2 slices per consumer warp keep twice the gathers in
// flight (3 stages); fp64/int32 streams are bandwidth-bound with one slice per warp (4 stages).
// AMG_TMA_VARIANT (experiments): 0 = 1 slice/warp 4 stages, 1 = 2 slices 3 stages, 2 = 1 slice 2 stages,
// 3 = 2 slices 2 stages.
template <class Epi, bool DOTS, int VM, int CM, int W>
static void launch_tma_v(const SpOp& op, const double* xg, const Epi& e, double* part, unsigned* tk, DotOut d,
                         cudaStream_t s) {
    static int var = -2;
    if (var == -2) var = getenv("AMG_TMA_VARIANT") ? atoi(getenv("AMG_TMA_VARIANT")) : -1;
    // measured: 2 slices per warp win for the narrow compressed 2D level (C3: 113.7 vs
    // 116.0 us), one slice per warp for the 7-wide 3D level (C4: 138.6 vs 158.4 us)
    const int v = var >= 0 ? var : ((VM == 1 && W <= 5) ? 1 : 0);
    switch (v) {
        case 1: launch_tma_w<Epi, DOTS, VM, CM, W, 2, 3>(op, xg, e, part, tk, d, s); break;
        case 2: launch_tma_w<Epi, DOTS, VM, CM, W, 1, 2>(op, xg, e, part, tk, d, s); break;
        case 3: launch_tma_w<Epi, DOTS, VM, CM, W, 2, 2>(op, xg, e, part, tk, d, s); break;
        default: launch_tma_w<Epi, DOTS, VM, CM, W, 1, 4>(op, xg, e, part, tk, d, s); break;
    }
}

template <class Epi, bool DOTS, int VM, int CM>
static void launch_tma_fmt(const SpOp& op, const double* xg, const Epi& e, double* part, unsigned* tk, DotOut d,
                           cudaStream_t s) {
    // exact-width instances up to 8 (the straight-line path then covers every full-width slice)
    switch (op.S.wmax) {
        case 1: case 2: case 3: case 4: launch_tma_v<Epi, DOTS, VM, CM, 4>(op, xg, e, part, tk, d, s); break;
        case 5: launch_tma_v<Epi, DOTS, VM, CM, 5>(op, xg, e, part, tk, d, s); break;
        case 6: launch_tma_v<Epi, DOTS, VM, CM, 6>(op, xg, e, part, tk, d, s); break;
        case 7: launch_tma_v<Epi, DOTS, VM, CM, 7>(op, xg, e, part, tk, d, s); break;
        case 8: launch_tma_v<Epi, DOTS, VM, CM, 8>(op, xg, e, part, tk, d, s); break;
        default:
            // (a 2-stage ring for the L2-resident W = 16 level measured slower: C3's level 1 17.1 vs
            // 14.7 us per step; ncu: L1/TEX 72% busy, 24% issue -- gather latency, not the ring, bounds it)
            if (op.S.wmax <= 12) launch_tma_w<Epi, DOTS, VM, CM, 12, 1, 3>(op, xg, e, part, tk, d, s);
            else if (op.S.wmax <= 16) launch_tma_w<Epi, DOTS, VM, CM, 16, 1, 3>(op, xg, e, part, tk, d, s);
            else if constexpr (tma_wide_fmt(VM, CM))  // 2-stage rings: 3 CTAs/SM with 1-byte value codes (C5's
                // level 0: 149.4 -> 134.3 us per step against 3 stages; 4 stages 258 us; 2 slices/warp 1.5 ms),
                // and the only ring of fp64 values that fits the 227 KB
                launch_tma_w<Epi, DOTS, VM, CM, 32, 1, 2>(op, xg, e, part, tk, d, s);
    }
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// TMA-staged path: SELL level with slices <= 8 wide, large enough to be bandwidth bound, and 16-byte
// aligned streams (bulk copies move 16-byte multiples).  Returns false if not eligible.
// the operator's format/size part of the TMA eligibility (the launch also needs 16-byte aligned vectors)
bool tma_eligible(const SpOp& op) {
    static int min_slices = -1;  // AMG_TMA_MIN_SLICES (experiments)
    if (min_slices < 0) min_slices = getenv("AMG_TMA_MIN_SLICES") ? atoi(getenv("AMG_TMA_MIN_SLICES")) : 8 * 148 * kTmaWarps;
    static int max_w = -1;  // AMG_TMA_MAX_W (experiments)
    if (max_w < 0) max_w = getenv("AMG_TMA_MAX_W") ? atoi(getenv("AMG_TMA_MAX_W")) : 32;
    const int wcap = tma_wide_fmt(op.S.vmode, op.S.cmode) ? 32 : 16;  // W = 32 instances: wide formats only
    return tma_enabled() && op.sell && op.vg == 0 && op.S.wmax <= std::min(max_w, wcap) && op.S.nslices >= min_slices;
}

template <class Epi, bool DOTS>
static bool launch_tma(const SpOp& op, const double* xg, const Epi& e, const double* v0, const double* v1,
                       const DotScratch* ds, DotOut d, cudaStream_t s) {
    if (!(tma_eligible(op) && aligned16(xg) && (!v0 || aligned16(v0)) && (!v1 || aligned16(v1)))) return false;
    double* part = ds ? ds->partials : nullptr;
    unsigned* tk = ds ? ds->ticket : nullptr;
    switch (op.S.vmode * 4 + op.S.cmode) {
        case 0: launch_tma_fmt<Epi, DOTS, 0, 0>(op, xg, e, part, tk, d, s); break;
        case 1: launch_tma_fmt<Epi, DOTS, 0, 1>(op, xg, e, part, tk, d, s); break;
        case 2: launch_tma_fmt<Epi, DOTS, 0, 2>(op, xg, e, part, tk, d, s); break;
        case 4: launch_tma_fmt<Epi, DOTS, 1, 0>(op, xg, e, part, tk, d, s); break;
        case 5: launch_tma_fmt<Epi, DOTS, 1, 1>(op, xg, e, part, tk, d, s); break;
        case 6: launch_tma_fmt<Epi, DOTS, 1, 2>(op, xg, e, part, tk, d, s); break;
        default: launch_tma_fmt<Epi, DOTS, 1, 3>(op, xg, e, part, tk, d, s); break;
    }
    CK(cudaGetLastError());
    ++g_launches;
    return true;
}

void launch_smooth(const SpOp& op, const double* xg, double cg, const double* f, const double* xprev, double cp,
                   double alpha, double beta, double* out, cudaStream_t s) {
    if (launch_tma<TEpiSmooth, false>(op, xg, TEpiSmooth{f, xprev, out, alpha, beta, cg, cp}, f, xprev, nullptr,
                                      DotOut{}, s))
        return;
    EpiSmooth e{f, xprev, out, alpha, beta, cg, cp};
    launch_op<EpiSmooth, false>(op, xg, e, nullptr, DotOut{}, s);
}

void launch_resid(const SpOp& op, const double* xg, const double* f, double* out, double* dot_rr, const DotScratch& ds,
                  cudaStream_t s) {
    if (dot_rr) {
        if (launch_tma<TEpiResid, true>(op, xg, TEpiResid{f, out}, f, nullptr, &ds, DotOut{{dot_rr}}, s)) return;
        launch_op<EpiResid, true>(op, xg, EpiResid{f, out}, &ds, DotOut{{dot_rr}}, s);
    } else {
        if (launch_tma<TEpiResid, false>(op, xg, TEpiResid{f, out}, f, nullptr, nullptr, DotOut{}, s)) return;
        launch_op<EpiResid, false>(op, xg, EpiResid{f, out}, nullptr, DotOut{}, s);
    }
}

void launch_spmv_dots(const SpOp& op, const double* d, const double* rho, double* q, double* dot_dq, double* dot_dr,
                      const DotScratch& ds, cudaStream_t s) {
    if (launch_tma<TEpiSpmvDots, true>(op, d, TEpiSpmvDots{rho, q}, rho, nullptr, &ds, DotOut{{dot_dq, dot_dr}}, s))
        return;
    EpiSpmvDots e{rho, q};
    launch_op<EpiSpmvDots, true>(op, d, e, &ds, DotOut{{dot_dq, dot_dr}}, s);
}

void launch_spmv_zdots(const SpOp& op, const double* z, const double* q0, const double* rho, double* out3,
                       const DotScratch& ds, cudaStream_t s) {
    launch_op<EpiZDots, true>(op, z, EpiZDots{q0, rho}, &ds, DotOut{{out3, out3 + 1, out3 + 2}}, s);
}

// ------------------------------------------------------------------ transfers
__global__ void __launch_bounds__(kBlock) k_restrict(int nc, const int* __restrict__ aptr,
                                                     const int* __restrict__ perm, const double* __restrict__ r,
                                                     double* __restrict__ rH) {
    for (int I = blockIdx.x * blockDim.x + threadIdx.x; I < nc; I += gridDim.x * blockDim.x) {
        const int t0 = aptr[I], t1 = aptr[I + 1];
        double s = 0.0;
        for (int t = t0; t < t1; ++t) s += __ldg(r + perm[t]);
        rH[I] = s;
    }
}

void launch_restrict(int nc, const int* aptr, const int* perm, const double* r, double* rH, cudaStream_t s) {
    const int grid = vgrid(nc);
    launch_k(k_restrict, dim3(grid), dim3(kBlock), 0, s, nc, aptr, perm, r, rH);
    CK(cudaGetLastError());
    ++g_launches;
}

// x_i += eH[agg_i].  V: quads of rows per thread and step (one int4 of agg, two double2 of x, four
// L2-resident gathers of eH), two quads in flight per thread; the scalar loop takes the tail.
template <bool V>
__global__ void __launch_bounds__(kBlock) k_prolong(int n, const int* __restrict__ agg,
                                                    const double* __restrict__ eH, double* __restrict__ x) {
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    int64_t i0 = 0;
    if constexpr (V) {
        const int64_t n4 = n >> 2;
        const int4* A4 = reinterpret_cast<const int4*>(agg);
        double2* X2 = reinterpret_cast<double2*>(x);
        int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        for (; q + st < n4; q += 2 * st) {
            const int4 a0 = A4[q], a1 = A4[q + st];
            double2 x0 = X2[2 * q], x1 = X2[2 * q + 1], x2 = X2[2 * (q + st)], x3 = X2[2 * (q + st) + 1];
            const double e0 = __ldg(eH + a0.x), e1 = __ldg(eH + a0.y), e2 = __ldg(eH + a0.z), e3 = __ldg(eH + a0.w);
            const double e4 = __ldg(eH + a1.x), e5 = __ldg(eH + a1.y), e6 = __ldg(eH + a1.z), e7 = __ldg(eH + a1.w);
            x0.x += e0; x0.y += e1; x1.x += e2; x1.y += e3;
            x2.x += e4; x2.y += e5; x3.x += e6; x3.y += e7;
            X2[2 * q] = x0; X2[2 * q + 1] = x1; X2[2 * (q + st)] = x2; X2[2 * (q + st) + 1] = x3;
        }
        for (; q < n4; q += st) {
            const int4 a0 = A4[q];
            double2 x0 = X2[2 * q], x1 = X2[2 * q + 1];
            x0.x += __ldg(eH + a0.x); x0.y += __ldg(eH + a0.y); x1.x += __ldg(eH + a0.z); x1.y += __ldg(eH + a0.w);
            X2[2 * q] = x0; X2[2 * q + 1] = x1;
        }
        i0 = n4 << 2;
    }
    for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += st) x[i] += __ldg(eH + agg[i]);
}

// The last inner-FCG update fused with the prolongation (E_l is read only by the prolongation):
// x_i += E'[agg_i], E' = alpha d + E (ASSIGN: alpha d), alpha = d.rho / d.q (0 when d.q = 0, reading
// A13) -- the same fma as k_fcg_update's E update, then the same single add as k_prolong.  One launch
// less per inner-FCG visit; E itself is not written.
template <bool V, bool ASSIGN>
__global__ void __launch_bounds__(kBlock) k_prolong_fcg(int n, const int* __restrict__ agg,
                                                        const double* __restrict__ eH, const double* __restrict__ dH,
                                                        const double* __restrict__ dr, const double* __restrict__ dq,
                                                        double* __restrict__ x) {
    const double den = *dq;
    const double alpha = (den != 0.0) ? (*dr) / den : 0.0;
    auto e = [&](int a) -> double {
        const double d = __ldg(dH + a);
        return ASSIGN ? alpha * d : fma(alpha, d, __ldg(eH + a));
    };
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    int64_t i0 = 0;
    if constexpr (V) {
        const int64_t n4 = n >> 2;
        const int4* A4 = reinterpret_cast<const int4*>(agg);
        double2* X2 = reinterpret_cast<double2*>(x);
        int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        for (; q + st < n4; q += 2 * st) {  // two quads in flight per thread (as k_prolong)
            const int4 a0 = A4[q], a1 = A4[q + st];
            double2 x0 = X2[2 * q], x1 = X2[2 * q + 1], x2 = X2[2 * (q + st)], x3 = X2[2 * (q + st) + 1];
            const double e0 = e(a0.x), e1 = e(a0.y), e2 = e(a0.z), e3 = e(a0.w);
            const double e4 = e(a1.x), e5 = e(a1.y), e6 = e(a1.z), e7 = e(a1.w);
            x0.x += e0; x0.y += e1; x1.x += e2; x1.y += e3;
            x2.x += e4; x2.y += e5; x3.x += e6; x3.y += e7;
            X2[2 * q] = x0; X2[2 * q + 1] = x1; X2[2 * (q + st)] = x2; X2[2 * (q + st) + 1] = x3;
        }
        for (; q < n4; q += st) {
            const int4 a0 = A4[q];
            double2 x0 = X2[2 * q], x1 = X2[2 * q + 1];
            x0.x += e(a0.x); x0.y += e(a0.y); x1.x += e(a0.z); x1.y += e(a0.w);
            X2[2 * q] = x0; X2[2 * q + 1] = x1;
        }
        i0 = n4 << 2;
    }
    for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += st) x[i] += e(agg[i]);
}

void launch_prolong_fcg(int n, const int* agg, const double* eH, const double* dH, const double* dr, const double* dq,
                        bool assign, double* x, cudaStream_t s) {
    const bool v = al16(agg) && al16(x);
    const dim3 g(vgrid(v ? (n + 3) / 4 : n)), b(kBlock);
    if (v) {
        if (assign) launch_k(k_prolong_fcg<true, true>, g, b, 0, s, n, agg, eH, dH, dr, dq, x);
        else launch_k(k_prolong_fcg<true, false>, g, b, 0, s, n, agg, eH, dH, dr, dq, x);
    } else {
        if (assign) launch_k(k_prolong_fcg<false, true>, g, b, 0, s, n, agg, eH, dH, dr, dq, x);
        else launch_k(k_prolong_fcg<false, false>, g, b, 0, s, n, agg, eH, dH, dr, dq, x);
    }
    CK(cudaGetLastError());
    ++g_launches;
}

// Prolongation of the nu = 2 inner-FCG result E = alpha_0 d_0 + alpha_1 d_1 with d_1 = z - beta_0 d_0
// never formed: x_i += c0 d_0[I] + c1 z[I], I = agg_i, c1 = alpha_1, c0 = alpha_0 - alpha_1 beta_0, from
// the scalars sc[0] = d_0.q_0, sc[W] = d_0.rho_0, sc[2W..2W+2] = (z.Az, z.q_0, z.rho_1) (W = kMaxWin):
//   beta_0 = z.q_0 / d_0.q_0,  d_1.q_1 = z.Az - beta_0 z.q_0  (A symmetric: d_0.Az = q_0.z),
//   d_1.rho_1 = z.rho_1 (d_0.rho_1 = 0: alpha_0 makes rho_1 orthogonal to d_0),
//   alpha_i = d_i.rho_i / d_i.q_i; every quotient with a zero denominator is 0 (reading A13).
__global__ void __launch_bounds__(kBlock) k_prolong_fcg2(int n, const int* __restrict__ agg,
                                                         const double* __restrict__ d0, const double* __restrict__ z,
                                                         const double* __restrict__ sc, double* __restrict__ x,
                                                         bool vec) {
    const double dq0 = sc[0], dr0 = sc[kMaxWin], zaz = sc[2 * kMaxWin], zq = sc[2 * kMaxWin + 1],
                 zr = sc[2 * kMaxWin + 2];
    const double a0 = dq0 != 0.0 ? dr0 / dq0 : 0.0;
    const double b0 = dq0 != 0.0 ? zq / dq0 : 0.0;
    const double dq1 = zaz - b0 * zq;
    const double a1 = dq1 != 0.0 ? zr / dq1 : 0.0;
    const double c0 = a0 - a1 * b0, c1 = a1;
    auto e = [&](int a) -> double { return fma(c1, __ldg(z + a), c0 * __ldg(d0 + a)); };
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    int64_t i0 = 0;
    if (vec) {
        const int64_t n4 = n >> 2;
        const int4* A4 = reinterpret_cast<const int4*>(agg);
        double2* X2 = reinterpret_cast<double2*>(x);
        for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n4; q += st) {
            const int4 a = A4[q];
            double2 x0 = X2[2 * q], x1 = X2[2 * q + 1];
            x0.x += e(a.x); x0.y += e(a.y); x1.x += e(a.z); x1.y += e(a.w);
            X2[2 * q] = x0; X2[2 * q + 1] = x1;
        }
        i0 = n4 << 2;
    }
    for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += st) x[i] += e(agg[i]);
}

void launch_prolong_fcg2(int n, const int* agg, const double* d0, const double* z, const double* sc, double* x,
                         cudaStream_t s) {
    const bool v = al16(agg) && al16(x);
    launch_k(k_prolong_fcg2, dim3(vgrid(v ? (n + 3) / 4 : n)), dim3(kBlock), 0, s, n, agg, d0, z, sc, x, v);
    CK(cudaGetLastError());
    ++g_launches;
}

void launch_prolong(int n, const int* agg, const double* eH, double* x, cudaStream_t s) {
    if (al16(agg) && al16(x)) launch_k(k_prolong<true>, dim3(vgrid((n + 3) / 4)), dim3(kBlock), 0, s, n, agg, eH, x);
    else launch_k(k_prolong<false>, dim3(vgrid(n)), dim3(kBlock), 0, s, n, agg, eH, x);
    CK(cudaGetLastError());
    ++g_launches;
}

// warp per row GEMV of the dense coarsest (pseudo-)inverse
__global__ void __launch_bounds__(kBlock) k_gemv(int n, const double* __restrict__ M, const double* __restrict__ r,
                                                 double* __restrict__ e) {
    const int lane = threadIdx.x & 31;
    const int nwarp = (gridDim.x * blockDim.x) >> 5;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarp) {
        double s = 0.0;
        for (int j = lane; j < n; j += 32) s = fma(M[(size_t)i * n + j], __ldg(r + j), s);
        s = warp_sum(s);
        if (lane == 0) e[i] = s;
    }
}

void launch_gemv(int n, const double* M, const double* r, double* e, cudaStream_t s) {
    int grid = (n * 32 + kBlock - 1) / kBlock;
    if (grid > vector_grid()) grid = vector_grid();
    launch_k(k_gemv, dim3(grid), dim3(kBlock), 0, s, n, M, r, e);
    CK(cudaGetLastError());
    ++g_launches;
}

// Dense B_{L-2} r (k_dense.cu): one CTA per row, each thread a strided share of the columns with
// four independent loads in flight, then a fixed-order block sum (deterministic).  A warp per row
// (k_gemv) kept too few loads in flight for the 1328^2 (C3) .. 2316^2 (C2) matrices: 15 us cold.
template <int T>
__global__ void __launch_bounds__(T) k_gemv_rows(int n, const double* __restrict__ M, const double* __restrict__ r,
                                                 double* __restrict__ e) {
    __shared__ double red[T / 32];
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const double* row = M + (size_t)i * n;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int j = threadIdx.x;
        for (; j + 3 * T < n; j += 4 * T) {
            const double a0 = __ldg(row + j), a1 = __ldg(row + j + T), a2 = __ldg(row + j + 2 * T),
                         a3 = __ldg(row + j + 3 * T);
            s0 = fma(a0, __ldg(r + j), s0);
            s1 = fma(a1, __ldg(r + j + T), s1);
            s2 = fma(a2, __ldg(r + j + 2 * T), s2);
            s3 = fma(a3, __ldg(r + j + 3 * T), s3);
        }
        for (; j < n; j += T) s0 = fma(__ldg(row + j), __ldg(r + j), s0);
        double v = warp_sum((s0 + s1) + (s2 + s3));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x < 32) {
            double t = threadIdx.x < T / 32 ? red[threadIdx.x] : 0.0;
            t = warp_sum(t);
            if (threadIdx.x == 0) e[i] = t;
        }
        __syncthreads();
    }
}

void launch_gemv_dense(int n, const double* M, const double* r, double* e, cudaStream_t s) {
    const int grid = n < 148 * 8 ? n : 148 * 8;
    if (n >= 1024) launch_k(k_gemv_rows<256>, dim3(grid), dim3(256), 0, s, n, M, r, e);
    else if (n >= 256) launch_k(k_gemv_rows<128>, dim3(grid), dim3(128), 0, s, n, M, r, e);
    else launch_k(k_gemv_rows<64>, dim3(grid), dim3(64), 0, s, n, M, r, e);
    CK(cudaGetLastError());
    ++g_launches;
}

// Residual fused with the restriction on the small (L2-resident, launch-latency-bound) levels: one
// warp per aggregate, lane = member (chunks of 32): each lane forms its row's residual f_i - (A x)_i
// with the fma chain in CSR order (the SELL kernels' order: the same r_i), then every lane sums the
// chunk's r in member order through shuffles starting from 0.0 (k_restrict's order): on a SELL level
// (and on a CSR-tile level whose rows all fit one thread's chain) bitwise the same rho_I as the
// unfused pair; k_tiled's block-summed long rows round differently (within the parity tolerance).
// One launch and the residual vector's round trip less per visit.
__global__ void __launch_bounds__(kBlock) k_resid_restrict(int nc, const int* __restrict__ aptr,
                                                           const int* __restrict__ perm, const int* __restrict__ rp,
                                                           const int* __restrict__ ci, const double* __restrict__ v,
                                                           const double* __restrict__ x, const double* __restrict__ f,
                                                           double* __restrict__ rho) {
    const int lane = threadIdx.x & 31;
    const int nwarp = (gridDim.x * blockDim.x) >> 5;
    for (int I = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; I < nc; I += nwarp) {
        const int t0 = aptr[I], t1 = aptr[I + 1];
        double s = 0.0;
        for (int tb = t0; tb < t1; tb += 32) {
            const int t = tb + lane;
            double r = 0.0;
            if (t < t1) {
                const int i = perm[t];
                // the row's chain in CSR order, its loads issued 8 entries at a time (one dependent
                // column -> gather round trip per 8 entries instead of per entry)
                double acc = 0.0;
                const int p1 = rp[i + 1];
                for (int p = rp[i]; p < p1; p += 8) {
                    int c[8];
                    double a[8], xv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        c[u] = p + u < p1 ? __ldg(ci + p + u) : -1;
                        a[u] = p + u < p1 ? __ldg(v + p + u) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) xv[u] = c[u] >= 0 ? ld_gather(x + c[u]) : 0.0;
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (c[u] >= 0) acc = fma(a[u], xv[u], acc);
                }
                r = ld_nc(f + i) - acc;
            }
            const int cnt = min(32, t1 - tb);
            for (int k = 0; k < cnt; ++k) s += __shfl_sync(0xffffffffu, r, k);
        }
        if (lane == 0) rho[I] = s;
    }
}

void launch_resid_restrict(int nc, const int* aptr, const int* perm, const Csr& A, const double* x, const double* f,
                           double* rho, cudaStream_t s) {
    int grid = (int)(((int64_t)nc * 32 + kBlock - 1) / kBlock);
    if (grid > vector_grid()) grid = vector_grid();
    launch_k(k_resid_restrict, dim3(grid), dim3(kBlock), 0, s, nc, aptr, perm, (const int*)A.rp, (const int*)A.ci,
             (const double*)A.v, x, f, rho);
    CK(cudaGetLastError());
    ++g_launches;
}

// Coarsest apply fused with the prolongation into the level above (one launch instead of two on every
// visit of level L-2): warp w takes fine rows i = w, w + nwarp, ...; it computes e_I, I = agg(i) + cb,
// exactly as k_gemv does for row I (the same lane split and warp_sum tree: bitwise the same e_I) and
// adds it to x_i (the same single add as k_prolong).  Each fine row recomputes its aggregate's dot:
// n_{L-2} * n_L fma, negligible next to the saved launch.
__global__ void __launch_bounds__(kBlock) k_gemv_prolong(int nf, const int* __restrict__ agg, int cb, int nL,
                                                         const double* __restrict__ M, const double* __restrict__ r,
                                                         double* __restrict__ x) {
    const int lane = threadIdx.x & 31;
    const int nwarp = (gridDim.x * blockDim.x) >> 5;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nf; i += nwarp) {
        const int I = __ldg(agg + i) + cb;
        double s = 0.0;
        for (int j = lane; j < nL; j += 32) s = fma(M[(size_t)I * nL + j], __ldg(r + j), s);
        s = warp_sum(s);
        if (lane == 0) x[i] += s;
    }
}

void launch_gemv_prolong(int nf, const int* agg, int cb, int nL, const double* M, const double* r, double* x,
                         cudaStream_t s) {
    int grid = (int)(((int64_t)nf * 32 + kBlock - 1) / kBlock);
    if (grid > vector_grid()) grid = vector_grid();
    launch_k(k_gemv_prolong, dim3(grid), dim3(kBlock), 0, s, nf, agg, cb, nL, M, r, x);
    CK(cudaGetLastError());
    ++g_launches;
}

// ------------------------------------------------------------------ FCG vector kernels
struct PtrArr {
    const double* p[kMaxWin];
};

// Vector kernels of the FCG iterations (outer: O8, inner: O7).  The level-0 vectors are 134 MB each
// on C3, so these are HBM streams: double2 loads, two steps in flight per thread, 8 CTAs/SM
// (tools/vec_micro.cu).  Each kernel has a scalar instance for vectors that are not 16-byte aligned
// (never on the library's own buffers) and the scalar loop takes the odd tail element.

// c_j = z . Q_j, j < W (deterministic two-stage reduction); W = 0: runtime w <= kMaxWin, scalar
template <int W, bool V>
__global__ void __launch_bounds__(kBlock) k_multidot(int n, const double* __restrict__ z, PtrArr Q, int w,
                                                     double* partials, unsigned* ticket, double* c) {
    constexpr int NA = W ? W : kMaxWin;
    double acc[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) acc[j] = 0.0;
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    int64_t i0 = 0;
    if constexpr (V && W > 0) {
        const int64_t n2 = n >> 1;
        const double2* Z2 = reinterpret_cast<const double2*>(z);
        int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        for (; i + st < n2; i += 2 * st) {
            const double2 za = Z2[i], zb = Z2[i + st];
            double2 qa[W], qb[W];
#pragma unroll
            for (int j = 0; j < W; ++j) {
                qa[j] = reinterpret_cast<const double2*>(Q.p[j])[i];
                qb[j] = reinterpret_cast<const double2*>(Q.p[j])[i + st];
            }
#pragma unroll
            for (int j = 0; j < W; ++j) {
                acc[j] += za.x * qa[j].x;
                acc[j] += za.y * qa[j].y;
                acc[j] += zb.x * qb[j].x;
                acc[j] += zb.y * qb[j].y;
            }
        }
        for (; i < n2; i += st) {
            const double2 za = Z2[i];
#pragma unroll
            for (int j = 0; j < W; ++j) {
                const double2 q = reinterpret_cast<const double2*>(Q.p[j])[i];
                acc[j] += za.x * q.x;
                acc[j] += za.y * q.y;
            }
        }
        i0 = n2 << 1;
    }
    const int ww = W ? W : w;
    for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += st) {
        const double zi = z[i];
#pragma unroll
        for (int j = 0; j < NA; ++j)
            if (j < ww) acc[j] += zi * Q.p[j][i];
    }
    // reduce only the first ww accumulators (ww is uniform)
    __shared__ bool amlast;
    const int G = gridDim.x;
    for (int j = 0; j < ww; ++j) {
        double b = block_sum(acc[j]);
        if (threadIdx.x == 0) partials[j * G + blockIdx.x] = b;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) amlast = (atomicAdd(ticket, 1u) == (unsigned)(G - 1));
    __syncthreads();
    if (amlast) {
        __threadfence();
        for (int j = 0; j < ww; ++j) {
            double v = 0.0;
            for (int b = threadIdx.x; b < G; b += blockDim.x) v += __ldcg(partials + j * G + b);
            v = block_sum(v);
            if (threadIdx.x == 0) c[j] = v;
        }
        if (threadIdx.x == 0) *ticket = 0u;
    }
}

static bool all_al16(const double* const* P, int w) {
    for (int j = 0; j < w; ++j)
        if (!al16(P[j])) return false;
    return true;
}

void launch_multidot(int n, const double* z, const double* const* Q, int w, double* c, const DotScratch& ds,
                     cudaStream_t s) {
    PtrArr a{};
    for (int j = 0; j < w; ++j) a.p[j] = Q[j];
    const bool v = al16(z) && all_al16(Q, w);
    const dim3 g(vgrid(v && w <= 4 ? (n + 1) / 2 : n)), b(kBlock);
    switch (v ? w : 0) {
        case 1: launch_k(k_multidot<1, true>, g, b, 0, s, n, z, a, w, ds.partials, ds.ticket, c); break;
        case 2: launch_k(k_multidot<2, true>, g, b, 0, s, n, z, a, w, ds.partials, ds.ticket, c); break;
        case 3: launch_k(k_multidot<3, true>, g, b, 0, s, n, z, a, w, ds.partials, ds.ticket, c); break;
        case 4: launch_k(k_multidot<4, true>, g, b, 0, s, n, z, a, w, ds.partials, ds.ticket, c); break;
        default: launch_k(k_multidot<0, false>, g, b, 0, s, n, z, a, w, ds.partials, ds.ticket, c); break;
    }
    CK(cudaGetLastError());
    ++g_launches;
}

// d = z - sum_{j<W} beta_j D_j, beta_j = c_j / (d_j.q_j) (0 when d_j.q_j = 0, reading A13)
template <int W, bool V>
__global__ void __launch_bounds__(kBlock) k_direction(int n, const double* __restrict__ z, PtrArr D,
                                                      const double* __restrict__ c, const double* __restrict__ dq,
                                                      int w, double* __restrict__ d) {
    constexpr int NA = W ? W : kMaxWin;
    const int ww = W ? W : w;
    double beta[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) beta[j] = (j < ww && dq[j] != 0.0) ? c[j] / dq[j] : 0.0;  // d_j = 0: no term (A13)
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    int64_t i0 = 0;
    if constexpr (V && W > 0) {
        const int64_t n2 = n >> 1;
        const double2* Z2 = reinterpret_cast<const double2*>(z);
        double2* O2 = reinterpret_cast<double2*>(d);
        int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        for (; i + st < n2; i += 2 * st) {
            double2 va = Z2[i], vb = Z2[i + st];
            double2 pa[W], pb[W];
#pragma unroll
            for (int j = 0; j < W; ++j) {
                pa[j] = reinterpret_cast<const double2*>(D.p[j])[i];
                pb[j] = reinterpret_cast<const double2*>(D.p[j])[i + st];
            }
#pragma unroll
            for (int j = 0; j < W; ++j) {
                va.x -= beta[j] * pa[j].x;
                va.y -= beta[j] * pa[j].y;
                vb.x -= beta[j] * pb[j].x;
                vb.y -= beta[j] * pb[j].y;
            }
            O2[i] = va;
            O2[i + st] = vb;
        }
        for (; i < n2; i += st) {
            double2 va = Z2[i];
#pragma unroll
            for (int j = 0; j < W; ++j) {
                const double2 p = reinterpret_cast<const double2*>(D.p[j])[i];
                va.x -= beta[j] * p.x;
                va.y -= beta[j] * p.y;
            }
            O2[i] = va;
        }
        i0 = n2 << 1;
    }
    for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += st) {
        double v = z[i];
#pragma unroll
        for (int j = 0; j < NA; ++j)
            if (j < ww) v -= beta[j] * D.p[j][i];
        d[i] = v;
    }
}

void launch_direction(int n, const double* z, const double* const* D, const double* c, const double* dq, int w,
                      double* d, cudaStream_t s) {
    PtrArr a{};
    for (int j = 0; j < w; ++j) a.p[j] = D[j];
    const bool v = al16(z) && al16(d) && all_al16(D, w);
    const dim3 g(vgrid(v && w <= 4 ? (n + 1) / 2 : n)), b(kBlock);
    switch (v ? w : 0) {
        case 1: launch_k(k_direction<1, true>, g, b, 0, s, n, z, a, c, dq, w, d); break;
        case 2: launch_k(k_direction<2, true>, g, b, 0, s, n, z, a, c, dq, w, d); break;
        case 3: launch_k(k_direction<3, true>, g, b, 0, s, n, z, a, c, dq, w, d); break;
        case 4: launch_k(k_direction<4, true>, g, b, 0, s, n, z, a, c, dq, w, d); break;
        default: launch_k(k_direction<0, false>, g, b, 0, s, n, z, a, c, dq, w, d); break;
    }
    CK(cudaGetLastError());
    ++g_launches;
}

// Outer FCG at the last window position p = W (W >= 1 earlier directions): the direction
// d_p = z - sum_j beta_j d_j of k_direction, fused with the deferred x updates of the window.  The
// d_j it loads anyway are reused for x += a_j d_j (j < p), and before d_p overwrites its slot the
// slot's old content -- the previous window's last direction, pending if *has_old -- is applied
// first.  The fma sequence is the one of the per-iteration updates (previous window's last, then
// this window's in order), so x is bitwise the same.
template <int W>
__global__ void __launch_bounds__(kBlock) k_direction_xf(int n, const double* __restrict__ z, PtrArr D,
                                                         const double* __restrict__ c, const double* __restrict__ dq,
                                                         double* __restrict__ d, double* __restrict__ x,
                                                         const double* __restrict__ alph, const int* __restrict__ has_old) {
    double beta[W], al[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
        beta[j] = dq[j] != 0.0 ? c[j] / dq[j] : 0.0;  // d_j = 0: no term (A13)
        al[j] = alph[j];
    }
    const bool ho = *has_old != 0;
    const double aold = alph[W];  // the slot d_p overwrites: the previous window's last alpha
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    const int64_t n2 = n >> 1;
    const double2* Z2 = reinterpret_cast<const double2*>(z);
    double2* O2 = reinterpret_cast<double2*>(d);
    double2* X2 = reinterpret_cast<double2*>(x);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += st) {
        double2 va = Z2[i], xi = X2[i], od = make_double2(0.0, 0.0);
        if (ho) od = O2[i];
        double2 pj[W];
#pragma unroll
        for (int j = 0; j < W; ++j) pj[j] = reinterpret_cast<const double2*>(D.p[j])[i];
        if (ho) { xi.x += aold * od.x; xi.y += aold * od.y; }
#pragma unroll
        for (int j = 0; j < W; ++j) {
            xi.x += al[j] * pj[j].x;
            xi.y += al[j] * pj[j].y;
            va.x -= beta[j] * pj[j].x;
            va.y -= beta[j] * pj[j].y;
        }
        X2[i] = xi;
        O2[i] = va;
    }
    for (int64_t i = (n2 << 1) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += st) {
        double v = z[i], xi = x[i];
        if (ho) xi += aold * d[i];
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const double p = D.p[j][i];
            xi += al[j] * p;
            v -= beta[j] * p;
        }
        x[i] = xi;
        d[i] = v;
    }
}

bool direction_xf_ok(int w, const double* z, const double* const* D, const double* d, const double* x) {
    return w >= 1 && w <= 4 && al16(z) && al16(d) && al16(x) && all_al16(D, w);
}

void launch_direction_xf(int n, const double* z, const double* const* D, const double* c, const double* dq, int w,
                         double* d, double* x, const double* alph, const int* has_old, cudaStream_t s) {
    if (!direction_xf_ok(w, z, D, d, x)) throw Error(-1, "launch_direction_xf: unsupported window");
    PtrArr a{};
    for (int j = 0; j < w; ++j) a.p[j] = D[j];
    const dim3 g(vgrid((n + 1) / 2)), b(kBlock);
    switch (w) {
        case 1: launch_k(k_direction_xf<1>, g, b, 0, s, n, z, a, c, dq, d, x, alph, has_old); break;
        case 2: launch_k(k_direction_xf<2>, g, b, 0, s, n, z, a, c, dq, d, x, alph, has_old); break;
        case 3: launch_k(k_direction_xf<3>, g, b, 0, s, n, z, a, c, dq, d, x, alph, has_old); break;
        default: launch_k(k_direction_xf<4>, g, b, 0, s, n, z, a, c, dq, d, x, alph, has_old); break;
    }
    CK(cudaGetLastError());
    ++g_launches;
}

// x (+)= alpha d; r -= alpha q; rr = r.r;  alpha = d.r / d.q (outer: d.q <= 0 or NaN is a breakdown)
// NOX: the x update is deferred (launch_x_flush); alpha goes to alpha_out, and d and x are not touched
template <bool ASSIGN, bool UPD_R, bool RR, bool V, bool NOX = false>
__global__ void __launch_bounds__(kBlock) k_fcg_update(int n, const double* __restrict__ dr,
                                                       const double* __restrict__ dq, const double* __restrict__ d,
                                                       const double* __restrict__ q, double* __restrict__ x,
                                                       double* __restrict__ r, int* breakdown, double* partials,
                                                       unsigned* ticket, double* rr, double* alpha_out, int* set_old) {
    const double den = *dq;
    double alpha;
    if (breakdown) {  // outer FCG: d.q <= 0 or NaN is a breakdown
        alpha = (den > 0.0) ? (*dr) / den : 0.0;
        if (!(den > 0.0) && blockIdx.x == 0 && threadIdx.x == 0) *breakdown = 1;
    } else {          // inner: rho = 0 => d = 0 => 0/0, take alpha = 0 (DESIGN.md readings)
        alpha = (den != 0.0) ? (*dr) / den : 0.0;
    }
    if (NOX && blockIdx.x == 0 && threadIdx.x == 0) {
        *alpha_out = alpha;
        if (set_old) *set_old = 1;  // this slot's update is now pending (k_direction_xf applies it)
    }
    double acc[1] = {0.0};
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    int64_t i0 = 0;
    if constexpr (V) {
        const int64_t n2 = n >> 1;
        const double2* D2 = reinterpret_cast<const double2*>(d);
        const double2* Q2 = reinterpret_cast<const double2*>(q);
        double2* X2 = reinterpret_cast<double2*>(x);
        double2* R2 = reinterpret_cast<double2*>(r);
        int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        for (; i < n2; i += st) {
            double2 ri, qi;
            if (UPD_R) { ri = R2[i]; qi = Q2[i]; }
            if (!NOX) {
                const double2 di = D2[i];
                double2 xi;
                if (!ASSIGN) xi = X2[i];
                if (ASSIGN) { xi.x = alpha * di.x; xi.y = alpha * di.y; } else { xi.x += alpha * di.x; xi.y += alpha * di.y; }
                X2[i] = xi;
            }
            if (UPD_R) {
                ri.x = ri.x - alpha * qi.x;
                ri.y = ri.y - alpha * qi.y;
                R2[i] = ri;
                if (RR) { acc[0] += ri.x * ri.x; acc[0] += ri.y * ri.y; }
            }
        }
        i0 = n2 << 1;
    }
    for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += st) {
        if (!NOX) {
            double di = d[i];
            if (ASSIGN) x[i] = alpha * di; else x[i] += alpha * di;
        }
        if (UPD_R) {
            double ri = r[i] - alpha * q[i];
            r[i] = ri;
            if (RR) acc[0] += ri * ri;
        }
    }
    if (RR) finalize_dots<1>(acc, partials, ticket, DotOut{{rr}});
}

template <bool V>
static void fcg_update_v(dim3 g, dim3 b, cudaStream_t s, int n, const double* dr, const double* dq, const double* d,
                         const double* q, double* x, bool assign_x, double* r, double* rr, int* breakdown,
                         const DotScratch& ds) {
    double* np = nullptr;
    unsigned* nt = nullptr;
    if (assign_x) {
        if (r) launch_k(k_fcg_update<true, true, false, V>, g, b, 0, s, n, dr, dq, d, q, x, r, breakdown, np, nt, np, np, nullptr);
        else   launch_k(k_fcg_update<true, false, false, V>, g, b, 0, s, n, dr, dq, d, q, x, r, breakdown, np, nt, np, np, nullptr);
    } else if (r && rr) {
        launch_k(k_fcg_update<false, true, true, V>, g, b, 0, s, n, dr, dq, d, q, x, r, breakdown, ds.partials, ds.ticket, rr, np, nullptr);
    } else if (r) {
        launch_k(k_fcg_update<false, true, false, V>, g, b, 0, s, n, dr, dq, d, q, x, r, breakdown, np, nt, np, np, nullptr);
    } else {
        launch_k(k_fcg_update<false, false, false, V>, g, b, 0, s, n, dr, dq, d, q, x, r, breakdown, np, nt, np, np, nullptr);
    }
}

void launch_fcg_update(int n, const double* dr, const double* dq, const double* d, const double* q, double* x,
                       bool assign_x, double* r, double* rr, int* breakdown, const DotScratch& ds, cudaStream_t s,
                       double* alpha_out, int* set_old) {
    const bool v = al16(d) && al16(x) && (!r || (al16(r) && al16(q)));
    const dim3 g(vgrid(v ? (n + 1) / 2 : n)), b(kBlock);
    if (!x) {  // deferred x update (outer FCG): r -= alpha q, rr = r.r, alpha stored
        if (!r || !rr || !alpha_out || assign_x) throw Error(-1, "launch_fcg_update: bad deferred update");
        if (v) launch_k(k_fcg_update<false, true, true, true, true>, g, b, 0, s, n, dr, dq, d, q, x, r, breakdown,
                        ds.partials, ds.ticket, rr, alpha_out, set_old);
        else   launch_k(k_fcg_update<false, true, true, false, true>, g, b, 0, s, n, dr, dq, d, q, x, r, breakdown,
                        ds.partials, ds.ticket, rr, alpha_out, set_old);
        CK(cudaGetLastError());
        ++g_launches;
        return;
    }
    if (v)
        fcg_update_v<true>(g, b, s, n, dr, dq, d, q, x, assign_x, r, rr, breakdown, ds);
    else
        fcg_update_v<false>(g, b, s, n, dr, dq, d, q, x, assign_x, r, rr, breakdown, ds);
    CK(cudaGetLastError());
    ++g_launches;
}

// deferred outer-FCG x update: x = (((x + a_{j0} d_{j0}) + a_{j1} d_{j1}) + ...) over the window
// slots sl.j[0..cnt) in that order (the order of the iterations they belong to).  One pass over x and
// the directions instead of one x read-modify-write per iteration.  C > 0: compile-time count (the C
// direction loads of a step in flight together); C = 0: runtime cnt.
template <int C, bool V>
__global__ void __launch_bounds__(kBlock) k_x_flush(int n, double* __restrict__ x, const double* __restrict__ D,
                                                    size_t ld, const double* __restrict__ a, Slots sl, int cnt) {
    constexpr int M = C > 0 ? C : kMaxWin;
    if (C > 0) cnt = C;
    double al[M];
    const double* dp[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
        al[j] = j < cnt ? a[sl.j[j]] : 0.0;
        dp[j] = D + (size_t)(j < cnt ? sl.j[j] : 0) * ld;
    }
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    int64_t i0 = 0;
    if constexpr (V && C > 0) {
        const int64_t n2 = n >> 1;
        double2* X2 = reinterpret_cast<double2*>(x);
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += st) {
            double2 dj[C];
#pragma unroll
            for (int j = 0; j < C; ++j) dj[j] = __ldcs(reinterpret_cast<const double2*>(dp[j]) + i);
            double2 xi = X2[i];
#pragma unroll
            for (int j = 0; j < C; ++j) {
                xi.x += al[j] * dj[j].x;
                xi.y += al[j] * dj[j].y;
            }
            X2[i] = xi;
        }
        i0 = n2 << 1;
    }
    for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += st) {
        double xi = x[i];
        for (int j = 0; j < cnt; ++j) xi += al[j] * dp[j][i];
        x[i] = xi;
    }
}

void launch_x_flush(int n, double* x, const double* D, size_t ld, const double* a, const Slots& sl, int cnt,
                    cudaStream_t s) {
    if (cnt <= 0) return;
    if (cnt > kMaxWin) throw Error(-1, "launch_x_flush: cnt > kMaxWin");
    const bool v = al16(x) && al16(D) && (ld % 2) == 0;
    const dim3 g(vgrid(v ? (n + 1) / 2 : n)), b(kBlock);
    if (v) {
        switch (cnt) {
            case 1: launch_k(k_x_flush<1, true>, g, b, 0, s, n, x, D, ld, a, sl, cnt); break;
            case 2: launch_k(k_x_flush<2, true>, g, b, 0, s, n, x, D, ld, a, sl, cnt); break;
            case 3: launch_k(k_x_flush<3, true>, g, b, 0, s, n, x, D, ld, a, sl, cnt); break;
            case 4: launch_k(k_x_flush<4, true>, g, b, 0, s, n, x, D, ld, a, sl, cnt); break;
            case 5: launch_k(k_x_flush<5, true>, g, b, 0, s, n, x, D, ld, a, sl, cnt); break;
            default: launch_k(k_x_flush<0, false>, dim3(vgrid(n)), b, 0, s, n, x, D, ld, a, sl, cnt); break;
        }
    } else {
        launch_k(k_x_flush<0, false>, g, b, 0, s, n, x, D, ld, a, sl, cnt);
    }
    CK(cudaGetLastError());
    ++g_launches;
}

// sum_i x_i y_i (y = null: sum_i x_i), deterministic two-stage reduction
template <bool V>
__global__ void __launch_bounds__(kBlock) k_dot(int n, const double* __restrict__ x, const double* __restrict__ y,
                                                double* partials, unsigned* ticket, double* out) {
    double acc[1] = {0.0};
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    int64_t i0 = 0;
    if constexpr (V) {
        const int64_t n2 = n >> 1;
        const double2* X2 = reinterpret_cast<const double2*>(x);
        const double2* Y2 = reinterpret_cast<const double2*>(y);
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += st) {
            const double2 a = X2[i];
            const double2 bb = y ? Y2[i] : make_double2(1.0, 1.0);
            acc[0] += a.x * bb.x;
            acc[0] += a.y * bb.y;
        }
        i0 = n2 << 1;
    }
    for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += st)
        acc[0] += x[i] * (y ? y[i] : 1.0);
    finalize_dots<1>(acc, partials, ticket, DotOut{{out}});
}

void launch_dot(int n, const double* x, const double* y, double* out, const DotScratch& ds, cudaStream_t s) {
    if (al16(x) && (!y || al16(y))) launch_k(k_dot<true>, dim3(vgrid((n + 1) / 2)), dim3(kBlock), 0, s, n, x, y, ds.partials, ds.ticket, out);
    else launch_k(k_dot<false>, dim3(vgrid(n)), dim3(kBlock), 0, s, n, x, y, ds.partials, ds.ticket, out);
    CK(cudaGetLastError());
    ++g_launches;
}

__global__ void __launch_bounds__(kBlock) k_sub_scalar(int n, double ntot, double* __restrict__ v,
                                                       const double* __restrict__ sum) {
    const double mu = (*sum) / ntot;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] -= mu;
}

void launch_mean_project(int n, double* v, double* tmp, const DotScratch& ds, cudaStream_t s) {
    launch_dot(n, v, nullptr, tmp, ds, s);
    launch_sub_mean(n, (double)n, v, tmp, s);
}

void launch_sub_mean(int n, double ntot, double* v, const double* sum, cudaStream_t s) {
    launch_k(k_sub_scalar, dim3(vgrid(n)), dim3(kBlock), 0, s, n, ntot, v, sum);
    CK(cudaGetLastError());
    ++g_launches;
}

__global__ void __launch_bounds__(kBlock) k_lincomb3(int n, double a, const double* x, double b, const double* y,
                                                     double c, const double* z, double* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double v = a * x[i];
        if (y) v += b * y[i];
        if (z) v += c * z[i];
        out[i] = v;
    }
}

void launch_lincomb3(int n, double a, const double* x, double b, const double* y, double c, const double* z,
                     double* out, cudaStream_t s) {
    launch_k(k_lincomb3, dim3(vgrid(n)), dim3(kBlock), 0, s, n, a, x, b, y, c, z, out);
    CK(cudaGetLastError());
    ++g_launches;
}

__global__ void __launch_bounds__(kBlock) k_copy(int n, const double* __restrict__ x, double* __restrict__ y) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = x[i];
}

void launch_copy(int n, const double* x, double* y, cudaStream_t s) {
    launch_k(k_copy, dim3(vgrid(n)), dim3(kBlock), 0, s, n, x, y);
    CK(cudaGetLastError());
    ++g_launches;
}

}  // namespace amg
