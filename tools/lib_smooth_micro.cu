// tools/lib_smooth_micro.cu -- times the LIBRARY's launch_smooth (k_solve.cu, compiled in) on the
// C3 level-0 operator in SELL-32 form, uncompressed and compressed, to compare with spmv_micro.cu.
#include "../paper_1307_6305_b200/csrc/k_solve.cu"

#include <cstdio>
#include <cstdlib>

namespace amg {
void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        printf("CUDA error %s in %s (%s:%d)\n", cudaGetErrorString(e), what, file, line);
        exit(1);
    }
}
}  // namespace amg

__global__ void build5(int N, int* sptr, int* col, double* val, unsigned char* vc, unsigned char* cc) {
    const int n = N * N, nsl = (n + 31) / 32;
    for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < (long)nsl * 32; t += (long)gridDim.x * blockDim.x) {
        int sl = (int)(t >> 5), lane = (int)(t & 31), i = sl * 32 + lane;
        if (lane == 0) sptr[sl] = sl * 5;
        if (t == 0) sptr[nsl] = nsl * 5;
        int iy = i / N, ix = i % N;
        int cs[5], vs[5], m = 0;
        double vv[5];
        int cols[5];
        if (i < n) {
            if (iy > 0) { cs[m] = 0; vs[m] = 0; cols[m] = i - N; vv[m++] = -1; }
            if (ix > 0) { cs[m] = 1; vs[m] = 0; cols[m] = i - 1; vv[m++] = -1; }
            cs[m] = 2; vs[m] = 1; cols[m] = i; vv[m++] = 4;
            if (ix < N - 1) { cs[m] = 3; vs[m] = 0; cols[m] = i + 1; vv[m++] = -1; }
            if (iy < N - 1) { cs[m] = 4; vs[m] = 0; cols[m] = i + N; vv[m++] = -1; }
        }
        for (int j = 0; j < 5; ++j) {
            size_t e = ((size_t)sl * 5 + j) * 32 + lane;
            vc[e] = (unsigned char)(j < m ? vs[j] : 2);
            cc[e] = (unsigned char)(j < m ? cs[j] : 2);
            col[e] = j < m ? cols[j] : (i < n ? i : 0);
            val[e] = j < m ? vv[j] : 0.0;
        }
    }
}

namespace amg {
__global__ void k_pair_codes_micro(int64_t m, const uint8_t* vc, const uint8_t* cc, uint16_t* pc) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
        pc[e] = (uint16_t)(vc[e] | (cc[e] << 8));
}
}  // namespace amg

__global__ void fill(double* x, size_t n, double s) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x)
        x[k] = s * (double)((k * 2654435761u) % 1000) / 1000.0;
}

int main(int argc, char** argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 4096;
    const int n = N * N, nsl = (n + 31) / 32;
    amg::init_device_props();
    amg::Sell S;
    S.n = n;
    S.nslices = nsl;
    S.padded = (int64_t)nsl * 160;
    S.wmax = 5;
    S.chi = n - 1;
    double *xg, *f, *xp, *out, *vd;
    int* cd;
    CK(cudaMalloc(&S.sptr, sizeof(int) * (nsl + 1)));
    CK(cudaMalloc(&S.col, sizeof(int) * S.padded + 256));
    CK(cudaMalloc(&S.val, sizeof(double) * S.padded + 256));
    CK(cudaMalloc(&S.vcode, S.padded + 256));
    CK(cudaMalloc(&S.ccode, S.padded + 256));
    CK(cudaMalloc(&vd, 256 * 8));
    CK(cudaMalloc(&cd, 256 * 4));
    for (double** p : {&xg, &f, &xp, &out}) CK(cudaMalloc(p, sizeof(double) * (size_t)n + 256));
    build5<<<4096, 256>>>(N, S.sptr, S.col, S.val, S.vcode, S.ccode);
    fill<<<4096, 256>>>(xg, n, 1.0);
    fill<<<4096, 256>>>(f, n, 2.0);
    fill<<<4096, 256>>>(xp, n, 3.0);
    double hv[256] = {-1.0, 4.0, 0.0};
    int hc[256] = {-N, -1, 0, 1, N};
    CK(cudaMemcpy(vd, hv, sizeof(hv), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(cd, hc, sizeof(hc), cudaMemcpyHostToDevice));
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, amg::SpOp& op, double bytes, bool inplace) {
        double* o = inplace ? xp : out;
        for (int r = 0; r < 3; ++r) amg::launch_smooth(op, xg, 1.0, f, xp, 0.0, 1.27, 0.29, o, 0);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int r = 0; r < 20; ++r) amg::launch_smooth(op, xg, 1.0, f, xp, 0.0, 1.27, 0.29, o, 0);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double us = 1e3 * ms / 20;
        printf("%-40s %8.1f us  %6.0f GB/s actual  model(12nnz+36n) %6.0f GB/s\n", name, us, bytes / us / 1e3,
               (12.0 * ((double)n + 4.0 * N * (N - 1)) + 36.0 * n) / us / 1e3);
    };
    amg::SpOp op;
    op.sell = true;
    op.S = S;
    run("library uncompressed", op, 12.0 * S.padded + 32.0 * n, false);
    run("library uncompressed in-place", op, 12.0 * S.padded + 32.0 * n, true);
    op.S.vmode = 1;
    op.S.cmode = 1;
    op.S.vdict = vd;
    op.S.cdict = cd;
    op.S.nvdict = 3;
    op.S.ncdict = 5;
    run("library compressed dict8/dict8", op, 2.0 * S.padded + 32.0 * n, false);
    run("library compressed in-place", op, 2.0 * S.padded + 32.0 * n, true);
    {
        uint16_t* pc;
        CK(cudaMalloc(&pc, 2 * S.padded + 256));
        amg::k_pair_codes_micro<<<4096, 256>>>(S.padded, S.vcode, S.ccode, pc);
        CK(cudaDeviceSynchronize());
        op.S.pcode = pc;
        op.S.cmode = 3;
        run("library compressed paired u16", op, 2.0 * S.padded + 32.0 * n, false);
    }
    return 0;
}
