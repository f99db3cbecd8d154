// tools/sync_micro.cu -- cost of a dependent phase on B200: grid.sync() in a cooperative persistent
// kernel vs a chain of tiny dependent kernels replayed from a CUDA graph (coarse-level latency floor).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_gridsync(int iters, double* buf) {
    cg::grid_group g = cg::this_grid();
    for (int k = 0; k < iters; ++k) {
        if (threadIdx.x == 0) buf[blockIdx.x] += 1.0;
        g.sync();
    }
}
// hand-rolled sense-reversal barrier (one atomic per CTA)
__global__ void k_mybar(int iters, unsigned* cnt, volatile unsigned* gen, double* buf) {
    for (int k = 0; k < iters; ++k) {
        if (threadIdx.x == 0) buf[blockIdx.x] += 1.0;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned g0 = *gen;
            __threadfence();
            if (atomicAdd(cnt, 1u) == gridDim.x - 1) {
                *cnt = 0;
                __threadfence();
                *gen = g0 + 1;
            } else {
                while (*gen == g0) {}
            }
            __threadfence();
        }
        __syncthreads();
    }
}
__global__ void k_tiny(double* buf, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) buf[i] += 1.0;
}

int main() {
    double* buf;
    unsigned* cnt;
    unsigned* gen;
    cudaMalloc(&buf, 1 << 24);
    cudaMalloc(&cnt, 8);
    cudaMalloc(&gen, 8);
    cudaMemset(buf, 0, 1 << 24);
    cudaMemset(cnt, 0, 8);
    cudaMemset(gen, 0, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int blocks : {148, 296, 592}) {
        int iters = 2000;
        void* args[] = {&iters, &buf};
        cudaLaunchCooperativeKernel((void*)k_gridsync, blocks, 256, args, 0, 0);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)k_gridsync, blocks, 256, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("grid.sync  %4d CTAs: %.3f us per barrier (%s)\n", blocks, 1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
        k_mybar<<<blocks, 256>>>(iters, cnt, gen, buf);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        k_mybar<<<blocks, 256>>>(iters, cnt, gen, buf);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("atomic bar %4d CTAs: %.3f us per barrier (%s)\n", blocks, 1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
    }
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int blocks : {1, 16, 148, 592}) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int k = 0; k < 500; ++k) k_tiny<<<blocks, 256, 0, s>>>(buf, blocks * 256);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        cudaEventRecord(e0, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("graph chain of tiny kernels, %4d CTAs: %.3f us per kernel\n", blocks, 1e3 * ms / 500);
    }
    return 0;
}
