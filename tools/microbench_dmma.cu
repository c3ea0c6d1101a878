// DMMA (mma.sync m8n8k4 f64) pipeline characterisation on B200: throughput
// vs warps per SM and independent accumulator chains per warp, plus the
// dependent-chain latency.  Informs the gate kernel's warp/chain layout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_dmma tools/microbench_dmma.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void chains(double* out, int iters, double a, double b, long long* cycles) {
    double c[2 * CH];
#pragma unroll
    for (int i = 0; i < 2 * CH; ++i) c[i] = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < CH; ++j) dmma(c[2 * j], c[2 * j + 1], a, b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 2 * CH; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

template <int CH>
void run(double* out, long long* dcyc, int warps_per_sm) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000 / CH;
    const int blocks = 148, threads = 32 * warps_per_sm;
    chains<CH><<<blocks, threads>>>(out, 10, 1.0, 1e-3, dcyc);
    cudaEventRecord(e0);
    chains<CH><<<blocks, threads>>>(out, iters, 1.0, 1e-3, dcyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long cyc;
    cudaMemcpy(&cyc, dcyc, sizeof(cyc), cudaMemcpyDeviceToHost);
    double dm = double(iters) * CH * blocks * warps_per_sm;
    printf("warps/SM=%2d chains=%d: %.2f TFLOP/s, %.2f cycles per DMMA per warp-chain-step, SM-cycles/DMMA=%.2f\n",
           warps_per_sm, CH, dm * 512 / ms / 1e9, double(cyc) / iters, double(cyc) / (double(iters) * CH * warps_per_sm));
}

int main() {
    double* out;
    long long* dcyc;
    cudaMalloc(&out, 148 * 1024 * sizeof(double));
    cudaMalloc(&dcyc, sizeof(long long));
    for (int w : {1, 4, 8, 16, 32}) {
        run<1>(out, dcyc, w);
        run<2>(out, dcyc, w);
        run<4>(out, dcyc, w);
        run<8>(out, dcyc, w);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
