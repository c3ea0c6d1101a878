// Microbenchmark: B200 fp64 throughput via DFMA (CUDA cores) vs DMMA
// (mma.sync.aligned.m8n8k4.row.col.f64, FP64 tensor path).  Used to choose
// the gate-kernel design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench_fp64.cu && ./mb
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters, double a, double b) {
    double c[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            dmma(c[0], c[1], a, b); dmma(c[2], c[3], a, b); dmma(c[4], c[5], a, b); dmma(c[6], c[7], a, b);
            dmma(c[8], c[9], a, b); dmma(c[10], c[11], a, b); dmma(c[12], c[13], a, b); dmma(c[14], c[15], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Mixed: warps with (warp % 4) < dmma_warps run the DMMA loop, the others
// the DFMA loop, on the same SM at the same time.  If the FP64 tensor path
// and the FP64 CUDA cores are separate units the two rates add up.
__global__ void mixed_kernel(double* out, int iters, int dfma_iters, double a, double b, int dmma_warps) {
    const int w = (threadIdx.x >> 5) & 3;
    if (w < dmma_warps) {
        double c[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) c[i] = 0.0;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                dmma(c[0], c[1], a, b); dmma(c[2], c[3], a, b); dmma(c[4], c[5], a, b); dmma(c[6], c[7], a, b);
                dmma(c[8], c[9], a, b); dmma(c[10], c[11], a, b); dmma(c[12], c[13], a, b); dmma(c[14], c[15], a, b);
            }
        }
        double s = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) s += c[i];
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    } else {
        double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
        for (int i = 0; i < dfma_iters; ++i) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
                x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
            }
        }
        out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    }
}

int main() {
    double* out;
    cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        for (int blocks_per_sm : {4, 8}) {
            int blocks = 148 * blocks_per_sm, threads = 256;
            cudaEventRecord(e0);
            dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double flops = 2.0 * 64 * iters * double(blocks) * threads;
            printf("DFMA  blocks/SM=%d: %.3f ms  %.2f TFLOP/s\n", blocks_per_sm, ms, flops / ms / 1e9);
            cudaEventRecord(e0);
            dmma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            // per warp per dmma: 8*8*4 FMA = 256 FMA = 512 flop
            double dflops = 512.0 * 64 * iters * double(blocks) * (threads / 32);
            printf("DMMA  blocks/SM=%d: %.3f ms  %.2f TFLOP/s\n", blocks_per_sm, ms, dflops / ms / 1e9);
        }
    }
    // mixed: per warp-slot 4 warps per SMSP group; vary the DMMA share and the DFMA work
    for (int dw : {1, 2, 3}) {
        for (int dfi : {1024, 2048, 4096, 8192}) {
            int blocks = 148 * 4, threads = 256;
            cudaEventRecord(e0);
            mixed_kernel<<<blocks, threads>>>(out, iters / 4, dfi, 0.999, 1e-3, dw);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double warps = double(blocks) * (threads / 32);
            const double dm = 512.0 * 64 * (iters / 4) * warps * dw / 4;
            const double df = 2.0 * 64 * dfi * warps * (4 - dw) / 4 * 32;
            printf("MIXED dmma_warps=%d/4 dfma_iters=%d: %.3f ms  DMMA %.2f + DFMA %.2f = %.2f TFLOP/s\n", dw, dfi, ms,
                   dm / ms / 1e9, df / ms / 1e9, (dm + df) / ms / 1e9);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
