// Legacy warp-level integer / fp8 tensor throughput on B200 (mma.sync, no
// tcgen05): int8 m16n8k32 -> s32 and e4m3 m16n8k32 -> f32, vs warps per SM and
// independent accumulator chains.  Decides whether an fp64-emulating (Ozaki)
// gate kernel could run on the legacy path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_imma tools/microbench_imma.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void imma(int (&d)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3, unsigned b0,
                                     unsigned b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int CH>
__global__ void chains(int* out, int iters, unsigned a, unsigned b) {
    int c[CH][4];
#pragma unroll
    for (int i = 0; i < CH; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) c[i][j] = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < CH; ++j) imma(c[j], a + j, a ^ j, a, b, b + j, b);
    }
    int s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s += c[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
void run(int* out, int warps_per_sm) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 40000 / CH;
    const int blocks = 148, threads = 32 * warps_per_sm;
    chains<CH><<<blocks, threads>>>(out, 10, 0x01020304u, 0x05060708u);
    cudaEventRecord(e0);
    chains<CH><<<blocks, threads>>>(out, iters, 0x01020304u, 0x05060708u);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = double(iters) * CH * blocks * warps_per_sm * 16 * 8 * 32 * 2;
    printf("int8 m16n8k32: warps/SM=%2d chains=%d: %.1f TOPS\n", warps_per_sm, CH, ops / ms / 1e9);
}

int main() {
    int* out;
    cudaMalloc(&out, 148 * 1024 * sizeof(int));
    for (int w : {4, 8, 16, 32}) {
        run<2>(out, w);
        run<4>(out, w);
        run<8>(out, w);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
