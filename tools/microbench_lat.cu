// Microbenchmark: dependent-chain latencies on B200 (one warp, clock64):
// DFMA, DMUL, DADD, LDS.64, LDS.128 and an indexed constant load.  Used to
// reason about the EVC coset kernel's per-mask dependency chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_lat tools/microbench_lat.cu && ./tools/mb_lat
#include <cstdio>
#include <cuda_runtime.h>

__constant__ double cst[256];

__global__ void lat_kernel(double* out, long long* cyc, int iters, double a, double b) {
    __shared__ double sm[1024];
    __shared__ double2 sm2[512];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 + 3) & 1023;
    for (int i = threadIdx.x; i < 512; i += blockDim.x) sm2[i] = make_double2((i * 5 + 1) & 511, 0.0);
    __syncthreads();
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    double y = x;
    for (int i = 0; i < iters; ++i) y = y * a;
    long long t2 = clock64();
    double z = y;
    for (int i = 0; i < iters; ++i) z = z + b;
    long long t3 = clock64();
    int idx = threadIdx.x & 1023;
    for (int i = 0; i < iters; ++i) idx = static_cast<int>(sm[idx]);
    long long t4 = clock64();
    int j = threadIdx.x & 511;
    for (int i = 0; i < iters; ++i) j = static_cast<int>(sm2[j].x);
    long long t5 = clock64();
    int k = threadIdx.x & 255;
    for (int i = 0; i < iters; ++i) k = static_cast<int>(cst[k]) & 255;
    long long t6 = clock64();
    out[threadIdx.x] = x + y + z + idx + j + k;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
    }
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaMallocManaged(&cyc, 8 * sizeof(long long));
    double h[256];
    for (int i = 0; i < 256; ++i) h[i] = (i * 11 + 5) & 255;
    cudaMemcpyToSymbol(cst, h, sizeof(h));
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        lat_kernel<<<1, 32>>>(out, cyc, iters, 0.999999, 1e-9);
        cudaDeviceSynchronize();
    }
    const char* names[] = {"DFMA", "DMUL", "DADD", "LDS.64 (+F2I)", "LDS.128 (+F2I)", "LDC indexed (+F2I)"};
    for (int i = 0; i < 6; ++i) printf("%-20s %.1f cycles per dependent op\n", names[i], double(cyc[i]) / iters);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
