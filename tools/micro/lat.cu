// Latency microbenchmarks (dependent chains, one warp): DADD, DMUL, FADD, LDS.64,
// SHFL, global load (L2 hit), integer division by a runtime value.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x, int n, int dv) {
    __shared__ double s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (double)((i * 7 + 1) & 1023);
    __syncthreads();
    double a = x, b = x * 0.5;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < n; ++i) { a = a + b; a = a + b; a = a + b; a = a + b; }
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < n; ++i) { a = a * 1.0000001; a = a * 0.9999999; a = a * 1.0000001; a = a * 0.9999999; }
    long long t2 = clock64();
    float f = (float)x;
#pragma unroll 1
    for (int i = 0; i < n; ++i) { f = f + 1.5f; f = f + 1.5f; f = f + 1.5f; f = f + 1.5f; }
    long long t3 = clock64();
    int idx = threadIdx.x & 1;
#pragma unroll 1
    for (int i = 0; i < n; ++i) { idx = (int)s[idx]; idx = (int)s[idx]; idx = (int)s[idx]; idx = (int)s[idx]; }
    long long t4 = clock64();
    double c = a;
#pragma unroll 1
    for (int i = 0; i < n; ++i) { c = __shfl_sync(0xffffffff, c, (threadIdx.x + 1) & 31); c = __shfl_sync(0xffffffff, c, (threadIdx.x + 1) & 31); c = __shfl_sync(0xffffffff, c, (threadIdx.x + 1) & 31); c = __shfl_sync(0xffffffff, c, (threadIdx.x + 1) & 31); }
    long long t5 = clock64();
    int q = n * 977 + 12345;
#pragma unroll 1
    for (int i = 0; i < n; ++i) { q = q / dv + 100000; q = q / dv + 100000; q = q / dv + 100000; q = q / dv + 100000; }
    long long t6 = clock64();
    double d = 0;
#pragma unroll 1
    for (int i = 0; i < n; ++i) { d = d + a / (b + d); }
    long long t7 = clock64();
    out[threadIdx.x] = a + f + idx + c + q + d;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6;
    }
}
int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 64);
    const int n = 1000;
    const char* nm[] = {"DADD", "DMUL", "FADD", "LDS.64+F2I", "SHFL.64", "IDIV(rt)", "DDIV"};
    // one warp, then 18 warps on one SM (the streaming kernel's residency): cycles
    // per dependent operation as seen by warp 0
    for (int threads : {32, 576}) {
        k<<<1, threads>>>(out, cyc, 1.25, n, 3);
        cudaDeviceSynchronize();
        k<<<1, threads>>>(out, cyc, 1.25, n, 3);
        cudaDeviceSynchronize();
        printf("-- %d warps on one SM\n", threads / 32);
        for (int i = 0; i < 7; ++i) printf("%-12s %6.1f cycles\n", nm[i], (double)cyc[i] / (i == 6 ? n : 4 * n));
    }
    return 0;
}
