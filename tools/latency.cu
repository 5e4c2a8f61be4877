// tools/latency.cu — dependent-chain latencies of the FP64 and data-movement
// instructions the Douglas-ADI kernels are built from (one warp, clock64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/latency tools/latency.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void k_lat(double* out, long long* cyc, double a, double b) {
    __shared__ double sm[64];
    const int t = threadIdx.x;
    sm[t] = a + t;
    __syncthreads();
    double x = a + t * 1e-9, y = b;
    long long c0, c1;
    // DFMA chain
    c0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = fma(x, y, 1e-12);
    c1 = clock64();
    if (t == 0) cyc[0] = c1 - c0;
    // DADD chain
    c0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = x + y;
    c1 = clock64();
    if (t == 0) cyc[1] = c1 - c0;
    // DMUL chain
    c0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = x * y;
    c1 = clock64();
    if (t == 0) cyc[2] = c1 - c0;
    // MUFU.RCP64H seed chain
    c0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) {
        double r;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        x = r;
    }
    c1 = clock64();
    if (t == 0) cyc[3] = c1 - c0;
    // 64-bit shuffle chain
    c0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
    c1 = clock64();
    if (t == 0) cyc[4] = c1 - c0;
    // LDS.64 pointer-chase-like chain (address depends on the loaded value)
    int idx = t;
    c0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) idx = (static_cast<int>(sm[idx]) + i) & 31;
    c1 = clock64();
    if (t == 0) cyc[5] = c1 - c0;
    // DSETP + select chain
    c0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = (x > y) ? x * 0.5 : x;
    c1 = clock64();
    if (t == 0) cyc[6] = c1 - c0;
    out[t] = x + idx;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64 * sizeof(double));
    cudaMalloc(&cyc, 8 * sizeof(long long));
    k_lat<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
    k_lat<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
    long long h[8];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    const char* names[] = {"DFMA", "DADD", "DMUL", "MUFU.RCP64H", "SHFL.BFLY (64-bit)", "LDS dependent", "DSETP+select+DMUL"};
    for (int i = 0; i < 7; ++i) printf("%-20s %6.1f cycles per dependent op\n", names[i], double(h[i]) / N);
    return 0;
}
