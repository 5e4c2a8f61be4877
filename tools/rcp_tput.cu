// tools/rcp_tput.cu — throughput of FP64 reciprocal recipes on a full SM
// (many warps, independent chains): the MUFU.RCP64H seed + cubic Newton step of
// kernels_fast.cu's frcp against an FP32 MUFU.RCP seed + the same step, and a
// pure DFMA baseline.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rcp_tput tools/rcp_tput.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 2048;
constexpr int ILP = 4;

__device__ __forceinline__ double rcp64h(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
}
__device__ __forceinline__ double rcp32seed(double x) {
    const double r = static_cast<double>(__frcp_rn(static_cast<float>(x)));
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
}

template <int MODE>
__global__ void k(double* out, double a) {
    double x[ILP];
#pragma unroll
    for (int q = 0; q < ILP; ++q) x[q] = a + 1e-3 * (threadIdx.x + q);
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int q = 0; q < ILP; ++q) {
            if (MODE == 0) x[q] = rcp64h(x[q]) + 1.5;
            else if (MODE == 1) x[q] = rcp32seed(x[q]) + 1.5;
            else x[q] = fma(fma(fma(x[q], 0.5, 1.5), 0.25, 1.5), 0.5, 0.75) + 1.5;  // 4 FP64 ops
        }
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < ILP; ++q) s += x[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double* out;
    const int blocks = 148 * 4, threads = 256;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[] = {"MUFU.RCP64H + 3 DFMA + DADD", "F32 MUFU.RCP seed + 3 DFMA + DADD", "4 DFMA + DADD"};
    for (int m = 0; m < 3; ++m) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (m == 0) k<0><<<blocks, threads>>>(out, 1.3);
            if (m == 1) k<1><<<blocks, threads>>>(out, 1.3);
            if (m == 2) k<2><<<blocks, threads>>>(out, 1.3);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = double(blocks) * threads * N * ILP;
            if (rep) printf("%-36s %8.2f G recipes/s  (%.2f per SM per clock at 1.965 GHz)\n", names[m],
                            ops / ms / 1e6, ops / ms / 1e6 / 148 / 1.965);
        }
    }
    return 0;
}
