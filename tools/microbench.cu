// tools/microbench.cu — calibration of the B200 memory system for the
// Douglas-ADI arrays (config 1: 256 x 128 x 128 FP64). Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NR = 256, NV = 128, NY = 128;
constexpr int SR = NV * NY;
constexpr size_t N = size_t(NR) * SR;

__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b) {
    size_t q = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (q < N) b[q] = a[q];
}

__global__ void k_fma(const double* __restrict__ a, double* __restrict__ b, int reps) {
    size_t q = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (q >= N) return;
    double x = a[q], y = 1.0;
    for (int r = 0; r < reps; ++r) y = fma(y, x, 1e-3);
    b[q] = y;
}

__global__ void k_stencil7(const double* __restrict__ u, double* __restrict__ d) {
    const int k = blockIdx.x * 32 + threadIdx.x, j = blockIdx.y * 8 + threadIdx.y, i = blockIdx.z;
    if (i == 0 || i == NR - 1 || j == 0 || j == NV - 1 || k == 0 || k == NY - 1) return;
    const size_t q = (size_t(i) * NV + j) * NY + k;
    const double* p = u + q;
    d[q] = 0.1 * (p[SR] + p[-SR]) + 0.2 * (p[NY] + p[-NY]) + 0.3 * (p[1] + p[-1]) - 1.2 * p[0] +
           0.05 * ((p[SR + NY] - p[SR - NY]) - (p[NY - SR] - p[-SR - NY]));
}

int main() {
    double *a, *b, *flush;
    cudaMalloc(&a, N * 8);
    cudaMalloc(&b, N * 8);
    cudaMalloc(&flush, 256 << 20);
    cudaMemset(a, 0, N * 8);
    cudaMemset(b, 0, N * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](const char* name, auto launch, double bytes, bool warm) {
        for (int w = 0; w < 3; ++w) launch();
        float best = 1e9;
        for (int it = 0; it < 10; ++it) {
            if (!warm) cudaMemset(flush, it, 256 << 20);
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("%-28s %s %8.2f us  %8.1f GB/s\n", name, warm ? "L2-warm" : "cold  ", best * 1e3,
               bytes / (best * 1e-3) / 1e9);
    };
    for (int warm = 0; warm < 2; ++warm) {
        time("copy", [&] { k_copy<<<(N + 255) / 256, 256>>>(a, b); }, 16.0 * N, warm);
        time("stencil7+cross", [&] { k_stencil7<<<dim3(NY / 32, NV / 8, NR), dim3(32, 8)>>>(a, b); },
             16.0 * N, warm);
        time("fma x32 (DP throughput)", [&] { k_fma<<<(N + 255) / 256, 256>>>(a, b, 32); }, 16.0 * N, warm);
    }
    // DP throughput: 32 FMA per node
    printf("DP rate check: 32 DFMA x %zu nodes\n", N);
    return 0;
}
