// tools/tma_probe.cu — standalone check of pass A's TMA window: one 4-D box
// {18, 3, 1, S} of U viewed as [P*S][16][nv][ny], completed on an mbarrier,
// compared element by element with the global array (zeros outside).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/_tma_probe tools/tma_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__global__ void k(const __grid_constant__ CUtensorMap map, int c0, int c1, int c2, int c3, double* out, int n) {
    extern __shared__ __align__(128) double sm[];
    __shared__ alignas(8) unsigned long long bar;
    const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(sm));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n * 8) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
            ::"r"(d), "l"(reinterpret_cast<unsigned long long>(&map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(b)
            : "memory");
    }
    asm volatile("{\n .reg .pred P;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n @!P bra W_%=;\n}" ::"r"(b)
                 : "memory");
    for (int e = threadIdx.x; e < n; e += blockDim.x) out[e] = sm[e];
}

int main(int argc, char** argv) {
    const int nr = 64, nv = 32, ny = 32, P = 2, S = nr / 16;
    const size_t N = static_cast<size_t>(P) * nr * nv * ny;
    std::vector<double> h(N);
    for (size_t q = 0; q < N; ++q) h[q] = 1.0 + q;
    double *U, *out;
    cudaMalloc(&U, N * 8);
    cudaMemcpy(U, h.data(), N * 8, cudaMemcpyHostToDevice);
    int n = 18 * 3 * S;
    cudaMalloc(&out, n * 8);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cuuint64_t dims[4] = {(cuuint64_t)ny, (cuuint64_t)nv, 16, (cuuint64_t)P * S};
    cuuint64_t strides[3] = {(cuuint64_t)ny * 8, (cuuint64_t)nv * ny * 8, (cuuint64_t)16 * nv * ny * 8};
    const int variant = argc > 1 ? atoi(argv[1]) : 0;
    cuuint32_t box[4] = {18, 3, 1, (cuuint32_t)S};
    if (variant == 1) box[0] = 16;                      // 128-byte inner box
    if (variant == 2) { box[0] = 16; box[1] = 1; box[3] = 1; }  // one row
    if (variant >= 10) box[0] = variant;                // inner box of `variant` doubles
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUtensorMap m;
    CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, U, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("variant %d encode %d (query %d)\n", variant, (int)r, (int)q);
    n = box[0] * box[1] * box[2] * box[3];
    int bad = 0;
    if (variant) {
        const int cx = argc > 2 ? atoi(argv[2]) : 0;
        k<<<1, 128, n * 8>>>(m, cx, 0, 0, 0, out, n);
        cudaError_t e = cudaDeviceSynchronize();
        printf("variant %d c0 %d: %s\n", variant, cx, cudaGetErrorString(e));
        return 0;
    }
    const int cases[3][4] = {{15, 4, 3, 1}, {-1, -1, 15, -1}, {15, 30, 0, 5}};
    for (auto& c : cases) {
        k<<<1, 128, n * 8>>>(m, c[0], c[1], c[2], c[3], out, n);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("kernel error %s\n", cudaGetErrorString(e));
            return 1;
        }
        std::vector<double> o(n);
        cudaMemcpy(o.data(), out, n * 8, cudaMemcpyDeviceToHost);
        for (int ss = 0; ss < S; ++ss)
            for (int jj = 0; jj < 3; ++jj)
                for (int kk = 0; kk < 18; ++kk) {
                    const int K = c[0] + kk, J = c[1] + jj, R = c[2], SG = c[3] + ss;
                    double want = 0.0;
                    if (K >= 0 && K < ny && J >= 0 && J < nv && SG >= 0 && SG < P * S)
                        want = h[((static_cast<size_t>(SG) * 16 + R) * nv + J) * ny + K];
                    if (o[(ss * 3 + jj) * 18 + kk] != want) ++bad;
                }
        printf("case %d %d %d %d: bad %d\n", c[0], c[1], c[2], c[3], bad);
    }
    return bad != 0;
}
