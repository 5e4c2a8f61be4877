// kernels_readout.cu — device readouts of a solved level, SURVEY §8f row 2:
// extract_greeks (instruments.cpp:90-132: rho = dU/dr~ and vega = dU/dv by
// central differences in computational coordinates over the Jacobian j1,
// 2nd-order one-sided on the faces), finish()'s rate scaling rho /= r0
// (instruments.cpp:150-152) and write_surface_csv's k-slice (job.cpp:300-310),
// so only the requested planes cross PCIe. Built with -fmad=false in the
// reference's operation order: bit-identical to the host loops.
#include "device_types.hpp"

namespace hjmsv_b200 {
namespace {

__global__ void k_greeks(BatchView v, int p, int scale, double r0, double* rho, double* vega) {
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (q >= v.N) return;
    const int k = static_cast<int>(q % ny);
    const int j = static_cast<int>((q / ny) % nv);
    const int i = static_cast<int>(q / (static_cast<long long>(ny) * nv));
    const double* u = v.U + static_cast<size_t>(p) * v.N;
    const double* t = v.axes + static_cast<size_t>(p) * v.axes_stride;
    const double* rj1 = t + nr;
    const double* vj1 = t + 3 * nr + nv;
    auto at = [&](int a, int b, int c) { return u[(static_cast<size_t>(a) * nv + b) * ny + c]; };
    double dr = 0.0;
    if (nr > 1) {
        if (i == 0)
            dr = (-3.0 * at(0, j, k) + 4.0 * at(1, j, k) - at(2, j, k)) / (2.0 * v.dxr);
        else if (i == nr - 1)
            dr = (3.0 * at(i, j, k) - 4.0 * at(i - 1, j, k) + at(i - 2, j, k)) / (2.0 * v.dxr);
        else
            dr = (at(i + 1, j, k) - at(i - 1, j, k)) / (2.0 * v.dxr);
        dr /= rj1[i];
    }
    double dv = 0.0;
    if (nv > 1) {
        if (j == 0)
            dv = (-3.0 * at(i, 0, k) + 4.0 * at(i, 1, k) - at(i, 2, k)) / (2.0 * v.dxv);
        else if (j == nv - 1)
            dv = (3.0 * at(i, j, k) - 4.0 * at(i, j - 1, k) + at(i, j - 2, k)) / (2.0 * v.dxv);
        else
            dv = (at(i, j + 1, k) - at(i, j - 1, k)) / (2.0 * v.dxv);
        dv /= vj1[j];
    }
    if (scale) dr /= r0;  // finish(): x /= mesh.r0
    if (rho) rho[q] = dr;
    if (vega) vega[q] = dv;
}

// write_surface_csv rows at slice k: (r0 z_r, z_v, U, rho, vega) per (i, j)
__global__ void k_surface(BatchView v, int p, int k, double r0, const double* rho,
                          const double* vega, double* out) {
    const int nv = v.nv, ny = v.ny;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= v.nr * nv) return;
    const int i = q / nv, j = q - i * nv;
    const double* t = v.axes + static_cast<size_t>(p) * v.axes_stride;
    const size_t idx = (static_cast<size_t>(i) * nv + j) * ny + k;
    double* o = out + static_cast<size_t>(q) * 5;
    o[0] = r0 * t[i];
    o[1] = t[3 * v.nr + j];
    o[2] = v.U[static_cast<size_t>(p) * v.N + idx];
    o[3] = rho[idx];
    o[4] = vega[idx];
}

}  // namespace

void greeks(const BatchView& v, int p, int scale, double r0, double* rho, double* vega,
            cudaStream_t stream) {
    k_greeks<<<static_cast<unsigned>((v.N + 255) / 256), 256, 0, stream>>>(v, p, scale, r0, rho, vega);
}

void surface(const BatchView& v, int p, int k, double r0, const double* rho, const double* vega,
             double* out, cudaStream_t stream) {
    const int n = v.nr * v.nv;
    k_surface<<<(n + 255) / 256, 256, 0, stream>>>(v, p, k, r0, rho, vega, out);
}

}  // namespace hjmsv_b200
