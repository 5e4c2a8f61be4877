// kernels_terminal.cu — the terminal level on the device (FAST mode), SURVEY
// §8f row 1: ZCB terminal 1 (instruments.cpp:200-204) and the caplet payoff
// max(1 - accrual * P(T, T_M; x, y), 0) (caplet_payoff, model.cpp:105-112;
// P = zcb_closed_form, model.cpp:48-54) averaged over smooth_terminal's cells
// (solver.cpp:180-211): m midpoint samples per axis inside the half-spacing cell
// of interior nodes, the node itself on faces. Built with -fmad=false and in the
// host restatement's operation order (lowering.cpp caplet_terminal), so only
// exp() may differ from the host by an ulp.
//
// One thread per (problem, i, k): the payoff does not depend on v, so the
// thread sums the samples for the two v-cell sizes (1 on the v faces, m inside)
// in the reference's (r, v, y) loop order and writes the whole j column.
#include "device_types.hpp"

namespace hjmsv_b200 {
namespace {

struct Cell {
    double lo, w;
    int n;
};

// smooth_terminal's per-axis cell samples (solver.cpp:184-194)
__device__ __forceinline__ Cell cell(const double* z, int n, int i, int m) {
    Cell c;
    if (n == 1 || i == 0 || i == n - 1) {
        c.lo = z[i];
        c.w = 0.0;
        c.n = 1;
        return c;
    }
    const double lo = z[i] - 0.5 * (z[i] - z[i - 1]);
    const double hi = z[i] + 0.5 * (z[i + 1] - z[i]);
    c.lo = lo;
    c.w = (hi - lo) / m;
    c.n = m;
    return c;
}

__device__ __forceinline__ double sample(const Cell& c, int q, const double* z, int i) {
    return c.n == 1 ? z[i] : c.lo + (q + 0.5) * c.w;
}

__global__ void k_terminal(BatchView v, const TermParam* tps, double* U0) {
    const int p = blockIdx.y;
    const TermParam tp = tps[p];
    if (tp.kind == TERM_HOST) return;
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nr * ny) return;
    const int i = q / ny, k = q - i * ny;
    double* out = U0 + static_cast<size_t>(p) * v.N + static_cast<size_t>(i) * nv * ny + k;
    if (tp.kind == TERM_ONES) {
        for (int j = 0; j < nv; ++j) out[static_cast<size_t>(j) * ny] = 1.0;
        return;
    }
    const double* t = v.axes + static_cast<size_t>(p) * v.axes_stride;
    const double* rz = t;
    const double* yz = t + 3 * nr + 3 * nv;
    const int m = tp.m;
    const double r0 = tp.r0;
    auto payoff = [&](double zr, double zy) {
        const double tr = r0 * zr, ty = r0 * r0 * zy;
        const double x = tr - tp.f_t;
        const double pb = tp.ratio * exp(-tp.g * x - 0.5 * tp.g * tp.g * ty);
        const double value = 1.0 - tp.accrual * pb;
        return value > 0.0 ? value : 0.0;
    };
    if (m == 1) {  // no smoothing: the payoff at the node
        const double val = payoff(rz[i], yz[k]);
        for (int j = 0; j < nv; ++j) out[static_cast<size_t>(j) * ny] = val;
        return;
    }
    const Cell cr = cell(rz, nr, i, m), cy = cell(yz, ny, k, m);
    // v-cell sizes: 1 on the v faces (and a collapsed v axis), m inside
    double acc1 = 0.0, accm = 0.0;
    for (int qr = 0; qr < cr.n; ++qr) {
        const double zr = sample(cr, qr, rz, i);
        for (int qy = 0; qy < cy.n; ++qy) acc1 += payoff(zr, sample(cy, qy, yz, k));
        for (int qv = 0; qv < m; ++qv)
            for (int qy = 0; qy < cy.n; ++qy) accm += payoff(zr, sample(cy, qy, yz, k));
    }
    const double v1 = acc1 / static_cast<double>(cr.n * cy.n);
    const double vm = accm / static_cast<double>(cr.n * m * cy.n);
    for (int j = 0; j < nv; ++j) {
        const bool face = nv == 1 || j == 0 || j == nv - 1;
        out[static_cast<size_t>(j) * ny] = face ? v1 : vm;
    }
}

}  // namespace

void device_terminal(const BatchView& v, const TermParam* tp, const int* host_kinds, double* U0,
                     cudaStream_t stream) {
    bool any = false;
    for (int p = 0; p < v.P; ++p) any = any || host_kinds[p] != TERM_HOST;
    if (!any) return;
    const int n = v.nr * v.ny;
    k_terminal<<<dim3((n + 127) / 128, v.P), 128, 0, stream>>>(v, tp, U0);
}

}  // namespace hjmsv_b200
