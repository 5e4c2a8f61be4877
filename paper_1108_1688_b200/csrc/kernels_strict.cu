// kernels_strict.cu — STRICT-mode Douglas-ADI step for sm_100a.
//
// Compiled with -fmad=false: every expression below keeps the reference's
// operation order and rounding (true IEEE divides, no FMA contraction), so the
// device step reproduces douglas_step (solver.cpp:81-178) bit for bit except
// for the libm ulp of exp() in closed-form face values. It is the parity
// baseline of the FAST kernels (kernels_fast.cu), not the benchmarked path.
//
// Kernels per step (one launch each, all problems of the batch at once):
//   k_explicit   dU0 = dt*F(U) + Dirichlet increments   solver.cpp:96-116,
//                F = apply_operator                     discretization.cpp:302-364
//   k_sweep<R>   r-lines (stride nv*ny), Thomas          solver.cpp:121-134
//   k_sweep<V>   v-lines (stride ny)                     solver.cpp:136-149
//   k_sweep<Y>   y-lines (contiguous)                    solver.cpp:151-161
//   k_update     U += dU, max|dU|, Dirichlet, guard      solver.cpp:163-176
#include <cfloat>
#include <cmath>

#include "kernels_common.cuh"

namespace hjmsv_b200 {
namespace {
using namespace dev;

struct G {
    double g1, g2, g3, g4, g5, g6, reaction;
};

// HjmCoefficientField::at (discretization.cpp:56-72), literal order
__device__ __forceinline__ G coeff(const ProblemConst& pc, const Tab& T, double c4, int i, int j,
                                   int k) {
    const double v = T.vz[j];
    const double yt = T.yz[k];
    const double h1 = T.a[i] * v;
    const double h2 = T.heps2 * v;
    const double jr = T.rj1[i], jv = T.vj1[j];
    G g;
    g.g1 = h1 / (jr * jr);
    g.g2 = h2 / (jv * jv);
    g.g3 = T.b[i] * v / (jr * jv);
    g.g4 = (c4 - pc.kappa * T.rz[i] + pc.r0 * yt) / jr - h1 * T.rj2[i] / (jr * jr * jr);
    g.g5 = pc.theta * (1.0 - v) / jv - h2 * T.vj2[j] / (jv * jv * jv);
    g.g6 = (2.0 * h1 - 2.0 * pc.kappa * yt) / T.yj1[k];
    g.reaction = T.rz[i] * pc.r0;
    return g;
}

// ---------------------------------------------------------------- explicit
__global__ void k_explicit(BatchView v, int s) {
    const int p = blockIdx.y;
    const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    DevStatus& st = v.st[p];
    if (failed_before(st, s)) return;
    if (q == 0) st.maxdelta_bits = 0ull;
    if (q >= v.N) return;
    const int nv = v.nv, ny = v.ny, nr = v.nr;
    const int k = static_cast<int>(q % ny);
    const int j = static_cast<int>((q / ny) % nv);
    const int i = static_cast<int>(q / (static_cast<long long>(ny) * nv));
    const ProblemConst& pc = v.pc[p];
    const Tab T = tables(v, p, s);
    const double* step = step_row(v, p, s);
    const double* U = v.U + static_cast<size_t>(p) * v.N;
    double* D = v.D + static_cast<size_t>(p) * v.N;

    const int face = dirichlet_face(v, pc, i, j, k);
    if (face >= 0) {  // solver.cpp:111-116 (apply_operator alone: 0, discretization.cpp:314-316)
        D[q] = v.apply_only ? 0.0 : face_value(pc, step, T, face, i, k) - U[q];
        return;
    }
    const double dxr = v.dxr, dxv = v.dxv, dxy = v.dxy;
    const double inv_dxr2 = nr > 1 ? 1.0 / (dxr * dxr) : 0.0;
    const double inv_2dxr = nr > 1 ? 0.5 / dxr : 0.0;
    const double inv_dxv2 = nv > 1 ? 1.0 / (dxv * dxv) : 0.0;
    const double inv_2dxv = nv > 1 ? 0.5 / dxv : 0.0;
    const double inv_2dxy = ny > 1 ? 0.5 / dxy : 0.0;
    const double inv_cross = 0.25 / (dxr * dxv);
    const long long sr = static_cast<long long>(nv) * ny, sv = ny;

    const G c = coeff(pc, T, step[ST_C4], i, j, k);
    const double u0 = U[q];
    double acc = -c.reaction * u0;
    if (nr > 1) {
        if (i == 0) {
            if (v.r_order == 1)
                acc += c.g4 * (U[q + sr] - u0) / dxr;
            else
                acc += c.g4 * (-U[q + 2 * sr] + 4.0 * U[q + sr] - 3.0 * u0) * inv_2dxr;
        } else {
            const double up = U[q + sr], dn = U[q - sr];
            acc += c.g1 * (up - 2.0 * u0 + dn) * inv_dxr2 + c.g4 * (up - dn) * inv_2dxr;
        }
    }
    if (nv > 1) {
        if (j == 0) {
            acc += c.g5 * (U[q + sv] - u0) / dxv;
        } else {
            const double up = U[q + sv], dn = U[q - sv];
            acc += c.g2 * (up - 2.0 * u0 + dn) * inv_dxv2 + c.g5 * (up - dn) * inv_2dxv;
        }
    }
    if (ny > 1) {
        if (k == 0) {
            if (v.y_order == 1)
                acc += c.g6 * (U[q + 1] - u0) / dxy;
            else
                acc += c.g6 * (-U[q + 2] + 4.0 * U[q + 1] - 3.0 * u0) * inv_2dxy;
        } else {
            acc += c.g6 * (U[q + 1] - U[q - 1]) * inv_2dxy;
        }
    }
    if (i > 0 && i < nr - 1 && j > 0 && j < nv - 1) {
        acc += c.g3 * inv_cross *
               (U[q + sr + sv] - U[q + sr - sv] - U[q - sr + sv] + U[q - sr - sv]);
    }
    D[q] = acc * pc.dt;  // solver.cpp:99
}

// ---------------------------------------------------------------- sweeps
// thomas_solve_inplace (solver.cpp:22-57) on a strided line held in x, with
// the modified superdiagonal c' in cs. Rows come from `row(i, l, d, u, s2)`.
template <class RowFn>
__device__ __forceinline__ int thomas_line(int n, double* x, double* cs, long long stride,
                                           RowFn row) {
    double l0, d0, u0, s2;
    row(0, l0, d0, u0, s2);
    double r0 = x[0] + 0.0;  // rhs += rhs_adjust (identically zero)
    if (s2 != 0.0 && n > 2) {
        double l1, d1, u1, t1;
        row(1, l1, d1, u1, t1);
        if (fabs(u1) > 1e-300) {
            const double f = s2 / u1;
            d0 -= f * l1;
            u0 -= f * d1;
            r0 -= f * (x[stride] + 0.0);
        } else {
            r0 -= s2 * (x[2 * stride] + 0.0);
        }
    }
    double piv = d0;
    if (fabs(piv) < 1e-300) return 0;
    double cp = u0 / piv;
    double dp = r0 / piv;
    cs[0] = cp;
    x[0] = dp;
    for (int i = 1; i < n; ++i) {
        double l, d, u, t;
        row(i, l, d, u, t);
        piv = d - l * cp;
        if (fabs(piv) < 1e-300) return i;
        cp = u / piv;
        dp = ((x[i * stride] + 0.0) - l * dp) / piv;
        cs[i * stride] = cp;
        x[i * stride] = dp;
    }
    double xn = dp;
    for (int i = n - 2; i >= 0; --i) {
        xn = x[i * stride] - cs[i * stride] * xn;
        x[i * stride] = xn;
    }
    return -1;
}

enum Axis3 { AX_R = 0, AX_V = 1, AX_Y = 2 };

template <int AX>
__global__ void k_sweep(BatchView v, int s) {
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (failed_before(st, s)) return;
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const int lines = AX == AX_R ? nv * ny : (AX == AX_V ? nr * ny : nr * nv);
    const int line = blockIdx.x * blockDim.x + threadIdx.x;
    if (line >= lines) return;
    int i = 0, j = 0, k = 0;
    if (AX == AX_R) { j = line / ny; k = line % ny; }
    if (AX == AX_V) { i = line / ny; k = line % ny; }
    if (AX == AX_Y) { i = line / nv; j = line % nv; }
    const ProblemConst& pc = v.pc[p];
    // whole line prescribed (solver.cpp:127, 142, 156)
    if (AX == AX_R && is_dirichlet(v, pc, 1, j, k)) return;
    if (AX == AX_V && is_dirichlet(v, pc, i, 1, k)) return;
    if (AX == AX_Y && ny > 1 && is_dirichlet(v, pc, i, j, 1)) return;

    const Tab T = tables(v, p, s);
    const double c4 = step_row(v, p, s)[ST_C4];
    const double th = pc.theta_dt;
    const long long base = static_cast<long long>(i) * nv * ny + static_cast<long long>(j) * ny + k;
    double* x = v.D + static_cast<size_t>(p) * v.N + base;
    double* cs = v.C + static_cast<size_t>(p) * v.N + base;
    int bad = -1;
    if (AX == AX_R) {
        const double dxr = v.dxr;
        const int order = v.r_order;
        // assemble_line_r (discretization.cpp:194-230)
        auto row = [&](int ii, double& l, double& d, double& u, double& s2) {
            l = 0.0; d = 1.0; u = 0.0; s2 = 0.0;
            if (is_dirichlet(v, pc, ii, j, k)) return;
            const G c = coeff(pc, T, c4, ii, j, k);
            if (ii == 0) {
                const double w = c.g4 / dxr;
                if (order == 1) {
                    d = 1.0 + th * w;
                    u = -th * w;
                } else {
                    d = 1.0 + th * 1.5 * w;
                    u = -th * 2.0 * w;
                    s2 = th * 0.5 * w;
                }
            } else {
                const double w2 = c.g1 / (dxr * dxr);
                const double w1 = c.g4 / (2.0 * dxr);
                l = -th * (w2 - w1);
                d = 1.0 + th * 2.0 * w2;
                u = -th * (w2 + w1);
            }
        };
        bad = thomas_line(nr, x, cs, static_cast<long long>(nv) * ny, row);
    } else if (AX == AX_V) {
        const double dxv = v.dxv;
        // assemble_line_v (discretization.cpp:232-259)
        auto row = [&](int jj, double& l, double& d, double& u, double& s2) {
            l = 0.0; d = 1.0; u = 0.0; s2 = 0.0;
            if (is_dirichlet(v, pc, i, jj, k)) return;
            const G c = coeff(pc, T, c4, i, jj, k);
            if (jj == 0) {
                d = 1.0 + th * c.g5 / dxv;
                u = -th * c.g5 / dxv;
            } else {
                const double w2 = c.g2 / (dxv * dxv);
                const double w1 = c.g5 / (2.0 * dxv);
                l = -th * (w2 - w1);
                d = 1.0 + th * 2.0 * w2;
                u = -th * (w2 + w1);
            }
        };
        bad = thomas_line(nv, x, cs, ny, row);
    } else {
        const double dxy = v.dxy;
        const int order = v.y_order;
        // assemble_line_y (discretization.cpp:261-300)
        auto row = [&](int kk, double& l, double& d, double& u, double& s2) {
            l = 0.0; d = 1.0; u = 0.0; s2 = 0.0;
            if (ny == 1) {
                if (is_dirichlet(v, pc, i, j, 0)) return;
                const G c = coeff(pc, T, c4, i, j, 0);
                d = 1.0 + th * c.reaction;
                return;
            }
            if (is_dirichlet(v, pc, i, j, kk)) return;
            const G c = coeff(pc, T, c4, i, j, kk);
            if (kk == 0) {
                const double w = c.g6 / dxy;
                if (order == 1) {
                    d = 1.0 + th * (w + c.reaction);
                    u = -th * w;
                } else {
                    d = 1.0 + th * (1.5 * w + c.reaction);
                    u = -th * 2.0 * w;
                    s2 = th * 0.5 * w;
                }
            } else {
                const double w1 = c.g6 / (2.0 * dxy);
                l = th * w1;
                d = 1.0 + th * c.reaction;
                u = -th * w1;
            }
        };
        bad = thomas_line(ny, x, cs, 1, row);
    }
    if (bad >= 0) {
        const unsigned long long key = (static_cast<unsigned long long>(AX) << 50) |
                                       (static_cast<unsigned long long>(line) << 20) |
                                       static_cast<unsigned long long>(bad);
        atomicMin(&st.pivot_key, key);
        mark_fail(st, s + 1, HJMSV_SINGULAR_PIVOT);
    }
}

// ---------------------------------------------------------------- update
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long x) {
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, x, o);
        x = y > x ? y : x;
    }
    return x;
}

__global__ void k_update(BatchView v, int s) {
    const int p = blockIdx.y;
    const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    DevStatus& st = v.st[p];
    if (failed_before(st, s)) return;  // uniform per block: p is per block
    unsigned long long md = 0ull;
    if (q < v.N) {
        const int nv = v.nv, ny = v.ny;
        const int k = static_cast<int>(q % ny);
        const int j = static_cast<int>((q / ny) % nv);
        const int i = static_cast<int>(q / (static_cast<long long>(ny) * nv));
        const ProblemConst& pc = v.pc[p];
        double* U = v.U + static_cast<size_t>(p) * v.N;
        const double dq = v.D[static_cast<size_t>(p) * v.N + q];
        double un = U[q] + dq;
        // std::max(max_delta, |d|) never adopts a NaN (solver.cpp:166)
        const double ad = fabs(dq);
        if (ad > 0.0) md = static_cast<unsigned long long>(__double_as_longlong(ad));
        const int face = dirichlet_face(v, pc, i, j, k);
        if (face >= 0) un = face_value(pc, step_row(v, p, s), tables(v, p, s), face, i, k);
        U[q] = un;
        // guard_finite (solver.cpp:69-77)
        if (!isfinite(un)) {
            atomicMin(&st.nonfinite_first, static_cast<unsigned long long>(q));
            mark_fail(st, s + 1, HJMSV_NONFINITE);
        } else if (fabs(un) > pc.bound) {
            atomicMin(&st.diverge_first, static_cast<unsigned long long>(q));
            mark_fail(st, s + 1, HJMSV_DIVERGED);
        }
    }
    md = warp_max_u64(md);
    if ((threadIdx.x & 31) == 0 && md) atomicMax(&st.maxdelta_bits, md);
}

__global__ void k_reset_status(DevStatus* st, int P) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    st[p].fail_step = 0;
    st[p].fail_code = 0;
    st[p].pivot_key = ~0ull;
    st[p].nonfinite_first = ~0ull;
    st[p].diverge_first = ~0ull;
    st[p].maxdelta_bits = 0ull;
}

// interpolate_at (instruments.cpp:71-88): the host resolves the 8 corner
// indices and weights; zero weights are skipped like the reference.
__global__ void k_gather_spot(BatchView v, const long long* idx, const double* w, double* out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= v.P) return;
    const double* U = v.U + static_cast<size_t>(p) * v.N;
    double acc = 0.0;
    for (int c = 0; c < 8; ++c) {
        const double ww = w[p * 8 + c];
        if (ww == 0.0) continue;
        acc += ww * U[idx[p * 8 + c]];
    }
    out[p] = acc;
}

__global__ void k_thomas_batch(int n, int count, const double* lower, const double* diag,
                               const double* upper, const double* super2, double* rhs,
                               double* scratch, int* fail_row) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= count) return;
    const size_t o = static_cast<size_t>(q) * n;
    auto row = [&](int i, double& l, double& d, double& u, double& s2) {
        l = lower[o + i];
        d = diag[o + i];
        u = upper[o + i];
        s2 = i == 0 ? super2[q] : 0.0;
    };
    fail_row[q] = thomas_line(n, rhs + o, scratch + o, 1, row);
}

}  // namespace

void strict_step(const BatchView& v, int s, cudaStream_t stream, long long* launches,
                 const LaunchHook* hook) {
    auto mark = [&](int idx, const char* name, double bytes) {
        if (launches) ++*launches;
        if (hook && hook->after) hook->after(hook->ctx, idx, name, bytes);
    };
    const int tpb = 256;
    const dim3 grid_pts(static_cast<unsigned>((v.N + tpb - 1) / tpb), v.P);
    // algorithmic bytes/point: read U, write dU (16) | read+write the line (16) |
    // read dU, read U, write U (24)
    k_explicit<<<grid_pts, tpb, 0, stream>>>(v, s);
    mark(0, "strict_explicit", 16.0);
    const int ltpb = 128;
    if (v.nr > 1) {
        k_sweep<AX_R><<<dim3((v.nv * v.ny + ltpb - 1) / ltpb, v.P), ltpb, 0, stream>>>(v, s);
        mark(1, "strict_sweep_r", 16.0);
    }
    if (v.nv > 1) {
        k_sweep<AX_V><<<dim3((v.nr * v.ny + ltpb - 1) / ltpb, v.P), ltpb, 0, stream>>>(v, s);
        mark(2, "strict_sweep_v", 16.0);
    }
    k_sweep<AX_Y><<<dim3((v.nr * v.nv + ltpb - 1) / ltpb, v.P), ltpb, 0, stream>>>(v, s);
    mark(3, "strict_sweep_y", 16.0);
    k_update<<<grid_pts, tpb, 0, stream>>>(v, s);
    mark(4, "strict_update", 24.0);
}

void strict_explicit(const BatchView& v, int s, cudaStream_t stream) {
    const int tpb = 256;
    k_explicit<<<dim3(static_cast<unsigned>((v.N + tpb - 1) / tpb), v.P), tpb, 0, stream>>>(v, s);
}

void reset_status(const BatchView& v, cudaStream_t stream) {
    k_reset_status<<<(v.P + 127) / 128, 128, 0, stream>>>(v.st, v.P);
}

void gather_spot(const BatchView& v, const long long* idx, const double* w, double* out,
                 cudaStream_t stream) {
    k_gather_spot<<<(v.P + 127) / 128, 128, 0, stream>>>(v, idx, w, out);
}

void thomas_batch(int n, int count, const double* lower, const double* diag, const double* upper,
                  const double* super2, double* rhs, double* scratch, int* fail_row, int fast,
                  cudaStream_t stream) {
    if (fast) {  // 1: pass A's partition solver, 2: pass B's twisted one
        fast_thomas_batch(n, count, lower, diag, upper, super2, rhs, fail_row, fast == 2, stream);
        return;
    }
    k_thomas_batch<<<(count + 127) / 128, 128, 0, stream>>>(n, count, lower, diag, upper, super2,
                                                            rhs, scratch, fail_row);
}

}  // namespace hjmsv_b200
