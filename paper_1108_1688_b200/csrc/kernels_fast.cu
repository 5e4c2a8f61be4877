// kernels_fast.cu — FAST-mode Douglas-ADI step for sm_100a (the benchmarked path).
//
// Same discretisation, boundary rules and time levels as douglas_step
// (solver.cpp:81-178); the arithmetic is reorganised for the GPU:
//   * coefficients come from per-axis factor tables (lowering.cpp
//     build_fast_tables) with the stencil 1/dx factors folded in: a few FMAs per
//     node instead of ~25 mul/add + 8 divides (discretization.cpp:56-72);
//   * every tridiagonal line is solved by the PARTITION method: the line is cut
//     into segments of M rows, one thread (or lane) per segment eliminates its
//     rows for three right-hand sides sharing one factorisation
//         T y = r,  T alpha = -l_first e_0,  T beta = -u_last e_{m-1},
//     so x_i = y_i + alpha_i x_{before} + beta_i x_{after}; the end rows of all
//     segments of a line form a small reduced system solved with an O(S)
//     recurrence, after which every thread finishes its rows. Lines stay in
//     registers from load to store, and the parallelism is S times the line
//     count (config 1 has only 16384 r-lines);
//   * pivots use a hardware reciprocal seed + Newton (1 MUFU + 3 DFMA);
//   * the v-line matrix depends on j only: its LU is a table and the segmented
//     v-solve is two affine scans (5 FP64 ops per node).
// Kernels per step (each launch covers every problem of the batch):
//   k_fx_explicit  dU0 = dt*F(U) + Dirichlet increments          16 B/node
//   k_fx_r         segmented r-lines (strided, coalesced over k)   16 B/node
//   k_fx_v         segmented v-lines (strided, coalesced over k)   16 B/node
//   k_fx_y         warp-segmented y-lines (contiguous) fused with
//                  U += dU, Dirichlet re-impose, max|dU|, guard    24 B/node
// The elimination order is the only difference from the reference's
// sequential Thomas (the north star's allowed source of difference); local and
// reduced pivots stand in for the global ones in the singular-pivot check.
// Parity with the reference is 1e-10 normwise (tests/test_gpu_parity.py).
#include <algorithm>
#include <cstdlib>

#include "kernels_common.cuh"

namespace hjmsv_b200 {
namespace {
using namespace dev;

constexpr int kSegR = 16;  // rows per r-segment
constexpr int kLanesR = 16;
constexpr int kSegY = 8;   // rows per lane of a y-line

// 1/x: MUFU.RCP64H seed, then e = 1 - x r and r (1 + e + e^2): error ~e^3
__device__ __forceinline__ double frcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
}

struct FT {
    const double *R, *V, *Y;
};
__device__ __forceinline__ FT ftab(const BatchView& v, int p) {
    const double* t = v.fast + static_cast<size_t>(p) * v.fast_stride;
    FT f;
    f.R = t;
    f.V = t + kFR * v.nr;
    f.Y = f.V + kFV * v.nv;
    return f;
}

__device__ __forceinline__ void record_pivot(DevStatus& st, int s, int ax, int line, int row) {
    const unsigned long long key = (static_cast<unsigned long long>(ax) << 50) |
                                   (static_cast<unsigned long long>(line) << 20) |
                                   static_cast<unsigned long long>(row);
    atomicMin(&st.pivot_key, key);
    mark_fail(st, s + 1, HJMSV_SINGULAR_PIVOT);
}

// Dirichlet face at (i,j,k) from the batch-uniform rule mask, with the
// precedence of dirichlet_value (discretization.cpp:172-192); -1 otherwise.
__device__ __forceinline__ int dface(const BatchView& v, int i, int j, int k) {
    const int m = v.dmask;
    if ((m >> F_RMAX & 1) && i == v.nr - 1) return F_RMAX;
    if ((m >> F_YMAX & 1) && k == v.ny - 1) return F_YMAX;
    if ((m >> F_VMAX & 1) && j == v.nv - 1) return F_VMAX;
    if ((m >> F_RMIN & 1) && i == 0) return F_RMIN;
    if ((m >> F_YMIN & 1) && k == 0) return F_YMIN;
    if ((m >> F_VMIN & 1) && j == 0) return F_VMIN;
    return -1;
}
__device__ __forceinline__ bool dir(const BatchView& v, int f) { return v.dmask >> f & 1; }

// ============================================================ explicit operator
// Thread per node; block = 32 k x 8 j of one plane i. dU0 = dt*F(U) at interior
// nodes (apply_operator, discretization.cpp:302-364), face(t_next) - U on
// Dirichlet nodes (solver.cpp:111-116). apply_only (stage) writes F(U) and 0.
__global__ void __launch_bounds__(256) k_fx_explicit(BatchView v, int s) {
    const int p = blockIdx.z, i = blockIdx.y;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    if (blockIdx.x == 0 && i == 0 && threadIdx.x == 0 && threadIdx.y == 0) st.maxdelta_bits = 0ull;
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const int tk = (ny + 31) >> 5;
    const int jt = blockIdx.x / tk;
    const int j = jt * 8 + threadIdx.y, k = (blockIdx.x - jt * tk) * 32 + threadIdx.x;
    if (j >= nv || k >= ny) return;
    const ProblemConst& pc = v.pc[p];
    const int sr = nv * ny;
    const size_t off = static_cast<size_t>(p) * v.N;
    const int q = (i * nv + j) * ny + k;
    const double* __restrict__ u = v.U + off + q;
    const double* step = step_row(v, p, s);
    const FT F = ftab(v, p);
    const double* R = F.R + kFR * i;
    const double* V = F.V + kFV * j;
    const double* Y = F.Y + kFY * k;
    double out;
    if (i > 0 && i < nr - 1 && j > 0 && j < nv - 1 && k > 0 && k < ny - 1) {
        // interior node: full 11-point stencil, no face logic
        const double vj = V[FV_V];
        const double g4h =
            fma(step[ST_C4], R[FR_G4C], fma(R[FR_G4Q], Y[FY_Y], fma(R[FR_G4V], vj, R[FR_G4P])));
        const double g6h = fma(R[FR_A] * vj, Y[FY_S6], Y[FY_T6]);
        const double u0 = u[0];
        const double rp = u[sr], rm = u[-sr], vp = u[ny], vm = u[-ny];
        double acc = -R[FR_REACT] * u0;
        acc = fma(R[FR_G1] * vj, (rp + rm) - 2.0 * u0, acc);
        acc = fma(g4h, rp - rm, acc);
        acc = fma(V[FV_G2], (vp + vm) - 2.0 * u0, acc);
        acc = fma(V[FV_G5], vp - vm, acc);
        acc = fma(g6h, u[1] - u[-1], acc);
        acc = fma(R[FR_G3] * V[FV_G3], (u[sr + ny] - u[sr - ny]) - (u[ny - sr] - u[-sr - ny]), acc);
        out = acc * pc.dt;
    } else {
        const int face = dface(v, i, j, k);
        if (face >= 0) {
            out = v.apply_only ? 0.0 : face_value(pc, step, tables(v, p), face, i, k) - u[0];
        } else {
            const double vj = V[FV_V];
            const double g1s = R[FR_G1] * vj;
            const double g4h = fma(step[ST_C4], R[FR_G4C],
                                   fma(R[FR_G4Q], Y[FY_Y], fma(R[FR_G4V], vj, R[FR_G4P])));
            const double g6h = fma(R[FR_A] * vj, Y[FY_S6], Y[FY_T6]);
            const double u0 = u[0];
            double acc = -R[FR_REACT] * u0;
            if (i == 0) {
                const double u1 = u[sr];
                if (v.r_order == 1)
                    acc = fma(2.0 * g4h, u1 - u0, acc);
                else
                    acc = fma(g4h, fma(4.0, u1, -u[2 * sr]) - 3.0 * u0, acc);
            } else {
                const double up = u[sr], dn = u[-sr];
                acc = fma(g1s, (up + dn) - 2.0 * u0, acc);
                acc = fma(g4h, up - dn, acc);
            }
            if (j == 0) {
                acc = fma(2.0 * V[FV_G5], u[ny] - u0, acc);
            } else {
                const double up = u[ny], dn = u[-ny];
                acc = fma(V[FV_G2], (up + dn) - 2.0 * u0, acc);
                acc = fma(V[FV_G5], up - dn, acc);
            }
            if (k == 0) {
                const double u1 = u[1];
                if (v.y_order == 1)
                    acc = fma(2.0 * g6h, u1 - u0, acc);
                else
                    acc = fma(g6h, fma(4.0, u1, -u[2]) - 3.0 * u0, acc);
            } else {
                acc = fma(g6h, u[1] - u[-1], acc);
            }
            if (i > 0 && i < nr - 1 && j > 0 && j < nv - 1)
                acc = fma(R[FR_G3] * V[FV_G3],
                          (u[sr + ny] - u[sr - ny]) - (u[ny - sr] - u[-sr - ny]), acc);
            out = acc * pc.dt;
        }
    }
    v.D[off + q] = out;
}

// ============================================================ partition solve
// Local elimination of one segment (rows 0..m-1) for the three right-hand
// sides; on entry x[] holds the rhs, row(r, l, d, u) gives row r. On exit
// x[] = y, al[] = alpha, cs[] = c', and the end-row values are set.
template <int M, class RowFn>
__device__ __forceinline__ bool seg_solve(int m, double (&x)[M], double (&cs)[M], double (&al)[M],
                                          double& yF, double& aF, double& bF, double& yL,
                                          double& aL, double& bL, int& bad_r, RowFn row) {
    // pivots in projective form: P_r = d_r P_{r-1} - l_r u_{r-1} P_{r-2},
    // 1/piv_r = P_{r-1}/P_r, so the recurrence chain is one FMA per row and the
    // reciprocal is off it; y' and alpha' then carry one FMA / MUL per row.
    double pm1 = 1.0, pm2 = 0.0, uprev = 0.0, yprev = 0.0, aprev = 0.0;
    bool ok = true;
#pragma unroll
    for (int r = 0; r < M; ++r) {
        if (r < m) {
            double l, d, u;
            row(r, l, d, u);
            const double P = r == 0 ? d : fma(d, pm1, -(l * uprev) * pm2);
            const double rp = pm1 * frcp(P);
            if (fabs(rp) > 1e300 && ok) {  // |pivot| < 1e-300 (solver.cpp:44-52)
                ok = false;
                bad_r = r;
            }
            const bool last = r == m - 1;
            const double lrp = l * rp;
            const double c = last ? 0.0 : u * rp;  // the last row's upper couples outside
            const double yy = r == 0 ? x[r] * rp : fma(-lrp, yprev, x[r] * rp);
            const double aa = r == 0 ? -lrp : -lrp * aprev;
            if (last) {
                yL = yy;
                aL = aa;
                bL = -u * rp;
            }
            cs[r] = c;
            x[r] = yy;
            al[r] = aa;
            yprev = yy;
            aprev = aa;
            uprev = u;
            pm2 = pm1;
            pm1 = P;
            if (r % 8 == 7) {  // exact power-of-two rescaling keeps P in range
                const int e = ((__double2hiint(pm1) >> 20) & 0x7ff) - 1023;
                const double sc = __hiloint2double((1023 - e) << 20, 0);
                pm1 *= sc;
                pm2 *= sc;
            }
        }
    }
    double yn = yL, an = aL, bn = bL;
#pragma unroll
    for (int r = M - 2; r >= 0; --r) {
        if (r < m - 1) {
            yn = fma(-cs[r], yn, x[r]);
            an = fma(-cs[r], an, al[r]);
            bn = -cs[r] * bn;
            x[r] = yn;
            al[r] = an;
        }
    }
    yF = yn;
    aF = an;
    bF = bn;
    return ok;
}

// Reduced system of a line with S segments, unknowns p_t = x_last(t) and
// q_t = x_first(t+1), t = 0..S-2:
//   p_t = yL_t + aL_t p_{t-1} + bL_t q_t,   q_t = yF_{t+1} + aF_{t+1} p_t + bF_{t+1} q_{t+1}
// Forward: q_t = Qc_t + Qd_t q_{t+1}, p_t = Pp_t + Pq_t q_{t+1}; backward from
// q_{S-1} = 0. Segment t's data at E[t*stride + f] (f: yF aF bF yL aL bL); the
// results p_t, q_t overwrite fields 6, 7.
__device__ __forceinline__ bool reduced_solve(double* E, int S, int stride, int& bad_t) {
    double Pp = 0.0, Pq = 0.0;
    bool ok = true;
#pragma unroll 1
    for (int t = 0; t < S - 1; ++t) {
        double* e0 = E + t * stride;
        const double* e1 = e0 + stride;
        const double A = fma(e0[4], Pp, e0[3]);
        const double B = fma(e0[4], Pq, e0[5]);
        const double den = fma(-e1[1], B, 1.0);
        if (fabs(den) < 1e-300 && ok) {
            ok = false;
            bad_t = t + 1;
        }
        const double inv = frcp(den);
        const double Qc = fma(e1[1], A, e1[0]) * inv;
        const double Qd = e1[2] * inv;
        Pp = fma(B, Qc, A);
        Pq = B * Qd;
        e0[6] = Qc;
        e0[7] = Qd;
        e0[3] = Pp;
        e0[4] = Pq;
    }
    double qn = 0.0;
#pragma unroll 1
    for (int t = S - 2; t >= 0; --t) {
        double* e0 = E + t * stride;
        const double qs = fma(e0[7], qn, e0[6]);
        e0[6] = fma(e0[4], qn, e0[3]);  // p_t
        e0[7] = qs;                     // q_t
        qn = qs;
    }
    return ok;
}

// ============================================================ r-lines
// Block = kLanesR consecutive k (same j) x S segments of M rows.
template <int M>
__global__ void __launch_bounds__(512) k_fx_r(BatchView v, int s) {
    extern __shared__ double red[];  // [kLanesR][S][8]
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const int S = blockDim.y;
    const int tx = threadIdx.x, sg = threadIdx.y;
    const int tk = (ny + kLanesR - 1) / kLanesR;
    const int j = blockIdx.x / tk;
    const int k = (blockIdx.x - j * tk) * kLanesR + tx;
    const ProblemConst& pc = v.pc[p];
    const bool active = k < ny;
    // is_dirichlet(1,j,k) (solver.cpp:127): the column lies on a v or y Dirichlet face
    const bool solve = active && !(k == ny - 1 && dir(v, F_YMAX)) &&
                       !(j == nv - 1 && dir(v, F_VMAX)) &&
                       !(k == 0 && dir(v, F_YMIN)) &&
                       !(j == 0 && dir(v, F_VMIN));
    const int a = sg * M;
    const int m = min(M, nr - a);
    const int sr = nv * ny;
    double* __restrict__ col = v.D + static_cast<size_t>(p) * v.N + static_cast<size_t>(j) * ny +
                               (active ? k : 0) + static_cast<size_t>(a) * sr;
    double x[M], cs[M], al[M];
    if (solve) {
#pragma unroll
        for (int r = 0; r < M; ++r) x[r] = r < m ? col[static_cast<size_t>(r) * sr] : 0.0;
    }
    double* E = red + (tx * S + sg) * 8;
    if (solve) {
        const FT F = ftab(v, p);
        const double c4 = step_row(v, p, s)[ST_C4];
        const double vj = F.V[kFV * j + FV_V];
        const double yk = F.Y[kFY * k + FY_Y];
        const double th = pc.theta_dt;
        const bool rmaxD = dir(v, F_RMAX);
        const bool rminD = dir(v, F_RMIN);
        // rows of I - th*L_r (assemble_line_r, discretization.cpp:194-230)
        auto coeffs = [&](int i, double& l, double& d, double& u, double& s2) {
            l = 0.0; d = 1.0; u = 0.0; s2 = 0.0;
            if ((i == nr - 1 && rmaxD) || (i == 0 && rminD)) return;
            const double* R = F.R + kFR * i;
            const double g4h = fma(c4, R[FR_G4C], fma(R[FR_G4Q], yk, fma(R[FR_G4V], vj, R[FR_G4P])));
            if (i == 0) {
                if (v.r_order == 1) {
                    d = fma(2.0 * th, g4h, 1.0);
                    u = -2.0 * th * g4h;
                } else {
                    d = fma(3.0 * th, g4h, 1.0);
                    u = -4.0 * th * g4h;
                    s2 = th * g4h;
                }
            } else {
                const double w2 = th * R[FR_G1] * vj, w1 = th * g4h;
                l = w1 - w2;
                d = fma(2.0, w2, 1.0);
                u = -(w2 + w1);
            }
        };
        // row 0 of the line carries the (0,2) entry: fold it against row 1 (solver.cpp:28-40)
        double f0d = 1.0, f0u = 0.0;
        if (a == 0) {
            double l0, d0, u0, s20, l1, d1, u1, t1;
            coeffs(0, l0, d0, u0, s20);
            f0d = d0;
            f0u = u0;
            if (s20 != 0.0 && nr > 2) {
                coeffs(1, l1, d1, u1, t1);
                if (fabs(u1) > 1e-300) {
                    const double f = s20 / u1;
                    f0d = fma(-f, l1, d0);
                    f0u = fma(-f, d1, u0);
                    x[0] = fma(-f, x[1], x[0]);
                } else {
                    x[0] = fma(-s20, x[2], x[0]);
                }
            }
        }
        auto row = [&](int r, double& l, double& d, double& u) {
            if (a == 0 && r == 0) {
                l = 0.0;
                d = f0d;
                u = f0u;
                return;
            }
            double s2;
            coeffs(a + r, l, d, u, s2);
        };
        double yF, aF, bF, yL, aL, bL;
        int bad_r = 0;
        if (!seg_solve<M>(m, x, cs, al, yF, aF, bF, yL, aL, bL, bad_r, row))
            record_pivot(st, s, 0, j * ny + k, a + bad_r);
        E[0] = yF; E[1] = aF; E[2] = bF; E[3] = yL; E[4] = aL; E[5] = bL;
    }
    __syncthreads();
    if (sg == 0 && solve && S > 1) {
        int bt = 0;
        if (!reduced_solve(red + tx * S * 8, S, 8, bt)) record_pivot(st, s, 0, j * ny + k, bt * M);
    }
    __syncthreads();
    if (!solve) return;
    const double left = sg > 0 ? E[-8 + 6] : 0.0;  // p_{s-1} = x_{a-1}
    const double right = sg < S - 1 ? E[7] : 0.0;  // q_s = x_{a+m}
    double b = E[5];                               // beta_{m-1}
#pragma unroll
    for (int r = M - 1; r >= 0; --r) {
        if (r < m) {
            if (r < m - 1) b = -cs[r] * b;
            col[static_cast<size_t>(r) * sr] = fma(b, right, fma(al[r], left, x[r]));
        }
    }
}

// ============================================================ v-lines
// The LU of the v-line is a table (depends on j only), so both substitutions
// are affine scans: a block of 32 k x S segments (kSegV rows) computes local
// scans, carries the segment boundary values across segments in shared memory,
// and fixes its rows up with the in-segment products BF/BB.
__global__ void __launch_bounds__(512, 2) k_fx_v(BatchView v, int s) {
    extern __shared__ double car[];  // [2][S][32]
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const int S = blockDim.y;
    const int tx = threadIdx.x, sg = threadIdx.y;
    const int tk = (ny + 31) >> 5;
    const int i = blockIdx.x / tk;
    const int k = (blockIdx.x - i * tk) * 32 + tx;
    const ProblemConst& pc = v.pc[p];
    // is_dirichlet(i,1,k) (solver.cpp:142)
    const bool solve = k < ny && !(i == nr - 1 && dir(v, F_RMAX)) &&
                       !(i == 0 && dir(v, F_RMIN)) &&
                       !(k == ny - 1 && dir(v, F_YMAX)) &&
                       !(k == 0 && dir(v, F_YMIN));
    const int a = sg * kSegV;
    const int m = min(kSegV, nv - a);
    const FT F = ftab(v, p);
    const double* T = F.V + kFV * a;
    double* __restrict__ col = v.D + static_cast<size_t>(p) * v.N +
                               (static_cast<size_t>(i) * nv + a) * ny + (k < ny ? k : 0);
    double x[kSegV];
    double loc = 0.0;
    bool ok = true;
    int bad = 0;
    if (solve) {
#pragma unroll
        for (int r = 0; r < kSegV; ++r) x[r] = r < m ? col[static_cast<size_t>(r) * ny] : 0.0;
        // local forward scan: dp_j = RP_j x_j + B_j dp_{j-1}, zero carry-in
#pragma unroll
        for (int r = 0; r < kSegV; ++r) {
            if (r < m) {
                const double rp = T[kFV * r + FV_RP];
                if (isnan(rp) && ok) {
                    ok = false;
                    bad = a + r;
                }
                loc = fma(T[kFV * r + FV_B], loc, rp * x[r]);
                x[r] = loc;
            }
        }
        car[sg * 32 + tx] = loc;  // local dp at the segment's last row
    }
    __syncthreads();
    if (sg == 0 && solve) {  // carries: true dp at row a-1 of every segment
        double c = 0.0;
        for (int t = 0; t < S; ++t) {
            const double endv = car[t * 32 + tx];
            const int last = min(nv, (t + 1) * kSegV) - 1;
            car[t * 32 + tx] = c;
            c = fma(F.V[kFV * last + FV_BF], c, endv);
        }
    }
    __syncthreads();
    double xb = 0.0;
    if (solve) {
        const double cin = car[sg * 32 + tx];
        // true dp, then the local backward scan x_j = dp_j + E_j x_{j+1}, zero carry-in
#pragma unroll
        for (int r = 0; r < kSegV; ++r)
            if (r < m) x[r] = fma(T[kFV * r + FV_BF], cin, x[r]);
#pragma unroll
        for (int r = kSegV - 1; r >= 0; --r) {
            if (r < m) {
                xb = fma(T[kFV * r + FV_E], xb, x[r]);
                x[r] = xb;
            }
        }
        car[S * 32 + sg * 32 + tx] = xb;  // local x at the segment's first row
    }
    __syncthreads();
    if (sg == 0 && solve) {  // carries: true x at row a+m of every segment, from the top
        double c = 0.0;
        for (int t = S - 1; t >= 0; --t) {
            const double firstv = car[S * 32 + t * 32 + tx];
            car[S * 32 + t * 32 + tx] = c;
            c = fma(F.V[kFV * (t * kSegV) + FV_BB], c, firstv);
        }
    }
    __syncthreads();
    if (!solve) return;
    if (!ok) record_pivot(st, s, 1, i * ny + k, bad);
    const double cout = car[S * 32 + sg * 32 + tx];
#pragma unroll
    for (int r = 0; r < kSegV; ++r)
        if (r < m) col[static_cast<size_t>(r) * ny] = fma(T[kFV * r + FV_BB], cout, x[r]);
}

// ============================================================ y-lines + update
// LY lanes per y-line (contiguous rows, kSegY per lane), 32/LY lines per warp.
// Each lane eliminates its rows; the reduced system of the line is solved
// redundantly by every lane of the line from shuffled end-row data (no block
// barrier); then each lane finishes its rows and applies U += dU, the Dirichlet
// re-imposition, max|dU| and the guard (solver.cpp:151-176).
template <int LY>
__global__ void __launch_bounds__(256, 2) k_fx_y(BatchView v, int s) {
    __shared__ double rs[8][32][8];  // per warp, per lane: segment end rows / reduced solution
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int LPW = 32 / LY;  // lines per warp
    const int sy = lane % LY;
    const int base = lane - sy;   // first lane of this line
    const int line = (blockIdx.x * 8 + wid) * LPW + lane / LY;
    const int lines = nr * nv;
    const bool live = line < lines;
    const int i = live ? line / nv : 0;
    const int j = live ? line - i * nv : 0;
    const int a = sy * kSegY;
    const int m = live ? max(0, min(kSegY, ny - a)) : 0;
    const ProblemConst& pc = v.pc[p];
    const size_t off = static_cast<size_t>(p) * v.N;
    const size_t lb = off + static_cast<size_t>(live ? line : 0) * ny + a;
    // is_dirichlet(i,j,1) (solver.cpp:156)
    const bool solve = live && ny > 1 && !(i == nr - 1 && dir(v, F_RMAX)) &&
                       !(i == 0 && dir(v, F_RMIN)) &&
                       !(j == nv - 1 && dir(v, F_VMAX)) &&
                       !(j == 0 && dir(v, F_VMIN));
    double x[kSegY], cs[kSegY], al[kSegY];
#pragma unroll
    for (int r = 0; r < kSegY; ++r) x[r] = r < m ? v.D[lb + r] : 0.0;
    const FT F = ftab(v, p);
    double yF = 0.0, aF = 0.0, bF = 0.0, yL = 0.0, aL = 0.0, bL = 0.0;
    if (solve && m > 0) {
        const double th = pc.theta_dt;
        const double* R = F.R + kFR * i;
        const double h1 = R[FR_A] * F.V[kFV * j + FV_V];
        const double react = R[FR_REACT];
        const double dint = fma(th, react, 1.0);
        const bool yminD = dir(v, F_YMIN);
        const bool ymaxD = dir(v, F_YMAX);
        const double* Y = F.Y;
        // row 0 of the line (assemble_line_y, discretization.cpp:280-289), folded
        double f0d = 1.0, f0u = 0.0;
        if (a == 0 && !yminD) {
            const double g6h = fma(h1, Y[FY_S6], Y[FY_T6]);
            if (v.y_order == 1) {
                f0d = fma(th, fma(2.0, g6h, react), 1.0);
                f0u = -2.0 * th * g6h;
            } else {
                f0d = fma(th, fma(3.0, g6h, react), 1.0);
                f0u = -4.0 * th * g6h;
                const double s20 = th * g6h;
                if (ny > 2) {  // fold against row 1, which is interior (solver.cpp:28-40)
                    const double l1 = th * fma(h1, Y[kFY + FY_S6], Y[kFY + FY_T6]);
                    const double u1 = -l1;
                    if (fabs(u1) > 1e-300) {
                        const double f = s20 / u1;
                        f0d = fma(-f, l1, f0d);
                        f0u = fma(-f, dint, f0u);
                        x[0] = fma(-f, x[1], x[0]);
                    } else {
                        x[0] = fma(-s20, x[2], x[0]);
                    }
                }
            }
        }
        auto row = [&](int r, double& l, double& d, double& u) {
            const int kk = a + r;
            if (kk == 0) {
                l = 0.0;
                d = f0d;
                u = f0u;
            } else if (kk == ny - 1 && ymaxD) {
                l = 0.0;
                d = 1.0;
                u = 0.0;
            } else {
                const double lk = th * fma(h1, Y[kFY * kk + FY_S6], Y[kFY * kk + FY_T6]);
                l = lk;
                d = dint;
                u = -lk;
            }
        };
        int bad_r = 0;
        if (!seg_solve<kSegY>(m, x, cs, al, yF, aF, bF, yL, aL, bL, bad_r, row))
            record_pivot(st, s, 2, line, a + bad_r);
    }
    // reduced system of the line: end rows -> shared memory, lane 0 of the line
    // runs the O(LY) recurrence, every lane then picks its two neighbours
    double left = 0.0, right = 0.0;
    if (LY > 1) {
        double* E = &rs[wid][base][0];
        double* e = E + sy * 8;
        e[0] = yF; e[1] = aF; e[2] = bF; e[3] = yL; e[4] = aL; e[5] = bL;
        __syncwarp();
        if (sy == 0 && solve) {
            int bt = 0;
            if (!reduced_solve(E, LY, 8, bt)) record_pivot(st, s, 2, line, bt * kSegY);
        }
        __syncwarp();
        left = sy > 0 ? E[(sy - 1) * 8 + 6] : 0.0;   // x_last(sy-1)
        right = sy < LY - 1 ? e[7] : 0.0;            // x_first(sy+1)
    }
    // finish rows, then U += dU, Dirichlet values, max|dU|, guard
    const double* step = step_row(v, p, s);
    double* __restrict__ Urow = v.U + lb;
    unsigned long long md = 0ull;
    double b = bL;
#pragma unroll
    for (int r = kSegY - 1; r >= 0; --r) {
        if (r < m) {
            double dq = x[r];
            if (solve) {
                if (r < m - 1) b = -cs[r] * b;
                dq = fma(b, right, fma(al[r], left, x[r]));
            }
            const int kk = a + r;
            double un = Urow[r] + dq;
            const double ad = fabs(dq);
            if (ad > 0.0) {
                const unsigned long long bits =
                    static_cast<unsigned long long>(__double_as_longlong(ad));
                md = bits > md ? bits : md;
            }
            const int face = dface(v, i, j, kk);
            if (face >= 0) un = face_value(pc, step, tables(v, p), face, i, kk);
            Urow[r] = un;
            const unsigned long long flat = static_cast<unsigned long long>(lb - off + r);
            if (!isfinite(un)) {
                atomicMin(&st.nonfinite_first, flat);
                mark_fail(st, s + 1, HJMSV_NONFINITE);
            } else if (fabs(un) > pc.bound) {
                atomicMin(&st.diverge_first, flat);
                mark_fail(st, s + 1, HJMSV_DIVERGED);
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y2 = __shfl_xor_sync(0xffffffffu, md, o);
        md = y2 > md ? y2 : md;
    }
    if (lane == 0 && md) atomicMax(&st.maxdelta_bits, md);
}

template <int LY>
void launch_y(const BatchView& v, int s, cudaStream_t stream) {
    constexpr int lpb = 8 * (32 / LY);
    const int lines = v.nr * v.nv;
    k_fx_y<LY><<<dim3((lines + lpb - 1) / lpb, v.P), 256, 0, stream>>>(v, s);
}

// ============================================================ face values
// Dirichlet values at t_next for the current step, one table per face, filled
// once per step (k_faces) so the hot kernels never evaluate exp():
//   r faces [ny] (at i = nr-1 / 0), y faces [nr] (at k = ny-1 / 0), v faces [nr][ny].
__device__ __forceinline__ int fb_offset(const BatchView& v, int face, int i, int k) {
    const int ny = v.ny, nr = v.nr;
    switch (face) {
        case F_RMAX: return k;
        case F_RMIN: return ny + k;
        case F_YMAX: return 2 * ny + i;
        case F_YMIN: return 2 * ny + nr + i;
        case F_VMAX: return 2 * ny + 2 * nr + i * ny + k;
        default: return 2 * ny + 2 * nr + nr * ny + i * ny + k;
    }
}

__device__ __forceinline__ double fval(const BatchView& v, int p, int face, int i, int k) {
    return __ldg(v.fb + static_cast<size_t>(p) * v.fb_stride + fb_offset(v, face, i, k));
}

__global__ void __launch_bounds__(256) k_faces(BatchView v, int s) {
    const int p = blockIdx.y;
    if (v.st[p].fail_step) return;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= v.fb_stride) return;
    const int nr = v.nr, ny = v.ny;
    int face, i, k;
    if (q < ny) {
        face = F_RMAX; i = nr - 1; k = q;
    } else if (q < 2 * ny) {
        face = F_RMIN; i = 0; k = q - ny;
    } else if (q < 2 * ny + nr) {
        face = F_YMAX; i = q - 2 * ny; k = ny - 1;
    } else if (q < 2 * ny + 2 * nr) {
        face = F_YMIN; i = q - 2 * ny - nr; k = 0;
    } else {
        int t = q - 2 * ny - 2 * nr;
        face = t < nr * ny ? F_VMAX : F_VMIN;
        if (t >= nr * ny) t -= nr * ny;
        i = t / ny;
        k = t - i * ny;
    }
    double val = 0.0;
    if (v.dmask >> face & 1)
        val = face_value(v.pc[p], step_row(v, p, s), tables(v, p), face, i, k);
    v.fb[static_cast<size_t>(p) * v.fb_stride + q] = val;
}

// out-of-line slow paths (take the view by value so the kernels' own copy stays
// in the parameter bank and their loads stay LDG)
__device__ __noinline__ void guard_fail(const BatchView v, int p, int s, unsigned long long flat,
                                        double un) {
    DevStatus& st = v.st[p];
    if (!isfinite(un)) {  // guard_finite (solver.cpp:69-77)
        atomicMin(&st.nonfinite_first, flat);
        mark_fail(st, s + 1, HJMSV_NONFINITE);
    } else {
        atomicMin(&st.diverge_first, flat);
        mark_fail(st, s + 1, HJMSV_DIVERGED);
    }
}

// dU0 at a node of a face plane i, a face row j (generic stencil, one-sided rows)
__device__ __noinline__ double explicit_slow(const BatchView v, int p, int s, int i, int j,
                                             int k) {
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const ProblemConst& pc = v.pc[p];
    const double* step = step_row(v, p, s);
    const int sr = nv * ny;
    const double* u = v.U + static_cast<size_t>(p) * v.N + (static_cast<size_t>(i) * nv + j) * ny + k;
    const int face = dface(v, i, j, k);
    if (face >= 0) return v.apply_only ? 0.0 : fval(v, p, face, i, k) - u[0];
    const FT F = ftab(v, p);
    const double* R = F.R + kFR * i;
    const double* V = F.V + kFV * j;
    const double* Y = F.Y + kFY * k;
    const double vj = V[FV_V];
    const double g1s = R[FR_G1] * vj;
    const double g4h =
        fma(step[ST_C4], R[FR_G4C], fma(R[FR_G4Q], Y[FY_Y], fma(R[FR_G4V], vj, R[FR_G4P])));
    const double g6h = fma(R[FR_A] * vj, Y[FY_S6], Y[FY_T6]);
    const double u0 = u[0];
    double acc = -R[FR_REACT] * u0;
    if (i == 0) {
        const double u1 = u[sr];
        if (v.r_order == 1)
            acc = fma(2.0 * g4h, u1 - u0, acc);
        else
            acc = fma(g4h, fma(4.0, u1, -u[2 * sr]) - 3.0 * u0, acc);
    } else {
        const double up = u[sr], dn = u[-sr];
        acc = fma(g1s, (up + dn) - 2.0 * u0, acc);
        acc = fma(g4h, up - dn, acc);
    }
    if (j == 0) {
        acc = fma(2.0 * V[FV_G5], u[ny] - u0, acc);
    } else {
        const double up = u[ny], dn = u[-ny];
        acc = fma(V[FV_G2], (up + dn) - 2.0 * u0, acc);
        acc = fma(V[FV_G5], up - dn, acc);
    }
    if (k == 0) {
        const double u1 = u[1];
        if (v.y_order == 1)
            acc = fma(2.0 * g6h, u1 - u0, acc);
        else
            acc = fma(g6h, fma(4.0, u1, -u[2]) - 3.0 * u0, acc);
    } else {
        acc = fma(g6h, u[1] - u[-1], acc);
    }
    if (i > 0 && i < nr - 1 && j > 0 && j < nv - 1)
        acc = fma(R[FR_G3] * V[FV_G3], (u[sr + ny] - u[sr - ny]) - (u[ny - sr] - u[-sr - ny]), acc);
    return acc * pc.dt;
}

// ============================================================ shape-specialised
// Instantiated for compile-time (NV, NY) so strides are immediate offsets;
// fast_step dispatches to them for the benchmark shapes and falls back to the
// runtime-shape kernels above otherwise.

// ------------------------------------------------------------ explicit, 2.5D
// Block = 32 k x 8 j; each thread marches TI planes of its column (fully
// unrolled) with a register window of U(i-1..i+1, j-1..j+1, k); k+-1 arrive by
// shuffles. Loads use clamped indices (no branches); the y faces and the
// one-sided y row are selects; face planes (i = 0, nr-1) and face rows
// (j = 0, nv-1) take the out-of-line generic path, uniformly per warp.
template <int NV, int NY, int TI, int MINB>
__global__ void __launch_bounds__(256, MINB) k_ex3(BatchView v, int s) {
    __shared__ double rt[TI][kFR];
    const int p = blockIdx.z;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    const int nr = v.nr;
    const int i0 = blockIdx.y * TI;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) st.maxdelta_bits = 0ull;
    const FT F = ftab(v, p);
    if (tid < TI * kFR) {
        const int ii = min(i0 + tid / kFR, nr - 1);
        rt[tid / kFR][tid % kFR] = F.R[kFR * ii + tid % kFR];
    }
    constexpr int TK = NY / 32 > 0 ? NY / 32 : 1;
    constexpr int SR = NV * NY;
    const int jt = blockIdx.x / TK;
    const int k = (blockIdx.x - jt * TK) * 32 + threadIdx.x;
    const int j = jt * 8 + threadIdx.y;
    const size_t off = static_cast<size_t>(p) * v.N;
    __syncthreads();
    if (j == 0 || j == NV - 1) {  // face rows: generic path (whole warp)
#pragma unroll 1
        for (int t = 0; t < TI; ++t) {
            const int i = i0 + t;
            if (i < nr)
                v.D[off + (static_cast<size_t>(i) * NV + j) * NY + k] = explicit_slow(v, p, s, i, j, k);
        }
        return;
    }
    const double* __restrict__ col = v.U + off + j * NY + k;
    double* __restrict__ dcol = v.D + off + j * NY + k;
    const double* Vt = F.V + kFV * j;
    const double* Yt = F.Y + kFY * k;
    const double vj = Vt[FV_V], g2s = Vt[FV_G2], g5h = Vt[FV_G5], g3v = Vt[FV_G3];
    const double yk = Yt[FY_Y], vs6 = vj * Yt[FY_S6], t6 = Yt[FY_T6];
    const double dtm = v.pc[p].dt;
    const double c4 = step_row(v, p, s)[ST_C4];
    const bool k0 = k == 0, kN = k == NY - 1;
    const bool ymaxF = kN && dir(v, F_YMAX) && !v.apply_only;
    const bool yminF = k0 && dir(v, F_YMIN) && !v.apply_only;
    const bool zeroF = (kN && dir(v, F_YMAX)) || (k0 && dir(v, F_YMIN));
    const bool order2y = v.y_order != 1;
    const double* fby = v.fb + static_cast<size_t>(p) * v.fb_stride + 2 * NY + (kN ? 0 : nr);
    auto load = [&](int ii, double& m, double& c, double& pl) {
        const double* q = col + static_cast<size_t>(min(max(ii, 0), nr - 1)) * SR;
        c = __ldg(q);
        m = __ldg(q - NY);
        pl = __ldg(q + NY);
    };
    double wm0, wm1, wm2, w00, w01, w02;
    load(i0 - 1, wm0, wm1, wm2);
    load(i0, w00, w01, w02);
#pragma unroll
    for (int t = 0; t < TI; ++t) {
        const int i = i0 + t;
        double wp0, wp1, wp2;
        load(i + 1, wp0, wp1, wp2);
        double kl = __shfl_up_sync(0xffffffffu, w01, 1);
        double kr = __shfl_down_sync(0xffffffffu, w01, 1);
        const double* q = col + static_cast<size_t>(min(i, nr - 1)) * SR;
        if (threadIdx.x == 0 && !k0) kl = __ldg(q - 1);
        if (threadIdx.x == 31 && !kN) kr = __ldg(q + 1);
        const double k2 = k0 ? __ldg(q + 2) : 0.0;
        const double fbv = (ymaxF || yminF) ? __ldg(fby + min(i, nr - 1)) : 0.0;
        if (i < nr) {
            double out;
            if (i > 0 && i < nr - 1) {
                const double* R = rt[t];
                const double g4h = fma(c4, R[FR_G4C], fma(R[FR_G4Q], yk, fma(R[FR_G4V], vj, R[FR_G4P])));
                const double u0 = w01;
                double acc = -R[FR_REACT] * u0;
                acc = fma(R[FR_G1] * vj, (wp1 + wm1) - 2.0 * u0, acc);
                acc = fma(g4h, wp1 - wm1, acc);
                acc = fma(g2s, (w02 + w00) - 2.0 * u0, acc);
                acc = fma(g5h, w02 - w00, acc);
                acc = fma(R[FR_G3] * g3v, (wp2 - wp0) - (wm2 - wm0), acc);
                // one-sided y row at k = 0 (discretization.cpp:346-352)
                const double yd = k0 ? (order2y ? fma(4.0, kr, -k2) - 3.0 * u0 : 2.0 * (kr - u0))
                                     : kr - kl;
                acc = fma(fma(R[FR_A], vs6, t6), yd, acc);
                out = acc * dtm;
                out = zeroF ? ((ymaxF || yminF) ? fbv - u0 : 0.0) : out;
            } else {
                out = explicit_slow(v, p, s, i, j, k);
            }
            dcol[static_cast<size_t>(i) * SR] = out;
        }
        wm0 = w00; wm1 = w01; wm2 = w02;
        w00 = wp0; w01 = wp1; w02 = wp2;
    }
}

// ------------------------------------------------------------ explicit, per node
// Thread per node, block = 32 k x 8 j of one plane: latency is hidden by
// occupancy (every load is independent), neighbours come from L1. Face planes
// and face rows (uniform per block / warp) take the generic out-of-line path;
// k edges are selects.
template <int NV, int NY>
__global__ void __launch_bounds__(256) k_ex4(BatchView v, int s) {
    const int p = blockIdx.z, i = blockIdx.y;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    constexpr int TK = NY / 32 > 0 ? NY / 32 : 1;
    constexpr int SR = NV * NY;
    const int jt = blockIdx.x / TK;
    const int k = (blockIdx.x - jt * TK) * 32 + threadIdx.x;
    const int j = jt * 8 + threadIdx.y;
    if (blockIdx.x == 0 && i == 0 && threadIdx.x == 0 && threadIdx.y == 0) st.maxdelta_bits = 0ull;
    const int nr = v.nr;
    const size_t off = static_cast<size_t>(p) * v.N;
    const int q = (i * NV + j) * NY + k;
    if (i == 0 || i == nr - 1 || j == 0 || j == NV - 1) {
        v.D[off + q] = explicit_slow(v, p, s, i, j, k);
        return;
    }
    const double* __restrict__ u = v.U + off + q;
    const double u0 = __ldg(u);
    double kl = __shfl_up_sync(0xffffffffu, u0, 1);
    double kr = __shfl_down_sync(0xffffffffu, u0, 1);
    const bool k0 = k == 0, kN = k == NY - 1;
    if (threadIdx.x == 0 && !k0) kl = __ldg(u - 1);
    if (threadIdx.x == 31 && !kN) kr = __ldg(u + 1);
    const double rp = __ldg(u + SR), rm = __ldg(u - SR);
    const double vp = __ldg(u + NY), vm = __ldg(u - NY);
    const double cross = (__ldg(u + SR + NY) - __ldg(u + SR - NY)) - (__ldg(u - SR + NY) - __ldg(u - SR - NY));
    const FT F = ftab(v, p);
    const double2* R2 = reinterpret_cast<const double2*>(F.R + kFR * i);
    const double2 r01 = __ldg(R2), r23 = __ldg(R2 + 1), r45 = __ldg(R2 + 2), r67 = __ldg(R2 + 3);
    // r01 = (G1, G4C), r23 = (G4P, G4Q), r45 = (G4V, G3), r67 = (REACT, A)
    const double2* V2 = reinterpret_cast<const double2*>(F.V + kFV * j);
    const double2 v01 = __ldg(V2), v23 = __ldg(V2 + 1);  // (V, G2), (G5, G3V)
    const double2* Y2 = reinterpret_cast<const double2*>(F.Y + kFY * k);
    const double2 y01 = __ldg(Y2), y23 = __ldg(Y2 + 1);  // (S6, T6), (Y, pad)
    const double vj = v01.x;
    const double c4 = __ldg(step_row(v, p, s) + ST_C4);
    const double g4h = fma(c4, r01.y, fma(r23.y, y23.x, fma(r45.x, vj, r23.x)));
    const double g6h = fma(r67.y * vj, y01.x, y01.y);
    double acc = -r67.x * u0;
    acc = fma(r01.x * vj, (rp + rm) - 2.0 * u0, acc);
    acc = fma(g4h, rp - rm, acc);
    acc = fma(v01.y, (vp + vm) - 2.0 * u0, acc);
    acc = fma(v23.x, vp - vm, acc);
    acc = fma(r45.y * v23.y, cross, acc);
    double yd = kr - kl;
    if (k0) {  // one-sided y row (discretization.cpp:346-352)
        const double k2 = __ldg(u + 2);
        yd = v.y_order != 1 ? fma(4.0, kr, -k2) - 3.0 * u0 : 2.0 * (kr - u0);
    }
    acc = fma(g6h, yd, acc);
    double out = acc * v.pc[p].dt;
    if ((kN && dir(v, F_YMAX)) || (k0 && dir(v, F_YMIN)))
        out = v.apply_only ? 0.0 : fval(v, p, kN ? F_YMAX : F_YMIN, i, k) - u0;
    v.D[off + q] = out;
}

// ------------------------------------------------------------ y-lines + update
// NY/MY lanes per line (MY contiguous rows per lane, 128-bit loads/stores).
template <int NV, int NY, int MY>
__global__ void __launch_bounds__(256, 2) k_y3(BatchView v, int s) {
    constexpr int kSegY = MY;
    constexpr int LY = NY / kSegY;
    constexpr int LPW = 32 / LY;
    __shared__ double rs[8][32][8];
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    const int nr = v.nr;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int sy = lane % LY;
    const int base = lane - sy;
    const int line = (blockIdx.x * 8 + wid) * LPW + lane / LY;
    const bool live = line < nr * NV;
    const int lc = live ? line : 0;
    const int i = lc / NV, j = lc - (lc / NV) * NV;
    const size_t off = static_cast<size_t>(p) * v.N;
    const size_t lb = off + static_cast<size_t>(lc) * NY + sy * kSegY;
    double x[kSegY], cs[kSegY], al[kSegY];
    {
        const double2* d2 = reinterpret_cast<const double2*>(v.D + lb);
#pragma unroll
        for (int q = 0; q < kSegY / 2; ++q) {
            const double2 t = __ldg(d2 + q);
            x[2 * q] = t.x;
            x[2 * q + 1] = t.y;
        }
    }
    const bool dI = (i == nr - 1 && dir(v, F_RMAX)) || (i == 0 && dir(v, F_RMIN));
    const bool dJ = (j == NV - 1 && dir(v, F_VMAX)) || (j == 0 && dir(v, F_VMIN));
    const bool solve = live && !dI && !dJ;  // !is_dirichlet(i,j,1) (solver.cpp:156)
    const bool yminD = dir(v, F_YMIN), ymaxD = dir(v, F_YMAX);
    double yF = 0.0, aF = 0.0, bF = 0.0, yL = 0.0, aL = 0.0, bL = 0.0;
    if (solve) {
        const ProblemConst& pc = v.pc[p];
        const FT F = ftab(v, p);
        const double th = pc.theta_dt;
        const double h1 = F.R[kFR * i + FR_A] * F.V[kFV * j + FV_V];
        const double react = F.R[kFR * i + FR_REACT];
        const double dint = fma(th, react, 1.0);
        double lr[kSegY];
        double g60 = 0.0;
#pragma unroll
        for (int r = 0; r < kSegY; ++r) {
            const double2 st6 = __ldg(reinterpret_cast<const double2*>(F.Y + kFY * (sy * kSegY + r)));
            const double g6h = fma(h1, st6.x, st6.y);
            if (r == 0) g60 = g6h;
            lr[r] = th * g6h;
        }
        double f0d = dint, f0u = -lr[0];
        if (sy == 0) {  // row 0 of the line (discretization.cpp:274-289), folded (solver.cpp:28-40)
            f0d = 1.0;
            f0u = 0.0;
            if (!yminD) {
                if (v.y_order == 1) {
                    f0d = fma(th, fma(2.0, g60, react), 1.0);
                    f0u = -2.0 * lr[0];
                } else {
                    f0d = fma(th, fma(3.0, g60, react), 1.0);
                    f0u = -4.0 * lr[0];
                    const double s20 = lr[0];
                    const double l1 = lr[1], u1 = -lr[1];
                    if (fabs(u1) > 1e-300) {
                        const double f = s20 / u1;
                        f0d = fma(-f, l1, f0d);
                        f0u = fma(-f, dint, f0u);
                        x[0] = fma(-f, x[1], x[0]);
                    } else {
                        x[0] = fma(-s20, x[2], x[0]);
                    }
                }
            }
        }
        const bool lastI = sy == LY - 1 && ymaxD;
        auto row = [&](int r, double& l, double& d, double& u) {
            if (r == 0 && sy == 0) {
                l = 0.0;
                d = f0d;
                u = f0u;
            } else if (r == kSegY - 1 && lastI) {
                l = 0.0;
                d = 1.0;
                u = 0.0;
            } else {
                l = lr[r];
                d = dint;
                u = -lr[r];
            }
        };
        int bad_r = 0;
        if (!seg_solve<kSegY>(kSegY, x, cs, al, yF, aF, bF, yL, aL, bL, bad_r, row))
            record_pivot(st, s, 2, line, sy * kSegY + bad_r);
    }
    double left = 0.0, right = 0.0;
    if (LY > 1) {
        double* E = &rs[wid][base][0];
        double* e = E + sy * 8;
        e[0] = yF; e[1] = aF; e[2] = bF; e[3] = yL; e[4] = aL; e[5] = bL;
        __syncwarp();
        if (sy == 0 && solve) {
            int bt = 0;
            if (!reduced_solve(E, LY, 8, bt)) record_pivot(st, s, 2, line, bt * kSegY);
        }
        __syncwarp();
        left = sy > 0 ? E[(sy - 1) * 8 + 6] : 0.0;
        right = sy < LY - 1 ? e[7] : 0.0;
    }
    // x_r, then U += dU, Dirichlet values, max|dU|, guard (solver.cpp:163-176)
    double md = 0.0;
    if (live) {
        double2* u2 = reinterpret_cast<double2*>(v.U + lb);
        double un[kSegY];
#pragma unroll
        for (int q = 0; q < kSegY / 2; ++q) {
            const double2 t = u2[q];
            un[2 * q] = t.x;
            un[2 * q + 1] = t.y;
        }
        double b = bL;
#pragma unroll
        for (int r = kSegY - 1; r >= 0; --r) {
            double dq = x[r];
            if (solve) {
                if (r < kSegY - 1) b = -cs[r] * b;
                dq = fma(b, right, fma(al[r], left, x[r]));
            }
            un[r] += dq;
            md = fmax(md, fabs(dq));
        }
        if (!solve) {
#pragma unroll
            for (int r = 0; r < kSegY; ++r) {
                const int kk = sy * kSegY + r;
                un[r] = fval(v, p, dface(v, i, j, kk), i, kk);
            }
        } else {
            const double* fby = v.fb + static_cast<size_t>(p) * v.fb_stride + 2 * NY;
            if (sy == 0 && yminD) un[0] = __ldg(fby + nr + i);
            if (sy == LY - 1 && ymaxD) un[kSegY - 1] = __ldg(fby + i);
        }
        const double bound = v.pc[p].bound;
#pragma unroll
        for (int r = 0; r < kSegY; ++r)
            if (!(fabs(un[r]) <= bound)) guard_fail(v, p, s, lb - off + r, un[r]);
#pragma unroll
        for (int q = 0; q < kSegY / 2; ++q) u2[q] = make_double2(un[2 * q], un[2 * q + 1]);
    }
    for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
    if (lane == 0 && md > 0.0)
        atomicMax(&st.maxdelta_bits, static_cast<unsigned long long>(__double_as_longlong(md)));
}

}  // namespace

// (nv, ny) pairs with compile-time kernels: nv == ny in {32, 64, 128, 256}
int specialised_shape(const BatchView& v) {
    if (v.nv != v.ny) return 0;
    return (v.ny == 32 || v.ny == 64 || v.ny == 128 || v.ny == 256) ? v.ny : 0;
}

bool fast_supported(int nr, int nv, int ny) {
    // collapsed axes are served by STRICT; segment counts bounded by the block shapes
    return nr >= 3 && nv >= 3 && ny >= 3 && (nr + kSegR - 1) / kSegR <= 32 &&
           (nv + kSegV - 1) / kSegV <= 16 && ny <= 32 * kSegY;
}

int fast_stride(int nr, int nv, int ny) { return fast_table_stride(nr, nv, ny); }

void fast_prepare(const BatchView& v, cudaStream_t) { (void)v; }

void fast_step(const BatchView& v, int s, cudaStream_t stream, long long* launches,
               const LaunchHook* hook) {
    auto mark = [&](int idx, const char* name, double bytes) {
        if (launches) ++*launches;
        if (hook && hook->after) hook->after(hook->ctx, idx, name, bytes);
    };
    // algorithmic bytes per node of each launch (SURVEY §8d accounting): read U,
    // write dU0 | read + write the line | read + write the line | read dU, read U, write U
    const int tk = (v.ny + 31) / 32, tj = (v.nv + 7) / 8;
    const int shape = specialised_shape(v);
    k_faces<<<dim3((v.fb_stride + 255) / 256, v.P), 256, 0, stream>>>(v, s);
    mark(4, "fx_faces", 0.0);
    constexpr int TI = 8;
    const dim3 gex(tk * tj, (v.nr + TI - 1) / TI, v.P);
    static const int exv = [] {
        const char* e = std::getenv("HJMSV_EX_MINB");
        return e ? std::atoi(e) : 0;
    }();
#define HJ_EX(NVV, MB) k_ex3<NVV, NVV, TI, MB><<<gex, dim3(32, 8), 0, stream>>>(v, s)
#define HJ_EXS(NVV)                   \
    if (exv == 0) k_ex4<NVV, NVV><<<dim3(tk * tj, v.nr, v.P), dim3(32, 8), 0, stream>>>(v, s); \
    else if (exv >= 4) HJ_EX(NVV, 4);       \
    else if (exv == 3) HJ_EX(NVV, 3);  \
    else HJ_EX(NVV, 2)
    switch (shape) {
        case 32: HJ_EXS(32); break;
        case 64: HJ_EXS(64); break;
        case 128: HJ_EXS(128); break;
        case 256: HJ_EXS(256); break;
        default: k_fx_explicit<<<dim3(tk * tj, v.nr, v.P), dim3(32, 8), 0, stream>>>(v, s);
    }
#undef HJ_EXS
#undef HJ_EX
    mark(0, "fx_explicit", 16.0);
    const int Sr = (v.nr + kSegR - 1) / kSegR;
    const int tkr = (v.ny + kLanesR - 1) / kLanesR;
    k_fx_r<kSegR><<<dim3(v.nv * tkr, v.P), dim3(kLanesR, Sr),
                    static_cast<size_t>(kLanesR) * Sr * 8 * sizeof(double), stream>>>(v, s);
    mark(1, "fx_sweep_r", 16.0);
    const int Sv = (v.nv + kSegV - 1) / kSegV;
    k_fx_v<<<dim3(v.nr * tk, v.P), dim3(32, Sv), 2ull * Sv * 32 * sizeof(double), stream>>>(v, s);
    mark(2, "fx_sweep_v", 16.0);
    const int ly = (v.ny + kSegY - 1) / kSegY;
    const int lines = v.nr * v.nv;
    static const int ymy = [] {
        const char* e = std::getenv("HJMSV_Y_ROWS");
        return e ? std::atoi(e) : 16;
    }();
    if (shape == 32) {
        if (ymy == 8) k_y3<32, 32, 8><<<dim3((lines + 63) / 64, v.P), 256, 0, stream>>>(v, s);
        else k_y3<32, 32, 16><<<dim3((lines + 127) / 128, v.P), 256, 0, stream>>>(v, s);
    } else if (shape == 64) {
        if (ymy == 8) k_y3<64, 64, 8><<<dim3((lines + 31) / 32, v.P), 256, 0, stream>>>(v, s);
        else k_y3<64, 64, 16><<<dim3((lines + 63) / 64, v.P), 256, 0, stream>>>(v, s);
    } else if (shape == 128) {
        if (ymy == 8) k_y3<128, 128, 8><<<dim3((lines + 15) / 16, v.P), 256, 0, stream>>>(v, s);
        else k_y3<128, 128, 16><<<dim3((lines + 31) / 32, v.P), 256, 0, stream>>>(v, s);
    } else if (shape == 256) {
        if (ymy == 8) k_y3<256, 256, 8><<<dim3((lines + 7) / 8, v.P), 256, 0, stream>>>(v, s);
        else k_y3<256, 256, 16><<<dim3((lines + 15) / 16, v.P), 256, 0, stream>>>(v, s);
    } else if (ly <= 1)
        launch_y<1>(v, s, stream);
    else if (ly <= 2)
        launch_y<2>(v, s, stream);
    else if (ly <= 4)
        launch_y<4>(v, s, stream);
    else if (ly <= 8)
        launch_y<8>(v, s, stream);
    else if (ly <= 16)
        launch_y<16>(v, s, stream);
    else
        launch_y<32>(v, s, stream);
    mark(3, "fx_sweep_y_update", 24.0);
}

void fast_explicit(const BatchView& v, int s, cudaStream_t stream) {
    const int tk = (v.ny + 31) / 32, tj = (v.nv + 7) / 8;
    k_fx_explicit<<<dim3(tk * tj, v.nr, v.P), dim3(32, 8), 0, stream>>>(v, s);
}

}  // namespace hjmsv_b200
