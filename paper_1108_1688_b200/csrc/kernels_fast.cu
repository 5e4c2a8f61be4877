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
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <type_traits>

#include <cooperative_groups.h>

#include "kernels_common.cuh"

namespace hjmsv_b200 {
namespace {
namespace cg = cooperative_groups;
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
__device__ __forceinline__ FT ftab(const BatchView& v, int p, int s) {
    const double* t = v.fast + static_cast<size_t>(p) * v.fast_stride + static_cast<size_t>(s) * v.fast_step;
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
    tl_begin(v, s, 0);
    const int p = blockIdx.z, i = blockIdx.y;
    DevStatus& st = v.st[p];
    if (failed_before(st, s)) return;
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
    const FT F = ftab(v, p, s);
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
            out = v.apply_only ? 0.0 : face_value(pc, step, tables(v, p, s), face, i, k) - u[0];
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
            if (nv == 1) {
                // a collapsed v axis has no v terms (apply_operator, discretization.cpp:336)
            } else if (j == 0) {
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
    tl_end_thread(v, s, 0);
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
    unsigned badm = 0u;  // rows with |pivot| < 1e-300 (solver.cpp:44-52); the first one is reported
#pragma unroll
    for (int r = 0; r < M; ++r) {
        if (r < m) {
            double l, d, u;
            row(r, l, d, u);
            const double P = r == 0 ? d : fma(d, pm1, -(l * uprev) * pm2);
            const double rp = pm1 * frcp(P);
            badm |= (fabs(rp) > 1e300 ? 1u : 0u) << r;
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
    if (badm) bad_r = __ffs(badm) - 1;
    return badm == 0u;
}

// ---- tensor memory (TMEM) as register-file extension for a thread's per-row
// values (tcgen05.st / tcgen05.ld of 32-bit columns in the warp's lane quarter;
// TMEM is otherwise idle in this FP64 path): pass A keeps the modified
// super-diagonal c' and the left spike alpha of its 16 rows there, so the march
// runs without register spills at 16 warps per SM (HJMSV_PA_TM=0: registers).
__device__ __forceinline__ void tm_st_d(unsigned taddr, double v) {
    const unsigned lo = static_cast<unsigned>(__double2loint(v)), hi = static_cast<unsigned>(__double2hiint(v));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(lo), "r"(hi) : "memory");
}
// four doubles (8 columns) starting at taddr
__device__ __forceinline__ void tm_ld_d4(unsigned taddr, double (&v)[4]) {
    unsigned w[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = __hiloint2double(static_cast<int>(w[2 * q + 1]), static_cast<int>(w[2 * q]));
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// two 4-double loads under one wait::ld
__device__ __forceinline__ void tm_ld_d4x2(unsigned ta, double (&va)[4], unsigned tb, double (&vb)[4]) {
    unsigned w[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "r"(ta)
                 : "memory");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]),
                   "=r"(w[15])
                 : "r"(tb)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        va[q] = __hiloint2double(static_cast<int>(w[2 * q + 1]), static_cast<int>(w[2 * q]));
        vb[q] = __hiloint2double(static_cast<int>(w[8 + 2 * q + 1]), static_cast<int>(w[8 + 2 * q]));
    }
}

// seg_solve with both c' (columns taddr + 2r) and the left spike alpha (columns
// taddr + 2M + 2r) in TMEM; only the right-hand side / y stays in registers
template <int M, class RowFn>
__device__ __forceinline__ bool seg_solve_tm2(double (&x)[M], unsigned taddr, double& yF, double& aF,
                                              double& bF, double& yL, double& aL, double& bL, int& bad_r,
                                              RowFn row) {
    double pm1 = 1.0, pm2 = 0.0, uprev = 0.0, yprev = 0.0, aprev = 0.0;
    unsigned badm = 0u;
#pragma unroll
    for (int r = 0; r < M; ++r) {
        double l, d, u;
        row(r, l, d, u);
        const double P = r == 0 ? d : fma(d, pm1, -(l * uprev) * pm2);
        const double rp = pm1 * frcp(P);
        badm |= (fabs(rp) > 1e300 ? 1u : 0u) << r;
        const bool last = r == M - 1;
        const double lrp = l * rp;
        const double yy = r == 0 ? x[r] * rp : fma(-lrp, yprev, x[r] * rp);
        const double aa = r == 0 ? -lrp : -lrp * aprev;
        if (last) {
            yL = yy;
            aL = aa;
            bL = -u * rp;
        } else {
            tm_st_d(taddr + 2 * r, u * rp);
            tm_st_d(taddr + 2 * M + 2 * r, aa);
        }
        x[r] = yy;
        yprev = yy;
        aprev = aa;
        uprev = u;
        pm2 = pm1;
        pm1 = P;
        if (r % 8 == 7) {
            const int e = ((__double2hiint(pm1) >> 20) & 0x7ff) - 1023;
            const double sc = __hiloint2double((1023 - e) << 20, 0);
            pm1 *= sc;
            pm2 *= sc;
        }
    }
    tm_wait_st();
    double yn = yL, an = aL, bn = bL;
#pragma unroll
    for (int c0 = M - 4; c0 >= 0; c0 -= 4) {
        double c[4], a4[4];
        tm_ld_d4x2(taddr + 2 * c0, c, taddr + 2 * M + 2 * c0, a4);
#pragma unroll
        for (int q = 3; q >= 0; --q) {
            const int r = c0 + q;
            if (r < M - 1) {
                yn = fma(-c[q], yn, x[r]);
                an = fma(-c[q], an, a4[q]);
                bn = -c[q] * bn;
                x[r] = yn;
                tm_st_d(taddr + 2 * M + 2 * r, an);
            }
        }
    }
    tm_st_d(taddr + 2 * M + 2 * (M - 1), aL);  // alpha of the last row
    tm_wait_st();
    yF = yn;
    aF = an;
    bF = bn;
    if (badm) bad_r = __ffs(badm) - 1;
    return badm == 0u;
}

// The segment solve of seg_solve by a twisted factorisation: rows 0..K-1 are
// eliminated from the top (LU) and rows M-1..K+1 from the bottom (UL) at the
// same time, and the two sweeps meet at row K = M/2, so each thread runs two
// independent chains of M/2 rows instead of one of M (the same three arrays:
// the top half keeps (c', y', alpha'), the bottom half (e', y'', beta'')).
// The right-hand side -l_0 e_0 (alpha) only enters the top sweep and
// -u_{M-1} e_{M-1} (beta) only the bottom one; pivots are continuant ratios in
// both directions (P_r = d_r P_{r-1} - l_r u_{r-1} P_{r-2} from the top,
// Q_r = d_r Q_{r+1} - u_r l_{r+1} Q_{r+2} from the bottom). On exit x[] = y,
// al[] = alpha, cs[] = beta (the right spike; callers use it directly) and the
// end-row values are set. Only the elimination order differs from seg_solve.
template <int M, class RowFn>
__device__ __forceinline__ bool seg_solve_tw(double (&x)[M], double (&cs)[M], double (&al)[M],
                                             double& yF, double& aF, double& bF, double& yL,
                                             double& aL, double& bL, int& bad_r, RowFn row) {
    static_assert(M >= 4 && M % 2 == 0, "twisted segment");
    constexpr int K = M / 2;
    unsigned badm = 0u;
    // top sweep, rows 0..K-1: cs = c' = u/piv, x = y', al = alpha'
    // bottom sweep, rows M-1..K+1: cs = e' = l/piv', x = y'', al = beta''
    double pm1 = 1.0, pm2 = 0.0, uprev = 0.0, yprev = 0.0, aprev = 0.0;
    double qm1 = 1.0, qm2 = 0.0, lnext = 0.0, ynext = 0.0, bnext = 0.0;
    double lK = 0.0, dK = 1.0, uK = 0.0;
#pragma unroll
    for (int h = 0; h < K; ++h) {
        {  // top row r = h
            const int r = h;
            double l, d, u;
            row(r, l, d, u);
            const double P = r == 0 ? d : fma(d, pm1, -(l * uprev) * pm2);
            const double rp = pm1 * frcp(P);  // 1/piv_r
            badm |= (fabs(rp) > 1e300 ? 1u : 0u) << r;
            const double lrp = l * rp;
            cs[r] = u * rp;
            x[r] = r == 0 ? x[r] * rp : fma(-lrp, yprev, x[r] * rp);
            al[r] = r == 0 ? -lrp : -lrp * aprev;
            yprev = x[r];
            aprev = al[r];
            uprev = u;
            pm2 = pm1;
            pm1 = P;
            if (r % 8 == 7) {
                const int e = ((__double2hiint(pm1) >> 20) & 0x7ff) - 1023;
                const double sc = __hiloint2double((1023 - e) << 20, 0);
                pm1 *= sc;
                pm2 *= sc;
            }
        }
        if (M - 1 - h > K) {  // bottom row r = M-1-h
            const int r = M - 1 - h;
            double l, d, u;
            row(r, l, d, u);
            const double Q = h == 0 ? d : fma(d, qm1, -(u * lnext) * qm2);
            const double rq = qm1 * frcp(Q);  // 1/piv'_r
            badm |= (fabs(rq) > 1e300 ? 1u : 0u) << r;
            const double urq = u * rq;
            cs[r] = l * rq;
            x[r] = h == 0 ? x[r] * rq : fma(-urq, ynext, x[r] * rq);
            al[r] = h == 0 ? -urq : -urq * bnext;
            ynext = x[r];
            bnext = al[r];
            lnext = l;
            qm2 = qm1;
            qm1 = Q;
            if (h % 8 == 7) {
                const int e = ((__double2hiint(qm1) >> 20) & 0x7ff) - 1023;
                const double sc = __hiloint2double((1023 - e) << 20, 0);
                qm1 *= sc;
                qm2 *= sc;
            }
        }
    }
    row(K, lK, dK, uK);
    // middle row K: both sweeps meet
    const double cK1 = cs[K - 1], eK1 = cs[K + 1];
    const double piv = fma(-lK, cK1, fma(-uK, eK1, dK));
    const double rk = frcp(piv);
    badm |= (fabs(rk) > 1e300 ? 1u : 0u) << K;
    const double yK = fma(-lK, x[K - 1], fma(-uK, x[K + 1], x[K])) * rk;
    const double aK = -lK * al[K - 1] * rk;
    const double bK = -uK * al[K + 1] * rk;
    x[K] = yK;
    al[K] = aK;
    cs[K] = bK;
    // outward back-substitution: upward rows K-1..0 and downward rows K+1..M-1
    double yu = yK, au = aK, bu = bK, yd = yK, ad = aK, bd = bK;
#pragma unroll
    for (int h = 1; h <= K; ++h) {
        {
            const int r = K - h;  // x_r = y'_r - c'_r x_{r+1}
            const double c = cs[r];
            yu = fma(-c, yu, x[r]);
            au = fma(-c, au, al[r]);
            bu = -c * bu;
            x[r] = yu;
            al[r] = au;
            cs[r] = bu;
        }
        if (K + h < M) {
            const int r = K + h;  // x_r = y''_r - e'_r x_{r-1}
            const double e = cs[r];
            yd = fma(-e, yd, x[r]);
            bd = fma(-e, bd, al[r]);
            ad = -e * ad;
            x[r] = yd;
            al[r] = ad;
            cs[r] = bd;
        }
    }
    yF = x[0];
    aF = al[0];
    bF = cs[0];
    yL = x[M - 1];
    aL = al[M - 1];
    bL = cs[M - 1];
    bad_r = badm ? __ffs(badm) - 1 : 0;
    return badm == 0u;
}

// Reduced system of a line with S segments, unknowns p_t = x_last(t) and
// q_t = x_first(t+1), t = 0..S-2:
//   p_t = yL_t + aL_t p_{t-1} + bL_t q_t,   q_t = yF_{t+1} + aF_{t+1} p_t + bF_{t+1} q_{t+1}
// Forward: q_t = Qc_t + Qd_t q_{t+1}, p_t = Pp_t + Pq_t q_{t+1}; backward from
// q_{S-1} = 0. Segment t's data at E[t*stride + f] (f: yF aF bF yL aL bL); the
// results p_t, q_t overwrite fields 6, 7.
__device__ __forceinline__ bool reduced_solve(double* E, int S, int stride, int& bad_t, int fs = 1) {
    // element (t, f) at E[t*stride + f*fs]
    double Pp = 0.0, Pq = 0.0;
    bool ok = true;
#pragma unroll 1
    for (int t = 0; t < S - 1; ++t) {
        double* e0 = E + t * stride;
        const double* e1 = e0 + stride;
        const double A = fma(e0[4 * fs], Pp, e0[3 * fs]);
        const double B = fma(e0[4 * fs], Pq, e0[5 * fs]);
        const double den = fma(-e1[1 * fs], B, 1.0);
        if (fabs(den) < 1e-300 && ok) {
            ok = false;
            bad_t = t + 1;
        }
        const double inv = frcp(den);
        const double Qc = fma(e1[1 * fs], A, e1[0]) * inv;
        const double Qd = e1[2 * fs] * inv;
        Pp = fma(B, Qc, A);
        Pq = B * Qd;
        e0[6 * fs] = Qc;
        e0[7 * fs] = Qd;
        e0[3 * fs] = Pp;
        e0[4 * fs] = Pq;
    }
    double qn = 0.0;
#pragma unroll 1
    for (int t = S - 2; t >= 0; --t) {
        double* e0 = E + t * stride;
        const double qs = fma(e0[7 * fs], qn, e0[6 * fs]);
        e0[6 * fs] = fma(e0[4 * fs], qn, e0[3 * fs]);  // p_t
        e0[7 * fs] = qs;                               // q_t
        qn = qs;
    }
    return ok;
}

// The same reduced system solved from both ends at once ("burn at both ends"):
// lanes with back == false run the forward recurrence over pairs 0..mF-1, their
// partner lanes (shfl_xor by `partner`) run the identical recurrence on the
// reversed system over pairs S-2 .. mF. Reversal maps segment s to S-1-s and
// swaps the roles of the end rows: first-row fields (yF, aF, bF) become
// (yL, bL, aL) and vice versa, so both halves execute the same instructions.
// The halves meet in a 2x2 solve at pair mF; each then back-substitutes its own
// pairs into fields 6, 7 (p_t, q_t) in the original orientation.
__device__ __forceinline__ bool reduced_solve_2way(double* E, int S, int stride, int fs, bool back,
                                                   unsigned mask, int partner, int& bad_t) {
    const int np = S - 1;
    const int mF = (np + 1) >> 1, mB = np - mF;
    const int fy0 = back ? 0 : 3, fa0 = back ? 2 : 4, fb0 = back ? 1 : 5;  // end row of s0
    const int fy1 = back ? 3 : 0, fa1 = back ? 5 : 1, fb1 = back ? 4 : 2;  // first row of s1
    const int sp = back ? 0 : 3, sq = back ? 2 : 4;                        // scratch Pp, Pq
    double Pp = 0.0, Pq = 0.0;
    bool ok = true;
#pragma unroll 1
    for (int k = 0; k < mF; ++k) {
        if (k < (back ? mB : mF)) {
            double* e0 = E + (back ? S - 1 - k : k) * stride;
            const double* e1 = E + (back ? S - 2 - k : k + 1) * stride;
            const double A = fma(e0[fa0 * fs], Pp, e0[fy0 * fs]);
            const double B = fma(e0[fa0 * fs], Pq, e0[fb0 * fs]);
            const double den = fma(-e1[fa1 * fs], B, 1.0);
            if (fabs(den) < 1e-300 && ok) {
                ok = false;
                bad_t = back ? S - 2 - k : k + 1;
            }
            const double inv = frcp(den);
            const double Qc = fma(e1[fa1 * fs], A, e1[fy1 * fs]) * inv;
            const double Qd = e1[fb1 * fs] * inv;
            Pp = fma(B, Qc, A);
            Pq = B * Qd;
            e0[6 * fs] = Qc;
            e0[7 * fs] = Qd;
            e0[sp * fs] = Pp;
            e0[sq * fs] = Pq;
        }
    }
    // meet: p_{mF-1} = PpF + PqF q_mF (forward), q_mF = PpB + PqB p_{mF-1} (backward)
    const double oPp = __shfl_xor_sync(mask, Pp, partner);
    const double oPq = __shfl_xor_sync(mask, Pq, partner);
    const double PpF = back ? oPp : Pp, PqF = back ? oPq : Pq;
    const double PpB = back ? Pp : oPp, PqB = back ? Pq : oPq;
    const double pm = (PpF + PqF * PpB) / (1.0 - PqF * PqB);
    const double qm = fma(PqB, pm, PpB);
    double qn = back ? pm : qm;
    const int n = back ? mB : mF;
#pragma unroll 1
    for (int k = n - 1; k >= 0; --k) {
        double* e0 = E + (back ? S - 1 - k : k) * stride;
        const double qs = fma(e0[7 * fs], qn, e0[6 * fs]);
        const double ps = fma(e0[sq * fs], qn, e0[sp * fs]);
        if (back) {  // reversed pair k is original pair t = S-2-k: p_t = qs, q_t = ps
            double* et = E + (S - 2 - k) * stride;
            et[6 * fs] = qs;
            et[7 * fs] = ps;
        } else {
            e0[6 * fs] = ps;
            e0[7 * fs] = qs;
        }
        qn = qs;
    }
    return ok;
}

// The reduced system of one line solved by L lanes at once (lane t = segment
// t; lanes t >= S pad), i.e. reduced_solve's recurrences as lane scans. With
// unprimed fields from segment t's last row and primed ones from segment t+1's
// first row, Pq alone obeys a Moebius recurrence,
//   Pq_t = bF' B_t / den_t,  B_t = aL Pq_{t-1} + bL,  den_t = 1 - aF' B_t,
// i.e. (Pq, 1) -> N_t (Pq, 1) projectively with N_t = [[bF' aL, bF' bL], [-aF' aL, 1 - aF' bL]],
// so an inclusive scan of 2x2 products (log2 L shuffle steps, each product
// rescaled by an exact power of two) gives every lane Pq_{t-1}; then, with
// r = 1/den_t,
//   Pp_t = r aL Pp_{t-1} + r (yL + yF' B_t)
// is an affine recurrence (a scan of (alpha, beta) pairs), and the
// back-substitution q_t = Qc_t + Qd_t q_{t+1} a suffix scan of affine maps.
// Returns left = p_{t-1} = x_{a-1} and right = q_t = x_{a+m} of segment t, and
// the pair index + 1 of a vanishing reduced pivot (0 if none) of this lane.
// Every lane of the warp must call it (full-warp shuffles of width L).
template <int L>
__device__ __forceinline__ int reduced_scan(double yF, double aF, double bF, double yL, double aL,
                                             double bL, int t, int S, double& left, double& right) {
    constexpr unsigned FULL = 0xffffffffu;
    const double nyF = __shfl_down_sync(FULL, yF, 1, L);
    const double naF = __shfl_down_sync(FULL, aF, 1, L);
    const double nbF = __shfl_down_sync(FULL, bF, 1, L);
    const bool pair = t < S - 1;  // pair t couples segments t and t+1
    double n11 = 1.0, n12 = 0.0, n21 = 0.0, n22 = 1.0;
    if (pair) {
        n11 = nbF * aL;
        n12 = nbF * bL;
        n21 = -naF * aL;
        n22 = fma(-naF, bL, 1.0);
    }
#pragma unroll
    for (int off = 1; off < L; off <<= 1) {  // N_t ... N_0
        const double q11 = __shfl_up_sync(FULL, n11, off, L);
        const double q12 = __shfl_up_sync(FULL, n12, off, L);
        const double q21 = __shfl_up_sync(FULL, n21, off, L);
        const double q22 = __shfl_up_sync(FULL, n22, off, L);
        {  // selects instead of a branch: the levels schedule as one block
            const double d11 = fma(n11, q11, n12 * q21);
            const double d12 = fma(n11, q12, n12 * q22);
            const double d21 = fma(n21, q11, n22 * q21);
            const double d22 = fma(n21, q12, n22 * q22);
            const int ex = (__double2hiint(d22) >> 20) & 0x7ff;
            const double sc = (ex != 0 && ex != 0x7ff) ? __hiloint2double((2046 - ex) << 20, 0) : 1.0;
            const bool on = t >= off;
            n11 = on ? d11 * sc : n11;
            n12 = on ? d12 * sc : n12;
            n21 = on ? d21 * sc : n21;
            n22 = on ? d22 * sc : n22;
        }
    }
    // Pq_{t-1} = n/d of the product up to pair t-1 (applied to (0, 1))
    const double pn = __shfl_up_sync(FULL, n12, 1, L);
    const double pd = __shfl_up_sync(FULL, n22, 1, L);
    const double Pq0 = t == 0 ? 0.0 : pn * frcp(pd);
    const double B = fma(aL, Pq0, bL);
    const double den = fma(-naF, B, 1.0);
    const double r = frcp(den);
    const int bad = (pair && fabs(den) < 1e-300) ? t + 1 : 0;
    const double Pq = pair ? B * (nbF * r) : 0.0;
    const double Qd = pair ? nbF * r : 0.0;
    // Pp_t = al Pp_{t-1} + be: inclusive affine scan
    double al = pair ? r * aL : 1.0, be = pair ? r * fma(nyF, B, yL) : 0.0;
#pragma unroll
    for (int off = 1; off < L; off <<= 1) {
        const double pa = __shfl_up_sync(FULL, al, off, L);
        const double pb = __shfl_up_sync(FULL, be, off, L);
        {
            const bool on = t >= off;
            be = on ? fma(al, pb, be) : be;
            al = on ? al * pa : al;
        }
    }
    double Pp0 = __shfl_up_sync(FULL, be, 1, L);  // Pp_{t-1}
    if (t == 0) Pp0 = 0.0;
    const double A = fma(aL, Pp0, yL);
    double c = pair ? fma(naF, A, nyF) * r : 0.0;  // Qc
    double g = Qd;
    const double Pp = pair ? be : 0.0;
#pragma unroll
    for (int off = 1; off < L; off <<= 1) {  // q_t = Qc_t + Qd_t q_{t+1}, q_{S-1} = 0
        const double c2 = __shfl_down_sync(FULL, c, off, L);
        const double g2 = __shfl_down_sync(FULL, g, off, L);
        {
            const bool on = t + off < L;
            c = on ? fma(g, c2, c) : c;
            g = on ? g * g2 : g;
        }
    }
    double qn = __shfl_down_sync(FULL, c, 1, L);
    if (t + 1 >= L) qn = 0.0;
    const double pt = fma(Pq, qn, Pp);  // p_t (pairs only)
    right = c;
    left = __shfl_up_sync(FULL, pt, 1, L);
    return bad;
}

// ============================================================ batched lines (stage test)
// Lines solved by the FAST partition method exactly as pass A's r-lines (and,
// with TW, pass B's y-lines) solve theirs: one warp per line, lane t owns rows
// 16t..16t+15 (rows past n are identity rows), the super2 fold of
// thomas_solve_inplace (solver.cpp:28-40, its lag branch included) applied to
// row 0 first, the segment solve (seg_solve / seg_solve_tw), the reduced
// system by the lane scan (reduced_scan), then x = y + alpha left + beta right.
// fail_row: -1, or a row of the first segment (or reduced pair) whose pivot
// vanished (|piv| < 1e-300; the partition pivots stand in for Thomas's).
template <bool TW>
__global__ void __launch_bounds__(128) k_thomas_fast(int n, int count, const double* __restrict__ lower,
                                                     const double* __restrict__ diag,
                                                     const double* __restrict__ upper,
                                                     const double* __restrict__ super2, double* rhs,
                                                     int* fail_row) {
    constexpr int M = 16;
    const int line = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (line >= count) return;  // warp-uniform
    const int t = threadIdx.x & 31;
    const int S = (n + M - 1) / M;
    const size_t o = static_cast<size_t>(line) * n;
    const int a = t * M;
    double x[M], cs[M], al[M];
#pragma unroll
    for (int r = 0; r < M; ++r) x[r] = a + r < n ? rhs[o + a + r] : 0.0;
    double f0d = 1.0, f0u = 0.0;
    if (t == 0) {
        f0d = diag[o];
        f0u = n > 1 ? upper[o] : 0.0;
        const double s2 = super2[line];
        if (s2 != 0.0 && n > 2) {
            if (fabs(upper[o + 1]) > 1e-300) {
                const double f = s2 / upper[o + 1];
                f0d = fma(-f, lower[o + 1], f0d);
                f0u = fma(-f, diag[o + 1], f0u);
                x[0] = fma(-f, x[1], x[0]);
            } else {  // vanishing coupling: lag the (0,2) term on the iterate
                x[0] = fma(-s2, x[2], x[0]);
            }
        }
    }
    auto row = [&](int r, double& l, double& d, double& u) {
        const int i = a + r;
        if (i >= n) {
            l = 0.0; d = 1.0; u = 0.0;
        } else if (i == 0) {
            l = 0.0; d = f0d; u = i == n - 1 ? 0.0 : f0u;
        } else {
            l = lower[o + i];
            d = diag[o + i];
            u = i == n - 1 ? 0.0 : upper[o + i];
        }
    };
    double yF = 0.0, aF = 0.0, bF = 0.0, yL = 0.0, aL = 0.0, bL = 0.0;
    int bad_r = 0;
    bool ok;
    if constexpr (TW) ok = seg_solve_tw<M>(x, cs, al, yF, aF, bF, yL, aL, bL, bad_r, row);
    else ok = seg_solve<M>(M, x, cs, al, yF, aF, bF, yL, aL, bL, bad_r, row);
    double lf = 0.0, rg = 0.0;
    const int bt = reduced_scan<32>(yF, aF, bF, yL, aL, bL, t, S, lf, rg);
    const double left = t > 0 && t < S ? lf : 0.0;
    const double right = t < S - 1 ? rg : 0.0;
    double b = bL;
#pragma unroll
    for (int r = M - 1; r >= 0; --r) {
        if constexpr (TW) b = cs[r];
        else if (r < M - 1) b = -cs[r] * b;
        if (a + r < n) rhs[o + a + r] = fma(b, right, fma(al[r], left, x[r]));
    }
    unsigned key = 0xffffffffu;
    if (t < S && !ok) key = static_cast<unsigned>(a + bad_r);
    if (t < S && bt) key = min(key, static_cast<unsigned>(bt * M));
    key = __reduce_min_sync(0xffffffffu, key);
    if (t == 0) fail_row[line] = key == 0xffffffffu ? -1 : static_cast<int>(key);
}

// ============================================================ r-lines
// Block = kLanesR consecutive k (same j) x S segments of M rows.
template <int M>
__global__ void __launch_bounds__(512) k_fx_r(BatchView v, int s) {
    tl_begin(v, s, 1);
    extern __shared__ double red[];  // [kLanesR][S][8]
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (failed_before(st, s)) return;
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
        const FT F = ftab(v, p, s);
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
    tl_end_thread(v, s, 1);
}

// ============================================================ v-lines
// The LU of the v-line is a table (depends on j only), so both substitutions
// are affine scans: a block of 32 k x S segments (kSegV rows) computes local
// scans, carries the segment boundary values across segments in shared memory,
// and fixes its rows up with the in-segment products BF/BB.
__global__ void __launch_bounds__(512, 2) k_fx_v(BatchView v, int s) {
    tl_begin(v, s, 2);
    extern __shared__ double car[];  // [2][S][32]
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (failed_before(st, s)) return;
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
    const FT F = ftab(v, p, s);
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
    tl_end_thread(v, s, 2);
}

// ============================================================ y-lines + update
// LY lanes per y-line (contiguous rows, kSegY per lane), 32/LY lines per warp.
// Each lane eliminates its rows; the reduced system of the line is solved
// redundantly by every lane of the line from shuffled end-row data (no block
// barrier); then each lane finishes its rows and applies U += dU, the Dirichlet
// re-imposition, max|dU| and the guard (solver.cpp:151-176).
template <int LY>
__global__ void __launch_bounds__(256, 2) k_fx_y(BatchView v, int s) {
    tl_begin(v, s, 3);
    __shared__ double rs[8][32][8];  // per warp, per lane: segment end rows / reduced solution
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (failed_before(st, s)) return;
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
    const FT F = ftab(v, p, s);
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
            if (face >= 0) un = face_value(pc, step, tables(v, p, s), face, i, kk);
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
    tl_end_thread(v, s, 3);
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

// entry q of the face buffer of step s (layout as fb_offset)
__device__ __forceinline__ double face_entry(const BatchView& v, int p, int s, int q) {
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
    if (!(v.dmask >> face & 1)) return 0.0;
    return face_value(v.pc[p], step_row(v, p, s), tables(v, p, s), face, i, k);
}

__global__ void __launch_bounds__(256) k_faces(BatchView v, int s) {
    tl_begin(v, s, 4);
    const int p = blockIdx.y;
    if (failed_before(v.st[p], s)) return;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= v.fb_stride) return;
    v.fb[static_cast<size_t>(p) * v.fb_stride + q] = face_entry(v, p, s, q);
    tl_end_thread(v, s, 4);
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

// guard_finite over the M values of a segment (solver.cpp:69-77): one integer
// max over the high words of |u| decides for all of them; only a segment with
// a value at or above the bound's high word (or Inf/NaN) runs the exact test
template <int M>
__device__ __forceinline__ void guard_seg(const BatchView& v, int p, int s, unsigned long long flat0,
                                          const double (&un)[M], double bound) {
    unsigned hm = 0u;
#pragma unroll
    for (int r = 0; r < M; ++r) hm = max(hm, static_cast<unsigned>(__double2hiint(un[r])) & 0x7fffffffu);
    if (hm >= static_cast<unsigned>(__double2hiint(bound))) {
#pragma unroll
        for (int r = 0; r < M; ++r)
            if (!(fabs(un[r]) <= bound)) guard_fail(v, p, s, flat0 + r, un[r]);
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
    const FT F = ftab(v, p, s);
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

// ------------------------------------------------------------ explicit, per node
// Thread per node, block = 32 k x 8 j of one plane: latency is hidden by
// occupancy (every load is independent), neighbours come from L1. Face planes
// and face rows (uniform per block / warp) take the generic out-of-line path;
// k edges are selects.
template <int NV, int NY>
__global__ void __launch_bounds__(256) k_ex4(BatchView v, int s) {
    tl_begin(v, s, 0);
    const int p = blockIdx.z, i = blockIdx.y;
    DevStatus& st = v.st[p];
    if (failed_before(st, s)) return;
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
    const FT F = ftab(v, p, s);
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
    tl_end_thread(v, s, 0);
}

// ------------------------------------------------------------ y-lines + update
// NY/MY lanes per line (MY contiguous rows per lane, 128-bit loads/stores).
template <int NV, int NY, int MY>
__global__ void __launch_bounds__(256, 2) k_y3(BatchView v, int s) {
    tl_begin(v, s, 3);
    constexpr int kSegY = MY;
    constexpr int LY = NY / kSegY;
    constexpr int LPW = 32 / LY;
    constexpr int TS = 8 * LPW + 1;                 // padded per-segment stride
    __shared__ double rsp[8][LY * TS + 1];           // per warp: [segment][field][line]
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (failed_before(st, s)) return;
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
        const FT F = ftab(v, p, s);
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
    } else {  // a line that is not solved keeps dU: zero spikes and couplings
#pragma unroll
        for (int r = 0; r < kSegY; ++r) cs[r] = al[r] = 0.0;
    }
    double left = 0.0, right = 0.0;
    if constexpr (LY >= 8) {  // the line's LY lanes solve its reduced system by a lane scan
        double lf, rg;
        const int bt = reduced_scan<LY>(yF, aF, bF, yL, aL, bL, sy, LY, lf, rg);
        const unsigned bm = __ballot_sync(0xffffffffu, solve && bt != 0);
        if (solve) {
            const int g0 = lane & ~(LY - 1);
            const unsigned lm = (bm >> g0) & ((LY < 32) ? ((1u << LY) - 1u) : 0xffffffffu);
            if (lm && sy == __ffs(lm) - 1) record_pivot(st, s, 2, line, bt * kSegY);
            if (sy > 0) left = lf;
            if (sy < LY - 1) right = rg;
        }
    } else if (LY > 1) {
        double* ew = &rsp[wid][lane / LY];
        double* e = ew + sy * TS;
        e[0] = yF; e[LPW] = aF; e[2 * LPW] = bF; e[3 * LPW] = yL; e[4 * LPW] = aL; e[5 * LPW] = bL;
        __syncwarp();
        if (sy == 0 && solve) {
            int bt = 0;
            if (!reduced_solve(ew, LY, TS, bt, LPW)) record_pivot(st, s, 2, line, bt * kSegY);
        }
        __syncwarp();
        left = (solve && sy > 0) ? e[-TS + 6 * LPW] : 0.0;
        right = (solve && sy < LY - 1) ? e[7 * LPW] : 0.0;
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
        double b = bL;  // 0 on lines that are not solved, as are cs, al, left, right
#pragma unroll
        for (int r = kSegY - 1; r >= 0; --r) {
            if (r < kSegY - 1) b = -cs[r] * b;
            const double dq = fma(b, right, fma(al[r], left, x[r]));
            un[r] += dq;
            x[r] = dq;
        }
        if (v.want_md) {
#pragma unroll
            for (int r = 0; r < kSegY; ++r) md = fmax(md, fabs(x[r]));
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
        guard_seg<kSegY>(v, p, s, lb - off, un, bound);
#pragma unroll
        for (int q = 0; q < kSegY / 2; ++q) u2[q] = make_double2(un[2 * q], un[2 * q + 1]);
    }
    for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
    if (lane == 0 && md > 0.0)
        atomicMax(&st.maxdelta_bits, static_cast<unsigned long long>(__double_as_longlong(md)));
    tl_end_thread(v, s, 3);
}

// ------------------------------------------------------------ pass A, fused
// Explicit operator + r-lines in one kernel. Block = 16 consecutive k (same j)
// x S segments of 16 rows i; each thread marches its segment with a register
// window of U at (i-1..i+1) x (j-1..j+1) fed by a per-thread cp.async ring
// (kRing rows ahead), k+-1 by shuffles inside the 16-lane group. It computes
// dU0 = dt F(U) (apply_operator, discretization.cpp:302-364; Dirichlet
// increments solver.cpp:111-116) for the row and feeds it straight into the
// segment elimination of I - th L_r (assemble_line_r, discretization.cpp:194-230;
// Thomas solver.cpp:22-57 by the partition method). Dirichlet v-face rows
// (block-uniform) take a load-store-only path (dU1 = dU0 = face - U); the
// degenerate v_min row runs the same fused march in its own instantiation.
// Columns on y Dirichlet faces (not solved, solver.cpp:127) run identity rows,
// so dU1 = dU0 there.
constexpr int kRing = 3;

__device__ __forceinline__ void cp_async8s(unsigned dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
// one-shot bulk (TMA engine) copies of contiguous tables into shared memory,
// completion tracked by an mbarrier (phase 0)
__device__ __forceinline__ void bulk_init(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, unsigned bar) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_wait(unsigned bar) {
    asm volatile("{\n .reg .pred P;\nWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n"
                 " @!P bra WAIT_%=;\n}" ::"r"(bar) : "memory");
}
// remote (cluster) stores that complete on the destination CTA's mbarrier: the
// consumer waits on its own barrier, no cluster-wide barrier or fence
__device__ __forceinline__ unsigned map_cluster(unsigned saddr, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_d2(unsigned raddr, double a, double b, unsigned rbar) {
    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                 ::"r"(raddr), "d"(a), "d"(b), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// phase 0 of a barrier that counts st.async bytes from peer CTAs: the completion
// of the transaction makes the stored data visible to the waiting thread, as
// for bulk copies (an acquire at cluster scope would invalidate all of L1:
// CCTL.IVALL, 6 % of pass B's stall samples when it was tried)
__device__ __forceinline__ void mbar_wait_cluster(unsigned bar) {
    asm volatile("{\n .reg .pred P;\nWAITC_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n"
                 " @!P bra WAITC_%=;\n}" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// TM: 0 or 2; SEG: rows per r-segment (16, or 32 with the arrays in TMEM)
template <int NV, int NY, bool SCAN, int KL = 16, int TPC = 1, bool PAD = false, int TM = 0, int SEG = 16>
__global__ void __launch_bounds__(512) k_pa(BatchView v, int s) {
    // launched as a programmatic dependent of the previous kernel: everything
    // below reads what it wrote (no-op without a programmatic dependency)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    tl_begin(v, s, 0);
    constexpr int M = SEG;
    // FOLD (the 32-row variant: 512-row lines): the (step, j) part of a row's
    // coefficients folded into the CTA's r-table. Config 3 pass A 265 -> 261 us;
    // on shorter lines the per-CTA table pass costs more than it saves (config 1
    // +7 %, configs 2 / 4 +6-8 %)
    constexpr bool FOLD = SEG == 32;
    static_assert(SEG == 16 || (SEG == 32 && TM == 2), "32-row segments keep their arrays in TMEM");
#ifdef HJMSV_BRFREE_ALL
    constexpr bool BRFREE = TM == 2;
#else
    constexpr bool BRFREE = SEG == 32;  // branch-free march rows
#endif
    // PAD: any nv, any ny <= NY and any nr <= 512 (the reference's own meshes):
    // the grid's real sizes are runtime values, k lanes past ny and rows past nr
    // run inert (identity rows, no stores); otherwise NV x NY exactly
    const int nyr = PAD ? v.ny : NY;
    const int nvr = PAD ? v.nv : NV;
    const int SR = PAD ? v.nv * v.ny : NV * NY;  // row stride (one r plane)
    extern __shared__ double sm[];
    const int S = blockDim.y;
    // KL consecutive k per segment group (16: one CTA of 16 S threads per SM on
    // 512-row lines; 8: two co-resident CTAs of 8 S threads — measured slower)
    static_assert(KL == 16 || KL == 8, "k-lane group");
    // TPC column tiles (KL consecutive k of one j) per CTA, marched one after the
    // other: the next tile's window and ring rows are queued (cp.async into the
    // thread's staging slots) as soon as a tile's march ends, so their latency
    // hides behind that tile's reduced systems and writes; per-CTA setup (tables,
    // r-table bulk copy) is paid once per TPC tiles
    static_assert(TPC == 1 || TPC == 2, "tiles per CTA");
    constexpr bool STAGE = TPC > 1;
    constexpr int RST = kRing * 4 + (STAGE ? 12 : 0) + 1;  // per-thread ring (+ window staging) stride
    const int nt = KL * S;
    double* red = sm;                          // [KL][8S+9] reduced-system rows
    double* ring = red + KL * (8 * S + 9);     // [nt][RST] window prefetch (padded)
    double* rt = ring + RST * nt;              // [nr][8] r-table (FastR)
    double* fy = rt + v.nr * kFR;              // [2][nr] y-face values (YMAX, YMIN)
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    const bool fail = !v.dbg && failed_before(st, s);  // checked after the prologue loads are in flight
    const int nr = v.nr;
    const int tx = threadIdx.x, sg = threadIdx.y;
    const int tid = sg * KL + tx;
    constexpr int TK = NY / KL;
    static_assert(TK % TPC == 0, "the tiles of a CTA share j");
    const int j = (blockIdx.x * TPC) / TK;
    const int kt0 = blockIdx.x * TPC - j * TK;  // first k tile of this CTA
    const ProblemConst& pc = v.pc[p];
    const bool yminD = dir(v, F_YMIN), ymaxD = dir(v, F_YMAX);
    // this KL-lane group of the warp (blockDim.x == KL)
    const unsigned hmask = (KL == 16 ? 0xffffu : 0xffu) << ((sg & (32 / KL - 1)) * KL);
    const int a = sg * M;
    const size_t off = static_cast<size_t>(p) * v.N;
    const FT F = ftab(v, p, s);
    // r-table and y-face values into shared memory by two bulk copies, overlapped
    // with the window prologue below
    __shared__ alignas(8) unsigned long long tbar;
    const unsigned tbar_s = static_cast<unsigned>(__cvta_generic_to_shared(&tbar));
    // TM 2: 64 TMEM columns per warp (its 15 c' and 16 alpha values) in the warp's lane quarter
    __shared__ unsigned tm_base_s;
    // ceil(warps / 4) slots per lane quarter x 4M columns, a
    // power of two >= 32: the co-resident CTAs of an SM fit its 512 columns
    // (16-warp CTAs: 256 columns, one per SM; 8-warp CTAs: 128, two per SM; 4-warp: 64, four)
    const unsigned tm_slots = (static_cast<unsigned>(blockDim.x * blockDim.y) / 32u + 3u) / 4u;
    const unsigned tm_need = tm_slots * (4u * M);
    const unsigned TM_COLS = tm_need <= 32u ? 32u : tm_need <= 64u ? 64u : tm_need <= 128u ? 128u
                             : tm_need <= 256u ? 256u : 512u;
    const int warp = tid >> 5;
    if constexpr (TM) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             static_cast<unsigned>(__cvta_generic_to_shared(&tm_base_s))),
                         "r"(TM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    if (tid == 0) {
        const unsigned rbytes = nr * kFR * sizeof(double), ybytes = 2 * nr * sizeof(double);
        bulk_init(tbar_s, rbytes + ybytes);
        bulk_copy(rt, F.R, rbytes, tbar_s);
        bulk_copy(fy, v.fb + static_cast<size_t>(p) * v.fb_stride + 2 * nyr, ybytes, tbar_s);
    }
    const double c4 = __ldg(step_row(v, p, s) + ST_C4);
    const double2* V2 = reinterpret_cast<const double2*>(F.V + kFV * j);
    double2 v01 = __ldg(V2);
    const double2 v23 = __ldg(V2 + 1);  // (V, G2), (G5, G3V)
    const double vj = v01.x;
    const double th = pc.theta_dt, dtm = pc.dt;
    const bool rmaxD = dir(v, F_RMAX), rminD = dir(v, F_RMIN);
    // v-face rows (block-uniform): j = nv-1 is the v_max Dirichlet face (an early,
    // load-store-only path); j = 0 is Dirichlet (same path) or the degenerate
    // one-sided row (below)
    const bool vminD = dir(v, F_VMIN), vmaxD = dir(v, F_VMAX);
    const bool jlo = j == 0, jhi = j == nvr - 1;
    const bool jdir = (jhi && vmaxD) || (jlo && vminD);
    // the degenerate j = 0 row uses the interior stencil with its missing j-1
    // column replaced by j+1 and G2 replaced by G5: that is exactly the
    // one-sided 2 g5 (u_{j+1} - u_j) term, and the cross term vanishes
    const bool jdeg = jlo && !jdir;
    if (jdeg) v01.y = v23.x;
    // FOLD: the stencil's coefficients carry dt, the line coefficients theta dt / dt
    const double g2c = FOLD ? v01.y * dtm : v01.y, g5c = FOLD ? v23.x * dtm : v23.x;
    const double thc = FOLD ? th / dtm : th;
    const bool order2y = v.y_order != 1, order2r = v.r_order != 1;
    const double* fbp = v.fb + static_cast<size_t>(p) * v.fb_stride;

    // ---- per-tile (k-dependent) state, set by tile_setup(t)
    int k = 0;
    bool klive = true, k0 = false, kN = false, solve = false, kface = false, edge = false;
    int eoff = 0;
    double yk = 0.0, vs6 = 0.0, t6 = 0.0, ths = 0.0, rminv = 0.0, rmaxv = 0.0, e3 = 0.0;
    bool k0o1 = false;
    const double* fyk = fy;
    const double* __restrict__ col = v.U;
    auto tile_k = [&](int t) { return (kt0 + t) * KL + tx; };
    auto tile_setup = [&](int t) {
        k = tile_k(t);
        klive = !PAD || k < nyr;
        if (PAD && !klive) k = nyr - 1;  // inert lane: reads a real column, stores nothing
        k0 = k == 0;
        kN = k == nyr - 1;
        e3 = k0 ? (order2y ? 3.0 : 1.0) : 0.0;
        k0o1 = k0 && !order2y;
        // is_dirichlet(1,j,k) (solver.cpp:127): the column lies on a v or y Dirichlet face
        solve = klive && !(kN && ymaxD) && !(j == nvr - 1 && dir(v, F_VMAX)) && !(k0 && yminD) &&
                !(j == 0 && dir(v, F_VMIN));
        const double2* Y2 = reinterpret_cast<const double2*>(F.Y + kFY * k);
        const double2 y01 = __ldg(Y2), y23 = __ldg(Y2 + 1);  // (S6, T6), (Y, pad)
        yk = y23.x;
        vs6 = FOLD ? y01.x : vj * y01.x;
        t6 = FOLD ? y01.y * dtm : y01.y;
        fyk = fy + (kN ? 0 : nr);
        kface = (kN && ymaxD) || (k0 && yminD);
        // r-face values this thread needs (first / last segment)
        rminv = (sg == 0 && rminD) ? __ldg(fbp + nyr + k) : 0.0;
        rmaxv = ((PAD ? (a <= nr - 1 && nr - 1 < a + M) : a + M == nr) && rmaxD) ? __ldg(fbp + k) : 0.0;
        col = v.U + off + static_cast<size_t>(j) * nyr + k;
        // the KL-lane group's edge lanes also carry their outside neighbour in k
        // (k-1 at tx 0, k+1 at tx KL-1; k+2 at k = 0 for the one-sided row)
        edge = klive && (tx == 0 || (tx == KL - 1 && !kN));
        eoff = tx == 0 ? (k0 ? 2 : -1) : 1;
        // interior rows (0 < i < nr-1); a column that is not solved runs identity rows
        ths = solve ? thc : 0.0;
    };
    tile_setup(0);
    double x[M], cs[M], al[M];
    // window for columns j-1 (0), j (1), j+1 (2): m = row ic-1, c = ic, p = ic+1;
    // rows ic+2 .. ic+1+kRing are in flight in this thread's ring slots (groups 1..kRing)
    // row ic-1 is kept as its centre value m1 and its j+1 - j-1 difference mx (the
    // cross term needs only that), saving two registers in the march
    double mx = 0.0, m1 = 0.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, p0 = 0.0, p1 = 0.0, p2 = 0.0;
    double ce = 0.0, pe = 0.0;
    auto gptr_c = [&](const double* cb, int ii) { return cb + static_cast<size_t>(min(max(ii, 0), nr - 1)) * SR; };
    auto gptr = [&](int ii) { return gptr_c(col, ii); };
    // this thread's ring slots (odd stride between threads, compile-time offsets
    // inside); STAGE: 12 more slots hold the next tile's window rows
    double* const myring = ring + tid * RST;
    const unsigned myring_s = static_cast<unsigned>(__cvta_generic_to_shared(myring));
    auto slot = [&](int q, int c) { return myring + q * 4 + c; };
    auto wslot = [&](int q, int c) { return myring + kRing * 4 + q * 4 + c; };
    // the j-1 column offset is a compile-time constant in each instantiation
    auto ring_rows = [&](auto jd, const double* cb, bool ed, int eo) {
        const int OFFM = decltype(jd)::value ? nyr : -nyr;
#pragma unroll
        for (int r = 0; r < kRing; ++r) {
            const double* g = gptr_c(cb, a + 2 + r);
            cp_async8s(myring_s + 8 * (r * 4 + 0), g + OFFM);
            cp_async8s(myring_s + 8 * (r * 4 + 1), g);
            cp_async8s(myring_s + 8 * (r * 4 + 2), g + nyr);
            if (ed) cp_async8s(myring_s + 8 * (r * 4 + 3), g + eo);
            cp_async_commit();
        }
    };
    auto prologue = [&](auto jd) {
        const int OFFM = decltype(jd)::value ? nyr : -nyr;
        const double* q = gptr(a - 1);
        m1 = __ldg(q);
        mx = __ldg(q + nyr) - __ldg(q + OFFM);
        q = gptr(a);
        c0 = __ldg(q + OFFM); c1 = __ldg(q); c2 = __ldg(q + nyr);
        if (edge) ce = __ldg(q + eoff);
        q = gptr(a + 1);
        p0 = __ldg(q + OFFM); p1 = __ldg(q); p2 = __ldg(q + nyr);
        if (edge) pe = __ldg(q + eoff);
        ring_rows(jd, col, edge, eoff);
    };
    // STAGE: the window rows a-1, a, a+1 of the tile at cb as one cp.async group
    // into the staging slots, then its ring rows (kRing groups)
    auto prologue_staged = [&](auto jd, const double* cb, bool ed, int eo) {
        const int OFFM = decltype(jd)::value ? nyr : -nyr;
        const unsigned ws = myring_s + 8 * (kRing * 4);
#pragma unroll
        for (int w = 0; w < 3; ++w) {
            const double* g = gptr_c(cb, a - 1 + w);
            cp_async8s(ws + 8 * (w * 4 + 0), g + OFFM);
            cp_async8s(ws + 8 * (w * 4 + 1), g);
            cp_async8s(ws + 8 * (w * 4 + 2), g + nyr);
            if (w > 0 && ed) cp_async8s(ws + 8 * (w * 4 + 3), g + eo);
        }
        cp_async_commit();
        ring_rows(jd, cb, ed, eo);
    };
    auto window_from_stage = [&] {
        cp_async_wait<kRing>();  // the staging group (the ring groups may be in flight)
        m1 = *wslot(0, 1);
        mx = *wslot(0, 2) - *wslot(0, 0);
        c0 = *wslot(1, 0); c1 = *wslot(1, 1); c2 = *wslot(1, 2);
        if (edge) ce = *wslot(1, 3);
        p0 = *wslot(2, 0); p1 = *wslot(2, 1); p2 = *wslot(2, 2);
        if (edge) pe = *wslot(2, 3);
    };
    if (!jdir) {
        if constexpr (STAGE) {
            if (jdeg) prologue_staged(std::true_type{}, col, edge, eoff);
            else prologue_staged(std::false_type{}, col, edge, eoff);
        } else {
            if (jdeg) prologue(std::true_type{});
            else prologue(std::false_type{});
        }
    }
    if constexpr (TM) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // the mbarrier is initialised
    if constexpr (TM) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned taddr = TM ? tm_base_s + ((static_cast<unsigned>(warp & 3) * 32u) << 16) +
                                   static_cast<unsigned>(warp >> 2) * (4u * M)
                              : 0u;
    auto tm_free = [&] {
        if constexpr (TM) {
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (warp == 0)
                asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base_s), "r"(TM_COLS)
                             : "memory");
        }
    };
    bulk_wait(tbar_s);  // rt, fy have landed
    // FOLD: everything of a row's coefficients that depends on (step, j) only is
    // folded into this CTA's copy of the r-table, scaled by dt:
    //   (G1 v_j dt, (c4 G4C + G4V v_j + G4P) dt | G4Q dt, G3 G3V_j dt | REACT dt, A v_j dt)
    // so a march row reads three 128-bit pairs and builds g4 with one FMA
    if constexpr (FOLD) {
        if (!jdir) {
            for (int i = tid; i < nr; i += nt) {
                double* R = rt + kFR * i;
                const double g1 = R[FR_G1], g4c = R[FR_G4C], g4p = R[FR_G4P], g4q = R[FR_G4Q], g4v = R[FR_G4V],
                             g3 = R[FR_G3], re = R[FR_REACT], aa = R[FR_A];
                R[0] = g1 * vj * dtm;
                R[1] = fma(c4, g4c, fma(g4v, vj, g4p)) * dtm;
                R[2] = g4q * dtm;
                R[3] = g3 * v23.y * dtm;
                R[4] = re * dtm;
                R[5] = aa * vj * dtm;
            }
        }
        __syncthreads();
    }
    if (fail) {  // the problem failed in an earlier step (block-uniform)
        cp_async_wait<0>();
        tm_free();
        return;
    }
    if (blockIdx.x == 0 && tid == 0) st.maxdelta_bits = 0ull;
    if (jdir) {
        // a Dirichlet v face: every column is an identity line, dU1 = dU0 =
        // face(t_next) - U (solver.cpp:111-116, 127), with the face precedence
        // r_max > y_max > v_max > r_min > y_min > v_min (discretization.cpp:153-192)
#pragma unroll 1
        for (int t = 0; t < TPC; ++t) {
            if (t > 0) tile_setup(t);
            const double* fv = fbp + 2 * nyr + 2 * nr + (jhi ? 0 : nr * nyr) + k;
            double* dcol = v.D + off + static_cast<size_t>(j) * nyr + k;
#pragma unroll 4
            for (int r = 0; r < M; ++r) {
                const int i = a + r;
                if (PAD && (i >= nr || !klive)) break;
                const double u0 = __ldg(col + static_cast<size_t>(i) * SR);
                double f = __ldg(fv + static_cast<size_t>(i) * nyr);
                if (!jhi) {  // v_min ranks last
                    if (i == 0 && rminD) f = rminv;
                    if (k0 && yminD) f = fyk[i];
                }
                if (kN && ymaxD) f = fyk[i];
                if (i == nr - 1 && rmaxD) f = rmaxv;
                dcol[static_cast<size_t>(i) * SR] = f - u0;
            }
        }
        tm_free();
        tl_end(v, s, 0);
        return;
    }

    // row coefficients of I - th L_r at row i (g4h shared with the stencil)
    auto coeffs = [&](int i, double g1s, double g4h, double& l, double& d, double& u, double& s2) {
        l = 0.0; d = 1.0; u = 0.0; s2 = 0.0;
        if (!solve || (i == nr - 1 && rmaxD) || (i == 0 && rminD)) return;
        if (i == 0) {
            if (!order2r) {
                d = fma(2.0 * thc, g4h, 1.0);
                u = -2.0 * thc * g4h;
            } else {
                d = fma(3.0 * thc, g4h, 1.0);
                u = -4.0 * thc * g4h;
                s2 = thc * g4h;
            }
        } else {
            const double w2 = thc * g1s, w1 = thc * g4h;
            l = w1 - w2;
            d = fma(2.0, w2, 1.0);
            u = -(w2 + w1);
        }
    };
    auto interior = [&](double g1s, double g4h, double& l, double& d, double& u) {
        const double w2 = ths * g1s, w1 = ths * g4h;
        l = w1 - w2;
        d = fma(2.0, w2, 1.0);
        u = -(w2 + w1);
    };
    auto rtab = [&](int i, double2& r01, double2& r23, double2& r45, double2& r67) {
        const double2* R2 = reinterpret_cast<const double2*>(rt + kFR * i);
        r01 = R2[0]; r23 = R2[1]; r45 = R2[2];
        if constexpr (!FOLD) r67 = R2[3];
        // r01 = (G1, G4C), r23 = (G4P, G4Q), r45 = (G4V, G3), r67 = (REACT, A); FOLD:
        // r01 = (G1 v dt, g4 part dt), r23 = (G4Q dt, G3 G3V dt), r45 = (REACT dt, A v dt)
    };
    auto g4 = [&](const double2& r01, const double2& r23, const double2& r45) {
        if constexpr (FOLD) return fma(r23.x, yk, r01.y);
        else return fma(c4, r01.y, fma(r23.y, yk, fma(r45.x, vj, r23.x)));
    };
    auto g1v = [&](const double2& r01) { return FOLD ? r01.x : r01.x * vj; };
    auto g3c = [&](const double2& r23, const double2& r45) { return FOLD ? r23.y : r45.y * v23.y; };
    auto rea = [&](const double2& r45, const double2& r67) { return FOLD ? r45.x : r67.x; };
    auto aiv = [&](const double2& r45, const double2& r67) { return FOLD ? r45.y : r67.y; };

    const int FS = S + 1, CST = 8 * S + 9;
#pragma unroll 1
    for (int t = 0; t < TPC; ++t) {
        if (t > 0) tile_setup(t);
        if constexpr (STAGE) window_from_stage();
        double yF = 0.0, aF = 0.0, bF = 0.0, yL = 0.0, aL = 0.0, bL = 0.0;
        int bad_r = 0;
        bool ok = true;
        auto march = [&](auto jd) {
            const int OFFM = decltype(jd)::value ? nyr : -nyr;
            // window for columns j-1 (0), j (1), j+1 (2): m = row ic-1, c = ic, p = ic+1;
            // rows ic+2 .. ic+1+kRing are in flight in this thread's ring slots
            // centre moves to row a+r: row a+r+1 comes out of ring slot (r-1) % kRing,
            // which is refilled with row a+r+kRing+1 while that row lies in the
            // segment's window (rows up to a+M); later shifts only drain the ring
            auto shift = [&](int r) {
                const int q = (r - 1) % kRing;
                if (r <= M - kRing) cp_async_wait<kRing - 1>();
                else if (r == M - 2) cp_async_wait<1>();
                else cp_async_wait<0>();
                mx = c2 - c0;
                m1 = c1;
                c0 = p0; c1 = p1; c2 = p2; ce = pe;
                p0 = *slot(q, 0); p1 = *slot(q, 1); p2 = *slot(q, 2);
                if (edge) pe = *slot(q, 3);
                if (r + kRing + 1 <= M) {
                    const double* g = gptr(a + r + kRing + 1);
                    {
                    cp_async8s(myring_s + 8 * (q * 4 + 0), g + OFFM);
                    cp_async8s(myring_s + 8 * (q * 4 + 1), g);
                    cp_async8s(myring_s + 8 * (q * 4 + 2), g + nyr);
                    if (edge) cp_async8s(myring_s + 8 * (q * 4 + 3), g + eoff);
                    }
                    cp_async_commit();
                }
            };
            // y-direction terms and the k faces (discretization.cpp:340-352)
            // full: every lane of the warp is here (rows r >= 1); row 0 runs the
            // face-row code in lane group 0 of warp 0 only, so it shuffles per group
            auto yterm = [&](bool full, double u0, double acc, double a_i, double ed) {
                const unsigned msk = full ? 0xffffffffu : hmask;
                double kl = __shfl_up_sync(msk, u0, 1, KL);
                double kr = __shfl_down_sync(msk, u0, 1, KL);
                double yd;
                if constexpr (BRFREE) {
                    // one-sided y row at k = 0 (discretization.cpp:346-352; ed = U(i, j, 2)) without a
                    // branch: 4 kr - ed - 3 u0 = (kr - ed) + 3 (kr - u0), and 2 (kr - u0) =
                    // (kr - u0) + (kr - u0); e3 = 0 on every other column. The unrolled march
                    // is then one basic block, which the scheduler interleaves across rows
                    // (config 3 pass A 296 -> 274 us; the register-resident variants spill
                    // twice as much that way and keep the branch)
                    if (tx == 0) kl = ed;
                    if (k0o1) kl = u0;
                    if (tx == KL - 1 && !kN) kr = ed;
                    yd = fma(e3, kr - u0, kr - kl);
                } else {
                    if (tx == 0 && !k0) kl = ed;
                    if (tx == KL - 1 && !kN) kr = ed;
                    yd = kr - kl;
                    if (k0)  // one-sided y row (discretization.cpp:346-352); ed = U(i, j, 2)
                        yd = order2y ? fma(4.0, kr, -ed) - 3.0 * u0 : 2.0 * (kr - u0);
                }
                acc = fma(fma(a_i, vs6, t6), yd, acc);
                return FOLD ? acc : acc * dtm;  // y-face Dirichlet columns are fixed up after the march
            };
            // dU0 at an interior row i from a window (mm, cc, pp)
            auto stencil = [&](bool full, const double2& r01, const double2& r23, const double2& r45, const double2& r67,
                               double g4h, double mqx, double mq1, double cq0, double cq1,
                               double cq2, double pq0, double pq1, double pq2, double ed) {
                const double u0 = cq1;
                double acc = -rea(r45, r67) * u0;
                acc = fma(g1v(r01), (pq1 + mq1) - 2.0 * u0, acc);
                acc = fma(g4h, pq1 - mq1, acc);
                acc = fma(g2c, (cq2 + cq0) - 2.0 * u0, acc);
                acc = fma(g5c, cq2 - cq0, acc);
                acc = fma(g3c(r23, r45), (pq2 - pq0) - mqx, acc);
                return yterm(full, u0, acc, aiv(r45, r67), ed);
            };
            auto row = [&](int r, double& l, double& d, double& u) {
                const int i = a + r;
                double2 r01, r23, r45, r67;
                rtab(PAD ? min(i, nr - 1) : i, r01, r23, r45, r67);
                const double g4h = g4(r01, r23, r45);
                if (r == 0) {
                    if (a == 0) {
                        // face plane i = 0 (discretization.cpp:318-329): one-sided g4 term, no cross
                        cp_async_wait<kRing - 1>();  // row 2 (ring slot 0)
                        const double n0 = *slot(0, 0), n1 = *slot(0, 1), n2 = *slot(0, 2);
                        const double u0 = c1;
                        double acc = -rea(r45, r67) * u0;
                        acc = fma(g4h, order2r ? fma(4.0, p1, -n1) - 3.0 * u0 : 2.0 * (p1 - u0), acc);
                        acc = fma(g2c, (c2 + c0) - 2.0 * u0, acc);
                        acc = fma(g5c, c2 - c0, acc);
                        double x0 = yterm(false, u0, acc, aiv(r45, r67), ce);
                        // r_min Dirichlet ranks below r_max / y_max / v_max (discretization.cpp:153-192)
                        if (rminD && !(kN && ymaxD)) x0 = rminv - u0;
                        x[0] = x0;
                        // the super2 fold needs row 1's rhs (solver.cpp:28-40)
                        double2 q01, q23, q45, q67;
                        rtab(1, q01, q23, q45, q67);
                        const double g4h1 = g4(q01, q23, q45);
                        const double x1 = stencil(false, q01, q23, q45, q67, g4h1, c2 - c0, c1, p0, p1, p2, n0, n1, n2, pe);
                        double d0, u0c, s20, l1, d1, u1, t1, l0;
                        coeffs(0, g1v(r01), g4h, l0, d0, u0c, s20);
                        double f0d = d0, f0u = u0c;
                        if (s20 != 0.0) {
                            coeffs(1, g1v(q01), g4h1, l1, d1, u1, t1);
                            if (fabs(u1) > 1e-300) {
                                const double f = s20 / u1;
                                f0d = fma(-f, l1, d0);
                                f0u = fma(-f, d1, u0c);
                                x[0] = fma(-f, x1, x[0]);
                            } else {  // lagged fold: row 2's rhs (rows 1..3 of the window)
                                cp_async_wait<kRing - 2>();
                                double2 w01, w23, w45, w67;
                                rtab(2, w01, w23, w45, w67);
                                const double x2 = stencil(false, w01, w23, w45, w67, g4(w01, w23, w45), p2 - p0, p1, n0,
                                                          n1, n2, *slot(1, 0), *slot(1, 1), *slot(1, 2),
                                                          edge ? *slot(0, 3) : 0.0);
                                x[0] = fma(-s20, x2, x[0]);
                            }
                        }
                        l = 0.0; d = f0d; u = f0u;
                        return;
                    }
                    x[0] = stencil(false, r01, r23, r45, r67, g4h, mx, m1, c0, c1, c2, p0, p1, p2, ce);
                } else {
                    shift(r);
                    const double xv = stencil(true, r01, r23, r45, r67, g4h, mx, m1, c0, c1, c2, p0, p1, p2, ce);
                    // face plane i = nr-1: r_max is always Dirichlet and ranks first
                    // (PAD: rows past nr-1 are inert identity rows)
                    if constexpr (PAD) x[r] = xv;
                    else x[r] = (r == M - 1 && i == nr - 1 && rmaxD) ? rmaxv - c1 : xv;
                }
                if constexpr (PAD) {  // the r_max face row anywhere in the segment; inert rows past it
                    if (i == nr - 1 && rmaxD) x[r] = rmaxv - c1;
                    else if (i >= nr) x[r] = 0.0;
                }
                // rows a+1 .. a+14 are always interior; a+15 may be the r_max face
                if (PAD ? (i >= nr - 1 && (i > nr - 1 || rmaxD)) : (r == M - 1 && i == nr - 1 && rmaxD)) {
                    l = 0.0; d = 1.0; u = 0.0;
                } else {
                    interior(g1v(r01), g4h, l, d, u);
                }
            };
            if constexpr (TM == 2) ok = seg_solve_tm2<M>(x, taddr, yF, aF, bF, yL, aL, bL, bad_r, row);
            else ok = seg_solve<M>(M, x, cs, al, yF, aF, bF, yL, aL, bL, bad_r, row);
            cp_async_wait<0>();
            // STAGE: queue the next tile's window and ring rows now (the ring and
            // the window registers are free), ahead of this tile's reduced systems
            if constexpr (STAGE) {
                if (t + 1 < TPC) {
                    const int kn = tile_k(t + 1);
                    const bool ed = tx == 0 || (tx == KL - 1 && kn != nyr - 1);
                    prologue_staged(jd, v.U + off + static_cast<size_t>(j) * nyr + kn, ed, tx == 0 ? -1 : 1);
                }
            }
        };
        if (jdeg) march(std::true_type{});
        else march(std::false_type{});
        if (!ok) record_pivot(st, s, 0, j * nyr + k, a + bad_r);
        // the next wave's U column -> L2: one 128-byte line per row of this thread's
        // segment, asked for now that this CTA's own window traffic has ended
        // (compiled into the tensor-memory variants only: the register-resident ones
        // of the small planes lose 2 % to the extra code and keep their grids in L2)
        if constexpr (!PAD && TPC == 1 && KL == 16 && TM == 2) {
            if (v.pf_ahead_a && tx == 0) {
                const unsigned nb = blockIdx.x + static_cast<unsigned>(v.pf_ahead_a);
                if (nb < gridDim.x) {
                    const unsigned j2 = nb / TK, kt2 = nb - j2 * TK;
                    const double* c2 = v.U + off + static_cast<size_t>(j2) * NY + kt2 * KL + static_cast<size_t>(a) * SR;
#pragma unroll
                    for (int r = 0; r < M; ++r)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(c2 + static_cast<size_t>(r) * SR));
                }
            }
        }
        // reduced-system rows as [column][field][segment] (field stride S+1, column
        // stride 8S+9: conflict-free for the writers, lanes = k, and for the
        // scans, lanes = segments)
        double* E = red + tx * CST + sg;
        E[0] = yF; E[FS] = aF; E[2 * FS] = bF; E[3 * FS] = yL; E[4 * FS] = aL; E[5 * FS] = bL;
        __syncthreads();
        if (S > 1) {
            if constexpr (SCAN) {
                // every thread solves: column tid / S, segment tid % S (KL S threads)
                const int cc = tid / S, ts = tid - cc * S;
                double* Ec = red + cc * CST + ts;
                const int kk = (kt0 + t) * KL + cc;
                const bool csolve = (!PAD || kk < nyr) && !(kk == nyr - 1 && ymaxD) &&
                                    !(j == nvr - 1 && dir(v, F_VMAX)) && !(kk == 0 && yminD) &&
                                    !(j == 0 && dir(v, F_VMIN));
                const double eyF = Ec[0], eaF = Ec[FS], ebF = Ec[2 * FS], eyL = Ec[3 * FS], eaL = Ec[4 * FS],
                             ebL = Ec[5 * FS];
                double lf = 0.0, rg = 0.0;
                int bad = 0;
                if (S == 16) bad = reduced_scan<16>(eyF, eaF, ebF, eyL, eaL, ebL, ts, S, lf, rg);
                else bad = reduced_scan<32>(eyF, eaF, ebF, eyL, eaL, ebL, ts, S, lf, rg);
                if (v.dbg & 1) lf = rg = 0.0;  // diagnostic: uncoupled segments (wrong results, finite)
                if (csolve && bad) record_pivot(st, s, 0, j * nyr + kk, bad * M);
                Ec[6 * FS] = lf;  // x_{a-1} of segment ts
                Ec[7 * FS] = rg;  // x_{a+m} of segment ts
            } else if (KL == 16 && sg < 2) {  // warp 0: segment rows 0 (forward) and 1 (backward) of every column
                const unsigned mask = __ballot_sync(0xffffffffu, solve);
                if (solve) {
                    int bt = 0;
                    if (!reduced_solve_2way(red + tx * CST, S, 1, FS, sg == 1, mask, 16, bt))
                        record_pivot(st, s, 0, j * nyr + k, bt * M);
                    __syncwarp(mask);
                    // p_t, q_t -> each segment's left (p_{t-1}) / right (q_t), as the scan leaves them
                    if (sg == 0) {
                        for (int ts = S - 1; ts >= 0; --ts) {
                            double* et = red + tx * CST + ts;
                            et[6 * FS] = ts > 0 ? et[-1 + 6 * FS] : 0.0;
                        }
                    }
                }
            }
        }
        __syncthreads();
        const double left = (solve && sg > 0) ? E[6 * FS] : 0.0;        // x_{a-1}
        const double right = (solve && sg < S - 1) ? E[7 * FS] : 0.0;   // x_{a+m}
        if (kface) {
            // y_max / y_min Dirichlet columns (identity rows): dU0 = face(t_next) - U
            // (solver.cpp:111-116) wherever the r faces do not take precedence
            // (discretization.cpp:153-192: r_max > y_max > v_max > r_min > y_min > v_min)
#pragma unroll
            for (int r = 0; r < M; ++r) {
                const int i = a + r;
                if (PAD && i >= nr) break;
                if (!((i == nr - 1 && rmaxD) || (i == 0 && rminD && !(kN && ymaxD))))
                    x[r] = fyk[i] - __ldg(col + static_cast<size_t>(i) * SR);
            }
        }
        double b = bL;
        double* __restrict__ dcol = v.D + off + static_cast<size_t>(j) * nyr + k + static_cast<size_t>(a) * SR;
        if constexpr (TM == 2) {
#pragma unroll
            for (int c0 = M - 4; c0 >= 0; c0 -= 4) {
                double c[4], a4[4];
                tm_ld_d4x2(taddr + 2 * c0, c, taddr + 2 * M + 2 * c0, a4);
#pragma unroll
                for (int q = 3; q >= 0; --q) {
                    const int r = c0 + q;
                    if (r < M - 1) b = -c[q] * b;
                    if (!PAD || (klive && a + r < nr))
                        dcol[static_cast<size_t>(r) * SR] = fma(b, right, fma(a4[q], left, x[r]));
                }
            }
        } else {
#pragma unroll
            for (int r = M - 1; r >= 0; --r) {
                if (r < M - 1) b = -cs[r] * b;
                if (!PAD || (klive && a + r < nr))
                    dcol[static_cast<size_t>(r) * SR] = fma(b, right, fma(al[r], left, x[r]));
            }
        }
        if (TPC > 1 && t + 1 < TPC) __syncthreads();  // the reduced rows are reused by the next tile
    }
    tm_free();
    tl_end(v, s, 0);
}

inline size_t pa_smem(int nr, int kl = 16, int tpc = 1, int seg = 16) {
    const int S = (nr + seg - 1) / seg, nt = kl * S;
    const int rst = kRing * 4 + (tpc > 1 ? 12 : 0) + 1;
    return sizeof(double) * (static_cast<size_t>(kl) * (8 * S + 9) + static_cast<size_t>(rst) * nt +
                             static_cast<size_t>(nr) * (kFR + 2));
}

// ------------------------------------------------------------ pass B, fused plane
// A cluster of CS CTAs per (problem, plane i); CTA c holds rows j in
// [c*RV, (c+1)*RV) of the plane of dU1 in shared memory. The v-lines (columns
// k) are solved by segmented affine scans of the table LU: every CTA scans its
// own 16-row segments, broadcasts the segment end values to all CTAs of the
// cluster through distributed shared memory, and each CTA then runs the (short)
// carry chain over all segments itself. The y-lines (rows j, CTA-local) use the
// partition method (16-row segments, per-line reduced systems inside a warp),
// and each y-segment finishes straight into U += dU3, Dirichlet re-imposition,
// max|dU| and the guard (solver.cpp:136-176).
// Element (j,k) lives at j*PITCH + (k/16)*17 + k%16: both the column walks
// (lanes = k) and the segment walks (lanes = segments) are at most 2-way bank
// conflicted.
template <int NV, int NY, int CS, int NTX, int MB = 0>
struct PlaneGeom {
    static constexpr int MS = 16;                 // rows per segment (v and y)
    static constexpr int RV = NV / CS;            // rows j per CTA
    static constexpr int LY = NY / MS;            // y segments per line
    static constexpr int SV = NV / MS;            // v segments per column
    static constexpr int SVL = RV / MS;           // v segments per CTA
    // rows of 16-element segments at an 18-element stride (16-byte aligned for
    // 128-bit accesses); PITCH = 4 (mod 16) spreads 4 consecutive rows over the banks
    static constexpr int P0 = LY * 18;
    static constexpr int PITCH = P0 + ((4 - (P0 % 16)) + 16) % 16;
    static constexpr int NT = NTX;
    static constexpr int YROUNDS = (RV * LY + NT - 1) / NT;
    static constexpr int TILE = RV * PITCH;
    static constexpr int VT = 6 * NV + 2;         // v tables: RP B E BF BB V, + the plane's 2 y-face values
    static constexpr int YT = 2 * (LY * 17);      // y tables: (S6, T6) pairs, 17-pair segments
    // v-lines of 64+ rows: register scans, segment carries as [segment][k]
    static constexpr bool REGV = NV >= 64;
    static constexpr int CP = NY;                 // carry row
    static constexpr int CAR = REGV ? 2 * SV * CP : 0;  // v carries (all segments, both directions)
    // y-line reduced rows in shared memory only for lines of < 8 segments (per warp: LY x TS + 1)
    static constexpr int EY = LY >= 8 ? 0 : (NT / 32) * ((NY / 16) * (8 * (32 / (NY / 16)) + 1) + 1);
    static constexpr size_t SMEM = sizeof(double) * (TILE + VT + YT + CAR + EY);
    // CTAs per SM the shared memory allows, capped at 128 registers per thread
    static constexpr int BY_SMEM = static_cast<int>((227 * 1024) / (SMEM + 1024));
    static constexpr int MINB = MB ? MB : (512 / NT) < BY_SMEM ? (512 / NT) : (BY_SMEM > 0 ? BY_SMEM : 1);
    static_assert(RV % MS == 0 && NY % MS == 0, "segments must tile the plane");
    static_assert(32 % LY == 0 && NT % 32 == 0, "y-lines must not straddle warps");
    static_assert((RV * NY / 2) % NT == 0, "plane rows must split evenly over the block");
    __device__ static int at(int j, int k) { return j * PITCH + (k >> 4) * 18 + (k & 15); }
    __device__ static int ci(int t, int k) { return t * CP + k; }
};

// Row 0 of a y-line (discretization.cpp:274-289) with its second super-diagonal
// folded into row 1 (solver.cpp:28-40): the row's diagonal f0d and upper f0u, and
// what the fold does to the right-hand side: x0 -= f x1 (f != 0), or the lagged
// x0 -= s20 x2 when row 1's upper coupling vanishes (lag). q0, q1 = theta dt
// g6 / (2 dxy) of rows 0 and 1. Shared by pass B and the pivot table build.
struct YRow0 {
    double d, u, f, s20;
    bool lag;
};
__device__ __forceinline__ YRow0 y_row0(bool yminD, int y_order, double q0, double q1, double th,
                                        double react, double dint) {
    YRow0 o{1.0, 0.0, 0.0, 0.0, false};
    if (yminD) return o;
    if (y_order == 1) {
        o.d = fma(2.0, q0, fma(th, react, 1.0));
        o.u = -2.0 * q0;
        return o;
    }
    o.d = fma(3.0, q0, fma(th, react, 1.0));
    o.u = -4.0 * q0;
    o.s20 = q0;
    const double l1 = q1, u1 = -q1;
    if (fabs(u1) > 1e-300) {
        o.f = o.s20 / u1;
        o.d = fma(-o.f, l1, o.d);
        o.u = fma(-o.f, dint, o.u);
    } else {
        o.lag = true;
    }
    return o;
}

// YLU: the y-lines of a constant model are solved from the precomputed pivots
// of the reference's own Thomas order (v.ylu, 1 / pivot per node): the forward
// and backward substitutions are affine recurrences with known coefficients,
// run as 16-row segment scans per lane with the segment carries resolved by two
// lane scans per line — one right-hand side and two arrays per thread instead of
// the partition method's three right-hand sides and per-step factorisation.
template <int NV, int NY, int CS, int NTX, int MB, bool PAD = false, bool YLU = false>
__global__ void __launch_bounds__(NTX, (PlaneGeom<NV, NY, CS, NTX, MB>::MINB))
k_plane(BatchView v, int s) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of pass A
    tl_begin(v, s, 2);
    using G = PlaneGeom<NV, NY, CS, NTX, MB>;
    constexpr int MS = G::MS, LY = G::LY, SV = G::SV, SVL = G::SVL, RV = G::RV, NT = G::NT;
    extern __shared__ double sm[];
    double* tile = sm;
    double* vtab = tile + G::TILE;   // [6][NV]: RP, B, E, BF, BB, V; then y-face values (YMAX, YMIN)
    double* ytab = vtab + G::VT;     // [LY*17] (S6, T6) pairs
    double* car = ytab + G::YT;      // [2][SV][NY]
    double* ey = car + G::CAR;       // [NT/LY lines][LY][8]
    const int nr = v.nr;
    // PAD: an nv x ny plane (nv, ny <= NV = NY) in the padded tile; rows j >= nv and
    // columns k >= ny are inert (identity lines, no loads or stores)
    static_assert(!PAD || CS == 1, "padded planes fit one CTA");
    const int nvr = PAD ? v.nv : NV, nyr = PAD ? v.ny : NY;
    const int tid = threadIdx.x;
    const int w = blockIdx.x / CS;
    const int c = CS > 1 ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
    const int j0 = c * RV;
    const int p = w / nr, i = w - (w / nr) * nr;
    DevStatus& st = v.st[p];
    // a failed problem skips the work but still takes part in the cluster barriers;
    // failed_before is uniform over the cluster (values written by earlier launches)
    const bool live_p = v.dbg || !failed_before(st, s);
    // distributed shared memory of a peer CTA may be written only once the whole
    // cluster is known to be running: arrive here, wait before the first bcast
    // the v-line carries of a cluster travel as asynchronous remote stores counted
    // by the receiving CTA's mbarrier (one per direction, used once)
    __shared__ alignas(8) unsigned long long vbar[2];
    const unsigned vbar_s = static_cast<unsigned>(__cvta_generic_to_shared(vbar));
    if constexpr (CS > 1) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(vbar_s) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(vbar_s + 8u) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    if constexpr (CS > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    auto cluster_sync = [] {
        if constexpr (CS > 1) cg::this_cluster().sync();
        else __syncthreads();
    };
    auto bcast = [&](int idx, double val) {  // write car[idx] in every CTA of the cluster
        if constexpr (CS > 1) {
#pragma unroll
            for (int r = 0; r < CS; ++r) cg::this_cluster().map_shared_rank(car, r)[idx] = val;
        } else {
            car[idx] = val;
        }
    };
    const size_t off = static_cast<size_t>(p) * v.N;
    const size_t pb = off + (static_cast<size_t>(i) * nvr + j0) * nyr;  // first row of this CTA
    const FT F = ftab(v, p, s);
    // per-plane scalars, loaded while the plane is staged
    const ProblemConst& pc = v.pc[p];
    const double th = pc.theta_dt, bound = pc.bound;
    const double a_i = __ldg(F.R + kFR * i + FR_A), react = __ldg(F.R + kFR * i + FR_REACT);
    // planes with 64+ rows solve the v-lines in registers: thread (kc, sl0)
    // holds column kc's local segments sl0, sl0 + SSTEP, ... (TPT of them)
    constexpr bool REGV = G::REGV;
    constexpr int TPT = REGV ? NY * SVL / NT : 1;
    constexpr int SSTEP = REGV ? NT / NY : 1;
    static_assert(!REGV || (NT % NY == 0 && (NY * SVL) % NT == 0), "register v-phase shape");
    const int kc = tid % NY, sl0 = tid / NY;
    // two segments per thread (the 128- and 256-wide planes): the thread takes two
    // adjacent columns of ONE segment instead, so every table value read from
    // shared memory serves two columns and rows move as 128-bit accesses
    constexpr bool VPAIR = REGV && !PAD && TPT == 2 && NT / (NY / 2) == SVL;

    const int kp = tid % (NY / 2), slp = tid / (NY / 2);
    constexpr bool LATE_PF = VPAIR;
    double xv[TPT][MS];
    {  // staged even for a failed problem: the loads need not wait for the status word
        // U (and pivot) rows -> L2 ahead of the update, so its loads hit L2; the
        // column-pair variant asks for them once its dU1 loads have landed (LATE_PF),
        // so the two streams do not share DRAM bandwidth and the v phase keeps DRAM busy
        if (!PAD && tid == 0 && !LATE_PF) {
            constexpr unsigned bytes = RV * NY * sizeof(double);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(v.U + pb), "r"(bytes) : "memory");
            if constexpr (YLU)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(v.ylu + pb), "r"(bytes) : "memory");
        }
        if constexpr (VPAIR) {
            // two adjacent columns of one 16-row segment per thread: 128-bit row loads
            const double2* src = reinterpret_cast<const double2*>(v.D + pb + static_cast<size_t>(slp) * MS * NY) + kp;
#pragma unroll
            for (int r = 0; r < MS; ++r) {
                const double2 t2 = __ldg(src + static_cast<size_t>(r) * (NY / 2));
                xv[0][r] = t2.x;
                xv[1][r] = t2.y;
            }
        } else if constexpr (REGV) {
            // column segments of dU1 straight into registers (lanes = k: coalesced rows)
#pragma unroll
            for (int q = 0; q < TPT; ++q)
#pragma unroll
                for (int r = 0; r < MS; ++r) {
                    const int jr = (sl0 + q * SSTEP) * MS + r;
                    if constexpr (PAD)
                        xv[q][r] = (jr < nvr && kc < nyr) ? __ldg(v.D + pb + static_cast<size_t>(jr) * nyr + kc) : 0.0;
                    else
                        xv[q][r] = __ldg(v.D + pb + static_cast<size_t>(jr) * NY + kc);
                }
        } else if constexpr (PAD) {
            for (int e = tid; e < RV * NY; e += NT) {
                const int j = e / NY, k = e - (e / NY) * NY;
                tile[G::at(j, k)] = (j < nvr && k < nyr) ? __ldg(v.D + pb + static_cast<size_t>(j) * nyr + k) : 0.0;
            }
        } else {
            // stage the rows of dU1: all 128-bit loads in flight, then the smem stores
            constexpr int PER = RV * NY / 2 / NT;
            const double2* src = reinterpret_cast<const double2*>(v.D + pb);
            double2 t[PER];
#pragma unroll
            for (int q = 0; q < PER; ++q) t[q] = __ldg(src + q * NT + tid);
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int e = q * NT + tid;
                const int j = (2 * e) / NY, k = 2 * e - j * NY;
                *reinterpret_cast<double2*>(tile + G::at(j, k)) = t[q];  // k even: 16-byte aligned
            }
        }
        for (int e = tid; e < NV; e += NT) {
            if (PAD && e >= nvr) {  // inert rows: identity v-line rows, decoupled
                vtab[e] = 1.0;
                vtab[NV + e] = vtab[2 * NV + e] = vtab[3 * NV + e] = vtab[4 * NV + e] = vtab[5 * NV + e] = 0.0;
                continue;
            }
            const double* Vr = F.V + kFV * e;
            vtab[e] = Vr[FV_RP];
            vtab[NV + e] = Vr[FV_B];
            vtab[2 * NV + e] = Vr[FV_E];
            vtab[3 * NV + e] = Vr[FV_BF];
            vtab[4 * NV + e] = Vr[FV_BB];
            vtab[5 * NV + e] = Vr[FV_V];
        }
        if (tid < 2)  // this plane's y-face values at t_next: YMAX, YMIN
            vtab[6 * NV + tid] = __ldg(v.fb + static_cast<size_t>(p) * v.fb_stride + 2 * nyr + tid * nr + i);
        for (int e = tid; e < NY; e += NT) {  // padded so the segments hit distinct banks
            // scaled by theta dt: a y-row coefficient is one FMA, th g6 = h1 (th S6) + (th T6)
            const int cc = 2 * ((e >> 4) * 17 + (e & 15));
            const double thp = v.pc[p].theta_dt;
            ytab[cc] = (PAD && e >= nyr) ? 0.0 : thp * F.Y[kFY * e + FY_S6];
            ytab[cc + 1] = (PAD && e >= nyr) ? 0.0 : thp * F.Y[kFY * e + FY_T6];
        }
    }
    __syncthreads();
    if constexpr (CS > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    const bool planeD = (i == nr - 1 && dir(v, F_RMAX)) || (i == 0 && dir(v, F_RMIN));
    const bool yminD = dir(v, F_YMIN), ymaxD = dir(v, F_YMAX);
    const bool vminD = dir(v, F_VMIN), vmaxD = dir(v, F_VMAX);
    const bool vwork = live_p && !planeD;

    // ---- v-lines (columns k), skip columns on y Dirichlet faces (solver.cpp:142)
    if constexpr (VPAIR) {
        // the table LU's two substitutions as segment scans in registers, columns
        // 2kp and 2kp+1 of local segment slp; segment end values go to every CTA of
        // the cluster, and each thread runs the carry chain up to its own segment
        const int g = c * SVL + slp;       // this thread's segment of the column (warp-uniform)
        const int ag = g * MS;             // its first row
        const bool vsa = vwork && !(kp == 0 && yminD);
        const bool vsb = vwork && !(kp == NY / 2 - 1 && ymaxD);
        const unsigned car_s = static_cast<unsigned>(__cvta_generic_to_shared(car));
        auto bcast2 = [&](int d, int idx, double va, double vb) {
            if constexpr (CS > 1) {
#pragma unroll
                for (int r = 0; r < CS; ++r)
                    st_async_d2(map_cluster(car_s + 8u * idx, r), va, vb, map_cluster(vbar_s + 8u * d, r));
            } else {
                *reinterpret_cast<double2*>(car + idx) = make_double2(va, vb);
            }
        };
        // every thread of every CTA of the cluster sends one pair per direction
        auto carry_wait = [&](int d) {
            if constexpr (CS > 1) {
                if (vwork) {  // cluster-uniform
                    if (tid == 0) mbar_expect(vbar_s + 8u * d, CS * NT * 16u);
                    mbar_wait_cluster(vbar_s + 8u * d);
                }
            } else {
                __syncthreads();
            }
        };
        if (vwork) {
            int bad = -1;  // first singular v pivot (table NaN), warp-uniform
#pragma unroll
            for (int jj = 0; jj < NV; jj += 32) {
                const unsigned m = __ballot_sync(0xffffffffu, isnan(vtab[jj + (tid & 31)]));
                if (m && bad < 0) bad = jj + __ffs(m) - 1;
            }
            if (bad >= 0 && c == 0 && slp == 0) {
                if (vsa) record_pivot(st, s, 1, i * nyr + 2 * kp, bad);
                if (vsb) record_pivot(st, s, 1, i * nyr + 2 * kp + 1, bad);
            }
            double la = 0.0, lb = 0.0;
#pragma unroll
            for (int r = 0; r < MS; ++r) {
                const double bq = vtab[NV + ag + r], rq = vtab[ag + r];
                la = fma(bq, la, rq * xv[0][r]);
                lb = fma(bq, lb, rq * xv[1][r]);
                xv[0][r] = la;
                xv[1][r] = lb;
            }
            bcast2(0, G::ci(g, 2 * kp), la, lb);
        }
        if (LATE_PF && tid == 0) {
            constexpr unsigned bytes = RV * NY * sizeof(double);
            if constexpr (YLU)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(v.ylu + pb), "r"(bytes) : "memory");
        }
        carry_wait(0);
        if (vwork) {
            double ca = 0.0, cb = 0.0;  // forward carry into segment g
#pragma unroll 1
            for (int t = 0; t < g; ++t) {
                const double bf = vtab[3 * NV + t * MS + MS - 1];
                const double2 e = *reinterpret_cast<const double2*>(car + G::ci(t, 2 * kp));
                ca = fma(bf, ca, e.x);
                cb = fma(bf, cb, e.y);
            }
            double xa = 0.0, xb = 0.0;
#pragma unroll
            for (int r = MS - 1; r >= 0; --r) {
                const double bf = vtab[3 * NV + ag + r], eq = vtab[2 * NV + ag + r];
                xa = fma(eq, xa, fma(bf, ca, xv[0][r]));
                xb = fma(eq, xb, fma(bf, cb, xv[1][r]));
                xv[0][r] = xa;
                xv[1][r] = xb;
            }
            bcast2(1, SV * G::CP + G::ci(g, 2 * kp), xa, xb);
        }
        carry_wait(1);
        {
            double ca = 0.0, cb = 0.0;  // backward carry into segment g, from the top
            if (vwork) {
#pragma unroll 1
                for (int t = SV - 1; t > g; --t) {
                    const double bb = vtab[4 * NV + t * MS];
                    const double2 e = *reinterpret_cast<const double2*>(car + SV * G::CP + G::ci(t, 2 * kp));
                    ca = fma(bb, ca, e.x);
                    cb = fma(bb, cb, e.y);
                }
#pragma unroll
                for (int r = 0; r < MS; ++r) {
                    const double bb = vtab[4 * NV + ag + r];
                    xv[0][r] = fma(bb, ca, xv[0][r]);
                    xv[1][r] = fma(bb, cb, xv[1][r]);
                }
                // a column on a y Dirichlet face is not solved (solver.cpp:142): its dU1 back
                if (!vsa || !vsb) {
                    const double* src = v.D + pb + static_cast<size_t>(slp) * MS * NY + 2 * kp + (vsa ? 1 : 0);
#pragma unroll
                    for (int r = 0; r < MS; ++r) {
                        const double o = __ldg(src + static_cast<size_t>(r) * NY);
                        if (!vsa) xv[0][r] = o;
                        else xv[1][r] = o;
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < MS; ++r)
                *reinterpret_cast<double2*>(tile + G::at(slp * MS + r, 2 * kp)) = make_double2(xv[0][r], xv[1][r]);
        }
        __syncthreads();
    } else if constexpr (REGV) {
        // the table LU's two substitutions as segmented affine scans in
        // registers (TPT independent chains per thread); segment end values go
        // to every CTA of the cluster, each CTA runs the (short) carry chains
        // itself; one store of dU2 into the tile
        const bool colD = (kc == 0 && yminD) || (kc == nyr - 1 && ymaxD) || (PAD && kc >= nyr);
        const bool vs = vwork && !colD && !(v.dbg & 16);  // cluster-uniform barriers below
        if (vwork) {
            int bad = -1;  // first singular v pivot (table NaN), warp-uniform
#pragma unroll
            for (int jj = 0; jj < NV; jj += 32) {
                const unsigned m = __ballot_sync(0xffffffffu, isnan(vtab[jj + (tid & 31)]));
                if (m && bad < 0) bad = jj + __ffs(m) - 1;
            }
            if (bad >= 0 && vs && c == 0) record_pivot(st, s, 1, i * nyr + kc, bad);
        }
        if (vs) {
#pragma unroll
            for (int q = 0; q < TPT; ++q) {
                const int a = (sl0 + q * SSTEP) * MS, ag = j0 + a;
                double loc = 0.0;
#pragma unroll
                for (int r = 0; r < MS; ++r) {
                    loc = fma(vtab[NV + ag + r], loc, vtab[ag + r] * xv[q][r]);
                    xv[q][r] = loc;
                }
                bcast(G::ci(c * SVL + sl0 + q * SSTEP, kc), loc);
            }
        }
        cluster_sync();
        // every thread runs the column's forward carry chain over the segment
        // end values itself and keeps the carry into each of its segments (no
        // serial pass by one thread per column, no extra barrier)
        double cins[TPT];
        if (vs) {
            double cc = 0.0;
#pragma unroll
            for (int t = 0; t < SV; ++t) {
#pragma unroll
                for (int q = 0; q < TPT; ++q)
                    if (t == c * SVL + sl0 + q * SSTEP) cins[q] = cc;
                cc = fma(vtab[3 * NV + (t * MS + MS - 1)], cc, car[G::ci(t, kc)]);
            }
        }
        if (vs) {
#pragma unroll
            for (int q = 0; q < TPT; ++q) {
                const int sv = c * SVL + sl0 + q * SSTEP, ag = sv * MS;
                const double cin = cins[q];
                double xb = 0.0;
#pragma unroll
                for (int r = MS - 1; r >= 0; --r) {
                    const double dp = fma(vtab[3 * NV + ag + r], cin, xv[q][r]);
                    xb = fma(vtab[2 * NV + ag + r], xb, dp);
                    xv[q][r] = xb;
                }
                bcast(SV * G::CP + G::ci(sv, kc), xb);
            }
        }
        cluster_sync();
        double cos_[TPT];  // backward carries into this thread's segments, from the top
        if (vs) {
            double cc = 0.0;
#pragma unroll
            for (int t = SV - 1; t >= 0; --t) {
#pragma unroll
                for (int q = 0; q < TPT; ++q)
                    if (t == c * SVL + sl0 + q * SSTEP) cos_[q] = cc;
                cc = fma(vtab[4 * NV + t * MS], cc, car[SV * G::CP + G::ci(t, kc)]);
            }
        }
#pragma unroll
        for (int q = 0; q < TPT; ++q) {
            const int a = (sl0 + q * SSTEP) * MS;
            const double co = vs ? cos_[q] : 0.0;
#pragma unroll
            for (int r = 0; r < MS; ++r) {
                const double xq = vs ? fma(vtab[4 * NV + j0 + a + r], co, xv[q][r]) : xv[q][r];
                tile[G::at(a + r, kc)] = xq;
            }
        }
        __syncthreads();
    } else if (!planeD) {
        static_assert(CS == 1 && NV <= 32, "short columns run one thread per column");
        // short columns: one thread per column runs the table LU's two
        // substitutions as plain recurrences (no segment carries or extra
        // passes; measured faster for 32-row columns, slower for longer ones)
        if (vwork && tid < NY) {
            const int k = tid;
            if (!((k == 0 && yminD) || (k == nyr - 1 && ymaxD) || (PAD && k >= nyr))) {
                double loc = 0.0;
                int bad = -1;
#pragma unroll 8
                for (int j = 0; j < NV; ++j) {
                    if (isnan(vtab[j]) && bad < 0) bad = j;  // singular v pivot (table NaN)
                    loc = fma(vtab[NV + j], loc, vtab[j] * tile[G::at(j, k)]);
                    tile[G::at(j, k)] = loc;
                }
                if (bad >= 0) record_pivot(st, s, 1, i * nyr + k, bad);
                double xb = 0.0;
#pragma unroll 8
                for (int j = NV - 1; j >= 0; --j) {
                    xb = fma(vtab[2 * NV + j], xb, tile[G::at(j, k)]);
                    tile[G::at(j, k)] = xb;
                }
            }
        }
        __syncthreads();
    }
    // (the U rows only now: the v phase's DRAM time went to the pivot rows)
    if (LATE_PF && tid == 0) {
        constexpr unsigned bytes = RV * NY * sizeof(double);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(v.U + pb), "r"(bytes) : "memory");
    }
    // the next wave's dU1 rows -> L2 while this CTA's y phase leaves DRAM idle
    auto next_wave = [&] {
        const long long w2 = static_cast<long long>(w) + v.pf_ahead;
        if (w2 < static_cast<long long>(nr) * v.P) {
            constexpr unsigned bytes = RV * NY * sizeof(double);
            const double* nx = v.D + (static_cast<size_t>(w2) * NV + j0) * NY;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nx), "r"(bytes) : "memory");
        }
    };
    // (measured on config 3: after the second carry broadcast or after the first
    // y round instead: 268 against 260.5 us)
    if (!PAD && v.pf_ahead && tid == 0) next_wave();
    if (!live_p) return;  // no cluster barrier follows

    // ---- y-lines (rows j) + update, in rounds of NT segment tasks
    const double dint = fma(th, react, 1.0);
    const bool wmd = v.want_md;
    double md = 0.0;
#pragma unroll 1
    for (int h = 0; h < G::YROUNDS; ++h) {
        const int task = h * NT + tid;
        constexpr bool ALL_LIVE = (RV * LY) % NT == 0;  // every round full: no tail lanes
        const int jl0 = (ALL_LIVE || task < RV * LY) ? task / LY : 0, sy = task % LY;
        const bool live = (ALL_LIVE || task < RV * LY) && (!PAD || j0 + jl0 < nvr);
        const int jl = live ? jl0 : 0;
        const int j = j0 + jl;
        const int a = sy * MS;
        const bool solve = live && !planeD && !((j == 0 && vminD) || (j == nvr - 1 && vmaxD));
        double* up = v.U + pb + static_cast<size_t>(jl) * nyr + a;
        double un[MS];
        auto load_u = [&] {
            if constexpr (PAD) {  // rows of ny doubles: no 16-byte alignment, masked tail
#pragma unroll
                for (int r = 0; r < MS; ++r) un[r] = a + r < nyr ? up[r] : 0.0;
            } else {
#pragma unroll
                for (int q = 0; q < MS / 2; ++q) {
                    const double2 t = reinterpret_cast<const double2*>(up)[q];
                    un[2 * q] = t.x;
                    un[2 * q + 1] = t.y;
                }
            }
        };
        // one CTA per SM (the 128- and 256-wide planes): the warp's rows of U
        // (32/LY lines x NY = 512 doubles, contiguous) move as coalesced 128-bit
        // chunks (lane l holds elements 64q + 2l) and are exchanged with the
        // lanes that own them through the warp's tile rows, which are free once
        // every lane has read its x; loads are in flight through the solve
        // registers for U in flight through the solve (one 8-warp CTA per SM; the
        // 16-warp variant keeps its 128 registers for the solve instead)
        constexpr bool early_u = G::MINB == 1 && NT <= 256;
        constexpr int WROWS = 32 / LY;
        constexpr bool stage_u = WROWS * NY == 512 && ALL_LIVE && !PAD;  // all benchmarked shapes
        const int jw = jl & ~(WROWS - 1);  // the warp's first row
        const int ln = tid & 31;
        double2 us[stage_u ? 8 : 1];
        auto load_us = [&] {
            const double2* gw = reinterpret_cast<const double2*>(v.U + pb + static_cast<size_t>(jw) * NY);
#pragma unroll
            for (int q = 0; q < 8; ++q) us[q] = gw[q * 32 + ln];
        };
        if constexpr (stage_u && early_u) load_us();
        double x[MS], cs[MS], al[MS];
        static_assert(!YLU || (stage_u && LY > 1), "table-driven y-lines: the exact two-pass shapes");
        if constexpr (YLU) {
            // this lane's 16 reciprocal pivots: the warp's block of the table moves
            // as coalesced 128-bit chunks (lane l, chunk q = rows 2q, 2q+1 of its segment)
            // (HJMSV_DBG bit 64, timing only: every warp reads the table's first block)
            const double2* gq = reinterpret_cast<const double2*>(
                v.ylu + ((v.dbg & 64) ? size_t(0) : pb + static_cast<size_t>(jw) * NY));
#pragma unroll
            for (int q = 0; q < MS / 2; ++q) {
                const double2 t2 = __ldg(gq + q * 32 + ln);
                cs[2 * q] = t2.x;
                cs[2 * q + 1] = t2.y;
            }
        }
#pragma unroll
        for (int q = 0; q < MS / 2; ++q) {
            const double2 t2 = live ? *reinterpret_cast<const double2*>(tile + G::at(jl, a + 2 * q))
                                    : make_double2(0.0, 0.0);
            x[2 * q] = t2.x;
            x[2 * q + 1] = t2.y;
        }
        double yF = 0.0, aF = 0.0, bF = 0.0, yL = 0.0, aL = 0.0, bL = 0.0;
        double left = 0.0, right = 0.0;
        if constexpr (YLU) {
            constexpr unsigned FULL = 0xffffffffu;
            // forward substitution x'_k = (x_k - l_k x'_{k-1}) / piv_k inside the
            // segment from a zero carry; fa = the carry's multiplier at the last row
            double fa = 0.0, fb = 0.0;
            if (solve) {
                const double h1 = a_i * vtab[5 * NV + j];
                auto lrv = [&](int r) {
                    const double2 st6 = reinterpret_cast<const double2*>(ytab)[sy * 17 + r];
                    return fma(h1, st6.x, st6.y);
                };
                double u0f = 0.0;
                if (sy == 0) {  // row 0, folded; its pivot is in the table
                    const YRow0 r0 = y_row0(yminD, v.y_order, lrv(0), lrv(1), th, react, dint);
                    u0f = r0.u;
                    if (r0.lag) x[0] = fma(-r0.s20, x[2], x[0]);
                    else x[0] = fma(-r0.f, x[1], x[0]);
                }
                const bool lastI = sy == LY - 1 && ymaxD;
                double xp = 0.0;
                fa = 1.0;
#pragma unroll
                for (int r = 0; r < MS; ++r) {
                    const double rp = cs[r];
                    double lrp = lrv(r) * rp;  // l / piv; u = -l on interior rows: c' = -l / piv
                    double cp = -lrp;
                    if (r == 0 && sy == 0) {
                        lrp = 0.0;
                        cp = u0f * rp;
                    }
                    if (r == MS - 1 && lastI) lrp = cp = 0.0;  // the y_max face row
                    xp = fma(-lrp, xp, x[r] * rp);
                    x[r] = xp;
                    fa *= -lrp;
                    cs[r] = cp;
                }
                fb = xp;
            }
            // x'_last of every segment: inclusive scan of the affine maps over the line's lanes
#pragma unroll
            for (int off = 1; off < LY; off <<= 1) {
                const double pa = __shfl_up_sync(FULL, fa, off, LY);
                const double pb2 = __shfl_up_sync(FULL, fb, off, LY);
                const bool on = sy >= off;  // selects: the levels schedule as one block
                fb = on ? fma(fa, pb2, fb) : fb;
                fa = on ? fa * pa : fa;
            }
            double cin = __shfl_up_sync(FULL, fb, 1, LY);
            if (sy == 0) cin = 0.0;
            // carry into the rows (the multiplier of row r is the product of -l/piv
            // up to r: c' on the rows that take a carry), then the backward
            // substitution x_k = x'_k - c'_k x_{k+1} from a zero carry
            double ba = 0.0, bb = 0.0;
            if (solve) {
                double m = cin;
#pragma unroll
                for (int r = 0; r < MS; ++r) {
                    m *= cs[r];
                    x[r] += m;
                }
                double xn = 0.0;
                ba = 1.0;
#pragma unroll
                for (int r = MS - 1; r >= 0; --r) {
                    xn = fma(-cs[r], xn, x[r]);
                    x[r] = xn;
                    ba *= -cs[r];
                }
                bb = xn;
            }
#pragma unroll
            for (int off = 1; off < LY; off <<= 1) {  // x_first of every segment: suffix scan
                const double na = __shfl_down_sync(FULL, ba, off, LY);
                const double nb = __shfl_down_sync(FULL, bb, off, LY);
                const bool on = sy + off < LY;
                bb = on ? fma(ba, nb, bb) : bb;
                ba = on ? ba * na : ba;
            }
            right = __shfl_down_sync(FULL, bb, 1, LY);  // x_{a+16}; its multipliers are applied below
            if (sy == LY - 1 || !solve) right = 0.0;
        } else if (solve && !(v.dbg & 4)) {
            const double h1 = a_i * vtab[5 * NV + j];
            // th g6 / (2 dxy) per row: a table (8-warp CTAs) or recomputed at each use
            // (16-warp CTAs, whose 128 registers hold the solve's arrays)
            constexpr bool LR_TAB = NT <= 256;
            double lr[LR_TAB ? MS : 1];
            auto lrv = [&](int r) {
                if constexpr (LR_TAB) {
                    return lr[r];
                } else {
                    const double2 st6 = reinterpret_cast<const double2*>(ytab)[sy * 17 + r];
                    return fma(h1, st6.x, st6.y);
                }
            };
            if constexpr (LR_TAB) {
#pragma unroll
                for (int r = 0; r < MS; ++r) {
                    const double2 st6 = reinterpret_cast<const double2*>(ytab)[sy * 17 + r];
                    lr[r] = fma(h1, st6.x, st6.y);
                }
            }
            double f0d = dint, f0u = -lrv(0);
            if (sy == 0) {  // row 0 (discretization.cpp:274-289), folded (solver.cpp:28-40)
                f0d = 1.0;
                f0u = 0.0;
                if (!yminD) {
                    if (v.y_order == 1) {
                        f0d = fma(2.0, lrv(0), fma(th, react, 1.0));
                        f0u = -2.0 * lrv(0);
                    } else {
                        f0d = fma(3.0, lrv(0), fma(th, react, 1.0));
                        f0u = -4.0 * lrv(0);
                        const double s20 = lrv(0);
                        const double l1 = lrv(1), u1 = -lrv(1);
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
                    l = 0.0; d = f0d; u = f0u;
                } else if (PAD ? (a + r >= nyr - 1 && (a + r > nyr - 1 || ymaxD)) : (r == MS - 1 && lastI)) {
                    l = 0.0; d = 1.0; u = 0.0;  // the y_max face row (PAD: and the inert rows past it)
                } else {
                    const double q = lrv(r);
                    l = q; d = dint; u = -q;
                }
            };
            int bad_r = 0;
            // phase-ordered solve where the registers allow it (one CTA per SM)
            bool sok;
            if constexpr (G::MINB == 1) sok = seg_solve_tw<MS>(x, cs, al, yF, aF, bF, yL, aL, bL, bad_r, row);
            else sok = seg_solve<MS>(MS, x, cs, al, yF, aF, bF, yL, aL, bL, bad_r, row);
            if (!sok) record_pivot(st, s, 2, i * nvr + j, a + bad_r);
        } else {  // a line that is not solved keeps dU: zero spikes and couplings
#pragma unroll
            for (int r = 0; r < MS; ++r) cs[r] = al[r] = 0.0;
        }
        // the line's reduced system: its LY segments are LY consecutive lanes of
        // one warp, solved by a lane scan (shuffles only)
        if constexpr (YLU) {
            // (the table-driven solve above resolved the carries by its own lane scans)
        } else if constexpr (LY > 1 && LY < 8) {
            // short systems: one lane per line through shared memory (measured
            // faster than the scan for 2 and 4 segments), rows as
            // [segment][field][line] (padded, bank-conflict free)
            constexpr int LPW = 32 / LY, TS = 8 * LPW + 1;
            double* ew = ey + (tid >> 5) * (LY * TS + 1) + (tid & 31) / LY;  // this line's (0, 0)
            double* e = ew + sy * TS;
            if (live) {
                e[0] = yF; e[LPW] = aF; e[2 * LPW] = bF; e[3 * LPW] = yL; e[4 * LPW] = aL; e[5 * LPW] = bL;
            }
            __syncwarp();  // a line's LY segments lie in one warp
            if (solve && sy == 0) {
                int bt = 0;
                if (!reduced_solve(ew, LY, TS, bt, LPW)) record_pivot(st, s, 2, i * nvr + j, bt * MS);
            }
            __syncwarp();
            if (solve && sy > 0) left = e[-TS + 6 * LPW];
            if (solve && sy < LY - 1) right = e[7 * LPW];
            __syncwarp();  // ey is reused by the next round
        } else if constexpr (LY > 1) {
            double lf, rg;
            const int bt = reduced_scan<LY>(yF, aF, bF, yL, aL, bL, sy, LY, lf, rg);
            const unsigned bm = __ballot_sync(0xffffffffu, solve && bt != 0);
            if (solve) {
                // the line's first vanishing reduced pivot (its lanes are g0 .. g0+LY-1)
                const int g0 = (tid & 31) & ~(LY - 1);
                const unsigned lm = (bm >> g0) & ((LY < 32) ? ((1u << LY) - 1u) : 0xffffffffu);
                if (lm && sy == __ffs(lm) - 1) record_pivot(st, s, 2, i * nvr + j, bt * MS);
                if (sy > 0) left = lf;
                if (sy < LY - 1) right = rg;
            }
        }
        // CTAIL: the update runs in the coalesced order (measured faster on 64-, 128-
        // and 256-wide planes, slower on the 32-wide planes of config 4)
        constexpr bool CTAIL = YLU && NY >= 64;
        if constexpr (CTAIL) {
            // dU3: the right carry times the product of -c' down to each row
            double b = right;  // 0 on lines that are not solved (they keep dU2)
#pragma unroll
            for (int r = MS - 1; r >= 0; --r) {
                b *= -cs[r];
                x[r] += b;
            }
            if (wmd) {
#pragma unroll
                for (int r = 0; r < MS; ++r) md = fmax(md, fabs(x[r]));
            }
            // U += dU3 in the coalesced order: only dU3 crosses the warp's tile rows
            // (each lane overwrites the segment it read), U stays in registers as
            // 128-bit chunks from load to store
#pragma unroll
            for (int q = 0; q < MS / 2; ++q)
                *reinterpret_cast<double2*>(tile + G::at(jl, a + 2 * q)) = make_double2(x[2 * q], x[2 * q + 1]);
            if constexpr (!early_u) load_us();
            __syncwarp();
            unsigned hm = 0u;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int e = q * 64 + 2 * ln;
                const int jr = jw + e / NY, k = e % NY, jg = j0 + jr;
                const double2 d2 = *reinterpret_cast<const double2*>(tile + G::at(jr, k));
                double2 u2 = make_double2(us[q].x + d2.x, us[q].y + d2.y);
                // Dirichlet nodes take their closed-form values at t_next (solver.cpp:169-174)
                if (planeD || (jg == 0 && vminD) || (jg == nvr - 1 && vmaxD)) {
                    u2.x = fval(v, p, dface(v, i, jg, k), i, k);
                    u2.y = fval(v, p, dface(v, i, jg, k + 1), i, k + 1);
                } else {
                    if (k == 0 && yminD) u2.x = vtab[6 * NV + 1];
                    if (k + 1 == NY - 1 && ymaxD) u2.y = vtab[6 * NV];
                }
                us[q] = u2;
                hm = max(hm, max(static_cast<unsigned>(__double2hiint(u2.x)) & 0x7fffffffu,
                                 static_cast<unsigned>(__double2hiint(u2.y)) & 0x7fffffffu));
            }
            // guard_finite (solver.cpp:69-77): one integer max decides for the lane's 16 values
            if (!(v.dbg & 32) && hm >= static_cast<unsigned>(__double2hiint(bound))) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int e = q * 64 + 2 * ln;
                    const unsigned long long flat =
                        (static_cast<unsigned long long>(i) * nvr + j0 + jw + e / NY) * nyr + e % NY;
                    if (!(fabs(us[q].x) <= bound)) guard_fail(v, p, s, flat, us[q].x);
                    if (!(fabs(us[q].y) <= bound)) guard_fail(v, p, s, flat + 1, us[q].y);
                }
            }
            double2* gw = reinterpret_cast<double2*>(v.U + pb + static_cast<size_t>(jw) * NY);
#pragma unroll
            for (int q = 0; q < 8; ++q) gw[q * 32 + ln] = us[q];
        } else if (live) {
            if constexpr (stage_u) {
                if constexpr (!early_u) load_us();
                __syncwarp();  // every lane has read its x from the warp's tile rows
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int e = q * 64 + 2 * ln;
                    *reinterpret_cast<double2*>(tile + G::at(jw + e / NY, e % NY)) = us[q];
                }
                __syncwarp();
#pragma unroll
                for (int q = 0; q < MS / 2; ++q) {
                    const double2 t = *reinterpret_cast<const double2*>(tile + G::at(jl, a + 2 * q));
                    un[2 * q] = t.x;
                    un[2 * q + 1] = t.y;
                }
            } else {
                load_u();
            }
            double b = YLU ? right : bL;  // 0 on lines that are not solved, as are cs, al, left, right
#pragma unroll
            for (int r = MS - 1; r >= 0; --r) {
                double dq;
                if constexpr (YLU) {  // the right carry times the product of -c' down to row r
                    b *= -cs[r];
                    dq = x[r] + b;
                } else {
                    if constexpr (G::MINB == 1) b = cs[r];  // the twisted solve left beta itself
                    else if (r < MS - 1) b = -cs[r] * b;
                    dq = fma(b, right, fma(al[r], left, x[r]));
                }
                un[r] += dq;
                x[r] = dq;
            }
            if (wmd) {
#pragma unroll
                for (int r = 0; r < MS; ++r) md = fmax(md, fabs(x[r]));
            }
            if (!solve) {
#pragma unroll
                for (int r = 0; r < MS; ++r)
                    un[r] = (PAD && a + r >= nyr) ? 0.0 : fval(v, p, dface(v, i, j, a + r), i, a + r);
            } else {
                if (sy == 0 && yminD) un[0] = vtab[6 * NV + 1];
                if constexpr (PAD) {
                    if (ymaxD && a <= nyr - 1 && nyr - 1 < a + MS) un[(nyr - 1) - a] = vtab[6 * NV];
                } else {
                    if (sy == LY - 1 && ymaxD) un[MS - 1] = vtab[6 * NV];
                }
            }
            if (!(v.dbg & 32)) guard_seg<MS>(v, p, s, (static_cast<size_t>(i) * nvr + j) * nyr + a, un, bound);
            if constexpr (stage_u) {  // back through the tile rows, out as coalesced chunks
#pragma unroll
                for (int q = 0; q < MS / 2; ++q)
                    *reinterpret_cast<double2*>(tile + G::at(jl, a + 2 * q)) = make_double2(un[2 * q], un[2 * q + 1]);
                __syncwarp();
                double2* gw = reinterpret_cast<double2*>(v.U + pb + static_cast<size_t>(jw) * NY);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int e = q * 64 + 2 * ln;
                    gw[q * 32 + ln] = *reinterpret_cast<const double2*>(tile + G::at(jw + e / NY, e % NY));
                }
            } else if constexpr (PAD) {
#pragma unroll
                for (int r = 0; r < MS; ++r)
                    if (a + r < nyr) up[r] = un[r];
            } else {
#pragma unroll
                for (int q = 0; q < MS / 2; ++q)
                    reinterpret_cast<double2*>(up)[q] = make_double2(un[2 * q], un[2 * q + 1]);
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
    if ((tid & 31) == 0 && md > 0.0)
        atomicMax(&st.maxdelta_bits, static_cast<unsigned long long>(__double_as_longlong(md)));
    // this plane's entries of the face table of step s+1 (read from the next step
    // on; the step's own table was filled one step earlier or by k_faces): the
    // v faces (i, k) of this CTA's rows, the y faces (i), and on the r-face
    // planes the r faces (k); one closed form per entry (model.cpp:48-54)
    if (v.fb_next && s + 1 < v.S) {
        double* fbn = v.fb_next + static_cast<size_t>(p) * v.fb_stride;
        const double* stp = step_row(v, p, s + 1);
        const Tab T = tables(v, p, s);
        const bool rface = i == 0 || i == nr - 1;
        const int nyc = nyr / CS;  // this CTA's share of k
        const int n_ent = (c == 0 ? 2 : 0) + 2 * nyc + (rface && c == 0 ? nyr : 0);
        for (int e = tid; e < n_ent; e += NT) {
            int face, k = 0, q;
            if (e < 2 * nyc) {  // v faces: this CTA's share of k
                face = e < nyc ? F_VMAX : F_VMIN;
                k = c * nyc + (e < nyc ? e : e - nyc);
                q = 2 * nyr + 2 * nr + (face == F_VMAX ? 0 : nr * nyr) + i * nyr + k;
            } else if (c == 0 && e < 2 * nyc + 2) {  // y faces
                face = e == 2 * nyc ? F_YMAX : F_YMIN;
                k = face == F_YMAX ? nyr - 1 : 0;
                q = 2 * nyr + (face == F_YMAX ? 0 : nr) + i;
            } else {  // r faces of the boundary planes
                face = i == nr - 1 ? F_RMAX : F_RMIN;
                k = e - 2 * nyc - 2;
                q = (face == F_RMAX ? 0 : nyr) + k;
            }
            fbn[q] = (v.dmask >> face & 1) ? face_value(v.pc[p], stp, T, face, i, k) : 0.0;
        }
    }
    tl_end(v, s, 2);
}

// cudaFuncAttributeMaxDynamicSharedMemorySize belongs to the device context the
// call is made on, so it is set once per (device, kernel, size): in-process
// multi-device batches (hjmsv_batch_run over several devices) launch the same
// kernels on every device.
void smem_attr(const void* fn, size_t bytes) {
    if (bytes <= 48 * 1024) return;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;  // the launch reports it
    static std::mutex mu;
    static std::set<std::tuple<int, const void*, size_t>> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({dev, fn, bytes})) return;
    // a failure stays the pending error: the caller's cudaGetLastError reports it
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)) ==
        cudaSuccess)
        done.insert({dev, fn, bytes});
}

// programmatic dependent launch of the two passes (HJMSV_PDL=0 turns it off)
int pdl_enabled() {
    static const int on = [] {
        const char* e = std::getenv("HJMSV_PDL");
        return e ? std::atoi(e) : 1;
    }();
    return on;
}

// CTAs of a kernel resident on the current device at once (cached per device,
// kernel and launch shape): the distance of the next-wave L2 prefetches
int resident_ctas(const void* fn, int threads, size_t smem) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int, size_t>, int> memo;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(dev, fn, threads, smem);
    const auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    // from the kernel's own resources (the occupancy API answers for the current
    // shared-memory carveout, not the one the launch will get)
    int per_sm = 0, sms = 0, regs_sm = 0, thr_sm = 0, smem_sm = 0, blk_sm = 0;
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess &&
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&blk_sm, cudaDevAttrMaxBlocksPerMultiprocessor, dev) == cudaSuccess) {
        const int warps = (threads + 31) / 32;
        const int regs_cta = ((fa.numRegs * 32 + 255) / 256 * 256) * warps;  // warp granularity 256
        const size_t smem_cta = smem + fa.sharedSizeBytes + 1024;            // + the per-CTA reserve
        per_sm = std::min({blk_sm, thr_sm / threads, regs_cta ? regs_sm / regs_cta : blk_sm,
                           static_cast<int>(static_cast<size_t>(smem_sm) / smem_cta)});
    } else {
        cudaGetLastError();
        per_sm = sms = 0;
    }
    if (std::getenv("HJMSV_TIMING"))
        std::fprintf(stderr, "[hjmsv] resident CTAs: %d per SM x %d SMs (threads %d, smem %zu)\n", per_sm, sms, threads, smem);
    return memo[key] = per_sm * sms;
}

// the arrays a march touches every step (U, dU, the pivot table) fit the L2 of the
// current device: next-wave prefetches have nothing to hide (config 1: 100 MB of 126 MB)
bool fits_l2(const BatchView& v) {
    int dev = 0, l2 = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    const double bytes = static_cast<double>(v.P) * static_cast<double>(v.N) * sizeof(double) * (v.ylu ? 3.0 : 2.0);
    return bytes <= static_cast<double>(l2);
}

template <class K>
void launch_pdl(K kernel, dim3 g, dim3 b, size_t sm, cudaStream_t stream, const BatchView& v, int s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = sm;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // next-wave prefetch distance: the CTAs resident at once (HJMSV_PF_AHEAD_A: 0 off, n fixed)
    BatchView w = v;
    static const int pfa_env = [] {
        const char* e = std::getenv("HJMSV_PF_AHEAD_A");
        return e ? std::atoi(e) : -1;
    }();
    w.pf_ahead_a = pfa_env >= 0 ? pfa_env : resident_ctas(reinterpret_cast<const void*>(kernel), b.x * b.y * b.z, sm);
    if (static_cast<long long>(g.x) <= w.pf_ahead_a) w.pf_ahead_a = 0;  // one wave: nothing to prefetch
    if (pfa_env < 0 && fits_l2(v)) w.pf_ahead_a = 0;  // the march's arrays stay in L2 anyway
    cudaLaunchKernelEx(&cfg, kernel, w, s);
}

// The pivots of every y-line of a constant-model batch in the reference's Thomas
// order (solver.cpp:42-50: piv_k = d_k - l_k c'_{k-1}, c'_k = u_k / piv_k), row 0
// folded (solver.cpp:28-40), the y_max face row an identity row; rows as pass B
// builds them (discretization.cpp:261-300). One thread per line (i, j); 1 / piv
// of node (i, j, k) goes to the slot pass B's lane reads it from: block of
// 32/LY lines, lane = (j mod 32/LY) LY + k/16, chunk (k mod 16)/2.
template <int NY>
__global__ void __launch_bounds__(128) k_ylu(BatchView v, double* out, int* flag) {
    constexpr int MS = 16, LY = NY / MS, WROWS = 32 / LY;
    static_assert(WROWS * NY == 512, "a warp's block of the table is 512 nodes");
    const int p = blockIdx.y;
    const int line = blockIdx.x * blockDim.x + threadIdx.x;
    if (line >= v.nr * v.nv) return;
    const int i = line / v.nv, j = line - i * v.nv;
    const FT F = ftab(v, p, 0);
    const double th = v.pc[p].theta_dt;
    const double a_i = F.R[kFR * i + FR_A], react = F.R[kFR * i + FR_REACT];
    const double dint = fma(th, react, 1.0);
    const double h1 = a_i * F.V[kFV * j + FV_V];
    const bool yminD = dir(v, F_YMIN), ymaxD = dir(v, F_YMAX);
    const bool planeD = (i == v.nr - 1 && dir(v, F_RMAX)) || (i == 0 && dir(v, F_RMIN));
    const bool solve = !planeD && !((j == 0 && dir(v, F_VMIN)) || (j == v.nv - 1 && dir(v, F_VMAX)));
    double* blk = out + static_cast<size_t>(p) * v.N + static_cast<size_t>(i) * v.nv * NY +
                  static_cast<size_t>(j / WROWS) * (WROWS * NY);
    const int lb = (j % WROWS) * LY;
    auto q_of = [&](int k) { return fma(h1, th * F.Y[kFY * k + FY_S6], th * F.Y[kFY * k + FY_T6]); };
    const YRow0 r0 = y_row0(yminD, v.y_order, q_of(0), q_of(1), th, react, dint);
    double cprev = 0.0;
    bool bad = false;
#pragma unroll 4
    for (int k = 0; k < NY; ++k) {
        double l, d, u;
        if (k == 0) {
            l = 0.0; d = r0.d; u = r0.u;
        } else if (k == NY - 1 && ymaxD) {
            l = 0.0; d = 1.0; u = 0.0;
        } else {
            const double q = q_of(k);
            l = q; d = dint; u = -q;
        }
        const double piv = k == 0 ? d : fma(-l, cprev, d);
        double rp = 1.0 / piv;
        if (!(fabs(piv) >= 1e-300) || !(fabs(rp) <= 1e300)) bad = true;  // solver.cpp:44
        cprev = u * rp;
        if (!solve) rp = 1.0;  // identity lines are not solved (solver.cpp:149)
        const int sy = k >> 4, r = k & 15;
        blk[((r >> 1) * 32 + lb + sy) * 2 + (r & 1)] = rp;
    }
    if (bad && solve) atomicOr(flag + p, 1);
}

template <int NV, int NY, int CS, int NT, int MB = 0, bool PAD = false, bool YLU = false>
void launch_plane(const BatchView& v, int s, cudaStream_t stream) {
    using G = PlaneGeom<NV, NY, CS, NT, MB>;
    // HJMSV_PB_PAD (diagnostic): extra dynamic shared memory, to pin fewer CTAs per SM
    static const size_t pb_pad = [] {
        const char* e = std::getenv("HJMSV_PB_PAD");
        return e ? static_cast<size_t>(std::atoll(e)) : size_t(0);
    }();
    smem_attr(reinterpret_cast<const void*>(k_plane<NV, NY, CS, NT, MB, PAD, YLU>), G::SMEM + pb_pad);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(v.nr * v.P * CS);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = G::SMEM + pb_pad;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // launch ahead, wait in-kernel
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    // next-wave prefetch distance: the clusters (planes) resident at once
    // (HJMSV_PF_AHEAD: 0 off, n fixed); measured on config 3: 33 resident, 30 / 33
    // planes ahead 291 -> 271 us, 66 ahead 295 us
    BatchView w = v;
    static const int pf_env = [] {
        const char* e = std::getenv("HJMSV_PF_AHEAD");
        return e ? std::atoi(e) : -1;
    }();
    if (pf_env >= 0) {
        w.pf_ahead = pf_env;
    } else {
        static std::mutex mu;
        static std::map<int, int> memo;  // per device, for this instantiation
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(mu);
        const auto it = memo.find(dev);
        if (it != memo.end()) {
            w.pf_ahead = it->second;
        } else {
            int n = 0;
            if (CS > 1) {
                if (cudaOccupancyMaxActiveClusters(&n, k_plane<NV, NY, CS, NT, MB, PAD, YLU>, &cfg) != cudaSuccess) {
                    cudaGetLastError();
                    n = 0;
                }
            } else {
                n = resident_ctas(reinterpret_cast<const void*>(k_plane<NV, NY, CS, NT, MB, PAD, YLU>), NT,
                                  G::SMEM + pb_pad);
            }
            w.pf_ahead = memo[dev] = n;
        }
    }
    if (static_cast<long long>(v.nr) * v.P <= w.pf_ahead) w.pf_ahead = 0;  // one wave
    cudaLaunchKernelEx(&cfg, k_plane<NV, NY, CS, NT, MB, PAD, YLU>, w, s);
}

int plane_kernels() {
    static const int on = [] {
        const char* e = std::getenv("HJMSV_PLANE");
        return e ? std::atoi(e) : 1;
    }();
    return on;
}

}  // namespace

// (nv, ny) pairs with compile-time kernels: nv == ny in {32, 64, 128, 256}
int specialised_shape(const BatchView& v) {
    if (v.nv != v.ny) return 0;
    return (v.ny == 32 || v.ny == 64 || v.ny == 128 || v.ny == 256) ? v.ny : 0;
}

bool fast_supported(int nr, int nv, int ny) {
    // a collapsed v axis (price_zcb's default mesh, instruments.cpp:140-143) runs the
    // four-kernel schedule without its v sweep; other collapsed axes are served by
    // STRICT; segment counts bounded by the block shapes
    return nr >= 3 && (nv >= 3 || nv == 1) && ny >= 3 && (nr + kSegR - 1) / kSegR <= 32 &&
           (nv + kSegV - 1) / kSegV <= 16 && ny <= 32 * kSegY;
}

int fast_stride(int nr, int nv, int ny) { return fast_table_stride(nr, nv, ny); }

// pass B reads the y-line pivots from a table on the exact two-pass shapes
// (HJMSV_YLU=0: the partition method on every handle, as with model functions of t)
bool fast_ylu_supported(const BatchView& v) {
    static const int on = [] {
        const char* e = std::getenv("HJMSV_YLU");
        return e ? std::atoi(e) : 1;
    }();
    return on && (plane_kernels() == 1 || plane_kernels() == 3) && specialised_shape(v) != 0 && v.fast_step == 0;
}

void fast_ylu_build(const BatchView& v, double* ylu, int* flag, cudaStream_t stream) {
    const dim3 g((v.nr * v.nv + 127) / 128, v.P), b(128);
    switch (specialised_shape(v)) {
        case 32: k_ylu<32><<<g, b, 0, stream>>>(v, ylu, flag); break;
        case 64: k_ylu<64><<<g, b, 0, stream>>>(v, ylu, flag); break;
        case 128: k_ylu<128><<<g, b, 0, stream>>>(v, ylu, flag); break;
        case 256: k_ylu<256><<<g, b, 0, stream>>>(v, ylu, flag); break;
        default: break;
    }
}


void fast_step(const BatchView& v0, int s, cudaStream_t stream, long long* launches,
               const LaunchHook* hook, int flags) {
    // face buffers alternate by step parity: kernels of step s read w.fb, the
    // plane kernel (last of the step) fills w.fb_next for step s+1
    BatchView w = v0;
    if (w.fb) {
        const size_t half = static_cast<size_t>(w.P) * w.fb_stride;
        w.fb = v0.fb + (s & 1) * half;
        w.fb_next = v0.fb + ((s + 1) & 1) * half;
    }
    w.want_md = (flags & STEP_LAST) ? 1 : 0;
    static const int dbg_env = [] {
        const char* e = std::getenv("HJMSV_DBG");
        return e ? std::atoi(e) : 0;
    }();
    w.dbg = dbg_env;
    const BatchView& v = w;
    auto mark = [&](int idx, const char* name, double bytes) {
        if (launches) ++*launches;
        if (hook && hook->after) hook->after(hook->ctx, idx, name, bytes);
    };
    // algorithmic bytes per node of each launch (SURVEY §8d accounting): read U,
    // write dU0 | read + write the line | read + write the line | read dU, read U, write U
    const int tk = (v.ny + 31) / 32, tj = (v.nv + 7) / 8;
    const int shape = specialised_shape(v);
    const int pl = plane_kernels();
    const bool plane_exact = pl && (shape == 32 || shape == 64 || shape == 128 || shape == 256);
    // any other plane up to 128 x 128 (nv, ny >= 3) runs pass B padded in a square
    // 32 / 64 / 128 tile (inert rows and columns), after the padded pass A
    const int pmax = std::max(v.nv, v.ny);
    const int plane_pad = (pl && !plane_exact && v.nv >= 3 && v.ny >= 3 && pmax <= 128)
                              ? (pmax <= 32 ? 32 : pmax <= 64 ? 64 : 128)
                              : 0;
    const bool plane = plane_exact || plane_pad;
    static const int pa_env = [] {
        const char* e = std::getenv("HJMSV_PA");
        return e ? std::atoi(e) : 1;
    }();
    const bool pa_exact = pa_env && shape != 0 && v.nr % 16 == 0 && v.nr / 16 <= 32;
    // any other shape with nv, ny >= 3, ny <= 256, nr <= 512 (e.g. the reference's own
    // 100x50x50 caplet mesh) runs pass A padded: ny rounded up to 32/64/128/256,
    // nr to a multiple of 16, the extra lanes and rows inert
    const bool pa_pad = pa_env && !pa_exact && v.nv >= 3 && v.ny >= 3 && v.ny <= 256 && v.nr >= 3 &&
                        v.nr <= 512;
    const bool pa = pa_exact || pa_pad;
    // folding the face table into pass A pays off for single grids; a large
    // batch computes it faster as its own full-occupancy launch (measured)
    static const int fold_env = [] {
        const char* e = std::getenv("HJMSV_FOLD");
        return e ? std::atoi(e) : -1;
    }();
    const bool fold = plane && fold_env != 0;  // pass B fills the next step's face table
    if (!fold) w.fb_next = nullptr;
    if (!fold || (flags & STEP_FIRST)) {  // otherwise pass A of step s-1 filled it
        k_faces<<<dim3((v.fb_stride + 255) / 256, v.P), 256, 0, stream>>>(v, s);
        mark(4, "fx_faces", 0.0);
    }
    if (pa_pad) {
        // pass A fused (padded shapes): explicit stencil + r-lines
        const int S = (v.nr + 15) / 16;
        const int nyp = v.ny <= 32 ? 32 : v.ny <= 64 ? 64 : v.ny <= 128 ? 128 : 256;
        const dim3 g(v.nv * (nyp / 16), v.P), b(16, S);
        const size_t sm = pa_smem(v.nr);
        const bool scan = (S == 16 || S == 32) && !(v.dbg & 2);
        auto go = [&](auto kern) {
            smem_attr(reinterpret_cast<const void*>(kern), sm);
            launch_pdl(kern, g, b, sm, stream, v, s);
        };
        switch (nyp) {
            case 32: go(k_pa<0, 32, false, 16, 1, true>); break;
            case 64: go(k_pa<0, 64, false, 16, 1, true>); break;
            case 128:
                if (scan) go(k_pa<0, 128, true, 16, 1, true, 2>);
                else go(k_pa<0, 128, false, 16, 1, true>);
                break;
            default:
                if (scan) go(k_pa<0, 256, true, 16, 1, true, 2>);
                else go(k_pa<0, 256, false, 16, 1, true>);
                break;
        }
        mark(0, "fx_explicit_sweep_r", 16.0);
    } else if (pa && [&] {
                   // 32-row segments for 512-row lines (config 3: two 256-thread CTAs
                   // per SM, half the per-segment overheads; measured 340 -> 299 us);
                   // HJMSV_PA_SEG=16 keeps 16-row segments, 32 forces them where they fit
                   static const int seg_env = [] {
                       const char* e = std::getenv("HJMSV_PA_SEG");
                       return e ? std::atoi(e) : 0;
                   }();
                   const bool fits = (shape == 128 || shape == 256) && v.nr % 32 == 0 &&
                                     (v.nr / 32 == 8 || v.nr / 32 == 16) && !(v.dbg & 2);
                   return fits && (seg_env == 32 || seg_env == 33 || (seg_env == 0 && v.nr == 512));
               }()) {
        // pass A fused, 32-row segments with c' and alpha in tensor memory
        const int S = v.nr / 32;
        const dim3 g(v.nv * (v.ny / 16), v.P), b(16, S);
        const size_t sm = pa_smem(v.nr, 16, 1, 32);
        auto go = [&](auto kern) {
            smem_attr(reinterpret_cast<const void*>(kern), sm);
            launch_pdl(kern, g, b, sm, stream, v, s);
        };
        static const bool seg_noscan = [] {  // HJMSV_PA_SEG=33: warp 0's two-ended recurrence
            const char* e = std::getenv("HJMSV_PA_SEG");
            return e && std::atoi(e) == 33;
        }();
        const bool scan = S == 16 && !seg_noscan;
        if (shape == 256) {
            if (scan) go(k_pa<256, 256, true, 16, 1, false, 2, 32>);
            else go(k_pa<256, 256, false, 16, 1, false, 2, 32>);
        } else {
            if (scan) go(k_pa<128, 128, true, 16, 1, false, 2, 32>);
            else go(k_pa<128, 128, false, 16, 1, false, 2, 32>);
        }
        mark(0, "fx_explicit_sweep_r", 16.0);
    } else if (pa) {
        // pass A fused: explicit stencil + r-lines
        const int S = v.nr / 16;
        // k-lane group width: 8 for 512-row lines (two 256-thread CTAs per SM
        // instead of one 512-thread CTA), 16 otherwise; HJMSV_PA_KL overrides
        static const int kl_env = [] {
            const char* e = std::getenv("HJMSV_PA_KL");
            return e ? std::atoi(e) : 0;
        }();
        const int KLw = (kl_env == 8 || kl_env == 16) ? kl_env : (S == 32 ? 16 : 16);
        const bool kl8 = KLw == 8 && S >= 16 && (S & (S - 1)) == 0 && !(v.dbg & 2) && v.ny % 8 == 0;
        const int KLu = kl8 ? 8 : 16;
        // column tiles per CTA (HJMSV_PA_TPC = 1 or 2)
        static const int tpc_env = [] {
            const char* e = std::getenv("HJMSV_PA_TPC");
            return e ? std::atoi(e) : 1;
        }();
        const int tpc = (tpc_env == 2 && !kl8 && (v.ny / KLu) % 2 == 0) ? 2 : 1;
        const dim3 g(v.nv * (v.ny / KLu) / tpc, v.P), b(KLu, S);
        // HJMSV_PA_PAD (diagnostic): extra dynamic shared memory per CTA, to pin
        // fewer CTAs per SM in occupancy experiments
        static const size_t pad_env = [] {
            const char* e = std::getenv("HJMSV_PA_PAD");
            return e ? static_cast<size_t>(std::atoll(e)) : size_t(0);
        }();
        const size_t sm = pa_smem(v.nr, KLu, tpc) + pad_env;
        // reduced systems of 16+ segments (nr >= 256) by lane scans over all
        // warps; shorter ones by warp 0's two-ended recurrence (measured faster:
        // the scan's registers make the march spill)
        const bool scan = S >= 16 && (S & (S - 1)) == 0 && !(v.dbg & 2);
        auto go = [&](auto kern) {
            smem_attr(reinterpret_cast<const void*>(kern), sm);
            launch_pdl(kern, g, b, sm, stream, v, s);
        };
        if (tpc == 2) {
            switch (shape) {
                case 32: go(k_pa<32, 32, false, 16, 2>); break;
                case 64: go(k_pa<64, 64, false, 16, 2>); break;
                case 128:
                    if (scan) go(k_pa<128, 128, true, 16, 2>);
                    else go(k_pa<128, 128, false, 16, 2>);
                    break;
                default:
                    if (scan) go(k_pa<256, 256, true, 16, 2>);
                    else go(k_pa<256, 256, false, 16, 2>);
                    break;
            }
        } else {
            // the lane-scan variants (16 / 32 segments, the large CTAs of configs 1
            // and 3) keep the partition solve's c' and alpha rows in tensor memory (no
            // spills; config 1 pass A -7 %); the small-CTA variants stay in registers
            // (the per-CTA TMEM allocation costs more than it saves there: config 4
            // +29 %); HJMSV_PA_TM=0: registers only
            static const int tm_env = [] {
                const char* e = std::getenv("HJMSV_PA_TM");
                return e ? std::atoi(e) : 2;
            }();
            const bool tm = tm_env != 0;
            switch (shape) {
                case 32: go(k_pa<32, 32, false>); break;
                case 64: go(k_pa<64, 64, false>); break;
                case 128:
                    if (kl8 && tm) go(k_pa<128, 128, true, 8, 1, false, 2>);
                    else if (kl8) go(k_pa<128, 128, true, 8>);
                    else if (scan && tm) go(k_pa<128, 128, true, 16, 1, false, 2>);
                    else if (scan) go(k_pa<128, 128, true>);
                    else go(k_pa<128, 128, false>);
                    break;
                default:
                    if (kl8 && tm) go(k_pa<256, 256, true, 8, 1, false, 2>);
                    else if (kl8) go(k_pa<256, 256, true, 8>);
                    else if (scan && tm) go(k_pa<256, 256, true, 16, 1, false, 2>);
                    else if (scan) go(k_pa<256, 256, true>);
                    else go(k_pa<256, 256, false>);
                    break;
            }
        }
        mark(0, "fx_explicit_sweep_r", 16.0);
    } else {
        switch (shape) {
            case 32: k_ex4<32, 32><<<dim3(tk * tj, v.nr, v.P), dim3(32, 8), 0, stream>>>(v, s); break;
            case 64: k_ex4<64, 64><<<dim3(tk * tj, v.nr, v.P), dim3(32, 8), 0, stream>>>(v, s); break;
            case 128: k_ex4<128, 128><<<dim3(tk * tj, v.nr, v.P), dim3(32, 8), 0, stream>>>(v, s); break;
            case 256: k_ex4<256, 256><<<dim3(tk * tj, v.nr, v.P), dim3(32, 8), 0, stream>>>(v, s); break;
            default: k_fx_explicit<<<dim3(tk * tj, v.nr, v.P), dim3(32, 8), 0, stream>>>(v, s);
        }
        mark(0, "fx_explicit", 16.0);
        const int Sr = (v.nr + kSegR - 1) / kSegR;
        const int tkr = (v.ny + kLanesR - 1) / kLanesR;
        k_fx_r<kSegR><<<dim3(v.nv * tkr, v.P), dim3(kLanesR, Sr),
                        static_cast<size_t>(kLanesR) * Sr * 8 * sizeof(double), stream>>>(v, s);
        mark(1, "fx_sweep_r", 16.0);
    }
    if (plane) {
        // pass B fused: v-lines + y-lines + update on an SMEM-resident plane
        if (plane_pad == 32) launch_plane<32, 32, 1, 64, 0, true>(v, s, stream);
        else if (plane_pad == 64) launch_plane<64, 64, 1, 256, 0, true>(v, s, stream);
        else if (plane_pad == 128) launch_plane<128, 128, 1, 256, 0, true>(v, s, stream);
        else if (v.ylu && pl == 1 && shape == 32) launch_plane<32, 32, 1, 64, 0, false, true>(v, s, stream);
        else if (v.ylu && pl == 1 && shape == 64) launch_plane<64, 64, 1, 256, 0, false, true>(v, s, stream);
        else if (v.ylu && pl == 1 && shape == 128) launch_plane<128, 128, 1, 512, 0, false, true>(v, s, stream);
        else if (v.ylu && pl == 1 && shape == 256) launch_plane<256, 256, 4, 512, 0, false, true>(v, s, stream);
        else if (shape == 32) launch_plane<32, 32, 1, 64>(v, s, stream);
        else if (shape == 64) launch_plane<64, 64, 1, 256>(v, s, stream);
        else if (shape == 128) {
            // 16 warps (512 threads at 128 registers: the y-row coefficients recomputed
            // at each use, U loaded after the solve) — measured faster than 8 warps at
            // 243 registers; HJMSV_PLANE=2: the 8-warp plane; 3: 2-CTA clusters (diagnostics)
            if (pl == 3 && v.ylu) launch_plane<128, 128, 2, 256, 0, false, true>(v, s, stream);
            else if (pl == 3) launch_plane<128, 128, 2, 256>(v, s, stream);
            else if (pl == 2) launch_plane<128, 128, 1, 256>(v, s, stream);
            else launch_plane<128, 128, 1, 512>(v, s, stream);
        } else if (pl == 2) launch_plane<256, 256, 4, 256>(v, s, stream);
        else launch_plane<256, 256, 4, 512>(v, s, stream);
        mark(2, "fx_plane_vy_update", 24.0);
        return;
    }
    if (v.nv > 1) {  // douglas_step skips the v sweep of a collapsed v axis (solver.cpp:136)
        const int Sv = (v.nv + kSegV - 1) / kSegV;
        k_fx_v<<<dim3(v.nr * tk, v.P), dim3(32, Sv), 2ull * Sv * 32 * sizeof(double), stream>>>(v, s);
        mark(2, "fx_sweep_v", 16.0);
    }
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

void fast_thomas_batch(int n, int count, const double* lower, const double* diag, const double* upper,
                       const double* super2, double* rhs, int* fail_row, bool twisted, cudaStream_t stream) {
    const int blocks = (count + 3) / 4;
    if (twisted)
        k_thomas_fast<true><<<blocks, 128, 0, stream>>>(n, count, lower, diag, upper, super2, rhs, fail_row);
    else
        k_thomas_fast<false><<<blocks, 128, 0, stream>>>(n, count, lower, diag, upper, super2, rhs, fail_row);
}

void fast_explicit(const BatchView& v, int s, cudaStream_t stream) {
    const int tk = (v.ny + 31) / 32, tj = (v.nv + 7) / 8;
    k_fx_explicit<<<dim3(tk * tj, v.nr, v.P), dim3(32, 8), 0, stream>>>(v, s);
}

}  // namespace hjmsv_b200
