// kernels_fast.cu — FAST-mode Douglas-ADI step for sm_100a (the benchmarked path).
//
// Same discretisation and boundary rules as douglas_step (solver.cpp:81-178);
// the arithmetic is reorganised for the GPU:
//   * coefficients g1..g6 come from per-axis factor tables with the stencil
//     1/dx factors folded in (lowering.cpp build_fast_tables), a few FMAs per
//     point instead of ~25 mul/add + 8 divides (discretization.cpp:56-72);
//   * pivots use a hardware reciprocal seed + two Newton steps (1 MUFU + 4 DFMA)
//     instead of IEEE divides; FMA contraction is allowed;
//   * the v-line matrix depends on j only, so its LU is precomputed once and the
//     v-sweep is 3 FP64 ops per point;
//   * the explicit operator is fused into the r-sweep's forward elimination.
// Kernels per step (all problems of a batch in one launch each):
//   k_fast_r   dU0 = dt*F(U) + Dirichlet increments, fused with the r-line Thomas
//   k_fast_v   v-lines from the precomputed LU (stride ny, coalesced over k)
//   k_fast_y   y-lines staged through shared memory + U += dU, Dirichlet, guard
// Parity with the reference is checked to 1e-10 (tests/test_gpu_parity.py).
#include <algorithm>

#include "kernels_common.cuh"

namespace hjmsv_b200 {
namespace {
using namespace dev;

struct FTab {
    const double *G1, *G4C, *G4P, *G4Q, *G4V, *G3, *REACT, *A;
    const double *V, *G2, *G5, *G3V, *L, *CP, *RP;
    const double *S6, *T6;
};

__device__ __forceinline__ FTab ftables(const BatchView& v, int p) {
    const double* t = v.fast + static_cast<size_t>(p) * v.fast_stride;
    const int nr = v.nr, nv = v.nv;
    FTab f;
    f.G1 = t + FR_G1 * nr;
    f.G4C = t + FR_G4C * nr;
    f.G4P = t + FR_G4P * nr;
    f.G4Q = t + FR_G4Q * nr;
    f.G4V = t + FR_G4V * nr;
    f.G3 = t + FR_G3 * nr;
    f.REACT = t + FR_REACT * nr;
    f.A = t + FR_A * nr;
    t += FR_COUNT * nr;
    f.V = t + FV_V * nv;
    f.G2 = t + FV_G2 * nv;
    f.G5 = t + FV_G5 * nv;
    f.G3V = t + FV_G3 * nv;
    f.L = t + FV_L * nv;
    f.CP = t + FV_CP * nv;
    f.RP = t + FV_RP * nv;
    t += FV_COUNT * nv;
    f.S6 = t + FY_S6 * v.ny;
    f.T6 = t + FY_T6 * v.ny;
    return f;
}

// 1/x: MUFU.RCP64H seed + two Newton steps (relative error ~1 ulp)
__device__ __forceinline__ double frcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

__device__ __forceinline__ double ld(const double* p) { return __ldg(p); }

// g4/(2 dxr) at (i, v_j, y_k) and g1/dxr^2
__device__ __forceinline__ double g4h_at(const FTab& F, double c4, int i, double vj, double yk) {
    return fma(c4, ld(F.G4C + i), fma(ld(F.G4Q + i), yk, fma(ld(F.G4V + i), vj, ld(F.G4P + i))));
}

// dt*F(U) at a non-Dirichlet node (apply_operator, discretization.cpp:302-364),
// with g1s = g1/dxr^2 and g4h = g4/(2dxr) supplied by the caller.
__device__ __forceinline__ double explicit_core(const BatchView& v, const ProblemConst& pc,
                                                const Tab& T, const FTab& F, const double* U,
                                                int q, int i, int j, int k, double g1s,
                                                double g4h) {
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const int sr = nv * ny, sv = ny;
    const double vj = ld(F.V + j);
    const double u0 = ld(U + q);
    double acc = -ld(F.REACT + i) * u0;
    if (nr > 1) {
        if (i == 0) {
            const double u1 = ld(U + q + sr);
            if (v.r_order == 1)
                acc = fma(2.0 * g4h, u1 - u0, acc);
            else
                acc = fma(g4h, fma(4.0, u1, -ld(U + q + 2 * sr)) - 3.0 * u0, acc);
        } else {
            const double up = ld(U + q + sr), dn = ld(U + q - sr);
            acc = fma(g1s, (up + dn) - 2.0 * u0, acc);
            acc = fma(g4h, up - dn, acc);
        }
    }
    if (nv > 1) {
        const double g5h = ld(F.G5 + j);
        if (j == 0) {
            acc = fma(2.0 * g5h, ld(U + q + sv) - u0, acc);
        } else {
            const double up = ld(U + q + sv), dn = ld(U + q - sv);
            acc = fma(ld(F.G2 + j), (up + dn) - 2.0 * u0, acc);
            acc = fma(g5h, up - dn, acc);
        }
    }
    if (ny > 1) {
        const double g6h = fma(ld(F.A + i) * vj, ld(F.S6 + k), ld(F.T6 + k));
        if (k == 0) {
            const double u1 = ld(U + q + 1);
            if (v.y_order == 1)
                acc = fma(2.0 * g6h, u1 - u0, acc);
            else
                acc = fma(g6h, fma(4.0, u1, -ld(U + q + 2)) - 3.0 * u0, acc);
        } else {
            acc = fma(g6h, ld(U + q + 1) - ld(U + q - 1), acc);
        }
    }
    if (i > 0 && i < nr - 1 && j > 0 && j < nv - 1) {
        const double cross = (ld(U + q + sr + sv) - ld(U + q + sr - sv)) -
                             (ld(U + q - sr + sv) - ld(U + q - sr - sv));
        acc = fma(ld(F.G3 + i) * ld(F.G3V + j), cross, acc);
    }
    return acc * pc.dt;
}

__device__ __forceinline__ void record_pivot(DevStatus& st, int s, int ax, int line, int row) {
    const unsigned long long key = (static_cast<unsigned long long>(ax) << 50) |
                                   (static_cast<unsigned long long>(line) << 20) |
                                   static_cast<unsigned long long>(row);
    atomicMin(&st.pivot_key, key);
    mark_fail(st, s + 1, HJMSV_SINGULAR_PIVOT);
}

// ------------------------------------------------------------- cp.async
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

constexpr int kRD = 16;  // prefetch depth (rows) of the per-thread line rings

// Per-thread ring of kRD rows of a strided line, slot-major in shared memory
// (slot*nt + tid: conflict free). Request q maps to row q (dir +1) or n-1-q.
struct LineStream {
    double* ring;
    int nt, tid;
    const double* src;
    int stride, n, dir;
    __device__ __forceinline__ const double* addr(int q) const {
        return src + static_cast<long long>(dir > 0 ? q : n - 1 - q) * stride;
    }
    __device__ __forceinline__ double* slot(int q) const { return ring + (q % kRD) * nt + tid; }
    __device__ __forceinline__ void issue(int q) const {
        if (q < n) cp_async8(slot(q), addr(q));
    }
    __device__ __forceinline__ void prologue() const {
        for (int q = 0; q < kRD - 1; ++q) {
            issue(q);
            cp_commit();
        }
    }
    // request q + kRD - 1, then wait until request q has landed
    __device__ __forceinline__ double next(int q) const {
        issue(q + kRD - 1);
        cp_commit();
        cp_wait<kRD - 1>();
        return *slot(q);
    }
};

// ------------------------------------------------------------- explicit
// dU0 = dt*F(U) at every node, Dirichlet increments on faces (solver.cpp:96-116).
__global__ void __launch_bounds__(256) k_fast_explicit(BatchView v, int s) {
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) st.maxdelta_bits = 0ull;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= v.N) return;
    const int nv = v.nv, ny = v.ny;
    const int line = q / ny;
    const int k = q - line * ny;
    const int i = line / nv, j = line - i * nv;
    const ProblemConst& pc = v.pc[p];
    const Tab T = tables(v, p);
    const FTab F = ftables(v, p);
    const double* step = step_row(v, p, s);
    const size_t off = static_cast<size_t>(p) * v.N;
    const double* __restrict__ U = v.U + off;
    const int face = dirichlet_face(v, pc, i, j, k);
    double out;
    if (face >= 0) {
        out = v.apply_only ? 0.0 : face_value(pc, step, T, face, i, k) - U[q];
    } else {
        const double vj = ld(F.V + j);
        const double g4h = g4h_at(F, step[ST_C4], i, vj, ld(T.yz + k));
        out = explicit_core(v, pc, T, F, U, q, i, j, k, ld(F.G1 + i) * vj, g4h);
    }
    v.D[off + q] = out;
}

// 2^-e for the binary exponent e of x: exact rescaling of the continuant
__device__ __forceinline__ double pow2_scale(double x) {
    const int e = ((__double2hiint(x) >> 20) & 0x7ff) - 1023;
    return __hiloint2double((1023 - e) << 20, 0);
}

// ------------------------------------------------------------- r-lines
// One thread per r-line (j,k), coalesced across k; the rhs (dU0) is streamed
// from D through a cp.async ring. Pivots in projective form
//   P_i = d_i P_{i-1} - l_i u_{i-1} P_{i-2},   1/beta_i = P_{i-1}/P_i,
// so the recurrence chain is one FMA per row and the reciprocal is off it.
// c' -> C, d' -> D, then back-substitution streams both back in reverse.
__global__ void __launch_bounds__(64) k_fast_r(BatchView v, int s) {
    extern __shared__ double ring[];
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const int line = blockIdx.x * blockDim.x + threadIdx.x;
    if (line >= nv * ny) return;
    const int j = line / ny, k = line - j * ny;
    const ProblemConst& pc = v.pc[p];
    if (is_dirichlet(v, pc, 1, j, k)) return;  // whole line prescribed (solver.cpp:127)
    const Tab T = tables(v, p);
    const FTab F = ftables(v, p);
    const size_t off = static_cast<size_t>(p) * v.N;
    double* __restrict__ D = v.D + off + line;
    double* __restrict__ C = v.C + off + line;
    const int sr = nv * ny;
    const double c4 = step_row(v, p, s)[ST_C4];
    const double vj = ld(F.V + j), yk = ld(T.yz + k);
    const double th = pc.theta_dt;
    const int nt = blockDim.x, tid = threadIdx.x;
    // rows of I - th*L_r (assemble_line_r, discretization.cpp:194-230)
    auto row = [&](int i, double& l, double& d, double& u, double& s2) {
        l = 0.0; d = 1.0; u = 0.0; s2 = 0.0;
        if (is_dirichlet(v, pc, i, j, k)) return;
        const double g4h = g4h_at(F, c4, i, vj, yk);
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
            const double w2 = th * ld(F.G1 + i) * vj, w1 = th * g4h;
            l = w1 - w2;
            d = fma(2.0, w2, 1.0);
            u = -(w2 + w1);
        }
    };
    const LineStream in{ring, nt, tid, D, sr, nr, +1};
    in.prologue();
    cp_wait<0>();
    double r0 = *in.slot(0);
    double l0, d0, u0, s20;
    row(0, l0, d0, u0, s20);
    if (s20 != 0.0 && nr > 2) {  // fold the (0,2) entry against row 1 (solver.cpp:28-40)
        double l1, d1, u1, t1;
        row(1, l1, d1, u1, t1);
        if (fabs(u1) > 1e-300) {
            const double f = s20 / u1;
            d0 = fma(-f, l1, d0);
            u0 = fma(-f, d1, u0);
            r0 = fma(-f, *in.slot(1), r0);
        } else {
            r0 = fma(-s20, *in.slot(2), r0);
        }
    }
    if (fabs(d0) < 1e-300) {
        record_pivot(st, s, 0, line, 0);
        return;
    }
    double rp = frcp(d0);
    double dp = r0 * rp;
    C[0] = u0 * rp;
    D[0] = dp;
    double pm2 = 1.0, pm1 = d0, uprev = u0;
    const double thv = th * vj;
    // interior rows 1..nr-2 (a solved line has only the r-faces as Dirichlet rows)
    for (int i = 1; i < nr - 1; ++i) {
        // requests stay contiguous: 0..kRD-2 were the prologue, i+kRD-2 now
        in.issue(i + kRD - 2);
        cp_commit();
        cp_wait<kRD - 2>();
        const double ri = *in.slot(i);
        const double w2 = thv * ld(F.G1 + i), w1 = th * g4h_at(F, c4, i, vj, yk);
        const double l = w1 - w2, d = fma(2.0, w2, 1.0), u = -(w2 + w1);
        const double P = fma(d, pm1, -(l * uprev) * pm2);
        rp = pm1 * frcp(P);
        if (fabs(rp) > 1e300) {  // |pivot| < 1e-300 (solver.cpp:49-52)
            record_pivot(st, s, 0, line, i);
            return;
        }
        dp = fma(-l * rp, dp, ri * rp);
        C[i * sr] = u * rp;
        D[i * sr] = dp;
        pm2 = pm1;
        pm1 = P;
        uprev = u;
        if ((i & 15) == 0) {
            const double sc = pow2_scale(pm1);
            pm1 *= sc;
            pm2 *= sc;
        }
    }
    // row nr-1 is the r_max Dirichlet identity row: dp = rhs, no pivot work
    in.issue(nr - 1 + kRD - 2);
    cp_commit();
    cp_wait<0>();
    dp = *in.slot(nr - 1);
    D[(nr - 1) * sr] = dp;
    cp_wait<0>();
    // back-substitution over rows nr-2..0 with c' and d' streamed in reverse
    const LineStream cs{ring, nt, tid, C, sr, nr - 1, -1};
    const LineStream ds{ring + kRD * nt, nt, tid, D, sr, nr - 1, -1};
    for (int q = 0; q < kRD - 1; ++q) {
        cs.issue(q);
        ds.issue(q);
        cp_commit();
    }
    double x = dp;
    for (int q = 0; q < nr - 1; ++q) {
        cs.issue(q + kRD - 1);
        ds.issue(q + kRD - 1);
        cp_commit();
        cp_wait<kRD - 1>();
        x = fma(-*cs.slot(q), x, *ds.slot(q));
        D[(nr - 2 - q) * sr] = x;
    }
}

// ------------------------------------------------------------------- v-lines
// The v-line matrix depends on j only: its LU (L, CP, RP) is a table and the
// sweep costs 3 FP64 ops per point, streamed through per-thread cp.async rings.
__global__ void __launch_bounds__(128) k_fast_v(BatchView v, int s) {
    extern __shared__ double ring[];
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const int line = blockIdx.x * blockDim.x + threadIdx.x;
    if (line >= nr * ny) return;
    const int i = line / ny, k = line - i * ny;
    const ProblemConst& pc = v.pc[p];
    if (is_dirichlet(v, pc, i, 1, k)) return;  // solver.cpp:142
    const FTab F = ftables(v, p);
    double* __restrict__ x =
        v.D + static_cast<size_t>(p) * v.N + static_cast<size_t>(i) * nv * ny + k;
    const int nt = blockDim.x, tid = threadIdx.x;
    const LineStream in{ring, nt, tid, x, ny, nv, +1};
    in.prologue();
    double dp = 0.0;
    for (int jj = 0; jj < nv; ++jj) {
        const double rj = in.next(jj);
        const double rp = ld(F.RP + jj);
        if (isnan(rp)) {
            record_pivot(st, s, 1, line, jj);
            return;
        }
        dp = (jj == 0 ? rj : fma(-ld(F.L + jj), dp, rj)) * rp;
        x[jj * ny] = dp;
    }
    cp_wait<0>();
    const LineStream bk{ring, nt, tid, x, ny, nv - 1, -1};
    bk.prologue();
    double xv = dp;
    for (int q = 0; q < nv - 1; ++q) {
        const int jj = nv - 2 - q;
        xv = fma(-ld(F.CP + jj), xv, bk.next(q));
        x[jj * ny] = xv;
    }
}

// ------------------------------------------------------------- y + update
// A CTA owns kTL consecutive y-lines = one contiguous chunk of kTL*ny values,
// staged in shared memory by cp.async (row pitch ny+1). One thread solves one
// line in place (projective pivots; c' in a transposed global scratch so its
// traffic is coalesced), then the CTA streams U += dU, re-imposes Dirichlet
// values, reduces max|dU| and runs the guard (solver.cpp:151-176).
constexpr int kTL = 64;   // y-lines per CTA
constexpr int kYT = 256;  // threads per CTA: all stage/update, the first kTL solve

__device__ __forceinline__ unsigned long long warp_max(unsigned long long x) {
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, x, o);
        x = y > x ? y : x;
    }
    return x;
}

__global__ void __launch_bounds__(kYT) k_fast_y(BatchView v, int s) {
    extern __shared__ double smem[];
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const int lines = nr * nv;
    const int L0 = blockIdx.x * kTL;
    const int nl = min(kTL, lines - L0);
    const int pitch = ny + 1;
    double* tile = smem;                  // [kTL][ny+1]
    double* ring = smem + kTL * pitch;    // [kRD][kTL] back-substitution prefetch
    const size_t off = static_cast<size_t>(p) * v.N;
    const size_t base = off + static_cast<size_t>(L0) * ny;
    const int cnt = nl * ny;
    for (int e = threadIdx.x; e < cnt; e += kYT) {
        const int ln = e / ny, kk = e - ln * ny;
        cp_async8(tile + ln * pitch + kk, v.D + base + e);
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    const ProblemConst& pc = v.pc[p];
    const Tab T = tables(v, p);
    const FTab F = ftables(v, p);
    const int t = threadIdx.x;
    if (t < nl) {
        const int line = L0 + t;
        const int i = line / nv, j = line - i * nv;
        if (!(ny > 1 && is_dirichlet(v, pc, i, j, 1))) {  // solver.cpp:156
            double* x = tile + t * pitch;
            double* __restrict__ cs = v.C + base + t;  // c'_k of line t at cs[k*nl]
            const double th = pc.theta_dt;
            const double h1 = ld(F.A + i) * ld(F.V + j);
            const double react = ld(F.REACT + i);
            const double dint = fma(th, react, 1.0);
            // row 0 (assemble_line_y, discretization.cpp:274-289)
            double d0 = 1.0, u0 = 0.0, s20 = 0.0;
            if (ny == 1) {
                if (!is_dirichlet(v, pc, i, j, 0)) d0 = dint;
            } else if (!is_dirichlet(v, pc, i, j, 0)) {
                const double g6h = fma(h1, ld(F.S6), ld(F.T6));
                if (v.y_order == 1) {
                    d0 = fma(th, fma(2.0, g6h, react), 1.0);
                    u0 = -2.0 * th * g6h;
                } else {
                    d0 = fma(th, fma(3.0, g6h, react), 1.0);
                    u0 = -4.0 * th * g6h;
                    s20 = th * g6h;
                }
            }
            double r0 = x[0];
            if (s20 != 0.0 && ny > 2) {  // fold (solver.cpp:28-40); row 1 is interior
                const double l1 = th * fma(h1, ld(F.S6 + 1), ld(F.T6 + 1));
                const double u1 = -l1, d1 = dint;
                if (fabs(u1) > 1e-300) {
                    const double f = s20 / u1;
                    d0 = fma(-f, l1, d0);
                    u0 = fma(-f, d1, u0);
                    r0 = fma(-f, x[1], r0);
                } else {
                    r0 = fma(-s20, x[2], r0);
                }
            }
            bool ok = fabs(d0) >= 1e-300;
            if (!ok) record_pivot(st, s, 2, line, 0);
            if (ok && ny == 1) {
                x[0] = r0 * frcp(d0);
            } else if (ok) {
                double rp = frcp(d0);
                double dp = r0 * rp;
                cs[0] = u0 * rp;
                x[0] = dp;
                double pm2 = 1.0, pm1 = d0, uprev = u0;
                // interior rows 1..ny-2: l = th*g6h, d = 1 + th*reaction, u = -l
                for (int kk = 1; kk < ny - 1; ++kk) {
                    const double l = th * fma(h1, ld(F.S6 + kk), ld(F.T6 + kk));
                    const double P = fma(dint, pm1, (l * uprev) * pm2 * -1.0);
                    rp = pm1 * frcp(P);
                    if (fabs(rp) > 1e300) {
                        record_pivot(st, s, 2, line, kk);
                        ok = false;
                        break;
                    }
                    dp = fma(-l * rp, dp, x[kk] * rp);
                    cs[kk * nl] = -l * rp;
                    x[kk] = dp;
                    pm2 = pm1;
                    pm1 = P;
                    uprev = -l;
                    if ((kk & 15) == 0) {
                        const double sc = pow2_scale(pm1);
                        pm1 *= sc;
                        pm2 *= sc;
                    }
                }
                if (ok) {
                    // row ny-1: the y_max Dirichlet identity row keeps its rhs
                    const LineStream bk{ring, kTL, t, cs, nl, ny - 1, -1};  // rows ny-2..0
                    bk.prologue();
                    double xv = x[ny - 1];
                    for (int q = 0; q < ny - 1; ++q) {
                        const int kk = ny - 2 - q;
                        xv = fma(-bk.next(q), xv, x[kk]);
                        x[kk] = xv;
                    }
                }
            }
        }
    }
    __syncthreads();
    if (st.fail_step) return;  // the reference throws before the update
    // U += dU, max|dU|, Dirichlet re-impose, guard (solver.cpp:163-176)
    unsigned long long md = 0ull;
    const double* step = step_row(v, p, s);
    double* __restrict__ U = v.U;
#pragma unroll 8
    for (int e = threadIdx.x; e < cnt; e += kYT) {
        const int ln = e / ny, kk = e - ln * ny;
        const double dq = tile[ln * pitch + kk];
        const size_t q = base + e;
        double un = U[q] + dq;
        const double ad = fabs(dq);
        if (ad > 0.0) {
            const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(ad));
            md = b > md ? b : md;
        }
        const int line = L0 + ln;
        const int i = line / nv, j = line - i * nv;
        const int face = dirichlet_face(v, pc, i, j, kk);
        if (face >= 0) un = face_value(pc, step, T, face, i, kk);
        U[q] = un;
        if (!isfinite(un)) {
            atomicMin(&st.nonfinite_first, static_cast<unsigned long long>(q - off));
            mark_fail(st, s + 1, HJMSV_NONFINITE);
        } else if (fabs(un) > pc.bound) {
            atomicMin(&st.diverge_first, static_cast<unsigned long long>(q - off));
            mark_fail(st, s + 1, HJMSV_DIVERGED);
        }
    }
    md = warp_max(md);
    if ((threadIdx.x & 31) == 0 && md) atomicMax(&st.maxdelta_bits, md);
}

// ===================================================================== v3
// Pass A: explicit operator fused with the r-line elimination, 2.5D march.
// A CTA of 32 x TJ threads owns the (j,k) columns j0..j0+TJ-1, k0..k0+31 and
// marches i = 0..nr-1. U planes arrive as (TJ+2) x 34 halo slabs through a
// cp.async ring (NB slabs, prefetch NB-3 ahead); the i-dependent factor tables
// sit in shared memory (block-uniform broadcast reads). Each thread computes
// dU0(i,j,k) from shared memory and immediately eliminates row i of its r-line
// (projective pivots), storing c' -> C and d' -> D; the back-substitution then
// streams C and D in reverse through per-thread rings.
constexpr int kNB = 6;     // plane slabs in the ring
constexpr int kSW = 34;    // slab row width: 32 columns + 2 halo

__device__ __forceinline__ double explicit_smem(const BatchView& v, double react, double g1s,
                                                double g4h, double g2s, double g5h, double g6h,
                                                double g3s, const double* Sm, const double* S0,
                                                const double* Sp, const double* S2, int c,
                                                int i, int j, int k) {
    // apply_operator (discretization.cpp:302-364) on a shared-memory stencil;
    // Sm/S0/Sp = slabs of planes i-1, i, i+1 (S2 = plane 2, used at i = 0)
    const double u0 = S0[c];
    double acc = -react * u0;
    if (i == 0) {
        const double u1 = Sp[c];
        if (v.r_order == 1)
            acc = fma(2.0 * g4h, u1 - u0, acc);
        else
            acc = fma(g4h, fma(4.0, u1, -S2[c]) - 3.0 * u0, acc);
    } else {
        const double up = Sp[c], dn = Sm[c];
        acc = fma(g1s, (up + dn) - 2.0 * u0, acc);
        acc = fma(g4h, up - dn, acc);
    }
    if (j == 0) {
        acc = fma(2.0 * g5h, S0[c + kSW] - u0, acc);
    } else {
        const double up = S0[c + kSW], dn = S0[c - kSW];
        acc = fma(g2s, (up + dn) - 2.0 * u0, acc);
        acc = fma(g5h, up - dn, acc);
    }
    if (k == 0) {
        const double u1 = S0[c + 1];
        if (v.y_order == 1)
            acc = fma(2.0 * g6h, u1 - u0, acc);
        else
            acc = fma(g6h, fma(4.0, u1, -S0[c + 2]) - 3.0 * u0, acc);
    } else {
        acc = fma(g6h, S0[c + 1] - S0[c - 1], acc);
    }
    if (i > 0 && i < v.nr - 1 && j > 0 && j < v.nv - 1) {
        const double cross = (Sp[c + kSW] - Sp[c - kSW]) - (Sm[c + kSW] - Sm[c - kSW]);
        acc = fma(g3s, cross, acc);
    }
    return acc;
}

template <int TJ>
__global__ void __launch_bounds__(32 * TJ) k_fast_rx(BatchView v, int s) {
    extern __shared__ double sm[];
    constexpr int NT = 32 * TJ;
    constexpr int SP = (TJ + 2) * kSW;
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    if (blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0) st.maxdelta_bits = 0ull;
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const int tiles_k = (ny + 31) >> 5;
    const int jt = blockIdx.x / tiles_k;
    const int j0 = jt * TJ, k0 = (blockIdx.x - jt * tiles_k) * 32;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
    const int j = j0 + ty, k = k0 + tx;
    const bool active = j < nv && k < ny;
    const ProblemConst& pc = v.pc[p];
    const size_t off = static_cast<size_t>(p) * v.N;
    const double* __restrict__ U = v.U + off;
    const int sr = nv * ny;

    // shared memory: r tables [FR_COUNT][nr] | slab ring [kNB][SP] (reused by the back rings)
    double* rt = sm;
    double* ring = sm + FR_COUNT * nr;
    const double* ftab = v.fast + static_cast<size_t>(p) * v.fast_stride;
    for (int e = tid; e < FR_COUNT * nr; e += NT) rt[e] = ftab[e];
    auto issue_slab = [&](int i) {
        if (i >= nr) return;
        double* dst = ring + (i % kNB) * SP;
        const double* src = U + static_cast<size_t>(i) * sr;
        for (int e = tid; e < SP; e += NT) {
            const int rr = e / kSW, cc = e - rr * kSW;
            const int jj = j0 - 1 + rr, kk = k0 - 1 + cc;
            if (jj >= 0 && jj < nv && kk >= 0 && kk < ny) cp_async8(dst + e, src + jj * ny + kk);
        }
    };
    for (int i = 0; i < kNB - 2; ++i) {
        issue_slab(i);
        cp_commit();
    }

    // per-column constants
    const double* vt = ftab + FR_COUNT * nr;
    const double* yt = vt + FV_COUNT * nv;
    const Tab T = tables(v, p);
    const int jc = active ? j : 0, kc = active ? k : 0;
    const double vj = ld(vt + FV_V * nv + jc), g2s = ld(vt + FV_G2 * nv + jc);
    const double g5h = ld(vt + FV_G5 * nv + jc), g3v = ld(vt + FV_G3 * nv + jc);
    const double yk = ld(T.yz + kc), s6 = ld(yt + FY_S6 * ny + kc), t6 = ld(yt + FY_T6 * ny + kc);
    const double th = pc.theta_dt, dtm = pc.dt;
    const double c4 = step_row(v, p, s)[ST_C4];
    const double* step = step_row(v, p, s);
    // Dirichlet faces of this column (precedence r_max > y_max > v_max > r_min > y_min > v_min)
    const bool rmaxD = pc.rule[F_RMAX] == RULE_DIRICHLET, rminD = pc.rule[F_RMIN] == RULE_DIRICHLET;
    int hi = -1, lo = -1;
    if (k == ny - 1 && pc.rule[F_YMAX] == RULE_DIRICHLET) hi = F_YMAX;
    else if (j == nv - 1 && pc.rule[F_VMAX] == RULE_DIRICHLET) hi = F_VMAX;
    if (k == 0 && pc.rule[F_YMIN] == RULE_DIRICHLET) lo = F_YMIN;
    else if (j == 0 && pc.rule[F_VMIN] == RULE_DIRICHLET) lo = F_VMIN;
    const bool solve = active && hi < 0 && lo < 0;  // !is_dirichlet(1,j,k) (solver.cpp:127)
    const int c = (ty + 1) * kSW + tx + 1;
    double* __restrict__ Dc = v.D + off + static_cast<size_t>(j) * ny + k;
    double* __restrict__ Cc = v.C + off + static_cast<size_t>(j) * ny + k;

    // elimination state
    double dp = 0.0, pm1 = 1.0, pm2 = 1.0, uprev = 0.0;
    double r0 = 0.0, d0 = 1.0, u0 = 0.0, s20 = 0.0;   // row 0 until the fold resolves
    double r1 = 0.0, l1 = 0.0, d1 = 1.0, u1 = 0.0;    // row 1 when the fold needs row 2
    int pending = 0;                                   // rows buffered before elimination
    bool failed = false;
    auto elim = [&](int i, double r, double l, double d, double u) {
        if (failed) return;
        if (i == 0) {
            if (fabs(d) < 1e-300) {
                record_pivot(st, s, 0, j * ny + k, 0);
                failed = true;
                return;
            }
            const double rp = frcp(d);
            dp = r * rp;
            Cc[0] = u * rp;
            Dc[0] = dp;
            pm2 = 1.0;
            pm1 = d;
            uprev = u;
            return;
        }
        if (i == nr - 1 && l == 0.0 && d == 1.0) {  // Dirichlet identity row
            dp = r;
            Dc[static_cast<size_t>(i) * sr] = dp;
            return;
        }
        const double P = fma(d, pm1, -(l * uprev) * pm2);
        const double rp = pm1 * frcp(P);
        if (fabs(rp) > 1e300) {  // |pivot| < 1e-300 (solver.cpp:49-52)
            record_pivot(st, s, 0, j * ny + k, i);
            failed = true;
            return;
        }
        dp = fma(-l * rp, dp, r * rp);
        Cc[static_cast<size_t>(i) * sr] = u * rp;
        Dc[static_cast<size_t>(i) * sr] = dp;
        pm2 = pm1;
        pm1 = P;
        uprev = u;
        if ((i & 15) == 0) {
            const double sc = pow2_scale(pm1);
            pm1 *= sc;
            pm2 *= sc;
        }
    };

    for (int i = 0; i < nr; ++i) {
        __syncthreads();  // slab i-2 is free for reuse
        issue_slab(i + kNB - 2);
        cp_commit();
        if (i == 0)
            cp_wait<0>();
        else
            cp_wait<kNB - 3>();
        __syncthreads();
        if (!active) continue;
        const double* S0 = ring + (i % kNB) * SP;
        const double* Sm = ring + ((i + kNB - 1) % kNB) * SP;
        const double* Sp = ring + ((i + 1) % kNB) * SP;
        const double* S2 = ring + (2 % kNB) * SP;
        // Dirichlet node? (dirichlet_value precedence, discretization.cpp:172-192)
        int face = -1;
        if (i == nr - 1 && rmaxD) face = F_RMAX;
        else if (hi >= 0) face = hi;
        else if (i == 0 && rminD) face = F_RMIN;
        else face = lo;
        double rhs, l = 0.0, d = 1.0, u = 0.0, s2 = 0.0;
        if (face >= 0) {
            rhs = face_value(pc, step, T, face, i, k) - S0[c];  // solver.cpp:111-116
        } else {
            const double a_i = rt[FR_A * nr + i];
            const double g1s = rt[FR_G1 * nr + i] * vj;
            const double g4h = fma(c4, rt[FR_G4C * nr + i],
                                   fma(rt[FR_G4Q * nr + i], yk,
                                       fma(rt[FR_G4V * nr + i], vj, rt[FR_G4P * nr + i])));
            const double g6h = fma(a_i * vj, s6, t6);
            const double g3s = rt[FR_G3 * nr + i] * g3v;
            rhs = dtm * explicit_smem(v, rt[FR_REACT * nr + i], g1s, g4h, g2s, g5h, g6h, g3s, Sm,
                                      S0, Sp, S2, c, i, j, k);
            if (i == 0) {  // degenerate row (discretization.cpp:207-218)
                if (v.r_order == 1) {
                    d = fma(2.0 * th, g4h, 1.0);
                    u = -2.0 * th * g4h;
                } else {
                    d = fma(3.0 * th, g4h, 1.0);
                    u = -4.0 * th * g4h;
                    s2 = th * g4h;
                }
            } else {
                const double w2 = th * g1s, w1 = th * g4h;
                l = w1 - w2;
                d = fma(2.0, w2, 1.0);
                u = -(w2 + w1);
            }
        }
        if (!solve) {
            Dc[static_cast<size_t>(i) * sr] = rhs;
            continue;
        }
        if (i == 0) {
            r0 = rhs; d0 = d; u0 = u; s20 = s2;
            pending = 1;
            continue;
        }
        if (pending == 1) {  // i == 1: resolve the (0,2) fold (solver.cpp:28-40)
            if (s20 != 0.0 && nr > 2) {
                if (fabs(u) > 1e-300) {
                    const double f = s20 / u;
                    d0 = fma(-f, l, d0);
                    u0 = fma(-f, d, u0);
                    r0 = fma(-f, rhs, r0);
                } else {  // needs rhs of row 2: keep row 1 buffered
                    r1 = rhs; l1 = l; d1 = d; u1 = u;
                    pending = 2;
                    continue;
                }
            }
            elim(0, r0, 0.0, d0, u0);
            elim(1, rhs, l, d, u);
            pending = 0;
            continue;
        }
        if (pending == 2) {  // i == 2, vanishing coupling: lag s2 on rhs[2]
            r0 = fma(-s20, rhs, r0);
            elim(0, r0, 0.0, d0, u0);
            elim(1, r1, l1, d1, u1);
            pending = 0;
        }
        elim(i, rhs, l, d, u);
    }
    cp_wait<0>();
    __syncthreads();
    if (!solve || failed) return;
    // back-substitution (solver.cpp:56) over rows nr-2..0
    const LineStream cs{ring, NT, tid, Cc, sr, nr - 1, -1};
    const LineStream ds{ring + kRD * NT, NT, tid, Dc, sr, nr - 1, -1};
    for (int q = 0; q < kRD - 1; ++q) {
        cs.issue(q);
        ds.issue(q);
        cp_commit();
    }
    double x = dp;
    for (int q = 0; q < nr - 1; ++q) {
        cs.issue(q + kRD - 1);
        ds.issue(q + kRD - 1);
        cp_commit();
        cp_wait<kRD - 1>();
        x = fma(-*cs.slot(q), x, *ds.slot(q));
        Dc[static_cast<size_t>(nr - 2 - q) * sr] = x;
    }
}

// Pass B: one CTA per i-plane (v,y) held in shared memory (pitch ny+1):
// v-sweep from the precomputed LU (thread per column k), y-sweep (thread per
// row j, projective pivots, c' in a transposed global scratch streamed back
// through per-thread rings), then U += dU, Dirichlet re-impose, max|dU| and
// the guard over the plane (solver.cpp:136-176).
constexpr int kPT = 256;

__global__ void __launch_bounds__(kPT) k_fast_plane(BatchView v, int s) {
    extern __shared__ double sm[];
    const int p = blockIdx.y;
    const int i = blockIdx.x;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const int pitch = ny + 1;
    double* tile = sm;                         // [nv][ny+1]
    double* vlu = tile + nv * pitch;           // L, CP, RP [3][nv]
    double* ys = vlu + 3 * nv;                 // S6, T6 [2][ny]
    double* ring = ys + 2 * ny;                // [kRD][nv] back rings of the y-sweep
    const size_t off = static_cast<size_t>(p) * v.N;
    const size_t pbase = off + static_cast<size_t>(i) * nv * ny;
    const int cnt = nv * ny;
    for (int e = threadIdx.x; e < cnt; e += kPT) {
        const int jj = e / ny, kk = e - jj * ny;
        cp_async8(tile + jj * pitch + kk, v.D + pbase + e);
    }
    cp_commit();
    const double* ftab = v.fast + static_cast<size_t>(p) * v.fast_stride;
    const double* vt = ftab + FR_COUNT * v.nr;
    const double* yt = vt + FV_COUNT * nv;
    for (int e = threadIdx.x; e < nv; e += kPT) {
        vlu[e] = vt[FV_L * nv + e];
        vlu[nv + e] = vt[FV_CP * nv + e];
        vlu[2 * nv + e] = vt[FV_RP * nv + e];
    }
    for (int e = threadIdx.x; e < ny; e += kPT) {
        ys[e] = yt[FY_S6 * ny + e];
        ys[ny + e] = yt[FY_T6 * ny + e];
    }
    const ProblemConst& pc = v.pc[p];
    const double th = pc.theta_dt;
    const double a_i = ftab[FR_A * nr + i], react = ftab[FR_REACT * nr + i];
    cp_wait<0>();
    __syncthreads();
    const bool plane_dir = (i == 0 && pc.rule[F_RMIN] == RULE_DIRICHLET) ||
                           (i == nr - 1 && pc.rule[F_RMAX] == RULE_DIRICHLET);
    // ---- v-sweep (solver.cpp:136-149): lines with !is_dirichlet(i,1,k)
    if (!plane_dir) {
        for (int kk = threadIdx.x; kk < ny; kk += kPT) {
            const bool kd = (kk == 0 && pc.rule[F_YMIN] == RULE_DIRICHLET) ||
                            (kk == ny - 1 && pc.rule[F_YMAX] == RULE_DIRICHLET);
            if (kd) continue;
            double* x = tile + kk;
            double dp = 0.0;
            bool ok = true;
            for (int jj = 0; jj < nv; ++jj) {
                const double rp = vlu[2 * nv + jj];
                if (isnan(rp)) {
                    record_pivot(st, s, 1, i * ny + kk, jj);
                    ok = false;
                    break;
                }
                const double r = x[jj * pitch];
                dp = (jj == 0 ? r : fma(-vlu[jj], dp, r)) * rp;
                x[jj * pitch] = dp;
            }
            if (!ok) continue;
            double xv = dp;
            for (int jj = nv - 2; jj >= 0; --jj) {
                xv = fma(-vlu[nv + jj], xv, x[jj * pitch]);
                x[jj * pitch] = xv;
            }
        }
    }
    __syncthreads();
    // ---- y-sweep (solver.cpp:151-161): lines with !is_dirichlet(i,j,1)
    const double dint = fma(th, react, 1.0);
    const double* vz = ftab + FR_COUNT * nr + FV_V * nv;
    double* __restrict__ cplane = v.C + pbase;  // c'_k of line j at cplane[k*nv + j]
    if (!plane_dir) {
        for (int jj = threadIdx.x; jj < nv; jj += kPT) {
            const bool jd = (jj == 0 && pc.rule[F_VMIN] == RULE_DIRICHLET) ||
                            (jj == nv - 1 && pc.rule[F_VMAX] == RULE_DIRICHLET);
            if (jd) continue;
            double* x = tile + jj * pitch;
            double* cs = cplane + jj;
            const double h1 = a_i * vz[jj];
            double d0 = 1.0, u0 = 0.0, s20 = 0.0;
            if (pc.rule[F_YMIN] != RULE_DIRICHLET) {  // row 0 (discretization.cpp:280-289)
                const double g6h = fma(h1, ys[0], ys[ny]);
                if (v.y_order == 1) {
                    d0 = fma(th, fma(2.0, g6h, react), 1.0);
                    u0 = -2.0 * th * g6h;
                } else {
                    d0 = fma(th, fma(3.0, g6h, react), 1.0);
                    u0 = -4.0 * th * g6h;
                    s20 = th * g6h;
                }
            }
            double r0 = x[0];
            if (s20 != 0.0 && ny > 2) {
                const double l1 = th * fma(h1, ys[1], ys[ny + 1]);
                const double u1 = -l1;
                if (fabs(u1) > 1e-300) {
                    const double f = s20 / u1;
                    d0 = fma(-f, l1, d0);
                    u0 = fma(-f, dint, u0);
                    r0 = fma(-f, x[1], r0);
                } else {
                    r0 = fma(-s20, x[2], r0);
                }
            }
            if (fabs(d0) < 1e-300) {
                record_pivot(st, s, 2, i * nv + jj, 0);
                continue;
            }
            double rp = frcp(d0);
            double dp = r0 * rp;
            cs[0] = u0 * rp;
            x[0] = dp;
            double pm2 = 1.0, pm1 = d0, uprev = u0;
            bool ok = true;
            for (int kk = 1; kk < ny - 1; ++kk) {
                const double l = th * fma(h1, ys[kk], ys[ny + kk]);
                const double P = fma(dint, pm1, (l * uprev) * pm2 * -1.0);
                rp = pm1 * frcp(P);
                if (fabs(rp) > 1e300) {
                    record_pivot(st, s, 2, i * nv + jj, kk);
                    ok = false;
                    break;
                }
                dp = fma(-l * rp, dp, x[kk] * rp);
                cs[static_cast<size_t>(kk) * nv] = -l * rp;
                x[kk] = dp;
                pm2 = pm1;
                pm1 = P;
                uprev = -l;
                if ((kk & 15) == 0) {
                    const double sc = pow2_scale(pm1);
                    pm1 *= sc;
                    pm2 *= sc;
                }
            }
            if (!ok) continue;
            // row ny-1 is the y_max identity row: x[ny-1] keeps its rhs
            const LineStream bk{ring, nv, jj, cs, nv, ny - 1, -1};
            bk.prologue();
            double xv = x[ny - 1];
            for (int q = 0; q < ny - 1; ++q) {
                const int kk = ny - 2 - q;
                xv = fma(-bk.next(q), xv, x[kk]);
                x[kk] = xv;
            }
            cp_wait<0>();
        }
    }
    __syncthreads();
    if (st.fail_step) return;  // the reference throws before the update
    // ---- U += dU, max|dU|, Dirichlet re-impose, guard (solver.cpp:163-176)
    const double* step = step_row(v, p, s);
    const Tab T = tables(v, p);
    unsigned long long md = 0ull;
    double* __restrict__ Up = v.U + pbase;
#pragma unroll 4
    for (int e = threadIdx.x; e < cnt; e += kPT) {
        const int jj = e / ny, kk = e - jj * ny;
        const double dq = tile[jj * pitch + kk];
        double un = Up[e] + dq;
        const double ad = fabs(dq);
        if (ad > 0.0) {
            const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(ad));
            md = b > md ? b : md;
        }
        const int face = dirichlet_face(v, pc, i, jj, kk);
        if (face >= 0) un = face_value(pc, step, T, face, i, kk);
        Up[e] = un;
        const unsigned long long flat = static_cast<unsigned long long>(pbase - off + e);
        if (!isfinite(un)) {
            atomicMin(&st.nonfinite_first, flat);
            mark_fail(st, s + 1, HJMSV_NONFINITE);
        } else if (fabs(un) > pc.bound) {
            atomicMin(&st.diverge_first, flat);
            mark_fail(st, s + 1, HJMSV_DIVERGED);
        }
    }
    md = warp_max(md);
    if ((threadIdx.x & 31) == 0 && md) atomicMax(&st.maxdelta_bits, md);
}

// ================================================================ pass A v4
// Explicit operator fused with a SEGMENTED r-line solve (partition method).
// Block = LANES consecutive k (same j) x S segments of M rows (S = ceil(nr/M)).
// Thread (k, s) computes dU0 for rows a..a+m-1 of column (j,k) from U (rolling
// register window over i; k+-1 through shuffles) and eliminates each row as it
// is produced, for three right-hand sides sharing one factorisation:
//     T y = r,   T alpha = -l_a e_0,   T beta = -u_{a+m-1} e_{m-1},
// so x_i = y_i + alpha_i x_{a-1} + beta_i x_{a+m}. The end rows of all segments
// form a reduced system in (x_last(s), x_first(s+1)), solved per line by one
// thread in shared memory; each thread then writes x_i = dU1 for its rows.
// Everything between the U loads and the dU1 stores stays in registers (no
// c'/d' scratch traffic). The elimination order differs from the reference's
// sequential Thomas (the north star's allowed source of difference); local and
// reduced pivots replace the global ones in the singular-pivot check.
template <int M, int LANES>
__global__ void __launch_bounds__(512) k_fast_rseg(BatchView v, int s) {
    extern __shared__ double red[];  // [8][S][LANES]: yF aF bF yL aL bL | p q
    const int p = blockIdx.y;
    DevStatus& st = v.st[p];
    if (st.fail_step) return;
    const int nr = v.nr, nv = v.nv, ny = v.ny;
    const int S = blockDim.y;
    const int tx = threadIdx.x, sg = threadIdx.y;
    if (blockIdx.x == 0 && tx == 0 && sg == 0) st.maxdelta_bits = 0ull;
    const int tiles_k = (ny + LANES - 1) / LANES;
    const int j = blockIdx.x / tiles_k;
    const int k = (blockIdx.x - j * tiles_k) * LANES + tx;
    const bool active = k < ny;
    const int kc = active ? k : ny - 1;
    const int a = sg * M;
    const int m = min(M, nr - a);
    const ProblemConst& pc = v.pc[p];
    const size_t off = static_cast<size_t>(p) * v.N;
    const int sr = nv * ny;
    const double* ftab = v.fast + static_cast<size_t>(p) * v.fast_stride;
    const double* rt = ftab;                  // r tables [FR_COUNT][nr]
    const double* vt = ftab + FR_COUNT * nr;  // v tables
    const double* yt = vt + FV_COUNT * nv;    // y tables
    const Tab T = tables(v, p);
    const double vj = ld(vt + FV_V * nv + j), g2s = ld(vt + FV_G2 * nv + j);
    const double g5h = ld(vt + FV_G5 * nv + j), g3v = ld(vt + FV_G3 * nv + j);
    const double yk = ld(T.yz + kc), vs6 = vj * ld(yt + FY_S6 * ny + kc);
    const double t6 = ld(yt + FY_T6 * ny + kc);
    const double th = pc.theta_dt, dtm = pc.dt;
    const double* step = step_row(v, p, s);
    const double c4 = step[ST_C4];
    const bool rmaxD = pc.rule[F_RMAX] == RULE_DIRICHLET, rminD = pc.rule[F_RMIN] == RULE_DIRICHLET;
    int hi = -1, lo = -1;  // Dirichlet faces of this column, precedence order
    if (k == ny - 1 && pc.rule[F_YMAX] == RULE_DIRICHLET) hi = F_YMAX;
    else if (j == nv - 1 && pc.rule[F_VMAX] == RULE_DIRICHLET) hi = F_VMAX;
    if (k == 0 && pc.rule[F_YMIN] == RULE_DIRICHLET) lo = F_YMIN;
    else if (j == 0 && pc.rule[F_VMIN] == RULE_DIRICHLET) lo = F_VMIN;
    const bool solve = active && hi < 0 && lo < 0;  // !is_dirichlet(1,j,k) (solver.cpp:127)
    const bool jlo = j > 0, jhi = j < nv - 1;
    const double* col = v.U + off + static_cast<size_t>(j) * ny + kc;  // U(0, j, k)
    double* dcol = v.D + off + static_cast<size_t>(j) * ny + kc;

    // rolling window of U(i', j-1..j+1, k) for i' = i-1, i, i+1
    auto load3 = [&](int ii, double& w0, double& w1, double& w2) {
        if (ii < 0 || ii >= nr) {
            w0 = w1 = w2 = 0.0;
            return;
        }
        const double* q = col + static_cast<size_t>(ii) * sr;
        w1 = __ldg(q);
        w0 = jlo ? __ldg(q - ny) : 0.0;
        w2 = jhi ? __ldg(q + ny) : 0.0;
    };
    double am0, am1, am2, a00, a01, a02, ap0, ap1, ap2;
    load3(a - 1, am0, am1, am2);
    load3(a, a00, a01, a02);
    load3(a + 1, ap0, ap1, ap2);
    double u2_0 = 0.0;  // U(2, j, k) for the one-sided r stencil at i = 0
    if (a == 0 && nr > 2) u2_0 = __ldg(col + 2 * static_cast<size_t>(sr));

    // elimination state: c'_r, y'_r, alpha'_r of the segment's rows
    double cs[M], ys[M], as[M];
    double cprev = 0.0, yprev = 0.0, aprev = 0.0;
    double bLs = 0.0, yLs = 0.0, aLs = 0.0;  // end-row values at r = m-1
    bool bad = false;
    int bad_row = 0;
    // row 0 of the line (segment 0): held until row 1 (or 2) resolves the fold
    double h0r = 0.0, h0d = 1.0, h0u = 0.0, h0s = 0.0;
    double h1r = 0.0, h1l = 0.0, h1d = 1.0, h1u = 0.0;
    int hold = 0;

    // eliminate row r (0-based in the segment) with coefficients (l, d, u)
    auto elim = [&](int r, double rhs, double l, double d, double u) {
        const double piv = r == 0 ? d : fma(-l, cprev, d);
        if (fabs(piv) < 1e-300 && !bad) {
            bad = true;
            bad_row = a + r;
        }
        const double rp = frcp(piv);
        const bool last = r == m - 1;
        const double c = last ? 0.0 : u * rp;  // the last row's upper couples to x_{a+m}
        const double yy = (r == 0 ? rhs : fma(-l, yprev, rhs)) * rp;
        const double aa = (r == 0 ? -l : -l * aprev) * rp;
        if (last) {
            bLs = -u * rp;
            yLs = yy;
            aLs = aa;
        }
        cprev = c;
        yprev = yy;
        aprev = aa;
        return c;
    };

#pragma unroll
    for (int r = 0; r < M; ++r) {
        const int i = a + r;
        double kl = __shfl_up_sync(0xffffffffu, a01, 1, LANES);
        double kr = __shfl_down_sync(0xffffffffu, a01, 1, LANES);
        if (r < m) {
            const double* q = col + static_cast<size_t>(i) * sr;
            if (tx == 0) kl = k > 0 ? __ldg(q - 1) : 0.0;
            if (tx == LANES - 1 || k == ny - 1) kr = k < ny - 1 ? __ldg(q + 1) : 0.0;
            int face;
            if (i == nr - 1 && rmaxD) face = F_RMAX;
            else if (hi >= 0) face = hi;
            else if (i == 0 && rminD) face = F_RMIN;
            else face = lo;
            double rhs, l = 0.0, d = 1.0, u = 0.0, s2 = 0.0;
            if (face >= 0) {
                rhs = face_value(pc, step, T, face, i, kc) - a01;  // solver.cpp:111-116
            } else {
                // dt*F(U) (apply_operator, discretization.cpp:302-364)
                const double g1s = ld(rt + FR_G1 * nr + i) * vj;
                const double g4h = fma(c4, ld(rt + FR_G4C * nr + i),
                                       fma(ld(rt + FR_G4Q * nr + i), yk,
                                           fma(ld(rt + FR_G4V * nr + i), vj,
                                               ld(rt + FR_G4P * nr + i))));
                const double g6h = fma(ld(rt + FR_A * nr + i), vs6, t6);
                const double u0 = a01;
                double acc = -ld(rt + FR_REACT * nr + i) * u0;
                if (i == 0) {
                    if (v.r_order == 1)
                        acc = fma(2.0 * g4h, ap1 - u0, acc);
                    else
                        acc = fma(g4h, fma(4.0, ap1, -u2_0) - 3.0 * u0, acc);
                } else {
                    acc = fma(g1s, (ap1 + am1) - 2.0 * u0, acc);
                    acc = fma(g4h, ap1 - am1, acc);
                }
                if (j == 0) {
                    acc = fma(2.0 * g5h, a02 - u0, acc);
                } else {
                    acc = fma(g2s, (a02 + a00) - 2.0 * u0, acc);
                    acc = fma(g5h, a02 - a00, acc);
                }
                if (k == 0) {
                    if (v.y_order == 1)
                        acc = fma(2.0 * g6h, kr - u0, acc);
                    else
                        acc = fma(g6h, fma(4.0, kr, -__ldg(q + 2)) - 3.0 * u0, acc);
                } else {
                    acc = fma(g6h, kr - kl, acc);
                }
                if (i > 0 && i < nr - 1 && jlo && jhi)
                    acc = fma(ld(rt + FR_G3 * nr + i) * g3v, (ap2 - ap0) - (am2 - am0), acc);
                rhs = dtm * acc;
                if (i == 0) {  // degenerate row (discretization.cpp:207-218)
                    if (v.r_order == 1) {
                        d = fma(2.0 * th, g4h, 1.0);
                        u = -2.0 * th * g4h;
                    } else {
                        d = fma(3.0 * th, g4h, 1.0);
                        u = -4.0 * th * g4h;
                        s2 = th * g4h;
                    }
                } else {
                    const double w2 = th * g1s, w1 = th * g4h;
                    l = w1 - w2;
                    d = fma(2.0, w2, 1.0);
                    u = -(w2 + w1);
                }
            }
            am0 = a00; am1 = a01; am2 = a02;  // advance the window
            a00 = ap0; a01 = ap1; a02 = ap2;
            load3(i + 2, ap0, ap1, ap2);
            if (!solve) {
                if (active) dcol[static_cast<size_t>(i) * sr] = rhs;
            } else if (a == 0 && r == 0) {
                h0r = rhs; h0d = d; h0u = u; h0s = s2;  // wait for row 1 (fold)
                hold = 1;
            } else if (a == 0 && r == 1) {
                if (h0s != 0.0 && nr > 2 && !(fabs(u) > 1e-300)) {
                    h1r = rhs; h1l = l; h1d = d; h1u = u;  // fold needs rhs of row 2
                    hold = 2;
                } else {
                    if (h0s != 0.0 && nr > 2) {  // fold (0,2) against row 1 (solver.cpp:28-40)
                        const double f = h0s / u;
                        h0d = fma(-f, l, h0d);
                        h0u = fma(-f, d, h0u);
                        h0r = fma(-f, rhs, h0r);
                    }
                    cs[0] = elim(0, h0r, 0.0, h0d, h0u);
                    ys[0] = yprev;
                    as[0] = aprev;
                    cs[1] = elim(1, rhs, l, d, u);
                    ys[1] = yprev;
                    as[1] = aprev;
                    hold = 0;
                }
            } else if (a == 0 && r == 2 && hold == 2) {
                h0r = fma(-h0s, rhs, h0r);  // vanishing coupling: lag s2 on rhs[2]
                cs[0] = elim(0, h0r, 0.0, h0d, h0u);
                ys[0] = yprev;
                as[0] = aprev;
                cs[1] = elim(1, h1r, h1l, h1d, h1u);
                ys[1] = yprev;
                as[1] = aprev;
                cs[2] = elim(2, rhs, l, d, u);
                ys[2] = yprev;
                as[2] = aprev;
                hold = 0;
            } else {
                cs[r] = elim(r, rhs, l, d, u);
                ys[r] = yprev;
                as[r] = aprev;
            }
        }
    }
    // local back-substitution of y and alpha (beta follows in the final pass)
    double yF = 0.0, aF = 0.0, bF = 0.0;
    if (solve) {
        double yn = yLs, an = aLs, bn = bLs;
#pragma unroll
        for (int r = M - 2; r >= 0; --r) {
            if (r < m - 1) {
                yn = fma(-cs[r], yn, ys[r]);
                an = fma(-cs[r], an, as[r]);
                bn = -cs[r] * bn;
                ys[r] = yn;
                as[r] = an;
            }
        }
        yF = m > 1 ? yn : yLs;
        aF = m > 1 ? an : aLs;
        bF = m > 1 ? bn : bLs;
        if (bad) record_pivot(st, s, 0, j * ny + k, bad_row);
    }
    const int L = LANES;
    const int SL = S * L;
    const int idx = sg * L + tx;
    double* R = red;
    if (solve) {
        R[0 * SL + idx] = yF;
        R[1 * SL + idx] = aF;
        R[2 * SL + idx] = bF;
        R[3 * SL + idx] = yLs;
        R[4 * SL + idx] = aLs;
        R[5 * SL + idx] = bLs;
    }
    __syncthreads();
    if (sg == 0 && solve && S > 1) {
        // reduced system in p_s = x_last(s), q_s = x_first(s+1), s = 0..S-2:
        //   p_s = yL_s + aL_s p_{s-1} + bL_s q_s
        //   q_s = yF_{s+1} + aF_{s+1} p_s + bF_{s+1} q_{s+1}
        double Pp = 0.0, Pq = 0.0;
        for (int q = 0; q < S - 1; ++q) {
            const int c0 = q * L + tx, c1 = c0 + L;
            const double aL = R[4 * SL + c0];
            const double A = fma(aL, Pp, R[3 * SL + c0]);
            const double B = fma(aL, Pq, R[5 * SL + c0]);
            const double aFn = R[1 * SL + c1];
            const double den = fma(-aFn, B, 1.0);
            if (fabs(den) < 1e-300) record_pivot(st, s, 0, j * ny + k, (q + 1) * M);
            const double inv = frcp(den);
            const double Qc = fma(aFn, A, R[0 * SL + c1]) * inv;
            const double Qd = R[2 * SL + c1] * inv;
            Pp = fma(B, Qc, A);
            Pq = B * Qd;
            R[6 * SL + c0] = Qc;
            R[7 * SL + c0] = Qd;
            R[3 * SL + c0] = Pp;
            R[4 * SL + c0] = Pq;
        }
        double qn = 0.0;  // q_{S-1} does not exist
        for (int q = S - 2; q >= 0; --q) {
            const int c0 = q * L + tx;
            const double qs = fma(R[7 * SL + c0], qn, R[6 * SL + c0]);
            const double ps = fma(R[4 * SL + c0], qn, R[3 * SL + c0]);
            R[6 * SL + c0] = ps;  // p_s = x_last(s)
            R[7 * SL + c0] = qs;  // q_s = x_first(s+1)
            qn = qs;
        }
    }
    __syncthreads();
    if (!solve) return;
    const double left = sg > 0 ? R[6 * SL + idx - L] : 0.0;
    const double right = sg < S - 1 ? R[7 * SL + idx] : 0.0;
    // x_r = y_r + alpha_r x_{a-1} + beta_r x_{a+m}, beta recomputed downwards
    double b = bLs;
#pragma unroll
    for (int r = M - 1; r >= 0; --r) {
        if (r < m) {
            if (r < m - 1) b = -cs[r] * b;
            const double yv = r == m - 1 ? yLs : ys[r];
            const double av = r == m - 1 ? aLs : as[r];
            dcol[static_cast<size_t>(a + r) * sr] = fma(b, right, fma(av, left, yv));
        }
    }
}

}  // namespace

bool fast_supported(int nr, int nv, int ny) {
    // collapsed axes and lines longer than the scratch layout are served by STRICT
    return nr >= 3 && nv >= 3 && ny >= 3;
}

int fast_stride(int nr, int nv, int ny) { return fast_table_stride(nr, nv, ny); }

namespace {
constexpr int kRXTJ = 2;
size_t rx_smem(const BatchView& v) {
    constexpr int NT = 32 * kRXTJ, SP = (kRXTJ + 2) * kSW;
    const size_t ring = std::max<size_t>(static_cast<size_t>(kNB) * SP, 2ull * kRD * NT);
    return (static_cast<size_t>(FR_COUNT) * v.nr + ring) * sizeof(double);
}
size_t plane_smem(const BatchView& v) {
    return (static_cast<size_t>(v.nv) * (v.ny + 1) + 3 * v.nv + 2 * v.ny +
            static_cast<size_t>(kRD) * v.nv) * sizeof(double);
}
size_t y_smem(const BatchView& v) {
    return (static_cast<size_t>(kTL) * (v.ny + 1) + kRD * kTL) * sizeof(double);
}
constexpr size_t kSmemCap = 220 * 1024;
constexpr int kSegM = 8;  // rows per r-segment
size_t seg_smem(int S, int lanes) { return 8ull * S * lanes * sizeof(double); }
}  // namespace

void fast_prepare(const BatchView& v, cudaStream_t) {
    cudaFuncSetAttribute(k_fast_y, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(y_smem(v)));
    cudaFuncSetAttribute(k_fast_rx<kRXTJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(rx_smem(v)));
    if (plane_smem(v) <= kSmemCap)
        cudaFuncSetAttribute(k_fast_plane, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(plane_smem(v)));
}

void fast_step(const BatchView& v, int s, cudaStream_t stream, long long* launches,
               const LaunchHook* hook) {
    auto mark = [&](int idx, const char* name, double bytes) {
        if (launches) ++*launches;
        if (hook && hook->after) hook->after(hook->ctx, idx, name, bytes);
    };
    // algorithmic bytes per point of each launch (SURVEY §8d accounting):
    //   pass A  read U, write dU1                         16
    //   pass B  read dU1, read U, write U                 24  (v + y + update fused)
    const int S = (v.nr + kSegM - 1) / kSegM;
    if (S <= 16) {
        const int tiles = v.nv * ((v.ny + 31) / 32);
        k_fast_rseg<kSegM, 32><<<dim3(tiles, v.P), dim3(32, S), seg_smem(S, 32), stream>>>(v, s);
    } else if (S <= 32) {
        const int tiles = v.nv * ((v.ny + 15) / 16);
        k_fast_rseg<kSegM, 16><<<dim3(tiles, v.P), dim3(16, S), seg_smem(S, 16), stream>>>(v, s);
    } else if (S <= 64) {
        const int tiles = v.nv * ((v.ny + 7) / 8);
        k_fast_rseg<kSegM, 8><<<dim3(tiles, v.P), dim3(8, S), seg_smem(S, 8), stream>>>(v, s);
    } else {
        const int tiles = ((v.nv + kRXTJ - 1) / kRXTJ) * ((v.ny + 31) / 32);
        k_fast_rx<kRXTJ><<<dim3(tiles, v.P), dim3(32, kRXTJ), rx_smem(v), stream>>>(v, s);
    }
    mark(0, "fast_explicit_r", 16.0);
    if (plane_smem(v) <= kSmemCap) {
        k_fast_plane<<<dim3(v.nr, v.P), kPT, plane_smem(v), stream>>>(v, s);
        mark(1, "fast_plane_vy_update", 24.0);
    } else {
        const int vt = 128;
        k_fast_v<<<dim3((v.nr * v.ny + vt - 1) / vt, v.P), vt, kRD * vt * sizeof(double),
                   stream>>>(v, s);
        mark(1, "fast_sweep_v", 16.0);
        const int lines = v.nr * v.nv;
        k_fast_y<<<dim3((lines + kTL - 1) / kTL, v.P), kYT, y_smem(v), stream>>>(v, s);
        mark(2, "fast_sweep_y_update", 24.0);
    }
}

void fast_explicit(const BatchView& v, int s, cudaStream_t stream) {
    k_fast_explicit<<<dim3(static_cast<unsigned>((v.N + 255) / 256), v.P), 256, 0, stream>>>(v,
                                                                                             s);
}

}  // namespace hjmsv_b200
