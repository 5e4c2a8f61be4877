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

}  // namespace

bool fast_supported(int nr, int nv, int ny) {
    // collapsed axes and lines longer than the scratch layout are served by STRICT
    return nr >= 3 && nv >= 3 && ny >= 3;
}

int fast_stride(int nr, int nv, int ny) { return fast_table_stride(nr, nv, ny); }

void fast_prepare(const BatchView& v, cudaStream_t) {
    const size_t ysm = (static_cast<size_t>(kTL) * (v.ny + 1) + kRD * kTL) * sizeof(double);
    cudaFuncSetAttribute(k_fast_y, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(ysm));
}

void fast_step(const BatchView& v, int s, cudaStream_t stream, long long* launches,
               const LaunchHook* hook) {
    auto mark = [&](int idx, const char* name, double bytes) {
        if (launches) ++*launches;
        if (hook && hook->after) hook->after(hook->ctx, idx, name, bytes);
    };
    // algorithmic bytes/point of each launch: read U + write dU0 (16) | read + write
    // the line (16) | read + write the line (16) | read dU, read U, write U (24)
    const unsigned npts = static_cast<unsigned>((v.N + 255) / 256);
    k_fast_explicit<<<dim3(npts, v.P), 256, 0, stream>>>(v, s);
    mark(0, "fast_explicit", 16.0);
    const int rt = 64;
    k_fast_r<<<dim3((v.nv * v.ny + rt - 1) / rt, v.P), rt, 2 * kRD * rt * sizeof(double),
               stream>>>(v, s);
    mark(1, "fast_sweep_r", 16.0);
    const int vt = 128;
    k_fast_v<<<dim3((v.nr * v.ny + vt - 1) / vt, v.P), vt, kRD * vt * sizeof(double), stream>>>(
        v, s);
    mark(2, "fast_sweep_v", 16.0);
    const int lines = v.nr * v.nv;
    const size_t ysm = (static_cast<size_t>(kTL) * (v.ny + 1) + kRD * kTL) * sizeof(double);
    k_fast_y<<<dim3((lines + kTL - 1) / kTL, v.P), kYT, ysm, stream>>>(v, s);
    mark(3, "fast_sweep_y_update", 24.0);
}

void fast_explicit(const BatchView& v, int s, cudaStream_t stream) {
    k_fast_explicit<<<dim3(static_cast<unsigned>((v.N + 255) / 256), v.P), 256, 0, stream>>>(v,
                                                                                             s);
}

}  // namespace hjmsv_b200
