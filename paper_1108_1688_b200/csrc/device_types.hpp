// device_types.hpp — plain-data layout shared by the host lowering and the
// sm_100a kernels. One BatchView describes P independent problems with equal
// (nr, nv, ny) and step count, laid out problem-major in HBM; each problem's
// level uses the reference index order idx(i,j,k) = (i*nv + j)*ny + k
// (discretization.hpp:27-29): r outermost, y contiguous.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace hjmsv_b200 {

// Per-step scalar table entry (doubles), one per (problem, step).
// c4(t_mid) (discretization.cpp:47) and the closed-form face scalars at t_next
// (ratio = p(0,T_x)/p(0,t_next), G = g_factor(T_x - t_next)), model.cpp:48-54.
constexpr int kMaxTerms = 12;  // two closed-form terms per face
constexpr int kStepStride = 32;
enum StepSlot : int {
    ST_C4 = 0,
    ST_FNEXT = 1,   // f(0, t_next)
    ST_TNEXT = 2,
    ST_TMID = 3,
    ST_RATIO = 4,   // [kMaxTerms]
    ST_G = 16,      // [kMaxTerms]
    ST_HEPS2 = 28   // eps(t_mid)^2 / 2 (discretization.cpp:45)
};

// Face order = reference Face enum (discretization.hpp:84).
enum FaceId : int { F_RMIN = 0, F_RMAX, F_VMIN, F_VMAX, F_YMIN, F_YMAX };
enum FaceRuleId : int { RULE_DIRICHLET = 0, RULE_DEGENERATE = 1, RULE_ONE_SIDED = 2 };
enum FaceValueKind : int { VAL_ZERO = 0, VAL_ZCB = 1, VAL_ZCB_DIFF = 2 };

struct ProblemConst {
    double kappa, theta, half_eps2, r0, dt, theta_dt, bound;
    double coef[kMaxTerms];   // term 2f: +coef*P(t,T), term 2f+1: -coef*P(t,T)
    int rule[6];
    int kind[6];
};

// Device status words per problem. A failing step sets fail_step (1-based);
// every later kernel of that problem returns immediately, mirroring the
// reference throwing out of douglas_step (solver.cpp:241-247).
struct DevStatus {
    int fail_step;
    int fail_code;                          // hjmsv_status of the failure
    unsigned long long pivot_key;           // (sweep<<50)|(line<<20)|row, first in loop order
    unsigned long long nonfinite_first;     // first flat index with !isfinite (solver.cpp:71)
    unsigned long long diverge_first;       // first flat index with |U| > bound (solver.cpp:73)
    unsigned long long maxdelta_bits;       // max |dU| of the latest step (solver.cpp:163-167)
};

struct BatchView {
    int P, nr, nv, ny;
    long long N;          // nr*nv*ny
    int S;                // steps in the march
    int y_order, r_order;
    double dxr, dxv, dxy;
    double* U;            // [P][N] level
    double* D;            // [P][N] delta / line workspace
    double* C;            // [P][N] Thomas c' scratch (strict sweeps)
    const double* axes;   // [P][axes_stride]: rz rj1 rj2 | vz vj1 vj2 | yz yj1 yj2 | a b
    int axes_stride;
    const ProblemConst* pc;
    const double* steps;  // [P][S][kStepStride]
    DevStatus* st;        // [P]
    const double* fast;   // [P][fast_stride] derived factor tables (FAST mode)
    int fast_stride;
    // time-dependent model functions (hjmsv_model::*_fn): the factor tables of
    // step s start fast_step doubles after step 0's (0: one table for every step)
    int fast_step;
    const double* ab;     // [P][S][2 nr] a_i, b_i of prepare(t_mid) per step, or null (constant: axes block)
    int apply_only;       // stage mode: D = F(U), Dirichlet nodes 0 (apply_operator)
    int dmask;            // bit f set when face f is Dirichlet (uniform across the batch)
    double* fb;           // [P][fb_stride] Dirichlet face values at t_next of the current step
    int fb_stride;        // 2ny (r faces) + 2nr (y faces) + 2 nr ny (v faces)
    double* fb_next;      // [P][fb_stride] the next step's values (filled by the last kernel of a step)
    int want_md;          // track max|dU| this step (the last step of a launched sequence)
    int dbg;              // diagnostic switches (HJMSV_DBG; 0 in production)
    // kernel timeline (profiling runs only, else null): per (step, kernel slot)
    // the earliest block start and the latest block end in %globaltimer ns, so
    // per-kernel durations are taken in the launch mode of the timed march
    unsigned long long* tl;
    // y-line LU of a constant model (the y-line matrices do not change between
    // steps): 1 / pivot of the reference's Thomas elimination (solver.cpp:42-50)
    // per node, [P][N] in pass B's warp-block order (fast_ylu_build), or null
    const double* ylu;
    // pass B: every CTA asks L2 for the dU1 rows of the plane pf_ahead planes on (the
    // plane its SM is likely to get next) while its own y phase runs; 0: off
    int pf_ahead;
    // pass A: the same for the U column of the CTA pf_ahead_a CTAs on, asked for
    // once this CTA's march has ended; 0: off
    int pf_ahead_a;
};
constexpr int kTlSlots = 5;  // 0 pass A / explicit, 1 r-lines, 2 pass B / v-lines, 3 y-lines, 4 faces

// fast_step flags: the first step of a launched sequence fills its own face
// buffer; the last one records max|dU| for the report (solver.cpp:163-167).
enum StepFlags : int { STEP_FIRST = 1, STEP_LAST = 2 };

inline int axes_stride(int nr, int nv, int ny) { return 5 * nr + 3 * nv + 3 * ny; }

// FAST-mode factor tables per problem (host-built, lowering.cpp), array-of-
// structs per node index so one base address serves every field. They hold the
// separable pieces of g1..g6 (discretization.cpp:56-72) with the stencil 1/dx
// factors folded in, plus the v-line LU, which depends on j only:
//   g1/dxr^2 = G1[i] v_j      g4/(2dxr) = c4 G4C[i] + G4P[i] + G4Q[i] y_k + G4V[i] v_j
//   g3/(4 dxr dxv) = G3[i] G3V[j]     g2/dxv^2 = G2[j]     g5/(2dxv) = G5[j]
//   g6/(2dxy) = A[i] v_j S6[k] + T6[k]                   reaction = REACT[i]
// v-line LU: dp_j = RP_j x_j + B_j dp_{j-1} (B = -RP L), x_j = dp_j + E_j x_{j+1}
// (E = -CP), with in-segment products BF/BB for the segmented v-solve.
constexpr int kFR = 8;
enum FastR : int { FR_G1 = 0, FR_G4C, FR_G4P, FR_G4Q, FR_G4V, FR_G3, FR_REACT, FR_A };
constexpr int kFV = 10;
enum FastV : int { FV_V = 0, FV_G2, FV_G5, FV_G3, FV_B, FV_E, FV_RP, FV_BF, FV_BB, FV_PAD };
constexpr int kFY = 4;
enum FastY : int { FY_S6 = 0, FY_T6, FY_Y, FY_PAD };
constexpr int kSegV = 16;  // rows per segment of the segmented v-solve
inline int fast_table_stride(int nr, int nv, int ny) { return kFR * nr + kFV * nv + kFY * ny; }

// Terminal level built on the device (FAST mode): ZCB = 1 everywhere; caplet =
// caplet_payoff (model.cpp:105-112) with smooth_terminal's cell averages
// (solver.cpp:180-211), from per-problem scalars of the host curve.
enum TermKind : int { TERM_HOST = 0, TERM_ONES = 1, TERM_CAPLET = 2 };
struct TermParam {
    int kind;
    int m;            // samples per axis (1 without smoothing)
    double r0;
    double f_t;       // f(0, T)
    double accrual;   // 1 + (T_M - T) K (model.hpp:55)
    double ratio;     // p(0, T_M) / p(0, T)
    double g;         // g_factor(T_M - T, kappa)
};

// Per-kernel hook for the live profiler: called after each launch with the
// kernel's index, name and ALGORITHMIC bytes per grid point of that launch.
struct LaunchHook {
    void (*after)(void* ctx, int idx, const char* name, double alg_bytes_per_point) = nullptr;
    void* ctx = nullptr;
};

// Kernel launch entry points (kernels_strict.cu / kernels_fast.cu).
void strict_step(const BatchView& v, int s, cudaStream_t stream, long long* launches,
                 const LaunchHook* hook = nullptr);
void fast_step(const BatchView& v, int s, cudaStream_t stream, long long* launches,
               const LaunchHook* hook = nullptr, int flags = STEP_FIRST | STEP_LAST);
// explicit stage alone (stage test of apply_operator / dU0)
void strict_explicit(const BatchView& v, int s, cudaStream_t stream);
void fast_explicit(const BatchView& v, int s, cudaStream_t stream);
int fast_stride(int nr, int nv, int ny);
// y-line pivots of a constant-model batch for pass B (exact two-pass shapes only):
// fills ylu [P][N] and sets flag[p] != 0 where a pivot vanished or left the
// finite range; false when the shape has no table-driven pass B
bool fast_ylu_supported(const BatchView& v);
void fast_ylu_build(const BatchView& v, double* ylu, int* flag, cudaStream_t stream);
bool fast_supported(int nr, int nv, int ny);
void reset_status(const BatchView& v, cudaStream_t stream);
// Monte Carlo validator (kernels_mc.cu): run_path's constants (montecarlo.cpp:38-79)
struct McParams {
    long long n_paths;
    int n_steps;
    int full_truncation;
    unsigned long long seed;
    double dt, sqrt_dt, decay_y, decay_h, f0;
    double kappa, theta, rho, sq1mr2;
    int caplet;
    double accrual, ratio, g;
};
// partial[2*b] = sum, partial[2*b+1] = sum of squares of block b's path samples;
// steps: per step (f(0, (s+1) dt), lambda, gamma, eps)
void mc_simulate(const McParams& mp, const double* steps, double* partial, int blocks,
                 cudaStream_t stream);
// extract_greeks of problem p's level (instruments.cpp:90-132); scale: rho /= r0
// as finish() does (instruments.cpp:150-152). rho / vega may be null.
void greeks(const BatchView& v, int p, int scale, double r0, double* rho, double* vega,
            cudaStream_t stream);
// write_surface_csv's rows at slice k (job.cpp:300-310): [nr*nv][5]
void surface(const BatchView& v, int p, int k, double r0, const double* rho, const double* vega,
             double* out, cudaStream_t stream);
// U0[p] = terminal level of problem p for every p with tp[p].kind != TERM_HOST
void device_terminal(const BatchView& v, const TermParam* tp, const int* host_kinds, double* U0,
                     cudaStream_t stream);
// trilinear readout: out[p] = sum_q w[p*8+q] * U[p][idx[p*8+q]] (instruments.cpp:71-88)
void gather_spot(const BatchView& v, const long long* idx, const double* w, double* out,
                 cudaStream_t stream);
// FAST partition-method lines (n <= 512): pass A's r-line solver, or with
// twisted pass B's y-line solver (kernels_fast.cu k_thomas_fast)
void fast_thomas_batch(int n, int count, const double* lower, const double* diag, const double* upper,
                       const double* super2, double* rhs, int* fail_row, bool twisted, cudaStream_t stream);
// standalone batched Thomas (parity stage test of solver.cpp:22-57)
void thomas_batch(int n, int count, const double* lower, const double* diag, const double* upper,
                  const double* super2, double* rhs, double* scratch, int* fail_row, int fast,
                  cudaStream_t stream);

}  // namespace hjmsv_b200
