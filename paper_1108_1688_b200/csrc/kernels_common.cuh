// kernels_common.cuh — device helpers shared by the STRICT and FAST kernels:
// per-problem table views, the reference's Dirichlet rules/precedence and the
// closed-form face values.
#pragma once

#include <cmath>

#include "device_types.hpp"
#include "hjmsv_b200.h"

namespace hjmsv_b200 {
namespace dev {

struct Tab {
    const double *rz, *rj1, *rj2, *vz, *vj1, *vj2, *yz, *yj1, *yj2, *a, *b;
    double heps2;  // eps(t_mid)^2 / 2 of the step (HjmCoefficientField::half_eps2_)
};

// the axes of problem p and the a_i, b_i of prepare(t_mid) at step s
// (discretization.cpp:40-54): the axes block for constant models, the per-step
// block for time-dependent model functions
__device__ __forceinline__ Tab tables(const BatchView& v, int p, int s) {
    const double* t = v.axes + static_cast<size_t>(p) * v.axes_stride;
    Tab x;
    x.rz = t;
    x.rj1 = t + v.nr;
    x.rj2 = t + 2 * v.nr;
    t += 3 * v.nr;
    x.vz = t;
    x.vj1 = t + v.nv;
    x.vj2 = t + 2 * v.nv;
    t += 3 * v.nv;
    x.yz = t;
    x.yj1 = t + v.ny;
    x.yj2 = t + 2 * v.ny;
    t += 3 * v.ny;
    x.a = v.ab ? v.ab + (static_cast<size_t>(p) * v.S + s) * 2 * v.nr : t;
    x.b = x.a + v.nr;
    x.heps2 = v.steps[(static_cast<size_t>(p) * v.S + s) * kStepStride + ST_HEPS2];
    return x;
}

// SpatialOperator::is_dirichlet (discretization.cpp:153-170)
__device__ __forceinline__ bool is_dirichlet(const BatchView& v, const ProblemConst& pc, int i,
                                             int j, int k) {
    if (v.nr > 1) {
        if (i == 0 && pc.rule[F_RMIN] == RULE_DIRICHLET) return true;
        if (i == v.nr - 1 && pc.rule[F_RMAX] == RULE_DIRICHLET) return true;
    }
    if (v.nv > 1) {
        if (j == 0 && pc.rule[F_VMIN] == RULE_DIRICHLET) return true;
        if (j == v.nv - 1 && pc.rule[F_VMAX] == RULE_DIRICHLET) return true;
    }
    if (v.ny > 1) {
        if (k == 0 && pc.rule[F_YMIN] == RULE_DIRICHLET) return true;
        if (k == v.ny - 1 && pc.rule[F_YMAX] == RULE_DIRICHLET) return true;
    }
    return false;
}

// dirichlet_value precedence r_max > y_max > v_max > r_min > y_min > v_min
// (discretization.cpp:172-192); -1 when the node is not Dirichlet.
__device__ __forceinline__ int dirichlet_face(const BatchView& v, const ProblemConst& pc, int i,
                                              int j, int k) {
    auto act = [&](int f, bool on) { return on && pc.rule[f] == RULE_DIRICHLET; };
    if (act(F_RMAX, v.nr > 1 && i == v.nr - 1)) return F_RMAX;
    if (act(F_YMAX, v.ny > 1 && k == v.ny - 1)) return F_YMAX;
    if (act(F_VMAX, v.nv > 1 && j == v.nv - 1)) return F_VMAX;
    if (act(F_RMIN, v.nr > 1 && i == 0)) return F_RMIN;
    if (act(F_YMIN, v.ny > 1 && k == 0)) return F_YMIN;
    if (act(F_VMIN, v.nv > 1 && j == 0)) return F_VMIN;
    return -1;
}

// closed-form face value: coef*P(t,T1) [- coef'*P(t,T2)], P = ratio*exp(-G x - G^2 y/2)
// with x = r0*zr - f(0,t), y = r0^2*zy (discretization.cpp:77-81,111-118; model.cpp:48-54)
__device__ __forceinline__ double face_value(const ProblemConst& pc, const double* step,
                                             const Tab& T, int face, int i, int k) {
    const int kind = pc.kind[face];
    if (kind == VAL_ZERO) return 0.0;
    const double x = pc.r0 * T.rz[i] - step[ST_FNEXT];
    const double y = pc.r0 * pc.r0 * T.yz[k];
    const int t0 = 2 * face;
    const double g1 = step[ST_G + t0];
    const double p1 = step[ST_RATIO + t0] * exp(-g1 * x - 0.5 * g1 * g1 * y);
    double val = pc.coef[t0] * p1;
    if (kind == VAL_ZCB_DIFF) {
        const double g2 = step[ST_G + t0 + 1];
        const double p2 = step[ST_RATIO + t0 + 1] * exp(-g2 * x - 0.5 * g2 * g2 * y);
        val = val - pc.coef[t0 + 1] * p2;
    }
    return val;
}

__device__ __forceinline__ const double* step_row(const BatchView& v, int p, int s) {
    return v.steps + (static_cast<size_t>(p) * v.S + s) * kStepStride;
}

// A problem stops at a failure recorded in an EARLIER step (the reference threw
// out of that douglas_step, solver.cpp:241-247). A failure recorded during the
// current step s (0-based; fail_step = s + 1) does not stop the other blocks of
// the step, so every singular pivot and guard hit of that step is recorded and
// the host picks the one the reference reports first (pivots before the guard,
// lowest index first; capi.cpp status_message). Values <= s were written by
// earlier launches, so all blocks of one launch (and of one cluster) agree.
__device__ __forceinline__ bool failed_before(const DevStatus& st, int s) {
    const int f = st.fail_step;
    return f != 0 && f <= s;
}

// kernel timeline (BatchView::tl): block start after the programmatic wait,
// block end after the block's last store (tl_end syncs the block, so every
// thread of the block must reach it; tl_end_thread records thread 0 only)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ bool tl_lead() { return threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0; }
__device__ __forceinline__ void tl_begin(const BatchView& v, int s, int slot) {
    if (v.tl && tl_lead()) atomicMin(v.tl + 2 * (static_cast<size_t>(s) * kTlSlots + slot), gtimer());
}
__device__ __forceinline__ void tl_end(const BatchView& v, int s, int slot) {
    if (v.tl) {
        __syncthreads();
        if (tl_lead()) atomicMax(v.tl + 2 * (static_cast<size_t>(s) * kTlSlots + slot) + 1, gtimer());
    }
}
__device__ __forceinline__ void tl_end_thread(const BatchView& v, int s, int slot) {
    if (v.tl && tl_lead()) atomicMax(v.tl + 2 * (static_cast<size_t>(s) * kTlSlots + slot) + 1, gtimer());
}

__device__ __forceinline__ void mark_fail(DevStatus& st, int step1, int code) {
    if (atomicCAS(&st.fail_step, 0, step1) == 0) st.fail_code = code;
}

}  // namespace dev
}  // namespace hjmsv_b200
