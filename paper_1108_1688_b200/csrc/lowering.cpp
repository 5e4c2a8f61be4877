// lowering.cpp — host lowering of a pricing problem to device tables.
#include "lowering.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <thread>

namespace hjmsv_b200 {

hjmsv_solver_config default_config() {
    hjmsv_solver_config c;
    c.theta_cn = 0.5;  // SolverConfig defaults, solver.hpp:10-20
    c.steps_per_year = 12;
    c.y_boundary_order = 2;
    c.r_boundary_order = 2;
    c.smoothing = 1;
    c.smoothing_subsamples = 3;
    c.divergence_bound = 1e6;
    return c;
}

namespace {

void validate_config(const hjmsv_solver_config& c) {  // solver.cpp:10-20
    if (c.theta_cn < 0.0 || c.theta_cn > 1.0)
        throw std::invalid_argument("theta_cn must lie in [0,1]");
    if (c.steps_per_year < 1) throw std::invalid_argument("steps_per_year must be >= 1");
    if (c.y_boundary_order != 1 && c.y_boundary_order != 2)
        throw std::invalid_argument("y_boundary_order must be 1 or 2");
    if (c.smoothing_subsamples < 1)
        throw std::invalid_argument("smoothing_subsamples must be >= 1");
    if (c.divergence_bound <= 0.0)
        throw std::invalid_argument("divergence_bound must be positive");
}

void validate_model(const hjmsv_model& m) {  // model.cpp:25-37
    if (m.kappa < 0.0) throw std::invalid_argument("kappa must be nonnegative");
    if (m.theta < 0.0) throw std::invalid_argument("theta must be nonnegative");
    if (m.rho < -1.0 || m.rho > 1.0) throw std::invalid_argument("rho must lie in [-1,1]");
    // a model function is checked at t = 0 only, as ModelParams::validate does
    const double g = m.gamma_fn ? m.gamma_fn(0.0, m.fn_user) : m.gamma;
    if (g <= 0.0 || g > 1.0) throw std::invalid_argument("gamma must lie in (0,1]");
}

Axis import_axis(const hjmsv_axis& a) {
    if (a.n != 1 && a.n < 3) throw std::invalid_argument("axis needs at least 3 nodes");
    if (!a.z || !a.j1 || !a.j2) throw std::invalid_argument("axis arrays must be set");
    Axis x;
    x.n = a.n;
    x.map = a.map;
    x.z.assign(a.z, a.z + a.n);
    x.j1.assign(a.j1, a.j1 + a.n);
    x.j2.assign(a.j2, a.j2 + a.n);
    x.center = a.center;
    x.alpha = a.alpha;
    x.z0 = a.z0;
    x.z_inf = a.z_inf;
    x.c1 = a.c1;
    x.c2 = a.c2;
    return x;
}

Curve import_curve(const hjmsv_curve& c) {
    if (c.kind == HJMSV_CURVE_FLAT) return Curve::flat(c.flat_base);
    if (c.n_nodes > 0 && (!c.maturities || !c.discounts))
        throw std::invalid_argument("curve arrays must be set");
    std::vector<std::pair<double, double>> nodes;
    nodes.reserve(c.n_nodes);
    for (int i = 0; i < c.n_nodes; ++i) nodes.emplace_back(c.maturities[i], c.discounts[i]);
    return Curve::from_nodes(std::move(nodes));
}

// smooth_terminal's per-axis cell samples (solver.cpp:184-194)
std::vector<double> cell_samples(const Axis& a, int i, int m) {
    if (a.n == 1 || i == 0 || i == a.n - 1) return {a.z[i]};
    const double lo = a.z[i] - 0.5 * (a.z[i] - a.z[i - 1]);
    const double hi = a.z[i] + 0.5 * (a.z[i + 1] - a.z[i]);
    const double w = (hi - lo) / m;
    std::vector<double> out(m);
    for (int q = 0; q < m; ++q) out[q] = lo + (q + 0.5) * w;
    return out;
}

template <class F>
void parallel_for(int n, F&& f) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int workers = static_cast<int>(std::min<unsigned>(hw, static_cast<unsigned>(n)));
    if (workers <= 1 || n < 8) {
        for (int i = 0; i < n; ++i) f(i);
        return;
    }
    std::vector<std::thread> pool;
    for (int w = 0; w < workers; ++w)
        pool.emplace_back([&, w] {
            for (int i = w; i < n; i += workers) f(i);
        });
    for (auto& t : pool) t.join();
}

// Caplet terminal condition (instruments.cpp:227-230 -> caplet_payoff,
// model.cpp:105-112) with optional cell-average smoothing (solver.cpp:180-211).
// The payoff does not depend on zv, so it is tabulated once per (r-sample,
// y-sample) and summed in the reference's (zr, zv, zy) loop order: the
// accumulation is bit-identical to 27 direct payoff calls per node.
void caplet_terminal(Lowered& L, const hjmsv_problem& p, const hjmsv_solver_config& cfg) {
    const double r0 = L.r0, expiry = p.maturity, payment = p.payment;
    const double accrual = 1.0 + (payment - expiry) * p.strike;  // model.hpp:55
    const double f_t = L.curve.forward(expiry);
    const double kappa = p.model.kappa;
    auto payoff = [&](double zr, double zy) {
        const double tr = r0 * zr, ty = r0 * r0 * zy;
        const double x = tr - f_t;
        const double pb = zcb_closed_form(expiry, payment, x, ty, L.curve, kappa);
        const double value = 1.0 - accrual * pb;
        return value > 0.0 ? value : 0.0;
    };
    const int nr = L.nr, nv = L.nv, ny = L.ny;
    const int m = cfg.smoothing ? cfg.smoothing_subsamples : 1;
    L.init.assign(static_cast<size_t>(nr) * nv * ny, 0.0);
    if (!cfg.smoothing) {
        parallel_for(nr, [&](int i) {
            for (int j = 0; j < nv; ++j)
                for (int k = 0; k < ny; ++k)
                    L.init[(static_cast<size_t>(i) * nv + j) * ny + k] = payoff(L.r.z[i], L.y.z[k]);
        });
        return;
    }
    std::vector<std::vector<double>> sy(ny);
    for (int k = 0; k < ny; ++k) sy[k] = cell_samples(L.y, k, m);
    std::vector<int> nsv(nv);
    for (int j = 0; j < nv; ++j) nsv[j] = static_cast<int>(cell_samples(L.v, j, m).size());
    parallel_for(nr, [&](int i) {
        const std::vector<double> sr = cell_samples(L.r, i, m);
        const int nsr = static_cast<int>(sr.size());
        // pv[(qr*ny + k)*m + qy]
        std::vector<double> pv(static_cast<size_t>(nsr) * ny * m);
        for (int qr = 0; qr < nsr; ++qr)
            for (int k = 0; k < ny; ++k)
                for (size_t qy = 0; qy < sy[k].size(); ++qy)
                    pv[(static_cast<size_t>(qr) * ny + k) * m + qy] = payoff(sr[qr], sy[k][qy]);
        for (int j = 0; j < nv; ++j)
            for (int k = 0; k < ny; ++k) {
                const int nsy = static_cast<int>(sy[k].size());
                double acc = 0.0;
                for (int qr = 0; qr < nsr; ++qr)
                    for (int qv = 0; qv < nsv[j]; ++qv)
                        for (int qy = 0; qy < nsy; ++qy)
                            acc += pv[(static_cast<size_t>(qr) * ny + k) * m + qy];
                const size_t count = static_cast<size_t>(nsr) * nsv[j] * nsy;
                L.init[(static_cast<size_t>(i) * nv + j) * ny + k] = acc / count;
            }
    });
}

}  // namespace

bool time_dependent(const hjmsv_model& m) { return m.lambda_fn || m.gamma_fn || m.eps_fn; }

ModelAt model_at(const hjmsv_model& m, double t) {
    // HjmCoefficientField::prepare's calls, in its order (discretization.cpp:41-43)
    ModelAt x;
    x.lambda = m.lambda_fn ? m.lambda_fn(t, m.fn_user) : m.lambda;
    x.gamma = m.gamma_fn ? m.gamma_fn(t, m.fn_user) : m.gamma;
    x.eps = m.eps_fn ? m.eps_fn(t, m.fn_user) : m.eps;
    return x;
}

void prepare_ab(const Lowered& L, const ModelAt& x, double* a, double* b) {
    // discretization.cpp:48-53, same operations
    const double r0_pow = std::pow(L.r0, x.gamma - 1.0);
    for (int i = 0; i < L.nr; ++i) {
        const double rp = L.r.z[i] > 0.0 ? std::pow(L.r.z[i], x.gamma) * r0_pow : 0.0;
        a[i] = 0.5 * x.lambda * x.lambda * rp * rp;
        b[i] = x.lambda * x.eps * L.model.rho * rp;
    }
}

void build_model_steps(Lowered& L) {
    const int S = static_cast<int>(L.steps.size() / kStepStride);
    if (!L.timedep) {
        for (int s = 0; s < S; ++s) L.steps[static_cast<size_t>(s) * kStepStride + ST_HEPS2] = L.pc.half_eps2;
        L.ab_steps.clear();
        return;
    }
    const int nr = L.nr;
    L.ab_steps.assign(static_cast<size_t>(S) * 2 * nr, 0.0);
    for (int s = 0; s < S; ++s) {
        double* e = &L.steps[static_cast<size_t>(s) * kStepStride];
        // prepare(t_mid) (solver.cpp:96): the model functions at the half level
        const ModelAt x = model_at(L.model, e[ST_TMID]);
        e[ST_HEPS2] = 0.5 * x.eps * x.eps;
        double* ab = &L.ab_steps[static_cast<size_t>(s) * 2 * nr];
        prepare_ab(L, x, ab, ab + nr);
    }
}

std::vector<double> march_levels(double maturity, int n_steps, int time_levels) {
    const double dt = maturity / n_steps;
    std::vector<double> t(n_steps);
    double t_from = maturity;
    for (int s = 0; s < n_steps; ++s) {
        if (time_levels == HJMSV_TIME_INDEXED) t_from = maturity - s * dt;
        t[s] = t_from;
        double t_next = t_from - dt;  // solver.cpp:85-87
        if (std::abs(t_next) < 1e-12 * dt) t_next = 0.0;
        t_from = t_next;
    }
    return t;
}

void build_step_table(Lowered& L, const std::vector<double>& t_from, double dt, bool faces) {
    const int S = static_cast<int>(t_from.size());
    L.steps.assign(static_cast<size_t>(S) * kStepStride, 0.0);
    const double kappa = L.pc.kappa;
    for (int s = 0; s < S; ++s) {
        double* e = &L.steps[static_cast<size_t>(s) * kStepStride];
        const double tf = t_from[s];
        double t_next = tf - dt;  // solver.cpp:85-88
        if (std::abs(t_next) < 1e-12 * dt) t_next = 0.0;
        const double t_mid = tf - 0.5 * dt;
        // HjmCoefficientField::prepare(t_mid) (discretization.cpp:47)
        e[ST_C4] = (L.curve.forward_slope(t_mid) + kappa * L.curve.forward(t_mid)) / L.r0;
        e[ST_FNEXT] = L.curve.forward(t_next);
        e[ST_TNEXT] = t_next;
        e[ST_TMID] = t_mid;
        // zcb_closed_form(t_next, T_x, ...) scalars, evaluated in the
        // reference's order so domain errors surface with its messages
        for (int f = 0; f < 6 && faces; ++f) {
            if (L.pc.rule[f] != RULE_DIRICHLET || L.pc.kind[f] == VAL_ZERO) continue;
            const int nterm = L.pc.kind[f] == VAL_ZCB_DIFF ? 2 : 1;
            for (int q = 0; q < nterm; ++q) {
                const int slot = 2 * f + q;
                const double mat = L.term_t[slot];
                if (mat < t_next)
                    throw std::domain_error("zcb_closed_form: maturity before valuation");
                e[ST_G + slot] = g_factor(mat - t_next, kappa);
                e[ST_RATIO + slot] = L.curve.discount(mat) / L.curve.discount(t_next);
            }
        }
    }
}

void locate_point(const Lowered& L, double zr, double zv, double zy, long long idx[8],
                  double w[8]) {
    struct Cell {
        int lo;
        double w;
    };
    auto locate = [](const Axis& a, double z) -> Cell {  // instruments.cpp:59-66
        if (a.n == 1) return {0, 0.0};
        const double x = physical_to_computational(a, z);
        const double s = x * (a.n - 1);
        const int lo = std::min(static_cast<int>(s), a.n - 2);
        return {lo, s - lo};
    };
    const Cell cr = locate(L.r, zr), cv = locate(L.v, zv), cy = locate(L.y, zy);
    int c = 0;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int d = 0; d < 2; ++d, ++c) {
                w[c] = (a ? cr.w : 1.0 - cr.w) * (b ? cv.w : 1.0 - cv.w) * (d ? cy.w : 1.0 - cy.w);
                const long long i = std::min(cr.lo + a, L.nr - 1);
                const long long j = std::min(cv.lo + b, L.nv - 1);
                const long long k = std::min(cy.lo + d, L.ny - 1);
                idx[c] = (i * L.nv + j) * L.ny + k;
            }
}

Lowered lower_problem(const hjmsv_problem& p, const hjmsv_solver_config& cfg, int init_mode) {
    validate_config(cfg);
    if (p.maturity <= 0.0) throw std::invalid_argument("run: maturity must be positive");
    if (p.instrument == HJMSV_INSTRUMENT_CAPLET) {  // CapletSpec::validate, model.cpp:35-39
        if (p.maturity <= 0.0) throw std::invalid_argument("caplet expiry must be positive");
        if (p.payment <= p.maturity)
            throw std::invalid_argument("caplet payment date must exceed expiry");
        if (p.strike <= 0.0) throw std::invalid_argument("caplet strike must be positive");
    } else if (p.instrument != HJMSV_INSTRUMENT_ZCB && p.instrument != HJMSV_INSTRUMENT_CUSTOM) {
        throw std::invalid_argument("unknown instrument kind");
    }
    if (p.time_levels != HJMSV_TIME_REFERENCE && p.time_levels != HJMSV_TIME_INDEXED)
        throw std::invalid_argument("unknown time-level mode");
    validate_model(p.model);

    Lowered L;
    L.r = import_axis(p.r);
    L.v = import_axis(p.v);
    L.y = import_axis(p.y);
    L.nr = L.r.n;
    L.nv = L.v.n;
    L.ny = L.y.n;
    L.curve = import_curve(p.curve);
    L.r0 = p.r0;
    L.maturity = p.maturity;
    if (L.r0 <= 0.0) throw std::invalid_argument("rate scale r0 must be positive");

    // boundary description (BoundarySpec::zcb / ::caplet, discretization.cpp:74-120)
    ProblemConst& pc = L.pc;
    for (int q = 0; q < kMaxTerms; ++q) pc.coef[q] = 0.0;
    for (double& t : L.term_t) t = 0.0;
    if (p.instrument == HJMSV_INSTRUMENT_CUSTOM) {
        for (int f = 0; f < 6; ++f) {
            pc.rule[f] = p.face_rule[f];
            if (pc.rule[f] < 0 || pc.rule[f] > 2) throw std::invalid_argument("unknown face rule");
            const hjmsv_face_value& fv = p.face_value[f];
            pc.kind[f] = fv.kind;
            if (fv.kind < 0 || fv.kind > 2) throw std::invalid_argument("unknown face value kind");
            pc.coef[2 * f] = fv.a;
            pc.coef[2 * f + 1] = fv.b;
            L.term_t[2 * f] = fv.t1;
            L.term_t[2 * f + 1] = fv.t2;
        }
    } else {
        const int rules[6] = {RULE_DEGENERATE, RULE_DIRICHLET, RULE_DEGENERATE,
                              RULE_DIRICHLET,  RULE_ONE_SIDED, RULE_DIRICHLET};
        for (int f = 0; f < 6; ++f) {
            pc.rule[f] = rules[f];
            pc.kind[f] = VAL_ZERO;
        }
        if (p.instrument == HJMSV_INSTRUMENT_ZCB) {
            for (int f : {F_VMAX, F_YMAX}) {
                pc.kind[f] = VAL_ZCB;
                pc.coef[2 * f] = 1.0;
                L.term_t[2 * f] = p.maturity;
            }
        } else {
            pc.kind[F_VMAX] = VAL_ZCB_DIFF;
            pc.coef[2 * F_VMAX] = 1.0;
            pc.coef[2 * F_VMAX + 1] = 1.0;
            L.term_t[2 * F_VMAX] = p.maturity;
            L.term_t[2 * F_VMAX + 1] = p.payment;
        }
    }
    // BoundarySpec::validate (discretization.cpp:130-137) + SpatialOperator checks
    for (int f : {F_RMAX, F_VMAX, F_YMAX})
        if (pc.rule[f] != RULE_DIRICHLET)
            throw std::invalid_argument("upper faces must carry Dirichlet rules");
    if (cfg.r_boundary_order != 1 && cfg.r_boundary_order != 2)
        throw std::invalid_argument("r boundary order must be 1 or 2");
    if (L.ny > 1 && L.ny < 3) throw std::invalid_argument("y axis needs at least 3 nodes");

    // constant model: HjmCoefficientField::prepare caches (discretization.cpp:40-54)
    const hjmsv_model& m = p.model;
    pc.kappa = m.kappa;
    pc.theta = m.theta;
    pc.half_eps2 = 0.5 * m.eps * m.eps;
    pc.r0 = p.r0;
    pc.bound = cfg.divergence_bound;
    L.n_steps = p.n_steps > 0
                    ? p.n_steps
                    : std::max(1, static_cast<int>(std::lround(cfg.steps_per_year * p.maturity)));
    L.dt = p.maturity / L.n_steps;
    pc.dt = L.dt;
    pc.theta_dt = cfg.theta_cn * L.dt;

    const int nr = L.nr, nv = L.nv, ny = L.ny;
    L.axes.assign(axes_stride(nr, nv, ny), 0.0);
    double* t = L.axes.data();
    auto put = [&](const std::vector<double>& src) {
        std::copy(src.begin(), src.end(), t);
        t += src.size();
    };
    put(L.r.z); put(L.r.j1); put(L.r.j2);
    put(L.v.z); put(L.v.j1); put(L.v.j2);
    put(L.y.z); put(L.y.j1); put(L.y.j2);
    L.model = m;
    L.timedep = time_dependent(m);
    // constant model: prepare's a_i, b_i once (a time-dependent one gets them per step)
    if (!L.timedep) prepare_ab(L, model_at(m, 0.0), t, t + nr);

    build_step_table(L, march_levels(p.maturity, L.n_steps, p.time_levels), L.dt, true);
    build_model_steps(L);

    // price readout at natural_spot (instruments.cpp:50-52, 145-149)
    const double f0 = L.curve.forward(0.0);
    locate_point(L, f0 / p.r0, 1.0, 0.0 / (p.r0 * p.r0), L.spot_idx, L.spot_w);

    if (init_mode == INIT_DEVICE && !p.initial_grid &&
        (p.instrument == HJMSV_INSTRUMENT_ZCB || p.instrument == HJMSV_INSTRUMENT_CAPLET)) {
        TermParam& tp = L.term;
        tp.m = cfg.smoothing ? cfg.smoothing_subsamples : 1;
        tp.r0 = p.r0;
        if (p.instrument == HJMSV_INSTRUMENT_ZCB) {
            tp.kind = TERM_ONES;
        } else {  // the scalars caplet_terminal's payoff closes over
            tp.kind = TERM_CAPLET;
            tp.f_t = L.curve.forward(p.maturity);
            tp.accrual = 1.0 + (p.payment - p.maturity) * p.strike;
            tp.ratio = L.curve.discount(p.payment) / L.curve.discount(p.maturity);
            tp.g = g_factor(p.payment - p.maturity, p.model.kappa);
        }
    } else if (init_mode != INIT_NONE) {
        const size_t N = static_cast<size_t>(nr) * nv * ny;
        if (p.initial_grid) {
            L.init.assign(p.initial_grid, p.initial_grid + N);
        } else if (p.instrument == HJMSV_INSTRUMENT_ZCB) {
            L.init.assign(N, 1.0);  // terminal 1; its cell average is exactly 1
        } else if (p.instrument == HJMSV_INSTRUMENT_CAPLET) {
            caplet_terminal(L, p, cfg);
        } else {
            throw std::invalid_argument("custom instrument needs an initial grid");
        }
    }
    return L;
}

std::vector<double> build_fast_tables(const Lowered& L, const hjmsv_solver_config& cfg,
                                      double th, int step) {
    const int nr = L.nr, nv = L.nv, ny = L.ny;
    std::vector<double> t(fast_table_stride(nr, nv, ny), 0.0);
    double* R = t.data();
    double* V = R + kFR * nr;
    double* Y = V + kFV * nv;
    const double dxr = L.r.dx(), dxv = L.v.dx(), dxy = L.y.dx();
    const double inv_dxr2 = nr > 1 ? 1.0 / (dxr * dxr) : 0.0;
    const double inv_2dxr = nr > 1 ? 0.5 / dxr : 0.0;
    const double inv_dxv2 = nv > 1 ? 1.0 / (dxv * dxv) : 0.0;
    const double inv_2dxv = nv > 1 ? 0.5 / dxv : 0.0;
    const double inv_2dxy = ny > 1 ? 0.5 / dxy : 0.0;
    // the cross term needs both axes resolved (apply_operator applies it only for
    // 0 < i < nr-1, 0 < j < nv-1, discretization.cpp:357-361); a singleton v axis has none
    const double inv_cross = (nr > 1 && nv > 1) ? 0.25 / (dxr * dxv) : 0.0;
    const ProblemConst& pc = L.pc;
    // prepare(t_mid)'s a_i, b_i and eps^2/2: the constants, or step `step`'s values
    const bool per_step = L.timedep && step >= 0;
    const double* a = per_step ? &L.ab_steps[static_cast<size_t>(step) * 2 * nr]
                               : L.axes.data() + 3 * nr + 3 * nv + 3 * ny;
    const double* b = a + nr;
    const double half_eps2 = per_step ? L.steps[static_cast<size_t>(step) * kStepStride + ST_HEPS2]
                                      : pc.half_eps2;
    for (int i = 0; i < nr; ++i) {
        const double jr = L.r.j1[i];
        double* e = R + kFR * i;
        e[FR_G1] = a[i] / (jr * jr) * inv_dxr2;
        e[FR_G4C] = inv_2dxr / jr;
        e[FR_G4P] = -pc.kappa * L.r.z[i] / jr * inv_2dxr;
        e[FR_G4Q] = pc.r0 / jr * inv_2dxr;
        e[FR_G4V] = -a[i] * L.r.j2[i] / (jr * jr * jr) * inv_2dxr;
        e[FR_G3] = b[i] / jr * inv_cross;
        e[FR_REACT] = L.r.z[i] * pc.r0;
        e[FR_A] = a[i];
    }
    for (int j = 0; j < nv; ++j) {
        const double v = L.v.z[j], jv = L.v.j1[j];
        double* e = V + kFV * j;
        e[FV_V] = v;
        e[FV_G2] = half_eps2 * v / (jv * jv) * inv_dxv2;
        e[FV_G5] = (pc.theta * (1.0 - v) / jv - half_eps2 * v * L.v.j2[j] / (jv * jv * jv)) *
                   inv_2dxv;
        e[FV_G3] = v / jv;
    }
    // v-line LU (rows of assemble_line_v, discretization.cpp:232-259, depend on j only)
    if (nv > 1) {
        double cp_prev = 0.0;
        for (int j = 0; j < nv; ++j) {
            double* e = V + kFV * j;
            double l = 0.0, d = 1.0, u = 0.0;
            const bool dir = (j == 0 && pc.rule[F_VMIN] == RULE_DIRICHLET) ||
                             (j == nv - 1 && pc.rule[F_VMAX] == RULE_DIRICHLET);
            if (!dir) {
                const double g5h = e[FV_G5];
                if (j == 0) {
                    d = 1.0 + th * 2.0 * g5h;
                    u = -th * 2.0 * g5h;
                } else {
                    const double w2 = th * e[FV_G2], w1 = th * g5h;
                    l = w1 - w2;
                    d = 1.0 + 2.0 * w2;
                    u = -(w2 + w1);
                }
            }
            const double piv = j == 0 ? d : d - l * cp_prev;
            const double rp = std::abs(piv) < 1e-300 ? std::nan("") : 1.0 / piv;
            cp_prev = u * rp;
            e[FV_B] = -rp * l;
            e[FV_E] = -cp_prev;
            e[FV_RP] = rp;
        }
        // in-segment products for the segmented solve
        for (int s0 = 0; s0 < nv; s0 += kSegV) {
            const int s1 = std::min(nv, s0 + kSegV) - 1;
            double pf = 1.0;
            for (int j = s0; j <= s1; ++j) {
                pf *= V[kFV * j + FV_B];
                V[kFV * j + FV_BF] = pf;
            }
            double pb = 1.0;
            for (int j = s1; j >= s0; --j) {
                pb *= V[kFV * j + FV_E];
                V[kFV * j + FV_BB] = pb;
            }
        }
    }
    for (int k = 0; k < ny; ++k) {
        const double jy = L.y.j1[k];
        double* e = Y + kFY * k;
        e[FY_S6] = 2.0 * inv_2dxy / jy;
        e[FY_T6] = -2.0 * pc.kappa * L.y.z[k] / jy * inv_2dxy;
        e[FY_Y] = L.y.z[k];
    }
    (void)cfg;
    return t;
}

McSetup lower_mc(const hjmsv_problem& p, const hjmsv_mc_config& c) {
    validate_model(p.model);  // simulate(): params.validate(), montecarlo.cpp:86-91
    if (c.n_paths < 1) throw std::invalid_argument("n_paths must be >= 1");
    if (c.steps_per_year < 1) throw std::invalid_argument("mc steps_per_year must be >= 1");
    McSetup m;
    const Curve curve = import_curve(p.curve);
    if (p.instrument == HJMSV_INSTRUMENT_CAPLET) {  // CapletSpec::validate, model.cpp:35-39
        if (p.maturity <= 0.0) throw std::invalid_argument("caplet expiry must be positive");
        if (p.payment <= p.maturity)
            throw std::invalid_argument("caplet payment date must exceed expiry");
        if (p.strike <= 0.0) throw std::invalid_argument("caplet strike must be positive");
        m.caplet = 1;
        m.accrual = 1.0 + (p.payment - p.maturity) * p.strike;  // model.hpp:55
        m.ratio = curve.discount(p.payment) / curve.discount(p.maturity);
        m.g = g_factor(p.payment - p.maturity, p.model.kappa);
    } else if (p.instrument != HJMSV_INSTRUMENT_ZCB) {
        throw std::invalid_argument("Monte Carlo prices ZCB and caplet instruments");
    }
    if (p.maturity < 0.0) throw std::invalid_argument("horizon must be nonnegative");
    m.horizon = p.maturity;
    m.f0 = curve.forward(0.0);
    if (p.maturity == 0.0) return m;
    m.n_steps = std::max(1, static_cast<int>(std::lround(c.steps_per_year * p.maturity)));
    m.dt = p.maturity / m.n_steps;  // run_path, montecarlo.cpp:44-48
    m.sqrt_dt = std::sqrt(m.dt);
    m.decay_y = std::exp(-2.0 * p.model.kappa * m.dt);
    m.decay_h = std::exp(-p.model.kappa * m.dt);
    m.steps.resize(4 * static_cast<size_t>(m.n_steps));
    for (int s = 0; s < m.n_steps; ++s) {
        // run_path's per-step model functions at t = s dt (montecarlo.cpp:54-58)
        const ModelAt x = model_at(p.model, s * m.dt);
        m.steps[4 * s] = curve.forward(s * m.dt + m.dt);
        m.steps[4 * s + 1] = x.lambda;
        m.steps[4 * s + 2] = x.gamma;
        m.steps[4 * s + 3] = x.eps;
    }
    return m;
}

}  // namespace hjmsv_b200
