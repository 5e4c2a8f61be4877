// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (parity checker, CPU baseline).
//
// A thin C-ABI harness over the UNMODIFIED reference library (compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/). It
// translates the plain-data hjmsv_problem of include/hjmsv_b200.h into the
// reference's own types and calls only the reference's public API:
//   run()            solver.cpp:213-258      douglas_step()   solver.cpp:81-178
//   apply_operator   discretization.cpp:302-364  assemble_line_* :194-300
//   thomas_solve_inplace solver.cpp:22-57    smooth_terminal  solver.cpp:180-211
//   interpolate_at   instruments.cpp:71-88   caplet_ladder pattern instruments.cpp:238-266
// The one deviation from run(), used only when time_levels == HJMSV_TIME_INDEXED,
// is the parity harness of SURVEY.md §8c: grid.time = T - s*dt before step s.
//
// Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline arm
// may load this library. The product (paper_1108_1688_b200/) never links it.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "hjmsv/curve.hpp"
#include "hjmsv/discretization.hpp"
#include "hjmsv/instruments.hpp"
#include "hjmsv/mesh.hpp"
#include "hjmsv/model.hpp"
#include "hjmsv/montecarlo.hpp"
#include "hjmsv/solver.hpp"
#include "hjmsv_b200.h"

using namespace hjmsv;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return HJMSV_OK;
    } catch (const std::invalid_argument& e) {
        return fail(HJMSV_INVALID_ARGUMENT, e.what());
    } catch (const std::domain_error& e) {
        return fail(HJMSV_DOMAIN, e.what());
    } catch (const std::logic_error& e) {
        return fail(HJMSV_LOGIC, e.what());
    } catch (const std::runtime_error& e) {
        const std::string m = e.what();
        if (m.find("singular pivot") != std::string::npos) return fail(HJMSV_SINGULAR_PIVOT, m);
        if (m.find("NaN/Inf") != std::string::npos) return fail(HJMSV_NONFINITE, m);
        if (m.find("divergence bound") != std::string::npos) return fail(HJMSV_DIVERGED, m);
        return fail(HJMSV_INVALID_ARGUMENT, m);
    } catch (const std::exception& e) {
        return fail(HJMSV_INVALID_ARGUMENT, e.what());
    }
}

Axis to_axis(const hjmsv_axis& a) {
    Axis ax;
    ax.n = a.n;
    ax.map = a.map == HJMSV_MAP_SINH     ? Axis::Map::sinh
             : a.map == HJMSV_MAP_LINEAR ? Axis::Map::linear
                                         : Axis::Map::singleton;
    ax.params = {a.center, a.alpha, a.z0, a.z_inf};
    ax.c1 = a.c1;
    ax.c2 = a.c2;
    ax.x.resize(a.n);
    for (int i = 0; i < a.n; ++i) ax.x[i] = a.n > 1 ? static_cast<double>(i) / (a.n - 1) : 0.0;
    ax.z.assign(a.z, a.z + a.n);
    ax.j1.assign(a.j1, a.j1 + a.n);
    ax.j2.assign(a.j2, a.j2 + a.n);
    return ax;
}

InitialCurve to_curve(const hjmsv_curve& c) {
    if (c.kind == HJMSV_CURVE_FLAT) return InitialCurve::flat(c.flat_base);
    std::vector<std::pair<double, double>> nodes;
    for (int i = 0; i < c.n_nodes; ++i) nodes.emplace_back(c.maturities[i], c.discounts[i]);
    return InitialCurve::from_nodes(std::move(nodes));
}

ModelParams to_model(const hjmsv_model& m) {
    if (!m.lambda_fn && !m.gamma_fn && !m.eps_fn)
        return ModelParams::constants(m.kappa, m.lambda, m.gamma, m.eps, m.theta, m.rho);
    // model functions of t (ModelParams::lambda_fn / gamma_fn / eps_fn, model.hpp:22-24)
    ModelParams p;
    p.kappa = m.kappa;
    p.theta = m.theta;
    p.rho = m.rho;
    auto fn = [&](hjmsv_time_fn f, double c) -> TimeFn {
        if (f) return [f, u = m.fn_user](double t) { return f(t, u); };
        return [c](double) { return c; };
    };
    p.lambda_fn = fn(m.lambda_fn, m.lambda);
    p.gamma_fn = fn(m.gamma_fn, m.gamma);
    p.eps_fn = fn(m.eps_fn, m.eps);
    p.validate();
    return p;
}

CapletSpec to_caplet(const hjmsv_problem& p) {
    CapletSpec s;
    s.expiry = p.maturity;
    s.payment = p.payment;
    s.strike = p.strike;
    return s;
}

BoundarySpec::ValueFn value_fn(const hjmsv_face_value& v, const InitialCurve& curve, double kappa,
                               double r0) {
    switch (v.kind) {
        case HJMSV_VALUE_ZERO:
            return [](double, double, double, double) { return 0.0; };
        case HJMSV_VALUE_ZCB: {
            const double a = v.a, t1 = v.t1;
            return [a, t1, curve, kappa, r0](double t, double zr, double, double zy) {
                double x = r0 * zr - curve.forward(t);
                return a * zcb_closed_form(t, t1, x, r0 * r0 * zy, curve, kappa);
            };
        }
        default: {
            const double a = v.a, t1 = v.t1, b = v.b, t2 = v.t2;
            return [a, t1, b, t2, curve, kappa, r0](double t, double zr, double, double zy) {
                double x = r0 * zr - curve.forward(t);
                double y = r0 * r0 * zy;
                return a * zcb_closed_form(t, t1, x, y, curve, kappa) -
                       b * zcb_closed_form(t, t2, x, y, curve, kappa);
            };
        }
    }
}

struct Built {
    PdeProblem problem;
    SolverConfig config;
};

SolverConfig to_config(const hjmsv_solver_config* c) {
    SolverConfig cfg;
    if (c) {
        cfg.theta_cn = c->theta_cn;
        cfg.steps_per_year = c->steps_per_year;
        cfg.y_boundary_order = c->y_boundary_order;
        cfg.r_boundary_order = c->r_boundary_order;
        cfg.smoothing = c->smoothing != 0;
        cfg.smoothing_subsamples = c->smoothing_subsamples;
        cfg.divergence_bound = c->divergence_bound;
    }
    return cfg;
}

// Builds the PdeProblem exactly as price_zcb (instruments.cpp:196-205) and
// price_caplet (instruments.cpp:219-232) do, from explicit axes.
PdeProblem to_problem(const hjmsv_problem& p) {
    PdeProblem pb;
    pb.r_axis = to_axis(p.r);
    pb.v_axis = to_axis(p.v);
    pb.y_axis = to_axis(p.y);
    pb.model = to_model(p.model);
    pb.curve = to_curve(p.curve);
    pb.r0 = p.r0;
    pb.maturity = p.maturity;
    const double r0 = p.r0;
    if (p.instrument == HJMSV_INSTRUMENT_ZCB) {
        pb.terminal = [](double, double, double) { return 1.0; };
        pb.boundary = BoundarySpec::zcb(p.maturity, pb.curve, pb.model, r0);
    } else if (p.instrument == HJMSV_INSTRUMENT_CAPLET) {
        CapletSpec spec = to_caplet(p);
        InitialCurve curve = pb.curve;
        ModelParams params = pb.model;
        pb.terminal = [spec, curve, params, r0](double zr, double, double zy) {
            StatePoint terminal{r0 * zr, 1.0, r0 * r0 * zy, spec.expiry};
            return caplet_payoff(terminal, spec, curve, params);
        };
        pb.boundary = BoundarySpec::caplet(spec, pb.curve, pb.model, r0);
    } else {
        BoundarySpec b;
        b.instrument = BoundarySpec::Instrument::custom;
        for (int f = 0; f < 6; ++f) {
            b.rule[f] = p.face_rule[f] == HJMSV_FACE_DIRICHLET  ? FaceRule::dirichlet
                        : p.face_rule[f] == HJMSV_FACE_DEGENERATE ? FaceRule::degenerate_pde
                                                                  : FaceRule::one_sided_convection;
            if (b.rule[f] == FaceRule::dirichlet)
                b.value[f] = value_fn(p.face_value[f], pb.curve, p.model.kappa, r0);
        }
        pb.boundary = b;
        pb.terminal = [](double, double, double) { return 0.0; };
    }
    return pb;
}

// terminal fill + smoothing, solver.cpp:220-227
Grid3 initial_level(const PdeProblem& pb, const SolverConfig& cfg, const hjmsv_problem& p) {
    Grid3 grid(pb.r_axis, pb.v_axis, pb.y_axis);
    grid.time = pb.maturity;
    if (p.initial_grid) {
        std::memcpy(grid.data.data(), p.initial_grid, grid.data.size() * sizeof(double));
        return grid;
    }
    if (p.instrument == HJMSV_INSTRUMENT_CUSTOM)
        throw std::invalid_argument("custom instrument needs an initial grid");
    for (int i = 0; i < grid.nr(); ++i)
        for (int j = 0; j < grid.nv(); ++j)
            for (int k = 0; k < grid.ny(); ++k)
                grid.at(i, j, k) = pb.terminal(grid.r.z[i], grid.v.z[j], grid.y.z[k]);
    if (cfg.smoothing) smooth_terminal(grid, pb.terminal, cfg.smoothing_subsamples);
    return grid;
}

int resolve_steps(const hjmsv_problem& p, const SolverConfig& cfg) {
    if (p.n_steps > 0) return p.n_steps;
    return std::max(1, static_cast<int>(std::lround(cfg.steps_per_year * p.maturity)));
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_mix_seed(uint64_t root, uint64_t stream) { return mix_seed(root, stream); }

int ref_uniform_axis(double z0, double z_inf, int n, double* z, double* j1, double* j2) {
    return guarded([&] {
        Axis a = uniform_axis(z0, z_inf, n);
        std::copy(a.z.begin(), a.z.end(), z);
        std::copy(a.j1.begin(), a.j1.end(), j1);
        std::copy(a.j2.begin(), a.j2.end(), j2);
    });
}

int ref_sinh_axis(double center, double alpha, double z0, double z_inf, int n, double* z,
                  double* j1, double* j2, double* c1c2) {
    return guarded([&] {
        Axis a = build_axis(MetricParams{center, alpha, z0, z_inf}, n);
        std::copy(a.z.begin(), a.z.end(), z);
        std::copy(a.j1.begin(), a.j1.end(), j1);
        std::copy(a.j2.begin(), a.j2.end(), j2);
        c1c2[0] = a.c1;
        c1c2[1] = a.c2;
    });
}

int ref_curve_eval(const hjmsv_curve* c, int what, int count, const double* t, double* out) {
    return guarded([&] {
        InitialCurve curve = to_curve(*c);
        for (int q = 0; q < count; ++q)
            out[q] = what == 0 ? curve.discount(t[q])
                     : what == 1 ? curve.forward(t[q])
                                 : curve.forward_slope(t[q]);
    });
}

int ref_g_factor(double s, double kappa, double* out) {
    return guarded([&] { *out = g_factor(s, kappa); });
}

int ref_zcb_closed_form(const hjmsv_curve* c, double kappa, double t, double maturity, double x,
                        double y, double* out) {
    return guarded([&] { *out = zcb_closed_form(t, maturity, x, y, to_curve(*c), kappa); });
}

int ref_initial_level(const hjmsv_problem* p, const hjmsv_solver_config* c, double* grid_out) {
    return guarded([&] {
        SolverConfig cfg = to_config(c);
        PdeProblem pb = to_problem(*p);
        Grid3 g = initial_level(pb, cfg, *p);
        std::copy(g.data.begin(), g.data.end(), grid_out);
    });
}

// The march of run() (solver.cpp:213-258). steps_to_do < 0 runs all steps.
int ref_run(const hjmsv_problem* p, const hjmsv_solver_config* c, int steps_to_do,
            double* grid_out, hjmsv_report* rep) {
    hjmsv_report r{};
    r.failed_row = -1;
    r.nan_guard_ok = 1;
    int code = guarded([&] {
        SolverConfig cfg = to_config(c);
        PdeProblem pb = to_problem(*p);
        const bool pure = p->time_levels == HJMSV_TIME_REFERENCE && p->n_steps == 0 &&
                          steps_to_do < 0 && !p->initial_grid &&
                          p->instrument != HJMSV_INSTRUMENT_CUSTOM;
        if (pure) {
            // the reference's own entry point, untouched
            auto [grid, report] = run(pb, cfg);
            r.wall_seconds = report.wall_seconds;
            r.n_steps = report.n_steps;
            r.steps_done = report.n_steps;
            r.last_max_delta = report.last_max_delta;
            r.nan_guard_ok = report.nan_guard_ok;
            r.time = grid.time;
            if (grid_out) std::copy(grid.data.begin(), grid.data.end(), grid_out);
            return;
        }
        cfg.validate();
        if (pb.maturity <= 0.0) throw std::invalid_argument("run: maturity must be positive");
        const auto t0 = std::chrono::steady_clock::now();
        Grid3 grid = initial_level(pb, cfg, *p);
        HjmCoefficientField coeffs(grid.r, grid.v, grid.y, pb.model, pb.curve, pb.r0);
        SpatialOperator op(grid.r, grid.v, grid.y, coeffs, pb.boundary,
                           {cfg.y_boundary_order, cfg.r_boundary_order});
        const int n_steps = resolve_steps(*p, cfg);
        const double dt = pb.maturity / n_steps;
        const int todo = steps_to_do < 0 ? n_steps : std::min(steps_to_do, n_steps);
        r.n_steps = n_steps;
        for (int step = 0; step < todo; ++step) {
            if (p->time_levels == HJMSV_TIME_INDEXED) grid.time = pb.maturity - step * dt;
            try {
                r.last_max_delta = douglas_step(grid, op, dt, cfg);
            } catch (const std::runtime_error& err) {
                r.nan_guard_ok = 0;
                r.failed_step = step + 1;
                throw std::runtime_error("step " + std::to_string(step + 1) + "/" +
                                         std::to_string(n_steps) + ": " + err.what());
            }
            r.steps_done = step + 1;
        }
        if (todo == n_steps) grid.time = 0.0;
        r.time = grid.time;
        r.wall_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (grid_out) std::copy(grid.data.begin(), grid.data.end(), grid_out);
    });
    r.status = code;
    if (rep) *rep = r;
    return code;
}

// A resumable march for the CPU baseline legs of bench.py: create() does the
// setup of run() (terminal fill + smooth_terminal, coefficient field, operator;
// solver.cpp:219-236) once, steps() advances the same march with douglas_step
// (solver.cpp:240-251, indexed time levels when the problem asks for them) and
// returns the time of the stepping loop alone, as SURVEY §8d's timed region.
struct RefSession {
    PdeProblem pb;
    SolverConfig cfg;
    std::unique_ptr<Grid3> grid;
    std::unique_ptr<HjmCoefficientField> coeffs;
    std::unique_ptr<SpatialOperator> op;
    int n_steps = 0, step = 0;
    bool indexed = false;
    double dt = 0.0;
};

void* ref_session_create(const hjmsv_problem* p, const hjmsv_solver_config* c) {
    RefSession* out = nullptr;
    const int code = guarded([&] {
        auto ses = std::make_unique<RefSession>();
        ses->cfg = to_config(c);
        ses->cfg.validate();
        ses->pb = to_problem(*p);
        ses->grid = std::make_unique<Grid3>(initial_level(ses->pb, ses->cfg, *p));
        Grid3& g = *ses->grid;
        ses->coeffs = std::make_unique<HjmCoefficientField>(g.r, g.v, g.y, ses->pb.model, ses->pb.curve,
                                                            ses->pb.r0);
        ses->op = std::make_unique<SpatialOperator>(
            g.r, g.v, g.y, *ses->coeffs, ses->pb.boundary,
            SpatialOperator::Options{ses->cfg.y_boundary_order, ses->cfg.r_boundary_order});
        ses->n_steps = resolve_steps(*p, ses->cfg);
        ses->dt = ses->pb.maturity / ses->n_steps;
        ses->indexed = p->time_levels == HJMSV_TIME_INDEXED;
        out = ses.release();
    });
    (void)code;
    return out;
}

// advances `count` steps (restarting from the terminal level is the caller's
// business: past the last step it wraps to step 0 of a fresh time sequence on
// the current level, which keeps the per-step work identical)
int ref_session_steps(void* h, int count, double* loop_seconds) {
    auto* ses = static_cast<RefSession*>(h);
    double secs = 0.0;
    const int code = guarded([&] {
        if (!ses) throw std::invalid_argument("null session");
        Grid3& g = *ses->grid;
        const auto t0 = std::chrono::steady_clock::now();
        for (int q = 0; q < count; ++q) {
            if (ses->step >= ses->n_steps) {
                ses->step = 0;
                g.time = ses->pb.maturity;
            }
            if (ses->indexed) g.time = ses->pb.maturity - ses->step * ses->dt;
            douglas_step(g, *ses->op, ses->dt, ses->cfg);
            ++ses->step;
        }
        secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
    if (loop_seconds) *loop_seconds = secs;
    return code;
}

void ref_session_destroy(void* h) { delete static_cast<RefSession*>(h); }

// douglas_step on an injected level (solver.hpp:45-47)
int ref_douglas_step(const hjmsv_problem* p, const hjmsv_solver_config* c, const double* u_in,
                     double t_from, double dt, double* u_out, double* max_delta,
                     double* t_next_out) {
    return guarded([&] {
        SolverConfig cfg = to_config(c);
        PdeProblem pb = to_problem(*p);
        Grid3 grid(pb.r_axis, pb.v_axis, pb.y_axis);
        std::memcpy(grid.data.data(), u_in, grid.data.size() * sizeof(double));
        grid.time = t_from;
        HjmCoefficientField coeffs(grid.r, grid.v, grid.y, pb.model, pb.curve, pb.r0);
        SpatialOperator op(grid.r, grid.v, grid.y, coeffs, pb.boundary,
                           {cfg.y_boundary_order, cfg.r_boundary_order});
        double md = douglas_step(grid, op, dt, cfg);
        if (max_delta) *max_delta = md;
        if (t_next_out) *t_next_out = grid.time;
        std::copy(grid.data.begin(), grid.data.end(), u_out);
    });
}

int ref_apply_operator(const hjmsv_problem* p, const hjmsv_solver_config* c, double t,
                       const double* u, double* out) {
    return guarded([&] {
        SolverConfig cfg = to_config(c);
        PdeProblem pb = to_problem(*p);
        Grid3 ug(pb.r_axis, pb.v_axis, pb.y_axis), og(pb.r_axis, pb.v_axis, pb.y_axis);
        std::memcpy(ug.data.data(), u, ug.data.size() * sizeof(double));
        HjmCoefficientField coeffs(ug.r, ug.v, ug.y, pb.model, pb.curve, pb.r0);
        SpatialOperator op(ug.r, ug.v, ug.y, coeffs, pb.boundary,
                           {cfg.y_boundary_order, cfg.r_boundary_order});
        coeffs.prepare(t);
        op.apply_operator(ug, og);
        std::copy(og.data.begin(), og.data.end(), out);
    });
}

// assemble_line_{r,v,y} (discretization.cpp:194-300); axis 0/1/2, (a,b) the
// two fixed indices in (j,k) / (i,k) / (i,j) order.
int ref_assemble_line(const hjmsv_problem* p, const hjmsv_solver_config* c, int axis, int a,
                      int b, double t, double theta_dt, double* lower, double* diag,
                      double* upper, double* super2) {
    return guarded([&] {
        SolverConfig cfg = to_config(c);
        PdeProblem pb = to_problem(*p);
        HjmCoefficientField coeffs(pb.r_axis, pb.v_axis, pb.y_axis, pb.model, pb.curve, pb.r0);
        SpatialOperator op(pb.r_axis, pb.v_axis, pb.y_axis, coeffs, pb.boundary,
                           {cfg.y_boundary_order, cfg.r_boundary_order});
        coeffs.prepare(t);
        TriDiagLine line = axis == 0   ? op.assemble_line_r(a, b, theta_dt)
                           : axis == 1 ? op.assemble_line_v(a, b, theta_dt)
                                       : op.assemble_line_y(a, b, theta_dt);
        std::copy(line.lower.begin(), line.lower.end(), lower);
        std::copy(line.diag.begin(), line.diag.end(), diag);
        std::copy(line.upper.begin(), line.upper.end(), upper);
        *super2 = line.first_row_super2;
    });
}

int ref_thomas(int n, int count, const double* lower, const double* diag, const double* upper,
               const double* super2, double* rhs) {
    return guarded([&] {
        std::vector<double> scratch(n);
        for (int q = 0; q < count; ++q) {
            TriDiagLine line(n);
            std::copy(lower + q * n, lower + (q + 1) * n, line.lower.begin());
            std::copy(diag + q * n, diag + (q + 1) * n, line.diag.begin());
            std::copy(upper + q * n, upper + (q + 1) * n, line.upper.begin());
            line.first_row_super2 = super2[q];
            thomas_solve_inplace(line, rhs + q * n, scratch.data());
        }
    });
}

int ref_interpolate(const hjmsv_problem* p, const double* grid_data, double zr, double zv,
                    double zy, double* out) {
    return guarded([&] {
        Grid3 g(to_axis(p->r), to_axis(p->v), to_axis(p->y));
        std::memcpy(g.data.data(), grid_data, g.data.size() * sizeof(double));
        *out = interpolate_at(g, zr, zv, zy);
    });
}

// spot readout of finish() (instruments.cpp:145-149) at natural_spot (:50-52)
int ref_spot_price(const hjmsv_problem* p, const double* grid_data, double* out) {
    return guarded([&] {
        Grid3 g(to_axis(p->r), to_axis(p->v), to_axis(p->y));
        std::memcpy(g.data.data(), grid_data, g.data.size() * sizeof(double));
        InitialCurve curve = to_curve(p->curve);
        StatePoint spot = natural_spot(curve);
        *out = interpolate_at(g, spot.r / p->r0, spot.v, spot.y / (p->r0 * p->r0));
    });
}

// extract_greeks (instruments.cpp:90-132) and finish()'s rho /= r0 (:150-152)
int ref_extract_greeks(const hjmsv_problem* p, const double* grid_data, int scale_rate,
                       double* rho_out, double* vega_out) {
    return guarded([&] {
        Grid3 g(to_axis(p->r), to_axis(p->v), to_axis(p->y));
        std::memcpy(g.data.data(), grid_data, g.data.size() * sizeof(double));
        auto [rho, vega] = extract_greeks(g);
        if (scale_rate)
            for (double& x : rho.data) x /= p->r0;
        std::memcpy(rho_out, rho.data.data(), rho.data.size() * sizeof(double));
        std::memcpy(vega_out, vega.data.data(), vega.data.size() * sizeof(double));
    });
}

// simulate_zcb / simulate_caplet (montecarlo.cpp:142-160): the reference's own
// Monte Carlo (mt19937_64 per 8192-path batch), the statistical check of the
// device validator
int ref_mc_price(const hjmsv_problem* p, const hjmsv_mc_config* c, int threads, double* mean,
                 double* std_error, long long* n_paths) {
    return guarded([&] {
        McConfig mc;
        mc.n_paths = c->n_paths;
        mc.steps_per_year = c->steps_per_year;
        mc.seed = c->seed;
        mc.full_truncation = c->full_truncation != 0;
        mc.threads = threads;
        const InitialCurve curve = to_curve(p->curve);
        const ModelParams mp = to_model(p->model);
        const McEstimate est = p->instrument == HJMSV_INSTRUMENT_CAPLET
                                   ? simulate_caplet(to_caplet(*p), curve, mp, mc)
                                   : simulate_zcb(p->maturity, curve, mp, mc);
        *mean = est.mean;
        *std_error = est.std_error;
        *n_paths = est.n_paths;
    });
}

// caplet_ladder's worker pool (instruments.cpp:242-264) over independent
// problems: each worker pulls the next index from an atomic counter and runs
// the full march + spot readout. Used as the batched CPU baseline.
int ref_batch_run(const hjmsv_problem* problems, int count, const hjmsv_solver_config* c,
                  int threads, double* prices, hjmsv_report* reports) {
    if (threads <= 0) threads = std::max(1u, std::thread::hardware_concurrency());
    std::atomic<int> next{0};
    std::atomic<int> first_err{HJMSV_OK};
    auto worker = [&]() {
        for (int q = next.fetch_add(1); q < count; q = next.fetch_add(1)) {
            const hjmsv_problem& p = problems[q];
            std::vector<double> grid(static_cast<size_t>(p.r.n) * p.v.n * p.y.n);
            hjmsv_report rep{};
            int code = ref_run(&p, c, -1, grid.data(), &rep);
            if (code == HJMSV_OK) {
                double price = 0.0;
                code = ref_spot_price(&p, grid.data(), &price);
                if (prices) prices[q] = price;
            } else if (prices) {
                prices[q] = std::nan("");
            }
            if (reports) reports[q] = rep;
            int expected = HJMSV_OK;
            if (code != HJMSV_OK) first_err.compare_exchange_strong(expected, code);
        }
    };
    if (threads == 1 || count <= 1) {
        worker();
    } else {
        std::vector<std::thread> pool;
        int n_workers = std::min(threads, count);
        for (int w = 0; w < n_workers; ++w) pool.emplace_back(worker);
        for (auto& th : pool) th.join();
    }
    return first_err.load();
}

}  // extern "C"
