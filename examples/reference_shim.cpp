// examples/reference_shim.cpp — the reference-side binding of INTEGRATION.md §1,
// compiled for real: the reference's own C++ API (hjmsv::PdeProblem, run(),
// BoundarySpec, InitialCurve, from /root/reference/proj/core/include) drives the
// B200 library through the C-ABI of include/hjmsv_b200.h.
//
// main() builds a ZCB and a caplet problem with the reference's API, prices each
// with the reference's run() (CPU) and with run_b200() (the GPU through the
// C-ABI), and prints one JSON line per problem with the normwise grid
// difference and both spot prices. Built by examples/Makefile against
// oracle/_ref/libhjmsv_ref.so (the compiled reference) and the product library.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hjmsv/curve.hpp"
#include "hjmsv/instruments.hpp"
#include "hjmsv/mesh.hpp"
#include "hjmsv/model.hpp"
#include "hjmsv/solver.hpp"
#include "hjmsv_b200.h"

namespace hjmsv {

// The problem must carry the instrument, because BoundarySpec keeps only its
// kind (discretization.hpp:96-100) and std::function cannot cross the ABI.
struct B200Instrument {
    int kind;
    double expiry, payment, strike;
};

static hjmsv_axis to_c(const Axis& a) {
    hjmsv_axis c{};
    c.n = a.n;
    c.map = a.map == Axis::Map::sinh     ? HJMSV_MAP_SINH
            : a.map == Axis::Map::linear ? HJMSV_MAP_LINEAR
                                         : HJMSV_MAP_SINGLETON;
    c.z = a.z.data();
    c.j1 = a.j1.data();
    c.j2 = a.j2.data();
    c.center = a.params.center;
    c.alpha = a.params.alpha;
    c.z0 = a.params.z0;
    c.z_inf = a.params.z_inf;
    c.c1 = a.c1;
    c.c2 = a.c2;
    return c;
}

// Drop-in for run(problem, cfg) (solver.cpp:213-258) on one B200.
std::pair<Grid3, SolveReport> run_b200(const PdeProblem& pb, const SolverConfig& cfg,
                                       const B200Instrument& ins,
                                       const std::vector<std::pair<double, double>>& quotes,
                                       double flat_base /* > 0: flat curve */, int mode,
                                       int n_steps, int time_levels) {
    hjmsv_problem p{};
    p.r = to_c(pb.r_axis);
    p.v = to_c(pb.v_axis);
    p.y = to_c(pb.y_axis);
    // ModelParams: the reference's TimeFn objects cross the C ABI as callbacks
    // (fn_user = the ModelParams; called while the problem is lowered)
    p.model = {pb.model.kappa, 0.0, 0.0, 0.0, pb.model.theta, pb.model.rho,
               [](double t, void* u) { return static_cast<const ModelParams*>(u)->lambda_fn(t); },
               [](double t, void* u) { return static_cast<const ModelParams*>(u)->gamma_fn(t); },
               [](double t, void* u) { return static_cast<const ModelParams*>(u)->eps_fn(t); },
               const_cast<ModelParams*>(&pb.model)};
    std::vector<double> T, D;
    for (auto& q : quotes) {
        T.push_back(q.first);
        D.push_back(q.second);
    }
    p.curve = flat_base > 0 ? hjmsv_curve{HJMSV_CURVE_FLAT, flat_base, 0, nullptr, nullptr}
                            : hjmsv_curve{HJMSV_CURVE_NODES, 0.0, static_cast<int32_t>(T.size()),
                                          T.data(), D.data()};
    p.r0 = pb.r0;
    p.maturity = pb.maturity;
    p.instrument = ins.kind;
    p.payment = ins.payment;
    p.strike = ins.strike;
    p.n_steps = n_steps;          // 0: lround(steps_per_year * T), as run()
    p.time_levels = time_levels;  // HJMSV_TIME_REFERENCE: run()'s own levels
    hjmsv_solver_config c{cfg.theta_cn, cfg.steps_per_year, cfg.y_boundary_order,
                          cfg.r_boundary_order, cfg.smoothing ? 1 : 0, cfg.smoothing_subsamples,
                          cfg.divergence_bound};
    hjmsv_solver* h = nullptr;
    auto check = [&](int32_t code) {
        if (code == HJMSV_OK) return;
        const std::string msg = hjmsv_last_error();
        if (h) hjmsv_solver_destroy(h);
        switch (code) {  // the reference's exception types
            case HJMSV_INVALID_ARGUMENT: throw std::invalid_argument(msg);
            case HJMSV_DOMAIN: throw std::domain_error(msg);
            case HJMSV_LOGIC: throw std::logic_error(msg);
            default: throw std::runtime_error(msg);
        }
    };
    check(hjmsv_solver_create(&p, 1, &c, /*device=*/0, mode, &h));
    check(hjmsv_solver_run(h));
    Grid3 grid(pb.r_axis, pb.v_axis, pb.y_axis);
    check(hjmsv_solver_get_grid(h, 0, grid.data.data()));
    hjmsv_report r{};
    check(hjmsv_solver_report(h, 0, &r));
    hjmsv_solver_destroy(h);
    grid.time = 0.0;
    SolveReport rep;
    rep.wall_seconds = r.wall_seconds;
    rep.n_steps = r.n_steps;
    rep.last_max_delta = r.last_max_delta;
    rep.nan_guard_ok = r.nan_guard_ok != 0;
    return {std::move(grid), rep};
}

}  // namespace hjmsv

using namespace hjmsv;

static double normwise(const Grid3& a, const Grid3& b) {
    double num = 0.0, den = 0.0;
    for (size_t q = 0; q < a.data.size(); ++q) {
        num = std::max(num, std::abs(a.data[q] - b.data[q]));
        den = std::max(den, std::abs(b.data[q]));
    }
    return num / std::max(den, 1e-300);
}

int main() {
    if (hjmsv_device_count() < 1) {
        std::printf("{\"skipped\": \"no CUDA device\"}\n");
        return 0;
    }
    const double base = 1.04, r0 = 0.01;
    const InitialCurve curve = InitialCurve::flat(base);
    const ModelParams model_const = ModelParams::constants(0.05, 0.15, 0.9, 0.4, 1.2, -0.3);
    // time-dependent model functions (ModelParams::lambda_fn / gamma_fn / eps_fn)
    ModelParams model_t = model_const;
    model_t.lambda_fn = [](double t) { return 0.15 * (1.0 + 0.3 * std::sin(2.0 * t)); };
    model_t.gamma_fn = [](double t) { return 0.9 - 0.05 * (1.0 - std::cos(t)); };
    model_t.eps_fn = [](double t) { return 0.4 * std::exp(-0.1 * t); };
    SolverConfig cfg;  // reference defaults (solver.hpp:10-20)
    cfg.steps_per_year = 24;
    struct Case {
        const char* name;
        B200Instrument ins;
        bool timefn;
    };
    const Case cases[] = {
        {"zcb", {HJMSV_INSTRUMENT_ZCB, 5.0, 0.0, 0.0}, false},
        {"caplet", {HJMSV_INSTRUMENT_CAPLET, 3.0, 3.25, 0.035}, false},
        {"caplet_timefn", {HJMSV_INSTRUMENT_CAPLET, 3.0, 3.25, 0.035}, true},
    };
    int bad = 0;
    for (const Case& cs : cases) {
        const ModelParams& model = cs.timefn ? model_t : model_const;
        PdeProblem pb;
        pb.r_axis = uniform_axis(0.0, 25.0, 48);
        pb.v_axis = uniform_axis(0.0, 1.5, 24);
        pb.y_axis = uniform_axis(0.0, 250.0, 24);
        pb.model = model;
        pb.curve = curve;
        pb.r0 = r0;
        pb.maturity = cs.ins.expiry;
        if (cs.ins.kind == HJMSV_INSTRUMENT_ZCB) {
            pb.terminal = [](double, double, double) { return 1.0; };
            pb.boundary = BoundarySpec::zcb(cs.ins.expiry, curve, model, r0);
        } else {
            CapletSpec spec;
            spec.expiry = cs.ins.expiry;
            spec.payment = cs.ins.payment;
            spec.strike = cs.ins.strike;
            pb.terminal = [spec, curve, model, r0](double zr, double, double zy) {
                StatePoint terminal{r0 * zr, 1.0, r0 * r0 * zy, spec.expiry};
                return caplet_payoff(terminal, spec, curve, model);
            };
            pb.boundary = BoundarySpec::caplet(spec, curve, model, r0);
        }
        const auto t0 = std::chrono::steady_clock::now();
        const auto ref = run(pb, cfg);  // the reference, CPU
        const auto t1 = std::chrono::steady_clock::now();
        for (int mode : {HJMSV_MODE_STRICT, HJMSV_MODE_FAST}) {
            const auto gpu = run_b200(pb, cfg, cs.ins, {}, base, mode, 0, HJMSV_TIME_REFERENCE);
            const double err = normwise(gpu.first, ref.first);
            const StatePoint spot = natural_spot(curve);
            const double p_ref = interpolate_at(ref.first, spot.r / r0, spot.v, spot.y / (r0 * r0));
            const double p_gpu = interpolate_at(gpu.first, spot.r / r0, spot.v, spot.y / (r0 * r0));
            const double perr = std::abs(p_gpu - p_ref) / std::abs(p_ref);
            std::printf("{\"case\": \"%s\", \"mode\": \"%s\", \"n_steps\": %d, \"grid_rel\": %.3e, "
                        "\"price_ref\": %.15g, \"price_gpu\": %.15g, \"price_rel\": %.3e, "
                        "\"ref_seconds\": %.3f}\n",
                        cs.name, mode == HJMSV_MODE_FAST ? "fast" : "strict", gpu.second.n_steps, err,
                        p_ref, p_gpu, perr, std::chrono::duration<double>(t1 - t0).count());
            if (!(err <= 1e-10 && perr <= 1e-10) || gpu.second.n_steps != ref.second.n_steps) ++bad;
        }
    }
    return bad ? 1 : 0;
}
