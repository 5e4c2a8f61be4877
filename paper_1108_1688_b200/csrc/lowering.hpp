// lowering.hpp — PdeProblem + SolverConfig (as hjmsv_problem / hjmsv_solver_config)
// lowered on the host to the plain tables the device kernels read.
#pragma once

#include <vector>

#include "device_types.hpp"
#include "hjmsv_b200.h"
#include "host_math.hpp"

namespace hjmsv_b200 {

struct Lowered {
    int nr = 0, nv = 0, ny = 0;
    int n_steps = 0;
    double maturity = 0.0, dt = 0.0, r0 = 0.0;
    Axis r, v, y;
    Curve curve;
    ProblemConst pc{};
    std::vector<double> axes;    // axes_stride(nr,nv,ny)
    std::vector<double> steps;   // n_steps * kStepStride
    std::vector<double> init;    // nr*nv*ny level at t = T
    double term_t[kMaxTerms] = {};  // maturity of each closed-form term slot
    long long spot_idx[8] = {};  // interpolate_at corners at natural_spot
    double spot_w[8] = {};
    TermParam term{};            // terminal built on the device (kind != TERM_HOST)
    hjmsv_model model{};         // ModelParams (with the model functions, if any)
    bool timedep = false;        // lambda/gamma/eps given as functions of t
    std::vector<double> ab_steps;  // timedep: n_steps * [a_i (nr), b_i (nr)] of prepare(t_mid)
};

/// lambda(t), gamma(t), eps(t) of a model (constants unless *_fn is set).
struct ModelAt {
    double lambda, gamma, eps;
};
bool time_dependent(const hjmsv_model& m);
ModelAt model_at(const hjmsv_model& m, double t);
/// prepare's a_i = lambda^2 rp^2 / 2, b_i = lambda eps rho rp (discretization.cpp:48-53).
void prepare_ab(const Lowered& L, const ModelAt& x, double* a, double* b);
/// Per-step model data from the step table's half levels: eps^2/2 into ST_HEPS2
/// and, for model functions, the a_i / b_i of every step (L.ab_steps).
void build_model_steps(Lowered& L);

/// How lower_problem provides the terminal level: on the host (L.init) or as
/// device terminal parameters (L.term) for ZCB / caplet problems without an
/// explicit initial grid (smooth_terminal + caplet_payoff, solver.cpp:180-211).
enum InitMode { INIT_NONE = 0, INIT_HOST = 1, INIT_DEVICE = 2 };

/// Validates exactly like run() (solver.cpp:214-216), SolverConfig::validate
/// (solver.cpp:10-20), ModelParams::validate (model.cpp:25-33), CapletSpec::validate
/// (model.cpp:35-39), HjmCoefficientField (discretization.cpp:34-35) and
/// SpatialOperator (discretization.cpp:144-150), then builds every table.
/// Throws the reference's exception types/messages.
Lowered lower_problem(const hjmsv_problem& p, const hjmsv_solver_config& cfg, int init_mode);

/// Per-step scalar table for explicit (t_from, dt) levels; used by the march
/// (time levels of run() or the indexed harness) and by the single-step stage.
void build_step_table(Lowered& L, const std::vector<double>& t_from, double dt, bool faces);

/// Time levels t_from[s] of the march (solver.cpp:85-87 or SURVEY §8c).
std::vector<double> march_levels(double maturity, int n_steps, int time_levels);

/// Corner indices/weights of interpolate_at (instruments.cpp:71-88) at (zr, zv, zy).
void locate_point(const Lowered& L, double zr, double zv, double zy, long long idx[8],
                  double w[8]);

hjmsv_solver_config default_config();

/// Host side of the Monte Carlo validator (montecarlo.cpp:83-139): validated
/// model, per-step forward curve f(0, t_s + dt) and the payout scalars.
struct McSetup {
    int n_steps = 0;
    double dt = 0.0, sqrt_dt = 0.0, decay_y = 0.0, decay_h = 0.0, f0 = 0.0;
    std::vector<double> steps;    // per step s: f(0, (s+1) dt), lambda(s dt), gamma(s dt), eps(s dt)
    int caplet = 0;
    double accrual = 0.0, ratio = 0.0, g = 0.0, horizon = 0.0;
};
McSetup lower_mc(const hjmsv_problem& p, const hjmsv_mc_config& c);

/// FAST-mode factor tables (layout: FastR/FastV/FastY in device_types.hpp).
/// step >= 0 with model functions: the tables of that step's prepare(t_mid).
std::vector<double> build_fast_tables(const Lowered& L, const hjmsv_solver_config& cfg,
                                      double theta_dt, int step = -1);

}  // namespace hjmsv_b200
