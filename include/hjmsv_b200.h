/*
 * hjmsv_b200.h — C-ABI of the B200-native Douglas-ADI solver for the 3D HJM-SV
 * pricing PDE (arXiv 1108.1688 reference: /root/reference/proj/core).
 *
 * The reference has no C ABI; its boundary is the C++ API of
 *   run(PdeProblem, SolverConfig)                  proj/core/include/hjmsv/solver.hpp:76
 *   douglas_step(Grid3&, SpatialOperator&, dt, cfg) proj/core/include/hjmsv/solver.hpp:45-47
 *   SpatialOperator::apply_operator / assemble_line_*  discretization.hpp:154-160
 *   thomas_solve_inplace(TriDiagLine, rhs, scratch) solver.hpp:37
 *   interpolate_at(Grid3, zr, zv, zy)              instruments.hpp:51 (instruments.cpp:71-88)
 *   caplet_ladder(...)                              instruments.hpp:77 (instruments.cpp:238-266)
 * Because std::function cannot cross a C ABI (PdeProblem::terminal/source/observer,
 * BoundarySpec::value[6], ModelParams::*_fn), the problem is described here as
 * plain data: explicit axes, constant model parameters, curve quotes, an
 * instrument kind and per-face rules/value forms.
 *
 * Conventions: plain pointers + sizes, host buffers are caller-owned, device
 * buffers are owned by the solver handle. Every entry point returns an
 * hjmsv_status; on failure hjmsv_last_error() holds the message the reference
 * would have thrown (thread-local).
 */
#ifndef HJMSV_B200_H
#define HJMSV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HJMSV_ABI_VERSION 2

/* Status codes. The C++ wrapper maps them back to the reference exception
 * types: INVALID_ARGUMENT -> std::invalid_argument, SINGULAR_PIVOT/NONFINITE/
 * DIVERGED -> std::runtime_error (solver.cpp:44-52, 69-77, 241-247),
 * DOMAIN -> std::domain_error (curve.cpp:136-137, model.cpp:42,50),
 * LOGIC -> std::logic_error (discretization.cpp:191,220,249,291). */
typedef enum {
    HJMSV_OK = 0,
    HJMSV_INVALID_ARGUMENT = 1,
    HJMSV_SINGULAR_PIVOT = 2,
    HJMSV_NONFINITE = 3,
    HJMSV_DIVERGED = 4,
    HJMSV_DOMAIN = 5,
    HJMSV_UNSUPPORTED = 6,
    HJMSV_CUDA_ERROR = 7,
    HJMSV_LOGIC = 8
} hjmsv_status;

/* Axis::Map (mesh.hpp:26) */
typedef enum { HJMSV_MAP_SINH = 0, HJMSV_MAP_LINEAR = 1, HJMSV_MAP_SINGLETON = 2 } hjmsv_axis_map;

/* One discretised direction, Axis (mesh.hpp:25-40): n nodes z, Jacobians
 * j1 = dz/dx, j2 = d2z/dx2, computational spacing dx = 1/(n-1).
 * center/alpha/z0/z_inf/c1/c2 are the sinh metric constants (used only by the
 * price readout's physical_to_computational, mesh.cpp:75-92). */
typedef struct {
    int32_t n;
    int32_t map;            /* hjmsv_axis_map */
    const double* z;
    const double* j1;
    const double* j2;
    double center, alpha, z0, z_inf;
    double c1, c2;
} hjmsv_axis;

/* TimeFn (model.hpp:10): a deterministic model function of calendar time t.
 * `user` is hjmsv_model::fn_user. Called on the host only, while a problem is
 * lowered (hjmsv_solver_create / the stage entry points), possibly from several
 * host threads at once for a batch. */
typedef double (*hjmsv_time_fn)(double t, void* user);

/* ModelParams (model.hpp:20-37). With every *_fn NULL this is
 * ModelParams::constants(kappa, lambda, gamma, eps, theta, rho) (model.cpp:12-23).
 * A non-NULL lambda_fn / gamma_fn / eps_fn replaces that constant by a function
 * of t: HjmCoefficientField::prepare (discretization.cpp:40-54) evaluates them
 * at every step's half level t_mid (solver.cpp:96), and so does the lowering,
 * which then uploads per-step coefficient tables. ModelParams::validate checks
 * gamma_fn(0) in (0,1] (model.cpp:36-37). */
typedef struct {
    double kappa, lambda, gamma, eps, theta, rho;
    hjmsv_time_fn lambda_fn, gamma_fn, eps_fn;
    void* fn_user;
} hjmsv_model;

/* InitialCurve (curve.hpp): flat(base) (curve.cpp:11-20) or natural cubic
 * spline of ln p through (maturity, discount) quotes (curve.cpp:22-48,68-127). */
typedef enum { HJMSV_CURVE_FLAT = 0, HJMSV_CURVE_NODES = 1 } hjmsv_curve_kind;
typedef struct {
    int32_t kind;
    double flat_base;
    int32_t n_nodes;
    const double* maturities;
    const double* discounts;
} hjmsv_curve;

/* FaceRule (discretization.hpp:86-90); faces ordered as Face (discretization.hpp:84):
 * r_min, r_max, v_min, v_max, y_min, y_max. */
typedef enum {
    HJMSV_FACE_DIRICHLET = 0,
    HJMSV_FACE_DEGENERATE = 1,
    HJMSV_FACE_ONE_SIDED = 2
} hjmsv_face_rule;

/* Dirichlet value forms. P(t,T) below is zcb_closed_form(t, T, x, y) with
 * x = r0*zr - f(0,t), y = r0^2*zy (discretization.cpp:77-81, model.cpp:48-54).
 *   ZERO:      0
 *   ZCB:       a * P(t,T1)                 (BoundarySpec::zcb faces use a = 1)
 *   ZCB_DIFF:  a * P(t,T1) - b * P(t,T2)   (BoundarySpec::caplet v_max uses a = b = 1) */
typedef enum { HJMSV_VALUE_ZERO = 0, HJMSV_VALUE_ZCB = 1, HJMSV_VALUE_ZCB_DIFF = 2 } hjmsv_value_kind;
typedef struct {
    int32_t kind;
    double a, t1, b, t2;
} hjmsv_face_value;

/* Instrument (BoundarySpec::Instrument, discretization.hpp:96) + terminal. */
typedef enum {
    HJMSV_INSTRUMENT_ZCB = 0,     /* terminal 1, BoundarySpec::zcb (instruments.cpp:200-201) */
    HJMSV_INSTRUMENT_CAPLET = 1,  /* caplet_payoff terminal, BoundarySpec::caplet (instruments.cpp:227-231) */
    HJMSV_INSTRUMENT_CUSTOM = 2   /* face_rule/face_value given, initial_grid required */
} hjmsv_instrument;

/* Time-level sequence. REFERENCE reproduces run()/douglas_step exactly:
 * t_next = t_from - dt by repeated subtraction, snapped to 0 below 1e-12*dt
 * (solver.cpp:85-87) — this throws at config 3.
 * INDEXED sets t_from = T - s*dt before step s (the parity harness). */
typedef enum { HJMSV_TIME_REFERENCE = 0, HJMSV_TIME_INDEXED = 1 } hjmsv_time_levels;

/* A complete pricing problem: PdeProblem (solver.hpp:59-72) + the instrument
 * descriptor of SURVEY §8b. */
typedef struct {
    hjmsv_axis r, v, y;
    hjmsv_model model;
    hjmsv_curve curve;
    double r0;                  /* rate scale of the axis coordinates */
    double maturity;            /* march length T (caplet: expiry) */
    int32_t instrument;         /* hjmsv_instrument */
    double payment;             /* caplet payment date T_M */
    double strike;              /* caplet strike K */
    int32_t face_rule[6];       /* CUSTOM only */
    hjmsv_face_value face_value[6]; /* CUSTOM only */
    int32_t n_steps;            /* 0 -> max(1, lround(steps_per_year*T)) (solver.cpp:234-236) */
    int32_t time_levels;        /* hjmsv_time_levels */
    const double* initial_grid; /* optional nr*nv*ny level at t = T (overrides terminal+smoothing) */
} hjmsv_problem;

/* SolverConfig (solver.hpp:10-20) */
typedef struct {
    double theta_cn;
    int32_t steps_per_year;
    int32_t y_boundary_order;
    int32_t r_boundary_order;
    int32_t smoothing;
    int32_t smoothing_subsamples;
    double divergence_bound;
} hjmsv_solver_config;

/* SolveReport (solver.hpp:22-27) plus device diagnostics. */
typedef struct {
    double wall_seconds;
    int32_t n_steps;
    int32_t steps_done;
    double last_max_delta;
    int32_t nan_guard_ok;
    int32_t status;             /* hjmsv_status of this problem */
    int32_t failed_step;        /* 1-based step index of the failure, 0 if none */
    int32_t failed_row;         /* singular pivot row, -1 if n/a */
    double time;                /* calendar time of the current level */
} hjmsv_report;

/* Arithmetic modes of the device kernels. STRICT follows the reference's
 * literal operation order with true divides and no FMA contraction (bit-level
 * parity up to libm ulps in face values). FAST uses per-axis factor tables,
 * reciprocal pivots, FMA and the fused two-pass step; it meets the 1e-10
 * normwise parity bar. */
typedef enum { HJMSV_MODE_STRICT = 0, HJMSV_MODE_FAST = 1 } hjmsv_mode;

void hjmsv_default_solver_config(hjmsv_solver_config* cfg);
const char* hjmsv_last_error(void);
int32_t hjmsv_abi_version(void);
int32_t hjmsv_device_count(void);

/* ---- host helpers (the framework's own restatements of the L0 layer) ---- */
/* uniform_axis (mesh.cpp:46-62) */
int32_t hjmsv_uniform_axis(double z0, double z_inf, int32_t n, double* z, double* j1, double* j2);
/* build_axis (mesh.cpp:16-44); c1c2 receives {c1, c2} */
int32_t hjmsv_sinh_axis(double center, double alpha, double z0, double z_inf, int32_t n,
                        double* z, double* j1, double* j2, double* c1c2);
/* InitialCurve::discount/forward/forward_slope (curve.cpp:135-160); what = 0,1,2 */
int32_t hjmsv_curve_eval(const hjmsv_curve* curve, int32_t what, int32_t count,
                         const double* t, double* out);
/* zcb_closed_form (model.cpp:48-54) */
int32_t hjmsv_zcb_closed_form(const hjmsv_curve* curve, double kappa, double t, double maturity,
                              double x, double y, double* out);

/* ---- solver handle: one device, a batch of problems with equal dims/steps ---- */
typedef struct hjmsv_solver hjmsv_solver;

/* Lowers `count` problems (same nr/nv/ny/n_steps) to device tables, builds the
 * terminal level (terminal + smooth_terminal, solver.cpp:220-227) and uploads it. */
int32_t hjmsv_solver_create(const hjmsv_problem* problems, int32_t count,
                            const hjmsv_solver_config* cfg, int32_t device, int32_t mode,
                            hjmsv_solver** out);
void hjmsv_solver_destroy(hjmsv_solver* h);
/* Restores the terminal level and step counter (for repeated timed marches). */
int32_t hjmsv_solver_reset(hjmsv_solver* h);
/* Advances every problem by `steps` Douglas steps (douglas_step, solver.cpp:81-178),
 * enqueued on the handle's stream; returns after the launches (asynchronous). */
int32_t hjmsv_solver_step_async(hjmsv_solver* h, int32_t steps);
/* Waits for the stream and converts device status words into per-problem
 * statuses; returns the first failing problem's status. */
int32_t hjmsv_solver_synchronize(hjmsv_solver* h);
/* step_async + synchronize */
int32_t hjmsv_solver_step(hjmsv_solver* h, int32_t steps);
/* All remaining steps (the march of run(), solver.cpp:240-251). */
int32_t hjmsv_solver_run(hjmsv_solver* h);
int32_t hjmsv_solver_report(hjmsv_solver* h, int32_t problem, hjmsv_report* out);
int32_t hjmsv_solver_dims(hjmsv_solver* h, int32_t* nr, int32_t* nv, int32_t* ny,
                          int32_t* count, int32_t* n_steps);
int32_t hjmsv_solver_get_grid(hjmsv_solver* h, int32_t problem, double* host_out);
/* All problems' levels in one copy: host_out[p*nr*nv*ny + idx] (batch readout). */
int32_t hjmsv_solver_get_grids(hjmsv_solver* h, double* host_out);
/* Injects a level (Grid3::data + Grid3::time are public, discretization.hpp:14-17). */
int32_t hjmsv_solver_set_grid(hjmsv_solver* h, int32_t problem, const double* host_in,
                              int32_t step_index);
/* interpolate_at (instruments.cpp:71-88) on the current level. */
int32_t hjmsv_solver_price(hjmsv_solver* h, int32_t problem, double zr, double zv, double zy,
                           double* out);
/* interpolate_at at natural_spot (f(0,0)/r0, 1, 0) (instruments.cpp:50-52,148) for all problems. */
int32_t hjmsv_solver_spot_prices(hjmsv_solver* h, double* out);
/* extract_greeks (instruments.cpp:90-132) of problem p's current level, on the
 * device: rho = dU/dr~ and vega = dU/dv (computational-coordinate differences over
 * j1, one-sided on the faces). scale_rate != 0 applies finish()'s rho /= r0
 * (instruments.cpp:150-152). rho / vega are caller host buffers of nr*nv*ny
 * doubles; either may be NULL. */
int32_t hjmsv_solver_greeks(hjmsv_solver* h, int32_t problem, int32_t scale_rate, double* rho,
                            double* vega);
/* write_surface_csv's rows (job.cpp:300-310) at y-slice k, computed on the device:
 * out[(i*nv + j)*5 + c] = (r0*z_r[i], z_v[j], U, rho/r0, vega)(i, j, k); only the
 * slice crosses PCIe. */
int32_t hjmsv_solver_surface(hjmsv_solver* h, int32_t problem, int32_t k, double* out);
/* ---- Monte Carlo validator on the device (montecarlo.cpp:38-139) ----
 * McConfig (montecarlo.hpp:15-24) without threads/observer. The device draws its
 * normals from a counter-based generator (Philox4x32-10 + Box-Muller) keyed by
 * (seed, path), so estimates are reproducible and independent of the launch
 * shape, but they are a different sample from the reference's mt19937_64
 * stream: parity with the reference is statistical (within standard errors). */
typedef struct {
    int64_t n_paths;
    int32_t steps_per_year;
    uint64_t seed;
    int32_t full_truncation;
} hjmsv_mc_config;
void hjmsv_default_mc_config(hjmsv_mc_config* cfg);
/* simulate_zcb / simulate_caplet (montecarlo.cpp:142-160) for problem p (its
 * model, curve, instrument, maturity, payment, strike; the axes are unused).
 * Writes McEstimate {mean, std_error, n_paths}. */
int32_t hjmsv_mc_price(const hjmsv_problem* problem, const hjmsv_mc_config* cfg, int32_t device,
                       double* mean, double* std_error, int64_t* n_paths);
/* Device pointer of problem p's level (stable for the handle's lifetime). */
int32_t hjmsv_solver_device_grid(hjmsv_solver* h, int32_t problem, double** dev_ptr);
/* Elapsed device time of the last step_async batch (CUDA events on the handle's stream). */
int32_t hjmsv_solver_last_device_ms(hjmsv_solver* h, double* ms);
/* Number of kernel launches issued by the last step_async call. */
int32_t hjmsv_solver_last_launches(hjmsv_solver* h, int64_t* launches);

/* Live per-kernel profile (FAST mode): runs `steps` steps launched exactly as
 * a handle's first march (direct launches, programmatic dependent launch),
 * every block recording its start/end on the device clock; returns each
 * kernel slot's average duration (ms, span of its blocks per launch), its
 * ALGORITHMIC bytes per launch (bytes/point x points; SURVEY §8d accounting),
 * the launch count, the names (name_len bytes each) and the event-timed
 * duration of the whole profiled sequence (march_ms, may be null). Used by
 * bench.py for the roofline. */
int32_t hjmsv_solver_kernel_timeline(hjmsv_solver* h, int32_t steps, int32_t max_kernels,
                                     double* avg_ms, double* alg_bytes, int64_t* launches,
                                     int32_t* n_kernels, char* names, int32_t name_len,
                                     double* march_ms);
/* hjmsv_solver_kernel_timeline without march_ms. */
int32_t hjmsv_solver_kernel_profile(hjmsv_solver* h, int32_t steps, int32_t max_kernels,
                                    double* avg_ms, double* alg_bytes, int64_t* launches,
                                    int32_t* n_kernels, char* names, int32_t name_len);

/* ---- stage entry points (parity tests: the reference's stage oracles) ----
 * They run on the calling thread's current CUDA device (cudaSetDevice). */
/* SpatialOperator::apply_operator after coefficients().prepare(t) (discretization.cpp:302-364) */
int32_t hjmsv_apply_operator(const hjmsv_problem* p, const hjmsv_solver_config* cfg, double t,
                             const double* u, double* out, int32_t mode);
/* One douglas_step from level u_in at calendar time t_from (solver.cpp:81-178). */
int32_t hjmsv_douglas_step(const hjmsv_problem* p, const hjmsv_solver_config* cfg,
                           const double* u_in, double t_from, double dt, double* u_out,
                           double* max_delta, int32_t mode);
/* Batched thomas_solve_inplace (solver.cpp:22-57) of `count` lines of length n
 * (arrays are count*n, line-major); super2 is per line. mode HJMSV_MODE_STRICT:
 * the reference's sequential Thomas; HJMSV_MODE_FAST: the partition method of
 * pass A's r-lines (16-row segments, lane-scan reduced system, n <= 512);
 * HJMSV_THOMAS_FAST_TWISTED: the same with pass B's twisted segment solve. */
#define HJMSV_THOMAS_FAST_TWISTED 2
int32_t hjmsv_thomas_batch(int32_t n, int32_t count, const double* lower, const double* diag,
                           const double* upper, const double* super2, double* rhs,
                           int32_t mode);

/* ---- batch driver (caplet_ladder, instruments.cpp:238-266, on GPUs) ----
 * Shards problems contiguously over `n_devices` devices (one host thread per
 * device, no inter-GPU traffic), runs every march and gathers spot prices and
 * reports. grids_out (nullable) receives every final level, problem-major. */
int32_t hjmsv_batch_run(const hjmsv_problem* problems, int32_t count,
                        const hjmsv_solver_config* cfg, const int32_t* devices,
                        int32_t n_devices, int32_t mode, double* prices_out,
                        hjmsv_report* reports_out, double* grids_out);

#ifdef __cplusplus
}
#endif
#endif /* HJMSV_B200_H */
