// host_math.hpp — the framework's host-side L0 layer: axes, initial curve and
// closed forms that produce the per-step scalar tables the device kernels
// consume. These are the framework's own restatements (no reference code is
// linked); arithmetic follows the reference's operation order so the tables
// are bit-identical to what the reference computes inside douglas_step.
#pragma once

#include <string>
#include <utility>
#include <vector>

namespace hjmsv_b200 {

/// One discretised direction (reference Axis, mesh.hpp:25-40).
struct Axis {
    enum Map { sinh = 0, linear = 1, singleton = 2 };
    int n = 0;
    int map = linear;
    std::vector<double> z, j1, j2;
    double center = 0.0, alpha = 1.0, z0 = 0.0, z_inf = 1.0;
    double c1 = 0.0, c2 = 0.0;
    double dx() const { return n > 1 ? 1.0 / (n - 1) : 1.0; }
};

/// uniform_axis (mesh.cpp:46-62)
Axis make_uniform_axis(double z0, double z_inf, int n);
/// build_axis (mesh.cpp:16-44)
Axis make_sinh_axis(double center, double alpha, double z0, double z_inf, int n);
/// physical_to_computational (mesh.cpp:75-92)
double physical_to_computational(const Axis& axis, double z);

/// Date-0 discount curve (reference InitialCurve, curve.hpp:11-61).
class Curve {
public:
    Curve() = default;
    static Curve flat(double base);                                      // curve.cpp:11-20
    static Curve from_nodes(std::vector<std::pair<double, double>> nodes);  // curve.cpp:22-48
    double discount(double maturity) const;      // curve.cpp:135-144
    double forward(double t) const;              // curve.cpp:146-152
    double forward_slope(double t) const;        // curve.cpp:154-160

private:
    void fit();                                  // curve.cpp:68-127
    int interval(double t) const;                // curve.cpp:129-133
    bool flat_ = true;
    double flat_fwd_ = 0.0;
    std::vector<double> knots_, a_, b_, c_, d_;
    double t_max_ = 1e9, extrap_ = 0.0, log_p_max_ = 0.0;
};

/// g_factor (model.cpp:41-46)
double g_factor(double s, double kappa);
/// zcb_closed_form (model.cpp:48-54)
double zcb_closed_form(double t, double maturity, double x, double y, const Curve& curve,
                       double kappa);

}  // namespace hjmsv_b200
