/* examples/capi_demo.c — the C-ABI from plain C (no C++ on the caller side):
 * host helpers that need no device (axes, curve, closed form), then, when a
 * CUDA device is present, one small ZCB march priced at the natural spot. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "hjmsv_b200.h"

int main(void) {
    enum { NR = 32, NV = 16, NY = 16 };
    static double rz[NR], rj1[NR], rj2[NR], vz[NV], vj1[NV], vj2[NV], yz[NY], yj1[NY], yj2[NY];
    if (hjmsv_uniform_axis(0.0, 25.0, NR, rz, rj1, rj2) || hjmsv_uniform_axis(0.0, 1.5, NV, vz, vj1, vj2) ||
        hjmsv_uniform_axis(0.0, 250.0, NY, yz, yj1, yj2)) {
        fprintf(stderr, "axis: %s\n", hjmsv_last_error());
        return 1;
    }
    hjmsv_curve curve = {HJMSV_CURVE_FLAT, 1.04, 0, NULL, NULL};
    double p5 = 0.0;
    if (hjmsv_zcb_closed_form(&curve, 0.05, 0.0, 5.0, 0.0, 0.0, &p5)) return 1;
    printf("{\"abi\": %d, \"p(0,5)\": %.15g}\n", hjmsv_abi_version(), p5);
    if (fabs(p5 - pow(1.04, -5.0)) > 1e-14) return 1;
    if (hjmsv_device_count() < 1) return 0;

    hjmsv_problem p = {0};
    p.r = (hjmsv_axis){NR, HJMSV_MAP_LINEAR, rz, rj1, rj2, 0.0, 1.0, 0.0, 25.0, 0.0, 0.0};
    p.v = (hjmsv_axis){NV, HJMSV_MAP_LINEAR, vz, vj1, vj2, 0.0, 1.0, 0.0, 1.5, 0.0, 0.0};
    p.y = (hjmsv_axis){NY, HJMSV_MAP_LINEAR, yz, yj1, yj2, 0.0, 1.0, 0.0, 250.0, 0.0, 0.0};
    p.model = (hjmsv_model){0.05, 0.15, 0.9, 0.4, 1.2, -0.3};
    p.curve = curve;
    p.r0 = 0.01;
    p.maturity = 5.0;
    p.instrument = HJMSV_INSTRUMENT_ZCB;
    p.n_steps = 60;
    p.time_levels = HJMSV_TIME_INDEXED;
    hjmsv_solver_config cfg;
    hjmsv_default_solver_config(&cfg);
    hjmsv_solver* h = NULL;
    double price = 0.0;
    if (hjmsv_solver_create(&p, 1, &cfg, 0, HJMSV_MODE_FAST, &h) || hjmsv_solver_run(h) ||
        hjmsv_solver_spot_prices(h, &price)) {
        fprintf(stderr, "solver: %s\n", hjmsv_last_error());
        if (h) hjmsv_solver_destroy(h);
        return 1;
    }
    hjmsv_solver_destroy(h);
    printf("{\"zcb_price\": %.15g, \"closed_form\": %.15g}\n", price, p5);
    return fabs(price - p5) < 1e-3 ? 0 : 1;
}
