// kernels_mc.cu — the Monte Carlo validator on the device:
// run_path / simulate (montecarlo.cpp:38-139). One thread per path: Euler step
// of x = r - f(0,t), the integrating-factor step of y, a full-truncation Euler
// step of v, trapezoidal integral of r, then the discounted payout (1 for ZCB,
// caplet_payoff at the terminal state, montecarlo.cpp:142-160).
//
// Normals: Philox4x32-10 keyed by the seed, counter (path, step) -> two 53-bit
// uniforms -> Box-Muller, so a path's draws do not depend on the launch shape.
// The reference draws from one mt19937_64 stream per 8192-path batch, which is
// inherently sequential; this generator is a different (independent) sample,
// so device-vs-reference parity is statistical. Partial sums are reduced in a
// fixed order per block and summed by the host in block order (deterministic).
#include <cstdint>

#include "device_types.hpp"

namespace hjmsv_b200 {
namespace {

__device__ __forceinline__ void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
    constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
        const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        k0 += W0;
        k1 += W1;
    }
}

// uniform in (0, 1) from 64 random bits (53-bit mantissa, never 0 or 1)
__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
    const uint64_t m = (static_cast<uint64_t>(a) << 21) ^ (b >> 11);
    return (static_cast<double>(m) + 0.5) * 0x1.0p-53;
}

// per step s: steps[4s..4s+3] = f(0, (s+1) dt), lambda(s dt), gamma(s dt), eps(s dt)
// (the model functions at the step's start, montecarlo.cpp:55-58)
__global__ void __launch_bounds__(256) k_mc(McParams mp, const double* __restrict__ steps,
                                            double* __restrict__ partial) {
    __shared__ double ssum[256], ssq[256];
    const long long tid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    const uint32_t k0 = static_cast<uint32_t>(mp.seed), k1 = static_cast<uint32_t>(mp.seed >> 32);
    double sum = 0.0, sq = 0.0;
    for (long long path = tid; path < mp.n_paths; path += stride) {
        double x = 0.0, y = 0.0, v = 1.0, integral_r = 0.0;
        double r = mp.f0;
        for (int s = 0; s < mp.n_steps; ++s) {
            const double2 fl = __ldg(reinterpret_cast<const double2*>(steps) + 2 * s);      // f_next, lambda
            const double2 ge = __ldg(reinterpret_cast<const double2*>(steps) + 2 * s + 1);  // gamma, eps
            const double v_pos = mp.full_truncation ? fmax(v, 0.0) : fabs(v);
            const double r_pos = fmax(r, 0.0);
            const double eta = sqrt(v_pos) * fl.y * (r_pos > 0.0 ? pow(r_pos, ge.x) : 0.0);
            uint32_t c[4] = {static_cast<uint32_t>(path), static_cast<uint32_t>(path >> 32),
                             static_cast<uint32_t>(s), 0x48534d43u};
            philox10(c, k0, k1);
            const double u1 = u53(c[0], c[1]), u2 = u53(c[2], c[3]);
            const double rad = sqrt(-2.0 * log(u1));
            double sn, cs;
            sincospi(2.0 * u2, &sn, &cs);
            const double dw = rad * cs;
            const double dz = mp.rho * dw + mp.sq1mr2 * (rad * sn);  // correlated_normals
            x += (-mp.kappa * x + y) * mp.dt + eta * mp.sqrt_dt * dw;
            y = y * mp.decay_y + eta * eta * mp.dt * mp.decay_h;
            v += mp.theta * (1.0 - v_pos) * mp.dt + ge.y * sqrt(v_pos) * mp.sqrt_dt * dz;
            const double r_next = x + fl.x;
            integral_r += 0.5 * (r + r_next) * mp.dt;
            r = r_next;
        }
        double pay = 1.0;
        if (mp.caplet) {  // caplet_payoff at the terminal state (model.cpp:105-112)
            const double pb = mp.ratio * exp(-mp.g * x - 0.5 * mp.g * mp.g * y);
            const double value = 1.0 - mp.accrual * pb;
            pay = value > 0.0 ? value : 0.0;
        }
        const double sample = pay * exp(-integral_r);
        sum += sample;
        sq += sample * sample;
    }
    ssum[threadIdx.x] = sum;
    ssq[threadIdx.x] = sq;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {  // fixed-order tree
        if (threadIdx.x < o) {
            ssum[threadIdx.x] += ssum[threadIdx.x + o];
            ssq[threadIdx.x] += ssq[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = ssum[0];
        partial[2 * blockIdx.x + 1] = ssq[0];
    }
}

}  // namespace

void mc_simulate(const McParams& mp, const double* steps, double* partial, int blocks,
                 cudaStream_t stream) {
    k_mc<<<blocks, 256, 0, stream>>>(mp, steps, partial);
}

}  // namespace hjmsv_b200
