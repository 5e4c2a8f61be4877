// kernels_fast.cu — FAST-mode step (placeholder until the fused kernels land).
#include "device_types.hpp"

namespace hjmsv_b200 {
bool fast_supported(int, int, int) { return false; }
int fast_stride(int, int, int) { return 1; }
void fast_prepare(const BatchView&, cudaStream_t) {}
void fast_step(const BatchView&, int, cudaStream_t, long long*) {}
void fast_explicit(const BatchView&, int, cudaStream_t) {}
}  // namespace hjmsv_b200
