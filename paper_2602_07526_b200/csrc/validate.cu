// validate.cu -- tape validation (SURVEY 8(b) "Errors": out-of-range idx
// passed to a backward is checked only on request, via a device flag word).
//
// A tape (idx, w) [B, H, k] is what a4 produced: per
// lookup k DISTINCT slot ids of the lookup's own table (i * n_sub + j, plus
// g * n_sub^2 for per-group tables, f4) and softmax weights, finite and >= 0.
// One warp per lookup (b, h); lane owns slots t = lane and lane + 32 (k <= 64).
// The number of violating slots is added to *bad (the caller zeroes it).
#include "common.cuh"
#include "kernels.h"

namespace msn {
namespace {

__global__ void __launch_bounds__(256) validate_tape_kernel(const int32_t* __restrict__ idx,
                                                            const float* __restrict__ w,
                                                            int64_t L, int H, int k, int hpg,
                                                            int64_t n_tab, bool group_tables,
                                                            int32_t* __restrict__ bad) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t l = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (l >= L) return;
  const int h = (int)(l % H);
  const int64_t lo = group_tables ? (int64_t)(h / hpg) * n_tab : 0;
  int32_t f[2];
  float v[2];
  int nbad = 0;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int t = lane + 32 * u;
    f[u] = t < k ? idx[l * k + t] : 0;
    v[u] = t < k ? w[l * k + t] : 0.f;
    if (t < k) {
      if ((int64_t)f[u] < lo || (int64_t)f[u] >= lo + n_tab) ++nbad;
      if (!(v[u] >= 0.f && v[u] <= 1.f)) ++nbad;  // also catches NaN
    }
  }
  // duplicates: every slot compared with every other slot of the lookup
  for (int j = 0; j < k; ++j) {
    const int32_t fj = __shfl_sync(0xffffffffu, j < 32 ? f[0] : f[1], j & 31);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int t = lane + 32 * u;
      if (t < k && t != j && f[u] == fj) ++nbad;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) nbad += __shfl_xor_sync(0xffffffffu, nbad, o);
  if (lane == 0 && nbad) atomicAdd(bad, nbad);
}

}  // namespace

cudaError_t launch_validate_tape(const Shape& s, const int32_t* idx, const float* w, int32_t* bad,
                                 cudaStream_t st, int* launches) {
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  const int64_t L = s.B * s.H;
  if (L == 0) return cudaSuccess;
  const int64_t blocks = (L + 7) / 8;
  e = launch_pdl(validate_tape_kernel, (unsigned)blocks, 256, 0, st, idx, w, L, s.H, s.k,
                 s.H / s.og, (int64_t)s.n_sub * s.n_sub, s.tab_stride != 0, bad);
  if (launches) ++*launches;
  return e;
}

}  // namespace msn
