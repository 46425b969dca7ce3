// gate.cu -- backward of the memory-gated fusion:
// for x~ = x (.) g(v_o) (Eq. gating; gates of the ablation
// PAPER.md:492) and an upstream gradient dx~,
//   dx   = dx~ (.) g(v_o)            (=)
//   dv_o = dx~ (.) x (.) g'(v_o)     (=)  -> the d_out of msn_pkm_backward.
// Elementwise and HBM-bound (3 reads + 2 writes of fp32 per element).
#include "common.cuh"
#include "kernels.h"

namespace msn {
namespace {

__global__ void __launch_bounds__(256) gate_backward_kernel(const float4* __restrict__ x,
                                                            const float4* __restrict__ vo,
                                                            const float4* __restrict__ dxt,
                                                            float4* __restrict__ dx,
                                                            float4* __restrict__ dvo, int64_t n4,
                                                            int kind) {
  pdl_enter();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 a = x[i], v = vo[i], d = dxt[i];
    dx[i] = make_float4(d.x * gate_g(v.x, kind), d.y * gate_g(v.y, kind), d.z * gate_g(v.z, kind),
                        d.w * gate_g(v.w, kind));
    dvo[i] = make_float4(d.x * a.x * gate_dg(v.x, kind), d.y * a.y * gate_dg(v.y, kind),
                         d.z * a.z * gate_dg(v.z, kind), d.w * a.w * gate_dg(v.w, kind));
  }
}

}  // namespace

cudaError_t launch_gate_backward(int64_t B, int d_v, int kind, const float* x, const float* vo,
                                 const float* dxt, float* dx, float* dvo, cudaStream_t st,
                                 int* launches) {
  const int64_t n4 = B * d_v / 4;  // d_v % 8 == 0
  if (n4 == 0) return cudaSuccess;
  int64_t blocks = (n4 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  cudaError_t e = launch_pdl(gate_backward_kernel, (unsigned)blocks, 256, 0, st,
                             (const float4*)x, (const float4*)vo, (const float4*)dxt, (float4*)dx,
                             (float4*)dvo, n4, kind);
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace msn
