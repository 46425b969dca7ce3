// gate.cuh -- the memory-gated fusion epilogue:
// x~ = x_in (.) g(v_o), Eq. gating PAPER.md:318-322 (g = tanh; the
// ablation's sigmoid / identity), applied where v_o is
// produced so that v_o and x~ leave the SM in the same pass.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace msn {

// x~ = x (.) g(v_o) for the lane's vectors of row b (f1 epilogue)
template <int VPL, int PER>
__device__ __forceinline__ void store_gated(const Gate& gate, int64_t b, int d_v, int gl,
                                            int row_vecs, const float (&acc)[VPL][PER]) {
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int vec = gl * VPL + v;
    if (vec < row_vecs) {
#pragma unroll
      for (int e = 0; e < PER; e += 4) {
        const int64_t off = b * d_v + vec * PER + e;
        const float4 x = *reinterpret_cast<const float4*>(gate.x + off);
        *reinterpret_cast<float4*>(gate.xt + off) =
            make_float4(x.x * gate_g(acc[v][e], gate.kind), x.y * gate_g(acc[v][e + 1], gate.kind),
                        x.z * gate_g(acc[v][e + 2], gate.kind), x.w * gate_g(acc[v][e + 3], gate.kind));
      }
    }
  }
}


}  // namespace msn
