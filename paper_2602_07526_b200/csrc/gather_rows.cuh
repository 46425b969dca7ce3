// gather_rows.cuh -- the weighted row sum of step a5 (Eq. vo_mem,
// PAPER.md:226-229) in a fixed order (reading R18): lane group g (of G) takes
// rows r0+g, r0+g+G, ... in ascending order, U rows in flight, an fp32 FMA
// chain per group, then the G group sums are combined by an xor tree.
// gather_rows_heads runs it over each head's k rows and adds the per-head
// partials in head order.
#pragma once
#include "common.cuh"

namespace msn {

// acc = sum over r in [r0, r1) with s_idx[r] >= 0 of s_w[r] * V[s_idx[r]],
// for the lane's VPL 16-byte vectors (vec = gl * VPL + v) of the row.  Every
// lane of the warp holds the full sum on return.  MASK = false: every index
// is a valid row (no per-row test, no zero fill: the same sum when none is
// masked).
template <typename VT, int VPL, int G, int U, bool MASK = true>
__device__ __forceinline__ void gather_rows(const int32_t* s_idx, const float* s_w, int r0, int r1,
                                            const VT* __restrict__ V, int d_v,
                                            float (&acc)[VPL][elem<VT>::per16]) {
  constexpr int PER = elem<VT>::per16;
  constexpr int LG = 32 / G;  // lanes per row
  const int lane = threadIdx.x % 32;
  const int g = lane / LG, gl = lane % LG;
  const int row_vecs = d_v / PER;
#pragma unroll
  for (int v = 0; v < VPL; ++v)
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[v][e] = 0.f;
  for (int base = r0 + g; base < r1; base += G * U) {
    uint4 x[U][VPL];
    float wt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = base + u * G;
      if constexpr (MASK) {
        const int f = r < r1 ? s_idx[r] : -1;
        wt[u] = f >= 0 ? s_w[r] : 0.f;
        const VT* row = V + (int64_t)(f >= 0 ? f : 0) * d_v;
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const int vec = gl * VPL + v;
          if (f >= 0 && vec < row_vecs) x[u][v] = ldg_nc_v4(row + vec * PER);
          else x[u][v] = make_uint4(0, 0, 0, 0);
        }
      } else {
        // (past r1: row 0 with weight 0 -- only in a ragged last group)
        const bool in = r < r1;
        const int f = in ? s_idx[r] : 0;
        wt[u] = in ? s_w[r] : 0.f;
        const VT* row = V + (int64_t)f * d_v;
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const int vec = gl * VPL + v;
          if (vec < row_vecs) x[u][v] = ldg_nc_v4(row + vec * PER);
          else x[u][v] = make_uint4(0, 0, 0, 0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        float f[PER];
        unpack16<VT>(x[u][v], f);
#pragma unroll
        for (int e = 0; e < PER; e += 2) ffma2(acc[v][e], acc[v][e + 1], f[e], f[e + 1], wt[u]);
      }
  }
#pragma unroll
  for (int m = LG; m < 32; m <<= 1)
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int e = 0; e < PER; ++e) acc[v][e] += __shfl_xor_sync(0xffffffffu, acc[v][e], m);
}

// The same sum organised by head (reading R18): the k rows of each head h in
// [h0, h1) into a partial, the partials added in ascending head order.  Every
// gather of the unsharded path uses this order -- per query (gather_kernel,
// gather_wide_kernel, cartesian_gather_kernel) or per lookup and then per
// query (cartesian_gather_lookup_kernel) -- so they agree bitwise.
template <typename VT, int VPL, int G, int U, bool MASK = true>
__device__ __forceinline__ void gather_rows_heads(const int32_t* s_idx, const float* s_w, int h0, int h1, int k,
                                                  const VT* __restrict__ V, int d_v,
                                                  float (&acc)[VPL][elem<VT>::per16]) {
  constexpr int PER = elem<VT>::per16;
#pragma unroll
  for (int v = 0; v < VPL; ++v)
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[v][e] = 0.f;
  for (int h = h0; h < h1; ++h) {
    float p[VPL][PER];
    gather_rows<VT, VPL, G, U, MASK>(s_idx, s_w, h * k, (h + 1) * k, V, d_v, p);
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int e = 0; e < PER; ++e) acc[v][e] += p[v][e];
  }
}

// (VPL, G, U) per row width R = d_v * sizeof(V) / 16 vectors (R <= 128).
#define MSN_GATHER_DISPATCH(R, X)                    \
  do {                                               \
    if ((R) > 128) return cudaErrorNotSupported;     \
    else if ((R) > 64) X(4, 1, 4);                   \
    else if ((R) > 32) X(2, 1, 8);                   \
    else if ((R) > 16) X(1, 1, 8);                   \
    else if ((R) > 8) X(1, 2, 8);                    \
    else if ((R) > 4) X(1, 4, 8);                    \
    else if ((R) > 2) X(1, 8, 8);                    \
    else if ((R) > 1) X(1, 16, 8);                   \
    else X(1, 32, 8);                                \
  } while (0)

}  // namespace msn
