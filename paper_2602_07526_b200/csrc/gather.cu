// gather.cu -- step a5: sparse gather + weighted sum over the value table,
// v_o = sum_{(i,j) in K} w_ij V[i*n_sub + j]  (Eq. vo_mem, PAPER.md:226-229,
// readings R1, R2), summed over heads (reading R7).
//
// HBM-bound: each lookup moves k value rows (k * d_v * sizeof(V) bytes).
// One warp per query streams its H*k rows with 128-bit non-coherent loads
// (ld.global.nc.L1::no_allocate.v4), U rows in flight per lane group, fp32
// accumulation in registers in a fixed (h, t) order.  A row of R 16-byte
// vectors is covered by 32/G lanes (G rows per warp step when R < 32, VPL
// vectors per lane when R > 32).
#include "common.cuh"
#include "kernels.h"
#include "gate.cuh"

namespace msn {
namespace {

constexpr int kWarps = 8;
constexpr int kMaxHK = 512;  // H*k entries staged per warp

template <typename VT, int VPL, int G, int U>
__global__ void __launch_bounds__(256) gather_kernel(const int32_t* __restrict__ idx,
                                                     const float* __restrict__ w,
                                                     const VT* __restrict__ V,
                                                     float* __restrict__ out, int64_t B, int HK,
                                                     int d_v, int64_t row_begin,
                                                     int64_t row_end, Gate gate, int og) {
  pdl_enter();
  constexpr int PER = elem<VT>::per16;
  constexpr int LG = 32 / G;  // lanes per row
  __shared__ int32_t s_idx[kWarps][kMaxHK];
  __shared__ float s_w[kWarps][kMaxHK];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t b = (int64_t)blockIdx.x * kWarps + wid;
  if (b >= B) return;
  for (int r = lane; r < HK; r += 32) {
    const int64_t f = idx[b * HK + r];
    const bool local = f >= row_begin && f < row_end;
    s_idx[wid][r] = local ? (int32_t)(f - row_begin) : -1;
    s_w[wid][r] = w[b * HK + r];
  }
  __syncwarp();
  const int g = lane / LG, gl = lane % LG;
  const int E = HK / og;  // entries of one output group (og = 1: all)
  for (int grp = 0; grp < og; ++grp) {
  float acc[VPL][PER];
#pragma unroll
  for (int v = 0; v < VPL; ++v)
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[v][e] = 0.f;
  const int row_vecs = d_v / PER;  // 16-byte vectors per row
  for (int base = grp * E + g; base < (grp + 1) * E; base += G * U) {
    uint4 x[U][VPL];
    float wt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = base + u * G;
      const int f = r < (grp + 1) * E ? s_idx[wid][r] : -1;
      wt[u] = f >= 0 ? s_w[wid][r] : 0.f;
      const VT* row = V + (int64_t)(f >= 0 ? f : 0) * d_v;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int vec = gl * VPL + v;
        if (f >= 0 && vec < row_vecs) x[u][v] = ldg_nc_v4(row + vec * PER);
        else x[u][v] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        float f[PER];
        unpack16<VT>(x[u][v], f);
#pragma unroll
        for (int e = 0; e < PER; ++e) acc[v][e] = fmaf(wt[u], f[e], acc[v][e]);
      }
  }
  // combine the G lane groups (fixed order)
#pragma unroll
  for (int m = LG; m < 32; m <<= 1)
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int e = 0; e < PER; ++e) acc[v][e] += __shfl_xor_sync(0xffffffffu, acc[v][e], m);
  if (g == 0) {
    const int64_t orow = b * og + grp;
    float* o = out + orow * d_v;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int vec = gl * VPL + v;
      if (vec < row_vecs) {
#pragma unroll
        for (int e = 0; e < PER; e += 4)
          *reinterpret_cast<float4*>(o + vec * PER + e) =
              make_float4(acc[v][e], acc[v][e + 1], acc[v][e + 2], acc[v][e + 3]);
      }
    }
    if (gate.kind) store_gated<VPL, PER>(gate, orow, d_v, gl, row_vecs, acc);
  }
  }  // output groups
}

template <typename VT>
cudaError_t dispatch(const Shape& s, const int32_t* idx, const float* w, const VT* V, float* out,
                     cudaStream_t st, const Gate& gate) {
  const int R = s.d_v * (int)sizeof(VT) / 16;
  const int HK = s.H * s.k;
  const unsigned blocks = (unsigned)((s.B + kWarps - 1) / kWarps);
#define GATHER(VPL, G, U)                                                                      \
  launch_pdl(gather_kernel<VT, VPL, G, U>, blocks, 256, 0, st, idx, w, V, out, s.B, HK, s.d_v,         \
                                                       s.row_begin, s.row_end, gate, s.og)
  if (R >= 128) { if (R > 128) return cudaErrorNotSupported; GATHER(4, 1, 4); }
  else if (R > 32) GATHER(2, 1, 8);
  else if (R > 16) GATHER(1, 1, 8);
  else if (R > 8) GATHER(1, 2, 8);
  else if (R > 4) GATHER(1, 4, 8);
  else if (R > 2) GATHER(1, 8, 8);
  else if (R > 1) GATHER(1, 16, 8);
  else GATHER(1, 32, 8);
#undef GATHER
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gather(const Shape& s, const int32_t* idx, const float* w, const void* V,
                          float* out, cudaStream_t st, int* launches, const Gate& gate) {
  if (s.H * s.k > kMaxHK) return cudaErrorNotSupported;
  cudaError_t e = s.v_dt == F32 ? dispatch<float>(s, idx, w, (const float*)V, out, st, gate)
                                : dispatch<__nv_bfloat16>(s, idx, w, (const __nv_bfloat16*)V, out, st, gate);
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace msn
