// gather.cu -- step a5: sparse gather + weighted sum over the value table,
// v_o = sum_{(i,j) in K} w_ij V[i*n_sub + j]  (Eq. vo_mem, PAPER.md:226-229,
// readings R1, R2), summed over heads (reading R7).
//
// HBM-bound: each lookup moves k value rows (k * d_v * sizeof(V) bytes).
// One warp per query streams its H*k rows with 128-bit non-coherent loads
// (ld.global.nc.L1::no_allocate.v4), U rows in flight per lane group, fp32
// accumulation in registers in a fixed (h, t) order (gather_rows.cuh over
// all H*k rows of an output group).  A row of R 16-byte vectors is covered by 32/G lanes (G
// rows per warp step when R < 32, VPL vectors per lane when R > 32).
#include "common.cuh"
#include "kernels.h"
#include "gate.cuh"
#include "gather_rows.cuh"

namespace msn {
namespace {

constexpr int kWarps = 8;
constexpr int kMaxHK = 512;  // H*k entries staged per warp

template <typename VT, int VPL, int G, int U>
__global__ void __launch_bounds__(256) gather_kernel(const int32_t* __restrict__ idx,
                                                     const float* __restrict__ w,
                                                     const VT* __restrict__ V,
                                                     float* __restrict__ out, int64_t B, int H, int k,
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
  const int HK = H * k;
  for (int r = lane; r < HK; r += 32) {
    const int64_t f = idx[b * HK + r];
    const bool local = f >= row_begin && f < row_end;
    s_idx[wid][r] = local ? (int32_t)(f - row_begin) : -1;
    s_w[wid][r] = w[b * HK + r];
  }
  __syncwarp();
  const int g = lane / LG, gl = lane % LG;
  const int row_vecs = d_v / PER;
  const int hpg = H / og;  // heads per output group (og = 1: all)
  for (int grp = 0; grp < og; ++grp) {
    float tot[VPL][PER];
    gather_rows_heads<VT, VPL, G, U>(s_idx[wid], s_w[wid], grp * hpg, (grp + 1) * hpg, k, V, d_v, tot);
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
                make_float4(tot[v][e], tot[v][e + 1], tot[v][e + 2], tot[v][e + 3]);
        }
      }
      if (gate.kind) store_gated<VPL, PER>(gate, orow, d_v, gl, row_vecs, tot);
    }
  }  // output groups
}

// Rows of R >= 64 16-byte vectors (e.g. d_v = 512 bf16): WPQ = R / 32 warps
// per query, each lane one 16-byte vector of every row.  Every output element
// is still one FMA chain over the query's rows in ascending order, the same
// additions as gather_kernel's VPL = R / 32 lanes (G = 1) and the fused
// kernel's: bitwise identical, with WPQ times the warps (small batches,
// e.g. C5, otherwise leave most SMs idle).
template <typename VT, int U>
__global__ void __launch_bounds__(256) gather_wide_kernel(const int32_t* __restrict__ idx,
                                                          const float* __restrict__ w,
                                                          const VT* __restrict__ V,
                                                          float* __restrict__ out, int64_t B, int HK,
                                                          int d_v, int wpq, int og, Gate gate, int k) {
  pdl_enter();
  constexpr int PER = elem<VT>::per16;
  __shared__ int32_t s_idx[kWarps][kMaxHK];
  __shared__ float s_w[kWarps][kMaxHK];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int qpb = kWarps / wpq;
  const int64_t b = (int64_t)blockIdx.x * qpb + wid / wpq;
  if (wid >= qpb * wpq || b >= B) return;  // (wpq divides kWarps for the R the launcher allows)
  const int vec = (wid % wpq) * 32 + lane;  // this lane's 16-byte vector of the row
  for (int r = lane; r < HK; r += 32) {
    s_idx[wid][r] = idx[b * HK + r];
    s_w[wid][r] = w[b * HK + r];
  }
  __syncwarp();
  const int E = HK / og;
  for (int grp = 0; grp < og; ++grp) {
    float acc[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = 0.f;
    // per head: the k rows into a partial, partials added in head order
    // (gather_rows_heads' order, gather_rows.cuh)
    for (int h0 = grp * E; h0 < (grp + 1) * E; h0 += k) {
      float part[PER];
#pragma unroll
      for (int e = 0; e < PER; ++e) part[e] = 0.f;
      for (int base = h0; base < h0 + k; base += U) {
        uint4 x[U];
        float wt[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int r = base + u;
          const int f = r < h0 + k ? s_idx[wid][r] : -1;
          wt[u] = f >= 0 ? s_w[wid][r] : 0.f;
          x[u] = f >= 0 ? ldg_nc_v4(V + (int64_t)f * d_v + vec * PER) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float f[PER];
          unpack16<VT>(x[u], f);
#pragma unroll
          for (int e = 0; e < PER; e += 2) ffma2(part[e], part[e + 1], f[e], f[e + 1], wt[u]);
        }
      }
#pragma unroll
      for (int e = 0; e < PER; ++e) acc[e] += part[e];
    }
    const int64_t orow = b * og + grp;
    float* o = out + orow * d_v + vec * PER;
#pragma unroll
    for (int e = 0; e < PER; e += 4) *reinterpret_cast<float4*>(o + e) = make_float4(acc[e], acc[e + 1], acc[e + 2], acc[e + 3]);
    if (gate.kind) {
#pragma unroll
      for (int e = 0; e < PER; e += 4) {
        const int64_t off = orow * d_v + vec * PER + e;
        const float4 xx = *reinterpret_cast<const float4*>(gate.x + off);
        *reinterpret_cast<float4*>(gate.xt + off) =
            make_float4(xx.x * gate_g(acc[e], gate.kind), xx.y * gate_g(acc[e + 1], gate.kind),
                        xx.z * gate_g(acc[e + 2], gate.kind), xx.w * gate_g(acc[e + 3], gate.kind));
      }
    }
  }
}

template <typename VT>
cudaError_t dispatch(const Shape& s, const int32_t* idx, const float* w, const VT* V, float* out,
                     cudaStream_t st, const Gate& gate) {
  const int R = s.d_v * (int)sizeof(VT) / 16;
  if ((R == 64 || R == 128) && s.row_begin == 0 &&
      s.row_end >= (int64_t)s.n_sub * s.n_sub * (s.tab_stride ? s.og : 1)) {
    const int wpq = R / 32, qpb = kWarps / wpq;
    launch_pdl(gather_wide_kernel<VT, 16>, (unsigned)((s.B + qpb - 1) / qpb), 256, 0, st, idx, w, V, out, s.B,
               s.H * s.k, s.d_v, wpq, s.og, gate, s.k);
    return cudaGetLastError();
  }
  const unsigned blocks = (unsigned)((s.B + kWarps - 1) / kWarps);
#define GATHER(VPL, G, U)                                                                      \
  launch_pdl(gather_kernel<VT, VPL, G, U>, blocks, 256, 0, st, idx, w, V, out, s.B, s.H, s.k, s.d_v, \
             s.row_begin, s.row_end, gate, s.og)
  MSN_GATHER_DISPATCH(R, GATHER);
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

namespace {
// out = recv[0] + recv[1] + ... in rank order, float4 per thread
__global__ void __launch_bounds__(256) reduce_partials_kernel(const float4* __restrict__ recv, int world,
                                                              int64_t n4, float4* __restrict__ out) {
  pdl_enter();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  float4 a = recv[i];
  for (int p = 1; p < world; ++p) {
    const float4 v = recv[(int64_t)p * n4 + i];
    a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
  }
  out[i] = a;
}
}  // namespace

cudaError_t launch_reduce_partials(const float* recv, int world, int64_t lb, int og, int d_v,
                                   float* out, cudaStream_t st, int* launches) {
  if (d_v % 4) return cudaErrorNotSupported;
  const int64_t n4 = lb * og * d_v / 4;
  if (n4 == 0) return cudaSuccess;
  launch_pdl(reduce_partials_kernel, (unsigned)((n4 + 255) / 256), 256, 0, st, (const float4*)recv, world,
             n4, (float4*)out);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace msn
