// select_simt.cu -- steps a1 + a2 with SIMT fp32 arithmetic: sub-key scoring
// (Eq. S_old) and per-half argtopk.
//
// Used for the fp32 configurations (BASELINE.json configs[0], configs[2]),
// whose scores must be fp32-accurate: every score is
// an fp32 FMA chain over d_h in ascending order.  The bf16 configurations use
// the tcgen05 kernel in select_tc.cu.
#include "common.cuh"
#include "kernels.h"

namespace msn {
namespace {

constexpr int TB = 64;   // queries per tile
constexpr int TN = 64;   // keys per tile
constexpr int TK = 16;   // reduction chunk

// S[b, h, half, n] = sum_e Q[b,h,half,e] * K[h,half,n,e]
template <typename T>
__global__ void __launch_bounds__(256) score_kernel(const T* __restrict__ Q, const T* __restrict__ K,
                                                    float* __restrict__ S, int64_t B, int H,
                                                    int n_sub, int d_h) {
  pdl_enter();
  __shared__ float As[TK][TB + 4];
  __shared__ float Bs[TK][TN + 4];
  const int hh = blockIdx.z;  // h*2 + half
  const int64_t b0 = (int64_t)blockIdx.y * TB;
  const int n0 = blockIdx.x * TN;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  float acc[4][4] = {};
  for (int kk = 0; kk < d_h; kk += TK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int id = tid + i * 256, r = id / TK, c = id % TK;
      const int64_t b = b0 + r;
      As[c][r] = (b < B && kk + c < d_h)
                     ? elem<T>::to_f(Q[((b * H) * 2 + hh) * (int64_t)d_h + kk + c])
                     : 0.f;
      const int n = n0 + r;
      Bs[c][r] = (n < n_sub && kk + c < d_h)
                     ? elem<T>::to_f(K[((int64_t)hh * n_sub + n) * d_h + kk + c])
                     : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < TK; ++c) {
      float a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[c][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[c][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t b = b0 + ty * 4 + i;
    if (b >= B) continue;
    float* row = S + ((b * H) * 2 + hh) * (int64_t)n_sub;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < n_sub) row[n] = acc[i][j];
    }
  }
}

// One warp per (b, h, half) row: k rounds of warp-wide argmax over the
// composite (score desc, index asc) keys held in registers.
template <int NPL>
__global__ void __launch_bounds__(256) topk_rows_kernel(const float* __restrict__ S, int64_t rows,
                                                        int n_sub, int k, uint2* __restrict__ vc,
                                                        int32_t* __restrict__ cn) {
  pdl_enter();
  const int64_t row = (int64_t)blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  const float* s = S + row * n_sub;
  uint64_t c[NPL];
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    const int col = lane + 32 * j;
    c[j] = col < n_sub ? sel_key(s[col], (uint32_t)col) : 0ull;
  }
  for (int t = 0; t < k; ++t) {
    uint64_t best = 0;
#pragma unroll
    for (int j = 0; j < NPL; ++j) best = c[j] > best ? c[j] : best;
    best = warp_max_u64(best);
#pragma unroll
    for (int j = 0; j < NPL; ++j)
      if (c[j] == best) c[j] = 0ull;
    if (lane == 0) {
      vc[row * kCandCap + t] = make_uint2(__float_as_uint(sel_key_score(best)), sel_key_index(best));
    }
  }
  if (lane == 0) cn[row] = k;
}

template <int NPL>
cudaError_t launch_topk(const float* S, int64_t rows, int n_sub, int k, const Cands& cd,
                        cudaStream_t st) {
  const int64_t blocks = (rows + 7) / 8;
  launch_pdl(topk_rows_kernel<NPL>, (unsigned)blocks, 256, 0, st, S, rows, n_sub, k, cd.vc, cd.n);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_select_simt(const Shape& s, const void* Q, const void* K, float* scores_ws,
                               const Cands& cd, cudaStream_t st, int* launches) {
  dim3 grid((s.n_sub + TN - 1) / TN, (unsigned)((s.B + TB - 1) / TB), s.H * 2);
  if (s.qk_dt == F32)
    launch_pdl(score_kernel<float>, grid, 256, 0, st, (const float*)Q, (const float*)K, scores_ws, s.B, s.H,
                                              s.n_sub, s.d_h);
  else
    launch_pdl(score_kernel<__nv_bfloat16>, grid, 256, 0, st, (const __nv_bfloat16*)Q,
                                                      (const __nv_bfloat16*)K, scores_ws, s.B,
                                                      s.H, s.n_sub, s.d_h);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ++*launches;
  const int64_t rows = s.B * s.H * 2;
  const int npl = (s.n_sub + 31) / 32;
  if (npl <= 1) e = launch_topk<1>(scores_ws, rows, s.n_sub, s.k, cd, st);
  else if (npl <= 2) e = launch_topk<2>(scores_ws, rows, s.n_sub, s.k, cd, st);
  else if (npl <= 4) e = launch_topk<4>(scores_ws, rows, s.n_sub, s.k, cd, st);
  else if (npl <= 8) e = launch_topk<8>(scores_ws, rows, s.n_sub, s.k, cd, st);
  else if (npl <= 16) e = launch_topk<16>(scores_ws, rows, s.n_sub, s.k, cd, st);
  else if (npl <= 32) e = launch_topk<32>(scores_ws, rows, s.n_sub, s.k, cd, st);
  else if (npl <= 64) e = launch_topk<64>(scores_ws, rows, s.n_sub, s.k, cd, st);
  else return cudaErrorNotSupported;
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace msn
