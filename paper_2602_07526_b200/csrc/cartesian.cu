// cartesian.cu -- steps a3 + a4: the Cartesian-candidate top-k over I x J
// and the softmax weights (reading R1), one warp
// per lookup, all in registers and shared memory.
//
// Candidates.  With both per-half lists sorted descending, the score
// c(a,b) = S_row[I_a] + S_col[J_b] is non-increasing in a and in b (fp32
// rounding is monotone).  Two exact prunings bound the work:
//   * tau = max_a c(a, ceil(k/(a+1)) - 1) is a lower bound on the k-th best
//     score: the (a+1) x ceil(k/(a+1)) >= k cells above-left of that cell all
//     score >= it;
//   * the top-k under (score desc, flat asc) is a down-set of the k x k grid,
//     so every selected (a,b) satisfies (a+1)(b+1) <= k.
// Each lane a scans the prefix b < k/(a+1) with c(a,b) >= tau; these m
// candidates (k <= m <= sum_a floor(k/(a+1))) are ranked exactly by their
// 64-bit composite key (score desc, flat asc) and the first k are written in
// that order (reading R5).  Under fp32 rounding a dominated cell can tie a
// dominating one; such exact score ties fall under the tie tolerance of the
// parity rule.
#include "common.cuh"
#include "kernels.h"

namespace msn {
namespace {

constexpr int kWarpsPerBlock = 8;

template <int KMAX, int MAXC>
__global__ void __launch_bounds__(256) cartesian_kernel(const float* __restrict__ topv,
                                                        const int32_t* __restrict__ topi,
                                                        int64_t L, int n_sub, int k,
                                                        int32_t* __restrict__ idx,
                                                        float* __restrict__ w) {
  constexpr int APL = KMAX / 32;  // rows a per lane
  __shared__ float sv2[kWarpsPerBlock][KMAX];
  __shared__ int32_t si2[kWarpsPerBlock][KMAX];
  __shared__ uint64_t cand[kWarpsPerBlock][MAXC];
  __shared__ uint64_t res[kWarpsPerBlock][KMAX];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t l = (int64_t)blockIdx.x * kWarpsPerBlock + wid;
  if (l >= L) return;
  const float* v1 = topv + (l * 2 + 0) * k;
  const float* v2 = topv + (l * 2 + 1) * k;
  const int32_t* i1 = topi + (l * 2 + 0) * k;
  const int32_t* i2 = topi + (l * 2 + 1) * k;

  float va[APL];
  int32_t ia[APL];
#pragma unroll
  for (int u = 0; u < APL; ++u) {
    const int a = lane + 32 * u;
    va[u] = a < k ? v1[a] : -INFINITY;
    ia[u] = a < k ? i1[a] : 0;
    if (a < k) {
      sv2[wid][a] = v2[a];
      si2[wid][a] = i2[a];
    }
  }
  __syncwarp();
  // tau: lower bound on the k-th best Cartesian score
  float tau = -INFINITY;
#pragma unroll
  for (int u = 0; u < APL; ++u) {
    const int a = lane + 32 * u;
    if (a < k) {
      const int ba = (k + a) / (a + 1) - 1;  // ceil(k/(a+1)) - 1 <= k-1
      tau = fmaxf(tau, va[u] + sv2[wid][ba]);
    }
  }
  tau = warp_max(tau);
  // prefix lengths p_a
  int p[APL];
  int mine = 0;
#pragma unroll
  for (int u = 0; u < APL; ++u) {
    const int a = lane + 32 * u;
    p[u] = 0;
    if (a < k) {
      const int lim = k / (a + 1);
      while (p[u] < lim && va[u] + sv2[wid][p[u]] >= tau) ++p[u];
    }
    mine += p[u];
  }
  // exclusive prefix over lanes
  int incl = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  const int m = __shfl_sync(0xffffffffu, incl, 31);
  int off = incl - mine;
#pragma unroll
  for (int u = 0; u < APL; ++u) {
    for (int q = 0; q < p[u]; ++q) {
      const float c = va[u] + sv2[wid][q];
      const uint32_t flat = (uint32_t)ia[u] * (uint32_t)n_sub + (uint32_t)si2[wid][q];
      cand[wid][off++] = sel_key(c, flat);
    }
  }
  __syncwarp();
  // exact rank by composite key; keys are distinct (flat ids are distinct)
  for (int x = lane; x < m; x += 32) {
    const uint64_t kx = cand[wid][x];
    int r = 0;
    for (int y = 0; y < m; ++y) r += cand[wid][y] > kx;
    if (r < k) res[wid][r] = kx;
  }
  __syncwarp();
  // softmax over the k selected scores, max = the first (reading R1)
  const float c0 = sel_key_score(res[wid][0]);
  float e[APL];
  float z = 0.f;
#pragma unroll
  for (int u = 0; u < APL; ++u) {
    const int t = lane + 32 * u;
    e[u] = t < k ? expf(sel_key_score(res[wid][t]) - c0) : 0.f;
    z += e[u];
  }
  z = warp_sum(z);
  const float inv = 1.0f / z;
#pragma unroll
  for (int u = 0; u < APL; ++u) {
    const int t = lane + 32 * u;
    if (t < k) {
      idx[l * k + t] = (int32_t)sel_key_index(res[wid][t]);
      w[l * k + t] = e[u] * inv;
    }
  }
}

}  // namespace

cudaError_t launch_cartesian(const Shape& s, const float* topv, const int32_t* topi,
                             int32_t* idx, float* w, cudaStream_t st, int* launches) {
  const int64_t L = s.B * s.H;
  const unsigned blocks = (unsigned)((L + kWarpsPerBlock - 1) / kWarpsPerBlock);
  if (s.k <= 32)
    cartesian_kernel<32, 119><<<blocks, 256, 0, st>>>(topv, topi, L, s.n_sub, s.k, idx, w);
  else if (s.k <= 64)
    cartesian_kernel<64, 280><<<blocks, 256, 0, st>>>(topv, topi, L, s.n_sub, s.k, idx, w);
  else
    return cudaErrorNotSupported;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace msn
