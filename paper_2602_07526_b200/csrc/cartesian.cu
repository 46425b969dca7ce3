// cartesian.cu -- steps a3 + a4: the Cartesian-candidate top-k over I x J
// and the softmax weights (reading R1), one warp
// per lookup, all in registers and shared memory.
//
// Per-half order (a2).  Each half arrives as an unordered candidate list
// (a superset of its top-k, up to 64 entries, 128 for k > 32, see kernels.h);
// the warp sorts it with a bitonic network across lanes (shuffles; element
// e = r*32 + lane, composite order (score desc, index asc) -- reading R5)
// and keeps the first k: I (row half) and J (column half).
//
// Candidates.  With both per-half lists sorted descending, the score
// c(a,b) = S_row[I_a] + S_col[J_b] is non-increasing in a and in b (fp32
// rounding is monotone).  Two exact prunings bound the work:
//   * tau = max_a c(a, ceil(k/(a+1)) - 1) is a lower bound on the k-th best
//     score: the (a+1) x ceil(k/(a+1)) >= k cells above-left of that cell all
//     score >= it;
//   * the top-k under (score desc, flat asc) is a down-set of the k x k grid,
//     so every selected (a,b) satisfies (a+1)(b+1) <= k.
// tau is then raised by three interpolation steps: x is a valid bound as
// soon as >= k cells of the region b < k/(a+1) score >= x (a warp count of
// per-lane binary searches).
// Each lane a scans the prefix b < k/(a+1) with c(a,b) >= tau; these m
// candidates (k <= m <= sum_a floor(k/(a+1))) are ranked exactly by their
// 64-bit composite key (score desc, flat asc) and the first k are written in
// that order (reading R5).  Under fp32 rounding a dominated cell can tie a
// dominating one; such exact score ties fall under the tie tolerance of the
// parity rule.
#include "common.cuh"
#include "kernels.h"
#include "gate.cuh"
#include "warp_sort.cuh"
#include "gather_rows.cuh"

namespace msn {
namespace {

constexpr int kWarpsPerBlock = 8;
#ifndef MSN_CART_TAU_STEPS
#define MSN_CART_TAU_STEPS 3  // counted interpolation steps on tau (see the header)
#endif
#ifndef MSN_FUSED_TAU_STEPS
#define MSN_FUSED_TAU_STEPS 0  // ... and in the fused kernels (see below)
#endif
// ... in the standalone Cartesian kernel only: in the fused Cartesian +
// gather kernel the steps lengthen every query warp's serial prologue before
// its row stream (measured: C3 +88 us, C4 +57 us per step), so it keeps tau0
constexpr int kMaxHK = 256;  // H*k staged per warp in the fused kernel

// Per-warp scratch of one lookup's Cartesian stage.
template <int KMAX, int MAXC>
struct CartSmem {
  float sv2[KMAX];
  int32_t si2[KMAX];
  float sva[KMAX];     // the row half's sorted scores / indices / candidate offsets
  int32_t sia[KMAX];
  int32_t soff[KMAX];
  uint64_t cand[MAXC];
  uint64_t res[KMAX];
};

// One warp computes lookup l: writes idx/w[l*k + t] to global and, when
// s_idx/s_w are given, to shared memory too (for a fused gather).
template <int KMAX, int MAXC, int TAU_STEPS, int SEG>
__device__ __forceinline__ void cartesian_lookup(CartSmem<KMAX, MAXC>& sm, int64_t l,
                                                 const uint2* __restrict__ cand,
                                                 const int32_t* __restrict__ cand_n, int n_sub,
                                                 int k, int32_t* __restrict__ idx,
                                                 float* __restrict__ w, int32_t* s_idx,
                                                 float* s_w, int32_t tab_off, int SC) {
  constexpr int APL = KMAX / 32;  // rows a per lane
  const int lane = threadIdx.x % 32;

  float va[APL];
  int32_t ia[APL];
  // the list: [0, n0) u [CAP - n1, CAP) (the scorer's two appending ends);
  // both halves are loaded, then sorted together (two interleaved networks)
  constexpr int CAP = cand_cap(KMAX);
  constexpr int R = CAP / 32;
  uint64_t key[2][R];  // composite keys (score desc, index asc) as one u64
  bool joined[2] = {false, false};
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int64_t row = l * 2 + half;
    const uint2* rc = cand + row * SC * CAP;
    if constexpr (KMAX == 32 && SEG == 2) {
      // column segments (select_tc.cu): every list holds its columns >= the
      // WHOLE row's bound, so together they are a superset of the row's
      // top-k; when they are compact and total <= 64 (the common case,
      // ~1.2k) they are read as one list: entry e of the concatenation
      // lies in segment g = #{segments whose inclusive prefix <= e}
      const int ng = lane < SC ? cand_n[row * SC + lane] : 0;
      int incl = ng & 0xffff;
#pragma unroll
      for (int d = 1; d < kMaxSeg; d <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += o;
      }
      int pre[kMaxSeg];
#pragma unroll
      for (int g = 0; g < kMaxSeg; ++g) pre[g] = __shfl_sync(0xffffffffu, incl, g < SC ? g : SC - 1);
      const int total = pre[kMaxSeg - 1];
      if (__all_sync(0xffffffffu, (ng >> 16) == 0) && total <= 64) {
        joined[half] = true;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int e = r * 32 + lane;
          int g = 0, base = 0;
#pragma unroll
          for (int t = 0; t < kMaxSeg - 1; ++t)
            if (e >= pre[t]) {
              g = t + 1;
              base = pre[t];
            }
          const uint2 c = e < total ? rc[g * CAP + (e - base)] : make_uint2(0u, 0u);
          key[half][r] = e < total ? sel_key(__uint_as_float(c.x), c.y) : 0ull;
        }
      }
    }
    if (!joined[half]) {
      const uint32_t nn = (uint32_t)cand_n[row * SC];
      const int n0 = (int)(nn & 0xffffu), n1 = (int)(nn >> 16);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int e = r * 32 + lane;
        const bool in = e < n0 || e >= CAP - n1;
        const uint2 c = in ? rc[e] : make_uint2(0u, 0u);
        key[half][r] = in ? sel_key(__uint_as_float(c.x), c.y) : 0ull;
      }
    }
  }
  // (k <= 32: only the top 32 are used -- two 32-sorts and a merge)
  if constexpr (KMAX == 32 && R == 2) {
    warp_top32_of_64_n<2>(*reinterpret_cast<uint64_t (*)[2][2]>(&key));
  } else {
    warp_sort_u64<R>(key[0]);
    warp_sort_u64<R>(key[1]);
  }
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int64_t row = l * 2 + half;
    const uint2* rc = cand + row * SC * CAP;
    float v[2];
    int32_t ix[2];
    if constexpr (KMAX == 32 && SEG == 2) if (!joined[half]) {
      // the row's other column segments (SC == S lists, see select_tc.cu):
      // each sorted likewise, then the best 32 of the running list and it by
      // the half-cleaner max(A_i, B_31-i) and a 5-step bitonic merge (k <= 32)
      for (int sg = 1; sg < SC; ++sg) {
        const uint32_t nb = (uint32_t)cand_n[row * SC + sg];
        const int m0 = (int)(nb & 0xffffu), m1 = (int)(nb >> 16);
        uint64_t k1[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int e = r * 32 + lane;
          const bool in = e < m0 || e >= CAP - m1;
          const uint2 c = in ? rc[sg * CAP + e] : make_uint2(0u, 0u);
          k1[r] = in ? sel_key(__uint_as_float(c.x), c.y) : 0ull;
        }
        warp_top32_of_64(k1);
        const uint32_t blo = __shfl_sync(0xffffffffu, (uint32_t)k1[0], 31 - lane);
        const uint32_t bhi = __shfl_sync(0xffffffffu, (uint32_t)(k1[0] >> 32), 31 - lane);
        const uint64_t bk = ((uint64_t)bhi << 32) | blo;
        uint64_t c = key[half][0] > bk ? key[half][0] : bk;
#pragma unroll
        for (int stride = 16; stride > 0; stride >>= 1) {
          const uint64_t o = shfl_xor_u64(c, stride);
          c = ((lane & stride) == 0) == (o > c) ? o : c;
        }
        key[half][0] = c;
        key[half][1] = 0ull;
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      v[r] = key[half][r] ? sel_key_score(key[half][r]) : -INFINITY;
      ix[r] = key[half][r] ? (int32_t)sel_key_index(key[half][r]) : 0x7fffffff;
    }
    if (half == 0) {
#pragma unroll
      for (int u = 0; u < APL; ++u) {
        const int a = lane + 32 * u;
        va[u] = a < k ? v[u] : -INFINITY;
        ia[u] = a < k ? ix[u] : 0;
        if (a < k) {
          sm.sva[a] = v[u];
          sm.sia[a] = ix[u];
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < APL; ++u) {
        const int a = lane + 32 * u;
        if (a < k) {
          sm.sv2[a] = v[u];
          sm.si2[a] = ix[u];
        }
      }
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
      tau = fmaxf(tau, va[u] + sm.sv2[ba]);
    }
  }
  tau = warp_max(tau);
  // tighten tau: x is also a lower bound on the k-th best score as soon as
  // at least k cells of the region b < k/(a+1) score >= x (distinct cells);
  // three interpolation steps between tau and c(0, 0) take the ~1.9k cells
  // above the staircase bound down to ~1.15k (random scores, k = 32)
  {
    float hi = __shfl_sync(0xffffffffu, va[0], 0) + sm.sv2[0];
#pragma unroll 1
    for (int it = 0; it < TAU_STEPS; ++it) {
      const float x = tau + 0.35f * (hi - tau);
      if (!(x > tau)) break;  // warp-uniform
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < APL; ++u) {
        const int a = lane + 32 * u;
        if (a < k) {
          int lo = 0, len = k / (a + 1);
          while (len > 0) {
            const int h = len >> 1;
            if (va[u] + sm.sv2[lo + h] >= x) {
              lo += h + 1;
              len -= h + 1;
            } else {
              len = h;
            }
          }
          cnt += lo;
        }
      }
      cnt = __reduce_add_sync(0xffffffffu, cnt);
      if (cnt >= k) tau = x;
      else hi = x;
    }
  }
  // prefix lengths p_a = #{b < k/(a+1) : c(a, b) >= tau}: c(a, b) is
  // non-increasing in b (sorted halves, monotone rounding), so a binary search
  int p[APL];
  int mine = 0;
#pragma unroll
  for (int u = 0; u < APL; ++u) {
    const int a = lane + 32 * u;
    int lo = 0;
    if (a < k) {
      int len = k / (a + 1);
      while (len > 0) {
        const int h = len >> 1;
        if (va[u] + sm.sv2[lo + h] >= tau) {
          lo += h + 1;
          len -= h + 1;
        } else {
          len = h;
        }
      }
    }
    p[u] = lo;
    mine += lo;
  }
  // exclusive prefix in row order (rows 0..31 on the lanes, then 32..63)
  int m = 0;
#pragma unroll
  for (int u = 0; u < APL; ++u) {
    int incl = p[u];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += o;
    }
    const int a = lane + 32 * u;
    if (a < k) sm.soff[a] = m + incl - p[u];
    m += __shfl_sync(0xffffffffu, incl, 31);
  }
  (void)mine;
  __syncwarp();
  // candidate x (lane-parallel): row a = the last row with soff[a] <= x (p_a is
  // non-increasing in a, so every row before the empty tail is non-empty),
  // column b = x - soff[a]
  for (int x = lane; x < m; x += 32) {
    int a = 0, len = k;
    while (len > 1) {
      const int h = len >> 1;
      if (sm.soff[a + h] <= x) a += h;
      len -= h;
    }
    const int b = x - sm.soff[a];
    const float c = sm.sva[a] + sm.sv2[b];
    const uint32_t flat = (uint32_t)sm.sia[a] * (uint32_t)n_sub + (uint32_t)sm.si2[b];
    sm.cand[x] = sel_key(c, flat);
  }
  __syncwarp();
  // exact rank by composite key; keys are distinct (flat ids are distinct).
  // Up to 64 candidates (the common case): each lane ranks its two in one
  // pass over the list (one shared load per two comparisons).
  if (KMAX == 32 && m <= 64) {
    // k <= 32: the top 32 of the (distinct, nonzero) keys by two 32-sorts and
    // a merge; lane t holds the t-th
    uint64_t c[2] = {lane < m ? sm.cand[lane] : 0ull, lane + 32 < m ? sm.cand[lane + 32] : 0ull};
    warp_top32_of_64(c);
    if (lane < k) sm.res[lane] = c[0];
  } else if (KMAX == 32 && MAXC <= 128) {  // (m <= MAXC)
    uint64_t c[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) c[r] = lane + 32 * r < m ? sm.cand[lane + 32 * r] : 0ull;
    warp_top32_of_128(c);
    if (lane < k) sm.res[lane] = c[0];
  } else if (m <= 64) {
    const uint64_t k0 = lane < m ? sm.cand[lane] : ~0ull;
    const uint64_t k1 = lane + 32 < m ? sm.cand[lane + 32] : ~0ull;
    int r0 = 0, r1 = 0;
    for (int y = 0; y < m; ++y) {
      const uint64_t ky = sm.cand[y];
      r0 += ky > k0;
      r1 += ky > k1;
    }
    if (lane < m && r0 < k) sm.res[r0] = k0;
    if (lane + 32 < m && r1 < k) sm.res[r1] = k1;
  } else {
    for (int x = lane; x < m; x += 32) {
      const uint64_t kx = sm.cand[x];
      int r = 0;
      for (int y = 0; y < m; ++y) r += sm.cand[y] > kx;
      if (r < k) sm.res[r] = kx;
    }
  }
  __syncwarp();
  // softmax over the k selected scores, max = the first (reading R1)
  const float c0 = sel_key_score(sm.res[0]);
  float e[APL];
  float z = 0.f;
#pragma unroll
  for (int u = 0; u < APL; ++u) {
    const int t = lane + 32 * u;
    e[u] = t < k ? expf(sel_key_score(sm.res[t]) - c0) : 0.f;
    z += e[u];
  }
  z = warp_sum(z);
  const float inv = 1.0f / z;
#pragma unroll
  for (int u = 0; u < APL; ++u) {
    const int t = lane + 32 * u;
    if (t < k) {
      const int32_t f = (int32_t)sel_key_index(sm.res[t]) + tab_off;  // + g n: per-group tables
      const float wt = e[u] * inv;
      idx[l * k + t] = f;
      w[l * k + t] = wt;
      if (s_idx) {
        s_idx[t] = f;
        s_w[t] = wt;
      }
    }
  }
  __syncwarp();
}

template <int KMAX, int MAXC, int SEG>
__global__ void __launch_bounds__(256) cartesian_kernel(const uint2* __restrict__ cand,
                                                        const int32_t* __restrict__ cand_n,
                                                        int64_t L, int n_sub, int k,
                                                        int32_t* __restrict__ idx,
                                                        float* __restrict__ w, int H, int hg,
                                                        int32_t tab_stride, int SC) {
  pdl_enter();
  __shared__ CartSmem<KMAX, MAXC> sm[kWarpsPerBlock];
  const int wid = threadIdx.x / 32;
  const int64_t l = (int64_t)blockIdx.x * kWarpsPerBlock + wid;
  if (l >= L) return;
  cartesian_lookup<KMAX, MAXC, MSN_CART_TAU_STEPS, SEG>(sm[wid], l, cand, cand_n, n_sub, k, idx, w, nullptr,
                                                        nullptr, (int32_t)((l % H) / hg) * tab_stride, SC);
}

// a3 + a4 + a5 fused: one warp per query runs the Cartesian stage of its H
// lookups (ALU-bound) and then streams their H*k value rows (HBM-bound);
// warps in different phases overlap the two.  Same arithmetic and
// summation order as cartesian_kernel + gather_kernel.
template <int KMAX, int MAXC, typename VT, int VPL, int G, int U>
__global__ void __launch_bounds__(256) cartesian_gather_kernel(
    const uint2* __restrict__ cand,
    const int32_t* __restrict__ cand_n, int64_t B, int H, int n_sub, int k,
    int32_t* __restrict__ idx, float* __restrict__ w, const VT* __restrict__ V,
    float* __restrict__ out, int d_v, Gate gate, int og, int32_t tab_stride, int SC) {
  pdl_enter();
  constexpr int PER = elem<VT>::per16;
  constexpr int LG = 32 / G;
  __shared__ CartSmem<KMAX, MAXC> sm[kWarpsPerBlock];
  __shared__ int32_t s_idx[kWarpsPerBlock][kMaxHK];
  __shared__ float s_w[kWarpsPerBlock][kMaxHK];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t b = (int64_t)blockIdx.x * kWarpsPerBlock + wid;
  if (b >= B) return;
  for (int h = 0; h < H; ++h)
    cartesian_lookup<KMAX, MAXC, MSN_FUSED_TAU_STEPS, 1>(sm[wid], b * H + h, cand, cand_n, n_sub, k, idx, w,
                                 &s_idx[wid][h * k], &s_w[wid][h * k],
                                 (int32_t)(h / (H / og)) * tab_stride, SC);
  const int HK = H * k;
  const int g = lane / LG, gl = lane % LG;
  const int E = HK / og;  // entries per output group
  const int row_vecs = d_v / PER;
  for (int grp = 0; grp < og; ++grp) {
    float acc[VPL][PER];
    gather_rows_heads<VT, VPL, G, U, false>(s_idx[wid], s_w[wid], grp * (E / k), (grp + 1) * (E / k), k, V, d_v, acc);
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

// a3 + a4 + a5 fused per LOOKUP (small batches, the latency regime): warp w
// of a block runs the Cartesian stage of lookup l = 8 blockIdx + w, then
// gathers its k value rows into a partial row (gather_rows); the block holds
// 8 / H whole queries, whose H partials are added in head order -- the order
// of gather_rows_heads, so the result is bitwise that of the phase calls.
// Eight times the warps of the per-query kernel for the same batch (C5: 2048
// instead of 512), so a small batch fills the GPU.  k <= 32, d_v <= 512,
// H | 8, one output group, no gate.
constexpr int kLkMaxDv = 512;
#ifndef MSN_LK_MASK
#define MSN_LK_MASK true  // per-row index test in the per-lookup gather (A/B: false)
#endif
template <int MAXC, int SEG, typename VT, int VPL, int G, int U>
__global__ void __launch_bounds__(256) cartesian_gather_lookup_kernel(
    const uint2* __restrict__ cand, const int32_t* __restrict__ cand_n, int64_t B, int H, int n_sub, int k,
    int32_t* __restrict__ idx, float* __restrict__ w, const VT* __restrict__ V, float* __restrict__ out, int d_v,
    int SC) {
  pdl_enter();
  constexpr int PER = elem<VT>::per16;
  constexpr int LG = 32 / G;
  __shared__ CartSmem<32, MAXC> sm[kWarpsPerBlock];
  __shared__ int32_t s_idx[kWarpsPerBlock][32];
  __shared__ float s_w[kWarpsPerBlock][32];
  __shared__ __align__(16) float part[kWarpsPerBlock][kLkMaxDv];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t l = (int64_t)blockIdx.x * kWarpsPerBlock + wid;
  const int64_t L = B * H;
  if (l < L) {
    cartesian_lookup<32, MAXC, MSN_FUSED_TAU_STEPS, SEG>(sm[wid], l, cand, cand_n, n_sub, k, idx, w, s_idx[wid], s_w[wid], 0, SC);
    float p[VPL][PER];
#ifndef MSN_LK_NOGATHER
    gather_rows<VT, VPL, G, U, MSN_LK_MASK>(s_idx[wid], s_w[wid], 0, k, V, d_v, p);  // (MASK = false measured slower here in round 2 r02c: C5 +4 us)
#else
    // (experiment builds only: the Cartesian stage alone)
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int e = 0; e < PER; ++e) p[v][e] = s_w[wid][0];
#endif
    const int g = lane / LG, gl = lane % LG;
    const int row_vecs = d_v / PER;
    if (g == 0) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int vec = gl * VPL + v;
        if (vec < row_vecs) {
#pragma unroll
          for (int e = 0; e < PER; e += 4)
            *reinterpret_cast<float4*>(&part[wid][vec * PER + e]) = make_float4(p[v][e], p[v][e + 1], p[v][e + 2], p[v][e + 3]);
        }
      }
    }
  }
  __syncthreads();
  // the block's queries: out[b] = ((0 + p_0) + p_1) + ... (head order)
  const int qpb = kWarpsPerBlock / H;
  const int64_t b0 = (int64_t)blockIdx.x * qpb;
  for (int i = threadIdx.x; i < qpb * d_v; i += blockDim.x) {
    const int q = i / d_v, e = i - q * d_v;
    if (b0 + q >= B) break;
    float t = 0.f;
    for (int h = 0; h < H; ++h) t += part[q * H + h][e];
    out[(b0 + q) * d_v + e] = t;
  }
}

template <int SEG, typename VT>
cudaError_t dispatch_lookup(const Shape& s, const Cands& cd, int32_t* idx, float* w, const VT* V, float* out,
                            cudaStream_t st) {
  const int R = s.d_v * (int)sizeof(VT) / 16;
  const int64_t L = s.B * s.H;
  const unsigned blocks = (unsigned)((L + kWarpsPerBlock - 1) / kWarpsPerBlock);
#define LK(VPL, G, U)                                                                                        \
  launch_pdl(cartesian_gather_lookup_kernel<119, SEG, VT, VPL, G, U>, blocks, 256, 0, st, cd.vc, cd.n, s.B, s.H, \
             s.n_sub, s.k, idx, w, V, out, s.d_v, cd.SC)
  MSN_GATHER_DISPATCH(R, LK);
#undef LK
  return cudaGetLastError();
}

// a3 + a4 + ROUTE + the local shard's a5 (the row-sharded table, a9): one
// warp per local query runs the Cartesian stage of its H lookups (the tape
// idx / w), then turns its H k slots into records {local row, w} in their
// owners' windows for this query (in (h, t) order: the position of slot r is
// the number of earlier slots with the same owner), writes the per-owner
// counts and every slot's position, and gathers the slots this rank owns
// into its own partial row -- the same rows, order and arithmetic as the
// owner-side gather of a remote window.  With peer memory the record stores
// cross NVLink as they are issued.
struct OwnerDiv {
  FastDiv div;
  uint32_t rpr;
};
template <int KMAX, int MAXC, int SEG, typename VT, int VPL, int G, int U>
__global__ void __launch_bounds__(256) cartesian_route_kernel(
    const uint2* __restrict__ cand, const int32_t* __restrict__ cand_n, int64_t B, int H, int n_sub, int k,
    int32_t* __restrict__ idx, float* __restrict__ w, const VT* __restrict__ V, int d_v, int SC, RouteArgs ra,
    OwnerDiv od) {
  pdl_enter();
  constexpr int PER = elem<VT>::per16;
  constexpr int LG = 32 / G;
  __shared__ CartSmem<KMAX, MAXC> sm[kWarpsPerBlock];
  __shared__ int32_t s_idx[kWarpsPerBlock][kMaxHK];
  __shared__ float s_w[kWarpsPerBlock][kMaxHK];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t b = (int64_t)blockIdx.x * kWarpsPerBlock + wid;
  if (b >= B) return;
  for (int h = 0; h < H; ++h)
    cartesian_lookup<KMAX, MAXC, MSN_FUSED_TAU_STEPS, SEG>(sm[wid], b * H + h, cand, cand_n, n_sub, k, idx, w, &s_idx[wid][h * k],
                                         &s_w[wid][h * k], 0, SC);
  const int HK = H * k;
  const int P = ra.P;
  int base = 0;  // lane o < P: the records of owner o so far in this query's window
  for (int r0 = 0; r0 < HK; r0 += 32) {
    const int r = r0 + lane;
    int o = -1;
    int32_t row = 0;
    float wt = 0.f;
    if (r < HK) {
      const uint32_t f = (uint32_t)s_idx[wid][r];
      const uint32_t q = od.div.div(f);
      o = (int)q;
      row = (int32_t)(f - q * od.rpr);
      wt = s_w[wid][r];
    }
    int my = 0, add = 0;
#pragma unroll
    for (int q = 0; q < kMaxWorld; ++q) {
      if (q < P) {
        const unsigned m = __ballot_sync(0xffffffffu, o == q);
        const int bq = __shfl_sync(0xffffffffu, base, q);
        if (o == q) my = bq + __popc(m & ((1u << lane) - 1u));
        if (lane == q) add = __popc(m);
      }
    }
    base += add;
    if (r < HK) {
      int32_t* prow = nullptr;
      float* pw = nullptr;
#pragma unroll
      for (int q = 0; q < kMaxWorld; ++q)
        if (q == o) {
          prow = ra.row.p[q];
          pw = ra.w.p[q];
        }
      prow[b * HK + my] = row;
      pw[b * HK + my] = wt;
      ra.pos[b * HK + r] = my;
      s_idx[wid][r] = o == ra.rank ? row : -1;  // the local shard's rows, in place
    }
  }
  if (lane < P) {
    int32_t* pc = nullptr;
#pragma unroll
    for (int q = 0; q < kMaxWorld; ++q)
      if (q == lane) pc = ra.cnt.p[q];
    pc[b] = base;
  }
  __syncwarp();
  // the local shard's rows: masked slots (-1) load nothing and add 0
  float acc[VPL][PER];
  if (P == 1) gather_rows<VT, VPL, G, U, false>(s_idx[wid], s_w[wid], 0, HK, V, d_v, acc);  // (every row local)
  else gather_rows<VT, VPL, G, U, true>(s_idx[wid], s_w[wid], 0, HK, V, d_v, acc);
  const int g = lane / LG, gl = lane % LG;
  if (g == 0) {
    float* o = ra.part + b * d_v;
    const int row_vecs = d_v / PER;
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
  }
}

template <int KMAX, int MAXC, int SEG, typename VT>
cudaError_t dispatch_route(const Shape& s, const Cands& cd, int32_t* idx, float* w, const VT* V,
                           const RouteArgs& ra, cudaStream_t st) {
  const int R = s.d_v * (int)sizeof(VT) / 16;
  const unsigned blocks = (unsigned)((s.B + kWarpsPerBlock - 1) / kWarpsPerBlock);
  OwnerDiv od;
  od.div = FastDiv((uint32_t)ra.rpr);
  od.rpr = (uint32_t)ra.rpr;
#define ROUTE(VPL, G, U)                                                                             \
  launch_pdl(cartesian_route_kernel<KMAX, MAXC, SEG, VT, VPL, G, U>, blocks, 256, 0, st, cd.vc, cd.n, s.B, s.H, \
             s.n_sub, s.k, idx, w, V, s.d_v, cd.SC, ra, od)
  MSN_GATHER_DISPATCH(R, ROUTE);
#undef ROUTE
  return cudaGetLastError();
}

template <int KMAX, int MAXC, typename VT>
cudaError_t dispatch_fused(const Shape& s, const Cands& cd, int32_t* idx, float* w, const VT* V,
                           float* out, cudaStream_t st, const Gate& gate) {
  const int R = s.d_v * (int)sizeof(VT) / 16;
  const unsigned blocks = (unsigned)((s.B + kWarpsPerBlock - 1) / kWarpsPerBlock);
#define FUSED(VPL, G, U)                                                                      \
  launch_pdl(cartesian_gather_kernel<KMAX, MAXC, VT, VPL, G, U>, blocks, 256, 0, st,                   \
      cd.vc, cd.n, s.B, s.H, s.n_sub, s.k, idx, w, V, out, s.d_v, gate, s.og, (int32_t)s.tab_stride, cd.SC)
  MSN_GATHER_DISPATCH(R, FUSED);
#undef FUSED
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_cartesian_gather(const Shape& s, const Cands& cd, int32_t* idx, float* w,
                                    const void* V, float* out, cudaStream_t st, int* launches,
                                    const Gate& gate) {
  if (s.H * s.k > kMaxHK || s.row_begin != 0 || cd.S != 1) return cudaErrorNotSupported;
  cudaError_t e;
  if (s.k <= 32) {
    e = s.v_dt == F32 ? dispatch_fused<32, 119, float>(s, cd, idx, w, (const float*)V, out, st, gate)
                      : dispatch_fused<32, 119, __nv_bfloat16>(s, cd, idx, w, (const __nv_bfloat16*)V, out, st, gate);
  } else {
    e = s.v_dt == F32 ? dispatch_fused<64, 280, float>(s, cd, idx, w, (const float*)V, out, st, gate)
                      : dispatch_fused<64, 280, __nv_bfloat16>(s, cd, idx, w, (const __nv_bfloat16*)V, out, st, gate);
  }
  if (e == cudaSuccess) ++*launches;
  return e;
}

bool cartesian_gather_lookup_ok(const Shape& s) {
  return s.k <= 32 && s.d_v <= kLkMaxDv && s.H <= kWarpsPerBlock && kWarpsPerBlock % s.H == 0 && s.og == 1 &&
         s.tab_stride == 0 && s.row_begin == 0;
}

cudaError_t launch_cartesian_gather_lookup(const Shape& s, const Cands& cd, int32_t* idx, float* w, const void* V,
                                          float* out, cudaStream_t st, int* launches) {
  if (!cartesian_gather_lookup_ok(s) || cd.S != cd.SC) return cudaErrorNotSupported;
  if (s.B == 0) return cudaSuccess;
  const bool bf = s.v_dt != F32;
  cudaError_t e;
  if (cd.S > 1)
    e = bf ? dispatch_lookup<2, __nv_bfloat16>(s, cd, idx, w, (const __nv_bfloat16*)V, out, st)
           : dispatch_lookup<2, float>(s, cd, idx, w, (const float*)V, out, st);
  else
    e = bf ? dispatch_lookup<1, __nv_bfloat16>(s, cd, idx, w, (const __nv_bfloat16*)V, out, st)
           : dispatch_lookup<1, float>(s, cd, idx, w, (const float*)V, out, st);
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t launch_cartesian_route(const Shape& s, const Cands& cd, int32_t* idx, float* w, const void* V,
                                   const RouteArgs& ra, cudaStream_t st, int* launches) {
  if (s.H * s.k > kMaxHK || s.og != 1 || s.tab_stride || ra.P < 1 || ra.P > kMaxWorld) return cudaErrorNotSupported;
  if (s.B == 0) return cudaSuccess;
  const bool bf = s.v_dt != F32;
  cudaError_t e;
  if (s.k <= 32 && cd.S > 1 && cd.S == cd.SC)
    e = bf ? dispatch_route<32, 119, 2, __nv_bfloat16>(s, cd, idx, w, (const __nv_bfloat16*)V, ra, st)
           : dispatch_route<32, 119, 2, float>(s, cd, idx, w, (const float*)V, ra, st);
  else if (cd.S != 1)
    return cudaErrorNotSupported;
  else if (s.k <= 32)
    e = bf ? dispatch_route<32, 119, 1, __nv_bfloat16>(s, cd, idx, w, (const __nv_bfloat16*)V, ra, st)
           : dispatch_route<32, 119, 1, float>(s, cd, idx, w, (const float*)V, ra, st);
  else
    e = bf ? dispatch_route<64, 280, 1, __nv_bfloat16>(s, cd, idx, w, (const __nv_bfloat16*)V, ra, st)
           : dispatch_route<64, 280, 1, float>(s, cd, idx, w, (const float*)V, ra, st);
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t launch_cartesian(const Shape& s, const Cands& cd, int32_t* idx, float* w,
                             cudaStream_t st, int* launches) {
  const int64_t L = s.B * s.H;
  const unsigned blocks = (unsigned)((L + kWarpsPerBlock - 1) / kWarpsPerBlock);
  if (s.k <= 32 && cd.S > 1 && cd.S == cd.SC)
    launch_pdl(cartesian_kernel<32, 119, 2>, blocks, 256, 0, st, cd.vc, cd.n, L, s.n_sub, s.k, idx, w,
               s.H, s.H / s.og, (int32_t)s.tab_stride, cd.SC);
  else if (cd.S != 1)
    return cudaErrorNotSupported;
  else if (s.k <= 32)
    launch_pdl(cartesian_kernel<32, 119, 1>, blocks, 256, 0, st, cd.vc, cd.n, L, s.n_sub, s.k, idx, w,
               s.H, s.H / s.og, (int32_t)s.tab_stride, cd.SC);
  else if (s.k <= 64)
    launch_pdl(cartesian_kernel<64, 280, 1>, blocks, 256, 0, st, cd.vc, cd.n, L, s.n_sub, s.k, idx, w,
               s.H, s.H / s.og, (int32_t)s.tab_stride, cd.SC);
  else
    return cudaErrorNotSupported;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace msn
