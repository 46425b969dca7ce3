// warp_sort.cuh -- warp-wide ordering of (score, index) pairs under the
// selection order of reading R5 (score desc, index asc): a 64-element bitonic
// network across the 32 lanes of a warp (element e = r*32 + lane in register
// r), and the exact rescoring of an overflowed per-half candidate list.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace msn {

__device__ __forceinline__ bool before(float av, int32_t ai, float bv, int32_t bi) {
  return av > bv || (av == bv && ai < bi);
}
// One bitonic step over the 64 elements e = r*32 + lane (stride < 32: across
// lanes; stride 32: the two registers of a lane); `size` selects the
// direction of each run (size 64: the whole sequence descending).
__device__ __forceinline__ void bitonic_step64(float (&v)[2], int32_t (&ix)[2], int size, int stride) {
  const int lane = threadIdx.x % 32;
  if (stride == 32) {
    const bool sw = before(v[1], ix[1], v[0], ix[0]);
    const float a = sw ? v[1] : v[0], b = sw ? v[0] : v[1];
    const int32_t c = sw ? ix[1] : ix[0], d = sw ? ix[0] : ix[1];
    v[0] = a; v[1] = b; ix[0] = c; ix[1] = d;
    return;
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int e = r * 32 + lane;
    const float ov = __shfl_xor_sync(0xffffffffu, v[r], stride);
    const int32_t oi = __shfl_xor_sync(0xffffffffu, ix[r], stride);
    const bool lower = (e & stride) == 0;
    const bool desc = (e & size) == 0;
    const bool want_better = desc == lower;
    const bool other_better = before(ov, oi, v[r], ix[r]);
    if (want_better == other_better) { v[r] = ov; ix[r] = oi; }
  }
}
__device__ __forceinline__ void warp_sort64(float (&v)[2], int32_t (&ix)[2]) {
#pragma unroll
  for (int size = 2; size <= 64; size <<= 1)
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) bitonic_step64(v, ix, size, stride);
}

// The same network over composite u64 keys (larger = better, sel_key):
// one 64-bit comparison per exchange.
__device__ __forceinline__ void warp_sort64_u64(uint64_t (&x)[2]) {
  const int lane = threadIdx.x % 32;
#pragma unroll
  for (int size = 2; size <= 64; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride == 32) {
        const uint64_t a = x[0] > x[1] ? x[0] : x[1], b = x[0] > x[1] ? x[1] : x[0];
        x[0] = a;
        x[1] = b;
      } else {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int e = r * 32 + lane;
          const uint64_t o = shfl_xor_u64(x[r], stride);
          const bool lower = (e & stride) == 0;
          const bool desc = (e & size) == 0;
          // keep the better of the pair when (lower == desc), else the worse
          x[r] = (lower == desc) == (o > x[r]) ? o : x[r];
        }
      }
    }
  }
}

// Descending sort of 32 R composite keys (element e = r*32 + lane), R a power
// of 2: strides >= 32 exchange registers of a lane, smaller ones lanes.
template <int R>
__device__ __forceinline__ void warp_sort_u64(uint64_t (&x)[R]) {
  const int lane = threadIdx.x % 32;
#pragma unroll
  for (int size = 2; size <= 32 * R; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int r2 = r ^ (stride / 32);
          if (r2 > r) {
            const bool desc = ((r * 32 + lane) & size) == 0;
            const uint64_t a = x[r], b = x[r2];
            const bool sw = desc ? (b > a) : (a > b);
            x[r] = sw ? b : a;
            x[r2] = sw ? a : b;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int e = r * 32 + lane;
          const uint64_t o = shfl_xor_u64(x[r], stride);
          const bool lower = (e & stride) == 0;
          const bool desc = (e & size) == 0;
          x[r] = (lower == desc) == (o > x[r]) ? o : x[r];
        }
      }
    }
  }
}

// The 32 largest of 64 u64 keys x[0..1] (element e = r*32 + lane), sorted
// descending in x[0] (lane i: the i-th largest): each register is sorted as a
// 32-sequence, the half-cleaner max(A_i, B_{31-i}) keeps the top 32 of A u B
// as a bitonic sequence, and a 5-step bitonic merge sorts it -- 36 shuffle
// compare-exchange steps instead of the 41 of a full 64-sort.
template <int N>
__device__ __forceinline__ void warp_top32_of_64_n(uint64_t (&x)[N][2]) {
  // N independent sets, their steps interleaved (N shuffle chains in flight)
  const int lane = threadIdx.x % 32;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int n = 0; n < N; ++n)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const uint64_t o = shfl_xor_u64(x[n][r], stride);
          const bool lower = (lane & stride) == 0;
          const bool desc = size == 32 || (lane & size) == 0;  // (a 32-sequence ends descending)
          x[n][r] = (lower == desc) == (o > x[n][r]) ? o : x[n][r];
        }
    }
  }
  uint64_t c[N];
#pragma unroll
  for (int n = 0; n < N; ++n) {
    const uint32_t blo = __shfl_sync(0xffffffffu, (uint32_t)x[n][1], 31 - lane);
    const uint32_t bhi = __shfl_sync(0xffffffffu, (uint32_t)(x[n][1] >> 32), 31 - lane);
    const uint64_t b = ((uint64_t)bhi << 32) | blo;
    c[n] = x[n][0] > b ? x[n][0] : b;
  }
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1)
#pragma unroll
    for (int n = 0; n < N; ++n) {
      const uint64_t o = shfl_xor_u64(c[n], stride);
      c[n] = ((lane & stride) == 0) == (o > c[n]) ? o : c[n];
    }
#pragma unroll
  for (int n = 0; n < N; ++n) {
    x[n][0] = c[n];
    x[n][1] = 0ull;
  }
}
__device__ __forceinline__ void warp_top32_of_64(uint64_t (&x)[2]) {
  uint64_t (&y)[1][2] = *reinterpret_cast<uint64_t (*)[1][2]>(&x);
  warp_top32_of_64_n<1>(y);
}

// The 32 largest of 128 u64 keys (four registers), sorted descending in x[0]:
// the top 32 of each pair (interleaved), then the half-cleaner of the two and
// a merge.
__device__ __forceinline__ void warp_top32_of_128(uint64_t (&x)[4]) {
  const int lane = threadIdx.x % 32;
  uint64_t ab[2][2] = {{x[0], x[1]}, {x[2], x[3]}};
  warp_top32_of_64_n<2>(ab);
  const uint32_t blo = __shfl_sync(0xffffffffu, (uint32_t)ab[1][0], 31 - lane);
  const uint32_t bhi = __shfl_sync(0xffffffffu, (uint32_t)(ab[1][0] >> 32), 31 - lane);
  const uint64_t br = ((uint64_t)bhi << 32) | blo;
  uint64_t c = ab[0][0] > br ? ab[0][0] : br;
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) {
    const uint64_t o = shfl_xor_u64(c, stride);
    c = ((lane & stride) == 0) == (o > c) ? o : c;
  }
  x[0] = c;
  x[1] = x[2] = x[3] = 0ull;
}

// Exact per-half top list of lookup l when the scorer's candidate list
// overflowed (its two ends met): rescore all n_sub sub-keys of this
// (head, half) and keep the best 64 under (score desc, index asc).  32
// sub-keys per step: lane e holds elements [8e, 8e+8) of q and of each K row
// (coalesced 16-B loads), the 32 partial dots are summed across lanes by a
// 31-shuffle butterfly that leaves sub-key base+lane's score in lane lane;
// a step whose scores all lose to the current 64th is skipped, the others are
// sorted and merged into the running top-64 (half-cleaner against the
// reversed batch + bitonic merge).  Only reached on degenerate data (massive
// exact ties); d_h <= 256 (the tcgen05 scorer's limit).  Result in (v, ix) as
// warp_sort64 leaves it.
template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&x)[8]);
template <>
__device__ __forceinline__ void load8<float>(const float* p, float (&x)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
}
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float (&x)[8]) {
  unpack16<__nv_bfloat16>(*reinterpret_cast<const uint4*>(p), x);
}
template <typename T>
__device__ __forceinline__ int exact_half_topk(const Rescore rq, int64_t l, int half, int H, int n_sub,
                                            uint2* vc, int col0 = 0, int ncols = -1) {
  // columns [col0, col0 + ncols) of the row (a column segment; default all)
  if (ncols < 0) ncols = n_sub;
  const int lane = threadIdx.x % 32;
  float v[2];
  int32_t ix[2];
  const int h = (int)(l % H);
  const int d = rq.d_h;
  const bool mine = lane * 8 < d;
  const T* q = (const T*)rq.Q + (l * 2 + half) * (int64_t)d;
  const T* kb = (const T*)rq.K + ((int64_t)(h * 2 + half) * n_sub + col0) * d + lane * 8;
  float qs[8];
  if (mine) load8<T>(q + lane * 8, qs);
  else
#pragma unroll
    for (int e = 0; e < 8; ++e) qs[e] = 0.f;
  v[0] = v[1] = -INFINITY;
  ix[0] = ix[1] = 0x7fffffff;
  for (int base = 0; base < ncols; base += 32) {
    float part[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      float acc = 0.f;
      if (mine && base + r < ncols) {
        float x[8];
        load8<T>(kb + (int64_t)(base + r) * d, x);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = fmaf(qs[e], x[e], acc);
      }
      part[r] = acc;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const bool upper = (lane & off) != 0;
#pragma unroll
      for (int j = 0; j < off; ++j) {
        const float send = upper ? part[j] : part[j + off];
        const float keep = upper ? part[j + off] : part[j];
        part[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    const int i = base + lane;
    float nv[2] = {i < ncols ? part[0] + 0.0f : -INFINITY, -INFINITY};
    int32_t ni[2] = {i < ncols ? col0 + i : 0x7fffffff, 0x7fffffff};
    const float wv = __shfl_sync(0xffffffffu, v[1], 31);  // current 64th
    const int32_t wi = __shfl_sync(0xffffffffu, ix[1], 31);
    if (!__any_sync(0xffffffffu, before(nv[0], ni[0], wv, wi))) continue;
    warp_sort64(nv, ni);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float ov = __shfl_sync(0xffffffffu, nv[1 - r], 31 - lane);
      const int32_t oi = __shfl_sync(0xffffffffu, ni[1 - r], 31 - lane);
      if (before(ov, oi, v[r], ix[r])) { v[r] = ov; ix[r] = oi; }
    }
#pragma unroll
    for (int stride = 32; stride > 0; stride >>= 1) bitonic_step64(v, ix, 64, stride);
  }
  // the row's new candidate list: its best min(64, ncols) sub-keys
  const int n = ncols < 64 ? ncols : 64;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int e = r * 32 + lane;
    if (e < n) vc[e] = make_uint2(__float_as_uint(v[r]), (uint32_t)ix[r]);
  }
  __syncwarp();
  return n;
}

}  // namespace msn
