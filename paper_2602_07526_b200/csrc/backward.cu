// backward.cu -- steps a6-a8 of the PKM lookup: the value-table and sub-key
// gradients ("scatter-adds gradients into the value table", PAPER.md:332;
// gradient only through the selected scores, reading R10).
//
// Deterministic path (default, BASELINE.json configs[2] "deterministic
// sort-based scatter-add"):
//   1. group the contributions by destination row (key = slot row, record
//      = contribution id cid = (b*H + h)*k + t): atomic counts, one
//      contiguous segment per touched row, placement (see "grouping");
//   2. row-major reduce: one warp per row with <= 32 contributions; longer
//      rows in fixed 32-entry slices (one warp each, then the slice sums in
//      slice order); each row's record ids are sorted first, so the sum
//      order is fixed (bitwise repeatable), and the row is read and written
//      once (G = G + sum).  For dV the same pass computes
//      dw[cid] = <V[row], dOut[b]>, reading each touched value row ONCE.
//   3. ds = w (dw - sum w dw) (softmax Jacobian), dQ (=) per lookup, and one
//      record per distinct (lookup, half, sub-key) with the aggregated dS;
//   4. group the records by sub-key row and reduce them into dK (+=) the same
//      way (bf16 configs with n_sub <= 2048 use the tensor cores instead).
// Atomic path (MSN_FLAG_ATOMIC_BWD): query-major re-gather with
// red.global.add.v4.f32 into dV (non-deterministic summation order).
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace msn {
namespace {

// ------------------------------------------------------------ slices ------
// EPL consecutive elements of a row per lane (row width = 32 * EPL).
template <typename T, int EPL>
__device__ __forceinline__ void load_slice(const T* p, float* f) {
  constexpr int BYTES = EPL * (int)sizeof(T);
  if constexpr (BYTES % 16 == 0) {
#pragma unroll
    for (int i = 0; i < BYTES / 16; ++i) {
      const uint4 v = ldg_v4(reinterpret_cast<const char*>(p) + 16 * i);
      unpack16<T>(v, f + i * elem<T>::per16);
    }
  } else {
#pragma unroll
    for (int i = 0; i < EPL; ++i) f[i] = elem<T>::to_f(p[i]);
  }
}
// ------------------------------------------------------------- grouping ----
// Contributions are grouped by destination row without a global sort:
//   1. count  (fused into the kernel that makes the keys):
//      rank[p] = atomicAdd(&cnt[key[p]], 1)            -- arbitrary order;
//   2. grp_runs_kernel: every row with cnt > 0 gets a contiguous segment
//      [off, off + cnt) (warp-aggregated atomic allocation) and a run record
//      {off, cnt, row} in the short (cnt <= 32) or the long list;
//   3. grp_place_kernel: ent[off[key] + rank[p]] = (p, wts[p]) (one 8-byte store).
// The order inside a segment, and of the runs in their lists, is arbitrary;
// the reducers sort each run's record ids before summing, so every gradient
// row is summed in a fixed order (ascending record id inside a warp's slice)
// -- bitwise repeatable, independent of the atomics.
#ifndef MSN_SHORT_U
#define MSN_SHORT_U 2  // x rows in flight per warp in the short-run reducer (8 values/lane)
#endif
#ifndef MSN_V_PREFETCH
#define MSN_V_PREFETCH 2  // L2 prefetch of the value row this many runs ahead of its load (0: off)
#endif
#ifndef MSN_G_PREFETCH
#define MSN_G_PREFETCH 0  // L2 prefetch of the gradient row two runs ahead of its reduction (off: the
                          // red.add is fire-and-forget; a prefetched line evicted before it is read
                          // twice -- C4 DRAM reads 4.77 -> 4.54 GB, reducer 1252 -> 1225 us)
#endif
#ifndef MSN_SHORT_U4
#define MSN_SHORT_U4 4  // ... (<= 4 values/lane: fp32 rows of <= 128)
#endif
#ifndef MSN_SHORT_BPS4
#define MSN_SHORT_BPS4 4  // ... (<= 4 values/lane)
#endif
#ifndef MSN_SHORT_BPS
#define MSN_SHORT_BPS 4  // resident blocks per SM of the short-run reducer (8 values/lane)
#endif
constexpr int GRP_SHORT = 32;     // runs up to this length: one warp, one entry per lane
constexpr int GRP_SLICE = 32;     // long runs are reduced in slices of this many entries (one warp each)
constexpr int GRP_WARP_SORT = 1024;   // long runs sorted by one warp in registers up to this length
enum { CTL_TOTAL = 0, CTL_NSHORT = 1, CTL_NLONG = 2, CTL_NPIECES = 3, CTL_NHUGE = 4, CTL_SORTQ = 5,
       CTL_WORDS = 8 };
__host__ __device__ __forceinline__ uint32_t grp_npieces(uint32_t c) {
  return c > GRP_SHORT ? (c + GRP_SLICE - 1) / GRP_SLICE : 0u;
}
// sum of grp_npieces over runs of total length n (every run > 32 entries):
// <= n / 32 + (number of runs) <= n / 32 + n / 33
inline int64_t grp_pieces_max(int64_t n) { return n / GRP_SLICE + n / (GRP_SHORT + 1) + 2; }
// runs longer than GRP_WARP_SORT: <= n / 1025
inline int64_t grp_huge_max(int64_t n) { return n / (GRP_WARP_SORT + 1) + 1; }

// Each block owns a contiguous range of rows: pass 1 counts its entries,
// short and long runs and long-run pieces; one atomic per counter per block
// reserves its output ranges; pass 2 writes the offsets, the run records
// {offset, length, row, first piece} and the piece records {long run, j}
// (block-ordered: block scans over 1024-row rounds, 4 rows per thread).
__global__ void __launch_bounds__(256) grp_runs_kernel(const uint32_t* __restrict__ cnt,
                                                       uint32_t nrows, uint32_t* __restrict__ off,
                                                       uint4* __restrict__ runs_short,
                                                       uint4* __restrict__ runs_long,
                                                       uint4* __restrict__ pieces,
                                                       uint32_t* __restrict__ huge,
                                                       uint32_t* __restrict__ ctl) {
  pdl_enter();
  __shared__ uint32_t sh[4][8];
  __shared__ uint32_t s_base[4];
  const int tid = threadIdx.x, lane = tid % 32, wid = tid / 32;
  const int64_t per = ((int64_t)nrows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * per;
  int64_t r1 = r0 + per;
  if (r1 > nrows) r1 = nrows;
  if (r0 >= r1) return;
  // pass 1: block totals
  uint32_t t4[4] = {0, 0, 0, 0};
  for (int64_t r = r0 + tid; r < r1; r += 256) {
    const uint32_t c = cnt[r];
    t4[0] += c;
    t4[1] += (c > 0 && c <= GRP_SHORT);
    t4[2] += (c > GRP_SHORT);
    t4[3] += grp_npieces(c);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    t4[i] = (uint32_t)warp_sum_int((int)t4[i]);
    if (lane == 0) sh[i][wid] = t4[i];
  }
  __syncthreads();
  if (tid < 4) {
    uint32_t t = 0;
    for (int w = 0; w < 8; ++w) t += sh[tid][w];
    s_base[tid] = t ? atomicAdd(&ctl[tid], t) : 0u;  // CTL_TOTAL, CTL_NSHORT, CTL_NLONG, CTL_NPIECES
  }
  __syncthreads();
  uint32_t base = s_base[0], sb = s_base[1], lb = s_base[2], pb = s_base[3];
  __syncthreads();
  // pass 2: ordered rounds of 1024 rows, four consecutive rows per thread
  for (int64_t rr = r0; rr < r1; rr += 1024) {
    const int64_t rb = rr + (int64_t)tid * 4;
    uint32_t c[4], isl[4], np[4];
    uint32_t x[3] = {0u, 0u, 0u};  // this thread's totals: entries, (short | long << 16), pieces
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      c[i] = rb + i < r1 ? cnt[rb + i] : 0u;
      isl[i] = (c[i] > 0 && c[i] <= GRP_SHORT) | ((uint32_t)(c[i] > GRP_SHORT) << 16);
      np[i] = grp_npieces(c[i]);
      x[0] += c[i];
      x[1] += isl[i];
      x[2] += np[i];
    }
    const uint32_t own[3] = {x[0], x[1], x[2]};
    // block exclusive scans of the thread totals
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, x[i], d);
        if (lane >= d) x[i] += o;
      }
    }
    if (lane == 31) { sh[0][wid] = x[0]; sh[1][wid] = x[1]; sh[2][wid] = x[2]; }
    __syncthreads();
    uint32_t pre[3] = {0, 0, 0}, tot[3] = {0, 0, 0};
#pragma unroll
    for (int w = 0; w < 8; ++w) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const uint32_t v = sh[i][w];
        if (w < wid) pre[i] += v;
        tot[i] += v;
      }
    }
    __syncthreads();
    uint32_t ec = base + pre[0] + x[0] - own[0];
    uint32_t es = pre[1] + x[1] - own[1];
    uint32_t ep = pb + pre[2] + x[2] - own[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (c[i] > 0) {
        const int64_t r = rb + i;
        off[r] = ec;
        if (isl[i] & 0xffffu) {
          runs_short[sb + (es & 0xffffu)] = make_uint4(ec, c[i], (uint32_t)r, 0u);
        } else {
          const uint32_t li = lb + (es >> 16);
          runs_long[li] = make_uint4(ec, c[i], (uint32_t)r, ep);
          // slice j: {first entry, entries (<= GRP_SLICE), row, long run}
          for (uint32_t j = 0; j < np[i]; ++j)
            pieces[ep + j] = make_uint4(ec + j * GRP_SLICE, min((uint32_t)GRP_SLICE, c[i] - j * GRP_SLICE), (uint32_t)r, li);
          if (c[i] > (uint32_t)GRP_WARP_SORT) huge[atomicAdd(&ctl[CTL_NHUGE], 1u)] = li;  // (any order)
        }
      }
      ec += c[i];
      es += isl[i];
      ep += np[i];
    }
    base += tot[0];
    sb += tot[1] & 0xffffu;
    lb += tot[1] >> 16;
    pb += tot[2];
  }
}

__global__ void __launch_bounds__(256) grp_place_kernel(const uint32_t* __restrict__ keys,
                                                        const uint32_t* __restrict__ rank,
                                                        const uint32_t* __restrict__ off,
                                                        const float* __restrict__ wts, int64_t n,
                                                        uint32_t nrows, uint2* __restrict__ ent) {
  pdl_enter();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t k = keys[p];
  if (k >= nrows) return;
  const uint32_t pos = off[k] + rank[p];
  ent[pos] = make_uint2((uint32_t)p, __float_as_uint(wts[p]));  // (one 8-byte scattered store)
}

// ------------------------------------------------------------- reducers ----
// MODE_DV : record = cid,            weight = w[cid],    x = dOut[b],          G = dV (local rows),
//           dot: dw[cid] = <V[row], dOut[b]>
// MODE_DK : record = 2*cid + half,   weight = dsS[rec],  x = Q[b,h,half,:],    G = dK rows (h,half,i)
enum { MODE_DV = 0, MODE_DK = 1 };

struct GrpArgs {
  const uint2* ent;       // (record id, weight bits), grouped by row
  const float* wts;       // weight by record id
  const uint4* runs_short;
  const uint4* runs_long;
  const uint4* pieces;    // long-run slices {first entry, entries, row, long run}
  float* part;            // per-slice partial rows
  const uint32_t* ctl;
  const void* X;          // x rows (dOut fp32 or Q)
  const void* Y;          // V (MODE_DV dot)
  float* dots;            // dw (MODE_DV)
  float* G;               // gradient rows (+=)
  uint2* ent_rw;          // = ent (long runs: sorted in place)
  FastDiv div_hk, div_k;  // record -> query: / (H k), / k
  // head groups: the x row of record cid is (b, group of h)
  int og = 1, H = 1;
  FastDiv div_h, div_hg;  // / H, / (H / og)
  // MODE_DV fused optimiser update: instead of G += g,
  // V[row] <- V[row] - lr g (upd 1, SGD) or, with s[row] += g^2,
  // V[row] - lr g / (sqrt(s[row]) + eps) (upd 2, Adagrad); 0: G += g.
  int upd = 0;
  float lr = 0.f, eps = 0.f;
  float* state = nullptr;  // Adagrad accumulator [rows, D]
  void* Vw = nullptr;      // the value table, written in place
  // row-sharded backward over peer memory (MODE_DV, P2P kernels): x row r of
  // the global batch lives on rank r / xl (px[rank] + (r % xl) D) and dw[rec]
  // goes to rank rec / dl (pd[rank] + rec % dl)
  PerRank<const float> px{};
  PerRank<float> pd{};
  uint32_t xl = 0, dl = 0;
  FastDiv div_xl, div_dl;
  const uint32_t* huge = nullptr;  // long runs > GRP_WARP_SORT entries (indices into runs_long)
  uint32_t* ctl_rw = nullptr;      // = ctl (the sort's work queue counter)
  uint32_t* keys_rw = nullptr;     // scratch for the ids of runs too long for shared memory
  uint32_t id_shift = 0;           // record id >> id_shift < 256 (the huge runs' bucket)
};

// Applies the fused update to VW consecutive elements at element offset off
// of the value table: y = their current values, g = their gradients.
template <typename YT, int VW>
__device__ __forceinline__ void update_vec(const GrpArgs& a, int64_t off, const float* y,
                                           const float* g) {
  float nv[VW];
#pragma unroll
  for (int v = 0; v < VW; ++v) {
    if (a.upd == 2) {
      const float s = a.state[off + v] + g[v] * g[v];
      a.state[off + v] = s;
      nv[v] = y[v] - a.lr * g[v] / (sqrtf(s) + a.eps);
    } else {
      nv[v] = y[v] - a.lr * g[v];
    }
  }
  YT* p = reinterpret_cast<YT*>(a.Vw) + off;
  if constexpr (sizeof(YT) == 4) {
    if constexpr (VW == 4) *reinterpret_cast<float4*>(p) = make_float4(nv[0], nv[1], nv[2], nv[3]);
    else {
#pragma unroll
      for (int v = 0; v < VW; ++v) reinterpret_cast<float*>(p)[v] = nv[v];
    }
  } else {
    if constexpr (VW == 4) {
      const __nv_bfloat162 lo = __floats2bfloat162_rn(nv[0], nv[1]);
      const __nv_bfloat162 hi = __floats2bfloat162_rn(nv[2], nv[3]);
      *reinterpret_cast<uint2*>(p) = make_uint2(*reinterpret_cast<const uint32_t*>(&lo),
                                                *reinterpret_cast<const uint32_t*>(&hi));
    } else {
#pragma unroll
      for (int v = 0; v < VW; ++v) p[v] = __float2bfloat16_rn(nv[v]);
    }
  }
}

// Batched butterfly: U per-lane partial sums -> full warp sums, with
// (U - 1) + log2(32 / U) shuffles instead of 5U.  Dot u ends in lane
// u * (32 / U) (fixed order: deterministic).
template <int U>
__device__ __forceinline__ float multi_warp_sum(float (&d)[U]) {
  const int lane = threadIdx.x % 32;
  float v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = d[u];
  int n = U;
#pragma unroll
  for (int m = 16; m >= 32 / U; m >>= 1) {
    const bool hi = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < U / 2; ++i) {
      if (i < n / 2) {
        const float keep = hi ? v[i + n / 2] : v[i];
        const float send = hi ? v[i] : v[i + n / 2];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
      }
    }
    n >>= 1;
  }
  float r = v[0];
#pragma unroll
  for (int m = 32 / U / 2; m > 0; m >>= 1) r += __shfl_xor_sync(0xffffffffu, r, m);
  return r;
}

// Per-lane element ownership: vector i (< NVEC) of a row holds the VW
// elements e = (i*32 + lane)*VW + v, so every row load/store of a warp is a
// contiguous, coalesced transaction for fp32 and bf16 alike.
template <typename T, int VW>
__device__ __forceinline__ void ldg_vec(const T* p, float* f) {
  if constexpr (sizeof(T) == 4) {
    if constexpr (VW == 4) {
      const uint4 v = ldg_v4(p);
      f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
      f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
    } else {
#pragma unroll
      for (int i = 0; i < VW; ++i) f[i] = reinterpret_cast<const float*>(p)[i];
    }
  } else {
    if constexpr (VW == 4) {
      const uint2 v = *reinterpret_cast<const uint2*>(p);
      f[0] = __uint_as_float(v.x << 16); f[1] = __uint_as_float(v.x & 0xffff0000u);
      f[2] = __uint_as_float(v.y << 16); f[3] = __uint_as_float(v.y & 0xffff0000u);
    } else {
#pragma unroll
      for (int i = 0; i < VW; ++i) f[i] = elem<T>::to_f(p[i]);
    }
  }
}
// G += v for a row that receives exactly this one update: a fire-and-forget
// reduction performed in L2 (no load round trip on the SM); with a single
// addend per element the result is bitwise that of G = G + v.
template <int VW>
__device__ __forceinline__ void red_vec(float* p, const float* v) {
  if constexpr (VW == 4) red_add_v4(p, v[0], v[1], v[2], v[3]);
  else {
#pragma unroll
    for (int i = 0; i < VW; ++i) atomicAdd(p + i, v[i]);
  }
}
// the same with an L2 eviction-priority policy (common.cuh)
template <typename T, int VW>
__device__ __forceinline__ void ldg_vec_pol(const T* p, float* f, uint64_t pol) {
  if constexpr (sizeof(T) == 4 && VW == 4) {
    const uint4 v = ldg_v4_pol(p, pol);
    f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
  } else if constexpr (sizeof(T) == 2 && VW == 4) {
    const uint2 v = ldg_v2_pol(p, pol);
    f[0] = __uint_as_float(v.x << 16); f[1] = __uint_as_float(v.x & 0xffff0000u);
    f[2] = __uint_as_float(v.y << 16); f[3] = __uint_as_float(v.y & 0xffff0000u);
  } else {
    ldg_vec<T, VW>(p, f);
  }
}
template <int VW>
__device__ __forceinline__ void red_vec_pol(float* p, const float* v, uint64_t pol) {
  if constexpr (VW == 4) red_add_v4_pol(p, v[0], v[1], v[2], v[3], pol);
  else red_vec<VW>(p, v);
}
template <int VW>
__device__ __forceinline__ void stg_vec(float* p, const float* v) {
  if constexpr (VW == 4) *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  else if constexpr (VW == 2) *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  else p[0] = v[0];
}

template <int MODE>
__device__ __forceinline__ uint32_t grp_xrow(const GrpArgs& a, uint32_t rec) {
  if constexpr (MODE == MODE_DV) {
    if (a.og == 1) return a.div_hk.div(rec);
    const uint32_t bh = a.div_k.div(rec);  // b * H + h
    const uint32_t b = a.div_h.div(bh);
    return b * (uint32_t)a.og + a.div_hg.div(bh - b * (uint32_t)a.H);
  } else {
    return a.div_k.div(rec >> 1) * 2u + (rec & 1u);
  }
}

// Sums the entries src(j), j in [j0, j1), of one row into acc (in j order),
// U x rows in flight at a time; MODE_DV also writes dw[rec] = <y, x>.
template <int MODE, typename XT, int EPL, int U, bool P2P, typename Src>
__device__ __forceinline__ void grp_accumulate(const GrpArgs& a, int j0, int j1, Src src,
                                               const float* y, float* acc, uint64_t xpol) {
  constexpr int VW = EPL < 4 ? EPL : 4;
  constexpr int NVEC = EPL / VW;
  constexpr int D = 32 * EPL;
  const int lane = threadIdx.x % 32;
  const XT* __restrict__ X = reinterpret_cast<const XT*>(a.X) + lane * VW;
  for (int jb = j0; jb < j1; jb += U) {
    float x[U][EPL];
    float wt[U];
    uint32_t rec[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = jb + u;
      if (j < j1) {
        float w_;
        rec[u] = src(j, w_);
        wt[u] = w_;
        const int64_t xr = grp_xrow<MODE>(a, rec[u]);
        const XT* xrow;
        if (P2P) {  // the home rank's d_out row (peer memory)
          const uint32_t home = a.div_xl.div((uint32_t)xr);
          const float* hb = nullptr;
#pragma unroll
          for (int q = 0; q < kMaxWorld; ++q)
            if (q == (int)home) hb = a.px.p[q];
          xrow = reinterpret_cast<const XT*>(hb) + lane * VW + (int64_t)(xr - (int64_t)home * a.xl) * D;
        } else {
          xrow = X + xr * D;
        }
#pragma unroll
        for (int i = 0; i < NVEC; ++i) {
          // d_out rows (MODE_DV) are re-read by ~H k records each: kept in L2
          if constexpr (MODE == MODE_DV) ldg_vec_pol<XT, VW>(xrow + i * 32 * VW, x[u] + i * VW, xpol);
          else ldg_vec<XT, VW>(xrow + i * 32 * VW, x[u] + i * VW);
        }
      } else {
        rec[u] = 0xffffffffu;
        wt[u] = 0.f;
#pragma unroll
        for (int i = 0; i < EPL; ++i) x[u][i] = 0.f;
      }
    }
    float d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      d[u] = 0.f;
      if constexpr (EPL % 2 == 0) {
#pragma unroll
        for (int i = 0; i < EPL; i += 2) ffma2(acc[i], acc[i + 1], x[u][i], x[u][i + 1], wt[u]);
      } else {
#pragma unroll
        for (int i = 0; i < EPL; ++i) acc[i] = fmaf(wt[u], x[u][i], acc[i]);
      }
      if constexpr (MODE == MODE_DV) {
#pragma unroll
        for (int i = 0; i < EPL; ++i) d[u] = fmaf(y[i], x[u][i], d[u]);
      }
    }
    if constexpr (MODE == MODE_DV) {
      const float r = multi_warp_sum<U>(d);
      if ((lane % (32 / U)) == 0) {
        const int u = lane / (32 / U);
#pragma unroll
        for (int uu = 0; uu < U; ++uu)
          if (uu == u && rec[uu] != 0xffffffffu) {
            if (P2P) {  // dw straight into the home rank's buffer (one owner per element)
              const uint32_t home = a.div_dl.div(rec[uu]);
              float* hd = nullptr;
#pragma unroll
              for (int q = 0; q < kMaxWorld; ++q)
                if (q == (int)home) hd = a.pd.p[q];
              hd[rec[uu] - home * a.dl] = r;
            } else {
              a.dots[rec[uu]] = r;
            }
          }
      }
    }
  }
}

// Short runs (<= 32 entries): one warp per run, persistent grid-stride over
// the short-run list.  Lane j holds entry j; the warp ranks the record ids
// (entries are then consumed in ascending record order).  The value row
// (MODE_DV) and the first U x rows of a run are requested together; the next
// run's record, ids and weights are loaded one iteration ahead (the record
// after that two ahead), so a run costs about one memory round trip.  The
// row sum is added to G by one vector reduction per lane (red.global.add,
// performed in L2): the row's only update, so G = G + sum bitwise.
template <int MODE, typename XT, typename YT, int EPL, bool UPD, bool P2P>
__global__ void __launch_bounds__(256, (EPL >= 32 ? 1 : (EPL >= 16 ? 2 : (EPL >= 8 ? MSN_SHORT_BPS : MSN_SHORT_BPS4)))) grp_reduce_short_kernel(GrpArgs a) {
  pdl_enter();
  constexpr int VW = EPL < 4 ? EPL : 4;
  constexpr int NVEC = EPL / VW;
  constexpr int D = 32 * EPL;
  constexpr int U = EPL >= 16 ? 2 : (EPL >= 8 ? MSN_SHORT_U : MSN_SHORT_U4);
  const int lane = threadIdx.x % 32;
  const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32;
  int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int64_t nruns = a.ctl[CTL_NSHORT];
  const YT* __restrict__ Y = reinterpret_cast<const YT*>(a.Y) + lane * VW;
  float* __restrict__ Gl = a.G + lane * VW;
  const uint64_t pol_once = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();
  uint4 cur = c < nruns ? a.runs_short[c] : make_uint4(0, 0, 0, 0);
  uint4 nxt = c + nw < nruns ? a.runs_short[c + nw] : make_uint4(0, 0, 0, 0);
  uint32_t me = 0xffffffffu;
  float mw = 0.f;
  if (lane < (int)cur.y) {
    const uint2 e0 = a.ent[cur.x + lane];
    me = e0.x;
    mw = __uint_as_float(e0.y);
  }
  for (; c < nruns; c += nw) {
    const uint32_t key = cur.z;
    const int len = (int)cur.y;
    const uint32_t ce = me;
    const float cw = mw;
    float y[MODE == MODE_DV ? EPL : 1], acc[EPL];
    if constexpr (MODE == MODE_DV) {
#pragma unroll
      for (int i = 0; i < NVEC; ++i) ldg_vec_pol<YT, VW>(Y + (int64_t)key * D + i * 32 * VW, y + i * VW, pol_once);
    }
    // next run's entries and the record after it; that run's value row is
    // pulled into L2 now (two iterations ahead of its use, no registers held)
    const uint4 nn = c + 2 * nw < nruns ? a.runs_short[c + 2 * nw] : make_uint4(0, 0, 0, 0);
    if constexpr (MODE == MODE_DV) {
      constexpr int LINES = (D * (int)sizeof(YT) + 127) / 128;
      const uint4& pv = MSN_V_PREFETCH == 1 ? nxt : nn;  // (1: one run ahead, 2: two)
      if (MSN_V_PREFETCH && lane < LINES && c + MSN_V_PREFETCH * nw < nruns)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(a.Y) +
                                                       (int64_t)pv.z * D * (int)sizeof(YT) + lane * 128));
    }
    {  // ... and its gradient row, which the row's single reduction updates in L2
      constexpr int GLINES = (D * 4 + 127) / 128;
      if (MSN_G_PREFETCH && !UPD && lane >= 32 - GLINES && c + 2 * nw < nruns)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(a.G) +
                                                       (int64_t)nn.z * D * 4 + (31 - lane) * 128));
    }
    me = 0xffffffffu;
    mw = 0.f;
    if (lane < (int)nxt.y) {
      const uint2 e1 = a.ent[nxt.x + lane];
      me = e1.x;
      mw = __uint_as_float(e1.y);
    }
    // rank of this lane's record id among the run's
    uint32_t rk = 0;
    for (int i = 0; i < len; ++i) rk += __shfl_sync(0xffffffffu, ce, i) < ce;
    if (lane >= len) rk = 0xffffffffu;
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
    grp_accumulate<MODE, XT, EPL, U, P2P>(
        a, 0, len,
        [&](int j, float& w_) {
          const int s = __ffs(__ballot_sync(0xffffffffu, rk == (uint32_t)j)) - 1;
          w_ = __shfl_sync(0xffffffffu, cw, s);
          return __shfl_sync(0xffffffffu, ce, s);
        },
        y, acc, pol_keep);
    if constexpr (MODE == MODE_DV && UPD) {
#pragma unroll
      for (int i = 0; i < NVEC; ++i)
        update_vec<YT, VW>(a, (int64_t)key * D + (i * 32 + lane) * VW, y + i * VW, acc + i * VW);
    } else {
#pragma unroll
      for (int i = 0; i < NVEC; ++i) red_vec_pol<VW>(Gl + (int64_t)key * D + i * 32 * VW, acc + i * VW, pol_once);
    }
    cur = nxt;
    nxt = nn;
  }
}

// Ascending bitonic sort of P = 2^m keys (padding: 0xffffffff at the end)
// by the block, in shared or global memory; the variant whose every
// compare-exchange puts the minimum at the lower index, so elements past
// the real length (treated as +inf) never move and need no storage.
__device__ void block_bitonic(uint32_t* v, int L, int P) {
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));  // (i / j) * 2j + i % j
        // first step of a stage compares lo with its mirror inside the k-block
        const int b = (j == (k >> 1)) ? ((lo & ~(k - 1)) | (k - 1 - (lo & (k - 1)))) : lo + j;
        if (b >= L) continue;  // partner is +inf padding: nothing moves
        const uint32_t x = v[lo], y = v[b];
        if (y < x) {
          v[lo] = y;
          v[b] = x;
        }
      }
      __syncthreads();
    }
  }
}

// Warp-wide ascending bitonic sort of 32*R keys held as x[r] (element
// e = r*32 + lane): shuffles for strides < 32, register swaps above.
template <int R>
__device__ __forceinline__ void warp_sort_asc(uint32_t (&x)[R]) {
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
            const bool asc = ((r * 32 + lane) & size) == 0;
            const uint32_t a = x[r], b = x[r2];
            const bool sw = asc ? (a > b) : (a < b);
            x[r] = sw ? b : a;
            x[r2] = sw ? a : b;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int e = r * 32 + lane;
          const uint32_t o = __shfl_xor_sync(0xffffffffu, x[r], stride);
          const bool keep_min = ((e & stride) == 0) == ((e & size) == 0);
          x[r] = keep_min ? min(x[r], o) : max(x[r], o);
        }
      }
    }
  }
}

template <int R>
__device__ __forceinline__ void warp_sort_run(uint32_t* g, int L) {
  const int lane = threadIdx.x % 32;
  uint32_t x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) x[r] = r * 32 + lane < L ? g[r * 32 + lane] : 0xffffffffu;
  warp_sort_asc<R>(x);
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (r * 32 + lane < L) g[r * 32 + lane] = x[r];
}

// Long runs (> 32 entries), step 1: every run's record ids are sorted
// ascending in place, fixing its summation order, and its weights are
// rewritten in that order (ent[e] = (id, wts[id])).  Runs of more than
// GRP_WARP_SORT entries (the `huge` list, few) go first, one CTA each: a
// two-level sort in shared memory -- bucket by the id's top 8 bits (a
// counting pass), then every bucket sorted by a warp in registers (a bucket
// of more than GRP_WARP_SORT entries by the CTA) -- the ascending order of the
// run either way.  Then every warp takes the other runs from a work queue
// (one atomic per run), sorting each in registers -- so a CTA held up by a
// huge run does not hold up a static share of the short ones.
template <int R>
__device__ __forceinline__ void warp_sort_run_w(const GrpArgs& a, uint2* g, int L) {
  const int lane = threadIdx.x % 32;
  uint32_t x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) x[r] = r * 32 + lane < L ? g[r * 32 + lane].x : 0xffffffffu;
  warp_sort_asc<R>(x);
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (r * 32 + lane < L) g[r * 32 + lane] = make_uint2(x[r], __float_as_uint(a.wts[x[r]]));
}
// a warp sorts the (id, weight) pairs g[0, L) by id (L <= GRP_WARP_SORT)
__device__ __forceinline__ void warp_sort_pairs(const GrpArgs& a, uint2* g, int L) {
  if (L <= 32) warp_sort_run_w<1>(a, g, L);
  else if (L <= 64) warp_sort_run_w<2>(a, g, L);
  else if (L <= 128) warp_sort_run_w<4>(a, g, L);
  else if (L <= 256) warp_sort_run_w<8>(a, g, L);
  else if (L <= 512) warp_sort_run_w<16>(a, g, L);
  else warp_sort_run_w<32>(a, g, L);
}
// a warp sorts the ids g[0, L) (L <= GRP_WARP_SORT)
__device__ __forceinline__ void warp_sort_any(uint32_t* g, int L) {
  {
    if (L <= 1) return;
    if (L <= 32) warp_sort_run<1>(g, L);
    else if (L <= 64) warp_sort_run<2>(g, L);
    else if (L <= 128) warp_sort_run<4>(g, L);
    else if (L <= 256) warp_sort_run<8>(g, L);
    else if (L <= 512) warp_sort_run<16>(g, L);
    else warp_sort_run<32>(g, L);
  }
}
constexpr int GRP_BUCKET_SMEM = 8192;  // huge runs bucket-sorted in shared memory up to this length
constexpr int GRP_SORT_SMEM_BYTES = (2 * GRP_BUCKET_SMEM + 2 * 256 + 8) * 4;

__global__ void __launch_bounds__(256) grp_sort_long_kernel(GrpArgs a) {
  pdl_enter();
  extern __shared__ __align__(16) uint32_t s_sort[];  // [2 * GRP_BUCKET_SMEM + 2 * 256 + 8]
  const int tid = threadIdx.x, lane = tid % 32, wid = tid / 32;
  const int64_t nruns = a.ctl[CTL_NLONG];
  const int64_t nhuge = a.ctl[CTL_NHUGE];
  for (int64_t h = blockIdx.x; h < nhuge; h += gridDim.x) {
    const uint4 run = a.runs_long[a.huge[h]];
    const int L = (int)run.y;
    uint2* g = a.ent_rw + run.x;
    if (L > GRP_BUCKET_SMEM) {  // (very long: the ids sorted in global scratch)
      uint32_t* gk = a.keys_rw + run.x;  // (the keys are dead once the records are placed)
      for (int i = tid; i < L; i += blockDim.x) gk[i] = g[i].x;
      __syncthreads();
      int P = 1;
      while (P < L) P <<= 1;
      block_bitonic(gk, L, P);
      for (int i = tid; i < L; i += blockDim.x) g[i] = make_uint2(gk[i], __float_as_uint(a.wts[gk[i]]));
      __syncthreads();
      continue;
    }
    uint32_t* sa = s_sort;
    uint32_t* sb = sa + GRP_BUCKET_SMEM;
    uint32_t* cnt = sb + GRP_BUCKET_SMEM;  // [256] counts, then the scatter cursors
    uint32_t* off = cnt + 256;             // [256] bucket offsets
    uint32_t* wsum = off + 256;            // [8]
    cnt[tid] = 0u;
    __syncthreads();
    for (int i = tid; i < L; i += blockDim.x) {
      const uint32_t v = g[i].x;
      sa[i] = v;
      atomicAdd(&cnt[v >> a.id_shift], 1u);
    }
    __syncthreads();
    // exclusive scan of the 256 bucket counts
    const uint32_t c = cnt[tid];
    uint32_t x = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += o;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    uint32_t pre = 0;
    for (int w = 0; w < wid; ++w) pre += wsum[w];
    off[tid] = pre + x - c;
    cnt[tid] = pre + x - c;  // cursor
    __syncthreads();
    for (int i = tid; i < L; i += blockDim.x) {
      const uint32_t v = sa[i];
      sb[atomicAdd(&cnt[v >> a.id_shift], 1u)] = v;  // (any order inside the bucket)
    }
    __syncthreads();
    // cnt[b] is now the end of bucket b
    for (int b = wid; b < 256; b += 8) {
      const int o = (int)off[b], n = (int)cnt[b] - o;
      if (n <= GRP_WARP_SORT) warp_sort_any(sb + o, n);
    }
    __syncthreads();
    for (int b = 0; b < 256; ++b) {  // (a bucket of more than GRP_WARP_SORT entries: the CTA)
      const int o = (int)off[b], n = (int)cnt[b] - o;
      if (n > GRP_WARP_SORT) {
        int P = 1;
        while (P < n) P <<= 1;
        block_bitonic(sb + o, n, P);
      }
    }
    for (int i = tid; i < L; i += blockDim.x) {
      const uint32_t v = sb[i];
      g[i] = make_uint2(v, __float_as_uint(a.wts[v]));
    }
    __syncthreads();
  }
  for (;;) {
    uint32_t r = 0;
    if (lane == 0) r = atomicAdd(a.ctl_rw + CTL_SORTQ, 1u);
    r = __shfl_sync(0xffffffffu, r, 0);
    if ((int64_t)r >= nruns) break;
    const uint4 run = a.runs_long[r];
    const int L = (int)run.y;
    if (L <= GRP_WARP_SORT) warp_sort_pairs(a, a.ent_rw + run.x, L);
  }
}

// Step 2: one warp per slice of GRP_SLICE consecutive sorted entries of a
// long run (a flat list over all runs: every warp has a full slice's work,
// many slices in flight); the slice sum, in entry order, goes to part[slice].
// The next slice's record is loaded one iteration ahead, so a slice costs
// two dependent round trips (its ids and weights, then the x rows).
template <int MODE, typename XT, typename YT, int EPL, bool P2P>
__global__ void __launch_bounds__(256, 4) grp_reduce_slice_kernel(GrpArgs a) {
  pdl_enter();
  constexpr int VW = EPL < 4 ? EPL : 4;
  constexpr int NVEC = EPL / VW;
  constexpr int D = 32 * EPL;
  constexpr int U = EPL >= 16 ? 2 : (EPL >= 8 ? 4 : 8);
  const int lane = threadIdx.x % 32;
  const int64_t np = a.ctl[CTL_NPIECES];
  const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32;
  const YT* __restrict__ Y = reinterpret_cast<const YT*>(a.Y) + lane * VW;
  int64_t pc = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  uint4 cur = pc < np ? a.pieces[pc] : make_uint4(0, 0, 0, 0);
  const uint64_t pol_once = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();
  for (; pc < np; pc += nw) {
    const uint4 nxt = pc + nw < np ? a.pieces[pc + nw] : make_uint4(0, 0, 0, 0);
    const int n = (int)cur.y;
    const uint2 me = lane < n ? a.ent[cur.x + lane] : make_uint2(0u, 0u);
    const uint32_t myid = me.x;
    const float myw = __uint_as_float(me.y);
    float y[MODE == MODE_DV ? EPL : 1], acc[EPL];
    if constexpr (MODE == MODE_DV) {
#pragma unroll
      for (int i = 0; i < NVEC; ++i) ldg_vec_pol<YT, VW>(Y + (int64_t)cur.z * D + i * 32 * VW, y + i * VW, pol_once);
    }
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
    grp_accumulate<MODE, XT, EPL, U, P2P>(
        a, 0, n,
        [&](int j, float& w_) {
          w_ = __shfl_sync(0xffffffffu, myw, j);
          return __shfl_sync(0xffffffffu, myid, j);
        },
        y, acc, pol_keep);
#pragma unroll
    for (int i = 0; i < NVEC; ++i) stg_vec<VW>(a.part + pc * D + lane * VW + i * 32 * VW, acc + i * VW);
    cur = nxt;
  }
}

// Step 3: one warp per long run (>= 2 slices): G += the slice sums, added in
// slice order (one update per element); the slice sums are requested CB at a
// time, so a run of many slices costs few memory round trips.
template <typename YT, int EPL>
__global__ void __launch_bounds__(256) grp_combine_long_kernel(GrpArgs a) {
  pdl_enter();
  constexpr int VW = EPL < 4 ? EPL : 4;
  constexpr int NVEC = EPL / VW;
  constexpr int D = 32 * EPL;
  const int lane = threadIdx.x % 32;
  const int64_t nruns = a.ctl[CTL_NLONG];
  const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < nruns; r += nw) {
    const uint4 run = a.runs_long[r];
    const int npc = (int)grp_npieces(run.y);
    constexpr int CB = EPL >= 16 ? 2 : (EPL >= 8 ? 4 : 8);
    float acc[EPL];
#pragma unroll
    for (int i = 0; i < NVEC; ++i) ldg_vec<float, VW>(a.part + (int64_t)run.w * D + lane * VW + i * 32 * VW, acc + i * VW);
    for (int j0 = 1; j0 < npc; j0 += CB) {
      float v[CB][EPL];
#pragma unroll
      for (int c = 0; c < CB; ++c)
        if (j0 + c < npc) {
#pragma unroll
          for (int i = 0; i < NVEC; ++i)
            ldg_vec<float, VW>(a.part + (int64_t)(run.w + j0 + c) * D + lane * VW + i * 32 * VW, v[c] + i * VW);
        }
#pragma unroll
      for (int c = 0; c < CB; ++c)
        if (j0 + c < npc) {
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[i] += v[c][i];
        }
    }
    if (a.upd) {
#pragma unroll
      for (int i = 0; i < NVEC; ++i) {
        const int64_t off = (int64_t)run.z * D + (i * 32 + lane) * VW;
        float y[VW];
        ldg_vec<YT, VW>(reinterpret_cast<const YT*>(a.Vw) + off, y);
        update_vec<YT, VW>(a, off, y, acc + i * VW);
      }
    } else {
#pragma unroll
      for (int i = 0; i < NVEC; ++i)
        red_vec_pol<VW>(a.G + (int64_t)run.z * D + lane * VW + i * 32 * VW, acc + i * VW, l2_policy_evict_first());
    }
  }
}

int num_sms() { return device_sms(); }

// scratch of the grouping (carved by carve_bwd_workspace)
struct GrpScratch {
  uint32_t* cnt;    // [rows]  (zeroed by grp_begin)
  uint32_t* off;    // [rows]
  uint32_t* rank;   // [n]
  uint32_t* keys;   // [n]
  uint2* ent;       // [n] (record id, weight bits)
  uint4* runs_short;  // [min(n, rows)]
  uint4* runs_long;   // [n / 33 + 1]
  uint4* pieces;    // [grp_pieces_max(n)]
  float* part;      // [grp_pieces_max(n) * D]
  uint32_t* ctl;    // CTL_WORDS
  uint32_t* huge;   // [grp_huge_max(n)]
};

// zero the row counters and the control words (the counts are accumulated by
// the kernel that produces the keys)
__global__ void __launch_bounds__(256) grp_zero_kernel(uint32_t* __restrict__ a, int64_t na,
                                                       uint32_t* __restrict__ b, int64_t nb) {
  pdl_enter();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na + nb; i += stride) {
    if (i < na) a[i] = 0u;
    else b[i - na] = 0u;
  }
}

cudaError_t grp_begin(const GrpScratch& g, uint32_t nrows, cudaStream_t st) {
  int64_t blocks = ((int64_t)nrows + CTL_WORDS + 255) / 256;
  if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
  return launch_pdl(grp_zero_kernel, (unsigned)blocks, 256, 0, st, g.ctl, (int64_t)CTL_WORDS, g.cnt,
                    (int64_t)nrows);
}

template <int MODE, typename XT, typename YT, int EPL>
cudaError_t grp_reduce_t(const GrpArgs& a, int64_t n, uint32_t nrows, cudaStream_t st,
                         int* launches, const TraceEvents& tr) {
  const int sms = num_sms();
  int64_t sb = (int64_t)sms * (EPL >= 32 ? 1 : (EPL >= 16 ? 2 : (EPL >= 8 ? MSN_SHORT_BPS : MSN_SHORT_BPS4)));
  const int64_t sneed = ((n < (int64_t)nrows ? n : (int64_t)nrows) + 7) / 8;
  if (sb > sneed) sb = sneed;
  if (sb < 1) sb = 1;
  if (tr.n > 0) cudaEventRecord(tr.ev[0], st);  // profiling: the short-run reducer alone
  if (MODE == MODE_DV && a.upd)
    launch_pdl(grp_reduce_short_kernel<MODE, XT, YT, EPL, true, false>, (unsigned)sb, 256, 0, st, a);
  else if (MODE == MODE_DV && a.xl)
    launch_pdl(grp_reduce_short_kernel<MODE, XT, YT, EPL, false, MODE == MODE_DV>, (unsigned)sb, 256, 0, st, a);
  else
    launch_pdl(grp_reduce_short_kernel<MODE, XT, YT, EPL, false, false>, (unsigned)sb, 256, 0, st, a);
  if (tr.n > 1) cudaEventRecord(tr.ev[1], st);
  // long runs: sort, pieces, combine
  static std::atomic<uint64_t> attr{0};
  {
    cudaError_t e = smem_attr_once(attr, grp_sort_long_kernel, GRP_SORT_SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  const int64_t lneed = n / (GRP_SHORT + 1) + 1;
  // (all three grids one wave of grid-stride / work-queue CTAs: with no long
  // run -- uniform traffic -- each launch reads its counter and exits)
  int64_t lb = (lneed + 7) / 8;
  if (lb > (int64_t)sms * 2) lb = (int64_t)sms * 2;
  launch_pdl(grp_sort_long_kernel, (unsigned)lb, 256, GRP_SORT_SMEM_BYTES, st, a);
  int64_t pb = (int64_t)sms * 4;
  const int64_t pneed = (grp_pieces_max(n) + 7) / 8;
  if (pb > pneed) pb = pneed;
  if (MODE == MODE_DV && a.xl)
    launch_pdl(grp_reduce_slice_kernel<MODE, XT, YT, EPL, MODE == MODE_DV>, (unsigned)pb, 256, 0, st, a);
  else
    launch_pdl(grp_reduce_slice_kernel<MODE, XT, YT, EPL, false>, (unsigned)pb, 256, 0, st, a);
  int64_t cb = (lneed + 7) / 8;
  if (cb > (int64_t)sms * 2) cb = (int64_t)sms * 2;
  launch_pdl(grp_combine_long_kernel<YT, EPL>, (unsigned)cb, 256, 0, st, a);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) *launches += 4;
  return e;
}

// runs + placement + reducers, after the keys and counts exist
struct UpdateArgs {
  int kind = 0;  // 0: G += g; 1 SGD; 2 Adagrad (on Y in place)
  float lr = 0.f, eps = 0.f;
  float* state = nullptr;
};

template <int MODE, typename XT, typename YT>
cudaError_t grp_finish(const GrpScratch& g, int64_t n, uint32_t nrows, const float* wts,
                       const void* X, const void* Y, float* dots, float* G, int H, int k, int D,
                       cudaStream_t st, int* launches, const TraceEvents& tr = TraceEvents{},
                       const UpdateArgs& up = UpdateArgs{}, int og = 1,
                       const ScatterPeers* peers = nullptr) {
  if (n == 0 || nrows == 0) return cudaSuccess;
  // blocks of >= 1024 rows, up to 8 per SM: a block's rows are walked in
  // 256-row rounds (two CTA barriers each), so fewer rounds per block keep
  // the pass off the latency chain (C4's 4M rows: 14 rounds instead of 56)
  int64_t rb = ((int64_t)nrows + 1023) / 1024;
  if (rb > (int64_t)num_sms() * 8) rb = (int64_t)num_sms() * 8;
  launch_pdl(grp_runs_kernel, (unsigned)rb, 256, 0, st, g.cnt, nrows, g.off, g.runs_short, g.runs_long,
                                                g.pieces, g.huge, g.ctl);
  launch_pdl(grp_place_kernel, (unsigned)((n + 255) / 256), 256, 0, st, g.keys, g.rank, g.off, wts, n, nrows,
                                                                g.ent);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  *launches += 2;
  GrpArgs a{g.ent, wts, g.runs_short, g.runs_long, g.pieces, g.part, g.ctl, X, Y, dots, G, g.ent,
            FastDiv((uint32_t)(H * k)), FastDiv((uint32_t)k)};
  a.huge = g.huge;
  a.ctl_rw = g.ctl;
  a.keys_rw = g.keys;
  {
    uint32_t bits = 0;
    while (bits < 32 && (uint64_t(1) << bits) < (uint64_t)n) ++bits;
    a.id_shift = bits > 8 ? bits - 8 : 0;
  }
  a.og = og;
  a.H = H;
  a.div_h = FastDiv((uint32_t)H);
  a.div_hg = FastDiv((uint32_t)(H / og));
  a.upd = up.kind;
  a.lr = up.lr;
  a.eps = up.eps;
  a.state = up.state;
  a.Vw = const_cast<void*>(Y);
  if (peers) {
    a.px = peers->d_out;
    a.pd = peers->dw;
    a.xl = (uint32_t)(peers->local_batch * og);
    a.dl = (uint32_t)(peers->cap ? peers->cap : peers->local_batch * H * k);
    a.div_xl = FastDiv(a.xl);
    a.div_dl = FastDiv(a.dl);
    if (!peers->p2p) a.xl = 0;  // (staged records: local X / dots)
  }

  switch (D / 32) {
    case 1: return grp_reduce_t<MODE, XT, YT, 1>(a, n, nrows, st, launches, tr);
    case 2: return grp_reduce_t<MODE, XT, YT, 2>(a, n, nrows, st, launches, tr);
    case 4: return grp_reduce_t<MODE, XT, YT, 4>(a, n, nrows, st, launches, tr);
    case 8: return grp_reduce_t<MODE, XT, YT, 8>(a, n, nrows, st, launches, tr);
    case 16: return grp_reduce_t<MODE, XT, YT, 16>(a, n, nrows, st, launches, tr);
    case 32:  // value rows of 1024 (the paper's inferred width)
      if constexpr (MODE == MODE_DV) return grp_reduce_t<MODE, XT, YT, 32>(a, n, nrows, st, launches, tr);
      else return cudaErrorNotSupported;
    default: return cudaErrorNotSupported;
  }
}

// ---------------------------------------------------- contribution keys ----
// key = local row of idx (or the nrows sentinel when the slot is held
// elsewhere; its dw is 0 here and the shards' dw are summed), and the
// grouping count: rank[p] = atomicAdd(&cnt[key], 1).
__global__ void dv_keys_kernel(const int32_t* __restrict__ idx, int64_t n, int64_t row_begin,
                               int64_t row_end, uint32_t sentinel, uint32_t* __restrict__ keys,
                               uint32_t* __restrict__ cnt, uint32_t* __restrict__ rank,
                               float* __restrict__ dw) {  // dw null: non-local slots are other ranks'
  pdl_enter();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t f = idx[p];
  const bool local = f >= row_begin && f < row_end;
  const uint32_t key = local ? (uint32_t)(f - row_begin) : sentinel;
  keys[p] = key;
  if (local) rank[p] = atomicAdd(&cnt[key], 1u);
  else if (dw) dw[p] = 0.f;
}

// ----------------------------------------------- ds, dQ and dK records ----
// One warp per lookup (b,h).  ds_t = w_t (dw_t - sum_u w_u dw_u).
// For each half, the dS of every distinct sub-key index r is summed over the
// t with r_t = r in t order; dQ[b,h,half] = sum_r dS_r K[h,half,r]; one dK
// record per distinct r (first occurrence, counted for the grouping), others
// get the sentinel key.
// OUT = OUT_DENSE: instead of grouping records, the dS of the lookup-half is
// written as one dense bf16 row dSd[b, h*2 + half, 0:n_sub] (zeros elsewhere)
// for the tensor-core dK (dk_tc.cu) and, unless DQ, the tensor-core dQ;
// n_sub <= kDenseMax.  OUT = OUT_COMPACT: the m distinct (sub-key, dS) pairs
// of the lookup-half as k uint2 slots {index, dS bits} (index 0xffffffff past
// m) from which the tensor-core dK builds its operand tiles in shared memory
// (no dense matrix in HBM).  DQ: dQ by the warp here (the m distinct K rows
// of the lookup-half from L2) -- cheaper than the dense GEMM when n_sub is
// large.
constexpr int kDenseMax = 2048;
enum { OUT_GROUP = 0, OUT_DENSE = 1, OUT_COMPACT = 2 };
template <typename QT, int KPL, int EPL, int OUT, bool DQ>
__global__ void __launch_bounds__(256) ds_dq_kernel(const QT* __restrict__ K,
                                                    const int32_t* __restrict__ idx,
                                                    const float* __restrict__ w,
                                                    const float* __restrict__ dw, int64_t L,
                                                    int H, int n_sub, int d_h, int k,
                                                    float* __restrict__ dQ,
                                                    uint32_t* __restrict__ rkeys,
                                                    float* __restrict__ dsS, uint32_t sentinel,
                                                    uint32_t* __restrict__ cnt,
                                                    uint32_t* __restrict__ rank,
                                                    uint16_t* __restrict__ dSd, int hg,
                                                    int32_t tab_stride, bool dq_bf16, int tile_rows = 0,
                                                    int ntiles = 0) {
  pdl_enter();
  constexpr int DQ_U = EPL >= 16 ? 2 : (EPL >= 8 ? 4 : 8);
  constexpr bool DENSE = OUT == OUT_DENSE;
  __shared__ int32_t s_r[8][2][64];
  __shared__ float s_d[8][2][64];
  __shared__ __align__(16) uint16_t s_row[DENSE ? 8 : 1][DENSE ? kDenseMax : 8];
  const int lane = threadIdx.x % 32, wid = threadIdx.x / 32;
  const int64_t l = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (l >= L) return;
  int mh[2] = {0, 0};  // distinct sub-keys per half
  const int h = (int)(l % H);
  float wt[KPL], g[KPL], ds[KPL];
  int32_t f[KPL];
  float part = 0.f;
#pragma unroll
  for (int u = 0; u < KPL; ++u) {
    const int t = lane + 32 * u;
    wt[u] = t < k ? w[l * k + t] : 0.f;
    g[u] = t < k ? dw[l * k + t] : 0.f;
    // slot within the group's table (per-group tables)
    f[u] = t < k ? idx[l * k + t] - (h / hg) * tab_stride : 0;
    part = fmaf(wt[u], g[u], part);
  }
  const float gbar = warp_sum(part);
#pragma unroll
  for (int u = 0; u < KPL; ++u) ds[u] = wt[u] * (g[u] - gbar);
  for (int half = 0; half < 2; ++half) {
    int r[KPL];
#pragma unroll
    for (int u = 0; u < KPL; ++u) {
      // (power-of-two codebooks -- every BASELINE config -- by shift and mask)
      if ((n_sub & (n_sub - 1)) == 0) {
        const int sh = __ffs(n_sub) - 1;
        r[u] = half == 0 ? f[u] >> sh : f[u] & (n_sub - 1);
      } else {
        r[u] = half == 0 ? f[u] / n_sub : f[u] % n_sub;
      }
    }
    float dS[KPL];
    bool first[KPL];
#pragma unroll
    for (int u = 0; u < KPL; ++u) { dS[u] = 0.f; first[u] = true; }
    if constexpr (KPL == 1) {
      // the lanes holding the same sub-key index r (one group per distinct r)
      // sum their ds in ascending lane (= t) order: the same additions as the
      // all-pairs loop below, in max(group size) steps instead of k
      const bool valid = lane < k;
      unsigned grp = __match_any_sync(0xffffffffu, valid ? r[0] : -1 - lane);
      first[0] = (grp & ((1u << lane) - 1u)) == 0u;
      int steps = __popc(grp);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) steps = max(steps, __shfl_xor_sync(0xffffffffu, steps, o));
      for (int j = 0; j < steps; ++j) {
        const int src = grp ? __ffs(grp) - 1 : lane;
        const float v = __shfl_sync(0xffffffffu, ds[0], src);
        if (grp) {
          dS[0] += v;
          grp &= grp - 1u;
        }
      }
      if (!valid) dS[0] = 0.f;
    } else {
      for (int v = 0; v < k; ++v) {
        const bool lo = KPL == 1 || v < 32;
        const int rv = __shfl_sync(0xffffffffu, lo ? r[0] : r[KPL - 1], v % 32);
        const float dsv = __shfl_sync(0xffffffffu, lo ? ds[0] : ds[KPL - 1], v % 32);
#pragma unroll
        for (int u = 0; u < KPL; ++u) {
          const int t = lane + 32 * u;
          if (rv == r[u]) {
            dS[u] += dsv;
            if (v < t) first[u] = false;
          }
        }
      }
    }
    // records
    if constexpr (OUT == OUT_GROUP) {
#pragma unroll
      for (int u = 0; u < KPL; ++u) {
        const int t = lane + 32 * u;
        if (t < k) {
          const int64_t rec = (l * k + t) * 2 + half;
          const uint32_t key = (uint32_t)((h * 2 + half) * n_sub + r[u]);
          rkeys[rec] = first[u] ? key : sentinel;
          if (first[u]) rank[rec] = atomicAdd(&cnt[key], 1u);
          dsS[rec] = dS[u];
        }
      }
    }
    // the distinct sub-keys of this half, compacted into shared memory in
    // first-occurrence order (dQ below, the dense / compact dS outputs)
    int m = 0;
#pragma unroll
    for (int u = 0; u < KPL; ++u) {
      const int t = lane + 32 * u;
      const bool fl = t < k && first[u];
      const unsigned bm = __ballot_sync(0xffffffffu, fl);
      if (fl) {
        const int pos = m + __popc(bm & ((1u << lane) - 1u));
        s_r[wid][half][pos] = r[u];
        s_d[wid][half][pos] = dS[u];
      }
      m += __popc(bm);
    }
    mh[half] = m;
    __syncwarp();
    if constexpr (DENSE) {
      // dense row: zero, place the m distinct values, copy out (16 B per lane)
      uint4* row4 = reinterpret_cast<uint4*>(s_row[wid]);
      const int n16 = n_sub / 8;
      for (int c = lane; c < n16; c += 32) row4[c] = make_uint4(0, 0, 0, 0);
      __syncwarp();
      for (int c = lane; c < m; c += 32)
        s_row[wid][s_r[wid][half][c]] = __bfloat16_as_ushort(__float2bfloat16_rn(s_d[wid][half][c]));
      __syncwarp();
      uint4* g4 = reinterpret_cast<uint4*>(dSd + (l * 2 + half) * (int64_t)n_sub);
      for (int c = lane; c < n16; c += 32) g4[c] = row4[c];
      __syncwarp();
    }
    if constexpr (OUT == OUT_COMPACT) {
      // the m records sorted by sub-key (rank = number of smaller indices;
      // the indices are distinct), and per block of tile_rows sub-keys
      // the end of its records: block t's records are [t ? off[t-1] : 0,
      // off[t]) (blocks of one dK tile, tile_rows sub-keys), so the dK tile
      // builder reads only its own (dk_tc.cu)
      // a record = bf16(dS) << 16 | sub-key (n_sub <= 2048; both consumers
      // multiply by the bf16-rounded dS), 0xffffffff past m
      uint32_t* rec = reinterpret_cast<uint32_t*>(dSd) + (l * 2 + half) * (int64_t)k;
      uint8_t* off = reinterpret_cast<uint8_t*>(reinterpret_cast<uint32_t*>(dSd) + (int64_t)L * 2 * k) +
                     (l * 2 + half) * 32;
      for (int c = lane; c < k; c += 32) {
        if (c < m) {
          const int32_t r = s_r[wid][half][c];
          int rk = 0;
          for (int j = 0; j < m; ++j) rk += s_r[wid][half][j] < r;
          rec[rk] = ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(s_d[wid][half][c])) << 16) | (uint32_t)r;
        } else {
          rec[c] = 0xffffffffu;
        }
      }
      int below = 0;  // lane t: records with sub-key < (t + 1) tile_rows
      for (int c = 0; c < m; c += 32) {
        const int idx0 = c + lane < m ? s_r[wid][half][c + lane] : 0x7fffffff;
        for (int t = 0; t < ntiles; ++t) {
          const int n = __popc(__ballot_sync(0xffffffffu, idx0 < (t + 1) * tile_rows));
          if (lane == t) below += n;
        }
      }
      if (lane < ntiles) off[lane] = (uint8_t)below;
    }
  }
  if constexpr (!DQ) return;  // dQ = dSd . K runs on the tensor cores (dk_tc.cu)
  // dQ[b,h,half] = sum_r dS_r K[h,half,r], lanes over d_h, both halves
  // together: DQ_U rows of each half in flight per step (the m distinct K
  // rows of a lookup-half come from L2), each half's sum in first-occurrence
  // order (the same additions as one half at a time)
  float acc[2][EPL];
#pragma unroll
  for (int i = 0; i < EPL; ++i) acc[0][i] = acc[1][i] = 0.f;
  const QT* Kh0 = K + (int64_t)(h * 2) * n_sub * d_h + lane * EPL;
  const QT* Kh1 = Kh0 + (int64_t)n_sub * d_h;
  const int mm = mh[0] > mh[1] ? mh[0] : mh[1];
  for (int b0 = 0; b0 < mm; b0 += DQ_U) {
    // unconditional loads (a row past m repeats row 0 and is added with 0): no
    // branches between them, so all 2 DQ_U rows are in flight together
    float kr[2][DQ_U][EPL];
    float dv[2][DQ_U];
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
      for (int u = 0; u < DQ_U; ++u) {
        const bool in = b0 + u < mh[hf];
        const int j = in ? b0 + u : 0;
        dv[hf][u] = in ? s_d[wid][hf][j] : 0.f;
        load_slice<QT, EPL>((hf ? Kh1 : Kh0) + (int64_t)s_r[wid][hf][j] * d_h, kr[hf][u]);
      }
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
      for (int u = 0; u < DQ_U; ++u) {
        if constexpr (EPL % 2 == 0) {
#pragma unroll
          for (int i = 0; i < EPL; i += 2) ffma2(acc[hf][i], acc[hf][i + 1], kr[hf][u][i], kr[hf][u][i + 1], dv[hf][u]);
        } else {
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[hf][i] = fmaf(dv[hf][u], kr[hf][u][i], acc[hf][i]);
        }
      }
  }
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    if (dq_bf16) {  // MSN_FLAG_DQ_QK_DTYPE: one RNE rounding
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(dQ) + (l * 2 + hf) * d_h + lane * EPL;
#pragma unroll
      for (int i = 0; i < EPL; ++i) o[i] = __float2bfloat16_rn(acc[hf][i]);
    } else {
      float* o = dQ + (l * 2 + hf) * d_h + lane * EPL;
#pragma unroll
      for (int i = 0; i < EPL; ++i) o[i] = acc[hf][i];
    }
  }
}

// ------------------------------------------------------- atomic scatter ---
template <typename VT, int EPL>
__global__ void __launch_bounds__(256) scatter_atomic_kernel(const int32_t* __restrict__ idx,
                                                             const float* __restrict__ w,
                                                             const float* __restrict__ dOut,
                                                             const VT* __restrict__ V,
                                                             float* __restrict__ dV,
                                                             float* __restrict__ dw, int64_t B,
                                                             int HK, int d_v, int64_t row_begin,
                                                             int64_t row_end) {
  pdl_enter();
  const int lane = threadIdx.x % 32;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (b >= B) return;
  float go[EPL];
  load_slice<float, EPL>(dOut + b * d_v + lane * EPL, go);
  for (int r = 0; r < HK; ++r) {
    const int64_t f = idx[b * HK + r];
    const float wt = w[b * HK + r];
    float d = 0.f;
    if (f >= row_begin && f < row_end) {
      const int64_t row = f - row_begin;
      float v[EPL];
      load_slice<VT, EPL>(V + row * d_v + lane * EPL, v);
#pragma unroll
      for (int i = 0; i < EPL; ++i) d = fmaf(v[i], go[i], d);
      float* p = dV + row * d_v + lane * EPL;
      if constexpr (EPL % 4 == 0) {
#pragma unroll
        for (int i = 0; i < EPL; i += 4)
          red_add_v4(p + i, wt * go[i], wt * go[i + 1], wt * go[i + 2], wt * go[i + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < EPL; ++i) atomicAdd(p + i, wt * go[i]);
      }
    }
    d = warp_sum(d);
    if (lane == 0) dw[b * HK + r] = d;
  }
}

int epl_of(int D) { return D / 32; }
bool epl_ok(int D) {
  const int e = D / 32;
  return D % 32 == 0 && (e == 1 || e == 2 || e == 4 || e == 8 || e == 16);
}
// value rows: also 1024 wide (EPL 32) in the value reducers
bool epl_ok_v(int D) { return epl_ok(D) || D == 1024; }

}  // namespace

bool backward_supported(const Shape& s, bool values, bool keys) {
  if (values && !epl_ok_v(s.d_v)) return false;
  if (keys && (!epl_ok(s.d_h) || s.k > 64)) return false;
  return true;
}

// ---------------------------------------------------------- workspace ------
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

namespace {
struct WsPlan {
  int64_t n, rows, D;
};
WsPlan ws_plan(const Shape& s, int64_t gather_batch) {
  const int64_t n_dv = gather_batch * s.H * s.k;
  const int64_t n_dk = 2 * s.B * s.H * s.k;
  const int64_t r_dv = s.row_end - s.row_begin;
  const int64_t r_dk = (int64_t)s.H * 2 * s.n_sub;
  return WsPlan{n_dv > n_dk ? n_dv : n_dk, r_dv > r_dk ? r_dv : r_dk, s.d_v > s.d_h ? s.d_v : s.d_h};
}
}  // namespace

size_t bwd_workspace_bytes(const Shape& s, int64_t gather_batch) {
  const WsPlan pl = ws_plan(s, gather_batch);
  const int64_t n_dv = gather_batch * s.H * s.k;
  const int64_t n_dk = 2 * s.B * s.H * s.k;
  const int64_t nshort = pl.n < pl.rows ? pl.n : pl.rows;
  size_t b = 0;
  b += 2 * align256(sizeof(uint32_t) * pl.rows);            // cnt, off
  b += 4 * align256(sizeof(uint32_t) * pl.n);               // rank, keys, ent (8-byte pairs)
  b += align256(sizeof(uint4) * nshort);                    // runs_short
  b += align256(sizeof(uint4) * (pl.n / (GRP_SHORT + 1) + 1));  // runs_long
  b += align256(sizeof(uint4) * grp_pieces_max(pl.n));             // slices
  b += align256(sizeof(float) * grp_pieces_max(pl.n) * pl.D);      // piece partials
  b += align256(sizeof(uint32_t) * CTL_WORDS);
  b += align256(sizeof(uint32_t) * grp_huge_max(pl.n));     // huge runs
  b += align256(sizeof(float) * n_dk);                      // dsS
  b += align256(sizeof(float) * n_dv);                      // dw
  b += align256(dk_tc_workspace_bytes(s));
  return b;
}

BwdWorkspace carve_bwd_workspace(const Shape& s, int64_t gather_batch, void* ws) {
  const WsPlan pl = ws_plan(s, gather_batch);
  const int64_t n_dv = gather_batch * s.H * s.k;
  const int64_t n_dk = 2 * s.B * s.H * s.k;
  const int64_t nshort = pl.n < pl.rows ? pl.n : pl.rows;
  char* p = (char*)ws;
  BwdWorkspace w;
  w.cnt = (uint32_t*)p; p += align256(sizeof(uint32_t) * pl.rows);
  w.off = (uint32_t*)p; p += align256(sizeof(uint32_t) * pl.rows);
  w.rank = (uint32_t*)p; p += align256(sizeof(uint32_t) * pl.n);
  w.keys = (uint32_t*)p; p += align256(sizeof(uint32_t) * pl.n);
  w.ent = (uint2*)p; p += 2 * align256(sizeof(uint32_t) * pl.n);
  w.runs_short = (uint4*)p; p += align256(sizeof(uint4) * nshort);
  w.runs_long = (uint4*)p; p += align256(sizeof(uint4) * (pl.n / (GRP_SHORT + 1) + 1));
  w.pieces = (uint4*)p; p += align256(sizeof(uint4) * grp_pieces_max(pl.n));
  w.part = (float*)p; p += align256(sizeof(float) * grp_pieces_max(pl.n) * pl.D);
  w.ctl = (uint32_t*)p; p += align256(sizeof(uint32_t) * CTL_WORDS);
  w.huge = (uint32_t*)p; p += align256(sizeof(uint32_t) * grp_huge_max(pl.n));
  w.dsS = (float*)p; p += align256(sizeof(float) * n_dk);
  w.dw = (float*)p; p += align256(sizeof(float) * n_dv);
  w.dk_ws = (void*)p; p += align256(dk_tc_workspace_bytes(s));
  return w;
}

// ------------------------------------------------------------ launchers ---
static GrpScratch grp_scratch(const BwdWorkspace& ws) {
  return GrpScratch{ws.cnt, ws.off, ws.rank, ws.keys, ws.ent, ws.runs_short, ws.runs_long,
                    ws.pieces, ws.part, ws.ctl, ws.huge};
}

cudaError_t launch_scatter_sorted(const Shape& s, const int32_t* idx, const float* w,
                                  const float* dOut, const void* V, float* dV, float* dw,
                                  const BwdWorkspace& ws, cudaStream_t st, int* launches,
                                  const TraceEvents& tr, int upd, float lr, float eps,
                                  float* state, const ScatterPeers* peers) {
  if (!epl_ok_v(s.d_v)) return cudaErrorNotSupported;
  const int64_t n = s.B * s.H * s.k;  // s.B is the gather batch here
  if (n == 0) return cudaSuccess;
  const uint32_t nrows = (uint32_t)(s.row_end - s.row_begin);
  const GrpScratch g = grp_scratch(ws);
  cudaError_t e = grp_begin(g, nrows, st);
  if (e != cudaSuccess) return e;
  launch_pdl(dv_keys_kernel, (unsigned)((n + 255) / 256), 256, 0, st, idx, n, s.row_begin, s.row_end,
                                                              nrows, g.keys, g.cnt, g.rank, peers ? nullptr : dw);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ++*launches;
  if (s.v_dt == F32)
    return grp_finish<MODE_DV, float, float>(g, n, nrows, w, dOut, V, dw, dV, s.H, s.k, s.d_v, st,
                                             launches, tr, UpdateArgs{upd, lr, eps, state}, s.og, peers);
  return grp_finish<MODE_DV, float, __nv_bfloat16>(g, n, nrows, w, dOut, V, dw, dV, s.H, s.k,
                                                   s.d_v, st, launches, tr, UpdateArgs{upd, lr, eps, state},
                                                   s.og, peers);
}

namespace {
// Keys of exchanged records (a9): record j = s * cap + b * HK + i (window
// (s, b), cap = lb * HK) is valid iff i < cnt[s * lb + b]; key = its local
// row.  The record id orders the contributions globally: source s's query b
// is the global query s * lb + b, so j / HK is the d_out row (as the cid of
// the unsharded path) and ascending j is ascending (query, h, t).
__global__ void rec_keys_kernel(const int32_t* __restrict__ row, const int32_t* __restrict__ cnt, FastDiv div_hk,
                                uint32_t HK, int64_t n, uint32_t sentinel, uint32_t* __restrict__ keys,
                                uint32_t* __restrict__ gcnt, uint32_t* __restrict__ rank) {
  pdl_enter();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t win = div_hk.div((uint32_t)p);  // s * lb + b
  const bool valid = (uint32_t)p - win * HK < (uint32_t)cnt[win];
  const uint32_t key = valid ? (uint32_t)row[p] : sentinel;
  keys[p] = key;
  if (valid) rank[p] = atomicAdd(&gcnt[key], 1u);
}
}  // namespace

cudaError_t launch_scatter_records(const Shape& s, const RecordsIn& r, const PerRank<const float>& x_src,
                                   const void* V, float* dV, const PerRank<float>& dw_dst,
                                   const BwdWorkspace& ws, cudaStream_t st, int* launches,
                                   const TraceEvents& tr) {
  if (!epl_ok_v(s.d_v) || s.og != 1) return cudaErrorNotSupported;
  const int64_t n = (int64_t)r.P * r.cap;
  if (n == 0) return cudaSuccess;
  if (n >= (int64_t(1) << 32)) return cudaErrorNotSupported;
  const uint32_t nrows = (uint32_t)(s.row_end - s.row_begin);
  const GrpScratch g = grp_scratch(ws);
  cudaError_t e = grp_begin(g, nrows, st);
  if (e != cudaSuccess) return e;
  launch_pdl(rec_keys_kernel, (unsigned)((n + 255) / 256), 256, 0, st, r.row, r.cnt, FastDiv((uint32_t)r.HK),
             (uint32_t)r.HK, n, nrows, g.keys, g.cnt, g.rank);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ++*launches;
  // the records' x rows and dw destinations are per source rank (peer memory,
  // or the staged local regions): the P2P reducers with record -> query map
  ScatterPeers peers;
  peers.d_out = x_src;
  peers.dw = dw_dst;
  peers.local_batch = r.lb;
  peers.p2p = true;
  peers.cap = r.cap;
  // one rank: the only source is this one -- the plain local reducers (x rows
  // and dw in single arrays), the same kernels as the unsharded backward
  const ScatterPeers* pp = r.P > 1 ? &peers : nullptr;
  const float* X = r.P > 1 ? nullptr : x_src.p[0];
  float* dots = r.P > 1 ? nullptr : dw_dst.p[0];
  if (s.v_dt == F32)
    return grp_finish<MODE_DV, float, float>(g, n, nrows, r.w, X, V, dots, dV, s.H, s.k, s.d_v, st,
                                             launches, tr, UpdateArgs{}, 1, pp);
  return grp_finish<MODE_DV, float, __nv_bfloat16>(g, n, nrows, r.w, X, V, dots, dV, s.H, s.k,
                                                   s.d_v, st, launches, tr, UpdateArgs{}, 1, pp);
}

cudaError_t launch_scatter_atomic(const Shape& s, const int32_t* idx, const float* w,
                                  const float* dOut, const void* V, float* dV, float* dw,
                                  cudaStream_t st, int* launches) {
  if (!epl_ok_v(s.d_v)) return cudaErrorNotSupported;
  const unsigned blocks = (unsigned)((s.B + 7) / 8);
  const int HK = s.H * s.k;
#define ATOMIC(VT, E)                                                                          \
  launch_pdl(scatter_atomic_kernel<VT, E>, blocks, 256, 0, st, idx, w, dOut, (const VT*)V, dV, dw, s.B, \
                                                       HK, s.d_v, s.row_begin, s.row_end)
  const int E = epl_of(s.d_v);
  if (s.v_dt == F32) {
    switch (E) { case 1: ATOMIC(float, 1); break; case 2: ATOMIC(float, 2); break;
      case 4: ATOMIC(float, 4); break; case 8: ATOMIC(float, 8); break;
      case 16: ATOMIC(float, 16); break; default: ATOMIC(float, 32); }
  } else {
    switch (E) { case 1: ATOMIC(__nv_bfloat16, 1); break; case 2: ATOMIC(__nv_bfloat16, 2); break;
      case 4: ATOMIC(__nv_bfloat16, 4); break; case 8: ATOMIC(__nv_bfloat16, 8); break;
      case 16: ATOMIC(__nv_bfloat16, 16); break; default: ATOMIC(__nv_bfloat16, 32); }
  }
#undef ATOMIC
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t launch_backward_keys(const Shape& s, const void* Q, const void* K,
                                 const int32_t* idx, const float* w, const float* dw, float* dQ,
                                 float* dK, const BwdWorkspace& ws, cudaStream_t st,
                                 int* launches) {
  if (!epl_ok(s.d_h) || s.k > 64) return cudaErrorNotSupported;
  const int64_t L = s.B * s.H;
  if (L == 0) return cudaSuccess;
  const uint32_t nrows = (uint32_t)(s.H * 2 * s.n_sub);
  const unsigned blocks = (unsigned)((L + 7) / 8);
  const int E = epl_of(s.d_h);
  const bool dense = dk_tc_supported(s);
  const bool dq_tc = dense && dq_tc_wanted(s);
  const bool dq_rec = dense && !dq_tc && dk_compact(s) && dq_rec_wanted(s);  // dQ on the tensor cores from the records
  const GrpScratch g = grp_scratch(ws);
  if (!dense) {
    cudaError_t e0 = grp_begin(g, nrows, st);
    if (e0 != cudaSuccess) return e0;
  }
#define DSDQ(QT, KPL, E_)                                                                      \
  if (dense && dq_tc)                                                                          \
    launch_pdl(ds_dq_kernel<QT, KPL, E_, OUT_DENSE, false>, blocks, 256, 0, st,                        \
        (const QT*)K, idx, w, dw, L, s.H, s.n_sub, s.d_h, s.k, dQ, g.keys, ws.dsS, nrows,       \
        g.cnt, g.rank, (uint16_t*)ws.dk_ws, s.H / s.og, (int32_t)s.tab_stride, s.dq_bf16, 0, 0);           \
  else if (dense && !dk_compact(s))                                                            \
    launch_pdl(ds_dq_kernel<QT, KPL, E_, OUT_DENSE, true>, blocks, 256, 0, st,                         \
        (const QT*)K, idx, w, dw, L, s.H, s.n_sub, s.d_h, s.k, dQ, g.keys, ws.dsS, nrows,       \
        g.cnt, g.rank, (uint16_t*)ws.dk_ws, s.H / s.og, (int32_t)s.tab_stride, s.dq_bf16, 0, 0);           \
  else if (dense && dq_rec)                                                                    \
    launch_pdl(ds_dq_kernel<QT, KPL, E_, OUT_COMPACT, false>, blocks, 256, 0, st,                      \
        (const QT*)K, idx, w, dw, L, s.H, s.n_sub, s.d_h, s.k, dQ, g.keys, ws.dsS, nrows,       \
        g.cnt, g.rank, (uint16_t*)ws.dk_ws, s.H / s.og, (int32_t)s.tab_stride, s.dq_bf16,        \
        dk_tile_rows(s), s.n_sub / dk_tile_rows(s));                                             \
  else if (dense)                                                                              \
    launch_pdl(ds_dq_kernel<QT, KPL, E_, OUT_COMPACT, true>, blocks, 256, 0, st,                       \
        (const QT*)K, idx, w, dw, L, s.H, s.n_sub, s.d_h, s.k, dQ, g.keys, ws.dsS, nrows,       \
        g.cnt, g.rank, (uint16_t*)ws.dk_ws, s.H / s.og, (int32_t)s.tab_stride, s.dq_bf16,        \
        dk_tile_rows(s), s.n_sub / dk_tile_rows(s));                                             \
  else                                                                                         \
    launch_pdl(ds_dq_kernel<QT, KPL, E_, OUT_GROUP, true>, blocks, 256, 0, st,                         \
        (const QT*)K, idx, w, dw, L, s.H, s.n_sub, s.d_h, s.k, dQ, g.keys, ws.dsS, nrows,       \
        g.cnt, g.rank, nullptr, s.H / s.og, (int32_t)s.tab_stride, s.dq_bf16, 0, 0)
#define DSDQ_E(QT, KPL)                                                                        \
  switch (E) { case 1: DSDQ(QT, KPL, 1); break; case 2: DSDQ(QT, KPL, 2); break;              \
    case 4: DSDQ(QT, KPL, 4); break; case 8: DSDQ(QT, KPL, 8); break;                          \
    default: DSDQ(QT, KPL, 16); }
  if (s.qk_dt == F32) {
    if (s.k <= 32) { DSDQ_E(float, 1) } else { DSDQ_E(float, 2) }
  } else {
    if (s.k <= 32) { DSDQ_E(__nv_bfloat16, 1) } else { DSDQ_E(__nv_bfloat16, 2) }
  }
#undef DSDQ_E
#undef DSDQ
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ++*launches;
  if (dense) return launch_dk_tc(s, Q, K, dQ, dK, ws.dk_ws, st, launches, dq_tc || dq_rec);
  const int64_t n = 2 * L * s.k;
  if (s.qk_dt == F32)
    return grp_finish<MODE_DK, float, float>(g, n, nrows, ws.dsS, Q, nullptr, nullptr, dK, s.H,
                                             s.k, s.d_h, st, launches);
  return grp_finish<MODE_DK, __nv_bfloat16, float>(g, n, nrows, ws.dsS, Q, nullptr, nullptr, dK,
                                                   s.H, s.k, s.d_h, st, launches);
}

}  // namespace msn
