// select_tc.cu -- steps a1 + a2 on the 5th-generation tensor cores:
// sub-key scoring S = K q (Eq. S_old) as a tcgen05 GEMM
// fed by TMA, with the per-half argtopk fused into the
// epilogue so that S never reaches HBM.
//
// One CTA per (128-query tile, head h, half): D[128 x n_sub] = Q_half . K_half^T
// with bf16 operands and fp32 accumulation in TMEM (kind::f16), computed in
// N-chunks of up to 256 columns that alternate between two TMEM accumulator
// buffers, so the MMA of chunk c+1 overlaps the epilogue of chunk c.
//
//   warp 0      TMA producer: the whole query tile once (resident), then the
//               sub-key tiles through a STAGES-deep mbarrier ring
//   warp 1      MMA issuer (one elected lane): tcgen05.mma + tcgen05.commit
//   warp 2      TMEM allocator (512 columns)
//   warps 4-7   epilogue: TMEM lane i = query row i, one thread per row.
//               tau = KT-th largest of the 2KT strided group maxima seen so
//               far is a provable lower bound on the row's KT-th score; the
//               columns >= tau (~1.4 KT for random scores) are kept in a
//               shared-memory buffer compacted as tau rises, and written out
//               unordered as the row's candidate list (<= 64 entries that
//               contain its top-k); cartesian_kernel orders them.  The first
//               segment is the first min(n_sub, 512) columns, resident in both
//               TMEM buffers, so tau is computed before any column is kept.
//               Rows whose buffer would overflow (massive exact ties) take an
//               exact bitwise search for their KT-th score instead.
#include <cuda.h>
#include <algorithm>
#include <vector>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace msn {
namespace {
using namespace tc;

constexpr int kThreads = 256;
constexpr int kEpiWarp0 = 4;
constexpr int kStages = 3;
constexpr int kMaxNTile = 256;
constexpr int kCap = 64;          // candidate buffer entries per row
constexpr int kRowBytes = 128;    // one 128-byte swizzle row per k-block (64 bf16 / 32 fp32)

// ------------------------------------------------------------- top-k -------
// In-register bitonic sort of N values, descending (group maxima -> tau).
template <int N>
__device__ __forceinline__ void bitonic_sort_vals(float (&v)[N]) {
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = (i & size) == 0;
          const float hi = fmaxf(v[i], v[j]), lo = fminf(v[i], v[j]);
          v[i] = desc ? hi : lo;
          v[j] = desc ? lo : hi;
        }
      }
    }
  }
}

__device__ unsigned long long g_dbg_ts[4096 * 32];
__device__ __forceinline__ unsigned long long gclk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
struct TcParams {
  int dbg;  // profiling only (MSN_SELECT_DBG): 1 = epilogue skips all processing
  int64_t B;
  int H, n_sub, d_h, k;
  int n_tile, n_chunks, k_blocks;
  float* cv;
  int32_t* cc;
  int32_t* cn;
};

template <int KT, bool TF32>
__global__ void __launch_bounds__(kThreads, 1)
    select_tc_kernel(const __grid_constant__ CUtensorMap tmap_q,
                     const __grid_constant__ CUtensorMap tmap_k,
                     const __grid_constant__ CUtensorMap tmap_klo, const TcParams p) {
  pdl_wait();
  constexpr int BK = TF32 ? 32 : 64;            // elements per k-block (one 128-B row)
  constexpr int B_PARTS = TF32 ? 2 : 1;         // B tiles per stage: (K_hi, K_lo) or K
  const int acc_stride = TF32 ? p.n_tile : kMaxNTile;  // TMEM columns between accumulators
  const uint32_t alo_col = 2u * (uint32_t)p.n_tile;     // TF32: A_lo columns [2 n_tile, +d_h)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // carve: A (k_blocks x 16 KB) | B ring (kStages x n_tile x 128 B) | cand vals | cand cols | bars
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* sA = smem_raw + pad;
  uint8_t* sB = sA + p.k_blocks * 16384;
  const int stage_bytes = B_PARTS * p.n_tile * kRowBytes;
  uint2* cand = reinterpret_cast<uint2*>(sB + kStages * stage_bytes);  // [kCap+1][128] (score bits, column)
  uint64_t* bars = reinterpret_cast<uint64_t*>(cand + (kCap + 1) * 128);
  uint64_t* a_full = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* a_ready = tempty + 2;  // TF32: A split into (hi in smem, lo in TMEM)
  uint32_t* tmem_slot = (uint32_t*)(a_ready + 1);

  const unsigned long long t_entry = gclk();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int hh = blockIdx.x;  // h*2 + half
  const int64_t m0 = (int64_t)blockIdx.y * 128;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap_q);
    prefetch_tmap(&tmap_k);
    if (TF32) prefetch_tmap(&tmap_klo);
    mbar_init(a_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    mbar_init(a_ready, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int cta_lin = blockIdx.y * gridDim.x + blockIdx.x;
  const bool ts_on = p.dbg >= 1 && cta_lin < 4096;
  if (ts_on && threadIdx.x == 0) {
    g_dbg_ts[cta_lin * 32 + 0] = gclk();
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_dbg_ts[cta_lin * 32 + 11] = smid;
    g_dbg_ts[cta_lin * 32 + 13] = t_entry;
  }

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_expect_tx(a_full, p.k_blocks * 16384);
      for (int kb = 0; kb < p.k_blocks; ++kb)
        tma_load_3d(sA + kb * 16384, &tmap_q, a_full, kb * BK, hh, (int)m0);
      int it = 0;
      for (int c = 0; c < p.n_chunks; ++c)
        for (int kb = 0; kb < p.k_blocks; ++kb, ++it) {
          const int s = it % kStages;
          mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          mbar_expect_tx(&full[s], stage_bytes);
          tma_load_2d(sB + s * stage_bytes, &tmap_k, &full[s], kb * BK, hh * p.n_sub + c * p.n_tile);
          if (TF32)
            tma_load_2d(sB + s * stage_bytes + p.n_tile * kRowBytes, &tmap_klo, &full[s], kb * BK,
                        hh * p.n_sub + c * p.n_tile);
        }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = TF32 ? idesc_tf32(128, p.n_tile) : idesc_bf16(128, p.n_tile);
      mbar_wait(a_full, 0);
      if (ts_on) g_dbg_ts[cta_lin * 32 + 1] = gclk();
      if (TF32) mbar_wait(a_ready, 0);
      tc_fence_after();
      int it = 0;
      for (int c = 0; c < p.n_chunks; ++c) {
        const int buf = c & 1;
        mbar_wait(&tempty[buf], ((c >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * acc_stride;
        for (int kb = 0; kb < p.k_blocks; ++kb, ++it) {
          const int s = it % kStages;
          mbar_wait(&full[s], (it / kStages) & 1);
          if (ts_on && it < 8) g_dbg_ts[cta_lin * 32 + 2 + it] = gclk();
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + kb * 16384);
          const uint32_t b0 = smem_u32(sB + s * stage_bytes);
          if constexpr (TF32) {
            // 3xTF32: A_hi.B_hi + A_hi.B_lo + A_lo.B_hi (the lo.lo term is below fp32 rounding)
            const uint32_t b1 = b0 + p.n_tile * kRowBytes;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint32_t acc = (kb | kk) != 0;
              tc_mma_tf32(d, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32), idesc, acc);
              tc_mma_tf32(d, sw128_desc(a0 + kk * 32), sw128_desc(b1 + kk * 32), idesc, 1);
              tc_mma_tf32_ts(d, tmem + alo_col + kb * BK + kk * 8, sw128_desc(b0 + kk * 32), idesc, 1);
            }
          } else {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              tc_mma(d, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32), idesc, (kb | kk) != 0);
          }
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[buf]);
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ---------------------------------------------------------- epilogue
    // One thread per query row (TMEM lane).  Running group maxima over
    // G = 2KT strided groups (g = column % G) give a lower bound tau on the
    // row's KT-th score (the KT largest group maxima are KT distinct columns
    // >= tau), valid for the whole row at every point of the stream; columns
    // >= tau are kept in a shared-memory buffer that is compacted as tau
    // rises.  A row whose buffer would overflow (massive exact ties) switches
    // to an exact bitwise search for its KT-th score over buffer + segment.
    const int q = warp & 3;            // TMEM lane quarter of this warp
    const int row = q * 32 + lane;     // query row within the tile
    const int tid = row;               // candidate buffer column
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    if constexpr (TF32) {
      // split this row of the resident query tile: hi (TF32-exact) back into
      // shared memory in place, lo = x - hi into TMEM columns [alo_col, +d_h)
      mbar_wait(a_full, 0);
      const int sw = row & 7;
      for (int kb = 0; kb < p.k_blocks; ++kb) {
        float* arow = reinterpret_cast<float*>(sA + kb * 16384 + row * kRowBytes);
        uint32_t lo[32];
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          float4* pc = reinterpret_cast<float4*>(arow) + (ch ^ sw);  // logical chunk ch
          float4 x = *pc;
          float4 h = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
          *pc = h;
          lo[ch * 4 + 0] = __float_as_uint(x.x - h.x);
          lo[ch * 4 + 1] = __float_as_uint(x.y - h.y);
          lo[ch * 4 + 2] = __float_as_uint(x.z - h.z);
          lo[ch * 4 + 3] = __float_as_uint(x.w - h.w);
        }
        tmem_st32(lane_base + alo_col + kb * BK, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_ready);
    }
    constexpr int G = 2 * KT;
    constexpr int STEP = G > 32 ? G : 32;
    float tau = -INFINITY;  // lower bound on this row's KT-th score
    int cnt = 0;
    // exact KT-th (index tie rule) over the buffered candidates -> new tau;
    // keeps exactly the entries that can still be in the top-KT (<= KT).
    int n_tight = 0;  // profiling (MSN_SELECT_DBG): buffer compactions of this thread
    auto tighten = [&]() {
      ++n_tight;
      float t[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) t[i] = i < cnt ? __uint_as_float(cand[i * 128 + tid].x) : -INFINITY;
      bitonic_sort_vals<64>(t);
      const float nt = t[KT - 1];
      int gt = 0;
#pragma unroll
      for (int i = 0; i < KT; ++i) gt += t[i] > nt ? 1 : 0;
      int need = KT - gt;  // entries equal to nt that survive (earliest columns first)
      const int mx = __reduce_max_sync(0xffffffffu, cnt);
      int w = 0;
      for (int i = 0; i < mx; ++i) {
        if (i < cnt) {
          const uint2 e = cand[i * 128 + tid];
          const float v = __uint_as_float(e.x);
          const bool keep = v > nt || (v == nt && need > 0);
          if (v == nt && keep) --need;
          if (keep) cand[w++ * 128 + tid] = e;
        }
      }
      cnt = w;
      tau = fmaxf(tau, nt);
    };
    for (int c = 0; c < p.n_chunks;) {
      const int nseg = (c == 0 && p.n_chunks >= 2) ? 2 : 1;  // first segment: both TMEM buffers
      for (int u = 0; u < nseg; ++u) mbar_wait(&tfull[(c + u) & 1], ((c + u) >> 1) & 1);
      tc_fence_after();
      if (p.dbg == 1) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
          for (int u = 0; u < nseg; ++u) mbar_arrive(&tempty[(c + u) & 1]);
        c += nseg;
        continue;
      }
      const int seg_cols = nseg * p.n_tile;
      const bool first = c == 0;
      const bool stamp = ts_on && warp == kEpiWarp0 && lane == 0 && first;
      if (stamp) g_dbg_ts[cta_lin * 32 + 16] = gclk();
      if (ts_on && warp == kEpiWarp0 && lane == 0 && c >= 2 && c < 8) g_dbg_ts[cta_lin * 32 + 18 + c] = gclk();
      // TMEM address of segment column j
      auto taddr = [&](int j) -> uint32_t {  // j < 2 * n_tile
        const int hi = j >= p.n_tile ? 1 : 0;
        return lane_base + (uint32_t)(((c + hi) & 1) * acc_stride + (j - hi * p.n_tile));
      };
      if (first) {
        // pass A: tau = KT-th largest of the 2KT strided group maxima of the
        // first segment (KT distinct columns score >= tau, so the row's KT-th
        // score is >= tau).  Segment start 0 is a multiple of G.
        float gm[G];
#pragma unroll
        for (int j = 0; j < G; ++j) gm[j] = -INFINITY;
        if (seg_cols % 64 == 0) {
          for (int j0 = 0; j0 < seg_cols; j0 += 64) {
            uint32_t r[64];
            tmem_ld64(taddr(j0), r);  // n_tile % 64 == 0: never straddles a buffer
#pragma unroll
            for (int jj = 0; jj < 64; ++jj) gm[jj % G] = fmaxf(gm[jj % G], __uint_as_float(r[jj]));
          }
        } else {
          for (int j0 = 0; j0 < seg_cols; j0 += STEP) {
#pragma unroll
            for (int piece = 0; piece < STEP / 32; ++piece) {
              const int j = j0 + piece * 32;
              if (j < seg_cols) {
                uint32_t r[32];
                tmem_ld32(taddr(j), r);
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) {
                  const int g = (piece * 32 + jj) % G;
                  gm[g] = fmaxf(gm[g], __uint_as_float(r[jj]));
                }
              }
            }
          }
        }
        if (stamp) g_dbg_ts[cta_lin * 32 + 17] = gclk() + (unsigned long long)(gm[0] > 1e30f);
        bitonic_sort_vals<G>(gm);
        tau = gm[KT - 1];
        if (stamp) g_dbg_ts[cta_lin * 32 + 18] = gclk() + (unsigned long long)(tau > 1e30f);
      }
      // pass B: buffer the columns that can still be in the top-KT.  In the
      // first segment tau came from these same columns (ties kept: >=);
      // later columns lose every tie to the KT earlier ones behind tau (>).
      // Branch-free: every column is stored, unselected ones (and any
      // first-segment overflow) into the dummy row kCap.
      const int cnt_old = cnt;
      const int col_base = c * p.n_tile;
      // One compact code path per 32-column piece (the unrolled variants did
      // not fit the instruction cache): a column is a hit when v > te, where
      // te = tau in later segments and the largest float below tau in the
      // first (ties with tau kept there).  Hit mask; if a later segment's
      // hits would not fit, compact the buffer first (tau rises) and redo the
      // mask; then every hit goes to slot cnt + (hits before it), with no
      // dependency between the stores.  A first-segment overflow stores what
      // fits and leaves the rest to the exact path below (cnt > kCap).
      auto piece = [&](const uint32_t (&r)[32], int j0) {
        const uint32_t colj = (uint32_t)(col_base + j0);
        uint32_t m;
        for (;;) {
          const float te = first ? nextafterf(tau, -INFINITY) : tau;
          m = 0;
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) m |= (__uint_as_float(r[jj]) > te ? 1u : 0u) << jj;
          if (first || !__any_sync(0xffffffffu, cnt + __popc(m) > kCap)) break;
          tighten();  // cnt <= KT; tau only rises
        }
        if (m) {
          const uint32_t base = smem_u32(cand + tid);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const uint32_t slot = (uint32_t)cnt + (uint32_t)__popc(m & ((1u << jj) - 1u));
            asm volatile(
                "{\n.reg .pred p, q;\n"
                "setp.ne.u32 p, %1, 0;\n"
                "setp.lt.and.u32 q, %2, %5, p;\n"
                "@q st.shared.v2.u32 [%0], {%3, %4};\n}\n" ::"r"(base + (slot << 10)),
                "r"(m & (1u << jj)), "r"(slot), "r"(r[jj]), "r"(colj + jj), "r"((uint32_t)kCap)
                : "memory");
          }
        }
        cnt += __popc(m);
      };
      for (int j0 = 0; j0 < seg_cols; j0 += 32) {
        uint32_t r[32];
        tmem_ld32(taddr(j0), r);
        piece(r, j0);
      }
      const bool ovf = cnt > kCap;  // first segment only (later pieces tighten first)
      if (ts_on && warp == kEpiWarp0 && lane == 0 && c >= 2 && c < 8) g_dbg_ts[cta_lin * 32 + 24 + c] = gclk();
      if (stamp) g_dbg_ts[cta_lin * 32 + 20] = gclk();
      if (stamp) g_dbg_ts[cta_lin * 32 + 19] = gclk() + (unsigned long long)(cnt > 100000);
      if (__any_sync(0xffffffffu, ovf)) {
        // exact path: the KT-th largest ordered key t over buffer u segment
        auto count_ge = [&](uint32_t t) -> int {
          int n = 0;
          for (int i = 0; i < cnt_old; ++i) n += ord_f32(__uint_as_float(cand[i * 128 + tid].x)) >= t ? 1 : 0;
          for (int j0 = 0; j0 < seg_cols; j0 += 32) {
            uint32_t r[32];
            tmem_ld32(taddr(j0), r);
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) n += ord_f32(__uint_as_float(r[jj])) >= t ? 1 : 0;
          }
          return n;
        };
        uint32_t t = 0;
        for (int bit = 31; bit >= 0; --bit) {
          const uint32_t ct = t | (1u << bit);
          if (count_ge(ct) >= KT) t = ct;
        }
        const int gt = (t == 0xffffffffu) ? 0 : count_ge(t + 1);
        int need = KT - gt;
        int w = 0;
        for (int i = 0; i < cnt_old; ++i) {
          const uint2 e = cand[i * 128 + tid];
          const uint32_t o = ord_f32(__uint_as_float(e.x));
          if (o > t || (o == t && need > 0)) {
            if (o == t) --need;
            cand[w++ * 128 + tid] = e;
          }
        }
        for (int j0 = 0; j0 < seg_cols; j0 += 32) {
          uint32_t r[32];
          tmem_ld32(taddr(j0), r);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const uint32_t o = ord_f32(__uint_as_float(r[jj]));
            if (o > t || (o == t && need > 0)) {
              if (o == t) --need;
              cand[w++ * 128 + tid] = make_uint2(r[jj], (uint32_t)(col_base + j0 + jj));
            }
          }
        }
        cnt = w;  // <= KT
        tau = fmaxf(tau, unord_f32(t));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        for (int u = 0; u < nseg; ++u) mbar_arrive(&tempty[(c + u) & 1]);
      c += nseg;
    }
    // coalesced write-out: the warp writes its 32 rows one after another
    // (lane = candidate slot), instead of 32 rows per store instruction
    // (row, slot half) tasks, 8 in flight: their shared-memory reads and
    // global stores are independent
    {
      const int64_t b_me = m0 + q * 32 + lane;
      if (b_me < p.B) p.cn[b_me * p.H * 2 + hh] = cnt;
    }
    for (int t0 = 0; t0 < 64; t0 += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + u, rr = t >> 1, i = (t & 1) * 32 + lane;
        const int n = __shfl_sync(0xffffffffu, cnt, rr);
        const int trow = q * 32 + rr;
        const int64_t b = m0 + trow;
        if (b < p.B && i < n) {
          const uint2 e = cand[i * 128 + trow];
          const int64_t o = (b * p.H * 2 + hh) * kCandCap + i;
          p.cv[o] = __uint_as_float(e.x);
          p.cc[o] = (int32_t)e.y;
        }
      }
    }
    if (ts_on && warp == kEpiWarp0 && lane == 0) g_dbg_ts[cta_lin * 32 + 14] = gclk();
    if (ts_on && warp == kEpiWarp0 && lane == 0) g_dbg_ts[cta_lin * 32 + 15] = (unsigned long long)n_tight;
  }
  tc_fence_before();
  __syncthreads();
  if (ts_on && threadIdx.x == 0) g_dbg_ts[cta_lin * 32 + 10] = gclk();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    if (ts_on && lane == 0) g_dbg_ts[cta_lin * 32 + 12] = gclk();
  }
}

// ------------------------------------------------------------- host --------
bool is_tf32(const Shape& s) { return s.qk_dt == F32; }

// Largest N tile (<= 256, multiple of 32, dividing n_sub); TF32 also keeps
// 2 accumulators + the A_lo operand (d_h columns) within 512 TMEM columns.
int n_tile_for(const Shape& s) {
  const int cap = is_tf32(s) ? (512 - s.d_h) / 2 : kMaxNTile;
  for (int nt = cap - cap % 32; nt >= 32; nt -= 32)
    if (s.n_sub % nt == 0) return nt;
  return 0;
}

size_t smem_bytes(const Shape& s) {
  const int nt = n_tile_for(s);
  const int bk = is_tf32(s) ? 32 : 64;
  const int parts = is_tf32(s) ? 2 : 1;
  return 1024 + (size_t)(s.d_h / bk) * 16384 + (size_t)kStages * parts * nt * kRowBytes +
         (size_t)(kCap + 1) * 128 * 8 + 8 * (1 + 2 * kStages + 5) + 16;
}

// K -> (K_hi, K_lo) for the 3xTF32 B operand.
__global__ void split_tf32_kernel(const float* __restrict__ k, float* __restrict__ hi,
                                  float* __restrict__ lo, int64_t n) {
  pdl_enter();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float x = k[i];
  const float h = tf32_hi(x);
  hi[i] = h;
  lo[i] = x - h;
}

template <int KT, bool TF32>
cudaError_t launch_kt(const Shape& s, const CUtensorMap& mq, const CUtensorMap& mk,
                      const CUtensorMap& mklo, TcParams p, cudaStream_t st) {
  const size_t sm = smem_bytes(s);
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(select_tc_kernel<KT, TF32>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  // x = head/half (fastest): concurrently resident CTAs spread over all 2H
  // sub-key codebooks instead of hammering one codebook's lines in L2
  dim3 grid(s.H * 2, (unsigned)((s.B + 127) / 128));
  launch_pdl(select_tc_kernel<KT, TF32>, grid, kThreads, sm, st, mq, mk, mklo, p);
  return cudaGetLastError();
}

}  // namespace

size_t select_tc_workspace_bytes(const Shape& s) {
  return is_tf32(s) ? 2 * sizeof(float) * (size_t)s.H * 2 * s.n_sub * s.d_h : 0;
}

bool select_tc_supported(const Shape& s) {
  const bool tf = is_tf32(s);
  if (s.qk_dt != BF16 && s.qk_dt != F32) return false;
  const int bk = tf ? 32 : 64;
  if (s.d_h % bk != 0 || s.d_h > (tf ? 128 : 256)) return false;
  const int nt = n_tile_for(s);
  if (nt == 0 || s.n_sub > 65535) return false;
  if (s.k > 32) return false;
  if (smem_bytes(s) > 227 * 1024) return false;
  return get_encode() != nullptr;
}

cudaError_t launch_select_tc(const Shape& s, const void* Q, const void* K, const Cands& cd,
                             void* ws, cudaStream_t st, int* launches) {
  if (!select_tc_supported(s)) return cudaErrorNotSupported;
  const bool tf = is_tf32(s);
  const int bk = tf ? 32 : 64;
  const int esz = tf ? 4 : 2;
  const CUtensorMapDataType dt = tf ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  EncodeTiledFn enc = get_encode();
  CUtensorMap mq, mk, mklo;
  {
    // Q [B, H*2, d_h]: dims (d_h, H*2, B); box (one 128-B row, 1, 128)
    cuuint64_t dims[3] = {(cuuint64_t)s.d_h, (cuuint64_t)(s.H * 2), (cuuint64_t)s.B};
    cuuint64_t strides[2] = {(cuuint64_t)s.d_h * esz, (cuuint64_t)s.H * 2 * s.d_h * esz};
    cuuint32_t box[3] = {(cuuint32_t)bk, 1, 128};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&mq, dt, 3, const_cast<void*>(Q), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int nt = n_tile_for(s);
  const int64_t kel = (int64_t)s.H * 2 * s.n_sub * s.d_h;
  const void* kb_hi = K;
  const void* kb_lo = K;
  if (tf) {
    float* hi = (float*)ws;
    float* lo = hi + kel;
    launch_pdl(split_tf32_kernel, (unsigned)((kel + 255) / 256), 256, 0, st, (const float*)K, hi, lo, kel);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ++*launches;
    kb_hi = hi;
    kb_lo = lo;
  }
  auto kmap = [&](CUtensorMap* m, const void* base) -> bool {
    // K [H*2*n_sub, d_h]: dims (d_h, H*2*n_sub); box (one 128-B row, n_tile)
    cuuint64_t dims[2] = {(cuuint64_t)s.d_h, (cuuint64_t)s.H * 2 * s.n_sub};
    cuuint64_t strides[1] = {(cuuint64_t)s.d_h * esz};
    cuuint32_t box[2] = {(cuuint32_t)bk, (cuuint32_t)nt};
    cuuint32_t es[2] = {1, 1};
    return enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  if (!kmap(&mk, kb_hi) || !kmap(&mklo, kb_lo)) return cudaErrorInvalidValue;
  static const int dbg = getenv("MSN_SELECT_DBG") ? atoi(getenv("MSN_SELECT_DBG")) : 0;
  TcParams p{dbg, s.B, s.H, s.n_sub, s.d_h, s.k, nt, s.n_sub / nt, s.d_h / bk, cd.v, cd.c, cd.n};
  cudaError_t e;
  if (tf) {
    if (s.k <= 8) e = launch_kt<8, true>(s, mq, mk, mklo, p, st);
    else if (s.k <= 16) e = launch_kt<16, true>(s, mq, mk, mklo, p, st);
    else e = launch_kt<32, true>(s, mq, mk, mklo, p, st);
  } else {
    if (s.k <= 8) e = launch_kt<8, false>(s, mq, mk, mklo, p, st);
    else if (s.k <= 16) e = launch_kt<16, false>(s, mq, mk, mklo, p, st);
    else e = launch_kt<32, false>(s, mq, mk, mklo, p, st);
  }
  if (e == cudaSuccess) ++*launches;
  if (dbg >= 2 && e == cudaSuccess) {
    cudaStreamSynchronize(st);
    static unsigned long long h[4096 * 32];
    cudaMemcpyFromSymbol(h, g_dbg_ts, sizeof(h));
    const int ncta = (int)std::min<int64_t>(4096, (s.B + 127) / 128 * s.H * 2);
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < ncta; ++c) t0 = std::min(t0, h[c * 32]);
    double acc[16] = {0};
    for (int c = 0; c < ncta; ++c)
      for (int j = 0; j < 15; ++j) if (j != 11 && j != 13 && j != 15) acc[j] += ((double)h[c * 32 + j] - (double)h[c * 32]) / ncta;
    double ph[4] = {0, 0, 0, 0};
    for (int c = 0; c < ncta; ++c)
      for (int j = 0; j < 4; ++j) ph[j] += ((double)h[c * 32 + 16 + j] - (double)h[c * 32]) / ncta;
    fprintf(stderr, "epilogue: tfull seen %.0f, passA %.0f, tau %.0f, passB %.0f, done %.0f; dealloc %.0f ns after CTA start\n",
            ph[0], ph[1], ph[2], ph[3], acc[14], acc[12]);
    double ch[16] = {0};
    for (int c = 0; c < ncta; ++c)
      for (int j = 20; j < 32; ++j) ch[j - 20] += ((double)h[c * 32 + j] - (double)h[c * 32]) / ncta;
    fprintf(stderr, "first seg passB stamp(20) %.0f; chunks 2..5 seen/done: %.0f/%.0f %.0f/%.0f %.0f/%.0f %.0f/%.0f\n",
            ch[0], ch[0 + 2 - 2 + 2], ch[6 + 2], ch[3], ch[9], ch[4], ch[10], ch[5], ch[11]);
    double span = 0;
    for (int c = 0; c < ncta; ++c) span = std::max(span, (double)(h[c * 32 + 10] - t0));
    {
      std::vector<double> st(ncta), en(ncta);
      for (int c = 0; c < ncta; ++c) { st[c] = (double)(h[c * 32] - t0); en[c] = (double)(h[c * 32 + 10] - t0); }
      std::vector<double> ss = st; std::sort(ss.begin(), ss.end());
      int per_sm[256] = {0};
      for (int c = 0; c < ncta; ++c) per_sm[h[c * 32 + 11] & 255]++;
      int maxc = 0, nsm = 0;
      for (int i = 0; i < 256; ++i) { maxc = std::max(maxc, per_sm[i]); nsm += per_sm[i] > 0; }
      // per SM: order CTAs by start, report gap between a CTA's dealloc and the next one's entry
      double gap = 0, ent = 0; int ng = 0;
      for (int c = 0; c < ncta; ++c) {
        ent += (double)(h[c * 32] - h[c * 32 + 13]) / ncta;
        int best = -1;
        for (int d = 0; d < ncta; ++d)
          if (h[d * 32 + 11] == h[c * 32 + 11] && h[d * 32 + 13] > h[c * 32 + 13] &&
              (best < 0 || h[d * 32 + 13] < h[best * 32 + 13])) best = d;
        if (best >= 0) { gap += (double)h[best * 32 + 13] - (double)h[c * 32 + 12]; ++ng; }
      }
      fprintf(stderr, "entry->start(alloc+init) %.0f ns; dealloc->next entry on same SM %.0f ns (n=%d)\n", ent, ng ? gap / ng : 0.0, ng);
      fprintf(stderr, "starts: p0 %.0f p25 %.0f p50 %.0f p75 %.0f p100 %.0f ns; SMs used %d, max CTAs/SM %d\n",
              ss[0], ss[ncta / 4], ss[ncta / 2], ss[3 * ncta / 4], ss[ncta - 1], nsm, maxc);
    }
    {
      double nt = 0;
      for (int c = 0; c < ncta; ++c) nt += (double)h[c * 32 + 15] / ncta;
      fprintf(stderr, "tighten calls per epilogue warp (warp 4): %.2f\n", nt);
    }
    fprintf(stderr, "select_tc ts (ns, mean rel. to CTA start): Afull %.0f  full0..7 %.0f %.0f %.0f %.0f %.0f %.0f %.0f %.0f  end %.0f  | kernel span %.0f\n",
            acc[1], acc[2], acc[3], acc[4], acc[5], acc[6], acc[7], acc[8], acc[9], acc[10], span);
  }
  return e;
}

}  // namespace msn
