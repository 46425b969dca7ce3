// select_tc.cu -- steps a1 + a2 on the 5th-generation tensor cores:
// sub-key scoring S = K q (Eq. S_old) as a tcgen05 GEMM
// fed by TMA, with the per-half argtopk fused into the
// epilogue so that S never reaches HBM.
//
// One CTA per (128-query tile, head h, half): D[128 x n_sub] = Q_half . K_half^T
// with bf16 operands and fp32 accumulation in TMEM (kind::f16; fp32 inputs:
// 3xTF32 kind::tf32), computed in N-chunks of up to 256 columns that
// alternate between two TMEM accumulator buffers.
//
//   warp 0       TMA producer: the whole query tile once (resident), then the
//                sub-key tiles through a kStages-deep mbarrier ring
//   warp 1       MMA issuer (one elected lane): tcgen05.mma + tcgen05.commit
//   warp 2       TMEM allocator (512 columns)
//   warps 4-11   epilogue, TWO threads per query row: warp 4+q and warp 8+q
//                both read TMEM lane quarter q (row = 32q + lane) and split the
//                row's columns (alternate 64-column blocks).
//
// Epilogue = two passes over the row, no data-dependent buffer management:
//   pass A  each thread folds its columns into KT group maxima (group =
//           column mod KT within its blocks); the two threads' KT maxima come
//           from 2KT disjoint column groups, so the KT-th largest of their
//           union, tau, is a provable lower bound on the row's KT-th score.
//           Both threads sort their KT maxima (descending), swap them through
//           shared memory, and take tau = min_i max(A_i, B_{KT-1-i}) -- the
//           half-cleaner of a bitonic merge, which is exactly the KT-th
//           largest of A u B.
//   pass B  every column with score >= tau is appended to the row's
//           64-entry candidate buffer, thread 0 filling it from the bottom,
//           thread 1 from the top (no atomics).  The row's top-KT under
//           (score desc, index asc) has scores >= tau, so the list contains
//           it (ties with tau are kept).
// For random scores ~1.3 KT columns pass.  A row with more than CAP (64; 128 for KT = 64)
// passing columns (massive exact ties, adversarial data) is written with
// is rescored exactly by its write-out warp (warp_sort.cuh, exact_half_topk)
// -- correctness never depends on the bound being tight.
//
// Small grids of bf16 rows with n_sub <= 1024 split every row over S = 2 or 4
// CTAs (select_segments; C5: 32 -> 128 CTAs, S = 4; blockIdx.z = column
// segment of n_sub / S >= 256 columns, each resident and scored once): each
// CTA writes the list of its own columns (a superset of that segment's
// top-KT), the Cartesian stage merges the S lists.
// Rows that fit TMEM (n_sub <= 512, two buffers) are scored once; longer rows
// are scored twice (the MMA pass is cheap next to the epilogue): the first
// pass feeds pass A, the second pass B, so tau is the whole row's bound.
// fp32 inputs score the first pass with ONE TF32 product (hi.hi) instead of
// three: |S_1x - S_3x| <= 2^-9 sum_e |q_e||k_e| + accumulation rounding
// (|x - hi(x)| < 2^-10 |x|), so with d = 2^-8 ||q|| max_i ||k_i|| every
// first-pass group maximum exceeds a column whose 3xTF32 score is >= it - d,
// and tau - d (rounded down) bounds the 3xTF32 KT-th score from below.
#include <cuda.h>
#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"
#include "warp_sort.cuh"

namespace msn {
namespace {
using namespace tc;

constexpr int kEpiWarp0 = 4;
constexpr int kEpiWarps = 8;                         // 2 threads per row
constexpr int kThreads = 32 * (kEpiWarp0 + kEpiWarps);
constexpr int kStages = 3;
constexpr int kMaxNTile = 256;
// candidate slots per row list: cand_cap(KT) (kernels.h)
constexpr int kCStride = 129;      // buffer entry (slot, row) at slot*129 + row: bank rotation
constexpr int kRowBytes = 128;     // one 128-byte swizzle row per k-block (64 bf16 / 32 fp32)

// In-register bitonic sort of N values, descending.
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

__device__ __forceinline__ void epi_bar() {  // the 8 epilogue warps only
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
}

// Thread-block cluster (the column segments of one row tile): a full cluster
// barrier (every thread of every CTA; release / acquire orders the shared
// stores before the peers' DSMEM loads), the rank, and a peer's copy of a
// shared address.
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t peer_addr(uint32_t local, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(local), "r"(rank));
  return a;
}
__device__ __forceinline__ void st_peer_f32(uint32_t a, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

// Sorts a bitonic sequence of N values descending (the merge half of a
// bitonic sort).
template <int N>
__device__ __forceinline__ void bitonic_merge_desc(float (&v)[N]) {
#pragma unroll
  for (int stride = N >> 1; stride > 0; stride >>= 1)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int j = i ^ stride;
      if (j > i) {
        const float hi = fmaxf(v[i], v[j]), lo = fminf(v[i], v[j]);
        v[i] = hi;
        v[j] = lo;
      }
    }
}

// MSN_SELECT_TS builds (profiling only): globaltimer stamps per CTA at the
// epilogue's phase boundaries (warp 4, lane 0), summarised by tools/select_ts.py.
#ifdef MSN_SELECT_TS
__device__ unsigned long long g_sel_ts[65536 * 16];
#define SEL_TS_ANY(i)                                                               \
  do {                                                                              \
    unsigned long long t_;                                                          \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
    const int c_ = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;                             \
    if (c_ < 65536) g_sel_ts[c_ * 16 + (i)] = t_;                                   \
  } while (0)
#define SEL_TS(i)                                                                   \
  do {                                                                              \
    if (threadIdx.x == 32 * kEpiWarp0) SEL_TS_ANY(i);                               \
  } while (0)
#else
#define SEL_TS(i) do {} while (0)
#define SEL_TS_ANY(i) do {} while (0)
#endif

struct TcParams {
  int64_t B;
  int H, n_sub, d_h, k;
  int n_tile, n_chunks, k_blocks, passes;
  uint2* vc;
  int32_t* cn;
  Rescore rq;
  const float* knorm;  // TF32, two sweeps: ||k_i|| (rounded up) per sub-key row [H*2*n_sub]  // overflowed rows are rescored exactly from these
  int seg_cols;        // columns per CTA: n_sub / S (blockIdx.z = column segment)
  int SC;              // segment slots per row in vc / cn
  void* qhat = nullptr;  // f2: LayerNorm the query tile on load, q^ written here (nullptr: off)
};

template <int KT, bool TF32, bool WIDE, bool SEG>
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
  constexpr int CAP = cand_cap(KT);
  // carve: A (k_blocks x 16 KB) | B ring | candidates [CAP][129] (score bits,
  //        column) | per-thread counts [2][128] | bars.  The tau exchange
  //        [KT][2][128] and ||q||^2 reuse the candidate area.
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* sA = smem_raw + pad;
  uint8_t* sB = sA + p.k_blocks * 16384;
  const int stage_bytes = B_PARTS * p.n_tile * kRowBytes;
  uint2* cand = reinterpret_cast<uint2*>(sB + kStages * stage_bytes);
  float* xch = reinterpret_cast<float*>(cand);            // [KT][2][128] sorted group maxima
  // ||q||^2 halves: the last 1 KB of the candidate area (written before pass A,
  // read at tau, before pass B fills the buffer; the tau exchange at its start
  // is at most KT KB < the area - 1 KB)
  float* qn = reinterpret_cast<float*>(cand + CAP * kCStride) - 256;  // [2][128]
  int* cnts = reinterpret_cast<int*>(cand + CAP * kCStride);          // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(cnts + 256);
  uint64_t* a_full = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* a_ready = tempty + 2;  // TF32: A split into (hi in smem, lo in TMEM)
  uint32_t* tmem_slot = (uint32_t*)(a_ready + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int hh = blockIdx.x;  // h*2 + half
  const int64_t m0 = (int64_t)blockIdx.y * 128;
  const int seg = SEG ? (int)blockIdx.z : 0;  // column segment [col_seg, col_seg + seg_cols)
  const int col_seg = SEG ? seg * p.seg_cols : 0;
  const int total_chunks = p.passes * p.n_chunks;

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
      mbar_init(&tempty[b], kEpiWarps);
    }
    mbar_init(a_ready, kEpiWarps);
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
  SEL_TS(0);

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_expect_tx(a_full, p.k_blocks * 16384);
      for (int kb = 0; kb < p.k_blocks; ++kb)
        tma_load_3d(sA + kb * 16384, &tmap_q, a_full, kb * BK, hh, (int)m0);
      int it = 0;
      for (int g = 0; g < total_chunks; ++g) {
        const int c = g % p.n_chunks;
        const bool one = TF32 && WIDE && g < p.n_chunks;  // 1xTF32 first sweep: K_hi only ...
        const int kstep = one ? 2 : 1;                     // ... two k-blocks per stage (both halves)
        const int krow = hh * p.n_sub + col_seg + c * p.n_tile;
        for (int kb = 0; kb < p.k_blocks; kb += kstep, ++it) {
          const int s = it % kStages;
          mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          const bool second = TF32 && (!one || kb + 1 < p.k_blocks);
          mbar_expect_tx(&full[s], second ? stage_bytes : p.n_tile * kRowBytes);
          tma_load_2d(sB + s * stage_bytes, &tmap_k, &full[s], kb * BK, krow);
          if (second)
            tma_load_2d(sB + s * stage_bytes + p.n_tile * kRowBytes, one ? &tmap_k : &tmap_klo, &full[s],
                        (one ? kb + 1 : kb) * BK, krow);
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = TF32 ? idesc_tf32(128, p.n_tile) : idesc_bf16(128, p.n_tile);
      mbar_wait(a_full, 0);
      SEL_TS_ANY(14);
      if (TF32 || p.qhat) mbar_wait(a_ready, 0);
      SEL_TS_ANY(15);
      tc_fence_after();
      int it = 0;
      for (int g = 0; g < total_chunks; ++g) {
        const int buf = g & 1;
        mbar_wait(&tempty[buf], ((g >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * acc_stride;
        const bool one = TF32 && WIDE && g < p.n_chunks;
        const int kstep = one ? 2 : 1;
        for (int kb = 0; kb < p.k_blocks; kb += kstep, ++it) {
          const int s = it % kStages;
          mbar_wait(&full[s], (it / kStages) & 1);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + kb * 16384);
          const uint32_t b0 = smem_u32(sB + s * stage_bytes);
          if constexpr (TF32) {
            // 3xTF32: A_hi.B_hi + A_hi.B_lo + A_lo.B_hi (the lo.lo term is below fp32 rounding);
            // the first sweep of a two-sweep row: A_hi.B_hi only (pass A, margin d), the
            // stage holding k-blocks kb and kb + 1
            const uint32_t b1 = b0 + p.n_tile * kRowBytes;
            if (one) {
#pragma unroll
              for (int kk = 0; kk < BK / 8; ++kk)
                tc_mma_tf32(d, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32), idesc, (kb | kk) != 0);
              if (kb + 1 < p.k_blocks) {
                const uint32_t a1 = a0 + 16384;
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk)
                  tc_mma_tf32(d, sw128_desc(a1 + kk * 32), sw128_desc(b1 + kk * 32), idesc, 1);
              }
            } else {
#pragma unroll
              for (int kk = 0; kk < BK / 8; ++kk) {
                const uint32_t acc = (kb | kk) != 0;
                tc_mma_tf32(d, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32), idesc, acc);
                tc_mma_tf32(d, sw128_desc(a0 + kk * 32), sw128_desc(b1 + kk * 32), idesc, 1);
                tc_mma_tf32_ts(d, tmem + alo_col + kb * BK + kk * 8, sw128_desc(b0 + kk * 32), idesc, 1);
              }
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
  }
  if (SEG && warp < kEpiWarp0) {
    // (the epilogue's tau exchange: every thread of the cluster arrives)
    cluster_sync();
  } else if (warp >= kEpiWarp0) {
    // ---------------------------------------------------------- epilogue
    const int ew = warp - kEpiWarp0;   // 0..7
    const int q = ew & 3;              // TMEM lane quarter (== warp % 4)
    const int sh = ew >> 2;            // column share of this thread: 0 or 1
    const int row = q * 32 + lane;     // query row within the tile
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    // f2: LayerNorm of the query row folded into the operand
    // load (reading R23: no affine, eps = 1e-5): the resident
    // query tile is normalised in place in shared memory before any MMA reads
    // it (two passes over the row: mean, then variance; the two threads of a
    // row exchange their halves' sums), and q^ is written out for the
    // backward (q_hat [B, H, 2, d_h], rounded once to the query dtype).
    if (p.qhat) {
      using QT = typename std::conditional<TF32, float, __nv_bfloat16>::type;
      constexpr int EPC = 16 / (int)sizeof(QT);  // elements per 16-byte chunk
      mbar_wait(a_full, 0);
      float* lnx = reinterpret_cast<float*>(cnts);  // [2][128] (the counts come much later)
      const int sw = row & 7;
      const int64_t b = m0 + row;
      auto chunk = [&](int kb, int ch) -> uint4* {
        return reinterpret_cast<uint4*>(sA + kb * 16384 + row * kRowBytes) + (ch ^ sw);
      };
      float sum = 0.f;
      for (int kb = sh; kb < p.k_blocks; kb += 2)
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          float f[EPC];
          unpack16<QT>(*chunk(kb, ch), f);
#pragma unroll
          for (int e = 0; e < EPC; ++e) sum += f[e];
        }
      lnx[sh * 128 + row] = sum;
      epi_bar();
      const float mu = (lnx[row] + lnx[128 + row]) / (float)p.d_h;
      epi_bar();
      float ss = 0.f;
      for (int kb = sh; kb < p.k_blocks; kb += 2)
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          float f[EPC];
          unpack16<QT>(*chunk(kb, ch), f);
#pragma unroll
          for (int e = 0; e < EPC; ++e) ss += (f[e] - mu) * (f[e] - mu);
        }
      lnx[sh * 128 + row] = ss;
      epi_bar();
      const float rs = rsqrtf((lnx[row] + lnx[128 + row]) / (float)p.d_h + 1e-5f);
      QT* qh = reinterpret_cast<QT*>(p.qhat) + (b * p.H * 2 + hh) * (int64_t)p.d_h;
      for (int kb = sh; kb < p.k_blocks; kb += 2)
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          uint4* c = chunk(kb, ch);
          float f[EPC];
          unpack16<QT>(*c, f);
          uint4 o;
          if constexpr (TF32) {
            o = make_uint4(__float_as_uint((f[0] - mu) * rs), __float_as_uint((f[1] - mu) * rs),
                           __float_as_uint((f[2] - mu) * rs), __float_as_uint((f[3] - mu) * rs));
          } else {
            uint32_t w[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const __nv_bfloat162 v = __floats2bfloat162_rn((f[2 * t] - mu) * rs, (f[2 * t + 1] - mu) * rs);
              w[t] = *reinterpret_cast<const uint32_t*>(&v);
            }
            o = make_uint4(w[0], w[1], w[2], w[3]);
          }
          *c = o;
          if (b < p.B) *reinterpret_cast<uint4*>(qh + kb * (kRowBytes / (int)sizeof(QT)) + ch * EPC) = o;
        }
      epi_bar();  // (the exchange slots are reused below)
      if constexpr (!TF32) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(a_ready);
      }
    }
    // TF32 two-sweep rows: margin d = 2^-8 ||q_row|| max_i ||k_i|| on the
    // 1xTF32 first sweep (see the header); ||q|| from the split below (qn)
    if constexpr (TF32) {
      {
        // split this row of the resident query tile: hi (TF32-exact) back into
        // shared memory in place, lo = x - hi into TMEM columns [alo_col, +d_h);
        // the two warps of a lane quarter take alternate k-blocks
        mbar_wait(a_full, 0);
        const int sw = row & 7;
        float qq = 0.f;
        for (int kb = sh; kb < p.k_blocks; kb += 2) {
          float* arow = reinterpret_cast<float*>(sA + kb * 16384 + row * kRowBytes);
          uint32_t lo[32];
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            float4* pc = reinterpret_cast<float4*>(arow) + (ch ^ sw);  // logical chunk ch
            float4 x = *pc;
            qq = fmaf(x.x, x.x, fmaf(x.y, x.y, fmaf(x.z, x.z, fmaf(x.w, x.w, qq))));
            float4 h = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
            *pc = h;
            lo[ch * 4 + 0] = __float_as_uint(x.x - h.x);
            lo[ch * 4 + 1] = __float_as_uint(x.y - h.y);
            lo[ch * 4 + 2] = __float_as_uint(x.z - h.z);
            lo[ch * 4 + 3] = __float_as_uint(x.w - h.w);
          }
          tmem_st32(lane_base + alo_col + kb * BK, lo);
        }
        if (WIDE) qn[sh * 128 + row] = qq;  // the two halves of ||q||^2, added at tau
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_ready);
      }
    }
    float kmax = 0.f;
    if constexpr (TF32 && WIDE) {
      for (int i = threadIdx.x - 32 * kEpiWarp0; i < p.n_sub; i += 32 * kEpiWarps)
        kmax = fmaxf(kmax, p.knorm[(int64_t)hh * p.n_sub + i]);
      kmax = warp_max(kmax);
      if (lane == 0) cnts[ew] = __float_as_int(kmax);
      epi_bar();
      kmax = 0.f;
#pragma unroll
      for (int i = 0; i < kEpiWarps; ++i) kmax = fmaxf(kmax, __int_as_float(cnts[i]));
    }
    // A segment = nseg consecutive chunks starting at global chunk g0, resident
    // in the TMEM buffers (g0 + u) & 1.  This thread owns the 32-column pieces
    // of the 64-column blocks b with b % 2 == sh (a lone last piece belongs to
    // the thread whose block it starts).
    auto piece_addr = [&](int g0, int j) -> uint32_t {  // segment column j (multiple of 32)
      const int u = j / p.n_tile;
      return lane_base + (uint32_t)(((g0 + u) & 1) * acc_stride + (j - u * p.n_tile));
    };
    auto wait_chunks = [&](int g0, int nseg) {
      for (int u = 0; u < nseg; ++u) mbar_wait(&tfull[(g0 + u) & 1], ((g0 + u) >> 1) & 1);
      tc_fence_after();
    };
    auto release_chunks = [&](int g0, int nseg) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        for (int u = 0; u < nseg; ++u) mbar_arrive(&tempty[(g0 + u) & 1]);
    };

    // ---- pass A: G group maxima over this thread's columns (G = KT; WIDE,
    // for rows longer than TMEM: G = 2KT, a tighter tau for the longer row)
    constexpr int G = (WIDE && KT <= 32) ? 2 * KT : KT;  // (KT = 64: 64 registers of maxima)
    constexpr int GP = G < 32 ? G : 32;  // groups fed by one 32-column piece
    float gm[G];
#pragma unroll
    for (int i = 0; i < G; ++i) gm[i] = -INFINITY;
    int gsel = 0;  // WIDE, G = 64: which half of gm this piece feeds (piece parity)
    auto fold32 = [&](const uint32_t (&r)[32]) {
#pragma unroll
      for (int jj = 0; jj < 32; jj += GP)
#pragma unroll
        for (int i = 0; i < GP; ++i) {
          if (G > 32 && gsel) gm[(G > 32 ? 32 : 0) + i] = fmaxf(gm[(G > 32 ? 32 : 0) + i], __uint_as_float(r[jj + i]));
          else gm[i] = fmaxf(gm[i], __uint_as_float(r[jj + i]));
        }
    };
    auto pass_a = [&](int g0, int seg_cols) {
      for (int j0 = 64 * sh; j0 < seg_cols; j0 += 128) {
        uint32_t ra[32], rb[32];
        const bool two = j0 + 32 < seg_cols;
        tmem_ld32_async(piece_addr(g0, j0), ra);
        if (two) tmem_ld32_async(piece_addr(g0, j0 + 32), rb);
        tmem_wait_ld(ra);
        if (two && G <= 32) {
          tmem_wait_ld(rb);
#pragma unroll
          for (int jj = 0; jj < 32; jj += GP)
#pragma unroll
            for (int i = 0; i < GP; ++i)
              gm[i] = fmaxf(gm[i], fmaxf(__uint_as_float(ra[jj + i]), __uint_as_float(rb[jj + i])));
        } else {
          gsel = 0;
          fold32(ra);
          if (two) {
            tmem_wait_ld(rb);
            gsel = 1;
            fold32(rb);
          }
        }
      }
    };
    const bool resident = p.passes == 1;  // whole row in the two TMEM buffers
    if (resident) {
      // chunk by chunk, so that pass A over chunk 0 runs under the MMA of chunk 1
      // (both stay resident for pass B)
      for (int c = 0; c < p.n_chunks; ++c) {
        wait_chunks(c, 1);
        if (c == 0) SEL_TS(1);
        pass_a(c, p.n_tile);
      }
    } else {
      for (int c = 0; c < p.n_chunks; ++c) {
        wait_chunks(c, 1);
        if (c < 7) SEL_TS(7 + c);
        pass_a(c, p.n_tile);
        release_chunks(c, 1);
      }
    }

    SEL_TS(2);
    // ---- tau = KT-th largest of the 2G group maxima of the row: each thread
    // sorts its G maxima, the two top-KT lists meet in the half-cleaner
    bitonic_sort_vals<G>(gm);
#pragma unroll
    for (int i = 0; i < KT; ++i) xch[(i * 2 + sh) * 128 + row] = gm[i];
    epi_bar();
    float tau = INFINITY;
    if constexpr (SEG) {
      // column segments (a cluster of S = gridDim.z CTAs along z): a bound on
      // the WHOLE row, so that each segment lists only its columns >= it
      // (~1.2 KT candidates per row over all S lists, not per list).  Each
      // CTA takes the sorted top-Q of its 2G group maxima (half-cleaner of
      // the two threads' sorted lists + merge) and publishes NP = 16 / S of
      // them, every T-th (T = KT / 8, Q = T NP): its j-th published value
      // has >= T (j+1) of the CTA's maxima >= it.  So with the 16 published
      // values of the cluster sorted, the 8th largest x has >= 8 T = KT
      // group maxima >= x over the row, from disjoint column groups: x is a
      // lower bound on the row's KT-th score.  One DSMEM round (one cluster
      // barrier); both threads of a row compute the same list.
      constexpr int T = KT / 8;
      const int S = (int)gridDim.z;
      float d[KT];  // the sorted top-Q, Q = KT (S = 2) or KT / 2 (S = 4)
      if (S == 2) {
#pragma unroll
        for (int i = 0; i < KT; ++i) d[i] = fmaxf(gm[i], xch[((KT - 1 - i) * 2 + (sh ^ 1)) * 128 + row]);
        bitonic_merge_desc<KT>(d);
      } else {
        float e[KT / 2];
#pragma unroll
        for (int i = 0; i < KT / 2; ++i) e[i] = fmaxf(gm[i], xch[((KT / 2 - 1 - i) * 2 + (sh ^ 1)) * 128 + row]);
        bitonic_merge_desc<KT / 2>(e);
#pragma unroll
        for (int i = 0; i < KT; ++i) d[i] = i < KT / 2 ? e[i] : -INFINITY;
      }
      // pushed, not pulled: thread 0 of the row stores its NP values into
      // slots [g NP, g NP + NP) of every cluster CTA's table (remote stores
      // are fire-and-forget; the barrier's release makes them visible), and
      // after the barrier every thread reads the 16 values locally.  The
      // table sits in the candidate area past the local exchange (KT x 2 x
      // 128 floats): peers write it only before the barrier, pass B
      // overwrites it only after.
      float* pub = xch + KT * 2 * 128;  // [16][128]
      if (sh == 0) {
        const int np = 16 / S, g = (int)blockIdx.z;
        for (int r = 0; r < S; ++r) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < np) st_peer_f32(peer_addr(smem_u32(pub + (g * np + j) * 128 + row), (uint32_t)r), d[T * (j + 1) - 1]);
        }
      }
      SEL_TS(7);
      cluster_sync();
      SEL_TS(8);
      float pv[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) pv[i] = pub[i * 128 + row];
      bitonic_sort_vals<16>(pv);
      tau = pv[7];
      SEL_TS(9);
    } else {
#pragma unroll
      for (int i = 0; i < KT; ++i) tau = fminf(tau, fmaxf(gm[i], xch[((KT - 1 - i) * 2 + (sh ^ 1)) * 128 + row]));
    }
    if constexpr (TF32 && WIDE) {
      // ||q||^2 summed in fp32 (relative error < 2^-17 for d_h <= 128): x 1.001
      // makes sqrt an upper bound; the margin itself has 2x slack (2^-8 vs 2^-9)
      const float d = 0x1p-8f * __fsqrt_ru((qn[row] + qn[128 + row]) * 1.001f) * kmax;
      tau = __fsub_rd(tau, d);
    }
    epi_bar();  // exchange read everywhere before the candidate area is written
    SEL_TS(3);

    // ---- pass B: append every column >= tau to the row's buffer
    // thread 0: slots 0, 1, ... ; thread 1: slots CAP-1, CAP-2, ...  (entry = slot*129 + row)
    const uint32_t cbase = smem_u32(cand) + (uint32_t)row * 8u;
    const uint32_t step = sh == 0 ? (uint32_t)(kCStride * 8) : (uint32_t)(-(kCStride * 8));
    uint32_t caddr = cbase + (sh == 0 ? 0u : (uint32_t)((CAP - 1) * kCStride * 8));
    int cnt = 0;  // this thread's appended columns (may exceed its room: row overflow)
    auto filter32 = [&](const uint32_t (&r)[32], uint32_t col0) {
      if (__any_sync(0xffffffffu, cnt > CAP - 32)) {
        // near the end of this thread's room: bounded stores, exact count
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          if (__uint_as_float(r[jj]) >= tau) {
            if (cnt < CAP) {
              asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(caddr), "r"(r[jj]), "r"(col0 + jj)
                           : "memory");
              caddr += step;
            }
            ++cnt;
          }
        }
        return;
      }
#ifndef MSN_PASSB_CHAIN
      // hit mask, then four independent store chains (columns g*8 .. g*8+7),
      // each starting at its prefix of the mask: no serial dependency across
      // the 32 columns
      uint32_t m = 0;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) m |= (__uint_as_float(r[jj]) >= tau ? 1u : 0u) << jj;
      uint32_t ca[4];
      ca[0] = caddr;
      ca[1] = ca[0] + (uint32_t)__popc(m & 0xffu) * step;
      ca[2] = ca[1] + (uint32_t)__popc(m & 0xff00u) * step;
      ca[3] = ca[2] + (uint32_t)__popc(m & 0xff0000u) * step;
      caddr = ca[3] + (uint32_t)__popc(m >> 24) * step;
      cnt += __popc(m);
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int col = g * 8 + jj;
          asm volatile(
              "{\n.reg .pred p;\n.reg .b32 t;\n"
              "and.b32 t, %1, %5;\n"
              "setp.ne.b32 p, t, 0;\n"
              "@p st.shared.v2.u32 [%0], {%2, %3};\n"
              "@p add.u32 %0, %0, %4;\n}\n"
              : "+r"(ca[g])
              : "r"(m), "r"(r[col]), "r"(col0 + col), "r"(step), "r"(1u << col)
              : "memory");
        }
#else
      const uint32_t a0 = caddr;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj)
        asm volatile(
            "{\n.reg .pred p;\n"
            "setp.ge.f32 p, %1, %2;\n"
            "@p st.shared.v2.u32 [%0], {%3, %4};\n"
            "@p add.u32 %0, %0, %5;\n}\n"
            : "+r"(caddr)
            : "f"(__uint_as_float(r[jj])), "f"(tau), "r"(r[jj]), "r"(col0 + jj), "r"(step)
            : "memory");
      // appended = |caddr - a0| / (129*8)
      const uint32_t moved = sh == 0 ? caddr - a0 : a0 - caddr;
      cnt += (int)(moved / (uint32_t)(kCStride * 8));
#endif
    };
    auto pass_b = [&](int g0, int seg_cols, int col_base) {
      for (int j0 = 64 * sh; j0 < seg_cols; j0 += 128) {
        uint32_t ra[32], rb[32];
        const bool two = j0 + 32 < seg_cols;
        tmem_ld32_async(piece_addr(g0, j0), ra);
        if (two) tmem_ld32_async(piece_addr(g0, j0 + 32), rb);
        tmem_wait_ld(ra);
        filter32(ra, (uint32_t)(col_base + j0));
        if (two) {
          tmem_wait_ld(rb);
          filter32(rb, (uint32_t)(col_base + j0 + 32));
        }
      }
    };
    if (resident) {
      pass_b(0, SEG ? p.seg_cols : p.n_sub, col_seg);
      release_chunks(0, p.n_chunks);
    } else {
      for (int c = 0; c < p.n_chunks; ++c) {
        const int g = p.n_chunks + c;
        wait_chunks(g, 1);
        pass_b(g, p.n_tile, col_seg + c * p.n_tile);
        release_chunks(g, 1);
      }
    }
    cnts[sh * 128 + row] = cnt;
    SEL_TS(4);
    epi_bar();
    SEL_TS(5);

    // ---- write-out: warp ew writes rows 16 ew .. 16 ew + 15, lane = slot;
    // the 16 rows' counts come in with one shared load per lane
    const int r0 = ew * 16;
    const int cn_l = cnts[(lane >> 4) * 128 + r0 + (lane & 15)];
    bool any_ovf = false;
    if constexpr (SEG) {
      // column segments: a few entries per row (the whole row's bound), so
      // each thread copies its own ones (thread 1's after thread 0's)
      const int n0 = cnts[row], n1 = cnts[128 + row];
      const int64_t b = m0 + row;
      const int n = n0 + n1;
      if (b < p.B && n <= CAP) {
        const int64_t grow = b * p.H * 2 + hh;
        uint2* dst = p.vc + (grow * p.SC + seg) * CAP + (sh ? n0 : 0);
        if (sh == 0) p.cn[grow * p.SC + seg] = n;
        const int mine = sh ? n1 : n0;
        for (int i = 0; i < mine; ++i) dst[i] = cand[(sh ? CAP - 1 - i : i) * kCStride + row];
      }
      const int nr = __shfl_sync(0xffffffffu, cn_l, lane & 15) + __shfl_sync(0xffffffffu, cn_l, 16 + (lane & 15));
      any_ovf = __any_sync(0xffffffffu, m0 + r0 + (lane & 15) < p.B && nr > CAP);
    } else {
#pragma unroll 4
    for (int rr = 0; rr < 16; ++rr) {
      const int trow = r0 + rr;
      const int64_t b = m0 + trow;
      const int n0 = __shfl_sync(0xffffffffu, cn_l, rr);
      const int n = n0 + __shfl_sync(0xffffffffu, cn_l, 16 + rr);
      if (b >= p.B) continue;
      if (n > CAP) { any_ovf = true; continue; }
      const int64_t grow = b * p.H * 2 + hh;
      if (lane == 0) p.cn[grow * p.SC + seg] = n;
      uint2* dst = p.vc + (grow * p.SC + seg) * CAP;
#pragma unroll
      for (int hf = 0; hf < CAP / 32; ++hf) {
        const int i = hf * 32 + lane;
        if (i < n) {
          const int slot = i < n0 ? i : CAP - 1 - (i - n0);
          dst[i] = cand[slot * kCStride + trow];
        }
      }
    }
    }
    if (any_ovf) {
      // more than CAP columns passed tau (massive exact ties): exact
      // rescoring of those rows by the warp, their best min(64, n_sub) sub-keys
      for (int rr = 0; rr < 16; ++rr) {
        const int64_t b = m0 + r0 + rr;
        const int n = __shfl_sync(0xffffffffu, cn_l, rr) + __shfl_sync(0xffffffffu, cn_l, 16 + rr);
        if (b >= p.B || n <= CAP) continue;
        const int64_t grow = b * p.H * 2 + hh;
        uint2* dst = p.vc + (grow * p.SC + seg) * CAP;
        const int nn = p.rq.qk_dt == F32
            ? exact_half_topk<float>(p.rq, b * p.H + (hh >> 1), hh & 1, p.H, p.n_sub, dst, col_seg,
                                     SEG ? p.seg_cols : -1)
            : exact_half_topk<__nv_bfloat16>(p.rq, b * p.H + (hh >> 1), hh & 1, p.H, p.n_sub, dst,
                                             col_seg, SEG ? p.seg_cols : -1);
        if (lane == 0) p.cn[grow * p.SC + seg] = nn;
      }
    }
  }
  SEL_TS(6);
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ------------------------------------------------------------- host --------
bool is_tf32(const Shape& s) { return s.qk_dt == F32; }

// Largest N tile (<= 256, multiple of 32, dividing n_sub); TF32 also keeps
// 2 accumulators + the A_lo operand (d_h columns) within 512 TMEM columns.
int kt_of(int k) { return k <= 8 ? 8 : k <= 16 ? 16 : k <= 32 ? 32 : 64; }

size_t smem_for_tile(const Shape& s, int nt) {
  const int bk = is_tf32(s) ? 32 : 64;
  const int parts = is_tf32(s) ? 2 : 1;
  return 1024 + (size_t)(s.d_h / bk) * 16384 + (size_t)kStages * parts * nt * kRowBytes +
         (size_t)cand_cap(kt_of(s.k)) * kCStride * 8 + 256 * 4 + 8 * (1 + 2 * kStages + 5) + 16;
}

// Largest N tile (<= 256, multiple of 32, dividing n_sub) whose stages fit
// shared memory; TF32 also keeps 2 accumulators + the A_lo operand (d_h
// columns) within 512 TMEM columns.
int n_tile_for(const Shape& s) {
  const int cap = is_tf32(s) ? (512 - s.d_h) / 2 : kMaxNTile;
  for (int nt = cap - cap % 32; nt >= 32; nt -= 32)
    if (s.n_sub % nt == 0 && smem_for_tile(s, nt) <= 227 * 1024) return nt;
  return 0;
}

size_t smem_bytes(const Shape& s) { return smem_for_tile(s, n_tile_for(s)); }

// K -> (K_hi, K_lo) for the 3xTF32 B operand, and ||k_i|| per sub-key row
// (fp32 sum of squares, x 1.001 before a rounded-up sqrt: an upper bound),
// one warp per row.
__global__ void split_tf32_kernel(const float* __restrict__ k, float* __restrict__ hi,
                                  float* __restrict__ lo, float* __restrict__ knorm, int64_t rows,
                                  int d) {
  pdl_enter();
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (r >= rows) return;
  float ss = 0.f;
  for (int e = lane; e < d; e += 32) {
    const int64_t i = r * d + e;
    const float x = k[i];
    const float h = tf32_hi(x);
    hi[i] = h;
    lo[i] = x - h;
    ss = fmaf(x, x, ss);
  }
  ss = warp_sum(ss);
  if (lane == 0) knorm[r] = __fsqrt_ru(ss * 1.001f);
}

template <int KT, bool TF32, bool WIDE, bool SEG>
cudaError_t launch_ktws(const Shape& s, const CUtensorMap& mq, const CUtensorMap& mk,
                       const CUtensorMap& mklo, TcParams p, cudaStream_t st) {
  const size_t sm = smem_bytes(s);
  static std::atomic<uint64_t> attr_done{0};
  {
    cudaError_t e = smem_attr_once(attr_done, select_tc_kernel<KT, TF32, WIDE, SEG>, 227 * 1024);
    if (e != cudaSuccess) return e;
  }
  // x = head/half (fastest): concurrently resident CTAs spread over all 2H
  // sub-key codebooks instead of hammering one codebook's lines in L2
  dim3 grid(s.H * 2, (unsigned)((s.B + 127) / 128), (unsigned)(s.n_sub / p.seg_cols));
  if constexpr (SEG) {
    // the S column segments of a row tile form one cluster (the tau exchange)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = grid.z;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool no_pdl = getenv("MSN_NO_PDL") != nullptr;
    cfg.numAttrs = no_pdl ? 1 : 2;
    return cudaLaunchKernelEx(&cfg, select_tc_kernel<KT, TF32, WIDE, SEG>, mq, mk, mklo, p);
  }
  launch_pdl(select_tc_kernel<KT, TF32, WIDE, SEG>, grid, kThreads, sm, st, mq, mk, mklo, p);
  return cudaGetLastError();
}

// How many clusters of S segment CTAs (smem bytes each) the device holds at
// once (cached per device and S; 0 when cluster launches are unavailable).
template <int KT>
int seg_clusters(int S, size_t smem) {
  static std::atomic<int> cache[64][3];  // [device][log2 S - 1], value + 1
  const int d = current_device();
  const int li = S == 2 ? 0 : S == 4 ? 1 : 2;
  if (d >= 0 && d < 64 && cache[d][li].load() > 0) return cache[d][li].load() - 1;
  static std::atomic<uint64_t> attr_done{0};
  int n = 0;
  if (smem_attr_once(attr_done, select_tc_kernel<KT, false, false, true>, 227 * 1024) == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1, 1, S);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = S;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&n, select_tc_kernel<KT, false, false, true>, &cfg) != cudaSuccess) {
      (void)cudaGetLastError();
      n = 0;
    }
  }
  if (d >= 0 && d < 64) cache[d][li].store(n + 1);
  return n;
}
template <int KT, bool TF32, bool WIDE>
cudaError_t launch_ktw(const Shape& s, const CUtensorMap& mq, const CUtensorMap& mk,
                       const CUtensorMap& mklo, TcParams p, cudaStream_t st) {
  if (!TF32 && !WIDE && p.seg_cols < p.n_sub) return launch_ktws<KT, TF32, WIDE, true>(s, mq, mk, mklo, p, st);
  return launch_ktws<KT, TF32, WIDE, false>(s, mq, mk, mklo, p, st);
}
template <int KT, bool TF32>
cudaError_t launch_kt(const Shape& s, const CUtensorMap& mq, const CUtensorMap& mk,
                      const CUtensorMap& mklo, TcParams p, cudaStream_t st) {
  return p.passes == 1 ? launch_ktw<KT, TF32, false>(s, mq, mk, mklo, p, st)
                       : launch_ktw<KT, TF32, true>(s, mq, mk, mklo, p, st);
}

}  // namespace

// Profiling builds only: copies the per-CTA stamps (16 per CTA) to host.
extern "C" int msn_select_ts_dump(unsigned long long* host, int n) {
#ifdef MSN_SELECT_TS
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, g_sel_ts, sizeof(unsigned long long) * (size_t)n * 16) == cudaSuccess ? n : -1;
#else
  (void)host; (void)n;
  return -1;
#endif
}

int select_cap(const Shape& s) { return cand_cap(kt_of(s.k)); }

int select_segments(const Shape& s, bool for_workspace) {
  (void)for_workspace;  // (the layout uses the same S: every call checks its own workspace size)
  if (is_tf32(s) || !select_tc_supported(s) || s.k > 32 || s.n_sub > 1024) return 1;
  const int nt = n_tile_for(s);
  // S segments of >= 256 columns (one full N chunk at least), each resident in TMEM
  auto ok = [&](int S) {
    return s.n_sub % S == 0 && s.n_sub / S >= 256 && (s.n_sub / S) % nt == 0;
  };
  static const int mode = getenv("MSN_SELECT_SPLIT") ? atoi(getenv("MSN_SELECT_SPLIT")) : -1;
  if (mode >= 0) return mode > 1 && ok(mode) ? mode : 1;  // (A/B and tests: force S)
  // the latency regime: as many segments as keep the grid within one wave
  // (and as many clusters of S CTAs as row tiles must be resident together)
  const int64_t ctas = (s.B + 127) / 128 * s.H * 2;
  const int kt = kt_of(s.k);
  for (int S = kMaxSeg; S >= 2; S /= 2) {
    if (!ok(S) || ctas * S > device_sms()) continue;
    const size_t sm = smem_bytes(s);
    const int fit = kt == 8 ? seg_clusters<8>(S, sm) : kt == 16 ? seg_clusters<16>(S, sm) : seg_clusters<32>(S, sm);
    if (ctas <= fit) return S;
  }
  return 1;
}

size_t select_tc_workspace_bytes(const Shape& s) {
  return is_tf32(s) ? 2 * sizeof(float) * (size_t)s.H * 2 * s.n_sub * s.d_h +
                          sizeof(float) * (size_t)s.H * 2 * s.n_sub : 0;
}

bool select_tc_supported(const Shape& s) {
  const bool tf = is_tf32(s);
  if (s.qk_dt != BF16 && s.qk_dt != F32) return false;
  const int bk = tf ? 32 : 64;
  if (s.d_h % bk != 0 || s.d_h > (tf ? 128 : 256)) return false;
  const int nt = n_tile_for(s);
  if (nt == 0 || s.n_sub > 65535) return false;
  if (s.k > 64) return false;
  return smem_bytes(s) <= 227 * 1024;
}

cudaError_t launch_select_tc(const Shape& s, const void* Q, const void* K, const Cands& cd,
                             void* ws, cudaStream_t st, int* launches, void* qhat) {
  if (!select_tc_supported(s) || get_encode() == nullptr || cd.cap != select_cap(s)) return cudaErrorNotSupported;
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
  float* knorm = nullptr;
  if (tf) {
    float* hi = (float*)ws;
    float* lo = hi + kel;
    knorm = lo + kel;
    const int64_t krows = (int64_t)s.H * 2 * s.n_sub;
    launch_pdl(split_tf32_kernel, (unsigned)((krows + 7) / 8), 256, 0, st, (const float*)K, hi, lo, knorm,
               krows, s.d_h);
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
  const int seg_cols = s.n_sub / cd.S;
  const int n_chunks = seg_cols / nt;
  TcParams p{s.B, s.H, s.n_sub, s.d_h, s.k, nt, n_chunks, s.d_h / bk, n_chunks <= 2 ? 1 : 2,
             cd.vc, cd.n, cd.rq, knorm, seg_cols, cd.SC, qhat};
  cudaError_t e;
  if (tf) {
    if (s.k <= 8) e = launch_kt<8, true>(s, mq, mk, mklo, p, st);
    else if (s.k <= 16) e = launch_kt<16, true>(s, mq, mk, mklo, p, st);
    else if (s.k <= 32) e = launch_kt<32, true>(s, mq, mk, mklo, p, st);
    else e = launch_kt<64, true>(s, mq, mk, mklo, p, st);
  } else {
    if (s.k <= 8) e = launch_kt<8, false>(s, mq, mk, mklo, p, st);
    else if (s.k <= 16) e = launch_kt<16, false>(s, mq, mk, mklo, p, st);
    else if (s.k <= 32) e = launch_kt<32, false>(s, mq, mk, mklo, p, st);
    else e = launch_kt<64, false>(s, mq, mk, mklo, p, st);
  }
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace msn
