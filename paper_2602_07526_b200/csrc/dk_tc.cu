// dk_tc.cu -- steps a7 (dq) and a8 (dK) on the tensor cores (bf16 configs):
//   dQ_half[b]  = dS[b,h,half] . K[h,half]      (= ; the query gradient)
//   dK[h,half] += dS[h,half]^T . Q_half      (only the
//   selected sub-keys receive gradient; dS is their aggregated score grad)
// as two dense tcgen05 GEMMs over the same dense score-gradient matrix.
//
// ds_dq_kernel (backward.cu) writes the aggregated score gradients as a
// dense bf16 matrix dSd [B, H*2, n_sub] (zeros for unselected sub-keys; one
// coalesced 2*n_sub-byte row per (query, head, half)).  For one
// (head, half) = hh:  M = n_sub sub-key rows (tiles of 128), N = d_h,
// K = the queries (blocks of 64).  Both operands are loaded by TMA straight
// from their natural layouts -- A = dSd[b, hh, i0:i0+128] and
// B = Q[b, hh, 0:d_h], whose contiguous dimension is M resp. N -- so both
// are "MN-major" UMMA operands (128-byte swizzle atoms of 64 elements x 8
// queries; LBO = stride between 64-element atoms, SBO = 1024 B between
// 8-query groups).  No transposes, no on-the-fly densification.
// Accumulation is fp32 in TMEM in a fixed k-block order; the query range is
// split S ways for parallelism and the S partials are added into dK in split
// order: bitwise deterministic.  Rounding dS to bf16 (2^-9 relative) is
// within the bf16-config tolerance; fp32 configs keep the sort-based path.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace msn {
namespace {
using namespace tc;

constexpr int kThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 TMEM alloc + epilogue (tile (w-2)/4)
constexpr int kCtasPerSm = 1;
constexpr int kDqStages = 4;
constexpr int kDqStagesRec = 4;   // REC: + the staged records (2 x 128 queries x k <= 32 records of 4 B)
constexpr int kDqRecBytes = 2 * 128 * 32 * 4;
// MT 128-row tiles per CTA share every B stage (M = 128 MT): stages of
// (16 MT + 32) KB at d_h = 256, up to ~192 KB of ring
__host__ __device__ constexpr int stages_for(int MT) { return MT == 1 ? 4 : 3; }
__host__ __device__ inline uint32_t tmem_cols(int n) {  // power of 2 >= 32
  uint32_t c = 32;
  while (c < (uint32_t)n) c <<= 1;
  return c;
}
constexpr int kBM = 128;  // sub-key rows per tile
constexpr int kBK = 64;   // queries per k-block
constexpr int kAtom = 64 * 64 * 2;  // one TMA box: 64 elements x 64 queries, bf16 = 8 KB

struct DkParams {
  int64_t B;
  int H, n_sub, d_h;
  int64_t q_per_split;  // queries per split (multiple of kBK)
  float* out;           // partials [S][H*2][n_sub][d_h] (or dK itself when S == 1)
  int accumulate;       // 1: out += acc (S == 1, out = dK); 0: out = acc
  const uint32_t* rec;  // REC: compact records [B][H*2][k] bf16(dS) << 16 | sub-key
  int k;
};

// MN-major, 128-byte-swizzled operand: atoms of 64 (M or N) elements x 8
// K-rows (1 KB); consecutive 64-element atoms kAtom bytes apart (LBO),
// consecutive 8-row groups 1024 B apart (SBO).
__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)(kAtom >> 4) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16, bf16 A/B, fp32 D, A and B MN-major (bits 15, 16).
constexpr uint32_t idesc_bf16_mn(int M, int N) {
  return idesc_bf16(M, N) | (1u << 15) | (1u << 16);
}

// REC: the A tiles (dS^T of the k-block's 64 queries over the CTA's MT x 128
// sub-keys) are built in shared memory from the compact records of
// ds_dq_kernel (p.rec: per (query, head, half) the records {sub-key, dS}
// sorted by sub-key, and per tile the offset of its first record) by the
// epilogue warps, which are idle until the last k-block: each query's row is
// cleared by its 4 threads, then its records in this tile are stored (one
// bf16 each) at their 128-byte-swizzle positions (the layout TMA would
// produce), fence.proxy.async, arrive.  No dense dS matrix in HBM; TMA loads
// only the Q tiles.
template <int MT, bool REC>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    dk_gemm_kernel(const __grid_constant__ CUtensorMap tmap_ds,
                   const __grid_constant__ CUtensorMap tmap_q, const DkParams p) {
  pdl_enter();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  const int nb = p.d_h / 64;                          // B atoms per stage
  constexpr int kStg = stages_for(MT);
  uint8_t* sA = smem_raw + pad;                       // kStg x MT x 2 atoms (16 KB each tile)
  uint8_t* sB = sA + kStg * MT * 2 * kAtom;           // kStg x nb atoms
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kStg * nb * kAtom);
  uint64_t* full = bars;
  uint64_t* empty = full + kStg;
  uint64_t* tdone = empty + kStg;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tdone + 1);
  const uint32_t tcols = tmem_cols(MT * p.d_h);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int i0 = blockIdx.x * kBM * MT;
  const int hh = blockIdx.y;
  const int64_t q0 = (int64_t)blockIdx.z * p.q_per_split;
  int64_t q1 = q0 + p.q_per_split;
  if (q1 > p.B) q1 = p.B;
  const int nkb = q1 > q0 ? (int)((q1 - q0 + kBK - 1) / kBK) : 0;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap_ds);
    prefetch_tmap(&tmap_q);
    for (int s = 0; s < kStg; ++s) {
      mbar_init(&full[s], REC ? 1 + 8 : 1);  // (REC: + one arrive per builder warp)
      mbar_init(&empty[s], 1);
    }
    mbar_init(tdone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)((REC ? 0 : 2 * MT) + nb) * kAtom;
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kStg;
        mbar_wait(&empty[s], ((kb / kStg) & 1) ^ 1);
        mbar_expect_tx(&full[s], bytes);
        const int b0 = (int)(q0 + (int64_t)kb * kBK);
        // queries >= B (ragged last block) are zero-filled by TMA
        if constexpr (!REC) {
#pragma unroll
          for (int t = 0; t < 2 * MT; ++t)
            tma_load_3d(sA + (s * MT * 2 + t) * kAtom, &tmap_ds, &full[s], i0 + 64 * t, hh, b0);
        }
        for (int j = 0; j < nb; ++j)
          tma_load_3d(sB + (s * nb + j) * kAtom, &tmap_q, &full[s], 64 * j, hh, b0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16_mn(kBM, p.d_h);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kStg;
        mbar_wait(&full[s], (kb / kStg) & 1);
        tc_fence_after();
        const uint32_t b0 = smem_u32(sB + s * nb * kAtom);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)  // 16 queries = two 8-row groups = 2 KB
#pragma unroll
          for (int t = 0; t < MT; ++t)          // the MT sub-key tiles share the Q block
            tc_mma(tmem + t * p.d_h, sw128_mn_desc(smem_u32(sA + (s * MT + t) * 2 * kAtom) + kk * 2048),
                   sw128_mn_desc(b0 + kk * 2048), idesc, (kb | kk) != 0);
        tc_commit(&empty[s]);
      }
      tc_commit(tdone);
    }
  } else {
    if constexpr (REC) {
      // ----- A-tile builders (warps 2..9, 256 threads): thread u handles the
      // k-block's query u / 4 and every 4th of its k record slots
      const int u = threadIdx.x - 64;
      const int ql = u >> 2, part = u & 3;
      const int HH = 2 * p.H;
      constexpr int kNr = 4;  // records per thread held one k-block ahead (more: loaded when used)
      constexpr uint32_t kNone = 0xffffffffu;
      const int64_t nlh = p.B * HH;  // lookup-halves (the per-tile offsets follow the records)
      const uint8_t* offs = reinterpret_cast<const uint8_t*>(p.rec + nlh * p.k);
      const int tile = blockIdx.x;   // this CTA's sub-key tile (kBM * MT rows)
      auto lh_of = [&](int kb) -> int64_t { return (q0 + (int64_t)kb * kBK + ql) * HH + hh; };
      // the records of query ql in this tile are [lo, hi) of its sorted list
      // (per-tile offsets written by ds_dq_kernel); the 4 threads of the query
      // take every 4th.  Offsets run two k-blocks ahead, records one.
      // (two byte loads whose values are only used a k-block later: no stall here)
      // (offsets per tile: tile t's records end at o[t])
      auto load_off = [&](int kb, int& lo, int& hi) {
        const bool ok = kb < nkb && q0 + (int64_t)kb * kBK + ql < q1;
        const uint8_t* o = offs + lh_of(ok ? kb : 0) * 32;
        lo = ok && tile ? (int)o[tile - 1] : 0;
        hi = ok ? (int)o[tile] : 0;
      };
      auto load_rec = [&](int kb, int lo, int hi, uint32_t (&x)[kNr]) {
        const uint32_t* r = p.rec + lh_of(kb < nkb ? kb : 0) * p.k;
#pragma unroll
        for (int c = 0; c < kNr; ++c) {
          const int j = lo + part + 4 * c;
          x[c] = j < hi ? r[j] : kNone;
        }
      };
      // offsets and records of k-block kb + kPre into L2 now
      constexpr int kPre = 4;
      auto prefetch_kb = [&](int kb) {
        if (kb < nkb && part < 2 && q0 + (int64_t)kb * kBK + ql < q1) {
          const char* a = part == 0 ? reinterpret_cast<const char*>(offs + lh_of(kb) * 32)
                                    : reinterpret_cast<const char*>(p.rec + lh_of(kb) * p.k);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
        }
      };
      // a stage's A tile must start zeroed: every query row is cleared by its
      // own 4 threads (lanes of one warp) before they write it, so a
      // __syncwarp orders clear and writes (no CTA barrier)
      for (int i = 0; i < kPre && i < nkb; ++i) prefetch_kb(i);
      int lo0, hi0, lo1, hi1;
      load_off(0, lo0, hi0);
      load_off(1, lo1, hi1);
      uint32_t cur[kNr], nr[kNr];
      load_rec(0, lo0, hi0, cur);
      int s = 0;
      uint32_t ph = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        prefetch_kb(kb + kPre);
        int lo2, hi2;
        load_off(kb + 2, lo2, hi2);
        load_rec(kb + 1, lo1, hi1, nr);
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* a = sA + s * MT * 2 * kAtom;
        const uint32_t abase = smem_u32(a) + (uint32_t)ql * 128;
#ifdef MSN_DK_ROWCLEAR
        // this query's row: MT * 2 atoms x 128 B, 4 threads x (MT * 2 * 8 / 4) x 16 B
#pragma unroll
        for (int i = 0; i < MT * 2 * 8 / 4; ++i) {
          const int c16 = part + 4 * i;  // 16-byte chunk of the query's row (8 per atom)
          *reinterpret_cast<uint4*>(a + (c16 >> 3) * kAtom + ql * 128 + (c16 & 7) * 16) = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
#else
        // the stage's A tiles zeroed by the 8 builder warps with contiguous
        // 16-byte stores (no bank conflicts; per-row clears by the row's own
        // 4 lanes hit 8-way conflicts), then a named barrier before the records
#pragma unroll
        for (int i = 0; i < MT * 2 * kAtom / 16 / 256; ++i)
          reinterpret_cast<uint4*>(a)[i * 256 + u] = make_uint4(0, 0, 0, 0);
        asm volatile("bar.sync 2, 256;" ::: "memory");
#endif
        auto put = [&](uint32_t r) {
          const uint32_t il = (r & 0xffffu) - (uint32_t)i0;  // (the sentinel's 0xffff is past every tile)
          if (il < (uint32_t)(kBM * MT)) {
            const uint32_t e = il & 63u;
            const uint32_t off = (il >> 6) * kAtom + ((((e >> 3) ^ (uint32_t)(ql & 7))) << 4) + (e & 7u) * 2;
            asm volatile("st.shared.b16 [%0], %1;" ::"r"(abase + off), "h"((unsigned short)(r >> 16)) : "memory");
          }
        };
#pragma unroll
        for (int c = 0; c < kNr; ++c) put(cur[c]);
        {  // (rare) more than 4 kNr records of this query in the tile
          const uint32_t* r = p.rec + lh_of(kb) * p.k;
          for (int j = lo0 + part + 4 * kNr; j < hi0; j += 4) put(r[j]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
        if (++s == kStg) {
          s = 0;
          ph ^= 1;
        }
#pragma unroll
        for (int c = 0; c < kNr; ++c) cur[c] = nr[c];
        lo0 = lo1;
        hi0 = hi1;
        lo1 = lo2;
        hi1 = hi2;
      }
    }
    if ((warp - 2) / 4 < MT) {
    // ----- epilogue (warps 2..: TMEM lane quarter warp % 4, tile (warp - 2) / 4): row i0 + 128 t + row
    const int q = warp & 3;
    const int t = (warp - 2) / 4;
    const int row = q * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + t * p.d_h;
    float* dst = p.out + ((int64_t)blockIdx.z * (gridDim.y) + hh) * (int64_t)p.n_sub * p.d_h +
                 (int64_t)(i0 + t * kBM + row) * p.d_h;
    if (nkb > 0) {
      mbar_wait(tdone, 0);
      tc_fence_after();
    }
    for (int c0 = 0; c0 < p.d_h; c0 += 32) {
      uint32_t r[32];
      if (nkb > 0) {
        tmem_ld32(lane_base + c0, r);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = 0u;
      }
      float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float4 v = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                               __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
        if (p.accumulate) {
          const float4 o = d4[j];
          v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
        }
        d4[j] = v;
      }
    }
    }  // epilogue warps
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
  }
}

// dQ[b, hh, :] = sum_i dSd[b, hh, i] K[hh, i, :]  (the dq half of step a7,
// dq_row = sum_i dS_row[i] K_row[i]) on the tensor cores: M = 128 queries,
// N = d_h, K = n_sub in blocks of 64.  A = dSd[b0:b0+128, hh, i-block] is
// K-major (contiguous along i), B = K[hh, i-block, :] is MN-major
// (contiguous along e) -- both straight from their natural layouts by TMA.
// Written (=), one fixed k-block order: deterministic.
struct DqParams {
  int64_t B;
  int H, n_sub, d_h;
  float* dQ;  // [B, H*2, d_h] (bf16 when bf16_out)
  int bf16_out = 0;
  const uint32_t* rec = nullptr;  // REC: compact records [B][H*2][k] (bf16(dS) << 16 | sub-key) + block offsets
  int k = 0;
};
// REC: 4 more warps (10..13) build the A tiles from the records
__host__ __device__ constexpr int dq_threads(bool rec) { return rec ? kThreads + 128 : kThreads; }

// Persistent: one CTA per SM walks the (query tile, head.half) tiles in
// hh-major order (the K block of an hh stays hot in L2); two TMEM
// accumulators, so the MMA of tile i+1 runs while the epilogue drains tile i,
// and the TMA ring streams the k-blocks of successive tiles without a break.
//
// REC (n_sub >= 1024: no dense dS in HBM): warps 10..13 build each stage's A
// tile -- dS of the tile's 128 queries over the k-block's 64 sub-keys, K-major
// in the 128-byte swizzle TMA would produce -- from the compact records of
// ds_dq_kernel: thread r walks query r's records (sorted by sub-key; the
// sentinel 0xffffffff past its m) block by block, clears its 128-byte row and
// stores each record of the block as one bf16, fence.proxy.async, arrive.
template <bool REC>
__global__ void __launch_bounds__(dq_threads(REC), 1)
    dq_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                   const __grid_constant__ CUtensorMap tmap_k, const DqParams p, int mtiles) {
  pdl_enter();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  const int nb = p.d_h / 64;                      // B atoms per stage
  constexpr int kABytes = 128 * 128;              // 128 queries x 64 sub-keys bf16
  constexpr int kStg = REC ? kDqStagesRec : kDqStages;
  uint8_t* sA = smem_raw + pad;                   // kStg x 16 KB
  uint8_t* sB = sA + kStg * kABytes;              // kStg x nb atoms
  uint32_t* sRec = reinterpret_cast<uint32_t*>(sB + kStg * nb * kAtom);  // REC: [2][128][32] records
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sRec) + (REC ? kDqRecBytes : 0));
  uint64_t* full = bars;
  uint64_t* empty = full + kStg;
  uint64_t* tfull = empty + kStg;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const uint32_t tcols = tmem_cols(2 * p.d_h);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nkb = p.n_sub / 64;
  const int ntiles = mtiles * 2 * p.H;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_k);
    for (int s = 0; s < kStg; ++s) {
      mbar_init(&full[s], REC ? 1 + 4 : 1);  // (REC: + one arrive per builder warp)
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = (REC ? 0u : (uint32_t)kABytes) + (uint32_t)nb * kAtom;
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int hh = t / mtiles, m0 = (t - hh * mtiles) * 128;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kStg;
          mbar_wait(&empty[s], ((it / kStg) & 1) ^ 1);
          mbar_expect_tx(&full[s], bytes);
          // queries >= B (ragged last tile) are zero-filled by TMA
          if constexpr (!REC) tma_load_3d(sA + s * kABytes, &tmap_a, &full[s], kb * 64, hh, m0);
          for (int j = 0; j < nb; ++j)
            tma_load_3d(sB + (s * nb + j) * kAtom, &tmap_k, &full[s], 64 * j, kb * 64, hh);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(128, p.d_h) | (1u << 16);  // B MN-major
      int it = 0, lt = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
        const int buf = lt & 1;
        mbar_wait(&tempty[buf], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * p.d_h;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kStg;
          mbar_wait(&full[s], (it / kStg) & 1);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * kABytes);
          const uint32_t b0 = smem_u32(sB + s * nb * kAtom);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // 16 sub-keys: +32 B in the A row, +2 KB in B
            tc_mma(d, sw128_desc(a0 + kk * 32), sw128_mn_desc(b0 + kk * 2048), idesc, (kb | kk) != 0);
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[buf]);
      }
    }
  } else if (REC && warp >= 10) {
    // ----- A-tile builders (warps 10..13): thread r = query row r of the tile.
    // The tile's records (k <= 32 per query) are staged in shared memory by
    // cp.async one tile ahead (each thread copies and reads only its own
    // query's, so its cp.async.wait_group is the only ordering needed); per
    // k-block the four warps zero the stage's A tile (contiguous 16-byte
    // stores: no bank conflicts), meet at a named barrier, and each thread
    // stores its query's records of the block.
    const int r = (warp - 10) * 32 + lane;
    const int bt = threadIdx.x - 10 * 32;  // 0..127
    const int HH = 2 * p.H;
    auto stage_recs = [&](int t, int buf) {
      const int hh = t / mtiles, m0 = (t - hh * mtiles) * 128;
      const int64_t b = (int64_t)m0 + r;
      if (t < ntiles && b < p.B) {
        const char* src = reinterpret_cast<const char*>(p.rec + (b * HH + hh) * p.k);
        const uint32_t dst = smem_u32(sRec + (buf * 128 + r) * 32);
        for (int c = 0; c < p.k / 4; ++c)  // (k % 4 == 0: 16 B = four records)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + c * 16), "l"(src + c * 16)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int it = 0, lt = 0;
    stage_recs(blockIdx.x, 0);
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const int hh = t / mtiles, m0 = (t - hh * mtiles) * 128;
      const bool valid = (int64_t)m0 + r < p.B;
      stage_recs(t + gridDim.x, (lt + 1) & 1);  // the next tile's records
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // this tile's have landed
      const uint32_t* my = sRec + ((lt & 1) * 128 + r) * 32;
      int j = 0;
      uint32_t x0 = valid ? my[0] : 0xffffffffu;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % kStg;
        mbar_wait(&empty[s], ((it / kStg) & 1) ^ 1);
        uint4* az = reinterpret_cast<uint4*>(sA + s * kABytes);
#pragma unroll
        for (int c = 0; c < kABytes / 16 / 128; ++c) az[c * 128 + bt] = make_uint4(0, 0, 0, 0);
        asm volatile("bar.sync 2, 128;" ::: "memory");  // the 4 builder warps: tile zeroed
        const uint32_t abase = smem_u32(sA + s * kABytes + r * 128);
        while (((x0 & 0xffffu) >> 6) == (uint32_t)kb) {  // (the sentinel's block 1023 is never reached)
          const uint32_t e = x0 & 63u;
          const uint32_t off = ((((e >> 3) ^ (uint32_t)(r & 7))) << 4) + (e & 7u) * 2;
          asm volatile("st.shared.b16 [%0], %1;" ::"r"(abase + off), "h"((unsigned short)(x0 >> 16)) : "memory");
          ++j;
          x0 = j < p.k ? my[j] : 0xffffffffu;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else {
    // epilogue: warps 2..9, TMEM lane quarter warp % 4, column half (warp - 2) / 4
    const int q = warp & 3;
    const int ch = (warp - 2) / 4;
    const int cw = p.d_h / 2;
    const int row = q * 32 + lane;
    int lt = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const int hh = t / mtiles, m0 = (t - hh * mtiles) * 128;
      const int buf = lt & 1;
      mbar_wait(&tfull[buf], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + buf * p.d_h;
      const int64_t b = (int64_t)m0 + row;
      const int64_t qoff = (b * (2 * p.H) + hh) * (int64_t)p.d_h;
      for (int c0 = ch * cw; c0 < (ch + 1) * cw; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(lane_base + c0, r);
        if (b < p.B) {
          if (p.bf16_out) {  // MSN_FLAG_DQ_QK_DTYPE: one RNE rounding, 16 B stores
            uint4* d8 = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.dQ) + qoff + c0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint32_t w[4];
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(r[8 * j + 2 * t]),
                                                               __uint_as_float(r[8 * j + 2 * t + 1]));
                w[t] = *reinterpret_cast<const uint32_t*>(&v);
              }
              d8[j] = make_uint4(w[0], w[1], w[2], w[3]);
            }
          } else {
            float4* d4 = reinterpret_cast<float4*>(p.dQ + qoff + c0);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              d4[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                  __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
  }
}

// Tiles per CTA.  Measured on the B200 (bench.py, MSN_DQ_MT / MSN_DK_MT
// override for A/B runs): dQ gains nothing from MT = 2 (C2 +1.7 us, C4 0);
// dK gains on long codebooks (C4, n_sub 2048: -21 us) and loses on short ones
// (C2, n_sub 512: +7.5 us, too few k-blocks per split).
int env_int(const char* n, int d) { const char* v = getenv(n); return v ? atoi(v) : d; }
int num_sms_dk() { return device_sms(); }
int dq_mt(const Shape&) { return 1; }
int dk_mt(const Shape& s) {
  static const int f = env_int("MSN_DK_MT", 0);
  const bool want = f == 0 ? s.n_sub >= 1024 : f >= 2;
  return (want && s.n_sub % (2 * kBM) == 0) ? 2 : 1;
}

size_t dq_smem_bytes(const Shape& s, int MT) {
  (void)MT;
  return 1024 + (size_t)kDqStages * (128 * 128 + (s.d_h / 64) * kAtom) + 8 * (2 * kDqStages + 4) + 16;
}
size_t dq_rec_smem_bytes(const Shape& s) {
  return 1024 + (size_t)kDqStagesRec * (128 * 128 + (s.d_h / 64) * kAtom) + kDqRecBytes +
         8 * (2 * kDqStagesRec + 4) + 16;
}

// dK += sum_s part[s] (fixed split order)
__global__ void dk_reduce_kernel(const float4* __restrict__ part, float4* __restrict__ dK,
                                 int64_t n4, int S) {
  pdl_enter();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  float4 acc = part[i];
  for (int s = 1; s < S; ++s) {
    const float4 v = part[(int64_t)s * n4 + i];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  float4 o = dK[i];
  o.x += acc.x; o.y += acc.y; o.z += acc.z; o.w += acc.w;
  dK[i] = o;
}

int splits_for(const Shape& s) {
  const int tiles = (s.n_sub / (kBM * dk_mt(s))) * s.H * 2;
  const int64_t kblocks = (s.B + kBK - 1) / kBK;
  int S = 1;
  while (tiles * S * 2 <= 148 * kCtasPerSm && kblocks / (S * 2) >= 4) S *= 2;
  return S;
}

size_t dk_smem_bytes(const Shape& s, int MT) {
  const int st = stages_for(MT);
  return 1024 + (size_t)st * (2 * MT + s.d_h / 64) * kAtom + 8 * (2 * st + 1) + 16;
}

bool dq_tc_wanted_(const Shape& s);
// the dense bf16 dS matrix (tensor-core dQ wanted), else the compact records
// (k slots of 8 B) and their per-tile offsets (32 B) per (query, head, half)
bool dk_compact_(const Shape& s);
size_t dense_ds_bytes(const Shape& s) {
  if (dk_compact_(s)) return ((size_t)s.B * s.H * 2 * (s.k * 4 + 32) + 255) & ~(size_t)255;
  return ((size_t)s.B * s.H * 2 * s.n_sub * 2 + 255) & ~(size_t)255;
}

}  // namespace

int dk_tile_rows(const Shape& s) { return kBM * dk_mt(s); }

bool dk_tc_supported(const Shape& s) {
  // The tensor-core path rounds dS to bf16 (2^-9 relative): only where the
  // bf16 tolerance applies, i.e. bf16 values (north_star: "1e-4 relative for
  // fp32 and 2e-2 relative for bf16 values"); bf16 q/K with fp32 values keep
  // dS in fp32 (grouped reducers, SIMT dQ) and meet 1e-4.
  return s.qk_dt == BF16 && s.v_dt == BF16 && s.n_sub <= 2048 && s.n_sub % kBM == 0 && s.d_h % 64 == 0 &&
         s.d_h >= 64 && s.d_h <= 256 && s.k <= 64 && dk_smem_bytes(s, dk_mt(s)) <= 227 * 1024 &&
         dq_smem_bytes(s, dq_mt(s)) <= 227 * 1024 && get_encode() != nullptr;
}

size_t dk_tc_workspace_bytes(const Shape& s) {
  if (!dk_tc_supported(s)) return 0;
  const int S = splits_for(s);
  const size_t part = S > 1 ? (size_t)S * s.H * 2 * s.n_sub * s.d_h * 4 : 0;
  return dense_ds_bytes(s) + part;
}

namespace {
bool dq_tc_wanted_(const Shape& s) {
  // MSN_DQ_TC=0/1 forces the choice (A/B measurements only)
  static const int f = env_int("MSN_DQ_TC", -1);
  return f >= 0 ? f != 0 : s.n_sub < 1024;
}
// the dK operand from compact records (no dense dS) whenever dQ is not on the
// tensor cores; MSN_DK_DENSE=1 keeps the dense matrix (A/B measurements only)
bool dk_compact_(const Shape& s) {
  static const int f = env_int("MSN_DK_DENSE", 0);
  return !dq_tc_wanted_(s) && !f;
}
}  // namespace
bool dq_tc_wanted(const Shape& s) { return dq_tc_wanted_(s); }
// compact records: dQ on the tensor cores with the A tiles built from them
// (MSN_DQ_REC=1 turns it on, else the SIMT dQ of ds_dq_kernel; A/B measurements only)
bool dq_rec_wanted(const Shape& s) {
  // default off: measured on C4, dq_gemm with built A tiles takes 316 us against
  // the ~240 us the SIMT dQ adds to ds_dq (builder-bound: 43 % tensor-pipe activity)
  static const int f = env_int("MSN_DQ_REC", 0);
  // (the records staged in shared memory: k <= 32, pairs of 16 bytes)
  return f != 0 && s.k <= 32 && s.k % 4 == 0 && dq_rec_smem_bytes(s) <= 227 * 1024;
}
bool dk_compact(const Shape& s) { return dk_compact_(s); }

cudaError_t launch_dk_tc(const Shape& s, const void* Q, const void* Kp, float* dQ, float* dK,
                         void* ws, cudaStream_t st, int* launches, bool with_dq) {
  if (!dk_tc_supported(s)) return cudaErrorNotSupported;
  const uint16_t* dSd = (const uint16_t*)ws;
  float* part = (float*)((char*)ws + dense_ds_bytes(s));
  const int HH = s.H * 2;
  CUtensorMap mds, mq;
  {
    // dSd [B, HH, n_sub]: dims (n_sub, HH, B), box (64, 1, 64)
    cuuint64_t dims[3] = {(cuuint64_t)s.n_sub, (cuuint64_t)HH, (cuuint64_t)s.B};
    cuuint64_t strides[2] = {(cuuint64_t)s.n_sub * 2, (cuuint64_t)HH * s.n_sub * 2};
    cuuint32_t box[3] = {64, 1, (cuuint32_t)kBK};
    cuuint32_t es[3] = {1, 1, 1};
    if (get_encode()(&mds, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)dSd, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    // Q [B, HH, d_h]: dims (d_h, HH, B), box (64, 1, 64)
    cuuint64_t dims[3] = {(cuuint64_t)s.d_h, (cuuint64_t)HH, (cuuint64_t)s.B};
    cuuint64_t strides[2] = {(cuuint64_t)s.d_h * 2, (cuuint64_t)HH * s.d_h * 2};
    cuuint32_t box[3] = {64, 1, (cuuint32_t)kBK};
    cuuint32_t es[3] = {1, 1, 1};
    if (get_encode()(&mq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(Q), dims, strides,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  // dQ = dS . K per (head, half) on the tensor cores: from the dense dS
  // matrix by TMA, or (compact records) with the A tiles built in shared memory
  if (with_dq && dk_compact(s)) {
    CUtensorMap mk;
    cuuint64_t kdims[3] = {(cuuint64_t)s.d_h, (cuuint64_t)s.n_sub, (cuuint64_t)HH};
    cuuint64_t kstrides[2] = {(cuuint64_t)s.d_h * 2, (cuuint64_t)s.n_sub * s.d_h * 2};
    cuuint32_t kbox[3] = {64, 64, 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (get_encode()(&mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(Kp), kdims,
                     kstrides, kbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    DqParams qp{s.B, s.H, s.n_sub, s.d_h, dQ, s.dq_bf16 ? 1 : 0};
    qp.rec = reinterpret_cast<const uint32_t*>(ws);
    qp.k = s.k;
    static std::atomic<uint64_t> qattr{0};
    cudaError_t e0 = smem_attr_once(qattr, dq_gemm_kernel<true>, 227 * 1024);
    if (e0 != cudaSuccess) return e0;
    const int mtiles = (int)((s.B + 127) / 128);
    const int ntiles = mtiles * HH;
    launch_pdl(dq_gemm_kernel<true>, (unsigned)std::min(ntiles, num_sms_dk()), dq_threads(true),
               dq_rec_smem_bytes(s), st, mk, mk, qp, mtiles);
    cudaError_t e1 = cudaGetLastError();
    if (e1 != cudaSuccess) return e1;
    ++*launches;
  } else if (with_dq) {
    CUtensorMap ma, mk;
    // dSd [B, HH, n_sub] as the K-major A operand: dims (n_sub, HH, B), box (64, 1, 128)
    cuuint64_t dims[3] = {(cuuint64_t)s.n_sub, (cuuint64_t)HH, (cuuint64_t)s.B};
    cuuint64_t strides[2] = {(cuuint64_t)s.n_sub * 2, (cuuint64_t)HH * s.n_sub * 2};
    cuuint32_t box[3] = {64, 1, 128};
    cuuint32_t es[3] = {1, 1, 1};
    if (get_encode()(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)dSd, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    // K [HH, n_sub, d_h] as the MN-major B operand: dims (d_h, n_sub, HH), box (64, 64, 1)
    cuuint64_t kdims[3] = {(cuuint64_t)s.d_h, (cuuint64_t)s.n_sub, (cuuint64_t)HH};
    cuuint64_t kstrides[2] = {(cuuint64_t)s.d_h * 2, (cuuint64_t)s.n_sub * s.d_h * 2};
    cuuint32_t kbox[3] = {64, 64, 1};
    if (get_encode()(&mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(Kp), kdims,
                     kstrides, kbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    DqParams qp{s.B, s.H, s.n_sub, s.d_h, dQ, s.dq_bf16 ? 1 : 0};
    static std::atomic<uint64_t> qattr{0};
    cudaError_t e0 = smem_attr_once(qattr, dq_gemm_kernel<false>, 227 * 1024);
    if (e0 != cudaSuccess) return e0;
    const int mtiles = (int)((s.B + 127) / 128);
    const int ntiles = mtiles * HH;
    launch_pdl(dq_gemm_kernel<false>, (unsigned)std::min(ntiles, num_sms_dk()), dq_threads(false),
               dq_smem_bytes(s, 1), st, ma, mk, qp, mtiles);
    cudaError_t e1 = cudaGetLastError();
    if (e1 != cudaSuccess) return e1;
    ++*launches;
  }
  const int S = splits_for(s);
  const int64_t kblocks = (s.B + kBK - 1) / kBK;
  const int64_t qps = ((kblocks + S - 1) / S) * kBK;
  DkParams p{s.B, s.H, s.n_sub, s.d_h, qps, S > 1 ? part : dK, S > 1 ? 0 : 1,
             reinterpret_cast<const uint32_t*>(ws), s.k};
  const int mtk = dk_mt(s);
  const bool rec = dk_compact(s);  // ds_dq_kernel wrote compact records (dQ done there)
  auto dkk = rec ? (mtk == 2 ? dk_gemm_kernel<2, true> : dk_gemm_kernel<1, true>)
                 : (mtk == 2 ? dk_gemm_kernel<2, false> : dk_gemm_kernel<1, false>);
  static std::atomic<uint64_t> attr[4];
  cudaError_t e = smem_attr_once(attr[(mtk - 1) * 2 + (rec ? 1 : 0)], dkk, 227 * 1024);
  if (e != cudaSuccess) return e;
  dim3 grid(s.n_sub / (kBM * mtk), HH, S);
  launch_pdl(dkk, grid, kThreads, dk_smem_bytes(s, mtk), st, mds, mq, p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ++*launches;
  if (S > 1) {
    const int64_t n4 = (int64_t)HH * s.n_sub * s.d_h / 4;
    launch_pdl(dk_reduce_kernel, (unsigned)((n4 + 255) / 256), 256, 0, st, (const float4*)part, (float4*)dK,
                                                                   n4, S);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ++*launches;
  }
  return cudaSuccess;
}

}  // namespace msn
