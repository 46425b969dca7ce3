// dk_tc.cu -- step a8's sub-key gradient on the tensor cores (bf16 configs):
//   dK[h,half] += dS[h,half]^T . Q_half      (only the
//   selected sub-keys receive gradient; dS is their aggregated score grad)
// as dense tcgen05 GEMM tiles whose sparse operand is densified on the fly.
//
// For one (head, half): M = n_sub sub-key rows (tiles of 128), N = d_h,
// K = the queries (blocks of 64).  The A tile dS^T[i0:i0+128, b0:b0+64] is
// built in shared memory (zeroed, then one bf16 write per distinct
// (query, sub-key) record of ds_dq_kernel, in the 128-byte-swizzled K-major
// layout the MMA descriptor expects); the B tile is Q^T[e, b0:b0+64] (a
// transposed copy of the query halves, so that the reduction dimension b is
// contiguous) loaded by TMA.  Accumulation is fp32 in TMEM in a fixed
// k-block order; the query range is split S ways for parallelism and the S
// partials are added into dK in split order: bitwise deterministic.
// Rounding dS to bf16 (2^-9 relative) is within the bf16-config tolerance;
// fp32 configs keep the sort-based path (backward.cu).
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace msn {
namespace {
using namespace tc;

constexpr int kThreads = 256;
constexpr int kStages = 3;
constexpr int kBM = 128;  // sub-key rows per tile
constexpr int kBK = 64;   // queries per k-block (one 128-byte bf16 row)

struct DkParams {
  int64_t B;
  int H, n_sub, d_h, k;
  int64_t q_per_split;  // queries per split (multiple of kBK)
  const uint32_t* rkeys;
  const float* dsS;
  float* out;           // partials [S][H*2][n_sub][d_h] (or dK itself when S == 1)
  int accumulate;       // 1: out += acc (S == 1, out = dK); 0: out = acc
};

__global__ void __launch_bounds__(kThreads, 1)
    dk_gemm_kernel(const __grid_constant__ CUtensorMap tmap_qt, const DkParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* sA = smem_raw + pad;                       // kStages x 16 KB
  uint8_t* sB = sA + kStages * kBM * 128;             // kStages x d_h x 128 B
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kStages * p.d_h * 128);
  uint64_t* full_b = bars;
  uint64_t* full_a = full_b + kStages;
  uint64_t* empty = full_a + kStages;
  uint64_t* tdone = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tdone + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int i0 = blockIdx.x * kBM;
  const int hh = blockIdx.y;
  const int h = hh >> 1, half = hh & 1;
  const int64_t q0 = (int64_t)blockIdx.z * p.q_per_split;
  int64_t q1 = q0 + p.q_per_split;
  if (q1 > p.B) q1 = p.B;
  const int nkb = q1 > q0 ? (int)((q1 - q0 + kBK - 1) / kBK) : 0;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap_qt);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_b[s], 1);
      mbar_init(&full_a[s], 4);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tdone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kStages;
        mbar_wait(&empty[s], ((kb / kStages) & 1) ^ 1);
        mbar_expect_tx(&full_b[s], p.d_h * 128);
        tma_load_2d(sB + s * p.d_h * 128, &tmap_qt, &full_b[s], (int)(q0 + kb * kBK), hh * p.d_h);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(kBM, p.d_h);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kStages;
        mbar_wait(&full_a[s], (kb / kStages) & 1);
        mbar_wait(&full_b[s], (kb / kStages) & 1);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + s * kBM * 128);
        const uint32_t b0 = smem_u32(sB + s * p.d_h * 128);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)
          tc_mma(tmem, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32), idesc, (kb | kk) != 0);
        tc_commit(&empty[s]);
      }
      tc_commit(tdone);
    }
  } else if (warp >= 4) {
    // ----- A builders: dS^T tile for queries [b0, b0+64), rows [i0, i0+128)
    const int t = threadIdx.x - 128;  // 0..127
    const uint32_t base_key = (uint32_t)hh * p.n_sub + i0;
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kStages;
      mbar_wait(&empty[s], ((kb / kStages) & 1) ^ 1);
      uint8_t* A = sA + s * kBM * 128;
      // zero: 16 KB, 128 B per thread
      uint4* z = reinterpret_cast<uint4*>(A) + t * 8;
#pragma unroll
      for (int i = 0; i < 8; ++i) z[i] = make_uint4(0, 0, 0, 0);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int qc = t & 63;  // query column of this thread
      const int64_t b = q0 + kb * kBK + qc;
      if (b < q1) {
        // this thread's records: t' = (t >> 6), (t >> 6) + 2, ... < k  (all loads first)
        constexpr int MAXR = 32;  // k <= 64
        uint32_t key[MAXR];
        float val[MAXR];
        const int64_t rec0 = ((b * p.H + h) * p.k) * 2 + half;
#pragma unroll
        for (int u = 0; u < MAXR; ++u) {
          const int tt = (t >> 6) + 2 * u;
          key[u] = tt < p.k ? __ldg(p.rkeys + rec0 + 2 * tt) : 0xffffffffu;
          val[u] = tt < p.k ? __ldg(p.dsS + rec0 + 2 * tt) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < MAXR; ++u) {
          const uint32_t r = key[u] - base_key;  // row within the tile (wraps if below)
          if (r < (uint32_t)kBM) {
            // SW128 K-major: row r = 128 B, 16-B chunk c XOR (r % 8)
            const int c = qc >> 3;
            uint16_t* dst = reinterpret_cast<uint16_t*>(A + r * 128 + ((c ^ (r & 7)) << 4)) + (qc & 7);
            *dst = __bfloat16_as_ushort(__float2bfloat16_rn(val[u]));
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (lane == 0) mbar_arrive(&full_a[s]);
    }
    // ----- epilogue: row i0 + t of the accumulator -> partial / dK
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    float* dst = p.out + ((int64_t)blockIdx.z * (gridDim.y) + hh) * (int64_t)p.n_sub * p.d_h +
                 (int64_t)(i0 + row) * p.d_h;
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
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

// Q [B, H, 2, d_h] -> QT [H*2, d_h, Bp] (the query index contiguous)
__global__ void __launch_bounds__(256) transpose_q_kernel(const __nv_bfloat16* __restrict__ Q,
                                                          __nv_bfloat16* __restrict__ QT, int64_t B,
                                                          int64_t Bp, int H, int d_h) {
  __shared__ uint16_t tile[64][65];
  const int hh = blockIdx.z;
  const int64_t b0 = (int64_t)blockIdx.x * 64;
  const int e0 = blockIdx.y * 64;
  const uint16_t* q = reinterpret_cast<const uint16_t*>(Q);
  uint16_t* qt = reinterpret_cast<uint16_t*>(QT);
  for (int i = threadIdx.x; i < 64 * 64; i += 256) {
    const int bb = i / 64, ee = i % 64;
    const int64_t b = b0 + bb;
    tile[bb][ee] = b < B ? q[((b * H) * 2 + hh) * (int64_t)d_h + e0 + ee] : (uint16_t)0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64 * 64; i += 256) {
    const int ee = i / 64, bb = i % 64;
    const int64_t b = b0 + bb;
    if (b < Bp) qt[((int64_t)hh * d_h + e0 + ee) * Bp + b] = tile[bb][ee];
  }
}

// dK += sum_s part[s] (fixed split order)
__global__ void dk_reduce_kernel(const float4* __restrict__ part, float4* __restrict__ dK,
                                 int64_t n4, int S) {
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

int64_t padded_batch(int64_t B) { return (B + 63) / 64 * 64; }

int splits_for(const Shape& s) {
  const int tiles = (s.n_sub / kBM) * s.H * 2;
  int S = 1;
  while (tiles * S < 148 && (padded_batch(s.B) / kBK) / (S * 2) >= 4) S *= 2;
  return S;
}

size_t dk_smem_bytes(const Shape& s) {
  return 1024 + (size_t)kStages * kBM * 128 + (size_t)kStages * s.d_h * 128 + 8 * (3 * kStages + 1) + 16;
}

}  // namespace

bool dk_tc_supported(const Shape& s) {
  // dense work = 2 n_sub d_h per (query, half) vs ~2 k d_h for the sparse path:
  // worth it while n_sub is small (C2: 512); C4 (2048) keeps the sort path.
  return s.qk_dt == BF16 && s.n_sub <= 1024 && s.d_h % 64 == 0 && s.d_h >= 64 && s.d_h <= 256 && s.n_sub % kBM == 0 &&
         s.k <= 64 && dk_smem_bytes(s) <= 227 * 1024 && get_encode() != nullptr;
}

size_t dk_tc_workspace_bytes(const Shape& s) {
  if (!dk_tc_supported(s)) return 0;
  const size_t qt = (size_t)s.H * 2 * s.d_h * padded_batch(s.B) * 2;
  const int S = splits_for(s);
  const size_t part = S > 1 ? (size_t)S * s.H * 2 * s.n_sub * s.d_h * 4 : 0;
  return ((qt + 255) & ~(size_t)255) + part;
}

cudaError_t launch_dk_tc(const Shape& s, const void* Q, const uint32_t* rkeys, const float* dsS,
                         float* dK, void* ws, cudaStream_t st, int* launches) {
  if (!dk_tc_supported(s)) return cudaErrorNotSupported;
  const int64_t Bp = padded_batch(s.B);
  __nv_bfloat16* QT = (__nv_bfloat16*)ws;
  const size_t qt_bytes = (((size_t)s.H * 2 * s.d_h * Bp * 2) + 255) & ~(size_t)255;
  float* part = (float*)((char*)ws + qt_bytes);
  dim3 tg((unsigned)(Bp / 64), s.d_h / 64, s.H * 2);
  transpose_q_kernel<<<tg, 256, 0, st>>>((const __nv_bfloat16*)Q, QT, s.B, Bp, s.H, s.d_h);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ++*launches;
  CUtensorMap m;
  {
    cuuint64_t dims[2] = {(cuuint64_t)Bp, (cuuint64_t)s.H * 2 * s.d_h};
    cuuint64_t strides[1] = {(cuuint64_t)Bp * 2};
    cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)s.d_h};
    cuuint32_t es[2] = {1, 1};
    if (get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, QT, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int S = splits_for(s);
  const int64_t qps = ((Bp / kBK + S - 1) / S) * kBK;
  DkParams p{s.B, s.H, s.n_sub, s.d_h, s.k, qps, rkeys, dsS, S > 1 ? part : dK, S > 1 ? 0 : 1};
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(dk_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(s.n_sub / kBM, s.H * 2, S);
  dk_gemm_kernel<<<grid, kThreads, dk_smem_bytes(s), st>>>(m, p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ++*launches;
  if (S > 1) {
    const int64_t n4 = (int64_t)s.H * 2 * s.n_sub * s.d_h / 4;
    dk_reduce_kernel<<<(unsigned)((n4 + 255) / 256), 256, 0, st>>>((const float4*)part, (float4*)dK,
                                                                   n4, S);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ++*launches;
  }
  return cudaSuccess;
}

}  // namespace msn
