// prologue.cu -- the query / key prologue of the lookup:
//   LayerNorm of query and sub-key vectors before scoring (
//   reading R23: no affine, eps = 1e-5) and its backward;
//   key over-parameterisation K~ = Theta K per (head, half)
//   and its gradients dTheta = sum_i dk~_i k_i^T, dk_i = Theta^T dk~_i
//   (PAPER.md:296-302).
// LN: one warp per row (the row lives in the lane registers), fp32 math,
// output rounded once to the storage type.  The Theta products (three per
// step: K~ = K^ Theta^T, dK^ = dK~ Theta, dTheta += dK~^T K^) run on the
// tensor cores as 3xTF32 tcgen05 GEMMs (pgemm_kernel: hi.hi + hi.lo + lo.hi,
// fp32-accurate for the fp32 configs' 1e-4), batched over the 2H codebooks.
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

#include <type_traits>

namespace msn {
namespace {

constexpr float kLnEps = 1e-5f;

template <typename T>
__device__ __forceinline__ float ld_f(const T* p) { return elem<T>::to_f(*p); }
template <typename T>
__device__ __forceinline__ void st_f(T* p, float v);
template <>
__device__ __forceinline__ void st_f<float>(float* p, float v) { *p = v; }
template <>
__device__ __forceinline__ void st_f<__nv_bfloat16>(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

template <typename T, int EPL>
__global__ void __launch_bounds__(256) ln_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                 int64_t rows) {
  pdl_enter();
  const int lane = threadIdx.x % 32;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (r >= rows) return;
  constexpr int D = 32 * EPL;
  float v[EPL];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    v[i] = ld_f(x + r * D + i * 32 + lane);
    s += v[i];
  }
  const float mu = warp_sum(s) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < EPL; ++i) q += (v[i] - mu) * (v[i] - mu);
  const float rs = rsqrtf(warp_sum(q) / D + kLnEps);
#pragma unroll
  for (int i = 0; i < EPL; ++i) st_f(y + r * D + i * 32 + lane, (v[i] - mu) * rs);
}

// dx = r (dy - mean(dy) - x_hat mean(dy x_hat)),  x_hat, r recomputed from x
template <typename T, int EPL>
__global__ void __launch_bounds__(256) ln_backward_kernel(const T* __restrict__ x,
                                                          const float* __restrict__ dy,
                                                          float* __restrict__ dx, int64_t rows) {
  pdl_enter();
  const int lane = threadIdx.x % 32;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (r >= rows) return;
  constexpr int D = 32 * EPL;
  float v[EPL], g[EPL];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    v[i] = ld_f(x + r * D + i * 32 + lane);
    g[i] = dy[r * D + i * 32 + lane];
    s += v[i];
  }
  const float mu = warp_sum(s) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < EPL; ++i) q += (v[i] - mu) * (v[i] - mu);
  const float rs = rsqrtf(warp_sum(q) / D + kLnEps);
  float sg = 0.f, sgx = 0.f;
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    v[i] = (v[i] - mu) * rs;  // x_hat
    sg += g[i];
    sgx += g[i] * v[i];
  }
  const float mg = warp_sum(sg) / D, mgx = warp_sum(sgx) / D;
#pragma unroll
  for (int i = 0; i < EPL; ++i) dx[r * D + i * 32 + lane] = rs * (g[i] - mg - v[i] * mgx);
}

// ---- 3xTF32 tcgen05 GEMM for the Theta products ---------------------------
// C[m][n] (=, or += with accumulate) = sum_k A(m, k) B(n, k) per batch z, with
// A(m, k) = A[z a_bs + m a_rs + k a_cs] and B(n, k) = B[z b_bs + k b_rs + n b_cs]
// (any layout: the operands are staged by the threads, which walk the source's
// contiguous dimension), C[z c_bs + m c_rs + n].  One CTA per (128-row tile,
// 64-column tile, batch), the tile in one TMEM accumulator; K in blocks of 32: every
// element is split x = hi + lo (hi = the TF32 value, lo exact in fp32) into
// two 128-byte-swizzled K-major tiles of each operand, and one elected thread
// issues D += Ahi.Bhi + Ahi.Blo + Alo.Bhi per 8-element step (the lo.lo term
// is below fp32 rounding).  Two stages: the threads stage k-block kb + 1
// while the tensor cores run kb (tcgen05.commit frees a stage).
constexpr int kPgThreads = 256;
constexpr int kPgM = 128;
constexpr int kPgN = 64;  // columns per CTA (C tiles of 128 x 64: 4x the CTAs of whole rows)
struct PgArgs {
  int M, N, K;
  const void* A;
  int64_t a_rs, a_cs, a_bs;
  const void* B;
  int64_t b_rs, b_cs, b_bs;
  void* C;
  int64_t c_rs, c_bs;
  int accumulate;
};
__device__ __forceinline__ uint32_t sw128_off(int r, int kk) {  // fp32 element (row r, k kk < 32)
  return (uint32_t)r * 128u + ((((uint32_t)kk >> 2) ^ ((uint32_t)r & 7u)) << 4) + ((uint32_t)kk & 3u) * 4u;
}
template <typename TA, typename TB, typename TC>
__global__ void __launch_bounds__(kPgThreads, 1) pgemm_kernel(PgArgs g) {
  using namespace tc;
  pdl_enter();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* base = smem_raw + pad;
  const int n0 = blockIdx.y * kPgN;
  const int NT = g.N - n0 < kPgN ? g.N - n0 : kPgN;  // this CTA's columns (multiple of 16)
  const int NP = kPgN;                           // B rows staged (whole swizzle atoms; zeros past N)
  const int a_bytes = kPgM * 128, b_bytes = NP * 128;
  const int stage = 2 * a_bytes + 2 * b_bytes;   // A_hi, A_lo, B_hi, B_lo
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + 2 * stage);
  uint64_t* empty = bars;                        // [2]
  uint64_t* done = bars + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 3);
  const uint32_t tcols = kPgN;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int m0 = blockIdx.x * kPgM;
  const int64_t z = blockIdx.z;
  const TA* A = reinterpret_cast<const TA*>(g.A) + z * g.a_bs;
  const TB* B = reinterpret_cast<const TB*>(g.B) + z * g.b_bs;
  if (tid == 0) {
    mbar_init(&empty[0], 1);
    mbar_init(&empty[1], 1);
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t idesc = idesc_tf32(kPgM, NP);
  const int nkb = (g.K + 31) / 32;
  // staging: element e of a [rows x 32] tile; the source's contiguous
  // dimension is the fastest over consecutive threads.  The global loads of
  // k-block kb + 1 are issued (into registers) right after k-block kb is
  // stored, so they overlap kb's barrier, MMA and the wait for a free stage.
  constexpr int NA = kPgM * 32 / kPgThreads, NB = kPgN * 32 / kPgThreads;
  auto load_tile = [&](auto* src, int64_t rs, int64_t cs, int rows, int row0, int rmax, int k0, auto& x) {
    constexpr int NE = sizeof(x) / sizeof(float);
    const bool kfast = cs == 1;
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int e = tid + i * kPgThreads;
      const int r = kfast ? e / 32 : e % rows;
      const int kk = kfast ? e % 32 : e / rows;
      const int gr = row0 + r, gk = k0 + kk;
      x[i] = 0.f;
      if (gr < rmax && gk < g.K)
        x[i] = elem<std::remove_cv_t<std::remove_pointer_t<decltype(src)>>>::to_f(src[(int64_t)gr * rs + (int64_t)gk * cs]);
    }
  };
  auto store_tile = [&](int64_t cs, int rows, uint8_t* hi, uint8_t* lo, const auto& x) {
    constexpr int NE = sizeof(x) / sizeof(float);
    const bool kfast = cs == 1;
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int e = tid + i * kPgThreads;
      const int r = kfast ? e / 32 : e % rows;
      const int kk = kfast ? e % 32 : e / rows;
      const float h = tf32_hi(x[i]);
      const uint32_t o = sw128_off(r, kk);
      *reinterpret_cast<float*>(hi + o) = h;
      *reinterpret_cast<float*>(lo + o) = x[i] - h;
    }
  };
  float xa[NA], xb[NB];
  if (nkb > 0) {
    load_tile(A, g.a_rs, g.a_cs, kPgM, m0, g.M, 0, xa);
    load_tile(B, g.b_cs, g.b_rs, NP, n0, g.N, 0, xb);
  }
  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb & 1;
    if (kb >= 2) mbar_wait(&empty[s], ((kb - 2) >> 1) & 1);
    uint8_t* st = base + s * stage;
    store_tile(g.a_cs, kPgM, st, st + a_bytes, xa);
    store_tile(g.b_rs, NP, st + 2 * a_bytes, st + 2 * a_bytes + b_bytes, xb);
    if (kb + 1 < nkb) {
      load_tile(A, g.a_rs, g.a_cs, kPgM, m0, g.M, (kb + 1) * 32, xa);
      load_tile(B, g.b_cs, g.b_rs, NP, n0, g.N, (kb + 1) * 32, xb);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t ah = smem_u32(st), al = ah + a_bytes, bh = al + a_bytes, bl = bh + b_bytes;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = (kb | kk) != 0;
        tc_mma_tf32(tmem, sw128_desc(ah + kk * 32), sw128_desc(bh + kk * 32), idesc, acc);
        tc_mma_tf32(tmem, sw128_desc(ah + kk * 32), sw128_desc(bl + kk * 32), idesc, 1);
        tc_mma_tf32(tmem, sw128_desc(al + kk * 32), sw128_desc(bh + kk * 32), idesc, 1);
      }
      tc_commit(&empty[s]);
      if (kb == nkb - 1) tc_commit(done);
    }
  }
  if (nkb > 0) mbar_wait(done, 0);
  tc_fence_after();
  // epilogue: warp w reads TMEM lane quarter w % 4 (rows), column half w / 4
  // (32 columns each); 4 consecutive columns per vector access
  {
    const int q = warp & 3, ch = warp >> 2;
    const int row = m0 + q * 32 + lane;
    const int c0 = ch * 32;
    if (c0 < NT) {
      uint32_t r[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, r);
      if (row < g.M) {
        TC* C = reinterpret_cast<TC*>(g.C) + z * g.c_bs + (int64_t)row * g.c_rs + n0 + c0;
        const int nc = NT - c0 < 32 ? NT - c0 : 32;  // 16 or 32
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          if (j >= nc) break;
          float v[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            v[t] = nkb > 0 ? __uint_as_float(r[j + t]) : 0.f;
            if (g.accumulate) v[t] += ld_f(C + j + t);
          }
          if constexpr (sizeof(TC) == 4) {
            *reinterpret_cast<float4*>(C + j) = make_float4(v[0], v[1], v[2], v[3]);
          } else {
            const __nv_bfloat162 lo = __floats2bfloat162_rn(v[0], v[1]), hi = __floats2bfloat162_rn(v[2], v[3]);
            *reinterpret_cast<uint2*>(C + j) =
                make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
  }
}

size_t pgemm_smem() { return 1024 + 2 * (2 * kPgM * 128 + 2 * kPgN * 128) + 64; }

template <typename TA, typename TB, typename TC>
cudaError_t pgemm(int batch, int M, int N, int K, const TA* A, int64_t a_rs, int64_t a_cs, int64_t a_bs,
                  const TB* B, int64_t b_rs, int64_t b_cs, int64_t b_bs, TC* C, int64_t c_rs, int64_t c_bs,
                  int accumulate, cudaStream_t st) {
  if (N % 32 || (N > kPgN && N % kPgN)) return cudaErrorNotSupported;
  static std::atomic<uint64_t> attr{0};
  cudaError_t e = smem_attr_once(attr, pgemm_kernel<TA, TB, TC>, 227 * 1024);
  if (e != cudaSuccess) return e;
  PgArgs g{M, N, K, A, a_rs, a_cs, a_bs, B, b_rs, b_cs, b_bs, C, c_rs, c_bs, accumulate};
  dim3 grid((M + kPgM - 1) / kPgM, (N + kPgN - 1) / kPgN, batch);
  return launch_pdl(pgemm_kernel<TA, TB, TC>, grid, kPgThreads, pgemm_smem(), st, g);
}

template <typename T>
cudaError_t ln_dispatch(const void* x, void* y, const float* dy, float* dx, int64_t rows, int d,
                        cudaStream_t st) {
  const unsigned blocks = (unsigned)((rows + 7) / 8);
#define LN(E)                                                                                   \
  return dy ? launch_pdl(ln_backward_kernel<T, E>, blocks, 256, 0, st, (const T*)x, dy, dx, rows) \
            : launch_pdl(ln_kernel<T, E>, blocks, 256, 0, st, (const T*)x, (T*)y, rows)
  switch (d / 32) {
    case 1: LN(1);
    case 2: LN(2);
    case 4: LN(4);
    case 8: LN(8);
    default: return cudaErrorNotSupported;
  }
#undef LN
}

}  // namespace

bool prologue_supported(const Shape& s) {
  const int e = s.d_h / 32;
  return s.d_h % 32 == 0 && (e == 1 || e == 2 || e == 4 || e == 8);
}

cudaError_t launch_layernorm(const Shape& s, int64_t rows, const void* x, void* y, const float* dy,
                             float* dx, cudaStream_t st, int* launches) {
  if (!prologue_supported(s)) return cudaErrorNotSupported;
  if (rows == 0) return cudaSuccess;
  cudaError_t e = s.qk_dt == F32 ? ln_dispatch<float>(x, y, dy, dx, rows, s.d_h, st)
                                 : ln_dispatch<__nv_bfloat16>(x, y, dy, dx, rows, s.d_h, st);
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t launch_key_transform(const Shape& s, const void* khat, const float* theta, void* keff,
                                 cudaStream_t st, int* launches) {
  const int d = s.d_h, n = s.n_sub, HH = 2 * s.H;
  // K~ [n x d] = K^ [n x d] Theta^T:  A(i, k) = K^[i][k], B(j, k) = Theta[j][k]
  cudaError_t e = s.qk_dt == F32
      ? pgemm<float, float, float>(HH, n, d, d, (const float*)khat, d, 1, (int64_t)n * d, theta, 1, d,
                                   (int64_t)d * d, (float*)keff, d, (int64_t)n * d, 0, st)
      : pgemm<__nv_bfloat16, float, __nv_bfloat16>(HH, n, d, d, (const __nv_bfloat16*)khat, d, 1,
                                                   (int64_t)n * d, theta, 1, d, (int64_t)d * d,
                                                   (__nv_bfloat16*)keff, d, (int64_t)n * d, 0, st);
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t launch_key_transform_backward(const Shape& s, const void* khat, const float* theta,
                                          const float* dkeff, float* dkhat, float* dtheta,
                                          cudaStream_t st, int* launches) {
  const int d = s.d_h, n = s.n_sub, HH = 2 * s.H;
  // dK^ [n x d] = dK~ [n x d] Theta [d x d] (=):  A(i, r) = dK~[i][r], B(c, r) = Theta[r][c]
  cudaError_t e = pgemm<float, float, float>(HH, n, d, d, dkeff, d, 1, (int64_t)n * d, theta, d, 1,
                                             (int64_t)d * d, dkhat, d, (int64_t)n * d, 0, st);
  if (e != cudaSuccess) return e;
  // dTheta [d x d] += dK~^T K^:  A(r, i) = dK~[i][r], B(c, i) = K^[i][c]
  e = s.qk_dt == F32
      ? pgemm<float, float, float>(HH, d, d, n, dkeff, 1, d, (int64_t)n * d, (const float*)khat, d, 1,
                                   (int64_t)n * d, dtheta, d, (int64_t)d * d, 1, st)
      : pgemm<float, __nv_bfloat16, float>(HH, d, d, n, dkeff, 1, d, (int64_t)n * d,
                                           (const __nv_bfloat16*)khat, d, 1, (int64_t)n * d, dtheta, d,
                                           (int64_t)d * d, 1, st);
  if (e == cudaSuccess) *launches += 2;
  return e;
}

}  // namespace msn
