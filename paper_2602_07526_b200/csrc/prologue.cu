// prologue.cu -- the query / key prologue of the lookup:
//   LayerNorm of query and sub-key vectors before scoring (
//   reading R23: no affine, eps = 1e-5) and its backward;
//   key over-parameterisation K~ = Theta K per (head, half)
//   and its gradients dTheta = sum_i dk~_i k_i^T, dk_i = Theta^T dk~_i
//   (PAPER.md:296-302).
// LN: one warp per row (the row lives in the lane registers), fp32 math,
// output rounded once to the storage type.  The Theta products are batched
// over the 2H codebooks as a 64x64-tiled fp32 SIMT GEMM (shared-memory
// staging, 4x4 outputs per thread): at n_sub x d x d per codebook this is a
// few hundred MFLOP per step, and fp32 keeps the fp32 configs exact enough
// for their 1e-4 tolerance.
#include "common.cuh"
#include "kernels.h"

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

// C[b] (= or +=) A[b] B[b]: A(i,k) = A[b*a_bs + i*a_rs + k*a_cs], likewise B;
// C row-major with row stride c_rs.  64 x 64 tile per CTA, k-steps of 16;
// the operand loads run kPf steps ahead of the math (a register ring), so a
// k-step costs its arithmetic rather than a global-load round trip.  The k
// order of the accumulation is unchanged (ascending).
constexpr int kPf = 4;
template <typename TA, typename TB, typename TC>
__global__ void __launch_bounds__(256) gemm_kernel(int M, int N, int K, const TA* __restrict__ A,
                                                   int64_t a_rs, int64_t a_cs, int64_t a_bs,
                                                   const TB* __restrict__ B, int64_t b_rs,
                                                   int64_t b_cs, int64_t b_bs, TC* __restrict__ C,
                                                   int64_t c_rs, int64_t c_bs, int accumulate) {
  pdl_enter();
  __shared__ float As[16][64 + 4], Bs[16][64 + 4];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int64_t bi = blockIdx.z;
  A += bi * a_bs;
  B += bi * b_bs;
  C += bi * c_bs;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const bool a_k = a_cs == 1;  // A contiguous along k
  const bool b_k = b_rs == 1;  // B contiguous along k
  // 16 x 64 elements per operand tile, 4 per thread; consecutive threads walk
  // the operand's contiguous dimension (coalesced loads)
  auto load = [&](int k0, float (&va)[4], float (&vb)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + u * 256;
      const int kk = a_k ? e % 16 : e / 64, ii = a_k ? e / 16 : e % 64;
      const int gk = k0 + kk;
      va[u] = (m0 + ii < M && gk < K) ? ld_f(A + (int64_t)(m0 + ii) * a_rs + (int64_t)gk * a_cs) : 0.f;
      const int kb = b_k ? e % 16 : e / 64, jj = b_k ? e / 16 : e % 64;
      const int gb = k0 + kb;
      vb[u] = (n0 + jj < N && gb < K) ? ld_f(B + (int64_t)gb * b_rs + (int64_t)(n0 + jj) * b_cs) : 0.f;
    }
  };
  float ra[kPf][4], rb[kPf][4];
#pragma unroll
  for (int d = 0; d < kPf; ++d) load(d * 16, ra[d], rb[d]);
  for (int k0 = 0; k0 < K; k0 += 16 * kPf) {
#pragma unroll
    for (int d = 0; d < kPf; ++d) {
      const int kc = k0 + d * 16;
      if (kc >= K) break;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = tid + u * 256;
        const int kk = a_k ? e % 16 : e / 64, ii = a_k ? e / 16 : e % 64;
        As[kk][ii] = ra[d][u];
        const int kb = b_k ? e % 16 : e / 64, jj = b_k ? e / 16 : e % 64;
        Bs[kb][jj] = rb[d][u];
      }
      __syncthreads();
      load(kc + 16 * kPf, ra[d], rb[d]);  // kPf steps ahead (zeros past K)
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        float a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      TC* p = C + (int64_t)m * c_rs + n;
      const float v = accumulate ? ld_f(p) + acc[i][j] : acc[i][j];
      st_f(p, v);
    }
  }
}

template <typename TA, typename TB, typename TC>
cudaError_t gemm(int batch, int M, int N, int K, const TA* A, int64_t a_rs, int64_t a_cs,
                 int64_t a_bs, const TB* B, int64_t b_rs, int64_t b_cs, int64_t b_bs, TC* C,
                 int64_t c_rs, int64_t c_bs, int accumulate, cudaStream_t st) {
  dim3 grid((N + 63) / 64, (M + 63) / 64, batch);
  return launch_pdl(gemm_kernel<TA, TB, TC>, grid, 256, 0, st, M, N, K, A, a_rs, a_cs, a_bs, B,
                    b_rs, b_cs, b_bs, C, c_rs, c_bs, accumulate);
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
  // K~ [n x d] = K^ [n x d] Theta^T:  B(k, j) = Theta[j][k]
  cudaError_t e = s.qk_dt == F32
      ? gemm<float, float, float>(HH, n, d, d, (const float*)khat, d, 1, (int64_t)n * d, theta, 1, d,
                                  (int64_t)d * d, (float*)keff, d, (int64_t)n * d, 0, st)
      : gemm<__nv_bfloat16, float, __nv_bfloat16>(HH, n, d, d, (const __nv_bfloat16*)khat, d, 1,
                                                  (int64_t)n * d, theta, 1, d, (int64_t)d * d,
                                                  (__nv_bfloat16*)keff, d, (int64_t)n * d, 0, st);
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t launch_key_transform_backward(const Shape& s, const void* khat, const float* theta,
                                          const float* dkeff, float* dkhat, float* dtheta,
                                          cudaStream_t st, int* launches) {
  const int d = s.d_h, n = s.n_sub, HH = 2 * s.H;
  // dK^ [n x d] = dK~ [n x d] Theta [d x d]   (=)
  cudaError_t e = gemm<float, float, float>(HH, n, d, d, dkeff, d, 1, (int64_t)n * d, theta, d, 1,
                                            (int64_t)d * d, dkhat, d, (int64_t)n * d, 0, st);
  if (e != cudaSuccess) return e;
  // dTheta [d x d] += dK~^T [d x n] K^ [n x d]:  A(i, k) = dK~[k][i]
  e = s.qk_dt == F32
      ? gemm<float, float, float>(HH, d, d, n, dkeff, 1, d, (int64_t)n * d, (const float*)khat, d, 1,
                                  (int64_t)n * d, dtheta, d, (int64_t)d * d, 1, st)
      : gemm<float, __nv_bfloat16, float>(HH, d, d, n, dkeff, 1, d, (int64_t)n * d,
                                          (const __nv_bfloat16*)khat, d, 1, (int64_t)n * d, dtheta, d,
                                          (int64_t)d * d, 1, st);
  if (e == cudaSuccess) *launches += 2;
  return e;
}

}  // namespace msn
