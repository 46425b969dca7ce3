// common.cuh -- small device helpers shared by the PKM kernels (sm_100a only).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <atomic>

#ifndef __CUDACC__
#error "CUDA only"
#endif

namespace msn {

constexpr int kWarp = 32;

// Programmatic dependent launch.  Every kernel of the library starts with
// pdl_enter(): wait until the previous grid in the stream has completed (and
// its writes are visible), then allow the next grid to be scheduled -- so a
// kernel's launch and prologue overlap its predecessor's tail, and, since
// every kernel waits, completion stays ordered transitively.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Wait only: the next grid is scheduled when this one exits (for a kernel
// whose CTAs must not share the machine with the next grid's waiting CTAs).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Host side: launch with programmatic stream serialization.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool off = getenv("MSN_NO_PDL") != nullptr;  // A/B measurements only
  cfg.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

// Host side: per-device state.  The current device's SM count (cached per
// device), and a one-time-per-device cudaFuncSetAttribute(max dynamic shared
// memory) for a kernel: `done` is that call site's bitmask of devices
// already set (atomic: several host threads may launch concurrently).
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
inline int device_sms() {
  static std::atomic<int> cache[64];
  const int d = current_device();
  if (d < 0 || d >= 64) return 148;
  int n = cache[d].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    if (n <= 0) n = 148;
    cache[d].store(n, std::memory_order_relaxed);
  }
  return n;
}
template <typename... KArgs>
inline cudaError_t smem_attr_once(std::atomic<uint64_t>& done, void (*kernel)(KArgs...), int bytes) {
  const int d = current_device();
  const uint64_t bit = (d >= 0 && d < 64) ? (uint64_t(1) << d) : 0;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// Order-preserving map fp32 -> uint32 (larger float -> larger uint).  -0 is
// canonicalised to +0 first so equal scores tie-break on the index
// (reading R6).
__device__ __forceinline__ uint32_t ord_f32(float f) {
  f = f + 0.0f;
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  return __uint_as_float(u);
}
// Composite selection key: (score desc, index asc) == composite desc.
__device__ __forceinline__ uint64_t sel_key(float s, uint32_t index) {
  return ((uint64_t)ord_f32(s) << 32) | (uint64_t)(0xffffffffu - index);
}
__device__ __forceinline__ float sel_key_score(uint64_t key) { return unord_f32((uint32_t)(key >> 32)); }
__device__ __forceinline__ uint32_t sel_key_index(uint64_t key) { return 0xffffffffu - (uint32_t)key; }

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  lo = __shfl_xor_sync(0xffffffffu, lo, m);
  hi = __shfl_xor_sync(0xffffffffu, hi, m);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    uint64_t o = shfl_xor_u64(v, m);
    v = o > v ? o : v;
  }
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, m));
  return v;
}
__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

// Division by a runtime constant d >= 1 without the integer-divide sequence:
// q = (umulhi(n, m) + n) >> s with s = ceil(log2 d) and
// m = floor(2^32 (2^s - d) / d) + 1, exact for every 32-bit n
// (Granlund-Montgomery); set up once on the host.
struct FastDiv {
  uint32_t m, s, d;
  __host__ FastDiv() : m(0), s(0), d(1) {}
  __host__ explicit FastDiv(uint32_t d_) : d(d_) {
    s = 0;
    while ((1ull << s) < d) ++s;
    m = (uint32_t)(((1ull << 32) * ((1ull << s) - d)) / d + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return (uint32_t)(((uint64_t)__umulhi(n, m) + n) >> s);
  }
};

// ---- element loads/conversions --------------------------------------------
template <typename T> struct elem;
template <> struct elem<float> {
  static constexpr int per16 = 4;  // elements per 16-byte vector
  __device__ __forceinline__ static float to_f(float x) { return x; }
};
template <> struct elem<__nv_bfloat16> {
  static constexpr int per16 = 8;
  __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
};

// 16-byte streaming load through the non-coherent path, no L1 allocation.
__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ldg_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// L2 eviction-priority policies (createpolicy) and loads / reductions
// carrying them: rows streamed once (value rows, gradient rows) are marked
// evict_first, rows re-read from L2 many times (d_out) evict_last, so the
// stream does not push the reused rows out of the 126 MB L2.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ldg_v4_pol(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint2 ldg_v2_pol(const void* p, uint64_t pol) {
  uint2 r;
  asm volatile("ld.global.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void red_add_v4_pol(float* p, float a, float b, float c, float d, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d), "l"(pol)
               : "memory");
}

// unpack a 16-byte vector of T into fp32
template <typename T>
__device__ __forceinline__ void unpack16(const uint4& v, float* f);
template <>
__device__ __forceinline__ void unpack16<float>(const uint4& v, float* f) {
  f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
  f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
}
template <>
__device__ __forceinline__ void unpack16<__nv_bfloat16>(const uint4& v, float* f) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

// Bulk prefetch of `bytes` (multiple of 16, 16-byte aligned) into L2: puts a
// gathered row's HBM read in flight without holding registers.
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Memory-gated fusion gate g and its derivative (tanh;
// the ablation's sigmoid and identity).  kind: 1 tanh,
// 2 sigmoid, 3 identity.
__device__ __forceinline__ float gate_g(float v, int kind) {
  if (kind == 1) return tanhf(v);
  if (kind == 2) return 1.0f / (1.0f + expf(-v));
  return v;
}
__device__ __forceinline__ float gate_dg(float v, int kind) {
  if (kind == 1) {
    const float t = tanhf(v);
    return 1.0f - t * t;
  }
  if (kind == 2) {
    const float sg = 1.0f / (1.0f + expf(-v));
    return sg * (1.0f - sg);
  }
  return 1.0f;
}

// Two independent fp32 FMAs in one instruction (FFMA2, sm_100):
// a0 = fma(x0, s, a0), a1 = fma(x1, s, a1) -- each exactly the scalar fmaf,
// so replacing a pair of fmaf by it changes no result bit.
__device__ __forceinline__ void ffma2(float& a0, float& a1, float x0, float x1, float s) {
  asm("{\n.reg .b64 A, X, S;\n"
      "mov.b64 A, {%0, %1};\n"
      "mov.b64 X, {%2, %3};\n"
      "mov.b64 S, {%4, %4};\n"
      "fma.rn.f32x2 A, X, S, A;\n"
      "mov.b64 {%0, %1}, A;\n}\n"
      : "+f"(a0), "+f"(a1)
      : "f"(x0), "f"(x1), "f"(s));
}

// fire-and-forget vector fp32 add into global memory (sm_90+).
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

}  // namespace msn
