// exchange.cu -- step a9: the record exchange of the row-sharded value table
// (BASELINE.json configs[3] "row-sharded across GPUs ... indices and partial
// weighted sums exchanged by all-to-all over NVLink"; north_star "index
// all-to-all and partial-sum return").
//
// Rank p owns rows [p n/P, (p+1) n/P).  The ROUTE is fused into the
// Cartesian kernel (cartesian.cu: every selected slot becomes an 8-byte record
// {local row, w} in its owner's window for (source, query), H k slots per
// window, records in (h, t) order, the local shard gathered on the spot); with
// peer memory the records are stored straight into the owner's buffer over
// NVLink.  Here: GATHER sums w V[row] per (remote source, query) window and
// stores the partial row into the home's receive slot; COMBINE
// (reduce_partials) adds the P partials in owner order; COLLECT maps the dw
// the owners return per record back to (b, h, t).  The barrier orders the
// ranks with device-side flags (release / acquire at system scope), no host
// synchronisation.
//
// HBM/NVLink bound: per lookup the route moves k records (8 B each) and the
// gather k value rows; the partial return is d_v * 4 B per (query, owner).
#include "common.cuh"
#include "gather_rows.cuh"
#include "kernels.h"

namespace msn {
namespace {

constexpr int kWarps = 8;
constexpr int kMaxHK = 512;  // H * k records per query (k <= 64, H * k <= 512)

// owner and local row of a global slot id f: rows per rank rpr = n / P
struct OwnerOf {
  FastDiv div_rpr;
  uint32_t rpr;
  __device__ __forceinline__ void operator()(int32_t f, int& o, int32_t& row) const {
    const uint32_t q = div_rpr.div((uint32_t)f);
    o = (int)q;
    row = (int32_t)((uint32_t)f - q * rpr);
  }
};

// GATHER: one warp per (remote source s, query b): the records of window
// (s, b) are staged in shared memory and summed in record order (= the (h, t)
// order of the home) by gather_rows; the partial row goes to dst[s] + b d_v
// (the home's receive slot).  Window pairs run over s != rank only (the home
// gathered its own shard's rows in the Cartesian kernel).
template <typename VT, int VPL, int G, int U>
__global__ void __launch_bounds__(256) gather_records_kernel(RecordsIn r, const VT* __restrict__ V, int d_v,
                                                             PerRank<float> dst) {
  pdl_enter();
  constexpr int PER = elem<VT>::per16;
  constexpr int LG = 32 / G;
  __shared__ int32_t s_idx[kWarps][kMaxHK];
  __shared__ float s_w[kWarps][kMaxHK];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t pair = (int64_t)blockIdx.x * kWarps + wid;
  if (pair >= (int64_t)(r.P - 1) * r.lb) return;
  int src = (int)(pair / r.lb);
  const int64_t b = pair - (int64_t)src * r.lb;
  if (src >= r.rank) ++src;  // skip the home's own shard
  const int64_t win = (int64_t)src * r.lb + b;
  const int n = r.cnt[win];  // <= H k
  const int64_t base = win * r.HK;
  for (int i = lane; i < n; i += 32) {
    s_idx[wid][i] = r.row[base + i];
    s_w[wid][i] = r.w[base + i];
  }
  __syncwarp();
  float tot[VPL][PER];
  gather_rows<VT, VPL, G, U>(s_idx[wid], s_w[wid], 0, n, V, d_v, tot);
  const int g = lane / LG, gl = lane % LG;
  if (g == 0) {
    float* o = nullptr;
#pragma unroll
    for (int q = 0; q < kMaxWorld; ++q)
      if (q == src) o = dst.p[q];  // (constant-index parameter loads, no local copy)
    o += b * d_v;
    const int row_vecs = d_v / PER;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int vec = gl * VPL + v;
      if (vec < row_vecs) {
#pragma unroll
        for (int e = 0; e < PER; e += 4)
          *reinterpret_cast<float4*>(o + vec * PER + e) =
              make_float4(tot[v][e], tot[v][e + 1], tot[v][e + 2], tot[v][e + 3]);
      }
    }
  }
}

// COLLECT: dw[p] = dw_in[owner(idx[p]) * cap + (p / HK) * HK + pos[p]]
__global__ void __launch_bounds__(256) collect_dw_kernel(const int32_t* __restrict__ idx,
                                                         const int32_t* __restrict__ pos,
                                                         const float* __restrict__ dw_in, int64_t n, int HK,
                                                         int64_t cap, OwnerOf own, float* __restrict__ dw) {
  pdl_enter();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  int o;
  int32_t row;
  own(idx[p], o, row);
  dw[p] = dw_in[(int64_t)o * cap + (p / HK) * HK + pos[p]];
}

// Device-side barrier: epoch = ++ctl[16]; every rank's flag [rank] <- epoch
// (release, system scope: NVLink peers), then wait until every flag of this
// rank is >= epoch (acquire).  Bounded wait (10 s by %globaltimer): on
// timeout ctl[17] = 1 and the kernel returns (no GPU hang).
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__global__ void exchange_barrier_kernel(int P, int rank, PerRank<uint32_t> flags, uint32_t* ctl) {
  pdl_enter();
  __shared__ uint32_t s_epoch;
  const int t = threadIdx.x;
  if (t == 0) {
    s_epoch = ctl[16] + 1u;
    ctl[16] = s_epoch;
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  __threadfence_system();  // this rank's earlier stores (previous kernels) before the flag
  if (t < P) st_release_sys(flags.p[t] + rank, epoch);
  if (t < P) {
    const uint64_t t0 = globaltimer();
    while ((int32_t)(ld_acquire_sys(ctl + t) - epoch) < 0) {
      if (globaltimer() - t0 > 10000000000ull) {
        ctl[17] = 1u;
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  __threadfence_system();
}

}  // namespace

static OwnerOf owner_of(int64_t rpr) {
  OwnerOf o;
  o.div_rpr = FastDiv((uint32_t)rpr);
  o.rpr = (uint32_t)rpr;
  return o;
}

template <typename VT>
static cudaError_t gather_records_t(const Shape& s, const RecordsIn& r, const VT* V, const PerRank<float>& dst,
                                    cudaStream_t st) {
  const int R = s.d_v * (int)sizeof(VT) / 16;
  const unsigned blocks = (unsigned)(((int64_t)(r.P - 1) * r.lb + kWarps - 1) / kWarps);
#define GREC(VPL, G, U) \
  launch_pdl(gather_records_kernel<VT, VPL, G, U>, blocks, 256, 0, st, r, V, s.d_v, dst)
  MSN_GATHER_DISPATCH(R, GREC);
#undef GREC
  return cudaGetLastError();
}

cudaError_t launch_gather_records(const Shape& s, const RecordsIn& r, const void* V, const PerRank<float>& dst,
                                  cudaStream_t st, int* launches) {
  if (s.H * s.k > kMaxHK || r.P < 1 || r.P > kMaxWorld) return cudaErrorNotSupported;
  if (r.lb == 0 || r.P == 1) return cudaSuccess;  // (no remote source)
  cudaError_t e = s.v_dt == F32 ? gather_records_t<float>(s, r, (const float*)V, dst, st)
                                : gather_records_t<__nv_bfloat16>(s, r, (const __nv_bfloat16*)V, dst, st);
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t launch_collect_dw(const Shape& s, const int32_t* idx, const int32_t* pos, const float* dw_in,
                              int64_t cap, int64_t rpr, float* dw, cudaStream_t st, int* launches) {
  const int64_t n = s.B * s.H * s.k;
  if (n == 0) return cudaSuccess;
  launch_pdl(collect_dw_kernel, (unsigned)((n + 255) / 256), 256, 0, st, idx, pos, dw_in, n, s.H * s.k, cap,
             owner_of(rpr), dw);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t launch_exchange_barrier(int P, int rank, const PerRank<uint32_t>& flags, uint32_t* ctl,
                                    cudaStream_t st, int* launches) {
  launch_pdl(exchange_barrier_kernel, 1, 32, 0, st, P, rank, flags, ctl);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace msn
