// exchange.cu -- step a9: the record exchange of the row-sharded value table
// (BASELINE.json configs[3] "row-sharded across GPUs ... indices and partial
// weighted sums exchanged by all-to-all over NVLink"; north_star "index
// all-to-all and partial-sum return").
//
// Rank p owns rows [p n/P, (p+1) n/P).  ROUTE turns every selected slot
// (b, h, t) of the home's queries into a 12-byte record {local row, w, b} in
// the owner's segment for this source, grouped by query in (b, h, t) order,
// plus per-query offsets; with peer memory the stores go straight into the
// owner's buffer over NVLink (the all-to-all is issued by the routing kernel
// itself).  GATHER sums w V[row] per (source, query) and stores the partial
// row into the home's receive slot; COMBINE (reduce_partials) adds the P
// partials in owner order.  COLLECT maps the dw the owners return per record
// back to (b, h, t).  The barrier orders the ranks with device-side flags
// (release / acquire at system scope), no host synchronisation.
//
// HBM/NVLink bound: per lookup the route moves k records (12 B each) and the
// gather k value rows; the partial return is d_v * 4 B per (query, owner).
#include "common.cuh"
#include "gather_rows.cuh"
#include "kernels.h"

namespace msn {
namespace {

constexpr int kWarps = 8;
constexpr int kMaxHK = 512;  // H * k records per query (k <= 64, H * k <= 512)
constexpr int kSlices = kMaxHK / 32;

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

// ROUTE pass 1: per (owner, query) record counts, one warp per query.
__global__ void __launch_bounds__(256) route_count_kernel(const int32_t* __restrict__ idx, int64_t lb, int HK,
                                                          OwnerOf own, int P, int32_t* __restrict__ cnt) {
  pdl_enter();
  const int lane = threadIdx.x % 32;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (b >= lb) return;
  int c[kMaxWorld];
#pragma unroll
  for (int o = 0; o < kMaxWorld; ++o) c[o] = 0;
  for (int r0 = 0; r0 < HK; r0 += 32) {
    int o = -1;
    int32_t row;
    if (r0 + lane < HK) own(idx[b * HK + r0 + lane], o, row);
#pragma unroll
    for (int q = 0; q < kMaxWorld; ++q)
      if (q < P) c[q] += __popc(__ballot_sync(0xffffffffu, o == q));
  }
  if (lane < P) {
    int v = 0;
#pragma unroll
    for (int q = 0; q < kMaxWorld; ++q)
      if (q == lane) v = c[q];
    cnt[(int64_t)lane * (lb + 1) + b] = v;
  }
}

// ROUTE pass 2: one CTA per owner: exclusive scan of its counts over the
// queries -> qoff[o][0..lb] (qoff[o][lb] = total), copied to the owner's
// offset destination, and the total into counts[o].
__global__ void __launch_bounds__(1024) route_scan_kernel(const int32_t* __restrict__ cnt, int64_t lb,
                                                          int32_t* __restrict__ qoff, PerRank<int32_t> off_dst,
                                                          int32_t* __restrict__ counts) {
  pdl_enter();
  __shared__ int32_t s_w[32];
  __shared__ int32_t s_carry;
  const int o = blockIdx.x;
  const int tid = threadIdx.x, lane = tid % 32, wid = tid / 32;
  const int32_t* c = cnt + (int64_t)o * (lb + 1);
  int32_t* q = qoff + (int64_t)o * (lb + 1);
  int32_t* d = off_dst.p[o];
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int64_t i0 = 0; i0 < lb; i0 += 1024) {
    const int64_t i = i0 + tid;
    const int32_t v = i < lb ? c[i] : 0;
    int32_t x = v;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, m);
      if (lane >= m) x += y;
    }
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int32_t t = s_w[lane];
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, t, m);
        if (lane >= m) t += y;
      }
      s_w[lane] = t;  // inclusive warp totals
    }
    __syncthreads();
    const int32_t carry = s_carry;
    const int32_t excl = carry + (wid ? s_w[wid - 1] : 0) + x - v;
    if (i < lb) {
      q[i] = excl;
      d[i] = excl;
    }
    __syncthreads();
    if (tid == 0) s_carry = carry + s_w[31];
    __syncthreads();
  }
  if (tid == 0) {
    q[lb] = s_carry;
    d[lb] = s_carry;
    counts[o] = s_carry;
  }
}

// ROUTE pass 3: one warp per query writes its records {row, w, b} in (h, t)
// order into the owners' segments at qoff[o][b] + (rank among this query's
// records of owner o), and the slot's position into pos.
__global__ void __launch_bounds__(256) route_write_kernel(const int32_t* __restrict__ idx,
                                                          const float* __restrict__ w, int64_t lb, int HK,
                                                          OwnerOf own, int P, const int32_t* __restrict__ qoff,
                                                          PerRank<int32_t> drow, PerRank<float> dw_,
                                                          PerRank<int32_t> dq, int32_t* __restrict__ pos) {
  pdl_enter();
  const int lane = threadIdx.x % 32;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (b >= lb) return;
  int base = 0;  // lane o (< P): this query's next position in owner o's segment
  if (lane < P) base = qoff[(int64_t)lane * (lb + 1) + b];
  for (int r0 = 0; r0 < HK; r0 += 32) {
    const int r = r0 + lane;
    int o = -1;
    int32_t row = 0;
    float wt = 0.f;
    if (r < HK) {
      own(idx[b * HK + r], o, row);
      wt = w[b * HK + r];
    }
    int my = 0, add = 0;
#pragma unroll
    for (int q = 0; q < kMaxWorld; ++q) {
      if (q < P) {
        const unsigned m = __ballot_sync(0xffffffffu, o == q);
        const int bq = __shfl_sync(0xffffffffu, base, q);
        if (o == q) my = bq + __popc(m & ((1u << lane) - 1u));
        if (lane == q) add = __popc(m);
      }
    }
    base += add;
    if (r < HK) {
      int32_t* prow = nullptr;
      float* pw = nullptr;
      int32_t* pq = nullptr;
#pragma unroll
      for (int q = 0; q < kMaxWorld; ++q)
        if (q == o) { prow = drow.p[q]; pw = dw_.p[q]; pq = dq.p[q]; }
      prow[my] = row;
      pw[my] = wt;
      pq[my] = (int32_t)b;
      pos[b * HK + r] = my;
    }
  }
}

// GATHER: one warp per (source s, query b): the records of IN segment s in
// [off[s][b], off[s][b+1]) are staged in shared memory and summed in record
// order (= the (h, t) order of the home) by gather_rows; the partial row goes
// to dst[s] + b d_v (the home's receive slot).
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
  if (pair >= (int64_t)r.P * r.lb) return;
  const int src = (int)(pair / r.lb);
  const int64_t b = pair - (int64_t)src * r.lb;
  const int32_t* off = r.off + (int64_t)src * (r.lb + 1);
  const int32_t j0 = off[b], j1 = off[b + 1];
  const int n = j1 - j0;  // <= H k
  const int64_t seg = (int64_t)src * r.cap + j0;
  for (int i = lane; i < n; i += 32) {
    s_idx[wid][i] = r.row[seg + i];
    s_w[wid][i] = r.w[seg + i];
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

// COLLECT: dw[p] = dw_in[owner(idx[p]) * cap + pos[p]]
__global__ void __launch_bounds__(256) collect_dw_kernel(const int32_t* __restrict__ idx,
                                                         const int32_t* __restrict__ pos,
                                                         const float* __restrict__ dw_in, int64_t n,
                                                         int64_t cap, OwnerOf own, float* __restrict__ dw) {
  pdl_enter();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  int o;
  int32_t row;
  own(idx[p], o, row);
  dw[p] = dw_in[(int64_t)o * cap + pos[p]];
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

cudaError_t launch_route(const Shape& s, const int32_t* idx, const float* w, const RouteArgs& a,
                         cudaStream_t st, int* launches) {
  const int HK = s.H * s.k;
  if (HK > kMaxHK || a.P < 1 || a.P > kMaxWorld) return cudaErrorNotSupported;
  if (a.lb == 0) return cudaSuccess;
  const OwnerOf own = owner_of(a.rpr);
  const unsigned blocks = (unsigned)((a.lb + kWarps - 1) / kWarps);
  launch_pdl(route_count_kernel, blocks, 256, 0, st, idx, a.lb, HK, own, a.P, a.cnt);
  launch_pdl(route_scan_kernel, (unsigned)a.P, 1024, 0, st, (const int32_t*)a.cnt, a.lb, a.qoff, a.off, a.counts);
  launch_pdl(route_write_kernel, blocks, 256, 0, st, idx, w, a.lb, HK, own, a.P, (const int32_t*)a.qoff, a.row,
             a.w, a.q, a.pos);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) *launches += 3;
  return e;
}

template <typename VT>
static cudaError_t gather_records_t(const Shape& s, const RecordsIn& r, const VT* V, const PerRank<float>& dst,
                                    cudaStream_t st) {
  const int R = s.d_v * (int)sizeof(VT) / 16;
  const unsigned blocks = (unsigned)(((int64_t)r.P * r.lb + kWarps - 1) / kWarps);
#define GREC(VPL, G, U) \
  launch_pdl(gather_records_kernel<VT, VPL, G, U>, blocks, 256, 0, st, r, V, s.d_v, dst)
  MSN_GATHER_DISPATCH(R, GREC);
#undef GREC
  return cudaGetLastError();
}

cudaError_t launch_gather_records(const Shape& s, const RecordsIn& r, const void* V, const PerRank<float>& dst,
                                  cudaStream_t st, int* launches) {
  if (s.H * s.k > kMaxHK || r.P < 1 || r.P > kMaxWorld) return cudaErrorNotSupported;
  if (r.lb == 0) return cudaSuccess;
  cudaError_t e = s.v_dt == F32 ? gather_records_t<float>(s, r, (const float*)V, dst, st)
                                : gather_records_t<__nv_bfloat16>(s, r, (const __nv_bfloat16*)V, dst, st);
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t launch_collect_dw(const Shape& s, const int32_t* idx, const int32_t* pos, const float* dw_in,
                              int64_t cap, int64_t rpr, float* dw, cudaStream_t st, int* launches) {
  const int64_t n = s.B * s.H * s.k;
  if (n == 0) return cudaSuccess;
  launch_pdl(collect_dw_kernel, (unsigned)((n + 255) / 256), 256, 0, st, idx, pos, dw_in, n, cap, owner_of(rpr),
             dw);
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
