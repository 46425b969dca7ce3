// backward.cu -- steps a6-a8 of the PKM lookup: the value-table and sub-key
// gradients ("scatter-adds gradients into the value table", PAPER.md:332;
// gradient only through the selected scores, reading R10).
//
// Deterministic path (default, BASELINE.json configs[2] "deterministic
// sort-based scatter-add"):
//   1. stable LSD radix sort of the contributions by destination row
//      (key = slot row, value = contribution id cid = (b*H + h)*k + t);
//   2. row-major segmented reduce: every row's contributions are summed in
//      cid order by one warp (runs crossing a tile boundary are summed from
//      per-tile partials, in tile order, by a fix-up kernel), then added once
//      into the gradient buffer.  For dV the same pass computes
//      dw[cid] = <V[row], dOut[b]>, reading each touched value row ONCE.
//   3. ds = w (dw - sum w dw) (softmax Jacobian), dQ (=) per lookup, and one
//      record per distinct (lookup, half, sub-key) with the aggregated dS;
//   4. sort the records by sub-key row and reduce them into dK (+=) the same way.
// Atomic path (MSN_FLAG_ATOMIC_BWD): query-major re-gather with
// red.global.add.v4.f32 into dV (non-deterministic summation order).
#include "common.cuh"
#include "kernels.h"

namespace msn {
namespace {

// ---------------------------------------------------------------- radix ----
constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 8;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 2048
constexpr int RS_BITS = 8;
constexpr int RS_BUCKETS = 1 << RS_BITS;

__global__ void __launch_bounds__(RS_THREADS) rs_hist_kernel(const uint32_t* __restrict__ keys,
                                                             int64_t n, int shift,
                                                             uint32_t* __restrict__ hist,
                                                             int nblocks) {
  __shared__ uint32_t cnt[RS_BUCKETS];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll
  for (int i = 0; i < RS_ITEMS; ++i) {
    const int64_t p = base + i * RS_THREADS + threadIdx.x;
    if (p < n) atomicAdd(&cnt[(keys[p] >> shift) & (RS_BUCKETS - 1)], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

// Exclusive scan of the digit-major histogram in three coalesced phases:
// per-chunk sums, a scan of the chunk sums, then per-chunk scans with carry.
constexpr int SCAN_T = 256;

__device__ __forceinline__ uint32_t block_excl_scan_256(uint32_t v, uint32_t* total,
                                                        uint32_t* sh /*[8]*/) {
  const int lane = threadIdx.x % 32, wid = threadIdx.x / 32;
  uint32_t incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) sh[wid] = incl;
  __syncthreads();
  uint32_t wpre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < SCAN_T / 32; ++w) {
    const uint32_t x = sh[w];
    wpre += (w < wid) ? x : 0u;
    tot += x;
  }
  __syncthreads();
  *total = tot;
  return wpre + incl - v;
}

__global__ void __launch_bounds__(SCAN_T) scan_reduce_kernel(const uint32_t* __restrict__ data,
                                                             int64_t len, int64_t chunk,
                                                             uint32_t* __restrict__ part) {
  __shared__ uint32_t sh[SCAN_T / 32];
  const int64_t s = (int64_t)blockIdx.x * chunk;
  const int64_t e = s + chunk < len ? s + chunk : len;
  uint32_t acc = 0;
  for (int64_t i = s + threadIdx.x; i < e; i += SCAN_T) acc += data[i];
  uint32_t tot;
  block_excl_scan_256(acc, &tot, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) scan_parts_kernel(uint32_t* __restrict__ part, int n) {
  __shared__ uint32_t sh[32];
  const int t = threadIdx.x, lane = t % 32, wid = t / 32;
  const uint32_t v = t < n ? part[t] : 0u;
  uint32_t incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) sh[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const uint32_t x = sh[lane];
    uint32_t xi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, xi, d);
      if (lane >= d) xi += o;
    }
    sh[lane] = xi - x;
  }
  __syncthreads();
  if (t < n) part[t] = sh[wid] + incl - v;
}

__global__ void __launch_bounds__(SCAN_T) scan_down_kernel(uint32_t* __restrict__ data, int64_t len,
                                                           int64_t chunk,
                                                           const uint32_t* __restrict__ part) {
  __shared__ uint32_t sh[SCAN_T / 32];
  const int64_t s = (int64_t)blockIdx.x * chunk;
  const int64_t e = s + chunk < len ? s + chunk : len;
  uint32_t carry = part[blockIdx.x];
  for (int64_t base = s; base < e; base += SCAN_T) {
    const int64_t i = base + threadIdx.x;
    const uint32_t v = i < e ? data[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan_256(v, &tot, sh);
    if (i < e) data[i] = carry + ex;
    carry += tot;
  }
}

cudaError_t excl_scan(uint32_t* data, int64_t len, uint32_t* part, cudaStream_t st, int* launches) {
  int nb = (int)((len + 255) / 256);
  if (nb > 1024) nb = 1024;
  const int64_t chunk = (len + nb - 1) / nb;
  nb = (int)((len + chunk - 1) / chunk);
  scan_reduce_kernel<<<nb, SCAN_T, 0, st>>>(data, len, chunk, part);
  scan_parts_kernel<<<1, 1024, 0, st>>>(part, nb);
  scan_down_kernel<<<nb, SCAN_T, 0, st>>>(data, len, chunk, part);
  *launches += 3;
  return cudaGetLastError();
}

// Stable scatter: items of a block are ranked per digit in input order with
// warp match-any; warp totals are scanned per digit across the 8 warps.
__global__ void __launch_bounds__(RS_THREADS) rs_scatter_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, int64_t n, int shift,
    const uint32_t* __restrict__ offs, int nblocks, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out) {
  constexpr int NW = RS_THREADS / 32;
  __shared__ uint32_t cnt[NW][RS_BUCKETS + 1];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < NW * (RS_BUCKETS + 1); i += RS_THREADS) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE + wid * (32 * RS_ITEMS);
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t key[RS_ITEMS], val[RS_ITEMS], dig[RS_ITEMS], rank[RS_ITEMS];
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    const int64_t p = base + j * 32 + lane;
    const bool ok = p < n;
    key[j] = ok ? keys_in[p] : 0u;
    val[j] = ok ? (vals_in ? vals_in[p] : (uint32_t)p) : 0u;
    dig[j] = ok ? ((key[j] >> shift) & (RS_BUCKETS - 1)) : RS_BUCKETS;
    const uint32_t peers = __match_any_sync(0xffffffffu, dig[j]);
    const int leader = __ffs(peers) - 1;
    const uint32_t before = cnt[wid][dig[j]];
    rank[j] = before + __popc(peers & lt);
    __syncwarp();
    if (lane == leader) cnt[wid][dig[j]] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {  // exclusive scan across warps, per digit
    const int d = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t c = cnt[w][d];
      cnt[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    if (dig[j] == RS_BUCKETS) continue;
    const uint32_t pos = offs[(int64_t)dig[j] * nblocks + blockIdx.x] + cnt[wid][dig[j]] + rank[j];
    keys_out[pos] = key[j];
    vals_out[pos] = val[j];
  }
}

int bits_for(uint32_t max_key) {
  int b = 1;
  while (b < 32 && (max_key >> b) != 0) ++b;
  return b;
}

// Sorts n keys (all <= max_key) stably, values = input positions.
// Result is in (*keys_res, *vals_res) (one of the ping-pong buffers).
cudaError_t radix_sort(uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b, uint32_t* vals_b,
                       uint32_t* hist, int64_t n, uint32_t max_key, cudaStream_t st, int* launches,
                       uint32_t** keys_res, uint32_t** vals_res) {
  const int bits = bits_for(max_key);
  const int passes = (bits + RS_BITS - 1) / RS_BITS;
  const int nblocks = (int)((n + RS_TILE - 1) / RS_TILE);
  uint32_t *kin = keys_a, *vin = nullptr, *kout = keys_b, *vout = vals_b;
  for (int p = 0; p < passes; ++p) {
    const int shift = p * RS_BITS;
    rs_hist_kernel<<<nblocks, RS_THREADS, 0, st>>>(kin, n, shift, hist, nblocks);
    const int64_t hl = (int64_t)RS_BUCKETS * nblocks;
    cudaError_t e = excl_scan(hist, hl, hist + hl, st, launches);
    if (e != cudaSuccess) return e;
    rs_scatter_kernel<<<nblocks, RS_THREADS, 0, st>>>(kin, vin, n, shift, hist, nblocks, kout,
                                                     vout);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    *launches += 2;
    // ping-pong
    uint32_t* nk = (kout == keys_b) ? keys_a : keys_b;
    uint32_t* nv = (vout == vals_b) ? vals_a : vals_b;
    kin = kout;
    vin = vout;
    kout = nk;
    vout = nv;
  }
  *keys_res = kin;
  *vals_res = vin;
  return cudaSuccess;
}

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
template <int EPL>
__device__ __forceinline__ void add_store_slice(float* p, const float* a) {
#pragma unroll
  for (int i = 0; i < EPL; ++i) p[i] += a[i];
}

// ------------------------------------------------- segmented reduce -------
// MODE_DV : record = cid,            weight = w[cid],    x = dOut[b],          G = dV (local rows),
//           dot: dw[cid] = <V[row], dOut[b]>
// MODE_DK : record = 2*cid + half,   weight = dsS[rec],  x = Q[b,h,half,:],    G = dK rows (h,half,i)
enum { MODE_DV = 0, MODE_DK = 1 };
constexpr int SEG_T = 64;  // entries per warp tile
constexpr int SEG_U = 4;   // entries prefetched per step

struct SegArgs {
  const uint32_t* keys;   // sorted rows (>= nrows: skip)
  const uint32_t* recs;   // record ids in key order
  int64_t n;              // entries
  uint32_t nrows;         // valid rows
  const float* wts;       // per-record weight
  const void* X;          // x rows (dOut fp32 or Q)
  const void* Y;          // V (MODE_DV dot)
  float* dots;            // dw (MODE_DV)
  float* G;               // gradient rows (+=)
  float* part_first;
  float* part_last;
  int H, k, d_h, D;       // D = row width of x / G
};

template <int MODE, typename XT, typename YT, int EPL>
__device__ __forceinline__ const XT* x_row(const SegArgs& a, uint32_t rec) {
  if constexpr (MODE == MODE_DV) {
    const uint32_t b = rec / (uint32_t)(a.H * a.k);
    return reinterpret_cast<const XT*>(a.X) + (int64_t)b * a.D;
  } else {
    const uint32_t cid = rec >> 1, half = rec & 1u;
    const uint32_t bh = cid / (uint32_t)a.k;  // b*H + h
    return reinterpret_cast<const XT*>(a.X) + ((int64_t)bh * 2 + half) * a.d_h;
  }
}

template <int MODE, typename XT, typename YT, int EPL>
__global__ void __launch_bounds__(256) segreduce_kernel(SegArgs a) {
  const int lane = threadIdx.x % 32;
  const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int64_t s = tile * SEG_T;
  if (s >= a.n) return;
  const int64_t e = s + SEG_T < a.n ? s + SEG_T : a.n;
  const int cnt = (int)(e - s);
  uint32_t rk[SEG_T / 32], rr[SEG_T / 32];
#pragma unroll
  for (int u = 0; u < SEG_T / 32; ++u) {
    const int64_t p = s + lane + 32 * u;
    rk[u] = p < e ? a.keys[p] : 0xffffffffu;
    rr[u] = p < e ? a.recs[p] : 0u;
  }
  const uint32_t prev_key = s > 0 ? a.keys[s - 1] : 0xffffffffu;
  const uint32_t next_key = e < a.n ? a.keys[e] : 0xffffffffu;

  float acc[EPL];
  float y[EPL];
  uint32_t cur = 0xffffffffu;
  int run_start = 0;
  auto flush = [&](int run_end) {
    if (cur >= a.nrows) return;
    const bool starts_here = run_start > 0 || s == 0 || prev_key != cur;
    const bool ends_here = run_end < cnt || e == a.n || next_key != cur;
    float* dst;
    if (starts_here && ends_here) {
      dst = a.G + (int64_t)cur * a.D + lane * EPL;
      add_store_slice<EPL>(dst, acc);
      return;
    }
    dst = (!starts_here ? a.part_first : a.part_last) + tile * a.D + lane * EPL;
#pragma unroll
    for (int i = 0; i < EPL; ++i) dst[i] = acc[i];
  };
  for (int j0 = 0; j0 < cnt; j0 += SEG_U) {
    uint32_t key[SEG_U], rec[SEG_U];
    float x[SEG_U][EPL];
    float yp[MODE == MODE_DV ? SEG_U : 1][EPL];
    float wt[SEG_U];
#pragma unroll
    for (int u = 0; u < SEG_U; ++u) {
      const int j = j0 + u;
      const int src = j % 32;
      uint32_t kk = 0xffffffffu, rr_ = 0;
#pragma unroll
      for (int q = 0; q < SEG_T / 32; ++q) {
        const uint32_t k2 = __shfl_sync(0xffffffffu, rk[q], src);
        const uint32_t r2 = __shfl_sync(0xffffffffu, rr[q], src);
        if (j / 32 == q) { kk = k2; rr_ = r2; }
      }
      if (j >= cnt) kk = 0xffffffffu;
      key[u] = kk;
      rec[u] = rr_;
      const bool valid = kk < a.nrows;
      wt[u] = valid ? a.wts[rr_] : 0.f;
      if (valid) load_slice<XT, EPL>(x_row<MODE, XT, YT, EPL>(a, rr_) + lane * EPL, x[u]);
      else
#pragma unroll
        for (int i = 0; i < EPL; ++i) x[u][i] = 0.f;
      if constexpr (MODE == MODE_DV) {
        // prefetch the value row too (repeats within a run hit L1)
        if (valid)
          load_slice<YT, EPL>(reinterpret_cast<const YT*>(a.Y) + (int64_t)kk * a.D + lane * EPL, yp[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < SEG_U; ++u) {
      const int j = j0 + u;
      if (j >= cnt) break;
      if (key[u] != cur) {
        flush(j);
        cur = key[u];
        run_start = j;
#pragma unroll
        for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
        if constexpr (MODE == MODE_DV) {
#pragma unroll
          for (int i = 0; i < EPL; ++i) y[i] = yp[u][i];
        }
      }
      if (cur >= a.nrows) continue;
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[i] = fmaf(wt[u], x[u][i], acc[i]);
      if constexpr (MODE == MODE_DV) {
        float d = 0.f;
#pragma unroll
        for (int i = 0; i < EPL; ++i) d = fmaf(y[i], x[u][i], d);
        d = warp_sum(d);
        if (lane == 0) a.dots[rec[u]] = d;
      }
    }
  }
  flush(cnt);
}

// Runs that cross tiles: the tile where the run starts (its "last" partial)
// sums the "first" partials of the following tiles in tile order.
__global__ void __launch_bounds__(256) seg_fixup_kernel(const uint32_t* __restrict__ keys,
                                                        int64_t n, uint32_t nrows,
                                                        const float* __restrict__ part_first,
                                                        const float* __restrict__ part_last,
                                                        float* __restrict__ G, int D) {
  const int lane = threadIdx.x % 32;
  const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int64_t s = tile * SEG_T;
  if (s >= n) return;
  const int64_t e = s + SEG_T < n ? s + SEG_T : n;
  if (e >= n) return;
  const uint32_t key = keys[e - 1];
  if (key >= nrows || keys[e] != key) return;  // last run ends inside this tile
  // owner test: the run containing entry e-1 starts in this tile
  if (keys[s] == key && s > 0 && keys[s - 1] == key) return;
  for (int c = lane; c < D; c += 32) {
    float acc = part_last[tile * D + c];
    for (int64_t t = tile + 1;; ++t) {
      acc += part_first[t * D + c];
      const int64_t ts = t * SEG_T, te = ts + SEG_T < n ? ts + SEG_T : n;
      if (te >= n || keys[te] != key || keys[te - 1] != key) break;
    }
    G[(int64_t)key * D + c] += acc;
  }
}

template <int MODE, typename XT, typename YT>
cudaError_t launch_seg(const SegArgs& a, int EPLn, cudaStream_t st, int* launches) {
  const int64_t tiles = (a.n + SEG_T - 1) / SEG_T;
  const unsigned blocks = (unsigned)((tiles + 7) / 8);
  switch (EPLn) {
    case 1: segreduce_kernel<MODE, XT, YT, 1><<<blocks, 256, 0, st>>>(a); break;
    case 2: segreduce_kernel<MODE, XT, YT, 2><<<blocks, 256, 0, st>>>(a); break;
    case 4: segreduce_kernel<MODE, XT, YT, 4><<<blocks, 256, 0, st>>>(a); break;
    case 8: segreduce_kernel<MODE, XT, YT, 8><<<blocks, 256, 0, st>>>(a); break;
    case 16: segreduce_kernel<MODE, XT, YT, 16><<<blocks, 256, 0, st>>>(a); break;
    default: return cudaErrorNotSupported;
  }
  seg_fixup_kernel<<<blocks, 256, 0, st>>>(a.keys, a.n, a.nrows, a.part_first, a.part_last, a.G,
                                           a.D);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) *launches += 2;
  return e;
}

// ---------------------------------------------------- contribution keys ----
// key = local row of idx (or nrows sentinel when the slot is held elsewhere)
// (dw of a slot held by another shard is 0 here; the shards' dw are summed)
__global__ void dv_keys_kernel(const int32_t* __restrict__ idx, int64_t n, int64_t row_begin,
                               int64_t row_end, uint32_t sentinel, uint32_t* __restrict__ keys,
                               float* __restrict__ dw) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t f = idx[p];
  const bool local = f >= row_begin && f < row_end;
  keys[p] = local ? (uint32_t)(f - row_begin) : sentinel;
  if (!local) dw[p] = 0.f;
}

// ----------------------------------------------- ds, dQ and dK records ----
// One warp per lookup (b,h).  ds_t = w_t (dw_t - sum_u w_u dw_u).
// For each half, the dS of every distinct sub-key index r is summed over the
// t with r_t = r in t order; dQ[b,h,half] = sum_r dS_r K[h,half,r]; one dK
// record per distinct r (first occurrence), others get the sentinel key.
template <typename QT, int KPL, int EPL>
__global__ void __launch_bounds__(256) ds_dq_kernel(const QT* __restrict__ K,
                                                    const int32_t* __restrict__ idx,
                                                    const float* __restrict__ w,
                                                    const float* __restrict__ dw, int64_t L,
                                                    int H, int n_sub, int d_h, int k,
                                                    float* __restrict__ dQ,
                                                    uint32_t* __restrict__ rkeys,
                                                    float* __restrict__ dsS, uint32_t sentinel) {
  const int lane = threadIdx.x % 32;
  const int64_t l = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (l >= L) return;
  const int h = (int)(l % H);
  float wt[KPL], g[KPL], ds[KPL];
  int32_t f[KPL];
  float part = 0.f;
#pragma unroll
  for (int u = 0; u < KPL; ++u) {
    const int t = lane + 32 * u;
    wt[u] = t < k ? w[l * k + t] : 0.f;
    g[u] = t < k ? dw[l * k + t] : 0.f;
    f[u] = t < k ? idx[l * k + t] : 0;
    part = fmaf(wt[u], g[u], part);
  }
  const float gbar = warp_sum(part);
#pragma unroll
  for (int u = 0; u < KPL; ++u) ds[u] = wt[u] * (g[u] - gbar);
  for (int half = 0; half < 2; ++half) {
    int r[KPL];
#pragma unroll
    for (int u = 0; u < KPL; ++u) r[u] = half == 0 ? f[u] / n_sub : f[u] % n_sub;
    float dS[KPL];
    bool first[KPL];
#pragma unroll
    for (int u = 0; u < KPL; ++u) { dS[u] = 0.f; first[u] = true; }
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
    // records
#pragma unroll
    for (int u = 0; u < KPL; ++u) {
      const int t = lane + 32 * u;
      if (t < k) {
        const int64_t rec = (l * k + t) * 2 + half;
        rkeys[rec] = first[u] ? (uint32_t)((h * 2 + half) * n_sub + r[u]) : sentinel;
        dsS[rec] = dS[u];
      }
    }
    // dQ: lanes over d_h
    float acc[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
    for (int v = 0; v < k; ++v) {
      const int src = v % 32;
      const bool lo = KPL == 1 || v < 32;
      const int rv = __shfl_sync(0xffffffffu, lo ? r[0] : r[KPL - 1], src);
      const float dSv = __shfl_sync(0xffffffffu, lo ? dS[0] : dS[KPL - 1], src);
      const bool fv = __shfl_sync(0xffffffffu, (int)(lo ? first[0] : first[KPL - 1]), src);
      if (!fv) continue;
      float kr[EPL];
      load_slice<QT, EPL>(K + ((int64_t)(h * 2 + half) * n_sub + rv) * d_h + lane * EPL, kr);
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[i] = fmaf(dSv, kr[i], acc[i]);
    }
    float* o = dQ + (l * 2 + half) * d_h + lane * EPL;
#pragma unroll
    for (int i = 0; i < EPL; ++i) o[i] = acc[i];
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

}  // namespace

// ---------------------------------------------------------- workspace ------
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t bwd_workspace_bytes(const Shape& s, int64_t gather_batch) {
  const int64_t n_dv = gather_batch * s.H * s.k;
  const int64_t n_dk = 2 * s.B * s.H * s.k;
  const int64_t n = n_dv > n_dk ? n_dv : n_dk;
  const int64_t nblocks = (n + RS_TILE - 1) / RS_TILE;
  const int64_t tiles = (n + SEG_T - 1) / SEG_T;
  const int64_t D = s.d_v > s.d_h ? s.d_v : s.d_h;
  size_t b = 0;
  b += 4 * align256(sizeof(uint32_t) * n);
  b += align256(sizeof(uint32_t) * (RS_BUCKETS * nblocks + 1024));
  b += 2 * align256(sizeof(float) * tiles * D);
  b += align256(sizeof(float) * n_dk);
  b += align256(sizeof(float) * n_dv);
  return b;
}

BwdWorkspace carve_bwd_workspace(const Shape& s, int64_t gather_batch, void* ws) {
  const int64_t n_dv = gather_batch * s.H * s.k;
  const int64_t n_dk = 2 * s.B * s.H * s.k;
  const int64_t n = n_dv > n_dk ? n_dv : n_dk;
  const int64_t nblocks = (n + RS_TILE - 1) / RS_TILE;
  const int64_t tiles = (n + SEG_T - 1) / SEG_T;
  const int64_t D = s.d_v > s.d_h ? s.d_v : s.d_h;
  char* p = (char*)ws;
  BwdWorkspace w;
  w.keys_a = (uint32_t*)p; p += align256(sizeof(uint32_t) * n);
  w.keys_b = (uint32_t*)p; p += align256(sizeof(uint32_t) * n);
  w.vals_a = (uint32_t*)p; p += align256(sizeof(uint32_t) * n);
  w.vals_b = (uint32_t*)p; p += align256(sizeof(uint32_t) * n);
  w.hist = (uint32_t*)p; p += align256(sizeof(uint32_t) * (RS_BUCKETS * nblocks + 1024));
  w.part_first = (float*)p; p += align256(sizeof(float) * tiles * D);
  w.part_last = (float*)p; p += align256(sizeof(float) * tiles * D);
  w.dsS = (float*)p; p += align256(sizeof(float) * n_dk);
  w.dw = (float*)p; p += align256(sizeof(float) * n_dv);
  return w;
}

// ------------------------------------------------------------ launchers ---
cudaError_t launch_scatter_sorted(const Shape& s, const int32_t* idx, const float* w,
                                  const float* dOut, const void* V, float* dV, float* dw,
                                  const BwdWorkspace& ws, cudaStream_t st, int* launches) {
  if (!epl_ok(s.d_v)) return cudaErrorNotSupported;
  const int64_t n = s.B * s.H * s.k;  // s.B is the gather batch here
  const uint32_t nrows = (uint32_t)(s.row_end - s.row_begin);
  dv_keys_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(idx, n, s.row_begin, s.row_end,
                                                              nrows, ws.keys_a, dw);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ++*launches;
  uint32_t *ks, *vs;
  e = radix_sort(ws.keys_a, ws.vals_a, ws.keys_b, ws.vals_b, ws.hist, n, nrows, st, launches, &ks,
                 &vs);
  if (e != cudaSuccess) return e;
  SegArgs a{ks, vs, n, nrows, w, dOut, V, dw, dV, ws.part_first, ws.part_last, s.H, s.k, s.d_h,
            s.d_v};
  if (s.v_dt == F32) return launch_seg<MODE_DV, float, float>(a, epl_of(s.d_v), st, launches);
  return launch_seg<MODE_DV, float, __nv_bfloat16>(a, epl_of(s.d_v), st, launches);
}

cudaError_t launch_scatter_atomic(const Shape& s, const int32_t* idx, const float* w,
                                  const float* dOut, const void* V, float* dV, float* dw,
                                  cudaStream_t st, int* launches) {
  if (!epl_ok(s.d_v)) return cudaErrorNotSupported;
  const unsigned blocks = (unsigned)((s.B + 7) / 8);
  const int HK = s.H * s.k;
#define ATOMIC(VT, E)                                                                          \
  scatter_atomic_kernel<VT, E><<<blocks, 256, 0, st>>>(idx, w, dOut, (const VT*)V, dV, dw, s.B, \
                                                       HK, s.d_v, s.row_begin, s.row_end)
  const int E = epl_of(s.d_v);
  if (s.v_dt == F32) {
    switch (E) { case 1: ATOMIC(float, 1); break; case 2: ATOMIC(float, 2); break;
      case 4: ATOMIC(float, 4); break; case 8: ATOMIC(float, 8); break;
      default: ATOMIC(float, 16); }
  } else {
    switch (E) { case 1: ATOMIC(__nv_bfloat16, 1); break; case 2: ATOMIC(__nv_bfloat16, 2); break;
      case 4: ATOMIC(__nv_bfloat16, 4); break; case 8: ATOMIC(__nv_bfloat16, 8); break;
      default: ATOMIC(__nv_bfloat16, 16); }
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
  const uint32_t nrows = (uint32_t)(s.H * 2 * s.n_sub);
  const unsigned blocks = (unsigned)((L + 7) / 8);
  const int E = epl_of(s.d_h);
#define DSDQ(QT, KPL, E_)                                                                      \
  ds_dq_kernel<QT, KPL, E_><<<blocks, 256, 0, st>>>((const QT*)K, idx, w, dw, L, s.H, s.n_sub, \
                                                    s.d_h, s.k, dQ, ws.keys_a, ws.dsS, nrows)
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
  const int64_t n = 2 * L * s.k;
  uint32_t *ks, *vs;
  e = radix_sort(ws.keys_a, ws.vals_a, ws.keys_b, ws.vals_b, ws.hist, n, nrows, st, launches, &ks,
                 &vs);
  if (e != cudaSuccess) return e;
  SegArgs a{ks, vs, n, nrows, ws.dsS, Q, nullptr, nullptr, dK, ws.part_first, ws.part_last, s.H,
            s.k, s.d_h, s.d_h};
  if (s.qk_dt == F32) return launch_seg<MODE_DK, float, float>(a, E, st, launches);
  return launch_seg<MODE_DK, __nv_bfloat16, float>(a, E, st, launches);
}

}  // namespace msn
