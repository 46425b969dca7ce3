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
constexpr int RS_MAX_BITS = 11;  // digit width <= 11 bits (<= 2048 buckets)

__global__ void __launch_bounds__(RS_THREADS) rs_hist_kernel(const uint32_t* __restrict__ keys,
                                                             int64_t n, int shift, int nb,
                                                             uint32_t* __restrict__ hist,
                                                             int nblocks) {
  extern __shared__ uint32_t cnt[];  // nb
  for (int d = threadIdx.x; d < nb; d += RS_THREADS) cnt[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
  const uint32_t mask = (uint32_t)nb - 1u;
#pragma unroll
  for (int i = 0; i < RS_ITEMS; ++i) {
    const int64_t p = base + i * RS_THREADS + threadIdx.x;
    if (p < n) atomicAdd(&cnt[(keys[p] >> shift) & mask], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < nb; d += RS_THREADS) hist[(int64_t)d * nblocks + blockIdx.x] = cnt[d];
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
// warp match-any; warp totals are scanned per digit across the 8 warps; the
// block's items are then reordered by digit in shared memory so that each
// digit's run is written to its global range with coalesced stores.
__global__ void __launch_bounds__(RS_THREADS) rs_scatter_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, int64_t n, int shift,
    int nb, const uint32_t* __restrict__ offs, int nblocks, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out) {
  constexpr int NW = RS_THREADS / 32;
  extern __shared__ uint32_t smem_rs[];
  const int stride_w = nb + 1;
  uint32_t* cnt_raw = smem_rs;                 // [NW][nb + 1]
  uint32_t* bstart = cnt_raw + NW * stride_w;  // [nb] block-local exclusive start per digit
  uint32_t* goff = bstart + nb;                // [nb] global start of this block's digit run
  uint32_t* skey = goff + nb;                  // [RS_TILE]
  uint32_t* sval = skey + RS_TILE;             // [RS_TILE]
  __shared__ uint32_t wsum[NW];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < NW * stride_w; i += RS_THREADS) cnt_raw[i] = 0;
  for (int d = threadIdx.x; d < nb; d += RS_THREADS) goff[d] = offs[(int64_t)d * nblocks + blockIdx.x];
  __syncthreads();
  uint32_t* cntw = cnt_raw + wid * stride_w;
  const uint32_t mask = (uint32_t)nb - 1u;
  const int64_t tile0 = (int64_t)blockIdx.x * RS_TILE;
  const int64_t base = tile0 + wid * (32 * RS_ITEMS);
  const int items = (int)((n - tile0) < RS_TILE ? (n - tile0) : RS_TILE);
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t key[RS_ITEMS], val[RS_ITEMS], dig[RS_ITEMS], rank[RS_ITEMS];
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    const int64_t p = base + j * 32 + lane;
    const bool ok = p < n;
    key[j] = ok ? keys_in[p] : 0u;
    val[j] = ok ? (vals_in ? vals_in[p] : (uint32_t)p) : 0u;
    dig[j] = ok ? ((key[j] >> shift) & mask) : (uint32_t)nb;
    const uint32_t peers = __match_any_sync(0xffffffffu, dig[j]);
    const int leader = __ffs(peers) - 1;
    const uint32_t before = cntw[dig[j]];
    rank[j] = before + __popc(peers & lt);
    __syncwarp();
    if (lane == leader) cntw[dig[j]] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive offsets across warps (in place) and the block total
  for (int d = threadIdx.x; d < nb; d += RS_THREADS) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t c = cnt_raw[w * stride_w + d];
      cnt_raw[w * stride_w + d] = run;
      run += c;
    }
    bstart[d] = run;
  }
  __syncthreads();
  // block-local exclusive scan of the digit totals (nb <= 2048, 8 per thread)
  {
    const int per = (nb + RS_THREADS - 1) / RS_THREADS;
    const int d0 = threadIdx.x * per;
    uint32_t loc[8];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int d = d0 + i;
      loc[i] = (i < per && d < nb) ? bstart[d] : 0u;
      sum += loc[i];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) wpre += (w < wid) ? wsum[w] : 0u;
    uint32_t run = wpre + incl - sum;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int d = d0 + i;
      if (i < per && d < nb) {
        bstart[d] = run;
        run += loc[i];
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    if (dig[j] == (uint32_t)nb) continue;
    const uint32_t local = bstart[dig[j]] + cntw[dig[j]] + rank[j];
    skey[local] = key[j];
    sval[local] = val[j];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < items; i += RS_THREADS) {
    const uint32_t k = skey[i];
    const uint32_t d = (k >> shift) & mask;
    const uint32_t pos = goff[d] + (uint32_t)i - bstart[d];
    keys_out[pos] = k;
    vals_out[pos] = sval[i];
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
  const int nblocks = (int)((n + RS_TILE - 1) / RS_TILE);
  // digit width: <= 11 bits and a histogram of <= 2^20 entries, balanced over the passes
  int wmax = RS_MAX_BITS;
  while (wmax > 4 && ((int64_t)nblocks << wmax) > (int64_t(1) << 20)) --wmax;
  const int passes = (bits + wmax - 1) / wmax;
  const int width = (bits + passes - 1) / passes;
  const int nb = 1 << width;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(rs_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         ((RS_THREADS / 32) * ((1 << RS_MAX_BITS) + 1) + 2 * (1 << RS_MAX_BITS) +
                          2 * RS_TILE) * 4);
    attr = true;
  }
  const size_t smem_scatter = ((size_t)(RS_THREADS / 32) * (nb + 1) + 2 * nb + 2 * RS_TILE) * 4;
  uint32_t *kin = keys_a, *vin = nullptr, *kout = keys_b, *vout = vals_b;
  for (int p = 0; p < passes; ++p) {
    const int shift = p * width;
    rs_hist_kernel<<<nblocks, RS_THREADS, nb * 4, st>>>(kin, n, shift, nb, hist, nblocks);
    const int64_t hl = (int64_t)nb * nblocks;
    cudaError_t e = excl_scan(hist, hl, hist + hl, st, launches);
    if (e != cudaSuccess) return e;
    rs_scatter_kernel<<<nblocks, RS_THREADS, smem_scatter, st>>>(kin, vin, n, shift, nb, hist,
                                                                nblocks, kout, vout);
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

// Raw 16-byte vectors of a row slice of EPL elements of T (prefetched as
// bytes, converted when consumed).
template <typename T, int EPL>
struct RawSlice {
  static constexpr int BYTES = EPL * (int)sizeof(T);
  static constexpr int NV = BYTES >= 16 ? BYTES / 16 : 1;
  uint4 v[NV];
  __device__ __forceinline__ void load(const T* p) {
    if constexpr (BYTES >= 16) {
#pragma unroll
      for (int i = 0; i < NV; ++i) v[i] = ldg_v4(reinterpret_cast<const char*>(p) + 16 * i);
    } else {
      uint32_t w[4] = {0, 0, 0, 0};
      const uint16_t* h = reinterpret_cast<const uint16_t*>(p);
      if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int i = 0; i < EPL; ++i) w[i] = reinterpret_cast<const uint32_t*>(p)[i];
      } else {
#pragma unroll
        for (int i = 0; i < EPL; ++i) w[i / 2] |= (uint32_t)h[i] << (16 * (i % 2));
      }
      v[0] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = make_uint4(0, 0, 0, 0);
  }
  __device__ __forceinline__ void to_float(float* f) const {
    if constexpr (BYTES >= 16) {
#pragma unroll
      for (int i = 0; i < NV; ++i) unpack16<T>(v[i], f + i * elem<T>::per16);
    } else {
      float t[16 / sizeof(T)];
      unpack16<T>(v[0], t);
#pragma unroll
      for (int i = 0; i < EPL; ++i) f[i] = t[i];
    }
  }
};

// Batched butterfly: U per-lane partial sums -> full warp sums, with
// (U - 1) + log2(32 / U) shuffles instead of 5U.  Dot u ends in lane
// u * (32 / U) (fixed order: deterministic).
template <int U>
__device__ __forceinline__ float multi_warp_sum(float (&d)[U]) {
  const int lane = threadIdx.x % 32;
  float v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = d[u];
  int n = U;
#pragma unroll
  for (int m = 16; m >= 32 / U; m >>= 1) {
    // keep half of the n values, send the other half to lane ^ m
    const bool hi = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < U / 2; ++i) {
      if (i < n / 2) {
        const float keep = hi ? v[i + n / 2] : v[i];
        const float send = hi ? v[i] : v[i + n / 2];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
      }
    }
    n >>= 1;
  }
  float r = v[0];
#pragma unroll
  for (int m = 32 / U / 2; m > 0; m >>= 1) r += __shfl_xor_sync(0xffffffffu, r, m);
  return r;
}

// Staged entry of a tile: key (row), record id, weight, x-row index and flags.
struct __align__(16) SegEntry {
  uint32_t key, rec;
  float wt;
  uint32_t xrow_flags;  // bits 0..29 x row, bit 30 starts_here, bit 31 new_run
};
constexpr uint32_t SF_NEW = 0x80000000u, SF_START = 0x40000000u, SF_XROW = 0x3fffffffu;

// One warp per tile of SEG_T sorted entries.  The tile's entries are staged
// in shared memory (row, record, weight, x-row index, run flags computed
// once), then consumed in groups of U: all loads of a group (x rows, value
// rows at run starts, gradient rows of runs that start in this tile) are
// issued before any is used.  Complete runs update the gradient row once
// (G = G + sum, in record order); runs that cross a tile boundary leave
// per-tile partials for seg_fixup_kernel.
template <int MODE, typename XT, typename YT, int EPL>
__global__ void __launch_bounds__(256, 2) segreduce_kernel(SegArgs a) {
  constexpr int U = EPL >= 16 ? 2 : (EPL >= 8 ? 4 : 8);
  __shared__ SegEntry stage[8][SEG_T];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int64_t s = tile * SEG_T;
  if (s >= a.n) return;
  const int64_t e = s + SEG_T < a.n ? s + SEG_T : a.n;
  const int cnt = (int)(e - s);
  if (a.keys[s] >= a.nrows) return;  // sorted: the rest of the array is sentinels
  const uint32_t prev_key = s > 0 ? a.keys[s - 1] : 0xffffffffu;
  const uint32_t next_key = e < a.n ? a.keys[e] : 0xffffffffu;
  {
    uint32_t k2[SEG_T / 32];
#pragma unroll
    for (int u = 0; u < SEG_T / 32; ++u) {
      const int j = lane + 32 * u;
      k2[u] = j < cnt ? a.keys[s + j] : 0xffffffffu;
    }
#pragma unroll
    for (int u = 0; u < SEG_T / 32; ++u) {
      const int j = lane + 32 * u;
      uint32_t pk = __shfl_up_sync(0xffffffffu, k2[u], 1);
      const uint32_t wrap = u > 0 ? __shfl_sync(0xffffffffu, k2[u > 0 ? u - 1 : 0], 31) : prev_key;
      if (lane == 0) pk = wrap;
      if (j < cnt) {
        const uint32_t kk = k2[u];
        const uint32_t rec = a.recs[s + j];
        const bool valid = kk < a.nrows;
        uint32_t xrow;
        if constexpr (MODE == MODE_DV) xrow = rec / (uint32_t)(a.H * a.k);
        else xrow = (rec >> 1) / (uint32_t)a.k * 2u + (rec & 1u);
        const bool newrun = (j == 0) || kk != pk;
        const bool starts = (j == 0) ? (s == 0 || prev_key != kk) : newrun;
        SegEntry en;
        en.key = kk;
        en.rec = rec;
        en.wt = valid ? a.wts[rec] : 0.f;
        en.xrow_flags = (xrow & SF_XROW) | (newrun ? SF_NEW : 0u) | (starts ? SF_START : 0u);
        stage[wid][j] = en;
      }
    }
  }
  __syncwarp();

  float acc[EPL], gcur[EPL];
  RawSlice<YT, EPL> ycur;
  uint32_t cur = 0xffffffffu;
  bool cur_starts = false;
  const uint32_t nrows = a.nrows;
  const int64_t D = a.D;
  const XT* __restrict__ Xl = reinterpret_cast<const XT*>(a.X) + lane * EPL;
  const YT* __restrict__ Yl = reinterpret_cast<const YT*>(a.Y) + lane * EPL;
  float* __restrict__ Gl = a.G + lane * EPL;
  auto store_row = [&](float* dst, const float* v) {
    if constexpr (EPL % 4 == 0) {
#pragma unroll
      for (int i = 0; i < EPL; i += 4)
        *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < EPL; ++i) dst[i] = v[i];
    }
  };
  auto flush = [&](bool ends_here) {
    if (cur >= nrows) return;
    if (cur_starts && ends_here) {
      float t[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) t[i] = gcur[i] + acc[i];
      store_row(Gl + (int64_t)cur * D, t);
      return;
    }
    store_row((!cur_starts ? a.part_first : a.part_last) + tile * D + lane * EPL, acc);
  };
  for (int j0 = 0; j0 < cnt; j0 += U) {
    SegEntry en[U];
    RawSlice<XT, EPL> xr[U];
    RawSlice<YT, EPL> yr[MODE == MODE_DV ? U : 1];
    float gp[U][EPL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u;
      if (j < cnt) en[u] = stage[wid][j];
      else en[u] = SegEntry{0xffffffffu, 0u, 0.f, 0u};
      const bool valid = en[u].key < nrows;
      if (valid) {
        xr[u].load(Xl + (int64_t)(en[u].xrow_flags & SF_XROW) * D);
        if constexpr (MODE == MODE_DV) {
          if (en[u].xrow_flags & SF_NEW) yr[u].load(Yl + (int64_t)en[u].key * D);
        }
        if (en[u].xrow_flags & SF_START) {
          const float* g = Gl + (int64_t)en[u].key * D;
          if constexpr (EPL % 4 == 0) {
#pragma unroll
            for (int i = 0; i < EPL; i += 4) {
              const float4 t = *reinterpret_cast<const float4*>(g + i);
              gp[u][i] = t.x; gp[u][i + 1] = t.y; gp[u][i + 2] = t.z; gp[u][i + 3] = t.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < EPL; ++i) gp[u][i] = g[i];
          }
        }
      }
    }
    float d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      d[u] = 0.f;
      if (j0 + u >= cnt) continue;
      if (en[u].xrow_flags & SF_NEW) {
        flush(true);
        cur = en[u].key;
        cur_starts = (en[u].xrow_flags & SF_START) != 0;
#pragma unroll
        for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
        if (cur_starts) {
#pragma unroll
          for (int i = 0; i < EPL; ++i) gcur[i] = gp[u][i];
        }
        if constexpr (MODE == MODE_DV) ycur = yr[u];
      }
      if (cur >= nrows) continue;
      float x[EPL];
      xr[u].to_float(x);
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[i] = fmaf(en[u].wt, x[i], acc[i]);
      if constexpr (MODE == MODE_DV) {
        float y[EPL];
        ycur.to_float(y);
#pragma unroll
        for (int i = 0; i < EPL; ++i) d[u] = fmaf(y[i], x[i], d[u]);
      }
    }
    if constexpr (MODE == MODE_DV) {
      const float r = multi_warp_sum<U>(d);
      const int u = lane / (32 / U);
      if ((lane % (32 / U)) == 0) {
#pragma unroll
        for (int uu = 0; uu < U; ++uu)
          if (uu == u && j0 + uu < cnt && en[uu].key < a.nrows) a.dots[en[uu].rec] = r;
      }
    }
  }
  flush(e == a.n || next_key != cur);
}

// Runs that cross tiles: the tile where the run starts (its "last" partial)
// sums the "first" partials of the following tiles in tile order.
__global__ void __launch_bounds__(256) seg_fixup_kernel(const uint32_t* __restrict__ keys,
                                                        int64_t n, uint32_t nrows,
                                                        const float* __restrict__ part_first,
                                                        const float* __restrict__ part_last,
                                                        float* __restrict__ G, int D) {
  // one warp per tile; only tiles where a run starts and continues into the
  // next tile do work: they sum the following tiles' partials in tile order
  const int lane = threadIdx.x % 32;
  const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int64_t s = tile * SEG_T;
  if (s >= n) return;
  const int64_t e = s + SEG_T < n ? s + SEG_T : n;
  if (e >= n) return;
  const uint32_t key = keys[e - 1];
  if (key >= nrows || keys[e] != key) return;  // last run ends inside this tile
  if (keys[s] == key && s > 0 && keys[s - 1] == key) return;  // ... or started before it
  for (int c = lane; c < D; c += 32) {
    float acc = part_last[tile * D + c];
    for (int64_t u = tile + 1;; ++u) {
      acc += part_first[u * D + c];
      const int64_t us = u * SEG_T, ue = us + SEG_T < n ? us + SEG_T : n;
      if (ue >= n || keys[ue] != key || keys[ue - 1] != key) break;
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
// DENSE: instead of records, the dS of the lookup-half is written as one
// dense bf16 row dSd[b, h*2 + half, 0:n_sub] (zeros elsewhere) for the
// tensor-core dQ and dK (dk_tc.cu), and dQ is not computed here;
// n_sub <= kDenseMax.
constexpr int kDenseMax = 1024;
template <typename QT, int KPL, int EPL, bool DENSE>
__global__ void __launch_bounds__(256) ds_dq_kernel(const QT* __restrict__ K,
                                                    const int32_t* __restrict__ idx,
                                                    const float* __restrict__ w,
                                                    const float* __restrict__ dw, int64_t L,
                                                    int H, int n_sub, int d_h, int k,
                                                    float* __restrict__ dQ,
                                                    uint32_t* __restrict__ rkeys,
                                                    float* __restrict__ dsS, uint32_t sentinel,
                                                    uint16_t* __restrict__ dSd) {
  constexpr int DQ_U = EPL >= 16 ? 2 : (EPL >= 8 ? 4 : 8);
  __shared__ int32_t s_r[8][64];
  __shared__ float s_d[8][64];
  __shared__ __align__(16) uint16_t s_row[DENSE ? 8 : 1][DENSE ? kDenseMax : 8];
  const int lane = threadIdx.x % 32, wid = threadIdx.x / 32;
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
    if constexpr (!DENSE) {
#pragma unroll
      for (int u = 0; u < KPL; ++u) {
        const int t = lane + 32 * u;
        if (t < k) {
          const int64_t rec = (l * k + t) * 2 + half;
          rkeys[rec] = first[u] ? (uint32_t)((h * 2 + half) * n_sub + r[u]) : sentinel;
          dsS[rec] = dS[u];
        }
      }
    }
    // dQ: lanes over d_h.  The distinct sub-keys of this half are compacted
    // into shared memory (first-occurrence order) and their K rows are
    // loaded DQ_U at a time, all loads of a group in flight together.
    int m = 0;
#pragma unroll
    for (int u = 0; u < KPL; ++u) {
      const int t = lane + 32 * u;
      const bool fl = t < k && first[u];
      const unsigned bm = __ballot_sync(0xffffffffu, fl);
      if (fl) {
        const int pos = m + __popc(bm & ((1u << lane) - 1u));
        s_r[wid][pos] = r[u];
        s_d[wid][pos] = dS[u];
      }
      m += __popc(bm);
    }
    __syncwarp();
    if constexpr (DENSE) {
      // dense row: zero, place the m distinct values, copy out (16 B per lane)
      uint4* row4 = reinterpret_cast<uint4*>(s_row[wid]);
      const int n16 = n_sub / 8;
      for (int c = lane; c < n16; c += 32) row4[c] = make_uint4(0, 0, 0, 0);
      __syncwarp();
      for (int c = lane; c < m; c += 32)
        s_row[wid][s_r[wid][c]] = __bfloat16_as_ushort(__float2bfloat16_rn(s_d[wid][c]));
      __syncwarp();
      uint4* g4 = reinterpret_cast<uint4*>(dSd + (l * 2 + half) * (int64_t)n_sub);
      for (int c = lane; c < n16; c += 32) g4[c] = row4[c];
    }
    if constexpr (DENSE) {
      __syncwarp();
      continue;  // dQ = dSd . K runs on the tensor cores (dk_tc.cu)
    }
    float acc[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
    const QT* Kh = K + (int64_t)(h * 2 + half) * n_sub * d_h + lane * EPL;
    for (int b0 = 0; b0 < m; b0 += DQ_U) {
      float kr[DQ_U][EPL];
#pragma unroll
      for (int u = 0; u < DQ_U; ++u)
        if (b0 + u < m) load_slice<QT, EPL>(Kh + (int64_t)s_r[wid][b0 + u] * d_h, kr[u]);
#pragma unroll
      for (int u = 0; u < DQ_U; ++u)
        if (b0 + u < m) {
          const float dSv = s_d[wid][b0 + u];
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[i] = fmaf(dSv, kr[u][i], acc[i]);
        }
    }
    __syncwarp();
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
  b += align256(sizeof(uint32_t) * ((int64_t(1) << 20) + (int64_t(1) << RS_MAX_BITS) * 0 + 1024 + 2048 * nblocks));
  b += 2 * align256(sizeof(float) * tiles * D);
  b += align256(sizeof(float) * n_dk);
  b += align256(sizeof(float) * n_dv);
  b += align256(dk_tc_workspace_bytes(s));
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
  w.hist = (uint32_t*)p; p += align256(sizeof(uint32_t) * ((int64_t(1) << 20) + (int64_t(1) << RS_MAX_BITS) * 0 + 1024 + 2048 * nblocks));
  w.part_first = (float*)p; p += align256(sizeof(float) * tiles * D);
  w.part_last = (float*)p; p += align256(sizeof(float) * tiles * D);
  w.dsS = (float*)p; p += align256(sizeof(float) * n_dk);
  w.dw = (float*)p; p += align256(sizeof(float) * n_dv);
  w.dk_ws = (void*)p; p += align256(dk_tc_workspace_bytes(s));
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
  const bool dense = dk_tc_supported(s);
#define DSDQ(QT, KPL, E_)                                                                      \
  if (dense)                                                                                   \
    ds_dq_kernel<QT, KPL, E_, true><<<blocks, 256, 0, st>>>(                                   \
        (const QT*)K, idx, w, dw, L, s.H, s.n_sub, s.d_h, s.k, dQ, ws.keys_a, ws.dsS, nrows,    \
        (uint16_t*)ws.dk_ws);                                                                  \
  else                                                                                         \
    ds_dq_kernel<QT, KPL, E_, false><<<blocks, 256, 0, st>>>(                                  \
        (const QT*)K, idx, w, dw, L, s.H, s.n_sub, s.d_h, s.k, dQ, ws.keys_a, ws.dsS, nrows,    \
        nullptr)
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
  if (dense) return launch_dk_tc(s, Q, K, dQ, dK, ws.dk_ws, st, launches);
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
