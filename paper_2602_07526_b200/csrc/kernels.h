// kernels.h -- internal launcher interface between the C-ABI host code
// (api.cu) and the kernels.  Not part of the public ABI (include/msn_pkm.h).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace msn {

enum Dt { F32 = 0, BF16 = 1 };

// Per-rank pointers of the row-sharded exchange (a9), passed by value in the
// kernel parameters (graph-capturable, no device pointer arrays).
constexpr int kMaxWorld = 8;
template <typename T>
struct PerRank {
  T* p[kMaxWorld];
};

struct Shape {
  int64_t B;       // queries in this call
  int H, n_sub, d_h, d_v, k;
  int qk_dt, v_dt;
  int64_t row_begin, row_end;  // local value rows
  int og = 1;                  // output head groups: out [B, og, d_v]
  int64_t tab_stride = 0;      // per-group tables: group g's rows start at g * tab_stride
  bool dq_bf16 = false;        // d_query written in bf16 (MSN_FLAG_DQ_QK_DTYPE, bf16 configs)
};

// Per-half candidate lists, the hand-off between a1+a2 and a3: for every
// (b, h, half) row r and column segment g, the list vc[(r*SC + g)*cap ...] of
// cap = cand_cap(KT) (score bits, sub-key index) pairs holds, in no particular
// order, a superset of the segment's top-k under (score desc, index asc):
// entries [0, n0) and [cap - n1, cap) with n[r*SC + g] = n0 | n1 << 16 (the
// tcgen05 scorer writes compact lists, n1 = 0).  n0 + n1 <= cap always: a row
// whose bound let more columns through (massive exact ties) is rescored
// exactly from the query and sub-keys in `rq` into [0, nn).
__host__ __device__ constexpr int cand_cap(int kt) { return kt > 32 ? 128 : 64; }
struct Rescore {
  const void* Q = nullptr;  // [B, H, 2, d_h] qk dtype
  const void* K = nullptr;  // [H, 2, n_sub, d_h] qk dtype
  int d_h = 0;
  int qk_dt = 0;
};
struct Cands {
  uint2* vc;     // [B*H*2, SC, cap] (float bits of the score, sub-key index)
  int32_t* n;    // [B*H*2, SC]: n0 | n1 << 16 per column segment's list
  Rescore rq;    // inputs, for rescoring overflowed rows
  int SC = 1;    // segment slots per row in the buffers (workspace layout)
  int S = 1;     // column segments in use (<= SC): the tcgen05 scorer splits a
                 // row over S CTAs, each writing the list of its columns
  int cap = 64;  // list capacity, cand_cap(KT)
};

// a1+a2 on tcgen05: fused scoring GEMM + candidate selection (the only
// scorer).  Returns cudaErrorNotSupported when the shape is not handled.
// fp32 inputs run 3xTF32 (kind::tf32); ws holds the split sub-keys
// (select_tc_workspace_bytes).
// Column segments of a scorer row (bf16, k <= 32, n_sub <= 1024): the largest
// S in {4, 2} with n_sub / S >= 256 columns (a multiple of the N tile) whose
// S x (the unsplit grid) still fits one wave of CTAs (the latency regime,
// e.g. C5: 32 CTAs -> S = 4), else 1.  MSN_SELECT_SPLIT=S forces it (A/B,
// tests).  The workspace layout uses the same S (SC == S).
constexpr int kMaxSeg = 4;
int select_segments(const Shape& s, bool for_workspace);
int select_cap(const Shape& s);  // candidate list capacity (64, or 128 for k > 32)
// qhat (f2, may be null): LayerNorm each query half-vector on load (no affine,
// eps 1e-5) and write q^ [B, H, 2, d_h] (query dtype) there; the exact
// rescoring of overflowed rows then reads cd.rq.Q = qhat.
cudaError_t launch_select_tc(const Shape& s, const void* Q, const void* K, const Cands& cd,
                             void* ws, cudaStream_t st, int* launches, void* qhat = nullptr);
bool select_tc_supported(const Shape& s);  // shape check only (no driver call)
size_t select_tc_workspace_bytes(const Shape& s);

// Memory-gated fusion: x~ = x (.) g(v_o), applied in the
// epilogue of the kernel that produces v_o (kind 0: none).
struct Gate {
  const float* x = nullptr;  // [B, d_v]
  float* xt = nullptr;       // [B, d_v]
  int kind = 0;              // 1 tanh, 2 sigmoid, 3 identity
};

// a2 (ordering) + a3 + a4: per-half top-k from the candidate lists, Cartesian
// top-k over I x J + softmax.  idx/w [B,H,k].
cudaError_t launch_cartesian(const Shape& s, const Cands& cd, int32_t* idx, float* w,
                             cudaStream_t st, int* launches);

// a2 (ordering) + a3 + a4 + a5 fused (unsharded forward): Cartesian stage of
// each query's H lookups, then the gather of their H*k rows.
cudaError_t launch_cartesian_gather(const Shape& s, const Cands& cd, int32_t* idx, float* w,
                                    const void* V, float* out, cudaStream_t st, int* launches,
                                    const Gate& gate = Gate{});

// a2 (ordering) + a3 + a4 + a5 fused per lookup (small batches): one warp per
// lookup, the block's H partials added per query in head order.
bool cartesian_gather_lookup_ok(const Shape& s);
cudaError_t launch_cartesian_gather_lookup(const Shape& s, const Cands& cd, int32_t* idx, float* w, const void* V,
                                          float* out, cudaStream_t st, int* launches);

// a5: out[b] = sum over local rows of w * V[idx - row_begin] (=).
cudaError_t launch_gather(const Shape& s, const int32_t* idx, const float* w, const void* V,
                          float* out, cudaStream_t st, int* launches, const Gate& gate = Gate{});

// out[b, g] = sum_p recv[p][b][g] in rank order (=).
cudaError_t launch_reduce_partials(const float* recv, int world, int64_t lb, int og, int d_v,
                                   float* out, cudaStream_t st, int* launches);

// f1 backward: dx = dxt (.) g(v_o) (=), dvo = dxt (.) x (.) g'(v_o) (=).
// validate.cu: *bad = number of invalid tape slots (range, duplicates, weight
// not in [0, 1]); zeroes *bad first.
cudaError_t launch_validate_tape(const Shape& s, const int32_t* idx, const float* w, int32_t* bad,
                                 cudaStream_t st, int* launches);
cudaError_t launch_gate_backward(int64_t B, int d_v, int kind, const float* x, const float* vo,
                                 const float* dxt, float* dx, float* dvo, cudaStream_t st,
                                 int* launches);

// ---- backward ----
struct BwdWorkspace {
  uint32_t *cnt, *off;            // per-row counts / segment offsets (grouping)
  uint32_t *rank, *keys;          // per-contribution rank, row key
  uint2* ent;                     // grouped (record id, weight bits) pairs
  uint4 *runs_short, *runs_long;  // run records {offset, length, row, first piece}
  uint4* pieces;                  // long-run slices {first entry, entries, row, long run}
  float* part;                    // piece partial rows
  uint32_t* ctl;                  // grouping counters
  uint32_t* huge;                 // long runs sorted by a CTA
  float* dsS;                     // 2*B*H*k aggregated score grads
  float* dw;                      // B*H*k (when the caller gives none)
  void* dk_ws;                    // tensor-core dQ/dK scratch (bf16 configs)
};

// Host-side shape check of the backward, made before anything is launched:
// the value reducers need d_v (values), the key path d_h (keys), each in
// 32 * {1, 2, 4, 8, 16}, and k <= 64.
bool backward_supported(const Shape& s, bool values, bool keys);

// a7 dQ + a8 dK on the tensor cores (bf16 q/K): dQ = dS . K, dK += dS^T . Q per (head, half).
bool dk_tc_supported(const Shape& s);
// sub-key rows per dK CTA tile (128 x tiles per CTA); the compact dS records
// carry per-tile offsets for it
int dk_tile_rows(const Shape& s);
size_t dk_tc_workspace_bytes(const Shape& s);
// ws starts with the dense bf16 score-gradient matrix dSd [B, H*2, n_sub]
// that ds_dq_kernel writes (dense mode).
// Also writes dQ = dSd . K (=) on the tensor cores.
cudaError_t launch_dk_tc(const Shape& s, const void* Q, const void* K, float* dQ, float* dK,
                         void* ws, cudaStream_t st, int* launches, bool with_dq = true);
// dQ on the tensor cores too (dense dS . K), or by ds_dq_kernel from the m
// distinct K rows of each lookup-half: the dense GEMM's work grows with n_sub.
bool dq_tc_wanted(const Shape& s);
// dK from the compact records (else from the dense bf16 dS matrix)
bool dk_compact(const Shape& s);
// with compact records: dQ on the tensor cores too, its dS tiles built in
// shared memory from the records (else the SIMT dQ of ds_dq_kernel)
bool dq_rec_wanted(const Shape& s);
size_t bwd_workspace_bytes(const Shape& s, int64_t gather_batch);
BwdWorkspace carve_bwd_workspace(const Shape& s, int64_t gather_batch, void* ws);

// Optional profiling events recorded around an internal stage.
struct TraceEvents {
  const cudaEvent_t* ev = nullptr;
  int n = 0;
};

// Row-sharded backward over peer memory: the d_out rows of query b are read
// from rank b / local_batch's buffer d_out[rank] ([local_batch, og, d_v]) and
// dw of record (b, h, t) is written into rank b / local_batch's dw[rank]
// ([local_batch, H, k]); each dw element has exactly one owner rank.
struct ScatterPeers {
  PerRank<const float> d_out{};  // rank p's [local_batch, og, d_v] rows
  PerRank<float> dw{};           // rank p's dw destination (pre-offset)
  int64_t local_batch = 0;
  bool p2p = true;               // false: x rows / dw in the local X / dots arrays
  int64_t cap = 0;               // dw destination segment per rank (0: local_batch H k)
};

// a6 deterministic: group (idx -> cid) by row, then fused row-major dV += / dw.
// tr: events around the short-run reducer (profiling only).
// upd: 0 -> dV += g; 1 -> SGD, 2 -> Adagrad applied to V in
// place (dV unused; state = the Adagrad accumulator [rows, d_v]).
cudaError_t launch_scatter_sorted(const Shape& s, const int32_t* idx, const float* w,
                                  const float* dOut, const void* V, float* dV, float* dw,
                                  const BwdWorkspace& ws, cudaStream_t st, int* launches,
                                  const TraceEvents& tr = TraceEvents{}, int upd = 0,
                                  float lr = 0.f, float eps = 0.f, float* state = nullptr,
                                  const ScatterPeers* peers = nullptr);
// a6 atomic: query-major re-gather + red.global.add.v4.f32.
cudaError_t launch_scatter_atomic(const Shape& s, const int32_t* idx, const float* w,
                                  const float* dOut, const void* V, float* dV, float* dw,
                                  cudaStream_t st, int* launches);
// a7+a8: ds, dQ (=), dK (+=) deterministic.
cudaError_t launch_backward_keys(const Shape& s, const void* Q, const void* K,
                                 const int32_t* idx, const float* w, const float* dw, float* dQ,
                                 float* dK, const BwdWorkspace& ws, cudaStream_t st,
                                 int* launches);

// ---- a9 record exchange of the row-sharded table (exchange.cu) ----
// a2-a4 + ROUTE + the local shard's a5, fused (cartesian.cu): one warp per
// local query runs the Cartesian stage of its H lookups (idx / w, the tape),
// writes every slot as a record {local row, w} into its owner's window
// row.p[o] / w.p[o] + b H k (in (h, t) order; cnt.p[o][b] = the count,
// pos[b H k + r] = the slot's place in the window) and gathers the slots this
// rank owns into part + b d_v.
struct RouteArgs {
  int P = 1, rank = 0;
  int64_t rpr = 0;          // value rows per rank (n / P)
  PerRank<int32_t> row{}, cnt{};
  PerRank<float> w{};
  int32_t* pos = nullptr;   // [B_l * H * k]
  float* part = nullptr;    // [B_l, d_v] the local shard's partial sums
};
cudaError_t launch_cartesian_route(const Shape& s, const Cands& cd, int32_t* idx, float* w, const void* V,
                                   const RouteArgs& r, cudaStream_t st, int* launches);
// The owner's view of the records it received: window (s, b) holds
// cnt[s * lb + b] records at s * cap + b * HK (cap = lb * HK).
struct RecordsIn {
  int P = 1, rank = 0;
  int64_t lb = 0, cap = 0;
  int HK = 0;
  const int32_t *row = nullptr, *cnt = nullptr;
  const float* w = nullptr;
};
// partial of remote source s's query b -> dst.p[s] + b * d_v (pre-offset per source)
cudaError_t launch_gather_records(const Shape& s, const RecordsIn& r, const void* V,
                                  const PerRank<float>& dst, cudaStream_t st, int* launches);
// dV (+=) and dw of the records; d_out row of (s, b) at x_src.p[s] + b * d_v,
// dw of the record at window position i of source s -> dw_dst.p[s] + i.
cudaError_t launch_scatter_records(const Shape& s, const RecordsIn& r, const PerRank<const float>& x_src,
                                   const void* V, float* dV, const PerRank<float>& dw_dst,
                                   const BwdWorkspace& ws, cudaStream_t st, int* launches,
                                   const TraceEvents& tr);
// dw[b,h,t] = dw_in[owner * cap + b * H * k + pos[b,h,t]]
cudaError_t launch_collect_dw(const Shape& s, const int32_t* idx, const int32_t* pos, const float* dw_in,
                              int64_t cap, int64_t rpr, float* dw, cudaStream_t st, int* launches);
// device barrier: flags.p[o] = rank o's CTL flag array, ctl = own CTL words
cudaError_t launch_exchange_barrier(int P, int rank, const PerRank<uint32_t>& flags, uint32_t* ctl,
                                    cudaStream_t st, int* launches);

// ---- prologue (prologue.cu) ----
bool prologue_supported(const Shape& s);
// LayerNorm of `rows` rows of width d_h (qk dtype): y = LN(x); with dy given,
// the backward dx (fp32, =) instead.
cudaError_t launch_layernorm(const Shape& s, int64_t rows, const void* x, void* y, const float* dy,
                             float* dx, cudaStream_t st, int* launches);
// K~ = K^ Theta^T per codebook (qk dtype in and out, Theta fp32 [2H, d, d]).
cudaError_t launch_key_transform(const Shape& s, const void* khat, const float* theta, void* keff,
                                 cudaStream_t st, int* launches);
// dK^ = dK~ Theta (=), dTheta += dK~^T K^ (fp32).
cudaError_t launch_key_transform_backward(const Shape& s, const void* khat, const float* theta,
                                          const float* dkeff, float* dkhat, float* dtheta,
                                          cudaStream_t st, int* launches);

}  // namespace msn
