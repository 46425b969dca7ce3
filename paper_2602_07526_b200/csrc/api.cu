// api.cu -- the C ABI declared in include/msn_pkm.h: validation, workspace
// carving and launch orchestration on the caller's stream.  No device
// allocation, no host synchronisation (except under MSN_FLAG_VALIDATE: one
// 4-byte flag word per handle, and a stream sync per tape check).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/msn_pkm.h"
#include "kernels.h"

using namespace msn;

struct msn_pkm {
  msn_pkm_config cfg;
  int last_launches;
  cudaEvent_t trace[4];  // optional stage-boundary events (msn_pkm_set_trace_events)
  int ntrace;
  int32_t* d_bad;  // MSN_FLAG_VALIDATE only: device word + pinned host copy
  int32_t* h_bad;
};

namespace {

thread_local std::string g_err;

msn_status fail(msn_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

msn_status cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaErrorNotSupported)
    return fail(MSN_ERR_UNSUPPORTED, "%s: shape not supported by this build", what);
  return fail(MSN_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

Shape shape_of(const msn_pkm_config& c, int64_t B) {
  Shape s;
  s.B = B;
  s.H = c.heads;
  s.n_sub = c.n_sub;
  s.d_h = c.d_half;
  s.d_v = c.d_value;
  s.k = c.k;
  s.qk_dt = c.qk_dtype;
  s.v_dt = c.value_dtype;
  s.row_begin = c.row_begin;
  s.row_end = c.row_end;
  s.og = c.head_groups > 1 ? c.head_groups : 1;
  s.tab_stride = (c.flags & MSN_FLAG_GROUP_TABLES) ? (int64_t)c.n_sub * c.n_sub : 0;
  s.dq_bf16 = (c.flags & MSN_FLAG_DQ_QK_DTYPE) && c.qk_dtype == MSN_BF16;
  return s;
}

// forward workspace layout: [cand (score, index) | cand_n | split sub-keys (3xTF32)]
size_t fwd_bytes(const Shape& s) {
  const int64_t rows = s.B * s.H * 2 * select_segments(s, true);  // (row, column segment) lists
  size_t b = align256(sizeof(uint2) * rows * select_cap(s)) + align256(sizeof(int32_t) * rows);
  b += align256(select_tc_workspace_bytes(s));
  return b;
}

// the candidate lists at the start of the forward workspace; returns the rest
char* carve_cands(const Shape& s, void* ws, Cands& cd) {
  cd.SC = select_segments(s, true);
  cd.S = select_segments(s, false);
  cd.cap = select_cap(s);
  const int64_t rows = s.B * s.H * 2 * cd.SC;
  char* p = (char*)ws;
  cd.vc = (uint2*)p;
  p += align256(sizeof(uint2) * rows * cd.cap);
  cd.n = (int32_t*)p;
  p += align256(sizeof(int32_t) * rows);
  return p;
}

// The scorer (a1-a2) is the tcgen05 kernel only: other shapes are refused on
// the host before anything is launched.
msn_status check_select_shape(const Shape& s) {
  if (select_tc_supported(s)) return MSN_OK;
  return fail(MSN_ERR_UNSUPPORTED,
              "the tcgen05 scorer needs n_sub %% 32 == 0, d_half %% 64 == 0 and <= 256 (bf16) or "
              "%% 32 == 0 and <= 128 (fp32), k <= 64 (n_sub %d, d_half %d, k %d); nothing was launched",
              s.n_sub, s.d_h, s.k);
}

msn_status check_bwd_shape(msn_pkm_t h, bool values, bool keys) {
  if (backward_supported(shape_of(h->cfg, 0), values, keys)) return MSN_OK;
  return fail(MSN_ERR_UNSUPPORTED,
              "backward needs d_value (%d) in 32 * {1, 2, 4, 8, 16, 32}, d_half (%d) in 32 * {1, 2, 4, 8, 16} and k <= 64; "
              "nothing was launched", h->cfg.d_value, h->cfg.d_half);
}

msn_status check_handle(msn_pkm_t h) {
  if (!h) return fail(MSN_ERR_INVALID_ARG, "null handle");
  return MSN_OK;
}

msn_status check_batch(msn_pkm_t h, int64_t B) {
  if (B < 0) return fail(MSN_ERR_INVALID_ARG, "B = %lld < 0", (long long)B);
  if (B > h->cfg.max_batch)
    return fail(MSN_ERR_INVALID_ARG, "B = %lld > max_batch = %lld", (long long)B,
                (long long)h->cfg.max_batch);
  return MSN_OK;
}

#define REQUIRE_PTR(p)                                                                       \
  do {                                                                                       \
    if (!(p)) return fail(MSN_ERR_INVALID_ARG, "%s is NULL", #p);                            \
    if (!aligned16(p)) return fail(MSN_ERR_INVALID_ARG, "%s is not 16-byte aligned", #p);   \
  } while (0)

// MSN_FLAG_VALIDATE: check the tape, synchronise, refuse an invalid one.
msn_status check_tape(msn_pkm_t h, void* stream, int64_t B, const int32_t* idx, const float* w) {
  if (!(h->cfg.flags & MSN_FLAG_VALIDATE) || B == 0) return MSN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = launch_validate_tape(shape_of(h->cfg, B), idx, w, h->d_bad, st, nullptr);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h->h_bad, h->d_bad, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "tape validation");
  if (*h->h_bad)
    return fail(MSN_ERR_INVALID_ARG,
                "tape: %d invalid slots (idx outside the table, repeated in a lookup, or weight not in [0, 1])",
                *h->h_bad);
  return MSN_OK;
}

// a1 + a2 into per-half candidate lists; then either the Cartesian stage
// alone (select) or fused with the gather (forward: values != NULL).
msn_status do_select(msn_pkm_t h, cudaStream_t st, int64_t B, const void* query,
                     const void* subkeys, int32_t* idx, float* weights, void* ws, size_t ws_bytes,
                     int* launches, const void* values = nullptr, float* out = nullptr,
                     const Gate& gate = Gate{}, bool per_lookup = false, void* qhat = nullptr) {
  const Shape s = shape_of(h->cfg, B);
  msn_status st0 = check_select_shape(s);
  if (st0) return st0;
  if (ws_bytes < fwd_bytes(s))
    return fail(MSN_ERR_WORKSPACE, "forward workspace %zu < %zu bytes", ws_bytes, fwd_bytes(s));
  Cands cd;
  char* p = carve_cands(s, ws, cd);
  cd.rq.Q = qhat ? qhat : query;  // (the exact rescoring scores the normalised query)
  cd.rq.K = subkeys;
  cd.rq.d_h = s.d_h;
  cd.rq.qk_dt = s.qk_dt;
  cudaError_t e = launch_select_tc(s, query, subkeys, cd, p, st, launches, qhat);
  if (e != cudaSuccess) return cuda_fail(e, "select (tcgen05 scoring + per-half candidates)");
  if (h->ntrace > 0) cudaEventRecord(h->trace[0], st);  // stage boundary: scoring done
  if (values && per_lookup) {  // small batches: Cartesian + gather fused per lookup
    if (h->ntrace > 1) cudaEventRecord(h->trace[1], st);
    e = launch_cartesian_gather_lookup(s, cd, idx, weights, values, out, st, launches);
    if (e != cudaSuccess) return cuda_fail(e, "cartesian top-k + softmax + gather (per lookup)");
    return MSN_OK;
  }
  if (values && cd.S == 1) {
    if (h->ntrace > 1) cudaEventRecord(h->trace[1], st);  // (fused: no separate Cartesian stage)
    e = launch_cartesian_gather(s, cd, idx, weights, values, out, st, launches, gate);
    if (e != cudaSuccess) return cuda_fail(e, "cartesian top-k + softmax + gather");
    return MSN_OK;
  }
  if (values) {  // column-segmented scorer rows: Cartesian stage, then the gather
    e = launch_cartesian(s, cd, idx, weights, st, launches);
    if (e != cudaSuccess) return cuda_fail(e, "cartesian top-k + softmax");
    if (h->ntrace > 1) cudaEventRecord(h->trace[1], st);
    e = launch_gather(s, idx, weights, values, out, st, launches, gate);
    if (e != cudaSuccess) return cuda_fail(e, "gather");
    return MSN_OK;
  }
  e = launch_cartesian(s, cd, idx, weights, st, launches);
  if (e != cudaSuccess) return cuda_fail(e, "cartesian top-k + softmax");
  if (h->ntrace > 1) cudaEventRecord(h->trace[1], st);  // stage boundary: Cartesian + softmax done
  return MSN_OK;
}

}  // namespace

extern "C" {

const char* msn_pkm_status_string(msn_status s) {
  switch (s) {
    case MSN_OK: return "ok";
    case MSN_ERR_INVALID_ARG: return "invalid argument";
    case MSN_ERR_UNSUPPORTED: return "unsupported";
    case MSN_ERR_CUDA: return "cuda error";
    case MSN_ERR_WORKSPACE: return "workspace too small";
    case MSN_ERR_INTERNAL: return "internal error";
  }
  return "unknown status";
}

const char* msn_pkm_last_error(void) { return g_err.c_str(); }

msn_status msn_pkm_create(const msn_pkm_config* c, msn_pkm_t* out) {
  if (!c || !out) return fail(MSN_ERR_INVALID_ARG, "null config or output pointer");
  *out = nullptr;
  if (c->abi_version != MSN_PKM_ABI_VERSION)
    return fail(MSN_ERR_INVALID_ARG, "abi_version %d != %d", c->abi_version, MSN_PKM_ABI_VERSION);
  if (c->heads < 1) return fail(MSN_ERR_INVALID_ARG, "heads must be >= 1");
  if (c->n_sub < 1 || (int64_t)c->n_sub * c->n_sub >= (int64_t(1) << 31))
    return fail(MSN_ERR_INVALID_ARG, "n_sub must satisfy 1 <= n_sub and n_sub^2 < 2^31");
  if (c->k < 1 || c->k > c->n_sub) return fail(MSN_ERR_INVALID_ARG, "need 1 <= k <= n_sub");
  if (c->k > 64) return fail(MSN_ERR_UNSUPPORTED, "k > 64 is not supported (Table 2 max is 64)");
  if (c->d_half < 16 || c->d_half % 16) return fail(MSN_ERR_INVALID_ARG, "d_half %% 16 != 0");
  if (c->qk_dtype != MSN_F32 && c->qk_dtype != MSN_BF16)
    return fail(MSN_ERR_INVALID_ARG, "qk_dtype must be MSN_F32 or MSN_BF16");
  if (c->value_dtype != MSN_F32 && c->value_dtype != MSN_BF16)
    return fail(MSN_ERR_INVALID_ARG, "value_dtype must be MSN_F32 or MSN_BF16");
  const int vsz = c->value_dtype == MSN_F32 ? 4 : 2;
  if (c->d_value < 1 || (c->d_value * vsz) % 16)
    return fail(MSN_ERR_INVALID_ARG, "d_value * sizeof(value) must be a multiple of 16 bytes");
  if (c->max_batch < 0) return fail(MSN_ERR_INVALID_ARG, "max_batch < 0");
  if (c->flags &
      ~(MSN_FLAG_ATOMIC_BWD | MSN_FLAG_GROUP_TABLES | MSN_FLAG_DQ_QK_DTYPE | MSN_FLAG_VALIDATE))
    return fail(MSN_ERR_INVALID_ARG, "unknown flags");
  const int G = c->head_groups > 1 ? c->head_groups : 1;
  if (c->head_groups < 0 || c->heads % G)
    return fail(MSN_ERR_INVALID_ARG, "head_groups must be >= 0 and divide heads");
  const int64_t n = (int64_t)c->n_sub * c->n_sub * ((c->flags & MSN_FLAG_GROUP_TABLES) ? G : 1);
  if (n >= (int64_t(1) << 31)) return fail(MSN_ERR_INVALID_ARG, "table rows must be < 2^31");
  if (c->world_size < 0 || c->world_size > MSN_MAX_WORLD)
    return fail(MSN_ERR_INVALID_ARG, "world_size %d not in [0, %d]", c->world_size, MSN_MAX_WORLD);
  if (c->rank < 0 || c->rank >= (c->world_size > 1 ? c->world_size : 1))
    return fail(MSN_ERR_INVALID_ARG, "rank %d outside [0, world_size)", c->rank);
  msn_pkm_config cc = *c;
  if (c->world_size > 1) {  // the row-sharded table: rank r owns rows [r n/P, (r+1) n/P)
    if (n % c->world_size)
      return fail(MSN_ERR_INVALID_ARG, "table rows %lld not divisible by world_size %d", (long long)n,
                  c->world_size);
    if (G > 1) return fail(MSN_ERR_UNSUPPORTED, "head groups need the unsharded table");
    const int64_t rpr = n / c->world_size;
    if (!(c->row_begin == 0 && c->row_end == 0) &&
        !(c->row_begin == c->rank * rpr && c->row_end == (c->rank + 1) * rpr))
      return fail(MSN_ERR_INVALID_ARG, "row_begin/row_end must be 0/0 or rank's rows [%lld, %lld)",
                  (long long)(c->rank * rpr), (long long)((c->rank + 1) * rpr));
    cc.row_begin = c->rank * rpr;
    cc.row_end = (c->rank + 1) * rpr;
  }
  c = &cc;
  if (c->row_begin < 0 || c->row_end > n || c->row_begin >= c->row_end)
    return fail(MSN_ERR_INVALID_ARG, "need 0 <= row_begin < row_end <= table rows");
  if (G > 1 && (c->row_begin != 0 || c->row_end != n))
    return fail(MSN_ERR_UNSUPPORTED, "head groups need the unsharded table");
  if (G > 1 && (c->flags & MSN_FLAG_ATOMIC_BWD))
    return fail(MSN_ERR_UNSUPPORTED, "head groups need the deterministic backward");
  if (c->n_sub > 2048) return fail(MSN_ERR_UNSUPPORTED, "n_sub > 2048 is not supported");

  msn_pkm* h = new (std::nothrow) msn_pkm;
  if (!h) return fail(MSN_ERR_INTERNAL, "out of host memory");
  h->cfg = *c;
  h->last_launches = 0;
  h->ntrace = 0;
  h->d_bad = nullptr;
  h->h_bad = nullptr;
  if (c->flags & MSN_FLAG_VALIDATE) {
    cudaError_t e = cudaMalloc(&h->d_bad, sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMallocHost(&h->h_bad, sizeof(int32_t));
    if (e != cudaSuccess) {
      msn_pkm_destroy(h);
      return cuda_fail(e, "MSN_FLAG_VALIDATE flag word");
    }
  }
  *out = h;
  return MSN_OK;
}

msn_status msn_pkm_destroy(msn_pkm_t h) {
  if (h && h->d_bad) cudaFree(h->d_bad);
  if (h && h->h_bad) cudaFreeHost(h->h_bad);
  delete h;
  return MSN_OK;
}

int32_t msn_pkm_last_launch_count(msn_pkm_t h) { return h ? h->last_launches : -1; }

msn_status msn_pkm_set_trace_events(msn_pkm_t h, void* const* events, int32_t n) {
  msn_status st = check_handle(h);
  if (st) return st;
  if (n < 0 || n > 4 || (n > 0 && !events)) return fail(MSN_ERR_INVALID_ARG, "0 <= n <= 4 events");
  for (int i = 0; i < n; ++i) h->trace[i] = (cudaEvent_t)events[i];
  h->ntrace = n;
  return MSN_OK;
}

msn_status msn_pkm_workspace_size(msn_pkm_t h, int64_t B, int64_t gather_batch, size_t* fwd,
                                  size_t* bwd) {
  msn_status st = check_handle(h);
  if (st) return st;
  if ((st = check_batch(h, B))) return st;
  if (gather_batch < B) return fail(MSN_ERR_INVALID_ARG, "gather_batch < B");
  const Shape s = shape_of(h->cfg, B);
  if (fwd) *fwd = fwd_bytes(s);
  if (bwd) *bwd = bwd_workspace_bytes(s, gather_batch);
  return MSN_OK;
}

msn_status msn_pkm_select(msn_pkm_t h, void* stream, int64_t B, const void* query,
                          const void* subkeys, int32_t* idx, float* weights, void* workspace,
                          size_t workspace_bytes) {
  msn_status st = check_handle(h);
  if (st) return st;
  if ((st = check_batch(h, B))) return st;
  h->last_launches = 0;
  if (B == 0) return MSN_OK;
  REQUIRE_PTR(query);
  REQUIRE_PTR(subkeys);
  REQUIRE_PTR(idx);
  REQUIRE_PTR(weights);
  REQUIRE_PTR(workspace);
  return do_select(h, (cudaStream_t)stream, B, query, subkeys, idx, weights, workspace,
                   workspace_bytes, &h->last_launches);
}

msn_status msn_pkm_gather(msn_pkm_t h, void* stream, int64_t B, const int32_t* idx,
                          const float* weights, const void* values, float* out) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  if (B < 0) return fail(MSN_ERR_INVALID_ARG, "B < 0");
  if (B == 0) return MSN_OK;
  REQUIRE_PTR(idx);
  REQUIRE_PTR(weights);
  REQUIRE_PTR(values);
  REQUIRE_PTR(out);
  if ((st = check_tape(h, stream, B, idx, weights))) return st;
  const Shape s = shape_of(h->cfg, B);
  cudaError_t e = launch_gather(s, idx, weights, values, out, (cudaStream_t)stream,
                                &h->last_launches);
  if (e != cudaSuccess) return cuda_fail(e, "gather");
  return MSN_OK;
}

msn_status msn_pkm_validate_tape(msn_pkm_t h, void* stream, int64_t B, const int32_t* idx,
                                 const float* weights, int32_t* bad) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  if (B < 0) return fail(MSN_ERR_INVALID_ARG, "B < 0");
  if (!bad) return fail(MSN_ERR_INVALID_ARG, "bad is NULL");
  if (B > 0) {
    REQUIRE_PTR(idx);
    REQUIRE_PTR(weights);
  }
  cudaError_t e = launch_validate_tape(shape_of(h->cfg, B), idx, weights, bad, (cudaStream_t)stream,
                                       &h->last_launches);
  if (e != cudaSuccess) return cuda_fail(e, "validate_tape");
  return MSN_OK;
}

static msn_status do_forward(msn_pkm_t h, void* stream, int64_t B, const void* query,
                             const void* subkeys, const void* values, float* out, int32_t* idx,
                             float* weights, void* workspace, size_t workspace_bytes,
                             const Gate& gate, void* qhat = nullptr) {
  msn_status st = check_handle(h);
  if (st) return st;
  if ((st = check_batch(h, B))) return st;
  h->last_launches = 0;
  if (B == 0) return MSN_OK;
  const Shape s0 = shape_of(h->cfg, 0);
  const int64_t n = (int64_t)h->cfg.n_sub * h->cfg.n_sub * (s0.tab_stride ? s0.og : 1);
  if (h->cfg.row_begin != 0 || h->cfg.row_end != n)
    return fail(MSN_ERR_INVALID_ARG, "msn_pkm_forward needs the whole table; use the phase calls when sharded");
  REQUIRE_PTR(query);
  REQUIRE_PTR(subkeys);
  REQUIRE_PTR(values);
  REQUIRE_PTR(out);
  REQUIRE_PTR(idx);
  REQUIRE_PTR(weights);
  REQUIRE_PTR(workspace);
  cudaStream_t cs = (cudaStream_t)stream;
  // fused Cartesian + gather when there are enough queries to fill the GPU
  // with warps (one warp per query); small batches keep one warp per lookup
  static const int64_t fuse_min_b = getenv("MSN_FUSE_MIN_B") ? atoll(getenv("MSN_FUSE_MIN_B")) : 8192;
  if (h->cfg.heads * h->cfg.k <= 256 && B >= fuse_min_b) {
    return do_select(h, cs, B, query, subkeys, idx, weights, workspace, workspace_bytes,
                     &h->last_launches, values, out, gate, false, qhat);
  }
  // smaller batches: Cartesian + gather fused per lookup (8x the warps of
  // the per-query kernel), unless a gate or head groups ask for the phases
  if (!gate.kind && cartesian_gather_lookup_ok(shape_of(h->cfg, B)))
    return do_select(h, cs, B, query, subkeys, idx, weights, workspace, workspace_bytes, &h->last_launches,
                     values, out, gate, true, qhat);
  if ((st = do_select(h, cs, B, query, subkeys, idx, weights, workspace, workspace_bytes,
                      &h->last_launches, nullptr, nullptr, Gate{}, false, qhat)))
    return st;
  cudaError_t e = launch_gather(shape_of(h->cfg, B), idx, weights, values, out, cs,
                                &h->last_launches, gate);
  if (e != cudaSuccess) return cuda_fail(e, "gather");
  return MSN_OK;
}

msn_status msn_pkm_forward(msn_pkm_t h, void* stream, int64_t B, const void* query,
                           const void* subkeys, const void* values, float* out, int32_t* idx,
                           float* weights, void* workspace, size_t workspace_bytes) {
  return do_forward(h, stream, B, query, subkeys, values, out, idx, weights, workspace,
                    workspace_bytes, Gate{});
}

msn_status msn_pkm_forward_qln(msn_pkm_t h, void* stream, int64_t B, const void* query,
                               const void* subkeys, const void* values, float* out, int32_t* idx,
                               float* weights, void* q_hat, void* workspace, size_t workspace_bytes) {
  if (B > 0) REQUIRE_PTR(q_hat);
  return do_forward(h, stream, B, query, subkeys, values, out, idx, weights, workspace, workspace_bytes,
                    Gate{}, q_hat);
}

msn_status msn_pkm_forward_gated(msn_pkm_t h, void* stream, int64_t B, const void* query,
                                 const void* subkeys, const void* values, const float* x_in,
                                 int32_t gate, float* out, float* x_tilde, int32_t* idx,
                                 float* weights, void* workspace, size_t workspace_bytes) {
  if (gate < MSN_GATE_TANH || gate > MSN_GATE_IDENTITY)
    return fail(MSN_ERR_INVALID_ARG, "gate %d is not MSN_GATE_TANH/SIGMOID/IDENTITY", gate);
  if (B > 0) {
    REQUIRE_PTR(x_in);
    REQUIRE_PTR(x_tilde);
  }
  Gate g;
  g.x = x_in;
  g.xt = x_tilde;
  g.kind = gate;
  return do_forward(h, stream, B, query, subkeys, values, out, idx, weights, workspace,
                    workspace_bytes, g);
}

msn_status msn_pkm_gate_backward(msn_pkm_t h, void* stream, int64_t B, int32_t gate,
                                 const float* x_in, const float* v_o, const float* d_x_tilde,
                                 float* d_x_in, float* d_out) {
  msn_status st = check_handle(h);
  if (st) return st;
  if ((st = check_batch(h, B))) return st;
  h->last_launches = 0;
  if (gate < MSN_GATE_TANH || gate > MSN_GATE_IDENTITY)
    return fail(MSN_ERR_INVALID_ARG, "gate %d is not MSN_GATE_TANH/SIGMOID/IDENTITY", gate);
  if (B == 0) return MSN_OK;
  REQUIRE_PTR(x_in);
  REQUIRE_PTR(v_o);
  REQUIRE_PTR(d_x_tilde);
  REQUIRE_PTR(d_x_in);
  REQUIRE_PTR(d_out);
  const int64_t rows = B * shape_of(h->cfg, 0).og;  // out is [B, G, d_value]
  cudaError_t e = launch_gate_backward(rows, h->cfg.d_value, gate, x_in, v_o, d_x_tilde, d_x_in, d_out,
                                       (cudaStream_t)stream, &h->last_launches);
  if (e != cudaSuccess) return cuda_fail(e, "gate backward");
  return MSN_OK;
}

msn_status msn_pkm_scatter(msn_pkm_t h, void* stream, int64_t B, const int32_t* idx,
                           const float* weights, const float* d_out, const void* values,
                           float* d_values, float* dw, void* workspace, size_t workspace_bytes) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  if (B < 0) return fail(MSN_ERR_INVALID_ARG, "B < 0");
  if (B == 0) return MSN_OK;
  REQUIRE_PTR(idx);
  REQUIRE_PTR(weights);
  REQUIRE_PTR(d_out);
  REQUIRE_PTR(values);
  REQUIRE_PTR(d_values);
  REQUIRE_PTR(dw);
  if ((st = check_bwd_shape(h, true, false))) return st;
  if ((st = check_tape(h, stream, B, idx, weights))) return st;
  const Shape s = shape_of(h->cfg, B);
  cudaStream_t cs = (cudaStream_t)stream;
  cudaError_t e;
  if (h->cfg.flags & MSN_FLAG_ATOMIC_BWD) {
    e = launch_scatter_atomic(s, idx, weights, d_out, values, d_values, dw, cs, &h->last_launches);
  } else {
    REQUIRE_PTR(workspace);
    const size_t need = bwd_workspace_bytes(shape_of(h->cfg, 0), B);
    if (workspace_bytes < need)
      return fail(MSN_ERR_WORKSPACE, "scatter workspace %zu < %zu bytes", workspace_bytes, need);
    const BwdWorkspace ws = carve_bwd_workspace(shape_of(h->cfg, 0), B, workspace);
    e = launch_scatter_sorted(s, idx, weights, d_out, values, d_values, dw, ws, cs,
                              &h->last_launches,
                              TraceEvents{h->trace, h->ntrace});
  }
  if (e != cudaSuccess) return cuda_fail(e, "scatter (dV, dw)");
  return MSN_OK;
}

msn_status msn_pkm_scatter_update(msn_pkm_t h, void* stream, int64_t B, const int32_t* idx,
                                  const float* weights, const float* d_out, void* values,
                                  int32_t update, float lr, float eps, float* state, float* dw,
                                  void* workspace, size_t workspace_bytes) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  if (B < 0) return fail(MSN_ERR_INVALID_ARG, "B < 0");
  if (update != MSN_UPDATE_SGD && update != MSN_UPDATE_ADAGRAD)
    return fail(MSN_ERR_INVALID_ARG, "update %d is not MSN_UPDATE_SGD/ADAGRAD", update);
  if (!(lr >= 0.f) || !(eps >= 0.f)) return fail(MSN_ERR_INVALID_ARG, "lr and eps must be >= 0");
  if (h->cfg.flags & MSN_FLAG_ATOMIC_BWD)
    return fail(MSN_ERR_UNSUPPORTED, "the fused update needs the deterministic (grouped) backward");
  if (B == 0) return MSN_OK;
  REQUIRE_PTR(idx);
  REQUIRE_PTR(weights);
  REQUIRE_PTR(d_out);
  REQUIRE_PTR(values);
  REQUIRE_PTR(dw);
  REQUIRE_PTR(workspace);
  if (update == MSN_UPDATE_ADAGRAD) REQUIRE_PTR(state);
  if ((st = check_bwd_shape(h, true, false))) return st;
  if ((st = check_tape(h, stream, B, idx, weights))) return st;
  const Shape s = shape_of(h->cfg, B);
  const size_t need = bwd_workspace_bytes(shape_of(h->cfg, 0), B);
  if (workspace_bytes < need)
    return fail(MSN_ERR_WORKSPACE, "scatter workspace %zu < %zu bytes", workspace_bytes, need);
  const BwdWorkspace ws = carve_bwd_workspace(shape_of(h->cfg, 0), B, workspace);
  cudaError_t e = launch_scatter_sorted(s, idx, weights, d_out, values, nullptr, dw, ws,
                                        (cudaStream_t)stream, &h->last_launches,
                                        TraceEvents{h->trace, h->ntrace}, update, lr, eps,
                                        update == MSN_UPDATE_ADAGRAD ? state : nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "scatter with fused update");
  return MSN_OK;
}

msn_status msn_pkm_backward_keys(msn_pkm_t h, void* stream, int64_t B, const void* query,
                                 const void* subkeys, const int32_t* idx, const float* weights,
                                 const float* dw, float* d_query, float* d_subkeys,
                                 void* workspace, size_t workspace_bytes) {
  msn_status st = check_handle(h);
  if (st) return st;
  if ((st = check_batch(h, B))) return st;
  h->last_launches = 0;
  if (B == 0) return MSN_OK;
  REQUIRE_PTR(query);
  REQUIRE_PTR(subkeys);
  REQUIRE_PTR(idx);
  REQUIRE_PTR(weights);
  REQUIRE_PTR(dw);
  REQUIRE_PTR(d_query);
  REQUIRE_PTR(d_subkeys);
  REQUIRE_PTR(workspace);
  if ((st = check_bwd_shape(h, false, true))) return st;
  if ((st = check_tape(h, stream, B, idx, weights))) return st;
  const Shape s = shape_of(h->cfg, B);
  const size_t need = bwd_workspace_bytes(s, B);
  if (workspace_bytes < need)
    return fail(MSN_ERR_WORKSPACE, "backward workspace %zu < %zu bytes", workspace_bytes, need);
  const BwdWorkspace ws = carve_bwd_workspace(s, B, workspace);
  cudaError_t e = launch_backward_keys(s, query, subkeys, idx, weights, dw, d_query, d_subkeys, ws,
                                       (cudaStream_t)stream, &h->last_launches);
  if (e != cudaSuccess) return cuda_fail(e, "backward (ds, dQ, dK)");
  return MSN_OK;
}

msn_status msn_pkm_backward(msn_pkm_t h, void* stream, int64_t B, const float* d_out,
                            const void* query, const void* subkeys, const void* values,
                            const int32_t* idx, const float* weights, float* d_query,
                            float* d_subkeys, float* d_values, float* dw, void* workspace,
                            size_t workspace_bytes) {
  msn_status st = check_handle(h);
  if (st) return st;
  if ((st = check_batch(h, B))) return st;
  h->last_launches = 0;
  if (B == 0) return MSN_OK;
  const Shape s0 = shape_of(h->cfg, 0);
  const int64_t n = (int64_t)h->cfg.n_sub * h->cfg.n_sub * (s0.tab_stride ? s0.og : 1);
  if (h->cfg.row_begin != 0 || h->cfg.row_end != n)
    return fail(MSN_ERR_INVALID_ARG, "msn_pkm_backward needs the whole table; use the phase calls when sharded");
  REQUIRE_PTR(d_out);
  REQUIRE_PTR(query);
  REQUIRE_PTR(subkeys);
  REQUIRE_PTR(values);
  REQUIRE_PTR(idx);
  REQUIRE_PTR(weights);
  REQUIRE_PTR(d_query);
  REQUIRE_PTR(d_subkeys);
  REQUIRE_PTR(d_values);
  REQUIRE_PTR(workspace);
  if ((st = check_bwd_shape(h, true, true))) return st;
  if ((st = check_tape(h, stream, B, idx, weights))) return st;
  const Shape s = shape_of(h->cfg, B);
  const size_t need = bwd_workspace_bytes(s, B);
  if (workspace_bytes < need)
    return fail(MSN_ERR_WORKSPACE, "backward workspace %zu < %zu bytes", workspace_bytes, need);
  const BwdWorkspace ws = carve_bwd_workspace(s, B, workspace);
  float* dwp = dw ? dw : ws.dw;
  if (dw && !aligned16(dw)) return fail(MSN_ERR_INVALID_ARG, "dw is not 16-byte aligned");
  cudaStream_t cs = (cudaStream_t)stream;
  int* L = &h->last_launches;
  cudaError_t e = (h->cfg.flags & MSN_FLAG_ATOMIC_BWD)
                      ? launch_scatter_atomic(s, idx, weights, d_out, values, d_values, dwp, cs, L)
                      : launch_scatter_sorted(s, idx, weights, d_out, values, d_values, dwp, ws,
                                              cs, L);
  if (e != cudaSuccess) return cuda_fail(e, "backward (dV, dw)");
  e = launch_backward_keys(s, query, subkeys, idx, weights, dwp, d_query, d_subkeys, ws, cs, L);
  if (e != cudaSuccess) return cuda_fail(e, "backward (ds, dQ, dK)");
  return MSN_OK;
}


// ------------------------------------------- a9 record exchange (sharded) --
}  // extern "C"
namespace {

struct XLayout {
  int64_t off[MSN_XREG_COUNT + 1];  // byte offsets; off[COUNT] = total
};

XLayout xlayout(const msn_pkm_config& c, int P, int64_t lb, bool staged) {
  const int64_t cap = lb * c.heads * c.k, dv = c.d_value;
  int64_t sz[MSN_XREG_COUNT] = {};
  sz[MSN_XREG_IN_ROW] = sz[MSN_XREG_IN_W] = sz[MSN_XREG_DW_IN] = 4 * P * cap;
  sz[MSN_XREG_IN_CNT] = 4 * P * lb;
  sz[MSN_XREG_PART_IN] = 4 * P * lb * dv;
  sz[MSN_XREG_DOUT] = 4 * lb * dv;
  sz[MSN_XREG_POS] = 4 * cap;
  sz[MSN_XREG_CTL] = 4 * 64;
  if (staged) {
    sz[MSN_XREG_OUT_ROW] = sz[MSN_XREG_OUT_W] = sz[MSN_XREG_DW_OUT] = 4 * P * cap;
    sz[MSN_XREG_OUT_CNT] = 4 * P * lb;
    sz[MSN_XREG_PART_OUT] = sz[MSN_XREG_DOUT_ALL] = 4 * P * lb * dv;
  }
  XLayout L;
  int64_t o = 0;
  for (int r = 0; r < MSN_XREG_COUNT; ++r) {
    L.off[r] = o;
    o += (int64_t)align256((size_t)sz[r]);
  }
  L.off[MSN_XREG_COUNT] = o;
  return L;
}

// The per-call view of the exchange: sizes and every pointer a phase needs.
struct XView {
  int P, rank, HK;
  bool staged;
  int64_t lb, cap, rpr;
  XLayout L;
  const msn_pkm_exchange* x;
  template <typename T>
  T* reg(int p, int r) const { return (T*)((char*)x->base[p] + L.off[r]); }
  template <typename T>
  T* own(int r) const { return reg<T>(rank, r); }
  RecordsIn records_in() const {
    RecordsIn ri;
    ri.P = P;
    ri.rank = rank;
    ri.lb = lb;
    ri.cap = cap;
    ri.HK = HK;
    ri.row = own<int32_t>(MSN_XREG_IN_ROW);
    ri.cnt = own<int32_t>(MSN_XREG_IN_CNT);
    ri.w = own<float>(MSN_XREG_IN_W);
    return ri;
  }
};

msn_status make_view(msn_pkm_t h, const msn_pkm_exchange* x, XView& v) {
  if (!x) return fail(MSN_ERR_INVALID_ARG, "exchange is NULL");
  const msn_pkm_config& c = h->cfg;
  const int P = c.world_size > 1 ? c.world_size : 1;
  if (x->world != P || x->rank != c.rank)
    return fail(MSN_ERR_INVALID_ARG, "exchange world/rank %d/%d != config %d/%d", x->world, x->rank, P, c.rank);
  if (x->transport != MSN_XCHG_PEER && x->transport != MSN_XCHG_STAGED)
    return fail(MSN_ERR_INVALID_ARG, "exchange transport %d", x->transport);
  if (x->local_batch < 0 || x->local_batch > c.max_batch)
    return fail(MSN_ERR_INVALID_ARG, "local_batch %lld outside [0, max_batch]", (long long)x->local_batch);
  if (c.head_groups > 1) return fail(MSN_ERR_UNSUPPORTED, "the exchange needs head_groups <= 1");
  if (c.heads * c.k > 256) return fail(MSN_ERR_UNSUPPORTED, "the exchange needs heads * k <= 256");
  if (c.flags & (MSN_FLAG_ATOMIC_BWD | MSN_FLAG_GROUP_TABLES))
    return fail(MSN_ERR_UNSUPPORTED, "the exchange runs the deterministic backward over one table");
  const int64_t n = (int64_t)c.n_sub * c.n_sub;
  if (c.row_begin != (int64_t)c.rank * (n / P) || c.row_end != (int64_t)(c.rank + 1) * (n / P))
    return fail(MSN_ERR_INVALID_ARG, "the exchange needs the rank's rows [rank n/P, (rank+1) n/P)");
  const bool staged = x->transport == MSN_XCHG_STAGED;
  for (int p = 0; p < P; ++p) {
    if (staged && p != c.rank) continue;
    if (!x->base[p] || ((uintptr_t)x->base[p] & 255u))
      return fail(MSN_ERR_INVALID_ARG, "exchange base[%d] is NULL or not 256-byte aligned", p);
  }
  v.P = P;
  v.rank = c.rank;
  v.staged = staged;
  v.lb = x->local_batch;
  v.HK = c.heads * c.k;
  v.cap = v.lb * v.HK;
  v.rpr = n / P;
  v.L = xlayout(c, P, v.lb, staged);
  v.x = x;
  return MSN_OK;
}

// SELECT: the scorer (a1-a2), then the fused Cartesian + route + local gather.
msn_status x_select(msn_pkm_t h, const XView& v, const void* query, const void* subkeys, const void* values,
                    int32_t* idx, float* w, float* out, void* ws, size_t ws_bytes, cudaStream_t st, int* L) {
  const Shape s = shape_of(h->cfg, v.lb);
  msn_status st0 = check_select_shape(s);
  if (st0) return st0;
  if (ws_bytes < fwd_bytes(s))
    return fail(MSN_ERR_WORKSPACE, "forward workspace %zu < %zu bytes", ws_bytes, fwd_bytes(s));
  Cands cd;
  char* p = carve_cands(s, ws, cd);
  cd.rq.Q = query;
  cd.rq.K = subkeys;
  cd.rq.d_h = s.d_h;
  cd.rq.qk_dt = s.qk_dt;
  cudaError_t e = launch_select_tc(s, query, subkeys, cd, p, st, L);
  if (e != cudaSuccess) return cuda_fail(e, "select (scoring + per-half candidates)");
  if (h->ntrace > 0) cudaEventRecord(h->trace[0], st);
  RouteArgs ra;
  ra.P = v.P;
  ra.rank = v.rank;
  ra.rpr = v.rpr;
  for (int o = 0; o < v.P; ++o) {
    if (v.staged) {  // OUT segment [o] of this rank
      ra.row.p[o] = v.own<int32_t>(MSN_XREG_OUT_ROW) + o * v.cap;
      ra.w.p[o] = v.own<float>(MSN_XREG_OUT_W) + o * v.cap;
      ra.cnt.p[o] = v.own<int32_t>(MSN_XREG_OUT_CNT) + o * v.lb;
    } else {  // owner o's IN segment [rank], over NVLink
      ra.row.p[o] = v.reg<int32_t>(o, MSN_XREG_IN_ROW) + v.rank * v.cap;
      ra.w.p[o] = v.reg<float>(o, MSN_XREG_IN_W) + v.rank * v.cap;
      ra.cnt.p[o] = v.reg<int32_t>(o, MSN_XREG_IN_CNT) + v.rank * v.lb;
    }
  }
  ra.pos = v.own<int32_t>(MSN_XREG_POS);
  const int64_t dv = h->cfg.d_value;
  ra.part = v.P == 1 ? out  // nothing to combine
                     : v.own<float>(v.staged ? MSN_XREG_PART_OUT : MSN_XREG_PART_IN) + v.rank * v.lb * dv;
  e = launch_cartesian_route(s, cd, idx, w, values, ra, st, L);
  if (e != cudaSuccess) return cuda_fail(e, "cartesian top-k + softmax + route + local gather");
  if (h->ntrace > 1) cudaEventRecord(h->trace[1], st);
  return MSN_OK;
}

cudaError_t x_gather(msn_pkm_t h, const XView& v, const void* values, cudaStream_t st, int* L) {
  PerRank<float> dst;
  for (int p = 0; p < kMaxWorld; ++p) dst.p[p] = nullptr;
  const int64_t dv = h->cfg.d_value;
  for (int p = 0; p < v.P; ++p)
    dst.p[p] = v.staged ? v.own<float>(MSN_XREG_PART_OUT) + p * v.lb * dv
                        : v.reg<float>(p, MSN_XREG_PART_IN) + v.rank * v.lb * dv;
  return launch_gather_records(shape_of(h->cfg, v.lb), v.records_in(), values, dst, st, L);
}

cudaError_t x_combine(msn_pkm_t h, const XView& v, float* out, cudaStream_t st, int* L) {
  if (v.P == 1) return cudaSuccess;  // SELECT wrote out
  return launch_reduce_partials(v.own<float>(MSN_XREG_PART_IN), v.P, v.lb, 1, h->cfg.d_value, out, st, L);
}

// dw_direct (P = 1 only, may be NULL): write dw straight into the caller's
// [B_l, H, k] array (one rank's windows are the slots in (b, h, t) order)
cudaError_t x_scatter(msn_pkm_t h, const XView& v, const void* values, float* d_values, void* ws,
                      cudaStream_t st, int* L, float* dw_direct = nullptr, const float* dout_direct = nullptr) {
  PerRank<const float> xs;
  PerRank<float> dd;
  for (int p = 0; p < kMaxWorld; ++p) {
    xs.p[p] = nullptr;
    dd.p[p] = nullptr;
  }
  const int64_t dv = h->cfg.d_value;
  for (int p = 0; p < v.P; ++p) {
    xs.p[p] = v.staged ? v.own<float>(MSN_XREG_DOUT_ALL) + p * v.lb * dv : v.reg<float>(p, MSN_XREG_DOUT);
    dd.p[p] = v.staged ? v.own<float>(MSN_XREG_DW_OUT) + p * v.cap
                       : v.reg<float>(p, MSN_XREG_DW_IN) + v.rank * v.cap;  // window order
  }
  if (v.P == 1 && dw_direct) dd.p[0] = dw_direct;
  if (v.P == 1 && dout_direct && !v.staged) xs.p[0] = dout_direct;
  const Shape s = shape_of(h->cfg, v.lb);
  const BwdWorkspace bw = carve_bwd_workspace(s, v.P * v.lb, ws);
  return launch_scatter_records(s, v.records_in(), xs, values, d_values, dd, bw, st, L,
                                TraceEvents{h->trace, h->ntrace});
}

cudaError_t x_collect(msn_pkm_t h, const XView& v, const int32_t* idx, float* dw, cudaStream_t st, int* L) {
  return launch_collect_dw(shape_of(h->cfg, v.lb), idx, v.own<int32_t>(MSN_XREG_POS), v.own<float>(MSN_XREG_DW_IN),
                           v.cap, v.rpr, dw, st, L);
}

cudaError_t x_barrier(const XView& v, cudaStream_t st, int* L, bool always = false) {
  // (the caller's collectives order the staged transport; one rank in the
  // composite calls: stream order)
  if (v.staged || (v.P == 1 && !always)) return cudaSuccess;
  PerRank<uint32_t> f;
  for (int p = 0; p < kMaxWorld; ++p) f.p[p] = nullptr;
  for (int p = 0; p < v.P; ++p) f.p[p] = v.reg<uint32_t>(p, MSN_XREG_CTL);
  return launch_exchange_barrier(v.P, v.rank, f, v.own<uint32_t>(MSN_XREG_CTL), st, L);
}

size_t x_ws_bytes(msn_pkm_t h, const XView& v) {
  const Shape s = shape_of(h->cfg, v.lb);
  const size_t a = fwd_bytes(s), b = bwd_workspace_bytes(s, v.P * v.lb);
  return a > b ? a : b;
}

}  // namespace
extern "C" {

msn_status msn_pkm_exchange_layout(msn_pkm_t h, int64_t local_batch, int32_t staged, int64_t* offsets,
                                   size_t* bytes) {
  msn_status st = check_handle(h);
  if (st) return st;
  if ((st = check_batch(h, local_batch))) return st;
  const int P = h->cfg.world_size > 1 ? h->cfg.world_size : 1;
  const XLayout L = xlayout(h->cfg, P, local_batch, staged != 0);
  if (offsets)
    for (int r = 0; r < MSN_XREG_COUNT; ++r) offsets[r] = L.off[r];
  if (bytes) *bytes = (size_t)L.off[MSN_XREG_COUNT];
  return MSN_OK;
}

#define XCALL(expr, what)                                      \
  do {                                                         \
    cudaError_t e_ = (expr);                                   \
    if (e_ != cudaSuccess) return cuda_fail(e_, what);         \
  } while (0)

msn_status msn_pkm_exchange_select(msn_pkm_t h, void* stream, const void* query, const void* subkeys,
                                   const void* values, const msn_pkm_exchange* x, int32_t* idx, float* weights,
                                   float* out, void* workspace, size_t workspace_bytes) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  XView v;
  if ((st = make_view(h, x, v))) return st;
  if (v.lb == 0) return MSN_OK;
  REQUIRE_PTR(query);
  REQUIRE_PTR(subkeys);
  REQUIRE_PTR(values);
  REQUIRE_PTR(idx);
  REQUIRE_PTR(weights);
  REQUIRE_PTR(workspace);
  if (v.P == 1) REQUIRE_PTR(out);
  return x_select(h, v, query, subkeys, values, idx, weights, out, workspace, workspace_bytes,
                  (cudaStream_t)stream, &h->last_launches);
}

msn_status msn_pkm_exchange_gather(msn_pkm_t h, void* stream, const void* values, const msn_pkm_exchange* x) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  XView v;
  if ((st = make_view(h, x, v))) return st;
  if (v.lb == 0) return MSN_OK;
  REQUIRE_PTR(values);
  XCALL(x_gather(h, v, values, (cudaStream_t)stream, &h->last_launches), "exchange gather");
  return MSN_OK;
}

msn_status msn_pkm_exchange_combine(msn_pkm_t h, void* stream, const msn_pkm_exchange* x, float* out) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  XView v;
  if ((st = make_view(h, x, v))) return st;
  if (v.lb == 0) return MSN_OK;
  REQUIRE_PTR(out);
  XCALL(x_combine(h, v, out, (cudaStream_t)stream, &h->last_launches), "exchange combine");
  return MSN_OK;
}

msn_status msn_pkm_exchange_scatter(msn_pkm_t h, void* stream, const void* values, float* d_values,
                                    const msn_pkm_exchange* x, void* workspace, size_t workspace_bytes) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  XView v;
  if ((st = make_view(h, x, v))) return st;
  if (v.lb == 0) return MSN_OK;
  REQUIRE_PTR(values);
  REQUIRE_PTR(d_values);
  REQUIRE_PTR(workspace);
  if ((st = check_bwd_shape(h, true, false))) return st;
  const size_t need = bwd_workspace_bytes(shape_of(h->cfg, v.lb), v.P * v.lb);
  if (workspace_bytes < need)
    return fail(MSN_ERR_WORKSPACE, "exchange scatter workspace %zu < %zu bytes", workspace_bytes, need);
  XCALL(x_scatter(h, v, values, d_values, workspace, (cudaStream_t)stream, &h->last_launches), "exchange scatter");
  return MSN_OK;
}

msn_status msn_pkm_exchange_collect(msn_pkm_t h, void* stream, const int32_t* idx, const msn_pkm_exchange* x,
                                    float* dw) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  XView v;
  if ((st = make_view(h, x, v))) return st;
  if (v.lb == 0) return MSN_OK;
  REQUIRE_PTR(idx);
  REQUIRE_PTR(dw);
  XCALL(x_collect(h, v, idx, dw, (cudaStream_t)stream, &h->last_launches), "exchange collect");
  return MSN_OK;
}

msn_status msn_pkm_exchange_barrier(msn_pkm_t h, void* stream, const msn_pkm_exchange* x) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  XView v;
  if ((st = make_view(h, x, v))) return st;
  XCALL(x_barrier(v, (cudaStream_t)stream, &h->last_launches, true), "exchange barrier");
  return MSN_OK;
}

msn_status msn_pkm_forward_sharded(msn_pkm_t h, void* stream, int64_t local_batch, const void* query,
                                   const void* subkeys, const void* values, const msn_pkm_exchange* x,
                                   float* out, int32_t* idx, float* weights, void* workspace,
                                   size_t workspace_bytes) {
  msn_status st = check_handle(h);
  if (st) return st;
  if ((st = check_batch(h, local_batch))) return st;
  h->last_launches = 0;
  XView v;
  if ((st = make_view(h, x, v))) return st;
  if (v.lb != local_batch) return fail(MSN_ERR_INVALID_ARG, "local_batch != exchange local_batch");
  if (v.staged) return fail(MSN_ERR_INVALID_ARG, "forward_sharded runs the PEER transport; STAGED: use the phases");
  REQUIRE_PTR(query);
  REQUIRE_PTR(subkeys);
  REQUIRE_PTR(values);
  REQUIRE_PTR(out);
  REQUIRE_PTR(idx);
  REQUIRE_PTR(weights);
  REQUIRE_PTR(workspace);
  if (workspace_bytes < x_ws_bytes(h, v))
    return fail(MSN_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, x_ws_bytes(h, v));
  cudaStream_t cs = (cudaStream_t)stream;
  int* L = &h->last_launches;
  // every rank takes part in every barrier, also with no local queries
  if (v.lb > 0 &&
      (st = x_select(h, v, query, subkeys, values, idx, weights, out, workspace, workspace_bytes, cs, L)))
    return st;
  XCALL(x_barrier(v, cs, L), "exchange barrier");
  if (v.lb > 0) XCALL(x_gather(h, v, values, cs, L), "exchange gather");
  XCALL(x_barrier(v, cs, L), "exchange barrier");
  if (v.lb > 0) XCALL(x_combine(h, v, out, cs, L), "exchange combine");
  return MSN_OK;
}

msn_status msn_pkm_backward_sharded(msn_pkm_t h, void* stream, int64_t local_batch, const float* d_out,
                                    const void* query, const void* subkeys, const void* values,
                                    const int32_t* idx, const float* weights, const msn_pkm_exchange* x,
                                    float* d_query, float* d_subkeys, float* d_values, float* dw,
                                    void* workspace, size_t workspace_bytes) {
  msn_status st = check_handle(h);
  if (st) return st;
  if ((st = check_batch(h, local_batch))) return st;
  h->last_launches = 0;
  XView v;
  if ((st = make_view(h, x, v))) return st;
  if (v.lb != local_batch) return fail(MSN_ERR_INVALID_ARG, "local_batch != exchange local_batch");
  if (v.staged) return fail(MSN_ERR_INVALID_ARG, "backward_sharded runs the PEER transport; STAGED: use the phases");
  REQUIRE_PTR(d_out);
  REQUIRE_PTR(query);
  REQUIRE_PTR(subkeys);
  REQUIRE_PTR(values);
  REQUIRE_PTR(idx);
  REQUIRE_PTR(weights);
  REQUIRE_PTR(d_query);
  REQUIRE_PTR(d_subkeys);
  REQUIRE_PTR(d_values);
  REQUIRE_PTR(workspace);
  if (dw && !aligned16(dw)) return fail(MSN_ERR_INVALID_ARG, "dw is not 16-byte aligned");
  if ((st = check_bwd_shape(h, true, true))) return st;
  if (workspace_bytes < x_ws_bytes(h, v))
    return fail(MSN_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, x_ws_bytes(h, v));
  if ((st = check_tape(h, stream, v.lb, idx, weights))) return st;
  cudaStream_t cs = (cudaStream_t)stream;
  int* L = &h->last_launches;
  const Shape s = shape_of(h->cfg, v.lb);
  const BwdWorkspace bw = carve_bwd_workspace(s, v.P * v.lb, workspace);
  float* dwp = dw ? dw : bw.dw;
  if (v.lb > 0 && v.P > 1)  // (one rank: the scatter reads the caller's d_out)
    XCALL(cudaMemcpyAsync(v.own<float>(MSN_XREG_DOUT), d_out, sizeof(float) * v.lb * h->cfg.d_value,
                          cudaMemcpyDeviceToDevice, cs), "d_out -> exchange");
  XCALL(x_barrier(v, cs, L), "exchange barrier");
  // one rank: the scatter's dw is already in (b, h, t) order, no collect
  XCALL(x_scatter(h, v, values, d_values, workspace, cs, L, v.P == 1 ? dwp : nullptr, d_out), "exchange scatter");
  XCALL(x_barrier(v, cs, L), "exchange barrier");
  if (v.lb > 0) {
    if (v.P > 1) XCALL(x_collect(h, v, idx, dwp, cs, L), "exchange collect");
    XCALL(launch_backward_keys(s, query, subkeys, idx, weights, dwp, d_query, d_subkeys, bw, cs, L),
          "backward (ds, dQ, dK)");
  }
  return MSN_OK;
}

// ------------------------------------------------ prologue --
msn_status msn_pkm_layernorm(msn_pkm_t h, void* stream, int64_t rows, const void* x, void* y) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  if (rows < 0) return fail(MSN_ERR_INVALID_ARG, "rows < 0");
  if (rows == 0) return MSN_OK;
  REQUIRE_PTR(x);
  REQUIRE_PTR(y);
  const Shape s = shape_of(h->cfg, 0);
  if (!prologue_supported(s)) return fail(MSN_ERR_UNSUPPORTED, "layernorm needs d_half in {32, 64, 128, 256}");
  cudaError_t e = launch_layernorm(s, rows, x, y, nullptr, nullptr, (cudaStream_t)stream, &h->last_launches);
  if (e != cudaSuccess) return cuda_fail(e, "layernorm");
  return MSN_OK;
}

msn_status msn_pkm_layernorm_backward(msn_pkm_t h, void* stream, int64_t rows, const void* x,
                                      const float* dy, float* dx) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  if (rows < 0) return fail(MSN_ERR_INVALID_ARG, "rows < 0");
  if (rows == 0) return MSN_OK;
  REQUIRE_PTR(x);
  REQUIRE_PTR(dy);
  REQUIRE_PTR(dx);
  const Shape s = shape_of(h->cfg, 0);
  if (!prologue_supported(s)) return fail(MSN_ERR_UNSUPPORTED, "layernorm needs d_half in {32, 64, 128, 256}");
  cudaError_t e = launch_layernorm(s, rows, x, nullptr, dy, dx, (cudaStream_t)stream, &h->last_launches);
  if (e != cudaSuccess) return cuda_fail(e, "layernorm backward");
  return MSN_OK;
}

msn_status msn_pkm_key_transform(msn_pkm_t h, void* stream, const void* k_hat, const float* theta,
                                 void* k_eff) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  REQUIRE_PTR(k_hat);
  REQUIRE_PTR(theta);
  REQUIRE_PTR(k_eff);
  cudaError_t e = launch_key_transform(shape_of(h->cfg, 0), k_hat, theta, k_eff, (cudaStream_t)stream,
                                       &h->last_launches);
  if (e != cudaSuccess) return cuda_fail(e, "key transform");
  return MSN_OK;
}

msn_status msn_pkm_key_transform_backward(msn_pkm_t h, void* stream, const void* k_hat,
                                          const float* theta, const float* d_k_eff, float* d_k_hat,
                                          float* d_theta) {
  msn_status st = check_handle(h);
  if (st) return st;
  h->last_launches = 0;
  REQUIRE_PTR(k_hat);
  REQUIRE_PTR(theta);
  REQUIRE_PTR(d_k_eff);
  REQUIRE_PTR(d_k_hat);
  REQUIRE_PTR(d_theta);
  cudaError_t e = launch_key_transform_backward(shape_of(h->cfg, 0), k_hat, theta, d_k_eff, d_k_hat,
                                                d_theta, (cudaStream_t)stream, &h->last_launches);
  if (e != cudaSuccess) return cuda_fail(e, "key transform backward");
  return MSN_OK;
}

}  // extern "C"
