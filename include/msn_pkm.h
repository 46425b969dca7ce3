/*
 * msn_pkm.h -- C ABI of the B200 (sm_100a) Product-Key Memory lookup, the
 * data-parallel hot path of MSN (arXiv 2602.07526, section 3.3).
 *
 * What one lookup (query b, head h) computes (PAPER.md, readings in DESIGN.md):
 *   a0  q_row = q[b,h,0,:], q_col = q[b,h,1,:]
 *   a1  S_row = K_row q_row, S_col = K_col q_col   (Eq. S_old)
 *   a2  I = argtopk_i S_row, J = argtopk_j S_col
 *   a3  K = argtopk_{(i,j) in I x J} S_row[i] + S_col[j]
 *   a4  w = softmax over the k selected scores (reading R1)
 *   a5  v_o = sum_{(i,j) in K} w_ij V[i*n_sub + j]  (Eq. vo_mem, reading R2)
 *                                                               PAPER.md:226-229
 *   a6-a8 backward: "scatter-adds gradients into the value table" and the
 *       sub-keys (north_star), gradient only through the
 *       selected scores ("unselected keys receive no gradients",
 *       PAPER.md:282-284).
 * Heads (reading R7): per-head sub-key codebooks, one shared value table,
 * out[b] = sum_h v_o(b,h).
 * Ties (reading R5): per half (score desc, index asc); final (score desc,
 * flat asc); idx/weights are listed in that order.
 *
 * Layouts (all row-major, element strides implied by the config):
 *   query    [B, H, 2, d_half]      qk_dtype   half 0 -> K_row (i), half 1 -> K_col (j)
 *   subkeys  [H, 2, n_sub, d_half]  qk_dtype
 *   values   [row_end-row_begin, d_value] value_dtype  (the local rows of the
 *            n_sub^2-row table; row_begin=0,row_end=n_sub^2 when unsharded)
 *   out      [B, d_value] fp32      sum over heads ([B, G, d_value] with head_groups G > 1)
 *   idx      [B, H, k]   int32      global flat slot ids i*n_sub + j
 *   weights  [B, H, k]   fp32       softmax weights, same order as idx
 *   d_out    [B, d_value] fp32
 *   d_query  [B, H, 2, d_half] fp32            written (=)  (qk_dtype with
 *            MSN_FLAG_DQ_QK_DTYPE)
 *   d_subkeys[H, 2, n_sub, d_half] fp32        accumulated (+=)
 *   d_values [row_end-row_begin, d_value] fp32 accumulated (+=)
 *   dw       [B, H, k] fp32   d loss / d weights (local rows only when sharded)
 *
 * Ownership: the caller owns every device buffer (inputs, outputs, the tape
 * idx/weights, workspace); the library never allocates device memory.  The
 * handle owns host state only.  All pointers are DEVICE pointers, 16-byte
 * aligned.  Every call enqueues work on the caller's stream and returns
 * without synchronising; buffers must stay alive until that work completes.
 * One in-flight call per handle; a handle is not thread-safe.
 *
 * Errors: every entry point returns msn_status and never aborts.  Arguments
 * are validated on the host before any launch (MSN_ERR_INVALID_ARG);
 * supported-but-unimplemented shapes give MSN_ERR_UNSUPPORTED; launch
 * failures give MSN_ERR_CUDA (asynchronous device faults surface on a later
 * CUDA call).  msn_pkm_last_error() returns a thread-local description of the
 * last failure.  B = 0 is a no-op returning MSN_OK.  Inputs must be finite.
 */
#ifndef MSN_PKM_H_
#define MSN_PKM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSN_PKM_ABI_VERSION 2
#define MSN_MAX_WORLD 8 /* ranks of one NVLink/NVSwitch node (8 x B200) */

typedef enum {
  MSN_OK = 0,
  MSN_ERR_INVALID_ARG = 1,
  MSN_ERR_UNSUPPORTED = 2,
  MSN_ERR_CUDA = 3,
  MSN_ERR_WORKSPACE = 5,
  MSN_ERR_INTERNAL = 6
} msn_status;

typedef enum { MSN_F32 = 0, MSN_BF16 = 1 } msn_dtype;

/* Memory-gated fusion gate g: x~ = x_in (.) g(v_o),
 * Eq. gating PAPER.md:318-322 (tanh); sigmoid and identity are the
 * alternatives of the paper's gate ablation. */
typedef enum { MSN_GATE_TANH = 1, MSN_GATE_SIGMOID = 2, MSN_GATE_IDENTITY = 3 } msn_gate;

/* Fused sparse optimiser update (the "gradient updates"
 * of the paper's Sparse-Gather op), reading R20. */
typedef enum { MSN_UPDATE_SGD = 1, MSN_UPDATE_ADAGRAD = 2 } msn_update;

/* flags */
#define MSN_FLAG_ATOMIC_BWD 0x1u /* value-gradient scatter with red.global.add
                                    (non-deterministic order) instead of the
                                    default deterministic grouped reduce */
#define MSN_FLAG_GROUP_TABLES 0x2u /* every head group has its
                                      own value table (per-token V):
                                      values hold G * n_sub^2 rows, group g's
                                      slots at rows g*n_sub^2 + i*n_sub + j, and
                                      idx reports those global rows */
#define MSN_FLAG_DQ_QK_DTYPE 0x4u /* d_query written in qk_dtype (bf16 for bf16
                                     configs, rounded once, RNE) instead of fp32:
                                     the gradient in the query's own dtype, half
                                     the bytes (e.g. for a host copy) */
#define MSN_FLAG_VALIDATE 0x8u /* SURVEY 8(b) MSN_VALIDATE: every call that
                                  consumes a tape (idx, weights) first checks
                                  it as msn_pkm_validate_tape does, SYNCHRONISES
                                  the stream, and returns MSN_ERR_INVALID_ARG
                                  (nothing launched) if any slot is invalid.
                                  A debugging mode: not graph-capturable; the
                                  handle then owns a 4-byte device word. */

typedef struct msn_pkm* msn_pkm_t;

typedef struct {
  int32_t abi_version; /* must equal MSN_PKM_ABI_VERSION */
  int32_t heads;       /* H >= 1 */
  int32_t n_sub;       /* sqrt(n): keys per codebook, n_sub^2 < 2^31 */
  int32_t d_half;      /* d: width of q_row / q_col and of a sub-key, % 16 == 0 */
  int32_t d_value;     /* value row width; d_value * sizeof(value) % 16 == 0 */
  int32_t k;           /* per-half and final top-k, 1 <= k <= min(n_sub, 64) */
  int64_t max_batch;   /* workspace is sized for B <= max_batch */
  int32_t qk_dtype;    /* msn_dtype of query and sub-keys */
  int32_t value_dtype; /* msn_dtype of the value table */
  uint32_t flags;      /* MSN_FLAG_* */
  int32_t head_groups; /* G (token-specific sub-keys):
                          0 or 1 = one group (out = sum over all heads); else H % G
                          == 0, consecutive blocks of H/G heads form a group (a
                          token with its own sub-key codebooks) and
                          out[b, g] = sum over the group's heads: out and d_out
                          are [B, G, d_value].  G > 1 needs the unsharded table
                          and the deterministic backward. */
  int64_t row_begin;   /* this process holds value rows [row_begin, row_end) */
  int64_t row_end;     /* (row-sharded table); 0 and n_sub^2 when unsharded */
  int32_t world_size;  /* P: 0 or 1 = no record exchange (the rows are row_begin..row_end);
                          2 <= P <= MSN_MAX_WORLD = the row-sharded table with the
                          library's record exchange (BASELINE.json
                          configs[3]): this rank holds rows [rank n/P, (rank+1) n/P),
                          n % P == 0, and row_begin/row_end must be 0/0 or exactly that
                          range.  A P = 1 exchange (the same sharded code path on one
                          GPU) is world_size = 1 with the msn_pkm_exchange calls. */
  int32_t rank;        /* 0 <= rank < max(world_size, 1) */
} msn_pkm_config;

/* Create / destroy a handle.  create validates the config. */
msn_status msn_pkm_create(const msn_pkm_config* cfg, msn_pkm_t* out);
msn_status msn_pkm_destroy(msn_pkm_t h);

/* Workspace bytes needed by forward / backward (and by the phase calls
 * below) for a batch of B <= max_batch queries.  gather_batch is the number
 * of queries the gather/scatter phases see (B for unsharded use; the
 * all-gathered batch when sharded). */
msn_status msn_pkm_workspace_size(msn_pkm_t h, int64_t B, int64_t gather_batch,
                                  size_t* fwd_bytes, size_t* bwd_bytes);

/* Full forward, steps a1-a5 (unsharded: requires row_begin=0, row_end=n).
 * Writes out, idx, weights (idx/weights are the backward tape). */
msn_status msn_pkm_forward(msn_pkm_t h, void* stream, int64_t B,
                           const void* query, const void* subkeys, const void* values,
                           float* out, int32_t* idx, float* weights,
                           void* workspace, size_t workspace_bytes);

/* Forward with the memory-gated fusion fused into the
 * kernel that produces v_o: everything msn_pkm_forward does, plus
 *   x_tilde = x_in (.) g(v_o)          (gate per msn_gate)
 * x_in, x_tilde: [B, d_value] fp32, 16-byte aligned device pointers (the
 * gate is elementwise, so x_in has the memory output's width).  out (= v_o,
 * sum over heads) is still written: the gate backward needs it.  Same errors
 * as msn_pkm_forward; an unknown gate -> MSN_ERR_INVALID_ARG. */
msn_status msn_pkm_forward_gated(msn_pkm_t h, void* stream, int64_t B,
                                 const void* query, const void* subkeys, const void* values,
                                 const float* x_in, int32_t gate, float* out, float* x_tilde,
                                 int32_t* idx, float* weights,
                                 void* workspace, size_t workspace_bytes);

/* Forward with the query LayerNorm folded into the scorer's operand load
 * (reading R23: LN over each d_half-wide query
 * half, no affine, eps = 1e-5): everything msn_pkm_forward does on
 * q^ = LN(query), and q^ [B, H, 2, d_half] (qk_dtype, rounded once) is
 * written to q_hat -- the backward's query (msn_pkm_backward(..., q_hat, ...)
 * gives d q^; msn_pkm_layernorm_backward(query, d q^) the gradient w.r.t. the
 * raw query).  Same errors as msn_pkm_forward; q_hat 16-byte aligned. */
msn_status msn_pkm_forward_qln(msn_pkm_t h, void* stream, int64_t B, const void* query,
                               const void* subkeys, const void* values, float* out, int32_t* idx,
                               float* weights, void* q_hat, void* workspace, size_t workspace_bytes);

/* Step a6 with the optimiser step fused into the row reduction (SURVEY 8(f)
 * f3): the value gradient g_r of every touched row r (this handle's rows) is
 * applied to the table in place instead of being accumulated into a
 * gradient buffer:
 *   MSN_UPDATE_SGD      values[r] -= lr * g_r
 *   MSN_UPDATE_ADAGRAD  state[r] += g_r^2;  values[r] -= lr * g_r / (sqrt(state[r]) + eps)
 * elementwise in fp32, rounded once (RNE) to value_dtype; untouched rows and
 * their state are not written.  dw (d loss / d weights) is computed from the
 * values BEFORE the update, exactly as msn_pkm_scatter does.
 *   values  [row_end-row_begin, d_value] value_dtype, read and written
 *   state   [row_end-row_begin, d_value] fp32 (+=), Adagrad only (else may be NULL)
 * Deterministic (grouped) backward only: with MSN_FLAG_ATOMIC_BWD it returns
 * MSN_ERR_UNSUPPORTED.  lr, eps >= 0 (else MSN_ERR_INVALID_ARG). */
msn_status msn_pkm_scatter_update(msn_pkm_t h, void* stream, int64_t B, const int32_t* idx,
                                  const float* weights, const float* d_out, void* values,
                                  int32_t update, float lr, float eps, float* state, float* dw,
                                  void* workspace, size_t workspace_bytes);

/* Query / key prologue, composed by the caller around
 * the lookup:  q^ = LN(q), k^ = LN(k) (reading R23: no affine,
 * eps = 1e-5), K~ = Theta k^ per (head, half), then the
 * lookup on (q^, K~); its d_query / d_subkeys are the gradients w.r.t. q^
 * and K~, which the backward calls below carry back to q, k and Theta
 * (PAPER.md:296-302).
 *
 * msn_pkm_layernorm: y = LN(x) row by row; x, y [rows, d_half] qk_dtype
 *   (queries: rows = B*H*2; sub-keys: rows = H*2*n_sub); output rounded once
 *   (RNE) to qk_dtype.  d_half in {32, 64, 128, 256} else MSN_ERR_UNSUPPORTED.
 * msn_pkm_layernorm_backward: dx = d LN(x)^T dy; x qk_dtype, dy and dx fp32
 *   [rows, d_half], dx written (=).
 * msn_pkm_key_transform: k_eff[h,c,i,:] = Theta[h,c] k_hat[h,c,i,:];
 *   k_hat, k_eff [H, 2, n_sub, d_half] qk_dtype; theta [H, 2, d_half, d_half]
 *   fp32 row-major (theta[h,c,r,col] multiplies k_hat component col).
 * msn_pkm_key_transform_backward: d_k_hat = Theta^T d_k_eff (=, fp32
 *   [H,2,n_sub,d_half]); d_theta += sum_i d_k_eff_i k_hat_i^T (fp32
 *   [H,2,d_half,d_half]).  All device pointers, 16-byte aligned. */
msn_status msn_pkm_layernorm(msn_pkm_t h, void* stream, int64_t rows, const void* x, void* y);
msn_status msn_pkm_layernorm_backward(msn_pkm_t h, void* stream, int64_t rows, const void* x,
                                      const float* dy, float* dx);
msn_status msn_pkm_key_transform(msn_pkm_t h, void* stream, const void* k_hat, const float* theta,
                                 void* k_eff);
msn_status msn_pkm_key_transform_backward(msn_pkm_t h, void* stream, const void* k_hat,
                                          const float* theta, const float* d_k_eff, float* d_k_hat,
                                          float* d_theta);

/* Backward of the gate for the upstream gradient d_x_tilde [B, d_value]:
 *   d_x_in = d_x_tilde (.) g(v_o)                       (written, =)
 *   d_out  = d_x_tilde (.) x_in (.) g'(v_o)             (written, =)
 * where v_o is the forward's out; d_out is then the upstream gradient of
 * msn_pkm_backward / msn_pkm_scatter.  All [B, d_value] fp32 device
 * pointers, 16-byte aligned.  One elementwise kernel; no workspace. */
msn_status msn_pkm_gate_backward(msn_pkm_t h, void* stream, int64_t B, int32_t gate,
                                 const float* x_in, const float* v_o, const float* d_x_tilde,
                                 float* d_x_in, float* d_out);

/* Full backward, steps a6-a8 (unsharded), for the loss with upstream
 * gradient d_out.  d_query is written; d_subkeys and d_values are
 * accumulated (+=).  dw may be NULL (then kept in the workspace). */
msn_status msn_pkm_backward(msn_pkm_t h, void* stream, int64_t B,
                            const float* d_out, const void* query, const void* subkeys,
                            const void* values, const int32_t* idx, const float* weights,
                            float* d_query, float* d_subkeys, float* d_values, float* dw,
                            void* workspace, size_t workspace_bytes);

/* ---- phase entry points: the steps of forward / backward one at a time
 * (select = a1-a4, gather = a5, scatter = a6, backward_keys = a7-a8), over
 * the handle's rows [row_begin, row_end); slots outside them contribute 0.
 * The row-sharded table's exchange has its own calls (msn_pkm_exchange_*). */

/* a1-a4: idx, weights for B queries. */
msn_status msn_pkm_select(msn_pkm_t h, void* stream, int64_t B,
                          const void* query, const void* subkeys,
                          int32_t* idx, float* weights, void* workspace, size_t workspace_bytes);

/* a5 over the local rows: out[b] = sum_{h,t: row_begin <= idx < row_end}
 * w * values[idx - row_begin]  (written, =). */
msn_status msn_pkm_gather(msn_pkm_t h, void* stream, int64_t B,
                          const int32_t* idx, const float* weights, const void* values,
                          float* out);

/* a6 over the local rows: d_values += w * d_out[b] and dw = <values[idx], d_out[b]>
 * for local slots (dw = 0 for slots held by other ranks). */
msn_status msn_pkm_scatter(msn_pkm_t h, void* stream, int64_t B,
                           const int32_t* idx, const float* weights, const float* d_out,
                           const void* values, float* d_values, float* dw,
                           void* workspace, size_t workspace_bytes);

/* a7-a8 given the full dw: d_query (=) and d_subkeys (+=). */
msn_status msn_pkm_backward_keys(msn_pkm_t h, void* stream, int64_t B,
                                 const void* query, const void* subkeys,
                                 const int32_t* idx, const float* weights, const float* dw,
                                 float* d_query, float* d_subkeys,
                                 void* workspace, size_t workspace_bytes);

/* ---- the row-sharded table with the library's record exchange (a9;
 * SURVEY.md 8(e); north_star: "row-sharded across the 8xB200 box, with ...
 * index all-to-all and partial-sum return"; BASELINE.json configs[3]).
 *
 * Rank p is home to its local_batch = B_l queries and owns value rows
 * [p n/P, (p+1) n/P) (owner(f) = f / (n/P)); the sub-keys are replicated.
 *   forward   SELECT: scoring a1-a2 and the Cartesian top-k + softmax a3-a4 of
 *             the local queries, fused with the ROUTE: every slot (b, h, t)
 *             becomes an 8-byte record {local row, w} in its owner's window for
 *             (this source, b) -- H*k slots per (source, query), records in
 *             (h, t) order, count in IN_CNT -- and the rows this rank owns are
 *             gathered right there into its own partial (a5, local shard);
 *             GATHER: every owner sums w V[row] over the records of each
 *             (remote source, query) and returns the partial row to the source;
 *             COMBINE: the home adds the P partials in owner order.
 *   backward  every owner reads the d_out rows its records need (from the
 *             home's DOUT), SCATTERs (dV shard +=, dw per record: the grouped
 *             deterministic reduction of msn_pkm_scatter, records summed in
 *             global contribution order -> dV shards bitwise equal to the
 *             unsharded dV) and returns dw per record -> COLLECT: the home puts
 *             dw back in (b, h, t) order -> backward_keys (a7-a8) locally.
 * Every rank has one exchange buffer of msn_pkm_exchange_layout() bytes (the
 * caller allocates it; zero-filled once before first use).  Two transports:
 *   MSN_XCHG_PEER   base[p] is rank p's buffer mapped into this process (torch
 *                   symmetric memory / CUDA IPC, NVLink peer memory): SELECT,
 *                   GATHER and SCATTER store straight into the peers' IN regions
 *                   (the all-to-all is issued by the compute kernels, record by
 *                   record and row by row: only the actual records and partials
 *                   cross NVLink); msn_pkm_exchange_barrier orders the ranks
 *                   (device-side flags, no host sync: graph-capturable).
 *                   msn_pkm_forward_sharded / msn_pkm_backward_sharded run the
 *                   whole step.
 *   MSN_XCHG_STAGED only base[rank] is used: outgoing data is staged in the OUT
 *                   regions (segment p for rank p) and the caller moves them
 *                   with fixed-size collectives (NCCL over NVLink, no host sync):
 *                   all-to-all OUT_ROW/OUT_W/OUT_CNT -> IN_ROW/IN_W/IN_CNT,
 *                   PART_OUT -> PART_IN, DW_OUT -> DW_IN, and an all-gather of
 *                   the homes' d_out into DOUT_ALL.  Whole windows move (P x
 *                   B_l*H*k records per rank): the baseline the peer transport
 *                   is measured against.
 * Region layout of one exchange buffer (cap = B_l*H*k: one window of H*k
 * records per query; offsets from msn_pkm_exchange_layout, 256-B aligned): */
enum {
  MSN_XREG_IN_ROW = 0,  /* int32 [P][B_l][H*k] local rows of the records source s sent here */
  MSN_XREG_IN_W,        /* fp32  [P][B_l][H*k] their weights */
  MSN_XREG_IN_CNT,      /* int32 [P][B_l]      records in window (s, b) */
  MSN_XREG_PART_IN,     /* fp32  [P][B_l][d_value] partial sums from owner o ([rank]: the local shard) */
  MSN_XREG_DOUT,        /* fp32  [B_l][d_value] this home's d_out (read by the owners) */
  MSN_XREG_DW_IN,       /* fp32  [P][B_l][H*k] dw returned by owner o, in o's window order */
  MSN_XREG_POS,         /* int32 [B_l*H*k] slot (b,h,t) -> its record's position in the window */
  MSN_XREG_CTL,         /* uint32 [64]: [0,P) barrier flags, [16] epoch, [17] barrier timeout */
  MSN_XREG_OUT_ROW,     /* STAGED only: int32 [P][B_l][H*k] records for owner p */
  MSN_XREG_OUT_W,       /*   fp32  [P][B_l][H*k] */
  MSN_XREG_OUT_CNT,     /*   int32 [P][B_l] */
  MSN_XREG_PART_OUT,    /*   fp32  [P][B_l][d_value] partials for home s */
  MSN_XREG_DOUT_ALL,    /*   fp32  [P][B_l][d_value] every home's d_out (all-gathered) */
  MSN_XREG_DW_OUT,      /*   fp32  [P][B_l][H*k] dw for home s, in this owner's window order */
  MSN_XREG_COUNT
};
typedef enum { MSN_XCHG_PEER = 0, MSN_XCHG_STAGED = 1 } msn_exchange_transport;
typedef struct {
  int32_t transport;    /* msn_exchange_transport */
  int32_t world;        /* P = max(config world_size, 1) */
  int32_t rank;         /* = config rank */
  int64_t local_batch;  /* B_l, the same on every rank */
  void* base[MSN_MAX_WORLD]; /* DEVICE pointers: base[p] = rank p's exchange buffer
                                (PEER: all P mapped here; STAGED: base[rank] only) */
} msn_pkm_exchange;

/* Byte offsets of the regions (offsets[MSN_XREG_COUNT], may be NULL) and the
 * total size of one exchange buffer for this handle and local_batch (STAGED
 * regions included when staged != 0). */
msn_status msn_pkm_exchange_layout(msn_pkm_t h, int64_t local_batch, int32_t staged,
                                   int64_t* offsets, size_t* bytes);

/* The whole sharded forward (PEER transport): SELECT (a1-a4 + route + the
 * local shard's gather), barrier, GATHER, barrier, COMBINE.  values = this rank's
 * rows [n/P, d_value]; out [B_l, d_value] fp32 (=); idx / weights [B_l,H,k]
 * (the tape, global slot ids).  Every rank calls it with the same B_l. */
msn_status msn_pkm_forward_sharded(msn_pkm_t h, void* stream, int64_t local_batch, const void* query,
                                   const void* subkeys, const void* values, const msn_pkm_exchange* x,
                                   float* out, int32_t* idx, float* weights, void* workspace,
                                   size_t workspace_bytes);
/* The whole sharded backward (PEER transport): d_out -> DOUT, barrier,
 * SCATTER (d_values += for this rank's rows), barrier, COLLECT (dw [B_l,H,k],
 * may be NULL), backward_keys (d_query =, d_subkeys += for the local
 * queries).  Workspace: msn_pkm_workspace_size(h, B_l, P * B_l). */
msn_status msn_pkm_backward_sharded(msn_pkm_t h, void* stream, int64_t local_batch, const float* d_out,
                                    const void* query, const void* subkeys, const void* values,
                                    const int32_t* idx, const float* weights, const msn_pkm_exchange* x,
                                    float* d_query, float* d_subkeys, float* d_values, float* dw,
                                    void* workspace, size_t workspace_bytes);

/* The phases (both transports; the STAGED caller moves the data in between;
 * ranks emulated on one GPU call them rank by rank, no barrier needed). */
/* SELECT: a1-a4 of the B_l local queries (idx / weights [B_l,H,k], the tape)
 * fused with the ROUTE into the owners' windows (+ POS, IN_CNT) and the gather
 * of the local shard's rows into PART_IN[rank] (PEER; PART_OUT[rank] when
 * STAGED; with P = 1 straight into out, which COMBINE then leaves as it is).
 * Workspace: msn_pkm_workspace_size(h, B_l, ...) forward bytes. */
msn_status msn_pkm_exchange_select(msn_pkm_t h, void* stream, const void* query, const void* subkeys,
                                   const void* values, const msn_pkm_exchange* x, int32_t* idx,
                                   float* weights, float* out, void* workspace, size_t workspace_bytes);
/* GATHER: for every REMOTE source s and query b, the partial sum of w V[row]
 * over the records of window (s, b) -> PART_IN[rank][b] of rank s (PEER) or
 * PART_OUT[s][b] (STAGED); zeros for an empty window. */
msn_status msn_pkm_exchange_gather(msn_pkm_t h, void* stream, const void* values, const msn_pkm_exchange* x);
/* COMBINE: out[b] = sum_o PART_IN[o][b], o ascending (=); P = 1: nothing to
 * add (SELECT wrote out). */
msn_status msn_pkm_exchange_combine(msn_pkm_t h, void* stream, const msn_pkm_exchange* x, float* out);
/* SCATTER: dV shard (+=) and dw of every record in the IN windows, d_out rows
 * from the homes' DOUT (PEER) or DOUT_ALL (STAGED); dw -> DW_IN[rank] of the
 * home (PEER) or DW_OUT[s] (STAGED), in window order.  Workspace as
 * msn_pkm_backward_sharded. */
msn_status msn_pkm_exchange_scatter(msn_pkm_t h, void* stream, const void* values, float* d_values,
                                    const msn_pkm_exchange* x, void* workspace, size_t workspace_bytes);
/* COLLECT: dw[b,h,t] = DW_IN[owner][b][POS[b,h,t]] (=). */
msn_status msn_pkm_exchange_collect(msn_pkm_t h, void* stream, const int32_t* idx,
                                    const msn_pkm_exchange* x, float* dw);
/* Device-side barrier over the P ranks (PEER): release-store of an epoch into
 * every rank's CTL flag [rank], then acquire-spin until all P flags of this
 * rank reach it.  Bounded: a rank that waits more than 10 s (a peer that
 * never arrives) sets CTL[17] = 1 and returns instead of hanging the GPU;
 * the results of that step are then invalid (the caller may check CTL[17]). */
msn_status msn_pkm_exchange_barrier(msn_pkm_t h, void* stream, const msn_pkm_exchange* x);

/* Tape check (SURVEY 8(b) "Errors"): *bad (DEVICE int32, written =, zeroed
 * on the stream first) = the number of slots (b, h, t) of idx / weights
 * [B, H, k] that are not what a4 produces: idx outside the
 * lookup's table ([0, n_sub^2), or [g n_sub^2, (g+1) n_sub^2) for head group g
 * under MSN_FLAG_GROUP_TABLES), an id repeated within one lookup (each copy
 * counts), or a weight that is not in [0, 1] (NaN included).  Asynchronous,
 * no host sync, graph-capturable.  The softmax normalisation itself is not
 * checked. */
msn_status msn_pkm_validate_tape(msn_pkm_t h, void* stream, int64_t B, const int32_t* idx,
                                 const float* weights, int32_t* bad);

/* Number of kernel launches the last forward/backward/phase call enqueued
 * (for the bench's gpu_launches count). */
int32_t msn_pkm_last_launch_count(msn_pkm_t h);

/* Tracing: caller-created cudaEvent_t handles (n <= 4, n = 0 disables) that
 * the library records on the call's stream at internal stage boundaries.
 * events[0]: after the scoring + per-half top-k stage of msn_pkm_forward /
 * msn_pkm_select; events[1]: after the Cartesian top-k + softmax stage (the
 * same point as events[0] when forward fuses that stage into the gather). */
msn_status msn_pkm_set_trace_events(msn_pkm_t h, void* const* events, int32_t n);

const char* msn_pkm_status_string(msn_status s);
const char* msn_pkm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* MSN_PKM_H_ */
