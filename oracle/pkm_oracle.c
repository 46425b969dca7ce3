/*
 * pkm_oracle.c -- plain, slow, fp64 CPU oracle of the PKM lookup
 * (MSN, arXiv 2602.07526, section 3.3), forward and backward.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or constant with the CUDA path
 * (paper_2602_07526_b200/csrc) and includes nothing from it.
 *
 * Every step follows the paper's equations in the paper's order, in fp64,
 * with plain loops and no blocking/fusion/reordering:
 *
 *   (S_old)   S_row = K_row q_row, S_col = K_col q_col
 *   (argtopk) I = argtopk_i S_row, J = argtopk_j S_col,
 *             K = argtopk_{(i,j) in I x J} S_row[i] + S_col[j] PAPER.md:218-222
 *   (vo_mem)  v_o = sum_{(i,j) in K} S[i,j] V[flat(i,j)]
 *
 * Readings of the paper taken here:
 *   R1 weights are a softmax over the k selected scores, temperature 1,
 *      max-subtracted (prose "softmax-weighted sum"; the printed
 *      linear normalisation, is not used).
 *   R2 flat(i,j) = i*n_sub + j (PAPER.md:229 prints (sqrt(n)-1)*i + j, which is
 *      not injective).
 *   R3 indices are 0-based ("i in [0, sqrt(n)-1]").
 *   R4 query half 0 scores against K_row (index i), half 1 against K_col (j).
 *   R5 ties: per half (score desc, index asc); pairs (score desc, flat asc);
 *      the output lists the k selected pairs in that order.
 *   R7 heads: per-head sub-key codebooks, one shared value table, output
 *      summed over heads (h ascending).
 *   R10 no gradient through the selection; gradient flows through the
 *      selected scores only ("unselected keys receive no gradients",
 *      PAPER.md:282-284).
 *   R11 "scatter-adds gradients into the value table" is read
 *      as dV += (a gradient buffer), not an optimiser update.
 *
 * Inputs are the exact stored values the GPU consumes (fp32 or bf16 bit
 * patterns, or fp64 for finite-difference tests), widened to fp64 here.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define DT_F32 0
#define DT_BF16 1
#define DT_F64 2

/* widen one stored element to fp64 */
static double load_elem(const void* base, int dtype, int64_t i) {
    if (dtype == DT_F32) return (double)((const float*)base)[i];
    if (dtype == DT_F64) return ((const double*)base)[i];
    /* bf16: the 16 stored bits are the top half of an fp32 pattern */
    uint32_t bits = ((uint32_t)((const uint16_t*)base)[i]) << 16;
    float f;
    memcpy(&f, &bits, sizeof f);
    return (double)f;
}

typedef struct { double s; int64_t i; } scored_t;

/* (score desc, index asc) -- the total order of reading R5 */
static int cmp_desc_asc(const void* a, const void* b) {
    const scored_t* x = (const scored_t*)a;
    const scored_t* y = (const scored_t*)b;
    if (x->s > y->s) return -1;
    if (x->s < y->s) return 1;
    if (x->i < y->i) return -1;
    if (x->i > y->i) return 1;
    return 0;
}

/* Q[b][h][half][e] */
static int64_t q_off(int64_t b, int h, int half, int H, int d_h) {
    return (((int64_t)b * H + h) * 2 + half) * d_h;
}
/* K[h][half][i][e] */
static int64_t k_off(int h, int half, int64_t i, int n_sub, int d_h) {
    return (((int64_t)h * 2 + half) * n_sub + i) * d_h;
}

/* Eq. (S_old): S[i] = sum_e K[h][half][i][e] * q[e], e ascending. */
static void score_half(const void* Q, int qdt, const void* K, int kdt, int64_t b, int h, int half,
                       int H, int n_sub, int d_h, double* S) {
    const int64_t qo = q_off(b, h, half, H, d_h);
    for (int64_t i = 0; i < n_sub; ++i) {
        const int64_t ko = k_off(h, half, i, n_sub, d_h);
        double acc = 0.0;
        for (int e = 0; e < d_h; ++e) acc += load_elem(K, kdt, ko + e) * load_elem(Q, qdt, qo + e);
        S[i] = acc;
    }
}

/* argtopk over one half: the first k entries of (S desc, i asc). */
static void argtopk_half(const double* S, int n_sub, int k, scored_t* tmp, int64_t* idx, double* val) {
    for (int64_t i = 0; i < n_sub; ++i) { tmp[i].s = S[i]; tmp[i].i = i; }
    qsort(tmp, (size_t)n_sub, sizeof(scored_t), cmp_desc_asc);
    for (int a = 0; a < k; ++a) { idx[a] = tmp[a].i; val[a] = tmp[a].s; }
}

/*
 * Forward.  For each query b and head h (lookups are independent):
 *   1. S1 = K[h,0] q[b,h,0], S2 = K[h,1] q[b,h,1]                  (S_old)
 *   2. I = argtopk S1, J = argtopk S2                              (argtopk)
 *   3. all k^2 pairs (i,j) in I x J: c = S1[i] + S2[j], f = i*n_sub + j (no pruning)
 *   4. T = first k pairs in (c desc, f asc) order
 *   5. w_t = exp(c_t - c_T0) / sum_u exp(c_u - c_T0)               (R1)
 *   6. out[b] += sum_t w_t V[f_t] (t ascending, then h ascending)  (vo_mem)
 * Outputs (any may be NULL except idx):
 *   I_out, J_out [B,H,k] int64; s1_out, s2_out [B,H,k] per-half top scores;
 *   idx [B,H,k] int64 flat slots; c_out, w_out [B,H,k];
 *   out [B,d_v] (sum over heads); out_ph [B,H,d_v] (per head).
 * Returns 0, or -1 on bad arguments / allocation failure.
 */
int pkm_oracle_forward(int64_t B, int H, int n_sub, int d_h, int d_v, int k,
                       const void* Q, int qdt, const void* K, int kdt, const void* V, int vdt,
                       int64_t* I_out, int64_t* J_out, double* s1_out, double* s2_out,
                       int64_t* idx, double* c_out, double* w_out,
                       double* out, double* out_ph, int nthreads) {
    if (B < 0 || H < 1 || n_sub < 1 || d_h < 1 || d_v < 1 || k < 1 || k > n_sub || !idx) return -1;
    int bad = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
#endif
    for (int64_t b = 0; b < B; ++b) {
        double* S1 = (double*)malloc(sizeof(double) * (size_t)n_sub);
        double* S2 = (double*)malloc(sizeof(double) * (size_t)n_sub);
        scored_t* tmp = (scored_t*)malloc(sizeof(scored_t) * (size_t)(n_sub > k * k ? n_sub : k * k));
        int64_t* I = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
        int64_t* J = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
        double* v1 = (double*)malloc(sizeof(double) * (size_t)k);
        double* v2 = (double*)malloc(sizeof(double) * (size_t)k);
        double* w = (double*)malloc(sizeof(double) * (size_t)k);
        if (!S1 || !S2 || !tmp || !I || !J || !v1 || !v2 || !w) { bad = 1; goto done; }
        if (out) for (int e = 0; e < d_v; ++e) out[b * d_v + e] = 0.0;
        for (int h = 0; h < H; ++h) {
            const int64_t o = ((int64_t)b * H + h) * k;
            /* 1 */
            score_half(Q, qdt, K, kdt, b, h, 0, H, n_sub, d_h, S1);
            score_half(Q, qdt, K, kdt, b, h, 1, H, n_sub, d_h, S2);
            /* 2 */
            argtopk_half(S1, n_sub, k, tmp, I, v1);
            argtopk_half(S2, n_sub, k, tmp, J, v2);
            if (I_out) for (int a = 0; a < k; ++a) I_out[o + a] = I[a];
            if (J_out) for (int a = 0; a < k; ++a) J_out[o + a] = J[a];
            if (s1_out) for (int a = 0; a < k; ++a) s1_out[o + a] = v1[a];
            if (s2_out) for (int a = 0; a < k; ++a) s2_out[o + a] = v2[a];
            /* 3 */
            for (int a = 0; a < k; ++a)
                for (int c = 0; c < k; ++c) {
                    tmp[a * k + c].s = S1[I[a]] + S2[J[c]];
                    tmp[a * k + c].i = I[a] * (int64_t)n_sub + J[c];
                }
            /* 4 */
            qsort(tmp, (size_t)k * (size_t)k, sizeof(scored_t), cmp_desc_asc);
            /* 5 */
            const double m = tmp[0].s;
            double z = 0.0;
            for (int t = 0; t < k; ++t) { w[t] = exp(tmp[t].s - m); z += w[t]; }
            for (int t = 0; t < k; ++t) w[t] /= z;
            for (int t = 0; t < k; ++t) {
                idx[o + t] = tmp[t].i;
                if (c_out) c_out[o + t] = tmp[t].s;
                if (w_out) w_out[o + t] = w[t];
            }
            /* 6 */
            if (out_ph) for (int e = 0; e < d_v; ++e) out_ph[o / k * d_v + e] = 0.0;
            for (int t = 0; t < k; ++t) {
                const int64_t row = tmp[t].i * (int64_t)d_v;
                for (int e = 0; e < d_v; ++e) {
                    const double x = w[t] * load_elem(V, vdt, row + e);
                    if (out) out[b * d_v + e] += x;
                    if (out_ph) out_ph[((int64_t)b * H + h) * d_v + e] += x;
                }
            }
        }
    done:
        free(S1); free(S2); free(tmp); free(I); free(J); free(v1); free(v2); free(w);
    }
    return bad ? -1 : 0;
}

/*
 * fp64 score S1[i] + S2[j] of arbitrary slots f = i*n_sub + j (used by the
 * tie rule of the parity comparator: "any swapped slot must have a score gap
 * <= 1e-5 relative", BASELINE.json north_star).  slots/out are [B,H,m].
 */
int pkm_oracle_slot_scores(int64_t B, int H, int n_sub, int d_h, const void* Q, int qdt,
                           const void* K, int kdt, const int64_t* slots, int m, double* out,
                           int nthreads) {
    if (B < 0 || H < 1 || n_sub < 1 || d_h < 1 || m < 0 || !slots || !out) return -1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t b = 0; b < B; ++b)
        for (int h = 0; h < H; ++h)
            for (int t = 0; t < m; ++t) {
                const int64_t o = ((int64_t)b * H + h) * m + t;
                const int64_t f = slots[o];
                const int64_t i = f / n_sub, j = f % n_sub;
                double s1 = 0.0, s2 = 0.0;
                const int64_t q0 = q_off(b, h, 0, H, d_h), q1 = q_off(b, h, 1, H, d_h);
                const int64_t k0 = k_off(h, 0, i, n_sub, d_h), k1 = k_off(h, 1, j, n_sub, d_h);
                for (int e = 0; e < d_h; ++e) s1 += load_elem(K, kdt, k0 + e) * load_elem(Q, qdt, q0 + e);
                for (int e = 0; e < d_h; ++e) s2 += load_elem(K, kdt, k1 + e) * load_elem(Q, qdt, q1 + e);
                out[o] = s1 + s2;
            }
    return 0;
}

/* position of row r in the sorted list rows[0..n) or -1 */
static int64_t find_row(const int64_t* rows, int64_t n, int64_t r) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (rows[mid] < r) lo = mid + 1; else hi = mid;
    }
    return (lo < n && rows[lo] == r) ? lo : -1;
}

/*
 * Backward at a given selection idx [B,H,k] (the oracle's own forward
 * output), for the scalar loss L = <dOut, out>:
 *   7.  dw_t = <V[f_t], dOut[b]>;  dV[f_t] += w_t dOut[b]
 *   8.  g = sum_t w_t dw_t;  ds_t = w_t (dw_t - g)          (softmax Jacobian)
 *   9.  i_t = f_t div n_sub, j_t = f_t mod n_sub; dS1[i_t] += ds_t; dS2[j_t] += ds_t
 *   10. dK[h,0,i] += dS1[i] q[b,h,0];  dK[h,1,j] += dS2[j] q[b,h,1]
 *   11. dQ[b,h,0] = sum_i dS1[i] K[h,0,i];  dQ[b,h,1] = sum_j dS2[j] K[h,1,j]
 * The weights w are recomputed from the scores at idx (step 1 and R1 with
 * the max over the k selected scores subtracted).
 * Outputs: dQ [B,H,2,d_h] (=), dK [H,2,n_sub,d_h] (=, fully written),
 * dV: if rows != NULL, compact [n_rows, d_v] over the sorted row list rows
 * (every selected slot must be in it), else dense [n_sub^2, d_v]; (=).
 * dw_out, ds_out [B,H,k] optional.  Accumulation into dV and dK runs in b
 * ascending, then h, then t order on one thread (deterministic).
 * Returns 0, -1 bad args, -2 a selected slot is missing from rows.
 */
int pkm_oracle_backward(int64_t B, int H, int n_sub, int d_h, int d_v, int k,
                        const void* Q, int qdt, const void* K, int kdt, const void* V, int vdt,
                        const int64_t* idx, const double* dOut,
                        double* dQ, double* dK, double* dV, const int64_t* rows, int64_t n_rows,
                        double* dw_out, double* ds_out, int nthreads) {
    if (B < 0 || H < 1 || n_sub < 1 || d_h < 1 || d_v < 1 || k < 1 || !idx || !dOut) return -1;
    const int64_t L = B * H;
    double* W = (double*)malloc(sizeof(double) * (size_t)(L * k + 1));
    double* DS = (double*)malloc(sizeof(double) * (size_t)(L * k + 1));
    if (!W || !DS) { free(W); free(DS); return -1; }
    int bad = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 4) reduction(| : bad)
#endif
    for (int64_t l = 0; l < L; ++l) {
        const int64_t b = l / H;
        const int h = (int)(l % H);
        const int64_t o = l * k;
        double* c = (double*)malloc(sizeof(double) * (size_t)k);
        double* dw = (double*)malloc(sizeof(double) * (size_t)k);
        if (!c || !dw) { bad = 1; free(c); free(dw); continue; }
        /* scores at the given selection (S_old), then R1 softmax */
        double m = -INFINITY;
        for (int t = 0; t < k; ++t) {
            const int64_t f = idx[o + t], i = f / n_sub, j = f % n_sub;
            double s1 = 0.0, s2 = 0.0;
            for (int e = 0; e < d_h; ++e)
                s1 += load_elem(K, kdt, k_off(h, 0, i, n_sub, d_h) + e) * load_elem(Q, qdt, q_off(b, h, 0, H, d_h) + e);
            for (int e = 0; e < d_h; ++e)
                s2 += load_elem(K, kdt, k_off(h, 1, j, n_sub, d_h) + e) * load_elem(Q, qdt, q_off(b, h, 1, H, d_h) + e);
            c[t] = s1 + s2;
            if (c[t] > m) m = c[t];
        }
        double z = 0.0;
        for (int t = 0; t < k; ++t) { W[o + t] = exp(c[t] - m); z += W[o + t]; }
        for (int t = 0; t < k; ++t) W[o + t] /= z;
        /* 7: dw */
        for (int t = 0; t < k; ++t) {
            const int64_t row = idx[o + t] * (int64_t)d_v;
            double acc = 0.0;
            for (int e = 0; e < d_v; ++e) acc += load_elem(V, vdt, row + e) * dOut[b * d_v + e];
            dw[t] = acc;
        }
        /* 8: ds */
        double g = 0.0;
        for (int t = 0; t < k; ++t) g += W[o + t] * dw[t];
        for (int t = 0; t < k; ++t) DS[o + t] = W[o + t] * (dw[t] - g);
        if (dw_out) for (int t = 0; t < k; ++t) dw_out[o + t] = dw[t];
        if (ds_out) for (int t = 0; t < k; ++t) ds_out[o + t] = DS[o + t];
        /* 9 + 11: dQ = sum_i dS1[i] K[h,0,i] -- dS1 accumulated first */
        if (dQ) {
            for (int half = 0; half < 2; ++half) {
                double* dq = dQ + q_off(b, h, half, H, d_h);
                for (int e = 0; e < d_h; ++e) dq[e] = 0.0;
                /* distinct sub-key indices in first-appearance order */
                for (int t = 0; t < k; ++t) {
                    const int64_t f = idx[o + t];
                    const int64_t r = half == 0 ? f / n_sub : f % n_sub;
                    int seen = 0;
                    for (int u = 0; u < t; ++u) {
                        const int64_t fu = idx[o + u];
                        if ((half == 0 ? fu / n_sub : fu % n_sub) == r) { seen = 1; break; }
                    }
                    if (seen) continue;
                    double dS = 0.0;
                    for (int u = t; u < k; ++u) {
                        const int64_t fu = idx[o + u];
                        if ((half == 0 ? fu / n_sub : fu % n_sub) == r) dS += DS[o + u];
                    }
                    for (int e = 0; e < d_h; ++e) dq[e] += dS * load_elem(K, kdt, k_off(h, half, r, n_sub, d_h) + e);
                }
            }
        }
        free(c);
        free(dw);
    }
    if (bad) { free(W); free(DS); return -1; }
    /* serial, fixed-order scatter-adds: dV (step 7) and dK (steps 9-10) */
    if (dK) memset(dK, 0, sizeof(double) * (size_t)H * 2 * (size_t)n_sub * (size_t)d_h);
    if (dV) {
        const int64_t nr = rows ? n_rows : (int64_t)n_sub * n_sub;
        memset(dV, 0, sizeof(double) * (size_t)nr * (size_t)d_v);
    }
    int rc = 0;
    for (int64_t l = 0; l < L; ++l) {
        const int64_t b = l / H;
        const int h = (int)(l % H);
        const int64_t o = l * k;
        for (int t = 0; t < k; ++t) {
            const int64_t f = idx[o + t];
            if (dV) {
                int64_t r = rows ? find_row(rows, n_rows, f) : f;
                if (r < 0) { rc = -2; continue; }
                for (int e = 0; e < d_v; ++e) dV[r * d_v + e] += W[o + t] * dOut[b * d_v + e];
            }
            if (dK) {
                const int64_t i = f / n_sub, j = f % n_sub;
                double* dk0 = dK + k_off(h, 0, i, n_sub, d_h);
                double* dk1 = dK + k_off(h, 1, j, n_sub, d_h);
                for (int e = 0; e < d_h; ++e) dk0[e] += DS[o + t] * load_elem(Q, qdt, q_off(b, h, 0, H, d_h) + e);
                for (int e = 0; e < d_h; ++e) dk1[e] += DS[o + t] * load_elem(Q, qdt, q_off(b, h, 1, H, d_h) + e);
            }
        }
    }
    free(W);
    free(DS);
    return rc;
}
