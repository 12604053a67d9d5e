/*
 * specexit_b200.h -- C ABI of the B200-native SpecEE speculative early-exit
 * predictor path (libspecexit_b200.so, sm_100a).
 *
 * This is the drop-in boundary.  In the reference (a numpy/Cython package,
 * /root/reference/pkg) the only native slot is the kernel backend registry
 * `_BACKENDS` (src/specexit/kernels/__init__.py:25-31) whose entries export
 * `matmul_f32` / `seq_sum_f32` (src/specexit/kernels/_ckern.pyx:16-46).  This
 * library replaces that slot at the OPERATOR level: each export is one fused
 * operator of the predictor path, called by the Python drop-in package
 * (paper_2504_08850_b200/, same names/signatures as `specexit`) through ctypes.
 *
 * Conventions (all exports):
 *   - every pointer is a DEVICE pointer allocated by the caller; the library
 *     never allocates, frees or synchronises;
 *   - all work is enqueued on `stream` (cudaStream_t passed as void*);
 *   - return 0 on success, SPX_EINVAL (-1) for arguments rejected on the
 *     host, SPX_ECUDA (-2) if the launch failed;
 *   - in-kernel input violations (token id out of range, non-finite values,
 *     bad probability vector) OR bits into the caller's device error word
 *     `err`; the Python wrapper maps them to the reference's ValueError
 *     messages at its next synchronisation point;
 *   - weight tensors are passed as void* with a SPX_DTYPE_* tag (bf16 = raw
 *     bfloat16 bits; f32 for reference weights that are not bf16-exact).
 */
#ifndef SPECEXIT_B200_H
#define SPECEXIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPX_EINVAL (-1)
#define SPX_ECUDA (-2)

#define SPX_MODE_FAST 0   /* canonical 128-partial reductions (production) */
#define SPX_MODE_STRICT 1 /* reference order: sequential, no FMA (parity)   */

#define SPX_DTYPE_BF16 0  /* weight storage: bfloat16 (production)           */
#define SPX_DTYPE_F32 1   /* weight storage: float32 (exact reference weights) */

#define SPX_POLICY_MLP 0      /* PredictorPolicy  (engine.py:83-92)             */
#define SPX_POLICY_CONST 1    /* Never/AlwaysExitPolicy (engine.py:67-80)       */

/* error-word bits */
#define SPX_ERR_ID_RANGE 1
#define SPX_ERR_HIDDEN_NONFINITE 2
#define SPX_ERR_LOGIT_NONFINITE 4
#define SPX_ERR_PREV_SUM 8
#define SPX_ERR_BAD_LAYER 16
#define SPX_ERR_ROW_CAP 32        /* a layer call selected more rows than row_cap */

/* K1+K2+K3 -- fused predictor evaluation for B rows at ONE layer.
 * Replaces, per row, the reference chain
 *   sliced_head_logits   (src/specexit/model.py:298-314)
 *   extract_features     (src/specexit/predictor.py:42-52)
 *   predictor_forward    (src/specexit/predictor.py:97-103)
 *   decide_exit          (src/specexit/predictor.py:106-109)
 * as used in ExitEngine.step (src/specexit/engine.py:192-200). */
typedef struct {
  const float *hidden;       /* (B, d) f32 residual rows                       */
  int64_t hidden_stride;     /* elements between rows (0 -> d)                 */
  const float *norm_g;       /* (d) final_norm.g                               */
  const float *norm_b;       /* (d) final_norm.b                               */
  const void *head;          /* (V, d) LM head, vocab-row major                */
  int32_t head_dtype;        /* SPX_DTYPE_*                                    */
  const float *head_bw;      /* (V) spx_head_bias output (FAST mode; NULL = 0) */
  const int32_t *ids;        /* (B, K) speculative token ids                   */
  float *prev;               /* (B, K) in: previous local probs, out: new ones */
  const float *w1;           /* (3K, H) predictor W1 (row-major, as reference) */
  const float *b1;           /* (H)                                            */
  const float *w2;           /* (H)                                            */
  float b2;                  /* f32 output bias                                */
  float z_cut;               /* fire iff z2 >= z_cut  (== sigmoid(z2) > thr)   */
  int32_t policy;            /* SPX_POLICY_*                                   */
  double const_prob;         /* SPX_POLICY_CONST: the policy's probability     */
  double threshold;          /* SPX_POLICY_CONST: fire iff const_prob > thr    */
  float *logits_out;         /* (B, K) optional                                */
  float *feat_out;           /* (B, 3K) optional FeatureVector.concat()        */
  float *z_out;              /* (B) optional pre-sigmoid f32                   */
  double *prob_out;          /* (B) optional f64 probability                   */
  uint8_t *fired;            /* (B) optional decision                          */
  const uint64_t *row_layer_mask; /* (B) optional: skip row unless bit `layer` */
  const uint8_t *row_done;   /* (B) optional: skip row if nonzero (exited)     */
  int32_t *evals;            /* (B) optional per-row evaluation counter        */
  int32_t layer;
  int32_t mode;              /* SPX_MODE_*                                     */
  int32_t pdl;               /* 1: programmatic dependent launch (overlap the  */
                             /*    prologue with the previous kernel);         */
                             /* 2: as 1, and `ids` is not written by the       */
                             /*    immediately preceding kernel, so the        */
                             /*    LM-head row prefetch of each team's first   */
                             /*    rows starts before griddepcontrol.wait     */
                             /*    (ignored when row_done / row_layer_mask     */
                             /*    are given: those flags are written late)    */
  int32_t *err;              /* device error word                              */
  int64_t B, d, V, K, H;
  /* ---- FAST-mode decision certification.  When
   * `recheck` is given, every FAST decision is either certified equal to the
   * reference's (|z2 - z_cut| beyond the stated FAST-vs-strict error bound of
   * that row) or the row is re-evaluated by the STRICT chain in a follow-up
   * launch enqueued by this same call, so `fired` matches the reference's
   * `prob > threshold` (predictor.py:106-109) row for row.               */
  const float *head_wmax;    /* (V) max_j |head[v][j]| (spx_head_stats)        */
  const float *cert;         /* (3K+2) spx_predictor_cert of this layer's MLP  */
  float cert_kappa;          /* 2 * lambda * 2^-24 * sqrt(d)  (lambda = 8)      */
  float cert_hnorm;          /* max|final_norm.g| * sqrt(d) + ||final_norm.b||  */
  float *prev_err;           /* (B) in: bound on |prev - prev_ref|; out: bound */
                             /*     for the new probabilities (0 after STRICT) */
  int32_t *recheck;          /* (5 + B) zeroed once by the caller, self-reset: */
                             /* [0] rows deferred, [1] CTA ticket, [2] pop     */
                             /* cursor, [3] total rows re-evaluated            */
                             /* (cumulative), [4] rows whose STRICT decision   */
                             /* still sat inside the carried prev bound        */
                             /* (cumulative), [5..] row list                   */
  uint8_t *fired_any;        /* (B) optional: fired_any[r] |= fired[r] (the    */
                             /*     token's predictor_fired, engine.py:199)    */
} spx_predictor_args;
int spx_predictor_eval(const spx_predictor_args *args, void *stream);

/* SPLIT form of spx_predictor_eval for large batches (FAST mode, bf16 head,
 * K <= 8, d in {2048, 4096, 8192}; spx_predictor_split_ok tells): the same
 * outputs, bit for bit, from two launches --
 *   spx_predictor_gather: LayerNorm + K-row gather + local logits (K1) into
 *     inter (B, 2K + 2) f32 = {local logits, wmax[id], lnf, flags}; reads neither
 *     prev nor the predictor.  args->pdl = 3: the inputs are not written by
 *     the preceding kernel, so consecutive gathers overlap (programmatic
 *     dependent launch, no griddepcontrol.wait).
 *   spx_predictor_tail: features + MLP + decision + certification (K2+K3)
 *     from inter; carries prev.  May run on another stream, concurrently
 *     with the next layer's gather.
 * Replaces the same reference chain as spx_predictor_eval
 * (src/specexit/model.py:298-314, src/specexit/predictor.py:42-109). */
int spx_predictor_split_ok(const spx_predictor_args *args);
int spx_predictor_gather(const spx_predictor_args *args, float *inter, void *stream);
int spx_predictor_tail(const spx_predictor_args *args, const float *inter, void *stream);
/* PIPELINED split form: ONE launch = the gather of `args` (layer l, into
 * inter) + the tail of `tail_args` (layer l-1, from tail_inter), the tail
 * warps starting once the preceding launch (layer l-1's gather) completes.
 * A chain gather(0), gather_tail(1, 0), ..., gather_tail(L-1, L-2),
 * tail(L-1) evaluates L layers with the prev chain carried and every gather
 * overlapping its neighbours (always programmatic dependent launch). */
int spx_predictor_gather_tail(const spx_predictor_args *args, float *inter,
                              const spx_predictor_args *tail_args, const float *tail_inter,
                              void *stream);
/* The chain's last step: the tail of `tail_args` by the pipelined kernel's
 * tail warps with an empty gather (one warp per row across the grid), after
 * the preceding launch completes. */
int spx_predictor_tail_pipelined(const spx_predictor_args *tail_args, const float *tail_inter,
                                 void *stream);

/* Per-layer constants of the certification bound for one predictor:
 * cert[i] = sum_j |w2[j]| |w1[i][j]| (i < 3K), cert[3K] = sum_j |w2[j] b1[j]|,
 * cert[3K+1] = sum_j |w2[j]|. */
int spx_predictor_cert(const float *w1, const float *b1, const float *w2, int64_t K, int64_t H,
                       float *cert, void *stream);
/* Per-vocabulary-row statistics of the LM head: wmax[v] = max_j |head[v][j]|. */
int spx_head_stats(const void *head, int32_t head_dtype, int64_t V, int64_t d, float *wmax,
                   void *stream);

/* extract_features alone (src/specexit/predictor.py:42-52) for B rows:
 * feats_out (B, 3K) = [logits | softmax | softmax - prev]; prev is read only. */
int spx_extract_features(const float *logits, const float *prev, float *feats_out, int32_t *err,
                         int64_t B, int64_t K, void *stream);
/* predictor_forward alone (src/specexit/predictor.py:97-103) + decide_exit
 * (:106-109) for B feature rows (B, 3K); any output pointer may be NULL. */
int spx_predictor_mlp(const float *feats, const float *w1, const float *b1, const float *w2,
                      float b2, float z_cut, float *z_out, double *prob_out, uint8_t *fired_out,
                      int64_t B, int64_t K, int64_t H, void *stream);

/* K4 -- full-head verification: argmax over V of LN(h) . head for each gated
 * row, lowest index on ties (np.argmax), membership in the row's verify set.
 * Replaces verify_exit (src/specexit/engine.py:59-64) / full_head_logits
 * (src/specexit/model.py:289-295) / the final-layer argmax (engine.py:208-210)
 * / TreeEngine._verify_path (src/specexit/tree.py:274-283).
 * On a verified row with `done_out` given it also writes the device exit
 * flag: done_out[r]=1, exit_layer_out[r]=layer -- later layer kernels read it
 * and return early (no host sync). */
typedef struct {
  const float *hidden; int64_t hidden_stride;   /* (B, d) */
  const float *norm_g, *norm_b;
  const void *head;                             /* (V, d) */
  int32_t head_dtype;                           /* SPX_DTYPE_* */
  const float *head_bw;                         /* (V) spx_head_bias (FAST); NULL = 0 */
  const uint8_t *gate;        /* (B) optional: row computed iff gate[r] != 0  */
  const uint8_t *row_done;    /* (B) optional: row skipped if nonzero         */
  const int32_t *spec_ptr;    /* (B+1) optional CSR offsets of verify sets    */
  const int32_t *spec_ids;    /* verify-set ids                               */
  int32_t *token_out;         /* (B) argmax token (written for computed rows) */
  uint8_t *verified_out;      /* (B) optional argmax in verify set            */
  float *maxlogit_out;        /* (B) optional                                 */
  float *logits_out;          /* (B, V) optional full logits                  */
  uint8_t *done_out;          /* (B) optional exit flag, set when verified    */
  int32_t *exit_layer_out;    /* (B) optional                                 */
  int32_t *full_heads;        /* (B) optional counter += 1 per computed row   */
  int32_t layer;
  unsigned long long *scratch;  /* (B) zeroed once by the caller; self-reset  */
  unsigned int *counter;        /* (1) zeroed once by the caller; self-reset  */
  int32_t mode;
  int32_t *err;
  int64_t B, d, V;
  /* optional (FAST, bf16 head, d % 64 == 0, B >= SPX_VERIFY_TC_MIN_ROWS, no
   * logits_out): the tensor-core form -- the head read once per 128 gated
   * rows (UMMA over an exact three-part bf16 split of the normalised rows),
   * candidates within a stated bound of the max re-evaluated in the CDOT
   * order, so tokens / max logits / flags are bit-identical to the CUDA-core
   * form.  tc_scratch >= spx_verify_tc_scratch_bytes(B, d, V) bytes. */
  const float *head_wmax;     /* (V) spx_head_stats                           */
  void *tc_scratch;
  /* optional, tensor-core form only: the stable top-K ids (value desc, index
   * asc; speculation.py:57-60) of each computed row's CDOT logits, (B, topk_k)
   * row-major, 1 <= topk_k <= 64 -- the draft proposal without full logits. */
  int32_t *topk_out;
  int32_t topk_k;
} spx_verify_args;
#define SPX_VERIFY_TC_MIN_ROWS 8
int spx_verify(const spx_verify_args *args, void *stream);
int64_t spx_verify_tc_scratch_bytes(int64_t B, int64_t d, int64_t V);
/* byte offset in tc_scratch of the tensor-core logits of the last
 * tensor-core verify call: (computed rows in row order, V) f32, r * D + bw
 * (FAST-tolerance logits; the exact ids come from topk_out / token_out).
 * The tensor-core form runs for B >= SPX_VERIFY_TC_MIN_ROWS, or any B when
 * topk_out is given. */
int64_t spx_verify_tc_logits_offset(int64_t B, int64_t d, int64_t V);

/* K5 -- two-level scheduler on device (src/specexit/scheduler.py:49-102).
 * Per row: ring of the last `queue_len` exit layers + neighbour counts. */
typedef struct {
  int32_t *queue;    /* (B, queue_len) ring storage                            */
  int32_t *head;     /* (B) slot of the oldest entry                           */
  int32_t *len;      /* (B) entries held                                       */
  int32_t *counts;   /* (B, L) neighbour counts (scheduler.py:54-58)           */
} spx_online_state;
/* update_online (scheduler.py:65-79) for each row r with gate[r] (or all). */
int spx_sched_update(spx_online_state st, const int32_t *exit_layer, const uint8_t *gate,
                     int64_t B, int32_t L, int32_t queue_len, int32_t radius, int32_t *err,
                     void *stream);
/* active_layers (scheduler.py:95-102): bit i of active_out[r] set iff
 * i <= L-2 and (offline bit i or counts[r][i] > 0); mode 0 = "all" layers
 * (engine.py:170-174). L <= 64. */
int spx_sched_active(spx_online_state st, uint64_t offline_mask, int64_t B, int32_t L,
                     int32_t mode, uint64_t *active_out, void *stream);

/* K6 -- context-aware merged mapping (src/specexit/tree.py:92-113): logits of
 * the (node, id) pairs with each UNIQUE id's LM-head row read once.  uniq (U)
 * are the distinct ids; the pairs of unique id u are uniq_ptr[u]..uniq_ptr[u+1]
 * with pair_node (row of xg) and pair_out (index into logits).  xg / r are the
 * spx_head_prep outputs of the N node rows.  FAST: logit = r*CDOT(xg,W)+bw,
 * bit-identical to K1's logits; STRICT: xg holds the reference LayerNorm rows
 * and each logit is the reference's sequential dot. */
int spx_tree_merged_logits(const float *xg, const float *r, int64_t N, const void *head,
                           int32_t head_dtype, const float *head_bw, int64_t V, int64_t d,
                           const int32_t *uniq, int64_t U, const int32_t *uniq_ptr,
                           const int32_t *pair_node, const int32_t *pair_out, float *logits,
                           int32_t mode, int32_t *err, void *stream);
/* K6 on the tensor cores (tcgen05.mma kind::f16, TMEM accumulators) for DENSE
 * node x unique-id tiles: the same pairs / outputs as spx_tree_merged_logits
 * (FAST mode; pair_uid[q] = the unique-id index of pair q, the CSR row), with xg split exactly into three bf16 parts so every product
 * is exact; only the accumulation order differs from the CUDA-core CDOT.
 * bf16 head, d % 64 == 0.  P = number of pairs; scratch: at least
 * spx_tree_tc_scratch_bytes(N, d, U, P) bytes (no initialisation needed). */
int64_t spx_tree_tc_scratch_bytes(int64_t N, int64_t d, int64_t U, int64_t P);
int spx_tree_merged_logits_tc(const float *xg, const float *r, int64_t N, const void *head,
                              int32_t head_dtype, const float *head_bw, int64_t V, int64_t d,
                              const int32_t *uniq, int64_t U, const int32_t *uniq_ptr,
                              const int32_t *pair_node, const int32_t *pair_out,
                              const int32_t *pair_uid, int64_t P, float *logits, void *scratch,
                              int32_t *err, void *stream);
/* Head-side normalisation of N rows for K6: FAST -> xg = (x-mean)*g and
 * r = 1/sqrt(var+eps) per row (canonical order); STRICT -> xg = the
 * reference LayerNorm (model.py:140-146), r = 1. */
int spx_head_prep(const float *hidden, int64_t hidden_stride, const float *g, const float *b,
                  float *xg, float *r, int64_t N, int64_t d, int32_t mode, int32_t *err,
                  void *stream);
/* bw[v] = CDOT(b, head_v): the final-norm bias folded through the head, once
 * per model (FAST path; all-zero b gives bw = 0). */
int spx_head_bias(const void *head, int32_t head_dtype, const float *b, int64_t V, int64_t d,
                  float *bw, void *stream);
/* final LayerNorm of N rows into hn (model.py:140-146), FAST or STRICT. */
int spx_final_norm(const float *hidden, int64_t hidden_stride, const float *g, const float *b,
                   float *hn, int64_t N, int64_t d, int32_t mode, int32_t *err, void *stream);

/* K7 -- hyper-token conjunction (src/specexit/tree.py:116-122, :389-390):
 * path_fire[p] = AND over nodes j of path p (CSR) of node_fired[j]; only for
 * live paths (live[p] != 0). */
int spx_path_and(const uint8_t *node_fired, const int32_t *path_ptr, const int32_t *path_nodes,
                 const uint8_t *live, int64_t P, uint8_t *path_fire, void *stream);

/* K7b -- rows that need the full-head check after the path AND
 * (src/specexit/tree.py:221-227, _verify_path :274-283): node_gate[j] = 1 for
 * every node j on a path with path_fire[p] != 0, node_gate[0] (the root) = 1
 * when any path fires, else 0.  n_nodes includes the root. */
int spx_tree_gate(const uint8_t *path_fire, const int32_t *path_ptr, const int32_t *path_nodes,
                  int64_t P, int64_t n_nodes, uint8_t *node_gate, void *stream);

/* Tree-node evaluation (src/specexit/tree.py:213-220; extract_features
 * src/specexit/predictor.py:42-52, predictor_forward :97-103): for each live
 * node i (node = live_idx[i]) take its K logits (row i of `logits`, the K6
 * output), build features against prev[node] (updated in place), evaluate
 * the MLP (policy SPX_POLICY_MLP: w1/b1/w2/b2, fire iff z2 >= z_cut) or the
 * constant policy (SPX_POLICY_CONST: fire iff const_prob > threshold), write
 * fired[node] and prob_out[node] (optional).  prev (n_nodes, K), fired and
 * prob_out (n_nodes) are indexed by node. */
int spx_tree_node_eval(const float *logits, const int32_t *live_idx, int64_t n_live, float *prev,
                       const float *w1, const float *b1, const float *w2, float b2, float z_cut,
                       int32_t policy, double const_prob, double threshold, double *prob_out,
                       uint8_t *fired, int32_t *err, int64_t K, int64_t H, void *stream);

/* Synthetic weights on device: reference rng.uniform (src/specexit/rng.py:24-27)
 * of stream `seed` over a (rows, cols) row-major tensor, written as bf16 (or
 * f32 when out_f32 != 0).  transpose != 0 stores element (r, c) at
 * out[c*rows + r] (e.g. the (d, V) lm_head as (V, d)). Bit-identical to
 * numpy's float32 result, then RNE-rounded to bf16. */
int spx_init_uniform(void *out, int32_t out_f32, int64_t rows, int64_t cols, int32_t transpose,
                     uint64_t seed, double low, double high, void *stream);

/* Flag-guarded decoder layer with lazy KV completion (model.py:220-270): advances
 * every unfrozen row whose frontier == layer through pre-LN MHA + ReLU FFN and
 * sets its frontier to layer+1.  All kernels return immediately when *done is
 * nonzero (the stream exited early this token: engine.py:205-207).  Weights
 * are out-major: wqkv (3d, d) = [wq^T; wk^T; wv^T], wo (d, d) = wo^T,
 * w1 (ffn, d) = ffn.w1^T, w2 (d, ffn) = ffn.w2^T. */
typedef struct {
  const float *ln1_g, *ln1_b, *ln2_g, *ln2_b;
  const void *wqkv, *wo, *w1, *w2;
  const float *b1, *b2;
  int32_t w_dtype;                 /* SPX_DTYPE_*                               */
  float *pending;                  /* (max_ctx, d) residual rows                */
  float *kcache, *vcache;          /* this layer's (max_ctx, d) K/V             */
  int32_t *frontier;               /* (max_ctx)                                 */
  const int32_t *n_ctx;            /* device scalar: rows in use                */
  const int32_t *new_row;          /* device scalar: newest row (cur_hidden)    */
  const uint8_t *frozen;           /* (max_ctx) optional (tree mode)            */
  const int32_t *attn_ptr;         /* (max_ctx+1) optional ancestor lists (CSR) */
  const int32_t *attn_idx;
  const uint8_t *done;             /* device exit flag (skip when nonzero)      */
  float *cur_hidden;               /* (d) optional copy of the newest row       */
  int32_t *rows, *nrows;           /* scratch: row set (max_ctx), count         */
  float *s_q, *s_att, *s_f;        /* scratch (max_ctx, d), (max_ctx, d), (max_ctx, ffn) */
  float *s_part;                   /* scratch: split-K partials (FAST), see spx_layer_part_floats */
  int32_t *s_flag;                 /* scratch: split-K arrival counters, zeroed once, self-reset */
  int32_t layer, mode;
  int32_t *err;
  int64_t max_ctx, d, n_heads, ffn;
  int32_t rows_hint;               /* new rows this call appends (begin() size), 0 =  */
                                   /* unknown; > 2 selects the multi-row kernel     */
                                   /* chain (prefill, token trees) over the         */
                                   /* persistent single-launch decode layer         */
  int32_t row_cap;                 /* max rows advanced by one call (shared-memory  */
                                   /* row set); 0 = max_ctx.  Batched streams: the  */
                                   /* new rows + lazily completed ones              */
  int32_t att_cap;                 /* max attention-list length (keys per row); 0 = */
                                   /* max_ctx.  Rows selecting more set SPX_ERR_ROW_CAP */
  void *tc_scratch;                /* optional: >= spx_layer_tc_scratch_bytes(d, ffn,  */
                                   /* row_cap or max_ctx) bytes; enables the tcgen05  */
                                   /* path for calls advancing >= 3 rows (FAST, bf16); */
                                   /* zero-initialised once by the caller           */
} spx_layer_args;
/* scratch of the tensor-core multi-row layer path: two regions of bf16 row
 * parts, the K-split partial sums and the K-split tile counters (which must
 * start at zero; they reset themselves after every use) */
int64_t spx_layer_tc_scratch_bytes(int64_t d, int64_t ffn, int64_t row_cap);
int spx_layer_forward(const spx_layer_args *args, void *stream);
/* floats needed for s_part and int32s for s_flag at these dimensions */
int64_t spx_layer_part_floats(int64_t d, int64_t ffn);
int64_t spx_layer_flag_ints(int64_t d, int64_t ffn);
/* begin() (model.py:181-212): append T rows, pending = emb[tok] + pe[pos],
 * frontier 0; *n_ctx += T; *new_row = last appended row. */
int spx_embed(const void *embedding, int32_t w_dtype, const float *pos_encoding,
              const int32_t *tokens, const int32_t *pos_ids, int64_t T, int64_t d, int64_t V,
              int64_t max_ctx, float *pending, int32_t *frontier, int32_t *n_ctx,
              int32_t *new_row, int32_t *err, void *stream);

/* Device-resident per-token state of a single-stream engine (engine.py:176-217)
 * and its trace record arrays (ExitRecord, engine.py:26-48). */
typedef struct {
  float *prev;                                  /* (K) local probs carried    */
  uint8_t *done, *fired, *fired_any;            /* exit flag, per-layer fire  */
  int32_t *exit_layer, *exit_token, *final_token, *evals, *full_heads;
  int32_t *next_in, *step;
  uint64_t *active;                             /* scheduled-layer bitmask    */
  int32_t *rec_token, *rec_exit_layer, *rec_evals, *rec_full_heads;
  uint8_t *rec_fired, *rec_verified;
  uint64_t *rec_active;
  float *prev_err;                              /* (1) bound carried with prev */
} spx_token_state;
/* stable top-K (value desc, lower id on ties) of n logits
 * (speculation.py:57-60 topk_from_logits). K <= 64. */
int spx_topk(const float *logits, int64_t n, int32_t K, int32_t *ids_out, void *stream);
/* softmax_1d (src/specexit/model.py:149-152) of each of `rows` rows of n
 * logits, evaluated at the K ids ids[r*K + j] (speculation.py:80-84
 * draft_probs).  STRICT: bit-identical to extract_features' local
 * probabilities (the reference's left-to-right denominator); FAST: the
 * denominator as a fixed-order parallel sum (FAST tolerance).  Non-finite
 * logits set ERR bit 4, ids outside [0, n) bit 1. */
int spx_softmax_pick(const float *logits, int64_t rows, int64_t n, const int32_t *ids,
                     int32_t K, float *probs_out, int32_t mode, int32_t *err, void *stream);
/* spx_topk for `rows` independent rows of n logits (row-major), K ids each. */
int spx_topk_rows(const float *logits, int64_t rows, int64_t n, int32_t K, int32_t *ids_out,
                  void *stream);
/* token start: prev = inv_k (= float32(1/K)), clear flags, exit_layer = L-1 */
int spx_token_begin(spx_token_state st, int32_t K, int32_t L, float inv_k, void *stream);
/* token end: pick verified exit token or the final argmax, record, next_in,
 * update_online (scheduler.py:65-79) of stream row 0 */
int spx_token_end(spx_token_state st, spx_online_state os, int32_t L, int32_t queue_len,
                  int32_t radius, int64_t max_steps, void *stream);
/* *dst |= *src (byte flags) */
int spx_or_flag(const uint8_t *src, uint8_t *dst, void *stream);
/* generate_forced (engine.py:227-246): *next_in = forced[*step - 1] */
int spx_force_next(const int32_t *forced, const int32_t *step, int32_t *next_in,
                   int64_t n_forced, void *stream);
/* injected-spec hook on _speculative_set (engine.py:162-168):
 * if flags[*step], forced[*step] (the target's final argmax under
 * generate_forced) replaces spec_ids[K-1] unless already among the K ids */
int spx_inject_spec(int32_t *spec_ids, int32_t K, const int32_t *forced, const int32_t *step,
                    const uint8_t *flags, int64_t n, void *stream);

/* numpy float32 exp restated on device (the exp of softmax_1d, model.py:151),
 * elementwise -- test hook for the bit-exactness of the softmax. */
int spx_np_expf(const float *x, float *y, int64_t n, void *stream);

/* Library identification (for the loaded-.so evidence). */
const char *spx_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPECEXIT_B200_H */
