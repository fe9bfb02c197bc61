/*
 * a2ats.h -- C ABI of the B200-native A^2ATS decode-time retrieval path.
 *
 * A^2ATS (arXiv 2502.12665).  "P:n" = line n of the paper's LaTeX source
 * (PAPER.md).  Readings Q1-Q24 of the paper's silent / ambiguous points are
 * listed in DESIGN.md.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - All tensor pointers are DEVICE pointers (cudaMalloc / PyTorch CUDA
 *    storage) unless a comment says "host".  With kv_location ==
 *    A2ATS_KV_HOST_MAPPED the K/V cache pointers may instead be device
 *    aliases of mapped pinned host memory (cudaHostAlloc(..Mapped) +
 *    cudaHostGetDevicePointer).
 *  - Every buffer is caller-owned.  The library allocates nothing on the hot
 *    path and retains no pointer after return.
 *  - bf16 tensors are passed as `const void*` (IEEE bfloat16 bit patterns,
 *    round-to-nearest-even conversions everywhere, reading Q17).
 *  - Layouts are dense row-major (C order); the last dimension is d = 128
 *    and is contiguous.  n_max % 8 == 0 so 16-byte vector loads of codes and
 *    rows are aligned; every pointer must be 16-byte aligned.
 *  - `stream` is a cudaStream_t passed as void*; NULL = the legacy default
 *    stream.  All work is enqueued asynchronously; nothing synchronises the
 *    host.  Asynchronous device faults surface at the caller's next sync.
 *  - Workspaces: query the size with the *_workspace_bytes function, hand
 *    over a device buffer of at least that many bytes that is ZERO-FILLED
 *    before its first use.  Every successful call leaves the workspace in
 *    that zero state again, so the same buffer can be reused call after call
 *    on one stream.  Concurrent calls need distinct workspaces.
 *  - Return value: A2ATS_OK (0) or a negative status (see below); no
 *    exception crosses the ABI.  Argument validation happens before any CUDA
 *    call, so EINVAL / EUNSUPPORTED / EWORKSPACE are returned without
 *    touching the device.
 *  - Results are bitwise deterministic for fixed inputs and shapes: no
 *    order-dependent floating-point atomics are used anywhere.
 */
#ifndef A2ATS_H_
#define A2ATS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define A2ATS_ABI_VERSION 10

/* ---- status codes ---------------------------------------------------- */
#define A2ATS_OK 0
#define A2ATS_EINVAL (-1)       /* bad argument: null required pointer, d odd, Hq % Hkv != 0,
                                   n_ctx <= 0 or > n_max, topk < 0, token range out of bounds,
                                   misalignment (mirrors SPEC "dimension mismatch", "odd-length
                                   row", "empty store") */
#define A2ATS_EUNSUPPORTED (-2) /* valid but not implemented: d != 128, G = Hq/Hkv not in
                                   {1,2,4,8}, L > 16384 */
#define A2ATS_EWORKSPACE (-3)   /* ws == NULL or ws_bytes smaller than the queried size */
#define A2ATS_ECUDA (-4)        /* a CUDA launch failed (cudaGetLastError after launch) */
#define A2ATS_ENCCL (-5)        /* an NCCL call failed (sharded entry points) */

/* group_reduce: how the G query heads of one KV head are folded into one
 * ranking score per token (paper silent; reading Q10).  PER_HEAD: no fold --
 * every query head selects its own top-K from its own LUT row and attends over
 * its own Sel (the paper's per-head retrieval): the
 * step runs G GQA-free sub-steps (G' = 1) over the same codes / hist / K / V,
 * sel_out is then [B, Hq, topk] (row b, hq), scores_out is not supported
 * (EUNSUPPORTED), and a workspace sized for one mode must be zeroed before it
 * is used with the other. */
#define A2ATS_GROUP_MAX 0
#define A2ATS_GROUP_SUM 1
#define A2ATS_GROUP_PER_HEAD 2

/* kv_location (reading: the paper's CPU-resident KV cache of P:392-394). */
#define A2ATS_KV_DEVICE 0       /* K/V cache in HBM */
#define A2ATS_KV_HOST_MAPPED 1  /* K/V cache in mapped pinned host memory, read over PCIe */

/* rope_mode (the ablation configurations of P:419-427). */
#define A2ATS_ROPE_WINDOWED 0   /* WRoPE, the method (Eqs. 11-12) */
#define A2ATS_ROPE_STANDARD 1   /* standard RoPE on post-PE keys (the "Baseline" / "QAVQ" ablations) */

/* lut_engine: which pipes compute the score table LUT = q~ C^T (a2, Eq. 21).  The
 * contraction is M = L, N = B*G, K = d per KV head: a dense GEMM for large B*G*L (tensor
 * cores, bf16 hi+lo split of q~), a few thousand FMAs per CTA otherwise. */
#define A2ATS_LUT_AUTO 0    /* FMA when B*G <= A2ATS_LUT_FMA_MAX_VECTORS, tensor cores above */
#define A2ATS_LUT_TENSOR 1  /* tcgen05 (TMEM accumulators)                             */
#define A2ATS_LUT_FMA 2     /* FP32 FMA, one thread per codeword                        */
#define A2ATS_LUT_FMA_MAX_VECTORS 8  /* measured crossover (reading Q26, profiles/lut_sweep_r1.json) */

typedef struct a2ats_shape {
  int32_t B;      /* batch size (sequences)                                   */
  int32_t Hq;     /* query heads                                              */
  int32_t Hkv;    /* KV heads (one codebook per KV head); Hq % Hkv == 0 */
  int32_t d;      /* head dimension; 128 in this version                      */
  int32_t L;      /* codebook size (P:431 uses 4096); 1 <= L <= 16384         */
  int32_t n_max;  /* capacity (tokens) of the K/V cache and code arrays; % 8 == 0 */
  int32_t code_bytes; /* width of a code: 2 (uint16; 0 means 2) or 1 (uint8, L <= 256:
                         half the index memory, aux-mem 1/256).  With 1
                         every `uint16_t* codes` argument points to uint8 codes
                         [B, Hkv, n_max]; supported by a2ats_build_codes, the posting-
                         list entry points (a2ats_postings_build, a2ats_*_postings) and
                         a2ats_qavq_prepare; the code-scan entry points, scores_out and
                         the sharded step return A2ATS_EUNSUPPORTED */
} a2ats_shape;

typedef struct a2ats_params {
  int32_t window;        /* w of Eq. 11: i-j < w is local; 64      */
  int32_t bridge;        /* b of Eq. 11/12: fixed relative position; 2048     */
  int32_t n_sink;        /* statically preserved initial tokens; 4            */
  int32_t topk;          /* K: number of retrieved candidates (absolute; reading Q9)  */
  double rope_theta;     /* RoPE base; 1e4 by default (reading Q1)                    */
  const double* inv_freq;/* optional HOST array [d/2] of rotation frequencies that
                            overrides rope_theta (e.g. Llama-3.1 scaled frequencies)   */
  int32_t group_reduce;  /* A2ATS_GROUP_MAX (default) | _SUM | _PER_HEAD               */
  int32_t kv_location;   /* A2ATS_KV_DEVICE (default) | A2ATS_KV_HOST_MAPPED          */
  int32_t lut_engine;    /* A2ATS_LUT_AUTO (default) | A2ATS_LUT_TENSOR | A2ATS_LUT_FMA */
  int32_t hist_lag;      /* deferred a0 (a new token's code is first read when
                            it leaves the window): the newest hist_lag tokens are not
                            encoded yet -- their codes are not read and hist covers
                            [0, N - hist_lag); 0 <= hist_lag <= min(window, N).  The
                            selection and output equal hist_lag = 0 exactly.  0 for the
                            append entry points, scores_out and the sharded step     */
  int32_t rope_mode;     /* A2ATS_ROPE_WINDOWED (default): WRoPE (Eq. 11-12) on pre-PE
                            keys | A2ATS_ROPE_STANDARD: the ablation "Baseline" / "QAVQ"
                            configurations: the cache holds POST-PE keys
                            k_j R_j (codes quantize them), q~ = q R_i with i = N - 1
                            (params.bridge ignored) and every selected row -- sinks,
                            top-K, window -- gets the standard logit q~ . k~_j; the
                            sharded step refuses it (EUNSUPPORTED)                      */
} a2ats_params;

/* Fills the paper's configuration: w = 64, b = 2048, n_sink = 4, topk = 0,
 * theta = 1e4, GROUP_MAX, KV on device, LUT engine AUTO. */
void a2ats_default_params(a2ats_params* p);

const char* a2ats_status_string(int status);
int a2ats_abi_version(void);
/* Description of the calling thread's last A2ATS_ECUDA failure ("" if none). */
const char* a2ats_last_cuda_error(void);

/* ---------------------------------------------------------------------
 * a2ats_qavq_prepare -- codebook-side terms of the query-aware quantizer.
 *
 * f'(k; C) = argmin_j (k - c_j) H (k - c_j)^T            (Eq. 14)
 *          = argmin_j ( n_j - 2 k . c^_j )
 * with S = (H + H^T)/2, c^_j = c_j S and n_j = c_j H c_j^T (the term k H k^T
 * does not depend on j).  Outputs:
 *   nrm      : [Hkv, L] fp32, n_j
 *   chat     : [Hkv, L, 2d] bf16 (16-B aligned), row j = hi(c^_j) | lo(c^_j)
 *              with hi = bf16(c^_j), lo = bf16(c^_j - hi) (round to nearest),
 *              so hi + lo carries c^_j to ~2^-16 relative
 * Inputs:
 *   codebook : [Hkv, L, d] bf16, the shared codebook C
 *   H        : [Hkv, d, d] fp32 positive definite second-moment matrix of
 *              post-PE queries; NULL => H = I (conventional VQ, Eq. 5,
 *              P:115-118; then chat = c | 0 and nrm = |c|^2)
 * Call once per codebook (offline state); no workspace.
 * Returns A2ATS_EINVAL on NULL / misaligned pointers.
 * ------------------------------------------------------------------- */
int a2ats_qavq_prepare(const a2ats_shape* shape, const void* codebook, const float* H,
                       float* nrm, void* chat, void* stream);

/* ---------------------------------------------------------------------
 * a2ats_build_codes -- inference-time quantization (Eq. 20).
 *
 * For every (b, h) and token t in [t_begin, t_end):
 *   codes[b,h,t] = f'(k_t; C_h)  (lowest codeword index on exact ties, Q12)
 * and, if hist != NULL, hist[b,h,codes[b,h,t]] += 1.
 *   keys     : [B, Hkv, n_max, d] bf16 PRE-PE keys (under WRoPE the post-PE
 *              key equals the pre-PE key, Eq. 12)
 *   chat, nrm: from a2ats_qavq_prepare (same C, H)
 *   codes    : [B, Hkv, n_max] uint16 out; only [t_begin, t_end) written
 *   hist     : optional [B, Hkv, L] int32 running histogram, accumulated
 *   ws       : zero-filled before first use, ws_bytes >= the query below;
 *              left zeroed again on return (reusable, one stream at a time)
 * 0 <= t_begin <= t_end <= n_max.  Used for prefill (whole prompt) and for
 * each decode step (the new token).
 * ------------------------------------------------------------------- */
size_t a2ats_build_codes_workspace_bytes(const a2ats_shape* shape);
int a2ats_build_codes(const a2ats_shape* shape, const void* keys, int32_t t_begin, int32_t t_end,
                      const void* chat, const float* nrm, uint16_t* codes, int32_t* hist,
                      void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------
 * a2ats_decode_step -- one decode step of the retrieval path, all pairs.
 *
 * Per (b, KV head h), with i = n_ctx - 1 the current token (in the cache):
 *  a1  q~ = q R_b                                     (Eq. 12)
 *  a2  LUT[l] = q~ . c_l                              (Eq. 21)
 *  a3  score[t] = LUT[codes[t]];  agg[t] = max (or sum) over the G query
 *      heads of the group                             (Eq. 21; reading Q10)
 *  a4  Sel = Sinks u TopK u Window: Window = {t >= n_ctx - w}, Sinks = the
 *      first n_sink tokens outside it, TopK = the first
 *      min(topk, |Cand|) candidates by (agg desc, t asc)  (readings Q8, Q12)
 *  a5  u_j = q~ . k_j for sinks/top-K (bridge), u_j = (q R_{i-j}) . k_j in
 *      the window (Eq. 11); o = softmax(u / sqrt(d)) V over Sel
 *      (Eq. 2), fp32 online softmax, split over row chunks
 *  a6  log-sum-exp combine of the chunks in fixed order
 * Arguments:
 *   n_ctx    : N, cached tokens including the current one; 1 <= N <= n_max
 *   q        : [B, Hq, d] bf16 PRE-PE queries (q of head hq uses KV head hq / G)
 *   k_cache, v_cache : [B, Hkv, n_max, d] bf16 (pre-PE keys; rows < N read)
 *   codes    : [B, Hkv, n_max] uint16, valid for all t < N
 *   codebook : [Hkv, L, d] bf16
 *   hist     : optional [B, Hkv, L] int32: counts of codes over tokens
 *              [0, N) exactly (as maintained by a2ats_build_codes).  With it
 *              the code stream is read once; NULL => histogram computed
 *              in-step with an extra pass.  Results are bitwise identical.
 *              Long contexts (> 32768 candidates) with hist, L <= 4096 and
 *              n_max % 64 == 0 take the threshold + persistent half-pair scan
 *              (code rows loaded by TMA as 128-B rows); other shapes the
 *              threshold + chunked scan.  Same results either way.
 *   out      : [B, Hq, d] fp32 attention output (device or mapped pinned
 *              host memory)
 *   sel_out  : optional [B, Hkv, K_eff] int32, the top-K token indices in
 *              ascending order, K_eff = min(topk, |Cand|)
 *   scores_out : optional [B, Hq, n_ctx] fp32 debug output of the
 *              approximate scores u^ (Eq. 21) of every token
 * ------------------------------------------------------------------- */
size_t a2ats_decode_workspace_bytes(const a2ats_shape* shape, const a2ats_params* params);
int a2ats_decode_step(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx,
                      const void* q, const void* k_cache, const void* v_cache,
                      const uint16_t* codes, const void* codebook, const int32_t* hist,
                      float* out, int32_t* sel_out, float* scores_out,
                      void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------
 * a2ats_select_topk -- a1..a4 only: the score table LUT = q~ C^T and the
 * top-K selection over the code stream, Sel written to sel_out; no K/V is
 * read and no attention runs.  This is the part the paper runs on the GPU
 * before handing Sel to its CPU attention.  Arguments as
 * a2ats_decode_step (same workspace); sel_out is required.  Results are
 * bitwise identical to the sel_out of a2ats_decode_step.
 * ------------------------------------------------------------------- */
int a2ats_select_topk(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx,
                      const void* q, const uint16_t* codes, const void* codebook,
                      const int32_t* hist, int32_t* sel_out, void* ws, size_t ws_bytes,
                      void* stream);

/* ---------------------------------------------------------------------
 * a2ats_stage_rows -- the step's inputs into device memory with one kernel
 * (no copy-engine operation): q_src [B, Hq, d] bf16 -> q_dst [B, Hq, d], and
 * the new token's key / value rows k_src, v_src [B, Hkv, d] bf16 ->
 * k_cache / v_cache [B, Hkv, n_max, d] at row n_ctx - 1.  Sources may be
 * device memory or MAPPED PINNED HOST memory (cudaHostAlloc / torch
 * pin_memory under UVA), read over PCIe by the kernel; any NULL source is
 * skipped.  All pointers 16-B aligned; 1 <= n_ctx <= n_max, else EINVAL.
 * Enqueued on `stream`, chained to the next library kernel (PDL).
 * Not a step of the paper: the plumbing of an end-to-end decode step.  The
 * output of a decode step may likewise be mapped pinned host memory (`out`
 * is written once per (b, hq) row by the attention kernel).
 * ------------------------------------------------------------------- */
int a2ats_stage_rows(const a2ats_shape* shape, int32_t n_ctx, const void* q_src, const void* k_src,
                     const void* v_src, void* q_dst, void* k_cache, void* v_cache, void* stream);

/* ---------------------------------------------------------------------
 * a2ats_decode_step_append -- a0 for the new token, then a1..a6 (one
 * decode step of the paper: the new key is quantized with Eq. 20,
 * P:369-373, and the query retrieves with Eqs. 21 / 11 / 2).
 *
 * Same as a2ats_build_codes(t_begin = n_ctx - 1, t_end = n_ctx) followed by
 * a2ats_decode_step(n_ctx), with identical results, but the encoding runs
 * concurrently with the score table (one kernel): the new token is inside
 * the window (w >= 1), so the selection never needs its code.
 *   codes, hist : on entry valid for tokens [0, n_ctx - 1); on return for
 *                 [0, n_ctx) (codes[.., n_ctx - 1] written, hist updated
 *                 if given)
 *   chat, nrm   : from a2ats_qavq_prepare
 * Requires B <= 256, kv_location = A2ATS_KV_DEVICE; other arguments and the
 * workspace as a2ats_decode_step.  EINVAL otherwise.
 * ------------------------------------------------------------------- */
int a2ats_decode_step_append(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx,
                             const void* q, const void* k_cache, const void* v_cache,
                             uint16_t* codes, const void* codebook, int32_t* hist,
                             const void* chat, const float* nrm,
                             float* out, int32_t* sel_out, float* scores_out,
                             void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------
 * Posting-list (inverted-index) selection.  A token's
 * approximate score is its code's (Eq. 21), so the top-K set is
 * the union of the token lists of the codes above v* plus the first m
 * tokens (lowest index, reading Q12) of the tied codes' lists: the selection
 * reads about K list entries per pair instead of every code.  The index is
 * query-independent: a2ats_postings_build groups the tokens [0, n_tokens) of
 * every pair by code, each list ascending (deterministic; postings:
 * a2ats_postings_bytes of device memory = int32 offsets [B*Hkv, LP] with
 * LP = (L + 4) & ~3 (row = the L+1 list starts, padded to 16 B), then,
 * 256-byte aligned, int32 tokens [B*Hkv, n_max], caller-owned); tokens
 * [n_post, n_ctx) not yet in the index are classified from their codes.
 * a2ats_select_topk_postings / a2ats_decode_step_postings = a2ats_select_topk /
 * a2ats_decode_step with that selection (hist required, L <= 4096, 0 <= n_post
 * <= n_ctx): the SAME SET per pair as the code scan.  Order of sel_out:
 *   n_post <= n_ctx - window (the index holds no window token; at most 64
 *   indexed sinks): index order -- the above-v* codes' lists (code order,
 *   each ascending), the above-v* unindexed tokens, then the m selected ties
 *   ascending; deterministic for a given index;
 *   otherwise: ascending, as a2ats_select_topk.
 * The attention output equals a2ats_decode_step's up to the summation order
 * of the rows (fp32 rounding).
 * ------------------------------------------------------------------- */
size_t a2ats_postings_bytes(const a2ats_shape* shape);
int a2ats_postings_build(const a2ats_shape* shape, const uint16_t* codes, int32_t n_tokens, void* postings,
                         void* stream);
int a2ats_select_topk_postings(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, const void* q,
                               const uint16_t* codes, const void* codebook, const int32_t* hist,
                               const void* postings, int32_t n_post, int32_t* sel_out, void* ws, size_t ws_bytes,
                               void* stream);
int a2ats_decode_step_postings(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, const void* q,
                               const void* k_cache, const void* v_cache, const uint16_t* codes,
                               const void* codebook, const int32_t* hist, const void* postings, int32_t n_post,
                               float* out, int32_t* sel_out, void* ws, size_t ws_bytes, void* stream);
/* One decode step of the paper with the posting-list selection: a0 for token
 * n_ctx-1 (as a2ats_decode_step_append: its code into codes, +1 into hist)
 * fused with a1..a6 over the index.  0 <= n_post <= n_ctx-1 (the new token is
 * never in the index); tokens [n_post, n_ctx) are classified from their codes,
 * so the caller rebuilds the index (a2ats_postings_build) as often as it likes
 * -- the result does not depend on n_post.  EINVAL / EUNSUPPORTED as above. */
int a2ats_decode_step_append_postings(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx,
                                      const void* q, const void* k_cache, const void* v_cache, uint16_t* codes,
                                      const void* codebook, int32_t* hist, const void* chat, const float* nrm,
                                      const void* postings, int32_t n_post, float* out, int32_t* sel_out, void* ws,
                                      size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------
 * Sequence-sharded decode step (the paper itself
 * is single-GPU).  R <= 8 ranks, one process per GPU.  Rank r holds,
 * for every (b, KV head), the global tokens [bounds[r], bounds[r+1]) of the
 * context in its own arrays of capacity shape->n_max (local row = global -
 * bounds[r]; n_max % 64 == 0): codes [B,Hkv,n_max] uint16 and k_cache /
 * v_cache [B,Hkv,n_max,d] bf16.  q, the codebook (and its prepared terms chat,
 * nrm of a2ats_qavq_prepare) and the shard STATE are replicated.  bounds is a
 * HOST array [R+1], bounds[0] = 0, non-decreasing, the same on every rank.
 *
 * State (a2ats_shard_state_bytes, caller-owned device memory, built by
 * a2ats_shard_state_build, then updated by every step identically on every
 * rank): the code histogram of all tokens [0, n) and every rank's histogram of
 * its tokens (int32 [B*Hkv, L] and [R, B*Hkv, L]), the codes of the first
 * n_sink tokens and of the latest WR tokens (WR = the power of two >= window).
 * From it every rank derives, with NO exchange, the K-th level v* and tie
 * quota m of the GLOBAL top-K (the LUT is bitwise identical on every rank)
 * and its own share of the ties (the first m tied tokens in global order,
 * reading Q12: lower ranks first) -- the collective-free exact global top-K
 * of SURVEY §8f.1.  The union of the ranks' selections equals the
 * single-GPU top-K exactly.
 *
 * a2ats_decode_step_sharded(n_ctx): token n_ctx-1 (its K/V row already in its
 * owner's cache: the rank with bounds[r] <= n_ctx-1 < bounds[r+1]) is encoded
 * on its owner (a0); every rank computes the LUT, its local selection and the
 * exact attention over its rows of Sel (a1..a5) into a partial (m, l, o) in the
 * base-2 logit domain; ONE ncclAllGather exchanges the partials and the new
 * token's code (msg = a2ats_shard_msg_bytes per rank, ~1 MB at C4); then the
 * log-sum-exp combine in rank order (a6) -> out [B,Hq,d] fp32 on EVERY rank,
 * and the state update.  All on the caller's stream, no host synchronisation:
 * one call per step, capturable in a CUDA graph.  sel_out (optional, [B,Hkv,
 * topk]): this rank's selected GLOBAL token indices, ascending.  ws: a2ats_
 * shard_workspace_bytes, zero-initialised once, reusable.  comm: from
 * a2ats_comm_init (NCCL, loaded with dlopen: the process's libnccl.so.2 or
 * A2ATS_NCCL_LIB); NULL only when R == 1.  Errors: A2ATS_EINVAL (bounds,
 * rank, pointers), A2ATS_EUNSUPPORTED (n_max % 64, L > 4096, B > 256, host
 * K/V), A2ATS_ENCCL.
 * ------------------------------------------------------------------- */
#define A2ATS_COMM_ID_BYTES 128
typedef struct a2ats_comm_id { char internal[A2ATS_COMM_ID_BYTES]; } a2ats_comm_id;  /* = ncclUniqueId */
typedef struct a2ats_comm a2ats_comm;
int a2ats_comm_unique_id(void* id);   /* rank 0; the caller broadcasts the 128 bytes (torch.distributed) */
int a2ats_comm_init(const void* id, int32_t world, int32_t rank, a2ats_comm** out);
int a2ats_comm_destroy(a2ats_comm* comm);
size_t a2ats_shard_state_bytes(const a2ats_shape* shape, const a2ats_params* params, int32_t world);
/* byte offsets in the state: [0] hist_g int32 [B*Hkv, L], [1] hist_r int32 [R, B*Hkv, L],
 * [2] ring uint16 [B*Hkv, WR], [3] sink codes uint16 [B*Hkv, n_sink_cap]; [4] WR, [5] n_sink_cap */
int a2ats_shard_state_layout(const a2ats_shape* shape, const a2ats_params* params, int32_t world, size_t* offsets);
size_t a2ats_shard_msg_bytes(const a2ats_shape* shape);
size_t a2ats_shard_workspace_bytes(const a2ats_shape* shape, const a2ats_params* params, int32_t world);
/* state of tokens [0, n_tokens) from every rank's codes (NCCL all-reduces; once, at prefill).
 * comm == NULL with world > 1: only this rank's contribution is written (zeros elsewhere);
 * the replicated state is then the element-wise sum of the ranks' contributions (int32
 * histograms, uint16 codes) -- single-process rank simulation (tests).  ws: workspace of
 * a2ats_shard_workspace_bytes. */
int a2ats_shard_state_build(const a2ats_shape* shape, const a2ats_params* params, int32_t world, int32_t rank,
                            const int32_t* bounds, int32_t n_tokens, const uint16_t* codes, void* state,
                            void* ws, size_t ws_bytes, a2ats_comm* comm, void* stream);
int a2ats_decode_step_sharded(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx,
                              int32_t world, int32_t rank, const int32_t* bounds, const void* q,
                              const void* k_cache, const void* v_cache, uint16_t* codes, const void* codebook,
                              const void* chat, const float* nrm, void* state, float* out, int32_t* sel_out,
                              void* ws, size_t ws_bytes, a2ats_comm* comm, void* stream);
/* The two halves of a2ats_decode_step_sharded around its all-gather (tests
 * simulate ranks in one process): partial writes this rank's message
 * (msg: a2ats_shard_msg_bytes, device); finish reads all ranks' messages
 * [R][msg] and writes out + updates the state. */
int a2ats_shard_step_partial(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, int32_t world,
                             int32_t rank, const int32_t* bounds, const void* q, const void* k_cache,
                             const void* v_cache, uint16_t* codes, const void* codebook, const void* chat,
                             const float* nrm, const void* state, void* msg, int32_t* sel_out, void* ws,
                             size_t ws_bytes, void* stream);
int a2ats_shard_step_finish(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, int32_t world,
                            const int32_t* bounds, const void* msgs, void* state, float* out, void* stream);
/* log-sum-exp combine of R partials [R,B,Hq,130] (base-2 domain) in rank order */
int a2ats_combine(const a2ats_shape* shape, int32_t nparts, const float* partials, float* out, void* stream);

/* ---------------------------------------------------------------------
 * a2ats_qavq_train -- OFFLINE query-aware codebook construction for one KV
 * head (§4.2):
 *   H = (1/m) sum_i q_i^T q_i over the m post-PE queries (Eq. 10)
 *       + eps * tr(H)/d * I (reading Q27; eps = 0: none), or H_in, or I
 *       (queries == H_in == NULL: conventional VQ, Eq. 4);
 *   H = L L^T (Cholesky), z = k L (Eq. 16);
 *   k-means++ on z with the caller's uniform draws u[0..L-1] in
 *       [0, 1): centre 0 = z[floor(u_0 n)], centre j = the first point whose
 *       running sum of D^2 exceeds u_j * sum D^2 (reading Q28);
 *   Lloyd on z: assignment argmin_j ||z - c^z_j||^2 (lowest j on ties),
 *       centroid = mean of its points, an empty cluster keeps its centre
 *       (reading Q29), until no assignment changes or max_iters (Eq. 18);
 *   C = C^z L^{-1} (Eq. 19).
 * keys [n_keys, d] bf16, queries [m_queries, d] bf16 (or NULL), H_in [d, d]
 * fp64 (or NULL), u [L] fp64, C_out [L, d] fp64, H_out [d, d] fp64 (optional),
 * labels_out [n_keys] int32 (optional), info_out int32[2] = {iterations run,
 * Cholesky failure flag} (optional): all DEVICE pointers.  d <= 128,
 * 1 <= L <= n_keys.  Computed in fp64 with fixed-order sums (deterministic);
 * asynchronous on `stream`, no host synchronisation.  ws: a2ats_qavq_train_
 * workspace_bytes.  Errors: A2ATS_EINVAL, A2ATS_EWORKSPACE, A2ATS_ECUDA.
 * ------------------------------------------------------------------- */
size_t a2ats_qavq_train_workspace_bytes(int32_t n_keys, int32_t d, int32_t L, int32_t m_queries);
int a2ats_qavq_train(int32_t n_keys, int32_t d, int32_t L, const void* keys, int32_t m_queries, const void* queries,
                     const double* H_in, double eps, const double* u, int32_t max_iters, double* C_out,
                     double* H_out, int32_t* labels_out, int32_t* info_out, void* ws, size_t ws_bytes,
                     void* stream);

/* ---------------------------------------------------------------------
 * a2ats_set_stage_events -- optional instrumentation for benchmarks.
 *
 * events: host array of n cudaEvent_t handles (passed as void*), or NULL to
 * disable.  While set, every a2ats_decode_step records events[0..4] on its
 * stream at the stage boundaries: [0] before a1/a2 (LUT), [1] after the LUT,
 * [2] after the code scan + top-K (a3 + a4), [3] after attention + combine
 * (a5 + a6), [4] at the end.  Requires n >= 5.
 * The array is copied; the events stay caller-owned.  Process-global, not
 * thread-safe: for single-threaded benchmarking only.
 * ------------------------------------------------------------------- */
int a2ats_set_stage_events(void* const* events, int n);

#ifdef __cplusplus
}
#endif
#endif /* A2ATS_H_ */
