/*
 * onmt.h - C-ABI of the B200-native OpenNMT beam-search translation hot path.
 *
 * The operation (PAPER.md, arXiv 1805.11462):
 *   P105-108 (§2)   p(w_{1:T}|x) = prod_t p(w_t | w_{1:t-1}, x; theta); a hypothesis
 *                   score is the sum of its token log-probabilities.
 *   P112-122 (§2)   source encoder RNN over word vectors -> h_1..h_S; target decoder
 *                   RNN; attention pooling over the source vectors; softmax layer.
 *   P129-136 (§2)   LSTM cells (a), stacked layers (b), input feeding (c).
 *   P136-139 (§2d)  test-time beam search.
 *   P233-237 (§4.1) "a batched CPU/GPU implementation for very quickly translating a
 *                   large set of sentences ... a specialized C implementation".
 *   P299-301, P315-316 (§4.2) general / dot attention; length normalisation.
 * The exact step-by-step rule implemented is DESIGN.md §2 (= SURVEY.md §8(c) O1-O11).
 *
 * Conventions
 *  - Every call returns onmt_status (0 = OK, < 0 = error).  No C++ exception crosses
 *    the ABI.  On error, onmt_last_error() returns a thread-local message that stays
 *    valid until the next call on the same thread.
 *  - Token ids: 0 = pad, 1 = unk, 2 = bos, 3 = eos (SPEC.md S170).
 *  - Source batches are batch-major, row-major int32 [B x S_max]; sentence b uses
 *    src_ids[b*S_max + 0 .. src_lens[b]-1]; ids at padded positions are ignored.
 *  - Ownership: the caller owns every buffer it passes; the library copies host
 *    inputs in once per call and results out once per call, and owns all device
 *    memory of a model handle (released by onmt_free).
 *  - Threading: at most one in-flight call per model handle.  Handles on DIFFERENT
 *    devices may run concurrently.  On one device, calls of distinct handles must not
 *    overlap in time (serialise them on one stream or with events): several kernels of a
 *    call are persistent grids whose CTAs (or thread-block clusters) wait for one another,
 *    planned so that the whole grid is co-resident on an otherwise idle device
 *    (cudaOccupancyMaxActiveClusters); if another grid holds the SMs such a wait times
 *    out after 4 s, the kernel traps and the call fails with ONMT_E_CUDA instead of
 *    hanging.
 */
#ifndef ONMT_H_
#define ONMT_H_

#include <stdint.h>

#if defined(__GNUC__)
#define ONMT_API __attribute__((visibility("default")))
#else
#define ONMT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ONMT_OK = 0,
  ONMT_E_INVALID_ARG = -1,   /* bad size/pointer/option (see each call)            */
  ONMT_E_IO = -2,            /* weight file cannot be opened/read                   */
  ONMT_E_FORMAT = -3,        /* bad magic, version, dtype, shape or tensor-name set */
  ONMT_E_UNSUPPORTED = -4,   /* beam > ONMT_K_MAX, not an sm_100 device, ...        */
  ONMT_E_ID_RANGE = -5,      /* a source id at a real position is outside [0,V_src) */
  ONMT_E_EMPTY_SOURCE = -6,  /* some src_lens[b] < 1 (SPEC.md S431)                 */
  ONMT_E_CUDA = -7,          /* CUDA runtime/driver failure (message has the error) */
  ONMT_E_OOM = -8            /* device allocation failed                            */
} onmt_status;

typedef enum { ONMT_PREC_FP32 = 0, ONMT_PREC_BF16 = 1 } onmt_precision;

#define ONMT_K_MAX 16

typedef struct onmt_model onmt_model; /* opaque, owned by the library */

typedef struct {
  int32_t layers, emb, hidden, v_src, v_tgt, bidir, attn_general, precision;
} onmt_model_info;

/*
 * onmt_load_weights - read an MNMT container (SPEC.md S83: magic "MNMT", u32 version 1,
 * per tensor u32 name length + name, u32 rank, u64 dims, u32 dtype tag f32 = 0, LE
 * payload) and build a device-resident model on CUDA device `device`.
 *   Tensor names/shapes (config inferred from them):
 *     enc.emb [V_src,E]; enc.l{l}.{fwd|bwd}.{w_ih [4Hd,In_l], w_hh [4Hd,Hd], b_ih, b_hh [4Hd]};
 *     dec.emb [V_tgt,E]; dec.l0.w_ih [4H,E+H] (columns: embedding | input feed);
 *     dec.l{l>0}.w_ih [4H,H]; dec.l{l}.{w_hh [4H,H], b_ih, b_hh [4H]};
 *     attn.w_in [H,H] (present <=> 'general'); attn.w_out [H,2H] (columns: context | h);
 *     gen.w [V_tgt,H]; gen.b [V_tgt].  LSTM gate row blocks are (i,f,g,o).
 *   prec = ONMT_PREC_BF16 rounds every tensor to bf16 (round-to-nearest-even) once at
 *   load (reading R23); ONMT_PREC_FP32 keeps the stored fp32 values.
 * Errors: INVALID_ARG (null path/out, bad precision), IO, FORMAT, UNSUPPORTED
 * (device is not compute capability 10.x), CUDA, OOM.  *out is NULL on error.
 */
ONMT_API onmt_status onmt_load_weights(const char* mnmt_path, int32_t device, onmt_precision prec,
                              onmt_model** out);

/* onmt_model_get_info - copy the inferred configuration.  INVALID_ARG on NULL. */
ONMT_API onmt_status onmt_model_get_info(const onmt_model* m, onmt_model_info* out);

/*
 * onmt_set_stream - the cudaStream_t (passed as void*) all later work of this handle is
 * issued on (e.g. torch.cuda.current_stream().cuda_stream).  NULL = the handle's own
 * stream.  The caller keeps the stream alive while the handle uses it.
 */
ONMT_API onmt_status onmt_set_stream(onmt_model* m, void* cuda_stream);

/*
 * onmt_encode - the encoder alone (P112-115, P129-133; DESIGN.md §2 steps A1-A4).
 *   Host inputs: src_ids [B*S_max], src_lens [B] (1 <= len <= S_max).
 *   Host outputs (each may be NULL): out_memory [B*S_max*H] fp32, memory bank
 *   (top-layer outputs, [fwd;bwd] per position; positions >= len are 0);
 *   out_h, out_c [L*B*H] fp32: final state per layer = decoder initial state
 *   (layer-major, then sentence).
 * Errors: B == 0 is OK (no-op); EMPTY_SOURCE if some len < 1; INVALID_ARG if
 * len > S_max, S_max < 1, B < 0 or null input pointers; ID_RANGE; CUDA/OOM.
 */
ONMT_API onmt_status onmt_encode(onmt_model* m, const int32_t* src_ids, const int32_t* src_lens,
                        int32_t B, int32_t S_max, float* out_memory, float* out_h, float* out_c);

/*
 * onmt_translate - batched beam-search translation (P136-139; DESIGN.md §2 A1-A11).
 *   beam K in [1, ONMT_K_MAX]; max_len >= 1 counts generated tokens including EOS;
 *   length_penalty = alpha >= 0 in lp(n) = ((5+n)/6)^alpha (P315-316, SPEC S439).
 *   Host outputs: out_hyps [B*max_len] int32, y_1..y_n then 0-filled (includes EOS
 *   when the hypothesis finished on EOS, excludes BOS); out_lens [B];
 *   out_scores [B] normalised score raw/lp(n); out_raw_scores [B] or NULL (sum of
 *   token log-probs); out_token_logp [B*max_len] or NULL (log p of each emitted token).
 * Errors: as onmt_encode, plus INVALID_ARG if max_len < 1, beam < 1, alpha < 0 or NaN,
 * or a required output pointer is NULL; UNSUPPORTED if beam > ONMT_K_MAX.
 */
ONMT_API onmt_status onmt_translate(onmt_model* m, const int32_t* src_ids, const int32_t* src_lens,
                           int32_t B, int32_t S_max, int32_t beam, int32_t max_len,
                           float length_penalty, int32_t* out_hyps, int32_t* out_lens,
                           float* out_scores, float* out_raw_scores, float* out_token_logp);

/*
 * onmt_translate_ex - onmt_translate with the paper's translation customisations
 * (PAPER.md P313-316 "beam search with various normalizations including length and
 * attention coverage normalization" and OOV handling; SPEC S421-448):
 *   coverage_penalty = beta >= 0: banked hypotheses are ranked by the GNMT final score
 *     raw / lp(n) + beta * sum_{s < len} log(min(sum_t a_{t,s}, 1)) over the hypothesis's
 *     attention history (S439); the ranking inside a step stays by raw score.
 *   n_best in [1, beam]: the n best bank entries per sentence, in final order
 *     (score desc, then earlier step, then lower rank).  A sentence that banked fewer
 *     entries reports len 0 and score -inf for the missing ranks.
 *   replace_unk != 0: out_unk_pos [B*n_best*max_len] receives, for every emitted <unk>
 *     (id 1), the source position argmax_s a_{t,s} (ties -> smallest s) whose word replaces
 *     it (S448; no phrase table), and -1 for every other position.
 *   Host outputs are [B][n_best][...]: out_hyps [B*n_best*max_len], out_lens,
 *   out_scores (final score), out_raw_scores (or NULL), out_token_logp (or NULL).
 *   With beta = 0, n_best = 1, replace_unk = 0 it equals onmt_translate.
 * Errors: as onmt_translate, plus INVALID_ARG for n_best outside [1, beam], beta < 0 or
 * NaN, out_unk_pos without replace_unk; UNSUPPORTED when coverage / unk replacement is
 * requested for a model whose generator partials exceed the one-CTA-per-sentence beam
 * step (fp32 models with V_tgt > 32768).
 */
typedef struct {
  int32_t beam, max_len;
  float length_penalty, coverage_penalty;
  int32_t n_best, replace_unk;
} onmt_decode_opts;
ONMT_API onmt_status onmt_translate_ex(onmt_model* m, const int32_t* src_ids, const int32_t* src_lens,
                              int32_t B, int32_t S_max, const onmt_decode_opts* opts, int32_t* out_hyps,
                              int32_t* out_lens, float* out_scores, float* out_raw_scores,
                              float* out_token_logp, int32_t* out_unk_pos);

/*
 * onmt_translate_copy - beam search of a COPY / POINTER-GENERATOR model (weights copy.w
 * [1,H], copy.b [1]; PAPER.md P302-304, P316-317; SPEC S293-301) over
 * the extended vocabulary: p(w) = g p_vocab(w) + (1 - g) sum_{s: src_ext[s] = w} a_s with
 * g = sigmoid(copy.w . h~ + copy.b) and a the step's attention weights.
 *   src_ext [B*S_max] host int32: the dynamic dictionary - for every real source position
 *   its extended id, < V_tgt for a word of the target vocabulary, V_tgt + k for the k-th
 *   source-only word of the sentence (ids of padded positions are ignored).
 *   Output hyps may hold extended ids >= V_tgt (copied source-only words; the caller maps
 *   them back through its dictionary); such a token is fed to the next step as <unk>.
 *   opts: beam, max_len, length_penalty as onmt_translate; n_best must be 1, coverage 0,
 *   replace_unk 0.  Outputs as onmt_translate.
 * Errors: as onmt_translate, plus UNSUPPORTED for a model without copy.* tensors or other
 * options, ID_RANGE for an extended id outside [0, V_tgt + S_max), INVALID_ARG for a null
 * src_ext.  onmt_translate on a copy model is INVALID_ARG (it needs src_ext).
 */
ONMT_API onmt_status onmt_translate_copy(onmt_model* m, const int32_t* src_ids, const int32_t* src_lens,
                                const int32_t* src_ext, int32_t B, int32_t S_max,
                                const onmt_decode_opts* opts, int32_t* out_hyps, int32_t* out_lens,
                                float* out_scores, float* out_raw_scores, float* out_token_logp);

/*
 * onmt_translate_trace - onmt_translate plus the per-step beam selections, for the
 * parity protocol: for step t (0-based), sentence b, rank r:
 *   sel_parent [max_len*B*beam]: parent slot k, or -1 if nothing was selected;
 *   sel_token: the token w; sel_score (fp64): cumulative raw score cum_k + log p(w).
 * Steps after a sentence stopped hold -1 / 0 / -inf.
 */
ONMT_API onmt_status onmt_translate_trace(onmt_model* m, const int32_t* src_ids, const int32_t* src_lens,
                                 int32_t B, int32_t S_max, int32_t beam, int32_t max_len,
                                 float length_penalty, int32_t* out_hyps, int32_t* out_lens,
                                 float* out_scores, float* out_raw_scores, float* out_token_logp,
                                 int32_t* sel_parent, int32_t* sel_token, double* sel_score);

/*
 * onmt_score - teacher-forced scoring (PAPER.md P105-108: log p(Y|X) = sum_t log p(y_t | y_<t, X);
 * SURVEY §8(f) rank 1).  The decoder is fed the GIVEN target tokens (y_0 = BOS, then
 * y_1 .. y_{n-1}) instead of beam selections; the generator runs once over every
 * (step, sentence) row.
 *   src_ids / src_lens / B / S_max: as onmt_translate (host memory).
 *   tgt_ids [B*T_max] row-major host int32: y_1 .. y_n of sentence b in row b (no BOS; an
 *     EOS, if wanted, is part of Y); ids past tgt_lens[b] are ignored.
 *   tgt_lens [B]: 1 <= n_b <= T_max.
 *   out_token_logp [B*T_max] (caller-allocated host float): log p(y_t | ...) for t < n_b,
 *     0 past the end.  out_nll [B] (host double, or NULL): -sum_t log p.
 * Errors: as onmt_translate for the source; EMPTY_SOURCE if a tgt_len < 1; INVALID_ARG if
 * tgt_len > T_max or T_max < 1; ID_RANGE for a target id outside [0, V_tgt); CUDA.
 * B == 0 is a no-op.
 */
ONMT_API onmt_status onmt_score(onmt_model* m, const int32_t* src_ids, const int32_t* src_lens, int32_t B,
                                int32_t S_max, const int32_t* tgt_ids, const int32_t* tgt_lens, int32_t T_max,
                                float* out_token_logp, double* out_nll);

/*
 * onmt_translate_dev - same as onmt_translate with every pointer a DEVICE pointer on
 * the model's device, and no host synchronisation: the work is enqueued on the
 * handle's stream (onmt_set_stream) and the outputs are valid once it completes.
 * src_lens are read on the host side for validation only if d_src_lens_host is
 * non-NULL (a host copy of the lengths); otherwise they are trusted.
 * Errors: INVALID_ARG / UNSUPPORTED as onmt_translate; CUDA.
 */
ONMT_API onmt_status onmt_translate_dev(onmt_model* m, const int32_t* d_src_ids, const int32_t* d_src_lens,
                               const int32_t* src_lens_host, int32_t B, int32_t S_max,
                               int32_t beam, int32_t max_len, float length_penalty,
                               int32_t* d_out_hyps, int32_t* d_out_lens, float* d_out_scores,
                               float* d_out_raw_scores, float* d_out_token_logp);

/*
 * onmt_set_option - tuning / measurement switches (name, integer value):
 *   "gemm_backend"  0 = tcgen05 tensor cores (bf16 models; default), 1 = SIMT FFMA
 *                   (always used for fp32 models).  Both compute the same sums.
 *   "profile"       1 = record CUDA events around every generator launch, 2 = around
 *                   every kernel family (see onmt_get_kernel_time); 0 = off (default).
 *   "use_graph"     1 = replay the whole translation as one cached CUDA graph (default),
 *                   0 = launch every kernel directly (profilers that cannot replay graph nodes).
 *   "fused_gemm"    1 = decoder gate and W_out GEMMs reduce their split-K partials in the
 *                   same kernel (L2 round trip + per-tile arrival counter) and apply the
 *                   LSTM cell / tanh there (default); 0 = separate partial GEMM + consumer
 *                   kernels.  Both give the same result up to fp32 summation order.
 *   "enc_persistent" 1 = an encoder layer's recurrence as one persistent launch (default),
 *                   0 = two launches per time step.
 *   "enc_cluster"   1 = a direction's recurrence as one thread-block cluster with h_{t-1} in
 *                   distributed shared memory where it fits (<= 16 gate tiles; default),
 *                   0 = the split-K grid kernel with a step barrier through L2.
 *   "enc_wavefront" 1 = unidirectional stacks as one layer-wavefront launch (default).
 *   "gen_step", "fold_wout", "rsplit"  1 = the fused generator step / folded W_out /
 *                   recurrent-split decode step where they apply (defaults), 0 = off.
 *   "regroup"       1 = single-split decoder gate GEMMs of the unfused per-layer step in row
 *                   groups sized to the SM count (default; bit-identical), 0 = the operand's
 *                   own row groups.
 *   All variants compute the same function up to fp32 summation order.
 * INVALID_ARG on an unknown name or value.
 */
ONMT_API onmt_status onmt_set_option(onmt_model* m, const char* name, int64_t value);

/*
 * onmt_get_kernel_time - with "profile" on: total milliseconds and launch count of the
 * kernel family `name` ("gen" = fused generator/log-softmax/top-k, "step" = whole
 * decode step, "encode") since the last reset; reset != 0 clears the counters.
 * Synchronises the handle's stream.
 */
ONMT_API onmt_status onmt_get_kernel_time(onmt_model* m, const char* name, int32_t reset,
                                 double* total_ms, int64_t* launches);

/* onmt_kernel_launches - number of this library's kernels launched by the handle since
 * the last call with reset != 0 (counted on the host at launch time). */
ONMT_API onmt_status onmt_kernel_launches(onmt_model* m, int32_t reset, int64_t* launches);

/* onmt_graph_captures - number of whole-call CUDA graphs the handle captured since load.
 * Every call replays a cached graph (LRU, 8 entries keyed by shape and buffer set); the
 * host-API calls pad S_max to a multiple of 8, so a corpus of batches with different
 * source lengths captures a few graphs once and then only replays (a corpus benchmark
 * reports this count).  INVALID_ARG on NULL. */
ONMT_API onmt_status onmt_graph_captures(onmt_model* m, int64_t* captures);

/*
 * Vocabulary-parallel generator (PAPER.md P219-224 names
 * multi-GPU parallelism).  `world` ranks (one process and one handle per GPU, the SAME model and
 * the SAME translate calls on every rank) split the generator's vocabulary: each rank streams
 * 1/world of W_gen per decode step and stores its per-CTA partials (max, sum exp, top-K) into
 * every rank's exchange buffer over NVLink peer memory, then raises a per-step flag there; each
 * rank's beam step waits for all flags and merges the same partials, so every rank selects the
 * same hypotheses (outputs are identical on all ranks).  The encoder and decoder layers run on
 * every rank.  Plain bf16 translation only (no copy / coverage / n-best customisations).
 *
 * onmt_vp_handle - allocate this handle's exchange buffer for up to max_rows = B x beam
 *   hypothesis rows and write its cudaIpcMemHandle (64 bytes) to handle_out.
 * onmt_vp_open   - map the other ranks' buffers: handles = world x 64 bytes in rank order (may be
 *   NULL for world == 1).  Later translate calls of the handle run vocabulary-parallel; rows above
 *   the capacity, beam > 16 or > 4 hypothesis-row groups return UNSUPPORTED.
 * onmt_vp_close  - unmap the peers and return to single-GPU decoding.
 * Errors: INVALID_ARG (bad world / rank, no handle yet), UNSUPPORTED (fp32 model), CUDA.
 */
ONMT_API onmt_status onmt_vp_handle(onmt_model* m, int32_t max_rows, void* handle_out);
ONMT_API onmt_status onmt_vp_open(onmt_model* m, int32_t world, int32_t rank, const void* handles);
ONMT_API onmt_status onmt_vp_close(onmt_model* m);

/*
 * onmt_last_plan - how the last translate / score call of the handle was executed (for
 * benchmarks and tests): rsplit = 1 if the recurrent-split decode step ran (DESIGN.md
 * §6.4b), fold = 1 if W_out was folded into attention, gen_parts = generator partials per
 * row, gate_tiles = gate tiles the generator computed per step (0 without rsplit), groups =
 * hypothesis-row groups of the generator.  INVALID_ARG on NULL.
 */
typedef struct {
  int32_t rsplit, fold, gen_parts, gate_tiles, groups;
} onmt_plan_info;
ONMT_API onmt_status onmt_last_plan(const onmt_model* m, onmt_plan_info* out);

/* onmt_free - release every device/host resource of the handle (NULL is a no-op). */
ONMT_API void onmt_free(onmt_model* m);

/* onmt_last_error - thread-local message of the last failing call ("" if none). */
ONMT_API const char* onmt_last_error(void);

/*
 * Kernel-level test entry points (C-ABI, device pointers, handle stream, synchronous).
 * onmt_test_gemm: P[s][r][m] = sum over the s-th K split of W[m][k]*X[r][k] with the
 * handle's GEMM backend; W [M x K] fp32 host, X [N x K] fp32 host, out [splits*N*M] host.
 * In bf16 handles W is rounded to bf16 and X is split into bf16 hi+lo planes
 * (DESIGN.md §6); in fp32 handles the SIMT kernel runs in fp32.
 */
ONMT_API onmt_status onmt_test_gemm(onmt_model* m, const float* W, const float* X, int32_t M, int32_t N,
                           int32_t K, int32_t splits, float* out);

/*
 * onmt_test_gen - the fused generator kernel alone: for hidden rows h~ [R x H] (host fp32)
 * returns per row the log-sum-exp of z = W_gen h~ + b over all V ids, and the top-k
 * (z, id) ordered by (z desc, id asc); lse [R], top_z [R*k], top_id [R*k].
 */
ONMT_API onmt_status onmt_test_gen(onmt_model* m, const float* htilde, int32_t R, int32_t k,
                          float* lse, float* top_z, int32_t* top_id);

#ifdef __cplusplus
}
#endif
#endif /* ONMT_H_ */
