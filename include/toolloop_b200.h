/*
 * toolloop-b200 — C ABI of the B200-native GRPO trajectory-to-loss hot path.
 *
 * Drop-in boundary for the reference's Python operators (paths relative to
 * /root/reference/pkg/src/toolloop/).  Every entry point:
 *   - takes plain device pointers + sizes and a cudaStream_t (as void*),
 *   - is stream-ordered and never synchronises the device,
 *   - never allocates device memory: scratch comes from a caller-owned
 *     workspace sized by the matching *_workspace_bytes() query,
 *   - returns TL_OK (0) or a tl_status; tl_last_error() has the message.
 * Length / shape validation that the reference performs eagerly
 * (MaskMismatch, GroupTooSmall, ValueError) is done by the host caller on
 * host-side metadata before launch; the codes below carry the same meaning.
 *
 * The F1 ingest (tl_ingest_*) and F4 tokeniser (tl_tokenizer_*,
 * tl_tokenize_segments) entry points are host-only: host pointers, no stream.
 *
 * Data types: token ids int32, masks uint8, bf16 tensors as uint16_t bit
 * patterns, log-probs float (perf mode) or double (parity mode).
 */
#ifndef TOOLLOOP_B200_H
#define TOOLLOOP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TL_ABI_VERSION 4  /* 2: tl_loss_config.entropy_norm, NCCL collectives
                             3: tl_pack_varlen traj_drop, dW-only / dH-only steps
                             4: factored store (TL_LMHEAD_NO_FACTORED / _DEBUG_FIXUP),
                                tl_grpo_lmhead_step_overlap */

typedef void* tl_stream_t; /* cudaStream_t */

typedef enum tl_status {
  TL_OK = 0,
  TL_ERR_INVALID_ARG = 1,     /* ValueError (config.py:70-78, loss.py:58-64)   */
  TL_ERR_MASK_MISMATCH = 2,   /* errors.MaskMismatch  (errors.py:28)           */
  TL_ERR_GROUP_TOO_SMALL = 3, /* errors.GroupTooSmall (errors.py:32)           */
  TL_ERR_CUDA = 4,
  TL_ERR_UNSUPPORTED = 5,
  TL_ERR_WORKSPACE = 6,
  TL_ERR_EPISODE_LOG = 7,     /* errors.EpisodeLogError (errors.py:44), "path:line: ..." */
  TL_ERR_COMM = 8             /* NCCL unavailable or a collective failed           */
} tl_status;

const char* tl_last_error(void);
int tl_abi_version(void);
/* Number of kernels this library has launched since load (monotonic). */
int64_t tl_launch_count(void);
/* Optional device timing per kernel category (CUDA events on the launching
 * stream).  enable(1) clears and starts recording, enable(0) stops;
 * read() synchronises the recorded events and returns per-category
 * milliseconds and launch counts; category(i) names category i. */
int tl_profile_enable(int32_t on);
int tl_profile_read(double* ms, int64_t* counts, int32_t n_categories);
const char* tl_profile_category(int32_t i);

/* ------------------------------------------------------------------------
 * K1 — trajectory packer.
 * Replaces trajectory.flatten (trajectory.py:154-159), trajectory.action_mask
 * (trajectory.py:162-167) and the per-token zip of rl.loss.token_records
 * (loss.py:76-100), batched over all trajectories of a step.
 *
 * Segment table: segments are listed in trajectory order; trajectory b owns
 * segments [traj_seg_off[b], traj_seg_off[b+1]).  Segment s has seg_len[s]
 * token ids stored at token_pool[seg_src_off[s] ...] (any order in the pool,
 * e.g. the arrival order of asynchronous rollout turns) and seg_is_action[s]
 * = 1 for Segment.origin == "action".
 * traj_drop [B] (nullable, build extension): 1 = drop the trajectory from the
 * update (error / timed-out episodes, whose gradients the paper masks,
 * PAPER.md:757): its tokens are packed with loss_mask 0 and no action rows,
 * so it contributes no log-prob work and no gradient and counts as an
 * all-observation trajectory of its group (loss.py:173-174, :193).
 * act_off / act_idx then count the remaining action tokens only.
 * Outputs (varlen, packed order, T = n_tokens, A = action tokens):
 *   input_ids[T], loss_mask[T], position_ids[T] (per-trajectory iota),
 *   traj_of_token[T], cu_seqlens[B+1], act_off[B+1], act_idx[A].
 * ---------------------------------------------------------------------- */
size_t tl_pack_workspace_bytes(int32_t n_traj, int32_t n_seg);
int tl_pack_varlen(const int32_t* token_pool, const int32_t* seg_src_off, const int32_t* seg_len,
                   const uint8_t* seg_is_action, const int32_t* traj_seg_off,
                   const uint8_t* traj_drop, int32_t n_traj, int32_t n_seg, int64_t n_tokens, int32_t* input_ids, uint8_t* loss_mask,
                   int32_t* position_ids, int32_t* traj_of_token, int32_t* cu_seqlens,
                   int32_t* act_off, int32_t* act_idx, void* workspace, size_t workspace_bytes,
                   tl_stream_t stream);
/* Padded [B, lmax] view of a varlen pack: pad slots get pad_id / mask 0 /
 * position 0.  Trajectories longer than lmax are an error (checked on host). */
int tl_pack_padded(const int32_t* input_ids, const uint8_t* loss_mask, const int32_t* cu_seqlens,
                   int32_t n_traj, int32_t lmax, int32_t pad_id, int32_t* ids_out,
                   uint8_t* mask_out, int32_t* pos_out, tl_stream_t stream);

/* ------------------------------------------------------------------------
 * K2 — GRPO group-normalised advantages.
 * Replaces rl.loss.group_advantages (loss.py:103-116): per group of G >= 2
 * rewards, mean = fsum(R)/G, var = fsum((R-mean)^2)/G (correctly rounded
 * sums, as math.fsum), A_i = (R_i - mean) / max(sqrt(var), std_floor).
 * Groups are contiguous runs of trajectories: group g = [group_off[g],
 * group_off[g+1]).  Also emits the per-trajectory gradient weight used by
 * the fused loss (build extension):
 *   agg = 0 (reference, cli.py:317-344): w_i = 1 / (n_i * G_g * norm_groups)
 *   agg = 1 (DAPO token-mean):           w_i = 1 / norm_tokens
 * with n_i = act_off[i+1] - act_off[i] (w_i = 0 when n_i = 0).
 * adv32 / traj_w / traj_group / act_off may be NULL.
 * ---------------------------------------------------------------------- */
int tl_group_advantages(const double* rewards, const int32_t* group_off, int32_t n_groups,
                        int32_t n_traj, double std_floor, const int32_t* act_off, int32_t agg,
                        double norm_groups, double norm_tokens, double* adv64, float* adv32,
                        float* traj_w, int32_t* traj_group, tl_stream_t stream);

/* F2 — verifiable rewards fused into K2.  Replaces the numeric part of
 * rl/rewards.py:15-68 (string matching stays on the host: `correct` is the
 * matcher's verdict, or terminated_ok for SWE):
 *   MATCH  +1 / -1 (:21-23)        MATH  +1 / -1.25 (:26-33)
 *   DEEPSEARCH  +-1 + 0.1*tool (:36-41)
 *   VISUAL_REASONER  r_acc + alpha*max(h - RaPR, 0)*invoked + beta*min(n - n_vo, 0)
 *     with RaPR = invoked responses / G of the group, computed in the warp (:43-63)
 *   SWE  1 iff terminated_ok and all tests pass (:66-68)
 * then the group advantages exactly as tl_group_advantages.  Unused signal
 * arrays may be NULL.  rapr_in [n_groups] (nullable) overrides the computed
 * RaPR (the reference takes it as an argument); rapr_out [n_groups] nullable. */
typedef enum tl_reward_kind {
  TL_REWARD_MATCH = 0,
  TL_REWARD_MATH = 1,
  TL_REWARD_DEEPSEARCH = 2,
  TL_REWARD_VISUAL_REASONER = 3,
  TL_REWARD_SWE = 4
} tl_reward_kind;
typedef struct tl_reward_params {
  int32_t kind;
  int32_t n;     /* visual reasoner: free tool calls (default 1)      */
  double h;      /* visual reasoner: RaPR target (default 0.3)        */
  double alpha;  /* visual reasoner: curiosity weight (default 0.5)   */
  double beta;   /* visual reasoner: over-use penalty (default 0.05)  */
} tl_reward_params;
int tl_group_rewards_advantages(const tl_reward_params* params, const uint8_t* correct,
                                const uint8_t* tool_called, const int32_t* n_vo,
                                const double* r_acc, const uint8_t* tests_pass,
                                const int32_t* group_off, int32_t n_groups, int32_t n_traj,
                                double std_floor, const double* rapr_in, double* rewards_out,
                                double* rapr_out, double* adv64, float* adv32,
                                tl_stream_t stream);

/* ------------------------------------------------------------------------
 * K3 — masked clipped surrogate (+ diagnostics, + per-token gradient).
 * Replaces rl.loss.grpo_multi_turn_loss (loss.py:150-201, use_mask=1),
 * grpo_single_turn_loss (loss.py:204-227, use_mask=0), unclipped_objective
 * (loss.py:230-270, objective=1), token_ratio (:119-126), _k3 (:139-147).
 * ---------------------------------------------------------------------- */
typedef struct tl_loss_config {
  double eps_low;      /* LossConfig.epsilon_clip                       */
  double eps_high;     /* = eps_low in the reference; DAPO clip-higher  */
  double kl_beta;      /* LossConfig.kl_beta                            */
  double entropy_coef; /* build extension (LM-head path only)           */
  int32_t use_mask;    /* 1 multi-turn (A11), 0 single-turn (A13)       */
  int32_t has_ref;     /* logp_ref present                              */
  int32_t objective;   /* 0 clipped (A11/A13), 1 unclipped (A14)        */
  int32_t agg;         /* 0 seq-mean-token-mean (reference), 1 token-mean */
  double entropy_norm; /* LM-head step: the entropy bonus is entropy_coef *
                          sum(entropy) / entropy_norm, i.e. the mean over the
                          step's GLOBAL action tokens when the step is split
                          into micro-batches or data-parallel shards
                          (<= 0: this call's action tokens)              */
} tl_loss_config;

/* Per-group result row of the fp64 parity path (TL_GROUP_OUT_LEN doubles):
 * objective, masked_tokens, total_tokens, clipped, clamp_count, kl_sum,
 * clip_fraction, kl  (LossDiagnostics, loss.py:67-73). */
#define TL_GROUP_OUT_LEN 8
/* Batch report (TL_REPORT_LEN doubles), cli.py:337-345 order first:
 * 0 objective, 1 clip_fraction, 2 masked_tokens, 3 kl, 4 groups, 5 episodes,
 * then additive partials for multi-rank reduction:
 * 6 total_tokens, 7 clamp_count, 8 clipped, 9 kl_sum, 10 entropy_sum,
 * 11 objective_sum (sum of per-group objectives, or of token terms for
 *    token-mean aggregation). */
#define TL_REPORT_LEN 12

/* fp64 parity mode: the reference's operation order (one sequential pass per
 * group for the sums, IEEE fp64 without contraction, correctly-rounded exp).
 * Inputs per packed token; grad (nullable) = d objective / d logp_new (A14
 * for objective=1, the clipped-arm restatement for objective=0). */
size_t tl_loss_f64_workspace_bytes(int64_t n_tokens);
int tl_loss_f64(const double* logp_new, const double* logp_old, const double* logp_ref,
                const uint8_t* mask, const int32_t* cu_seqlens, const int32_t* group_off,
                const double* adv, int32_t n_traj, int32_t n_groups, int64_t n_tokens,
                const tl_loss_config* cfg, double* grad, double* group_out, void* workspace,
                size_t workspace_bytes, tl_stream_t stream);
/* cli.loss aggregation over per-group rows (cli.py:309-345), reference order. */
int tl_report_f64(const double* group_out, int32_t n_groups, int32_t n_traj, double* report,
                  tl_stream_t stream);
/* Exact-reference elementwise helpers (token_ratio / _k3) for API parity. */
int tl_token_ratio_f64(const double* logp_new, const double* logp_old, int64_t n, double* ratio,
                       tl_stream_t stream);

/* fp32 performance mode: per-token terms in fp32, deterministic fixed-order
 * reductions (per trajectory -> per group -> batch) in fp64.  grad (nullable)
 * = d objective / d logp_new (report objective, i.e. already scaled by
 * traj_w).  traj_w from tl_group_advantages. */
size_t tl_loss_f32_workspace_bytes(int64_t n_tokens, int32_t n_traj, int32_t n_groups);
int tl_loss_f32(const float* logp_new, const float* logp_old, const float* logp_ref,
                const uint8_t* mask, const int32_t* traj_of_token, const int32_t* cu_seqlens,
                const int32_t* group_off, const float* adv32, const float* traj_w,
                int32_t n_traj, int32_t n_groups, int64_t n_tokens, const tl_loss_config* cfg,
                float* grad, double* report, void* workspace, size_t workspace_bytes,
                tl_stream_t stream);

/* ------------------------------------------------------------------------
 * K4/K5 — fused LM-head log-prob / entropy (+ surrogate epilogue) and its
 * backward, on tcgen05/TMEM/TMA.  No reference implementation: contract of
 * PolicyAction.token_logprobs (rollout/policy.py:25-28) / TokenRecord.logp_new
 * (loss.py:30).  hidden row t predicts target input_ids[t] (caller shifts).
 * Only action rows (act_idx) are computed, in chunks of chunk_rows action
 * rows.  The forward sweeps the vocabulary in 256-wide tiles with an online
 * log-sum-exp, so the log-probs never need [T, V] logits.  The backward
 * needs p = softmax(z) once the final LSE is known: STORE_LOGITS keeps ONE
 * chunk's [chunk_rows, V] 2-byte buffer (46 GB at 4 x 37,888 rows and
 * V = 152,064) — bf16 q = e^(z - m0) that the dH / dW GEMMs read directly
 * (factored, no entropy bonus), or fp16 logits turned into bf16 dS in place
 * (entropy bonus on); RECOMPUTE keeps no logits and recomputes them in a
 * second GEMM.  [T, V] is never allocated: one chunk at a time.
 * ---------------------------------------------------------------------- */
/* Workspace of tl_grpo_lmhead_step in the serial modes (STORE_LOGITS,
 * RECOMPUTE) with the backward: one chunk's [chunk_rows, V] dS buffer, the
 * split-K tail slices and the step's per-token / per-trajectory state. */
size_t tl_lmhead_workspace_bytes(int32_t chunk_rows, int32_t hidden, int32_t vocab, int64_t n_tokens,
                                 int32_t n_traj, int32_t n_groups);
/* Workspace of tl_lmhead_logprobs (forward only: h_c rows + per-row stats,
 * no dS buffer — ~C*H*2 bytes, 1.1 GB at C = 151,552 rows and H = 3,584). */
size_t tl_lmhead_logprobs_workspace_bytes(int32_t chunk_rows, int32_t hidden, int32_t vocab);
/* Forward only: logp/entropy/lse for rows idx[0..n_rows) of hidden
 * (F3: rollout-side logp_old / logp_ref).  Outputs indexed like idx
 * (out[k] for row idx[k]); idx NULL = rows 0..n_rows-1. */
int tl_lmhead_logprobs(const uint16_t* hidden, const uint16_t* weight, const int32_t* targets,
                       const int32_t* idx, int64_t n_rows, int32_t hidden_dim, int32_t vocab,
                       float* logp, float* entropy, float* lse, int32_t chunk_rows,
                       void* workspace, size_t workspace_bytes, tl_stream_t stream);
/* Backward modes of tl_grpo_lmhead_step.
 *  STORE_LOGITS: the forward epilogue also writes the chunk's logits into the
 *    [chunk_rows, V] workspace (6*T*H*V issued FLOPs; [T, V] is never
 *    allocated — only one chunk at a time).  Without the entropy bonus
 *    (entropy_coef == 0) dS = alpha_r * q row by row, so the forward stores
 *    bf16 q = e^(z - m0) against a per-row anchor m0 and the dH / dW GEMMs
 *    read q with alpha folded into the dH epilogue and into h_c ("factored",
 *    no elementwise pass); with the bonus it stores fp16 logits and an
 *    elementwise pass turns them into bf16 dS in place.
 *  RECOMPUTE: the backward recomputes the logits with a second GEMM whose
 *    epilogue writes dS (8*T*H*V issued FLOPs; no logits ever leave TMEM). */
#define TL_LMHEAD_STORE_LOGITS 0
#define TL_LMHEAD_RECOMPUTE 1
/*  STORE_LOGITS_PIPELINED: STORE_LOGITS with two chunk buffers; chunk i's
 *    elementwise dS pass runs on an internal side stream concurrently with
 *    chunk i+1's forward GEMM (workspace: tl_lmhead_step_workspace_bytes). */
#define TL_LMHEAD_STORE_LOGITS_PIPELINED 2
/* Flag OR-ed into `mode`: dweight += this call's dW instead of dweight = dW
 * (micro-batches of one optimizer step; pass the step's global norm_groups /
 * norm_tokens to tl_group_advantages so every micro-batch scales alike). */
#define TL_LMHEAD_ACCUMULATE_DW 0x100
/* Debug flag OR-ed into `mode`: run the dW GEMM's partial last wave unsplit
 * (no split-K tail); results agree to fp32 summation order (tests). */
#define TL_LMHEAD_NO_SPLIT_TAIL 0x200
/* Debug flag OR-ed into `mode`: keep the fp16-logit store + dS pass even
 * when the factored store applies.  STORE_LOGITS without the entropy bonus
 * (entropy_coef == 0) otherwise writes bf16 q = e^(z - m0) against a per-row
 * anchor m0 and runs dH / dW on q with a per-row scale (dS = alpha_r q plus
 * one element per row): no elementwise dS pass, same workspace. */
#define TL_LMHEAD_NO_FACTORED 0x400
/* Test hook OR-ed into `mode`: the factored store treats every row as out of
 * its anchor's range and rewrites it on CUDA cores (slow; exercises the
 * fallback that rows with lse - m0 outside [-45, 80] take). */
#define TL_LMHEAD_DEBUG_FIXUP 0x800
/* Workspace for tl_grpo_lmhead_step in `mode` (PIPELINED holds two chunks). */
size_t tl_lmhead_step_workspace_bytes(int32_t chunk_rows, int32_t hidden, int32_t vocab,
                                      int64_t n_tokens, int32_t n_traj, int32_t n_groups,
                                      int32_t mode);
/* Whole GRPO step on device-resident tensors:
 *   logp_new = LMhead(hidden[act rows]); surrogate (K3 math) fused into the
 *   log-prob epilogue; report; loss = -(objective + entropy_coef * mean
 *   entropy); dhidden = dloss/dhidden (bf16 [T, H], observation rows zeroed),
 *   dweight = dloss/dW (fp32 [V, H], overwritten; accumulated with
 *   TL_LMHEAD_ACCUMULATE_DW).  dweight NULL = frozen LM head (dS and dH
 *   only, 4*T_act*H*V issued FLOPs in store mode); dhidden NULL = detached
 *   hidden states (dW only); both NULL = forward + report only. */
int tl_grpo_lmhead_step(const uint16_t* hidden, const uint16_t* weight, const int32_t* input_ids,
                        const uint8_t* loss_mask, const int32_t* act_idx, int64_t n_act,
                        const int32_t* traj_of_token, const int32_t* cu_seqlens,
                        const int32_t* group_off, const float* logp_old, const float* logp_ref,
                        const float* adv32, const float* traj_w, int64_t n_tokens,
                        int32_t hidden_dim, int32_t vocab, int32_t n_traj, int32_t n_groups,
                        const tl_loss_config* cfg, float* logp_out, float* entropy_out,
                        uint16_t* dhidden, float* dweight, double* report, int32_t chunk_rows,
                        int32_t mode, void* workspace, size_t workspace_bytes,
                        tl_stream_t stream);

/* N2 overlap (data parallel, see tl_allreduce_f32 below).  With
 * dw_ready_event != NULL the step runs its last chunk's dW GEMM before that
 * chunk's dH GEMM and records the event (a cudaEvent_t) on `stream` as soon
 * as dweight is final; the last dH GEMM then leaves reserve_sms SMs free.  A
 * caller that makes another stream wait on the event and issues the dW
 * all-reduce / reduce-scatter there gets the collective running beside the
 * last dH GEMM instead of after the step (every GEMM otherwise holds all
 * SMs).  Outputs are bitwise those of tl_grpo_lmhead_step. */
typedef struct tl_step_overlap {
  void* dw_ready_event;  /* cudaEvent_t, or NULL */
  int32_t reserve_sms;   /* >= 0; rounded up to whole CTA pairs */
} tl_step_overlap;
int tl_grpo_lmhead_step_overlap(const uint16_t* hidden, const uint16_t* weight,
                                const int32_t* input_ids, const uint8_t* loss_mask,
                                const int32_t* act_idx, int64_t n_act,
                                const int32_t* traj_of_token, const int32_t* cu_seqlens,
                                const int32_t* group_off, const float* logp_old,
                                const float* logp_ref, const float* adv32, const float* traj_w,
                                int64_t n_tokens, int32_t hidden_dim, int32_t vocab,
                                int32_t n_traj, int32_t n_groups, const tl_loss_config* cfg,
                                float* logp_out, float* entropy_out, uint16_t* dhidden,
                                float* dweight, double* report, int32_t chunk_rows, int32_t mode,
                                void* workspace, size_t workspace_bytes, tl_stream_t stream,
                                const tl_step_overlap* overlap);

/* ------------------------------------------------------------------------
 * F1 — episode-log / sidecar ingest (host, multithreaded C++).
 * Replaces rollout/episodes.read_episodes (episodes.py:132-147) +
 * EpisodeRecord.from_dict (:95-120) + trajectory_from_dict
 * (trajectory.py:182-200), cli._read_sidecar (cli.py:255-269),
 * cli._flat_logps (cli.py:233-252) and the task_id grouping of cli.loss
 * (cli.py:309-311).  Produces the SoA segment table of tl_pack_varlen with
 * episodes permuted so each task_id group (first-appearance order) is
 * contiguous, plus per-token fp64 log-probs (logp_ref NaN where a sidecar row
 * has none).  sidecar_path NULL = log-probs embedded in the episode log
 * (logp_old := logp_new, observation positions 0.0).
 * ---------------------------------------------------------------------- */
typedef struct tl_episode_batch tl_episode_batch;
int tl_ingest_open(const char* episodes_path, const char* sidecar_path, tl_episode_batch** out);
int tl_ingest_sizes(const tl_episode_batch* batch, int64_t* n_episodes, int64_t* n_segments,
                    int64_t* n_tokens, int64_t* n_groups, int32_t* has_ref);
int tl_ingest_fill(const tl_episode_batch* batch, int32_t* token_pool, int32_t* seg_src_off,
                   int32_t* seg_len, uint8_t* seg_is_action, int32_t* traj_seg_off,
                   int32_t* group_off, double* rewards, double* logp_new, double* logp_old,
                   double* logp_ref);
void tl_ingest_free(tl_episode_batch* batch);

/* ------------------------------------------------------------------------
 * F4 — incremental tokenisation of rollout segments (host, multithreaded C++).
 * Replaces tokenizer.ToyMergeTokenizer (tokenizer.py:36-87: byte ids 0..255,
 * ordered merge table, rule k -> id 256+k, one left-to-right pass per rule)
 * applied segment by segment with the token cap of trajectory._tokenize
 * (trajectory.py:97-104) / orchestrator.feed_action, feed_response
 * (orchestrator.py:112-117, :156-161).
 * ---------------------------------------------------------------------- */
typedef struct tl_tokenizer tl_tokenizer;
/* Merge k = (left, right) byte strings: left = merge_bytes[off[2k], off[2k+1]),
 * right = merge_bytes[off[2k+1], off[2k+2]).  Both must already be tokens
 * (TL_ERR_INVALID_ARG otherwise, tokenizer.py:55-58 ValueError). */
int tl_tokenizer_create(const uint8_t* merge_bytes, const int64_t* merge_off, int32_t n_merges,
                        tl_tokenizer** out);
void tl_tokenizer_free(tl_tokenizer* tok);
int32_t tl_tokenizer_vocab_size(const tl_tokenizer* tok);
/* Encode segment i = text[text_off[i], text_off[i+1]) on its own (never across
 * a segment boundary), keep its first max_tokens[i] ids (max_tokens NULL or
 * < 0: no cap).  Ids go to token_pool[text_off[i] ...] (never more ids than
 * bytes), so (token_pool, seg_src_off = text_off, seg_len) is directly the
 * segment table of tl_pack_varlen.  n_threads <= 0: all hardware threads. */
int tl_tokenize_segments(const tl_tokenizer* tok, const uint8_t* text, const int64_t* text_off,
                         int64_t n_segments, const int32_t* max_tokens, int32_t* token_pool,
                         int32_t* seg_len, int32_t n_threads);
/* Bytes of ids[0..n) (ToyMergeTokenizer.decode before UTF-8 decoding): *len =
 * total bytes; copied into out only if they fit in cap (out NULL: size only). */
int tl_tokenizer_decode(const tl_tokenizer* tok, const int32_t* ids, int64_t n, uint8_t* out,
                        int64_t cap, int64_t* len);

/* ------------------------------------------------------------------------
 * N1 / N2 — data-parallel collectives (NCCL, stream-ordered).
 * Replaces the serial per-group loop + aggregation of cli.loss
 * (cli.py:317-344; groups are independent): each rank runs the
 * step on its own whole groups with the global normalisers, then
 *   N1  tl_allreduce_report: the TL_REPORT_LEN report summed over ranks
 *       (additive partials) and its ratio fields recomputed, in place;
 *   N2  tl_allreduce_f32 (dW, in place) or tl_reduce_scatter_f32 (dW row
 *       shard [V / nranks, H] when W is partitioned).
 * `comm` is an ncclComm_t (void*): create one with tl_nccl_unique_id on one
 * rank, broadcast the id, tl_nccl_comm_init on every rank (current device),
 * or pass a communicator the caller already owns.  NCCL is loaded at run
 * time (libnccl.so.2); without it these return TL_ERR_COMM and
 * tl_nccl_available() is 0.
 * ---------------------------------------------------------------------- */
#define TL_NCCL_UNIQUE_ID_BYTES 128
int tl_nccl_available(void);
int tl_nccl_version(void);
int tl_nccl_unique_id(uint8_t* id_out /* TL_NCCL_UNIQUE_ID_BYTES */);
int tl_nccl_comm_init(void** comm_out, const uint8_t* id, int32_t nranks, int32_t rank);
int tl_nccl_comm_destroy(void* comm);
int tl_nccl_comm_size(void* comm, int32_t* nranks);
/* sum of n doubles over ranks, in place (SURVEY §8(b) tl_allreduce_scalars) */
int tl_allreduce_scalars(void* comm, double* x, int32_t n, tl_stream_t stream);
/* N1: report[TL_REPORT_LEN] of each rank -> the global report (agg as tl_loss_config.agg) */
int tl_allreduce_report(void* comm, double* report, int32_t agg, tl_stream_t stream);
/* N2: dW all-reduce (in place) / reduce-scatter (rank r receives elements
 * [r * shard_n, (r + 1) * shard_n) of the sum; buf holds nranks * shard_n) */
int tl_allreduce_f32(void* comm, float* buf, int64_t n, tl_stream_t stream);
int tl_reduce_scatter_f32(void* comm, const float* buf, float* shard, int64_t shard_n,
                          tl_stream_t stream);

/* Plain tcgen05 GEMM (building block, exported for tests):
 * C[M,N] (+)= A[M,K] * B[N,K]^T with A given K-major ([M,K], lda) or MN-major
 * ([K,M], lda) and B K-major ([N,K], ldb) or MN-major ([K,N], ldb).
 * C is bf16 (c_fp32=0) or fp32 (c_fp32=1, accumulate allowed). */
int tl_gemm_bf16(const uint16_t* A, int32_t a_mn_major, int64_t lda, const uint16_t* B,
                 int32_t b_mn_major, int64_t ldb, int32_t M, int32_t N, int32_t K, void* C,
                 int32_t c_fp32, int64_t ldc, int32_t accumulate, tl_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* TOOLLOOP_B200_H */
