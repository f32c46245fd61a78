/*
 * wanspec_b200.h — C ABI of the B200-native WANSpec verify / draft hot path.
 *
 * The reference (arxiv 2602.18931, /root/reference/proj) is header-only C++20 with no
 * ABI: the hot path sits behind three in-process model calls made at step completion
 * by the harnesses:
 *
 *   1. target verify  ValidationResult run_target_step(const SequenceTrace&, uint64_t base,
 *                                                      span<const TokenId>)   oracle.hpp:127-139
 *                     callers sim.hpp:297, runtime.hpp:308/:425/:475
 *   2. worker draft   Prediction SequenceTrace::draft_prediction(uint64_t pos)  oracle.hpp:96-98
 *                     callers sim.hpp:314, runtime.hpp:197
 *   3. local draft    same function, callers sim.hpp:307, runtime.hpp:319/:434/:480
 *
 * and the results are folded back by apply_target_result (controller.hpp:235),
 * apply_local_draft (controller.hpp:273) and apply_draft_output (worker.hpp:110).
 *
 * This header is what a maintainer binds instead: plain pointers and
 * sizes, caller-owned host buffers, every entry point total and returning 0 or a negative
 * WS_E* code (the reference's error classes, types.hpp:35-45). Model calls are batched
 * over many requests/leaves per launch; the batched event driver (ws_run_sim) replaces
 * run_sim_full (sim.hpp:429-442) with the same per-request semantics.
 *
 * There is no CPU fallback: every model call runs on the GPU of the context; without a
 * CUDA device ws_create fails with WS_ECUDA.
 */
#ifndef WANSPEC_B200_H
#define WANSPEC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WS_ABI_VERSION 1

/* ---- status codes (types.hpp:35-45 error classes; sim.hpp:198/:200 logic errors) ---- */
#define WS_OK 0
#define WS_ECONFIG (-1) /* ConfigError  types.hpp:35 (OracleConfig/SimConfig::validate) */
#define WS_EPARSE (-2)  /* ParseError   types.hpp:39 */
#define WS_EPROTO (-3)  /* ProtocolError types.hpp:43 */
#define WS_ELOGIC (-4)  /* std::logic_error: event budget / unfinished request sim.hpp:198,:200 */
#define WS_ECUDA (-5)   /* CUDA runtime/driver failure, or no device */
#define WS_EARG (-6)    /* null pointer / size out of range / buffer too small */

/* ---- verify modes ---- */
#define WS_VERIFY_GREEDY 0     /* run_target_step oracle.hpp:127-139 (parity-pinned) */
#define WS_VERIFY_REJECTION 1  /* Philox4x32-10 speculative rejection sampling (extension) */

/* ---- sim modes (sim.hpp:26) ---- */
#define WS_MODE_BASELINE 0
#define WS_MODE_WANSPEC 1

/* TokenRecord (types.hpp:67-72) with the top-2 Prediction (types.hpp:56-63) the stochastic
 * oracle synthesizes (oracle.hpp:313-345). Fixed layout, 64 bytes. */
typedef struct ws_token_record {
  uint32_t target_token;  /* == target top-1 */
  uint32_t target_top2;
  double target_p1, target_p2, target_entropy;
  uint32_t draft_top1, draft_top2;
  double draft_p1, draft_p2, draft_entropy;
} ws_token_record;

/* Prediction reduced to what the protocol consumes (types.hpp:56-63): n = 1 or 2 candidates
 * in descending probability (ties by ascending id), entropy in nats. Past-end positions
 * yield {(eos, 1.0)}, entropy 0 (oracle.hpp:88-102, :118). */
typedef struct ws_pred {
  uint32_t n;
  uint32_t id[2];
  uint32_t pad;
  double prob[2];
  double entropy;
} ws_pred;

/* OracleConfig (oracle.hpp:37-47), stochastic kind only. */
typedef struct ws_oracle_cfg {
  uint64_t seed;
  uint32_t vocab_size;
  uint32_t eos_id;
  double match_prob;
  double entropy_low;
  double entropy_high;
  double second_correct_prob;
  uint32_t sequence_length;
  uint32_t pad;
} ws_oracle_cfg;

/* SimConfig (sim.hpp:28-80) plus the verify mode / sampling key of the extension. */
typedef struct ws_sim_cfg {
  int32_t mode;        /* WS_MODE_* */
  int32_t verify;      /* WS_VERIFY_* */
  int64_t rtt;         /* µs */
  int64_t jitter;      /* µs, uniform +/- per frame */
  int64_t r_estimate;  /* µs, <0 = use rtt */
  int64_t t_target;    /* µs */
  int64_t t_draft;     /* µs */
  uint32_t k, b, s;
  uint32_t catchup_batch_limit;
  double theta, phi;
  uint32_t max_nodes;
  int32_t wait_backstop;
  uint32_t num_requests;  /* requests dealt from the oracle stream, in order */
  uint32_t first_request; /* shard: run requests [first_request, first_request+local_requests) */
  uint32_t local_requests;/* 0 = all from first_request */
  uint32_t host_threads;  /* protocol threads for ws_run_sim (0 = 1); one CUDA stream each */
  uint64_t sample_seed;   /* Philox key for WS_VERIFY_REJECTION */
  ws_oracle_cfg oracle;
  /* model path, WS_VERIFY_REJECTION only (K4R, kernels/sample.cuh): nucleus mass (0 or >= 1 =
   * no truncation) and softmax temperature (0 = 1) of the target distribution */
  float top_p;
  float temperature;
} ws_sim_cfg;

/* RequestMetrics (sim.hpp:121-134). */
typedef struct ws_request_metrics {
  int64_t latency;
  uint64_t tokens_committed;
  uint64_t target_steps;
  uint64_t ctrl_draft_passes;
  uint64_t ctrl_local_draft_steps;
  uint64_t ctrl_catchup_batches;
  uint64_t worker_draft_steps;
  uint64_t sync_stalls;
  uint64_t entropy_resets;
  uint64_t stale_specs;
} ws_request_metrics;

/* One verify step as folded by apply_target_result (controller.hpp:235-266). */
#define WS_STEP_SYNC_STALL 1u     /* length < k+1: resync-on-mismatch, t_update = now */
#define WS_STEP_ENTROPY_RESET 2u  /* full accept, final_entropy > phi: t_update = now */
typedef struct ws_step_log {
  uint32_t request;
  uint32_t step;
  uint64_t base;
  uint32_t accepted;
  uint32_t bonus;
  double final_entropy;
  int64_t time;  /* virtual µs at fold time */
  uint32_t flags;
  uint32_t pad;
} ws_step_log;

/* Outputs of a run (RunOutputs sim.hpp:420-427). All buffers caller-owned; any may be
 * NULL to skip. Token buffers are [local_requests * max_len]. */
typedef struct ws_run_out {
  ws_request_metrics* metrics;
  uint32_t* ctrl_tokens;
  uint32_t* ctrl_len;
  uint32_t* wrk_tokens;
  uint32_t* wrk_len;
  uint32_t max_len;
  uint32_t pad;
  ws_step_log* steps;
  uint64_t max_steps;
  uint64_t n_steps;       /* out */
  /* execution statistics (out) */
  uint64_t rounds;        /* batched GPU rounds */
  uint64_t gpu_launches;  /* kernels launched by this run */
  uint64_t verify_rows;   /* verify jobs executed */
  uint64_t draft_rows;    /* draft rows executed */
  double kernel_ms;       /* summed device time of the hot-path kernels (CUDA events) */
  uint64_t h2d_bytes;     /* host->device bytes copied by the run */
  uint64_t d2h_bytes;     /* device->host bytes copied by the run */
} ws_run_out;

typedef struct ws_ctx ws_ctx;

/* ---- lifetime ---- */
int ws_abi_version(void);
int ws_device_count(int* out);
int ws_create(int device, ws_ctx** out);
int ws_destroy(ws_ctx* ctx);
/* Thread-local message of the last failing call ("" if none). */
const char* ws_last_error(void);

/* ---- the tiny draft/target pair (oracle.hpp:262-352) ----
 * Host synthesis of n_seq sequences in the reference's draw order (oracle.hpp:320) from
 * one mt19937_64 stream; out is [n_seq * sequence_length]. Pure host arithmetic (it is
 * the "model weights" of the tiny pair) — no GPU needed. */
int ws_oracle_synth(const ws_oracle_cfg* cfg, uint32_t n_seq, ws_token_record* out);

/* Upload tables to device memory (K9 mode): n_seq sequences of seq_len records. */
int ws_load_oracle(ws_ctx* ctx, uint32_t n_seq, uint32_t seq_len, uint32_t vocab_size,
                   uint32_t eos_id, const ws_token_record* records);

/* ---- batched model calls over the device tables (host buffers in/out) ---- */
/* run_target_step × n (oracle.hpp:127-139): job j verifies cand[j*k .. j*k+k) anchored at
 * base[j] of sequence seq[j]. Outputs accepted length, bonus token, final entropy. */
int ws_verify(ws_ctx* ctx, uint32_t n, uint32_t k, const uint32_t* seq, const uint64_t* base,
              const uint32_t* cand, uint32_t* acc_len, uint32_t* bonus, double* final_entropy);

/* Rejection-sampling verify × n (extension, parity unpinned by the reference): accept c_i
 * iff u_i * p_d(c_i) < p_t(c_i), u from Philox4x32-10 keyed (sample_seed) with counter
 * (request[j], step[j], i); residual/bonus draw from the same counter's upper words. */
int ws_verify_rejection(ws_ctx* ctx, uint32_t n, uint32_t k, uint64_t sample_seed,
                        const uint32_t* seq, const uint64_t* request, const uint32_t* step,
                        const uint64_t* base, const uint32_t* cand, uint32_t* acc_len,
                        uint32_t* bonus, double* final_entropy);

/* draft_prediction × n (oracle.hpp:96-98). */
int ws_draft(ws_ctx* ctx, uint32_t n, const uint32_t* seq, const uint64_t* pos, ws_pred* out);

/* ---- whole runs: run_sim_full (sim.hpp:429-442) through the batched driver ----
 * Synthesizes cfg->num_requests sequences in order (host), uploads them, and runs the
 * shard [first_request, first_request+local_requests) with every model step batched
 * across requests on the GPU. Per-request results are identical to the reference. */
int ws_run_sim(ws_ctx* ctx, const ws_sim_cfg* cfg, ws_run_out* out);

/* Same, with tables already resident (ws_load_oracle) — the device-resident timing path. */
int ws_run_sim_resident(ws_ctx* ctx, const ws_sim_cfg* cfg, ws_run_out* out);

/* ---- batched job records (driver rounds, K9 kernel, model seam) ---- */
typedef struct ws_verify_job {
  uint32_t seq;       /* request's table block */
  uint32_t k;
  uint64_t base;
  uint64_t request;   /* Philox counter words (rejection mode) */
  uint32_t step;      /* per-request verify step index */
  uint32_t cand_off;  /* offset into the round's candidate array */
} ws_verify_job;
typedef struct ws_draft_job {
  uint32_t seq;
  uint32_t pad;
  uint64_t pos;
} ws_draft_job;
typedef struct ws_verify_out {
  uint32_t accepted;
  uint32_t bonus;
  double final_entropy;
} ws_verify_out;
/* ---- device-pointer kernel entry points (the model path's building blocks) ----
 * All pointers are device memory; `stream` is a cudaStream_t (NULL = legacy default). */
#define WS_EPI_BF16 0    /* out bf16 = A·W^T */
#define WS_EPI_ADD_F32 1 /* out fp32 += A·W^T (residual stream) */
#define WS_EPI_SWIGLU 2  /* out bf16 = silu(gate)·up, W rows interleaved in 32-row gate/up blocks */
/* K1: C[M,N] = A[M,K]·W[N,K]^T, bf16 operands, fp32 accumulation in TMEM (tcgen05 + TMA).
 * bn: N-tile width (0 = auto); splits: split-K factor (1 = none, 0 = the (N,K)-determined
 * count the model uses), partials summed in fixed split order (deterministic). */
int ws_op_gemm_bf16(const void* A, const void* W, void* out, int M, int N, int K, int lda, int ldw,
                    int ldo, int epi, int bn, int splits, void* stream);

/* K3: per row of bf16 logits [rows, ld]: top-2 (id, prob) of softmax(x·inv_temp), ties to the
 * lower id, and the entropy in nats (entropy_of semantics, oracle.hpp:21-33), fp32 reductions.
 * out: ws_pred[rows]; stats (optional): float4[rows] = {max·cl, Z, cl, H}, cl = inv_temp·log2 e.
 * workspace: >= ws_op_row_stats_workspace_bytes(), zero-filled once (self-resetting). */
size_t ws_op_row_stats_workspace_bytes(uint32_t rows, uint32_t vocab, uint32_t n_req);
int ws_op_row_stats_bf16(const void* logits, uint32_t rows, uint32_t vocab, uint32_t ld,
                         float inv_temp, ws_pred* out, void* stats, void* workspace, void* stream);
/* K3+K4: greedy verify over n_req groups of k+1 logits rows (row i of request j predicts
 * position base_j + i): run_target_step (oracle.hpp:127-139) on the argmaxes, fused. */
int ws_op_verify_greedy_bf16(const void* logits, uint32_t n_req, uint32_t k, uint32_t vocab,
                             uint32_t ld, const uint32_t* cand, ws_verify_out* out,
                             ws_pred* rows_out, void* workspace, void* stream);

/* K4R: speculative rejection sampling over n_req groups of k+1 bf16 logits rows (extension,
 * kernels/sample.cuh): accept c_i iff u * q_i < p'(c_i) with u from Philox4x32-10 keyed seed,
 * counter (request[j], step[j], i); residual / bonus draws over the full vocabulary; optional
 * top-p nucleus and temperature. All pointers device memory; forced (may be NULL): per row,
 * >= 0 = a point mass on that token. */
int ws_op_verify_rejection_bf16(const void* logits, uint32_t n_req, uint32_t k, uint32_t vocab, uint32_t ld,
                                float inv_temp, float top_p, const uint32_t* cand, const double* cand_prob,
                                uint64_t seed, const uint64_t* request, const uint32_t* step,
                                const int32_t* forced, ws_verify_out* out, void* stream);

/* ---- real-model pair (BASELINE config 3): Llama-shape target + draft on one GPU ----
 * Random-init bf16 weights of the named shapes ("llama3-8b", "llama3.2-1b", "tiny", ...),
 * prompts of prompt_len seeded tokens, and a planted shared bigram bias (a seeded hash of the
 * input token receives +plant logits; the draft sees it for draft_plant_rate of input tokens)
 * so draft and target agree at a controllable rate. Generation is capped like the tiny pair:
 * rows predicting committed index >= sequence_length-1 emit EOS with probability 1. */
typedef struct ws_model_cfg {
  const char* target;
  const char* draft;
  uint64_t seed;
  uint32_t prompt_len;
  uint32_t max_requests;
  uint32_t max_ctx;
  uint32_t trie_slots;
  float plant_target;
  float plant_draft;
  float draft_plant_rate;
  uint32_t tp;  /* target tensor-parallel ranks on GPUs device .. device+tp-1 (0/1 = one GPU) */
} ws_model_cfg;
int ws_model_load(ws_ctx* ctx, const ws_model_cfg* cfg);
/* Split placement: the target (verify) model on the context's GPU and the draft
 * model — the worker's rollout and the controller's local drafts — on `draft_device`, each lane
 * on its own GPU; requests' proposals and verify results meet in the host driver. A negative
 * draft_device is ws_model_load. */
int ws_model_load_split(ws_ctx* ctx, const ws_model_cfg* cfg, int draft_device);
/* Teacher-forced trace export (the reference's docs/trace_format.md records):
 * for requests [first_request, first_request + n) of the loaded pair, the target's greedy
 * continuation of each prompt for `length` positions; every record holds the target's and the
 * draft's top-2 and entropy on the same committed context (the reference's TokenRecord,
 * oracle.hpp:52-70). out: n * length records, request-major. Resets the pair's KV caches. */
int ws_model_export_trace(ws_ctx* ctx, uint32_t first_request, uint32_t n, uint32_t length,
                          ws_token_record* out);
/* run_sim_full (sim.hpp:429-442) with the verify / draft model calls on the loaded models;
 * cfg->oracle supplies vocab_size (must equal the models'), eos_id and sequence_length. */
int ws_run_model_sim(ws_ctx* ctx, const ws_sim_cfg* cfg, ws_run_out* out);
/* Wall-clock mode (the reference's networked runtime, runtime.hpp:153-386, in-box): every
 * request's controller and worker state machines run on the host against real time; model steps
 * complete when their GPU work completes (not after t_target / t_draft); proposals and
 * validations cross per-request host queues whose frames become visible rtt/2 (+/- jitter) after
 * sending, FIFO-clamped (LatencyEmulator, net.hpp:149-163). metrics.latency is real µs.
 * decision_log (may be NULL): an NDJSON controller decision log (DecisionLog, runtime.hpp:227-237,
 * plus the model results) that a fresh state machine replays to the same decisions. */
int ws_run_model_wallclock(ws_ctx* ctx, const ws_sim_cfg* cfg, ws_run_out* out, const char* decision_log);
/* model-step timing of the last ws_run_model_sim: device ms and rows fed per model */
int ws_model_stats(ws_ctx* ctx, double* target_ms, double* draft_ms, uint64_t* target_rows,
                   uint64_t* draft_rows, uint64_t* target_forwards, uint64_t* draft_forwards);

/* ---- per-call model boundary (the reference's three model calls) ----
 * For callers that keep their own controller / worker state machines (the reference's
 * RequestSim or runtime) and call the loaded models once per step:
 *   run_target_step  (oracle.hpp:127-139; callers sim.hpp:297, runtime.hpp:308)  -> ws_model_verify
 *   draft_prediction (oracle.hpp:96-98;  callers sim.hpp:307/:314, runtime.hpp:197/:319)
 *                                                                                 -> ws_model_draft
 * A job names a request (its seeded prompt and KV region in the loaded pair) and the tokens
 * after the prompt: the committed output, then (drafts) the speculative path. Real models are
 * context-dependent, so the draft calls take the leaf's path where the reference passes only
 * its anchor position. KV caches are content-addressed: every job's context is matched
 * against the request's cached tokens (longest common prefix for the verify and controller
 * draft caches, a token trie of speculative nodes over the committed prefix for the worker),
 * only the missing rows are fed, and accepted speculative KV migrates into the prefix on the
 * next job — commit and fork need no call (a fork is two children in the trie; attention
 * masks let them share every ancestor's KV in place). Results equal ws_run_model_sim's for the
 * same contexts bit for bit (batch-invariant kernels). Rows predicting committed index >=
 * sequence_length - 1 emit eos_id with probability 1, the tiny pair's past-end rule
 * (oracle.hpp:88-102). */
#define WS_JOB_VERIFY 0u
#define WS_JOB_CTRL_DRAFT 1u   /* controller local draft / catch-up (controller.hpp:194-208) */
#define WS_JOB_WORKER_DRAFT 2u /* worker frontier leaf (worker.hpp:93-96) */
typedef struct ws_model_job {
  uint32_t request;
  uint32_t kind;        /* WS_JOB_* */
  uint32_t n_committed; /* committed tokens at the head of the context */
  uint32_t len;         /* context tokens after the prompt (verify: == n_committed) */
  uint64_t off;         /* offset of this job's context in the tokens array */
} ws_model_job;
/* Starts a per-call session on the loaded pair: forgets every cached KV, sets k and the
 * generation cap. */
int ws_model_open(ws_ctx* ctx, uint32_t k, uint32_t sequence_length, uint32_t eos_id);
/* Prompt prefill of the listed requests (optional: a first job would feed its prompt too). */
int ws_model_prefill(ws_ctx* ctx, uint32_t n, const uint32_t* requests);
/* run_target_step x n in one target forward + K3/K4: job j verifies cand[j*k .. j*k+k) after
 * its committed context. out[j] = (accepted, bonus, final_entropy); rows_opt (may be NULL):
 * the n*(k+1) per-row predictions (top-2 + entropy) the walk read. */
int ws_model_verify(ws_ctx* ctx, uint32_t n, const ws_model_job* jobs, const uint32_t* tokens,
                    const uint32_t* cand, ws_verify_out* out, ws_pred* rows_opt);
/* draft_prediction x n in one draft forward + K3: the prediction after each job's context. */
int ws_model_draft(ws_ctx* ctx, uint32_t n, const ws_model_job* jobs, const uint32_t* tokens, ws_pred* out);
/* Forget one request's cached KV (its slots are reused by the next job naming it). */
int ws_model_evict(ws_ctx* ctx, uint32_t request);

/* Per-unit device time of the last ws_run_model_sim (CUDA events on each unit's stream): the
 * prompt-prefill phase (prefill_rows prompt tokens; target and draft forwards, no LM head), the
 * verify forwards (verify_rows fed, verify_out_rows through the LM head + K3/K4 — k+1 per
 * verify job) and the draft forwards (draft_rows fed, draft_out_rows = leaves + local drafts). */
typedef struct ws_run_stats {
  double verify_ms, draft_ms, prefill_target_ms, prefill_draft_ms;
  uint64_t verify_rows, verify_out_rows, verify_forwards;
  uint64_t draft_rows, draft_out_rows, draft_forwards;
  uint64_t prefill_rows, prefill_forwards;  /* target-side prefill forwards */
  /* attention work per unit: keys read (sum over groups of prefix + extras) and rows x keys */
  uint64_t verify_kv_pos, verify_attn_pairs, draft_kv_pos, draft_attn_pairs;
  uint64_t prefill_kv_pos, prefill_attn_pairs;
} ws_run_stats;
int ws_model_run_stats(ws_ctx* ctx, ws_run_stats* out);

/* single-model forward surface (tests): rows (token, position, KV slot), attention groups
 * {row0, n_rows, prefix_slot, prefix_len, extra_off, extra_len, masked} (7 int32 each) over
 * the slot pool — causal within a group, or (masked) row j sees the extras whose bits are set
 * in row_mask[row0 + j] — and the logits of out_rows → logits_out (device bf16 [n_out, V]). */
typedef struct ws_model ws_model;
int ws_model_create(const char* shape, uint64_t seed, int64_t n_slots, int max_rows, int device,
                    ws_model** out);
/* The same model split tensor-parallel over GPUs device .. device + tp - 1 (config 5's layout:
 * column-parallel QKV / gate-up, row-parallel O / down with the peer-memory all-reduce fused into
 * the residual update, vocabulary-parallel LM head); weights identical to the one-GPU model of
 * the same seed. Logits land on `device`. */
int ws_model_create_tp(const char* shape, uint64_t seed, int64_t n_slots, int max_rows, int device, int tp,
                       ws_model** out);
int ws_model_destroy(ws_model* m);
int ws_model_copy_weight(ws_model* m, const char* which, int layer, void* dst_dev, int64_t numel);
int ws_model_forward(ws_model* m, int n_rows, const int32_t* tok, const int32_t* pos,
                     const int32_t* slot, int n_groups, const int32_t* groups, int n_extra,
                     const int32_t* extra, const uint64_t* row_mask, int n_out,
                     const int32_t* out_rows, void* logits_out, void* stream);

/* ---- wire framing (wire.hpp:149-323, docs/protocol.md) ----
 * The reference's frame format for the protocol messages (big-endian u32 length, kind tag, then
 * the kind's fields), for a cross-host deployment; in-box, the wall-clock driver carries these
 * exact frames on its RTT queues. Speculations carry at most two candidates (the worker's top-2,
 * worker.hpp:121-125) and validations at most WS_WIRE_MAX_ACCEPTED accepted tokens. */
#define WS_MSG_HELLO 1
#define WS_MSG_SPECULATION 2
#define WS_MSG_VALIDATION 3
#define WS_MSG_EOS 4
#define WS_MSG_BYE 5
#define WS_WIRE_MAX_PATH 1024
#define WS_WIRE_MAX_ACCEPTED 255
#define WS_WIRE_NEED_MORE 1  /* ws_wire_decode: the frame is truncated */
typedef struct ws_wire_msg {
  uint32_t kind;                            /* WS_MSG_* */
  uint32_t n_path;                          /* speculation */
  uint64_t request_id, seq_no, base;
  uint64_t config_digest;                   /* hello */
  uint64_t final_length;                    /* eos */
  uint32_t n_cands;                         /* speculation: 1 or 2 */
  uint32_t cand_token[2];
  double cand_prob[2], cand_entropy[2];
  uint32_t n_accepted, bonus;               /* validation */
  double final_entropy;
  uint32_t path[WS_WIRE_MAX_PATH];
  uint32_t accepted[WS_WIRE_MAX_ACCEPTED];
  uint32_t pad;
} ws_wire_msg;
/* Encodes one frame into out[0, cap); *len = its size (WS_EARG when cap is too small). */
int ws_wire_encode(const ws_wire_msg* m, uint8_t* out, size_t cap, size_t* len);
/* Decodes the frame at the head of bytes[0, n) (decode_frame, wire.hpp:198-280): WS_OK with
 * *consumed = its size, WS_WIRE_NEED_MORE on truncation, WS_EPROTO on a malformed frame (bad tag,
 * length outside (0, 1 MiB], short or overlong payload; ws_last_error has the reason). */
int ws_wire_decode(const uint8_t* bytes, size_t n, ws_wire_msg* out, size_t* consumed);

/* ---- host-logic seam (tests / alternative model providers) ----
 * The batched driver with the model round supplied by the caller instead of the GPU: one
 * callback per round receives every pending verify job and draft row, exactly what the K9
 * kernel receives. Used by the CPU test-suite to check the host state machines against the
 * reference without a GPU; ws_run_sim never falls back to it. */
typedef int (*ws_model_round_fn)(void* user, uint32_t n_verify, const ws_verify_job* verify,
                                 const uint32_t* cands, uint32_t n_draft, const ws_draft_job* draft,
                                 ws_verify_out* verify_out, ws_pred* draft_out, int verify_mode,
                                 uint64_t sample_seed);
int ws_run_sim_with_model(const ws_sim_cfg* cfg, ws_model_round_fn fn, void* user, ws_run_out* out);

#ifdef __cplusplus
}
#endif
#endif /* WANSPEC_B200_H */
