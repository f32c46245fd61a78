/*
 * ORACLE — TEST INFRASTRUCTURE ONLY. Nothing under paper_2602_18931_b200/ may include,
 * link or call this; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs use it, and only as the checker.
 *
 * Plain-C restatement of the reference's hot-path arithmetic (arxiv 2602.18931,
 * /root/reference/proj/include/wanspec). Each function cites the file:line it follows.
 * Pinned against (a) the reference's own known-answer tests (tests/unit/test_oracle.cpp),
 * (b) the reference itself compiled into oracle/_ref/ (ref_shim.cpp), and (c) committed
 * golden fixtures in tests/golden/.
 *
 * The rejection-sampling verify (or_rejection_verify) and Philox are EXTENSIONS the
 * reference does not implement (SPEC.md:102 greedy only): parity for them is "unpinned"
 * by the reference — this restatement is the definition the GPU kernel is checked against.
 */
#ifndef WANSPEC_ORACLE_RESTATE_H
#define WANSPEC_ORACLE_RESTATE_H

#include <stddef.h>
#include <stdint.h>

#include "wanspec_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* std::mt19937_64 (fully specified by [rand.eng.mers]); rng.hpp:9-12 relies on it. */
typedef struct or_mt64 {
  uint64_t mt[312];
  int mti;
} or_mt64;

void or_mt64_seed(or_mt64* g, uint64_t seed);
uint64_t or_mt64_next(or_mt64* g);
double or_uniform_unit(or_mt64* g);                   /* rng.hpp:15-17 */
uint64_t or_uniform_below(or_mt64* g, uint64_t n);    /* rng.hpp:20-34 */
double or_exponential(or_mt64* g, double mean);       /* rng.hpp:37-41 */
int64_t or_uniform_jitter(or_mt64* g, int64_t spread);/* rng.hpp:44-48 */

/* OracleConfig::validate (oracle.hpp:49-60), stochastic kind. 0 or WS_ECONFIG. */
int or_oracle_validate(const ws_oracle_cfg* cfg);

/* Oracle::open + n_seq × next_sequence → synth_sequence (oracle.hpp:264-290, :313-345).
 * out: [n_seq * sequence_length]. */
int or_synth(const ws_oracle_cfg* cfg, uint32_t n_seq, ws_token_record* out);

/* entropy_of (oracle.hpp:21-33). Returns 0, or WS_EARG for negative / unnormalised input. */
int or_entropy_of(const double* p, size_t n, double* out);

/* run_target_step (oracle.hpp:127-139) over one sequence's records (len records; positions
 * >= len resolve to eos with entropy 0, oracle.hpp:88-102). */
void or_run_target_step(const ws_token_record* recs, uint32_t len, uint32_t eos, uint64_t base,
                        const uint32_t* cand, uint32_t k, uint32_t* acc_len, uint32_t* bonus,
                        double* final_entropy);

/* SequenceTrace::draft_prediction / target_prediction (oracle.hpp:92-98). */
void or_draft_prediction(const ws_token_record* recs, uint32_t len, uint32_t eos, uint64_t pos,
                         ws_pred* out);
void or_target_prediction(const ws_token_record* recs, uint32_t len, uint32_t eos,
                          uint64_t pos, ws_pred* out);

/* commit_tokens (oracle.hpp:356-363): appends until EOS. Returns new length. */
uint32_t or_commit_tokens(uint32_t* committed, uint32_t len, int* finished, const uint32_t* toks,
                          uint32_t n, uint32_t eos);

/* ---- extension: Philox4x32-10 rejection sampling (parity unpinned by the reference) ---- */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* 53-bit uniform in [0,1) from two words: ((hi<<32|lo) >> 11) * 2^-53. */
double or_unit_from_words(uint32_t hi, uint32_t lo);
/* Probability of token x under the completed distribution of a top-n prediction: listed ids
 * keep their prob; the remaining mass max(0,(1-p1)-p2) is spread uniformly over the V-n
 * unlisted ids. */
double or_completed_prob(const ws_pred* p, uint32_t vocab, uint32_t x);
/* Draw from max(0, Pt - Pd) (normalised; falls back to Pt when the residual is empty) by an
 * ascending-id inverse-CDF walk with uniform u. Pd may be NULL (sample from Pt). */
uint32_t or_sample_residual(const ws_pred* pt, const ws_pred* pd, uint32_t vocab, double u);
/* Speculative rejection verify: for i<k accept cand[i] iff u_i*pd < pt with
 * u_i = unit(philox(ctr=(req_lo, req_hi, step, i), key=(seed_lo, seed_hi)).w0,w1); on the
 * first reject the bonus is the residual draw with unit(w2,w3) of the same counter; after k
 * accepts the bonus is drawn from Pt(base+k) with counter i=k. final_entropy is the stored
 * target entropy at the bonus position (as run_target_step). */
void or_rejection_verify(const ws_token_record* recs, uint32_t len, uint32_t eos, uint32_t vocab,
                         uint64_t sample_seed, uint64_t request, uint32_t step, uint64_t base,
                         const uint32_t* cand, uint32_t k, uint32_t* acc_len, uint32_t* bonus,
                         double* final_entropy);

/* One batched model round over host tables (the CPU checker behind ws_run_sim_with_model):
 * verify jobs → run_target_step or or_rejection_verify; draft jobs → or_draft_prediction. */
void or_model_round(const ws_token_record* recs, uint32_t seq_len, uint32_t eos, uint32_t vocab,
                    uint32_t nv, const ws_verify_job* vj, const uint32_t* cands, uint32_t nd,
                    const ws_draft_job* dj, ws_verify_out* vo, ws_pred* dout, int mode,
                    uint64_t sample_seed);

/* FNV-1a 64 over the little-endian bytes of a u32 token stream (fingerprints). */
uint64_t or_fnv1a_tokens(uint64_t h, const uint32_t* toks, size_t n);

/* ---- K3 restatement: fp64 softmax statistics of one logits row ----
 * top-2 of softmax(x * inv_temp) (ties to the lower id) and entropy in nats. */
void or_row_stats(const float* logits, uint32_t vocab, double inv_temp, ws_pred* out);
/* K4R restated (kernels/sample.cuh): rejection sampling over k+1 float rows (the bf16 logits of
 * one request's verify rows, row stride ld) — extension, parity unpinned by the reference. */
void or_model_rejection_verify(const float* rows, uint32_t k, uint32_t vocab, uint32_t ld, float inv_temp,
                               float top_p, const uint32_t* cand, const double* cand_prob, uint64_t seed,
                               uint64_t request, uint32_t step, const int32_t* forced, uint32_t* acc_len,
                               uint32_t* bonus, double* final_entropy);

#ifdef __cplusplus
}
#endif
#endif
