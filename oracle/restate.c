/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see restate.h). Plain-C restatement of the reference's
 * hot-path arithmetic; compiled with -ffp-contract=off so every double op rounds like the
 * reference's (and like the GPU kernels, which use explicit _rn intrinsics).
 */
#include "restate.h"

#include <math.h>
#include <string.h>

/* ---------------- std::mt19937_64 ---------------- */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void or_mt64_seed(or_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = MT_N;
}

uint64_t or_mt64_next(or_mt64* g) {
  if (g->mti >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t y = (g->mt[i] & MT_UPPER) | (g->mt[(i + 1) % MT_N] & MT_LOWER);
      g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
    }
    g->mti = 0;
  }
  uint64_t x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* rng.hpp:15-17 */
double or_uniform_unit(or_mt64* g) { return (double)(or_mt64_next(g) >> 11) * 0x1.0p-53; }

/* rng.hpp:20-34 — Lemire multiply-shift with rejection of the biased zone. */
uint64_t or_uniform_below(or_mt64* g, uint64_t n) {
  uint64_t x = or_mt64_next(g);
  unsigned __int128 m = (unsigned __int128)x * n;
  uint64_t lo = (uint64_t)m;
  if (lo < n) {
    uint64_t threshold = (0 - n) % n;
    while (lo < threshold) {
      x = or_mt64_next(g);
      m = (unsigned __int128)x * n;
      lo = (uint64_t)m;
    }
  }
  return (uint64_t)(m >> 64);
}

/* rng.hpp:37-41 */
double or_exponential(or_mt64* g, double mean) {
  double u = or_uniform_unit(g);
  double v = -mean * log(1.0 - u);
  return v > 1e-12 ? v : 1e-12;
}

/* rng.hpp:44-48 */
int64_t or_uniform_jitter(or_mt64* g, int64_t spread) {
  if (spread <= 0) return 0;
  uint64_t span = (uint64_t)(2 * spread + 1);
  return (int64_t)or_uniform_below(g, span) - spread;
}

/* ---------------- the tiny pair ---------------- */
/* oracle.hpp:49-60 */
int or_oracle_validate(const ws_oracle_cfg* c) {
  if (!c) return WS_EARG;
  if (c->vocab_size < 2) return WS_ECONFIG;
  if (c->eos_id >= c->vocab_size) return WS_ECONFIG;
  if (!(c->match_prob >= 0.0 && c->match_prob <= 1.0)) return WS_ECONFIG;
  if (!(c->second_correct_prob >= 0.0 && c->second_correct_prob <= 1.0)) return WS_ECONFIG;
  if (c->entropy_low <= 0.0 || c->entropy_high <= 0.0) return WS_ECONFIG;
  if (c->sequence_length < 1) return WS_ECONFIG;
  return WS_OK;
}

/* oracle.hpp:295-303 — uniform over V minus the excluded ids, skipping them in sorted order. */
static uint32_t draw_excluding(or_mt64* g, uint32_t vocab, const uint32_t* ex, int n_ex) {
  uint32_t s[2];
  for (int i = 0; i < n_ex; ++i) s[i] = ex[i];
  if (n_ex == 2 && s[1] < s[0]) {
    uint32_t t = s[0];
    s[0] = s[1];
    s[1] = t;
  }
  uint32_t t = (uint32_t)or_uniform_below(g, (uint64_t)(vocab - (uint32_t)n_ex));
  for (int i = 0; i < n_ex; ++i)
    if (t >= s[i]) ++t;
  return t;
}

/* oracle.hpp:305-311 */
static void fill_probs(double entropy, double* p1, double* p2) {
  double e = exp(-entropy);
  double a = e < 0.05 ? 0.05 : (e > 0.99 ? 0.99 : e);
  double b1 = 0.9 * a, b2 = 0.5 * (1.0 - a);
  *p1 = a;
  *p2 = b1 < b2 ? b1 : b2;
}

/* oracle.hpp:313-345 — the draw order (:320) is the replay contract. */
int or_synth(const ws_oracle_cfg* c, uint32_t n_seq, ws_token_record* out) {
  int rc = or_oracle_validate(c);
  if (rc) return rc;
  or_mt64 g;
  or_mt64_seed(&g, c->seed);
  const uint32_t L = c->sequence_length, V = c->vocab_size, eos = c->eos_id;
  for (uint32_t s = 0; s < n_seq; ++s) {
    for (uint32_t pos = 0; pos < L; ++pos) {
      ws_token_record* r = &out[(size_t)s * L + pos];
      memset(r, 0, sizeof(*r));
      int last = pos + 1 == L;
      int match = or_uniform_unit(&g) < c->match_prob;
      uint32_t ex1[1] = {eos};
      r->target_token = last ? eos : draw_excluding(&g, V, ex1, 1);
      double th = or_exponential(&g, match ? c->entropy_low : c->entropy_high);
      double dh = or_exponential(&g, match ? c->entropy_low : c->entropy_high);
      uint32_t d1, d2;
      if (match) {
        d1 = r->target_token;
        uint32_t e[1] = {d1};
        d2 = draw_excluding(&g, V, e, 1);
      } else {
        uint32_t e[1] = {r->target_token};
        d1 = draw_excluding(&g, V, e, 1);
        int second_correct = or_uniform_unit(&g) < c->second_correct_prob;
        if (second_correct) {
          d2 = r->target_token;
        } else {
          uint32_t e2[2] = {r->target_token, d1};
          d2 = draw_excluding(&g, V, e2, 2);
        }
      }
      uint32_t et[1] = {r->target_token};
      r->target_top2 = draw_excluding(&g, V, et, 1);
      r->target_entropy = th;
      fill_probs(th, &r->target_p1, &r->target_p2);
      r->draft_top1 = d1;
      r->draft_top2 = d2;
      r->draft_entropy = dh;
      fill_probs(dh, &r->draft_p1, &r->draft_p2);
    }
  }
  return WS_OK;
}

/* oracle.hpp:21-33 */
int or_entropy_of(const double* p, size_t n, double* out) {
  double sum = 0.0;
  for (size_t i = 0; i < n; ++i) {
    if (p[i] < 0.0) return WS_EARG;
    sum += p[i];
  }
  if (fabs(sum - 1.0) > 1e-9) return WS_EARG;
  double h = 0.0;
  for (size_t i = 0; i < n; ++i)
    if (p[i] > 0.0) h -= p[i] * log(p[i]);
  *out = h < 0.0 ? 0.0 : h;
  return WS_OK;
}

/* oracle.hpp:88-90 */
static uint32_t target_token(const ws_token_record* r, uint32_t len, uint32_t eos, uint64_t pos) {
  return pos < len ? r[pos].target_token : eos;
}
/* oracle.hpp:100-102 */
static double target_entropy(const ws_token_record* r, uint32_t len, uint64_t pos) {
  return pos < len ? r[pos].target_entropy : 0.0;
}

/* oracle.hpp:127-139 */
void or_run_target_step(const ws_token_record* recs, uint32_t len, uint32_t eos, uint64_t base,
                        const uint32_t* cand, uint32_t k, uint32_t* acc_len, uint32_t* bonus,
                        double* final_entropy) {
  uint64_t pos = base;
  uint32_t a = 0;
  for (uint32_t i = 0; i < k; ++i) {
    if (cand[i] != target_token(recs, len, eos, pos)) break;
    ++a;
    ++pos;
  }
  *acc_len = a;
  *bonus = target_token(recs, len, eos, pos);
  *final_entropy = target_entropy(recs, len, pos);
}

/* oracle.hpp:96-98 with the past-end EOS prediction of :118 */
void or_draft_prediction(const ws_token_record* recs, uint32_t len, uint32_t eos, uint64_t pos,
                         ws_pred* out) {
  memset(out, 0, sizeof(*out));
  if (pos < len) {
    const ws_token_record* r = &recs[pos];
    out->n = 2;
    out->id[0] = r->draft_top1;
    out->id[1] = r->draft_top2;
    out->prob[0] = r->draft_p1;
    out->prob[1] = r->draft_p2;
    out->entropy = r->draft_entropy;
  } else {
    out->n = 1;
    out->id[0] = eos;
    out->prob[0] = 1.0;
  }
}

/* oracle.hpp:92-94 */
void or_target_prediction(const ws_token_record* recs, uint32_t len, uint32_t eos,
                          uint64_t pos, ws_pred* out) {
  memset(out, 0, sizeof(*out));
  if (pos < len) {
    const ws_token_record* r = &recs[pos];
    out->n = 2;
    out->id[0] = r->target_token;
    out->id[1] = r->target_top2;
    out->prob[0] = r->target_p1;
    out->prob[1] = r->target_p2;
    out->entropy = r->target_entropy;
  } else {
    out->n = 1;
    out->id[0] = eos;
    out->prob[0] = 1.0;
  }
}

/* oracle.hpp:356-363 */
uint32_t or_commit_tokens(uint32_t* committed, uint32_t len, int* finished, const uint32_t* toks,
                          uint32_t n, uint32_t eos) {
  for (uint32_t i = 0; i < n; ++i) {
    if (*finished) return len;
    committed[len++] = toks[i];
    if (toks[i] == eos) *finished = 1;
  }
  return len;
}

/* ---------------- extension: Philox4x32-10 rejection sampling ---------------- */
/* Salmon et al., "Parallel random numbers: as easy as 1, 2, 3" (SC'11), Philox4x32 with
 * 10 rounds; multipliers 0xD2511F53 / 0xCD9E8D57, Weyl key increments 0x9E3779B9 /
 * 0xBB67AE85. */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

double or_unit_from_words(uint32_t hi, uint32_t lo) {
  uint64_t x = ((uint64_t)hi << 32) | lo;
  return (double)(x >> 11) * 0x1.0p-53;
}

static double tail_per_token(const ws_pred* p, uint32_t vocab) {
  double t = 1.0;
  for (uint32_t j = 0; j < p->n; ++j) t = t - p->prob[j];
  if (t < 0.0) t = 0.0;
  if (vocab <= p->n) return 0.0;
  return t / (double)(vocab - p->n);
}

double or_completed_prob(const ws_pred* p, uint32_t vocab, uint32_t x) {
  for (uint32_t j = 0; j < p->n; ++j)
    if (p->id[j] == x) return p->prob[j];
  return tail_per_token(p, vocab);
}

/* Inverse-CDF walk in ascending id order over: runs of unlisted ids (mass rho each) and the
 * listed ids s[0..ns) (mass m[j]). Returns the drawn id. */
static uint32_t walk_sample(const uint32_t* s, const double* m, int ns, double rho,
                            uint32_t vocab, double u) {
  /* total mass, accumulated in the same order as the walk */
  double z = 0.0;
  uint32_t prev = 0;
  for (int j = 0; j < ns; ++j) {
    z = z + (double)(s[j] - prev) * rho;
    z = z + m[j];
    prev = s[j] + 1;
  }
  z = z + (double)(vocab - prev) * rho;
  double target = u * z;
  double acc = 0.0;
  prev = 0;
  uint32_t last_pos = 0;
  int have_last = 0;
  for (int j = 0; j <= ns; ++j) {
    uint32_t end = j < ns ? s[j] : vocab;
    uint32_t run = end - prev;
    if (run > 0 && rho > 0.0) {
      double seg = (double)run * rho;
      if (acc + seg > target) {
        double off = floor((target - acc) / rho);
        uint32_t o = off < 0.0 ? 0u : (off >= (double)run ? run - 1 : (uint32_t)off);
        return prev + o;
      }
      acc = acc + seg;
      last_pos = end - 1;
      have_last = 1;
    }
    if (j < ns) {
      if (m[j] > 0.0) {
        if (acc + m[j] > target) return s[j];
        acc = acc + m[j];
        last_pos = s[j];
        have_last = 1;
      }
      prev = s[j] + 1;
    }
  }
  return have_last ? last_pos : 0u;
}

uint32_t or_sample_residual(const ws_pred* pt, const ws_pred* pd, uint32_t vocab, double u) {
  uint32_t s[4];
  int ns = 0;
  const ws_pred* ps[2] = {pt, pd};
  for (int w = 0; w < 2; ++w) {
    if (!ps[w]) continue;
    for (uint32_t j = 0; j < ps[w]->n; ++j) {
      uint32_t id = ps[w]->id[j];
      int dup = 0;
      for (int q = 0; q < ns; ++q) dup |= s[q] == id;
      if (!dup) s[ns++] = id;
    }
  }
  /* insertion sort ascending */
  for (int i = 1; i < ns; ++i)
    for (int j = i; j > 0 && s[j - 1] > s[j]; --j) {
      uint32_t t = s[j];
      s[j] = s[j - 1];
      s[j - 1] = t;
    }
  double m[4];
  double rho;
  double tt = tail_per_token(pt, vocab);
  if (pd) {
    double td = tail_per_token(pd, vocab);
    double zr = 0.0;
    for (int j = 0; j < ns; ++j) {
      double d = or_completed_prob(pt, vocab, s[j]) - or_completed_prob(pd, vocab, s[j]);
      m[j] = d > 0.0 ? d : 0.0;
      zr = zr + m[j];
    }
    double dr = tt - td;
    rho = dr > 0.0 ? dr : 0.0;
    if (zr > 0.0 || (rho > 0.0 && (uint32_t)ns < vocab))
      return walk_sample(s, m, ns, rho, vocab, u);
  }
  for (int j = 0; j < ns; ++j) m[j] = or_completed_prob(pt, vocab, s[j]);
  return walk_sample(s, m, ns, tt, vocab, u);
}

void or_rejection_verify(const ws_token_record* recs, uint32_t len, uint32_t eos, uint32_t vocab,
                         uint64_t sample_seed, uint64_t request, uint32_t step, uint64_t base,
                         const uint32_t* cand, uint32_t k, uint32_t* acc_len, uint32_t* bonus,
                         double* final_entropy) {
  const uint32_t key[2] = {(uint32_t)sample_seed, (uint32_t)(sample_seed >> 32)};
  for (uint32_t i = 0; i <= k; ++i) {
    uint64_t q = base + i;
    ws_pred pt;
    or_target_prediction(recs, len, eos, q, &pt);
    const uint32_t ctr[4] = {(uint32_t)request, (uint32_t)(request >> 32), step, i};
    uint32_t w[4];
    or_philox4x32_10(ctr, key, w);
    if (i == k) {
      *acc_len = k;
      *bonus = or_sample_residual(&pt, NULL, vocab, or_unit_from_words(w[2], w[3]));
      *final_entropy = target_entropy(recs, len, q);
      return;
    }
    ws_pred pd;
    or_draft_prediction(recs, len, eos, q, &pd);
    double p_t = or_completed_prob(&pt, vocab, cand[i]);
    double p_d = or_completed_prob(&pd, vocab, cand[i]);
    double u = or_unit_from_words(w[0], w[1]);
    if (u * p_d < p_t) continue;
    *acc_len = i;
    *bonus = or_sample_residual(&pt, &pd, vocab, or_unit_from_words(w[2], w[3]));
    *final_entropy = target_entropy(recs, len, q);
    return;
  }
}

void or_model_round(const ws_token_record* recs, uint32_t seq_len, uint32_t eos, uint32_t vocab,
                    uint32_t nv, const ws_verify_job* vj, const uint32_t* cands, uint32_t nd,
                    const ws_draft_job* dj, ws_verify_out* vo, ws_pred* dout, int mode,
                    uint64_t sample_seed) {
  for (uint32_t j = 0; j < nv; ++j) {
    const ws_token_record* r = recs + (size_t)vj[j].seq * seq_len;
    const uint32_t* c = cands + vj[j].cand_off;
    if (mode == WS_VERIFY_REJECTION)
      or_rejection_verify(r, seq_len, eos, vocab, sample_seed, vj[j].request, vj[j].step, vj[j].base, c,
                          vj[j].k, &vo[j].accepted, &vo[j].bonus, &vo[j].final_entropy);
    else
      or_run_target_step(r, seq_len, eos, vj[j].base, c, vj[j].k, &vo[j].accepted, &vo[j].bonus,
                         &vo[j].final_entropy);
  }
  for (uint32_t j = 0; j < nd; ++j)
    or_draft_prediction(recs + (size_t)dj[j].seq * seq_len, seq_len, eos, dj[j].pos, &dout[j]);
}

uint64_t or_fnv1a_tokens(uint64_t h, const uint32_t* toks, size_t n) {
  for (size_t i = 0; i < n; ++i)
    for (int b = 0; b < 4; ++b) {
      h ^= (toks[i] >> (8 * b)) & 0xFFu;
      h *= 0x100000001B3ULL;
    }
  return h;
}

/* K3 restatement in fp64: softmax(x*it) top-2 (ties → lower id) and H = ln Z - S/Z with
 * m = max, Z = sum e^{l-m}, S = sum e^{l-m} (l-m). */
void or_row_stats(const float* x, uint32_t vocab, double it, ws_pred* out) {
  memset(out, 0, sizeof(*out));
  double m = -INFINITY;
  uint32_t i1 = 0, i2 = 0;
  double v1 = -INFINITY, v2 = -INFINITY;
  for (uint32_t v = 0; v < vocab; ++v) {
    double l = (double)x[v] * it;
    if (l > v1) {
      v2 = v1;
      i2 = i1;
      v1 = l;
      i1 = v;
    } else if (l > v2) {
      v2 = l;
      i2 = v;
    }
  }
  m = v1;
  double z = 0.0, s = 0.0;
  for (uint32_t v = 0; v < vocab; ++v) {
    double d = (double)x[v] * it - m;
    double e = exp(d);
    z += e;
    if (e > 0.0) s += e * d; /* entropy_of's 0 ln 0 = 0 (oracle.hpp:21-33): -inf logits add nothing */
  }
  out->n = vocab >= 2 ? 2 : 1;
  out->id[0] = i1;
  out->id[1] = i2;
  out->prob[0] = exp(v1 - m) / z;
  out->prob[1] = vocab >= 2 ? exp(v2 - m) / z : 0.0;
  double h = log(z) - s / z;
  out->entropy = h < 0.0 ? 0.0 : h;
}

/* ---------------- extension: K4R rejection sampling over real-model rows ---------------- */
/* Restates paper_2602_18931_b200/csrc/kernels/sample.cuh (the rule) step for step: the same
 * fp64 operations in the same order — per-chunk sequential sums over ceil(V/512)-id chunks, a
 * fixed pairwise tree over the 512 partials, a sequential prefix over the chunks for the
 * inverse CDF. Parity is unpinned by the reference (greedy only); this is the
 * checker. Only exp() may differ by an ulp between glibc and libdevice. */
#define OR_T 512

typedef struct {
  const float* x;
  uint32_t V;
  double tau, zmax, Z, S, M;
  int32_t forced;
  uint32_t t_star;
} or_row;

static uint32_t or_key16(float x) {
  uint32_t b;
  memcpy(&b, &x, 4);
  b >>= 16;
  return (b & 0x8000u) ? (~b & 0xFFFFu) : (b | 0x8000u);
}

static double or_tree(double* s) {
  for (int st = OR_T / 2; st > 0; st >>= 1)
    for (int i = 0; i < st; ++i) s[i] = s[i] + s[i + st];
  return s[0];
}

static void or_chunk(uint32_t V, int t, uint32_t* lo, uint32_t* hi) {
  uint32_t C = (V + OR_T - 1) / OR_T;
  uint64_t l = (uint64_t)t * C;
  *lo = l > V ? V : (uint32_t)l;
  *hi = *lo + C > V ? V : *lo + C;
}

static double or_z(const or_row* r, uint32_t i) { return (double)r->x[i] * r->tau; }

static double or_pprime(const or_row* r, uint32_t i) {
  if (r->forced >= 0) return (uint32_t)r->forced == i ? 1.0 : 0.0;
  if (or_key16(r->x[i]) < r->t_star) return 0.0;
  double p = exp(or_z(r, i) - r->zmax) / r->Z;
  return r->M == 1.0 ? p : p / r->M;
}

static void or_row_dist(or_row* r, float top_p) {
  r->t_star = 0;
  r->M = 1.0;
  if (r->forced >= 0) {
    r->Z = 1.0;
    r->S = 0.0;
    r->zmax = 0.0;
    return;
  }
  float mx = -INFINITY;
  for (uint32_t i = 0; i < r->V; ++i) mx = r->x[i] > mx ? r->x[i] : mx;
  r->zmax = (double)mx * r->tau;
  double pz[OR_T], ps[OR_T];
  for (int t = 0; t < OR_T; ++t) {
    uint32_t lo, hi;
    or_chunk(r->V, t, &lo, &hi);
    double z = 0.0, sv = 0.0;
    for (uint32_t i = lo; i < hi; ++i) {
      double d = or_z(r, i) - r->zmax;
      double e = exp(d);
      z = z + e;
      if (e > 0.0) sv = sv + e * d;
    }
    pz[t] = z;
    ps[t] = sv;
  }
  r->Z = or_tree(pz);
  r->S = or_tree(ps);
  if (top_p < 1.f) {
    double tp = (double)top_p;
    uint32_t lo = 0, hi = 65536;
    double m_lo = 1.0;
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) / 2;
      double part[OR_T];
      for (int t = 0; t < OR_T; ++t) {
        uint32_t a, b;
        or_chunk(r->V, t, &a, &b);
        double s = 0.0;
        for (uint32_t i = a; i < b; ++i)
          if (or_key16(r->x[i]) >= mid) s = s + exp(or_z(r, i) - r->zmax);
        part[t] = s;
      }
      double mass = or_tree(part) / r->Z;
      if (mass >= tp) {
        lo = mid;
        m_lo = mass;
      } else {
        hi = mid;
      }
    }
    r->t_star = lo;
    r->M = m_lo;
  }
}

static double or_w(const or_row* r, int resid, uint32_t c, double q, double tail, uint32_t i) {
  double p = or_pprime(r, i);
  if (!resid) return p;
  double d = p - (i == c ? q : tail);
  return d > 0.0 ? d : 0.0;
}

static uint32_t or_sample_row(const or_row* r, int has_d, uint32_t c, double q, double u) {
  uint32_t V = r->V;
  double tail = V > 1 ? (1.0 - q) / (double)(V - 1) : 0.0;
  for (int pass = 0; pass < 2; ++pass) {
    int resid = has_d && pass == 0;
    double part[OR_T], start[OR_T];
    for (int t = 0; t < OR_T; ++t) {
      uint32_t a, b;
      or_chunk(V, t, &a, &b);
      double s = 0.0;
      for (uint32_t i = a; i < b; ++i) s = s + or_w(r, resid, c, q, tail, i);
      part[t] = s;
    }
    double acc = 0.0;
    for (int t = 0; t < OR_T; ++t) {
      start[t] = acc;
      acc = acc + part[t];
    }
    double R = acc;
    if (resid && !(R > 0.0)) continue;
    double target = u * R;
    uint32_t pick = 0xFFFFFFFFu, lastpos = 0;
    for (int t = 0; t < OR_T; ++t) {
      if (!(part[t] > 0.0)) continue;
      uint32_t a, b;
      or_chunk(V, t, &a, &b);
      if (pick == 0xFFFFFFFFu && target >= start[t] && target < start[t] + part[t]) {
        double w_acc = start[t];
        for (uint32_t i = a; i < b; ++i) {
          double v = or_w(r, resid, c, q, tail, i);
          if (v > 0.0) {
            double nx = w_acc + v;
            if (nx > target) {
              pick = i;
              break;
            }
            w_acc = nx;
          }
        }
      }
      for (uint32_t i = a; i < b; ++i)
        if (or_w(r, resid, c, q, tail, i) > 0.0 && i > lastpos) lastpos = i;
    }
    return pick != 0xFFFFFFFFu ? pick : lastpos;
  }
  return 0;
}

void or_model_rejection_verify(const float* rows, uint32_t k, uint32_t vocab, uint32_t ld, float inv_temp,
                               float top_p, const uint32_t* cand, const double* cand_prob, uint64_t seed,
                               uint64_t request, uint32_t step, const int32_t* forced, uint32_t* acc_len,
                               uint32_t* bonus, double* final_entropy) {
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  or_row r;
  r.V = vocab;
  r.tau = (double)inv_temp;
  for (uint32_t i = 0; i <= k; ++i) {
    r.x = rows + (size_t)i * ld;
    r.forced = forced ? forced[i] : -1;
    or_row_dist(&r, top_p);
    const uint32_t ctr[4] = {(uint32_t)request, (uint32_t)(request >> 32), step, i};
    uint32_t w[4];
    or_philox4x32_10(ctr, key, w);
    double u2 = or_unit_from_words(w[2], w[3]);
    int reject = 0;
    uint32_t c = 0;
    double q = 0.0;
    if (i < k) {
      c = cand[i];
      q = cand_prob[i];
      q = q < 0.0 ? 0.0 : (q > 1.0 ? 1.0 : q);
      double u = or_unit_from_words(w[0], w[1]);
      reject = !(u * q < or_pprime(&r, c));
    }
    if (i == k || reject) {
      *acc_len = i;
      *bonus = or_sample_row(&r, reject, c, q, u2);
      if (r.forced >= 0) {
        *final_entropy = 0.0;
      } else {
        double h = log(r.Z) - r.S / r.Z;
        *final_entropy = h < 0.0 ? 0.0 : h;
      }
      return;
    }
  }
}
