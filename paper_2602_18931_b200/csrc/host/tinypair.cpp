// The tiny draft/target pair (BASELINE configs 1-2): per-position TokenRecords synthesized
// from one std::mt19937_64 stream in the reference's draw order (oracle.hpp:313-345, draw-order
// contract :320), dealt to requests in order (oracle.hpp:282-290). These records are the
// "weights" of the tiny pair; they are generated on the host (libm-identical log/exp and the
// sequential engine) and uploaded once as device tables for K9.
#include "tinypair.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>

namespace wsb {

namespace {

double uniform_unit(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }  // rng.hpp:15

std::uint64_t uniform_below(std::mt19937_64& g, std::uint64_t n) {  // rng.hpp:20-34
  std::uint64_t x = g();
  unsigned __int128 m = static_cast<unsigned __int128>(x) * n;
  auto lo = static_cast<std::uint64_t>(m);
  if (lo < n) {
    const std::uint64_t threshold = (0 - n) % n;
    while (lo < threshold) {
      x = g();
      m = static_cast<unsigned __int128>(x) * n;
      lo = static_cast<std::uint64_t>(m);
    }
  }
  return static_cast<std::uint64_t>(m >> 64);
}

double exponential(std::mt19937_64& g, double mean) {  // rng.hpp:37-41
  const double u = uniform_unit(g);
  const double v = -mean * std::log(1.0 - u);
  return v > 1e-12 ? v : 1e-12;
}

// oracle.hpp:295-303
TokenId draw_excluding(std::mt19937_64& g, std::uint32_t vocab, TokenId a) {
  TokenId t = static_cast<TokenId>(uniform_below(g, vocab - 1u));
  if (t >= a) ++t;
  return t;
}
TokenId draw_excluding(std::mt19937_64& g, std::uint32_t vocab, TokenId a, TokenId b) {
  const TokenId lo = std::min(a, b), hi = std::max(a, b);
  TokenId t = static_cast<TokenId>(uniform_below(g, vocab - 2u));
  if (t >= lo) ++t;
  if (t >= hi) ++t;
  return t;
}

// oracle.hpp:305-311
void fill_probs(double entropy, double& p1, double& p2) {
  p1 = std::clamp(std::exp(-entropy), 0.05, 0.99);
  p2 = std::min(0.9 * p1, 0.5 * (1.0 - p1));
}

}  // namespace

// oracle.hpp:49-60 (stochastic kind)
void validate_oracle(const ws_oracle_cfg& c) {
  if (c.vocab_size < 2) throw ConfigError("oracle: vocab_size must be >= 2");
  if (c.eos_id >= c.vocab_size) throw ConfigError("oracle: eos_id must be < vocab_size");
  if (c.match_prob < 0.0 || c.match_prob > 1.0) throw ConfigError("oracle: match_prob must be in [0,1]");
  if (c.second_correct_prob < 0.0 || c.second_correct_prob > 1.0)
    throw ConfigError("oracle: second_correct_prob must be in [0,1]");
  if (c.entropy_low <= 0.0 || c.entropy_high <= 0.0) throw ConfigError("oracle: entropy means must be > 0");
  if (c.sequence_length < 1) throw ConfigError("oracle: sequence_length must be >= 1");
}

void synth_tiny_pair(const ws_oracle_cfg& c, std::uint32_t n_seq, ws_token_record* out) {
  validate_oracle(c);
  std::mt19937_64 g(c.seed);
  const std::uint32_t L = c.sequence_length, V = c.vocab_size;
  const TokenId eos = c.eos_id;
  for (std::uint32_t s = 0; s < n_seq; ++s) {
    for (std::uint32_t pos = 0; pos < L; ++pos) {
      ws_token_record& r = out[static_cast<std::size_t>(s) * L + pos];
      std::memset(&r, 0, sizeof(r));
      const bool last = pos + 1 == L;
      const bool match = uniform_unit(g) < c.match_prob;
      r.target_token = last ? eos : draw_excluding(g, V, eos);
      const double th = exponential(g, match ? c.entropy_low : c.entropy_high);
      const double dh = exponential(g, match ? c.entropy_low : c.entropy_high);
      TokenId d1, d2;
      if (match) {
        d1 = r.target_token;
        d2 = draw_excluding(g, V, d1);
      } else {
        d1 = draw_excluding(g, V, r.target_token);
        const bool second_correct = uniform_unit(g) < c.second_correct_prob;
        d2 = second_correct ? r.target_token : draw_excluding(g, V, r.target_token, d1);
      }
      r.target_top2 = draw_excluding(g, V, r.target_token);
      r.target_entropy = th;
      fill_probs(th, r.target_p1, r.target_p2);
      r.draft_top1 = d1;
      r.draft_top2 = d2;
      r.draft_entropy = dh;
      fill_probs(dh, r.draft_p1, r.draft_p2);
    }
  }
}

}  // namespace wsb
