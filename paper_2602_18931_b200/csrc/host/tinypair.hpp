#pragma once

#include "common.hpp"
#include "wanspec_b200.h"

#include <cstdint>

namespace wsb {

// OracleConfig::validate (oracle.hpp:49-60); throws ConfigError.
void validate_oracle(const ws_oracle_cfg& c);

// Oracle::open + n_seq × synth_sequence (oracle.hpp:264-290, :313-345).
void synth_tiny_pair(const ws_oracle_cfg& c, std::uint32_t n_seq, ws_token_record* out);

}  // namespace wsb
