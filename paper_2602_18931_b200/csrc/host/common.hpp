// Host-side vocabulary of the B200 WANSpec hot path. New code: the names follow the
// reference's domain (types.hpp, spectree.hpp, wire.hpp) so parity reviews line up, but the
// layouts are flat and allocation-light for the batched multi-request driver.
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace wsb {

using TokenId = std::uint32_t;  // types.hpp:14
using SimTime = std::int64_t;   // types.hpp:18 (µs)
using NodeId = std::uint32_t;   // spectree.hpp:18
constexpr NodeId kRootId = 0;   // spectree.hpp:19
constexpr SimTime kInfiniteTime = std::numeric_limits<SimTime>::max();  // types.hpp:20

// types.hpp:30-33
inline SimTime sat_add(SimTime a, SimTime b) {
  if (a > 0 && b > kInfiniteTime - a) return kInfiniteTime;
  return a + b;
}

// Error classes (types.hpp:35-45), mapped to WS_E* codes at the C ABI.
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ProtocolError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// A model output reduced to the protocol's needs (types.hpp:56-63): n ∈ {1,2} candidates,
// descending probability, ties by ascending id; entropy in nats.
struct Pred {
  std::uint32_t n = 0;
  TokenId id[2] = {0, 0};
  double prob[2] = {0.0, 0.0};
  double entropy = 0.0;
};

// spectree.hpp:52-58
struct CandIn {
  TokenId token = 0;
  double prob = 0.0;
  double entropy = 0.0;
};

// spectree.hpp:37-45
struct Validation {
  std::vector<TokenId> accepted;
  TokenId bonus = 0;
  double final_entropy = 0.0;
  std::size_t length() const { return accepted.size() + 1; }
};

enum class Origin : std::uint8_t { worker, controller };  // spectree.hpp:21

// Message vocabulary (wire.hpp:24-83). In-box the WAN is an injected RTT on host queues,
// so messages stay as structs (no framing); one flat struct per message, kind-tagged.
enum class MsgKind : std::uint8_t { hello = 1, speculation = 2, validation = 3, eos = 4, bye = 5 };

struct Message {
  std::uint64_t request_id = 0;
  std::uint64_t seq_no = 0;
  MsgKind kind = MsgKind::hello;
  std::uint64_t base = 0;          // speculation / validation
  std::vector<TokenId> path;       // speculation: anchor path below base
  CandIn cands[2];                 // speculation: 1 or 2 candidates
  std::uint32_t n_cands = 0;
  Validation result;               // validation
  std::uint64_t final_length = 0;  // eos
  std::uint64_t config_digest = 0; // hello (wire.hpp:32-34)
};

}  // namespace wsb
