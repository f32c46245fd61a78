// Wire framing of the protocol messages (wire.hpp:149-323 of the reference; docs/protocol.md):
// big-endian u32 payload length, then kind tag u8, request_id u64, seq_no u64 (not for Bye), and
// the kind's fields — Hello: config digest u64; Speculation: base u64, path u16 + u32 each,
// candidates u8 + (u32 token, f64 prob, f64 entropy); Validation: base u64, accepted u8 + u32
// each, bonus u32, final entropy f64; Eos: final length u64. Payloads are capped at 1 MiB.
// decode_frame is strict (truncation -> need_more; bad tag, bad length, short or overlong
// payload -> error), FrameReader enforces the per-request FIFO seq contract.
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "common.hpp"

namespace wsb {

constexpr std::size_t kMaxFramePayload = 1u << 20;

void wire_encode(const Message& m, std::vector<std::uint8_t>& out);  // appends one frame

enum class DecodeStatus { ok, need_more, error };
struct Decoded {
  DecodeStatus status = DecodeStatus::error;
  std::size_t consumed = 0;
  Message message;
  std::string error;
};
Decoded wire_decode_frame(const std::uint8_t* bytes, std::size_t n);
Decoded wire_decode(const std::uint8_t* bytes, std::size_t n);  // exactly one frame

class FrameReader {
 public:
  void feed(const std::uint8_t* bytes, std::size_t n) { buf_.insert(buf_.end(), bytes, bytes + n); }
  // next complete message (false: need more bytes); throws ProtocolError on a bad frame or a
  // seq gap within a request's stream
  bool next(Message& out);

 private:
  std::vector<std::uint8_t> buf_;
  std::size_t head_ = 0;
  std::map<std::uint64_t, std::uint64_t> last_seq_;
};

}  // namespace wsb
