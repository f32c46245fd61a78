// Wall-clock driver (the reference's networked runtime, runtime.hpp:153-386, brought in-box):
// every request runs its controller and worker state machines on the host against real time;
// each model step is launched on the GPU lanes when the state machine asks for it and completes
// when its CUDA work completes (not after a virtual t_target / t_draft); proposals and
// validations cross per-request host queues whose frames become visible one_way = rtt/2 (+/-
// uniform jitter) after they are sent, never out of order — the LatencyEmulator's
// visible_at = max(sent + delay, last_visible) (net.hpp:149-163); every message travels as its
// wire frame (host/wire.hpp, the reference's encoding) through a FrameReader that enforces the
// per-request FIFO seq contract (wire.hpp:296-323). Requests run concurrently and
// share the GPU lanes (continuous batching); each one's protocol is the reference's.
//
// Optional decision log (the reference's DecisionLog, runtime.hpp:227-237, extended with the
// model results a real model cannot recompute): one NDJSON line per controller turn — its
// clock, the frames folded in, the target / local-draft completions with their results, the
// steps it launched and t_update after the turn — so a fresh state machine (the reference's
// own, oracle/ref_shim.cpp ref_replay_model_log) can replay the run and must reproduce every
// launch decision, the t_update trace and the committed streams (runtime.hpp:404-454).
#pragma once

#include <cstdint>
#include <string>

#include "driver.hpp"

namespace wsb {

struct WallclockStats {
  double wall_ms = 0.0;
  std::uint64_t turns = 0;
};

void run_requests_wallclock(const SimCfg& cfg, const std::uint32_t* requests, std::size_t n, ModelBackend& backend,
                            RequestOutput* outs, const std::string& decision_log_path, WallclockStats* stats);

}  // namespace wsb
