// SPDX-License-Identifier: Apache-2.0
// Shared metric finalization (internal): RunMetrics from a timeline, used by
// the pricing simulator and by the B200 executor on measured timestamps
// (reference definitions: proj/src/simulator.cpp:256-285).
#pragma once

#include <span>

#include "moesim/simulator.hpp"

namespace moesim::detail {

void finalize_metrics(const Schedule& schedule, std::span<const SimEvent> timeline,
                      byte_count peak_vram, RunMetrics& m);

// Ledger replay on a timeline (the run()'s accounting, simulator.cpp
// replay_ledger, applied to measured start/end times): resident tensors at
// t = 0, then every op's LedgerEffects at its start or end, frees first at
// equal times. Frees of tags allocated before the window (a run that starts
// mid-stream) are skipped and counted. Returns the number of such frees.
std::int64_t replay_ledger_on_timeline(const Schedule& schedule, std::span<const SimEvent> timeline,
                                       const PipelinePlan& plan, MemoryLedger& ledger);

}  // namespace moesim::detail
