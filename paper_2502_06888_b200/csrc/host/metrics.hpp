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

}  // namespace moesim::detail
