// Private seams between the scheduler and the GPU runtime.
#pragma once

#include <cstdint>
#include <vector>

#include "cake/scheduler.hpp"
#include "cake/transfer.hpp"

namespace cake::detail {

// sort + exactly-once check + ttft/busy/merge (reference scheduler.cpp:105-124)
void finalize_report(RunReport& report, std::uint32_t merge_point);
std::uint32_t merge_from_records(const RunReport& report);

RunReport run_live_gpu(const RunPlan& plan, const std::vector<std::uint32_t>& tokens, const CostModel& cost,
                       const BandwidthTrace& trace, const Codec& codec, const ChunkStore& store, RunMode mode,
                       double power, const RunOptions& options);

}  // namespace cake::detail
