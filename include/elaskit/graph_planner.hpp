// elaskit graph planner — B200 build, hot-path subset.
//
// The recovery path consumes only the LayerMove value type from the
// reference's graph planner (reference: graph_planner.hpp:56-62, used by
// rng.hpp:71-73 and migration.hpp:56-57).  The minimax layer partitioner
// itself (plan_partition / diff_assignments, graph_planner.cpp:31-155) is
// pipeline-domain replanning and is out of scope for this library; see
// DESIGN.md "Out of scope".
#pragma once

namespace elaskit {

// One layer changing pipeline stage (1-based stage ids).
struct LayerMove {
  int layer = 0;
  int src_stage = 0;
  int dst_stage = 0;

  bool operator==(const LayerMove&) const = default;
};

}  // namespace elaskit
