// Cluster model: resource pool, stage x DP-slot grid, elastic events (host
// side).  The recovery path derives its old/new DP membership from
// apply_event + dp_group (b200::dp_transition in layout.cpp).  Behaviour
// follows the reference (cluster.cpp, cited per function); to_string /
// event_kind_from_string live in communicator.cpp.
#include "elaskit/cluster.hpp"

#include <algorithm>
#include <string>

namespace elaskit {

namespace {

Device& live_target(ClusterState& st, DeviceId id) {
  const auto it = st.devices.find(id);
  if (it == st.devices.end()) throw UnknownDevice("unknown device " + std::to_string(id));
  if (!it->second.alive)
    throw EventOnDeadDevice("device " + std::to_string(id) + " already dead");
  return it->second;
}

void check_stage(const ClusterState& st, int stage) {
  if (stage < 1 || stage > static_cast<int>(st.topology.rank_grid.size()))
    throw BadEvent("stage out of range: " + std::to_string(stage));
}

}  // namespace

// reference: cluster.cpp:25-35
std::vector<int> Topology::dp_per_stage() const {
  std::vector<int> per;
  per.reserve(rank_grid.size());
  for (const auto& stage : rank_grid)
    per.push_back(static_cast<int>(std::count_if(stage.begin(), stage.end(),
                                                 [](DeviceId d) { return d >= 0; })));
  return per;
}

// reference: cluster.cpp:37-94.  Targets are processed in order; the first
// bad target throws and the partially edited copy is discarded, so the
// caller's state is never half-applied.
ClusterState apply_event(const ClusterState& state, const ElasticEvent& ev) {
  if (ev.targets.empty()) throw BadEvent("event has no targets");
  ClusterState out = state;
  if (ev.kind == EventKind::FailSlow) {
    if (!(ev.slow_factor > 1.0)) throw BadEvent("fail_slow requires slow_factor > 1");
    for (const DeviceId id : ev.targets) live_target(out, id).slow_factor = ev.slow_factor;
    return out;
  }
  if (ev.kind == EventKind::ScaleOut) {
    for (const DeviceId id : ev.targets) {
      const auto it = out.devices.find(id);
      if (it != out.devices.end() && it->second.alive)
        throw DuplicateDeviceId("device id " + std::to_string(id) + " already present");
      // a newcomer copies the capacity / clock envelope of the lowest id
      // present at its arrival (earlier targets of the same event included)
      Device d = out.devices.empty() ? Device{} : out.devices.begin()->second;
      d.id = id;
      d.node_id = -1;
      d.slow_factor = 1.0;
      d.alive = true;
      out.devices[id] = d;
      out.free_pool.push_back(id);
    }
    std::sort(out.free_pool.begin(), out.free_pool.end());
    return out;
  }
  // FailStop / ScaleIn: the device leaves its slot and the free pool
  for (const DeviceId id : ev.targets) {
    live_target(out, id).alive = false;
    for (auto& stage : out.topology.rank_grid)
      std::replace(stage.begin(), stage.end(), id, DeviceId{-1});
    out.free_pool.erase(std::remove(out.free_pool.begin(), out.free_pool.end(), id),
                        out.free_pool.end());
  }
  return out;
}

// reference: cluster.cpp:96-105
std::vector<DeviceId> dp_group(const ClusterState& state, int stage) {
  check_stage(state, stage);
  std::vector<DeviceId> members;
  for (const DeviceId d : state.topology.rank_grid[static_cast<std::size_t>(stage - 1)]) {
    if (d < 0) continue;
    const auto it = state.devices.find(d);
    if (it != state.devices.end() && it->second.alive) members.push_back(d);
  }
  if (members.empty())
    throw EmptyStage("stage " + std::to_string(stage) + " has no alive members");
  return members;
}

// reference: cluster.cpp:107-116
std::pair<std::optional<int>, std::optional<int>> pp_neighbors(const ClusterState& state,
                                                               int stage) {
  check_stage(state, stage);
  const int last = static_cast<int>(state.topology.rank_grid.size());
  return {stage > 1 ? std::optional<int>(stage - 1) : std::nullopt,
          stage < last ? std::optional<int>(stage + 1) : std::nullopt};
}

// reference: cluster.cpp:118-123
int alive_device_count(const ClusterState& state) {
  return static_cast<int>(std::count_if(state.devices.begin(), state.devices.end(),
                                        [](const auto& kv) { return kv.second.alive; }));
}

// reference: cluster.cpp:125-149
ClusterState make_uniform_cluster(int pp, int dp, std::int64_t mem_capacity_bytes, int freq_mhz,
                                  int freq_max_mhz, int devices_per_node, int tp) {
  ClusterState st;
  st.topology.tp = tp;
  st.topology.pp = pp;
  st.topology.rank_grid.assign(static_cast<std::size_t>(std::max(pp, 0)),
                               std::vector<DeviceId>(static_cast<std::size_t>(std::max(dp, 0)), -1));
  const int units_per_node = std::max(1, devices_per_node / std::max(1, tp));
  for (int slot = 0; slot < dp; ++slot) {
    for (int s = 0; s < pp; ++s) {
      const DeviceId id = slot * pp + s;
      Device d;
      d.id = id;
      d.node_id = id / units_per_node;
      d.mem_capacity_bytes = mem_capacity_bytes;
      d.freq_mhz = freq_mhz;
      d.freq_max_mhz = freq_max_mhz;
      st.devices[id] = d;
      st.topology.rank_grid[static_cast<std::size_t>(s)][static_cast<std::size_t>(slot)] = id;
    }
  }
  return st;
}

}  // namespace elaskit
