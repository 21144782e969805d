// Dynamic-communicator edit planning (host side).
//
// plan_edit decides which peer links a membership change adds and removes;
// on B200 the executor (capi.cpp: ew_comm_shrink, ew_peer_*) maps removals to
// NCCL communicator shrink + IPC unmaps.  Outputs match the reference
// (communicator.cpp, cited per function).
#include "elaskit/communicator.hpp"

#include <algorithm>
#include <map>

namespace elaskit {

// reference: cluster.cpp:7-15
std::string to_string(EventKind k) {
  switch (k) {
    case EventKind::FailStop: return "fail_stop";
    case EventKind::FailSlow: return "fail_slow";
    case EventKind::ScaleIn: return "scale_in";
    case EventKind::ScaleOut: return "scale_out";
  }
  return "?";
}

// reference: cluster.cpp:17-23
std::optional<EventKind> event_kind_from_string(const std::string& s) {
  static const std::map<std::string, EventKind> kinds = {{"fail_stop", EventKind::FailStop},
                                                          {"fail_slow", EventKind::FailSlow},
                                                          {"scale_in", EventKind::ScaleIn},
                                                          {"scale_out", EventKind::ScaleOut}};
  const auto it = kinds.find(s);
  if (it == kinds.end()) return std::nullopt;
  return it->second;
}

// reference: communicator.cpp:8
Link make_link(int a, int b) { return {std::min(a, b), std::max(a, b)}; }

// reference: communicator.cpp:10-21
std::set<Link> CommGroup::required_links() const {
  std::set<Link> links;
  const std::size_t n = members.size();
  if (n < 2) return links;
  if (topo == GroupTopology::Ring) {
    for (std::size_t i = 0; i < n; ++i) links.insert(make_link(members[i], members[(i + 1) % n]));
    return links;
  }
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = i + 1; j < n; ++j) links.insert(make_link(members[i], members[j]));
  return links;
}

// reference: communicator.cpp:23-25
bool CommGroup::contains(int rank) const {
  return std::find(members.begin(), members.end(), rank) != members.end();
}

namespace {

// Are all `nodes` reachable from nodes[0] using only edges between nodes?
// (reference: communicator.cpp:29-50)
bool spans(const std::vector<int>& nodes, const std::set<Link>& edges) {
  if (nodes.size() <= 1) return true;
  const std::set<int> wanted(nodes.begin(), nodes.end());
  std::map<int, std::vector<int>> adj;
  for (const Link& e : edges) {
    adj[e.first].push_back(e.second);
    adj[e.second].push_back(e.first);
  }
  std::set<int> reached = {nodes.front()};
  std::vector<int> frontier = {nodes.front()};
  while (!frontier.empty()) {
    const int v = frontier.back();
    frontier.pop_back();
    for (const int w : adj[v])
      if (wanted.contains(w) && reached.insert(w).second) frontier.push_back(w);
  }
  return reached.size() == wanted.size();
}

bool touches(const CommGroup& g, const std::vector<int>& targets) {
  return std::any_of(targets.begin(), targets.end(), [&](int r) { return g.contains(r); });
}

}  // namespace

// reference: communicator.cpp:54-105
EditPlan plan_edit(const std::vector<CommGroup>& groups, const ElasticEvent& ev,
                   const std::set<Link>& global_link_pool) {
  EditPlan plan;
  const std::set<int> moving(ev.targets.begin(), ev.targets.end());
  const auto incident = [&](const Link& l) {
    return moving.contains(l.first) || moving.contains(l.second);
  };

  for (const CommGroup& g : groups) {
    if (!touches(g, ev.targets)) continue;
    plan.groups_touched.insert(g.id);

    if (ev.kind == EventKind::ScaleOut) {
      for (const Link& l : g.required_links())
        if (incident(l) && !global_link_pool.contains(l)) plan.links_to_add.insert(l);
      continue;
    }

    std::vector<int> survivors;
    for (const int m : g.members)
      if (!moving.contains(m)) survivors.push_back(m);

    for (const Link& l : global_link_pool)
      if (incident(l) && g.contains(l.first) && g.contains(l.second))
        plan.links_to_remove.insert(l);

    if (g.topo == GroupTopology::Ring && survivors.size() >= 2) {
      CommGroup healed = g;
      healed.members = survivors;
      for (const Link& l : healed.required_links())
        if (!global_link_pool.contains(l)) plan.links_to_add.insert(l);
    }

    std::set<Link> remaining;
    for (const Link& l : g.required_links())
      if (global_link_pool.contains(l) && !plan.links_to_remove.contains(l)) remaining.insert(l);
    for (const Link& l : plan.links_to_add)
      if (g.contains(l.first) && g.contains(l.second)) remaining.insert(l);
    if (!spans(survivors, remaining))
      throw DisconnectedGroup("edit disconnects group " + g.id + "; replanning must regroup");
  }
  for (const Link& l : plan.links_to_add) plan.links_to_remove.erase(l);
  return plan;
}

// reference: communicator.cpp:107-110
double estimate_recovery_time(const EditPlan& plan, const CommCostModel& cost) {
  return cost.per_group_fixed_s * static_cast<double>(plan.groups_touched.size()) +
         cost.per_link_setup_s * static_cast<double>(plan.links_to_add.size());
}

namespace {

// Shared body of the two rebuild baselines (reference: communicator.cpp:112-152).
RebuildEstimate rebuild(const std::vector<CommGroup>& groups, const ElasticEvent& ev,
                        const CommCostModel& cost, double fixed, bool only_touched) {
  const std::set<int> moving(ev.targets.begin(), ev.targets.end());
  RebuildEstimate est;
  est.time_s = fixed;
  for (const CommGroup& g : groups) {
    if (only_touched && !touches(g, ev.targets)) continue;
    CommGroup fresh = g;
    if (ev.kind != EventKind::ScaleOut) {
      fresh.members.clear();
      for (const int m : g.members)
        if (!moving.contains(m)) fresh.members.push_back(m);
    }
    est.links_created += static_cast<std::int64_t>(fresh.required_links().size());
    est.time_s += cost.per_group_fixed_s;
  }
  est.time_s += cost.per_link_setup_s * static_cast<double>(est.links_created);
  return est;
}

}  // namespace

RebuildEstimate estimate_partial_rebuild(const std::vector<CommGroup>& groups,
                                         const ElasticEvent& ev, const CommCostModel& cost) {
  return rebuild(groups, ev, cost, cost.partial_restart_fixed_s, true);
}

RebuildEstimate estimate_full_rebuild(const std::vector<CommGroup>& groups,
                                      const ElasticEvent& ev, const CommCostModel& cost) {
  return rebuild(groups, ev, cost, cost.full_restart_fixed_s, false);
}

}  // namespace elaskit
