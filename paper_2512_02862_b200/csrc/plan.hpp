// Declarative query plan — same JSON contract and validation as the reference
// (QueryPlan::from_json_text, /root/reference/proj/src/pipeline.cpp:108-156; validate :178-196;
// ScanNode/JoinNode/AggregateNode pipeline.hpp:82-122).
#pragma once

#include <optional>
#include <string>
#include <vector>

#include "common.hpp"

namespace psg {

struct ScanNode {
  std::string table;
  std::vector<std::string> paths;  // this node's shards ({node} resolved, globs expanded)
  std::vector<std::string> columns;
  Predicate predicate;
  bool replicated = false;
};

struct JoinNode {
  std::string id, build, probe, build_key, probe_key;
  bool shuffle = false;
};

struct AggregateNode {
  std::string group_by;  // empty = global aggregate; else must equal the shuffle probe key
  std::vector<std::string> sums;
};

struct QueryPlan {
  std::vector<ScanNode> scans;
  std::vector<JoinNode> joins;
  std::optional<AggregateNode> aggregate;
  uint64_t buffer_target_bytes = 8ull << 20;
  uint64_t memory_budget_bytes = 0;
  uint64_t ht_estimate_bytes = 0;
  int io_workers = 4;

  static QueryPlan from_json_text(const std::string& text, const std::string& data_root, int node, int node_count);
  void validate() const;
  const ScanNode& scan(const std::string& table) const;
  const JoinNode* shuffle_join() const;
};

std::vector<std::string> expand_glob(const std::string& pattern);

}  // namespace psg
