#include "plan.hpp"

#include <algorithm>
#include <filesystem>
#include <json.hpp>

namespace psg {

CmpOp cmp_op_from_string(const std::string& s) {
  if (s == "<") return CmpOp::Lt;
  if (s == "<=") return CmpOp::Le;
  if (s == "==" || s == "=") return CmpOp::Eq;
  if (s == "!=") return CmpOp::Ne;
  if (s == ">=") return CmpOp::Ge;
  if (s == ">") return CmpOp::Gt;
  throw InvalidInput("unknown comparison operator: " + s);
}

std::vector<std::string> expand_glob(const std::string& pattern) {
  namespace fs = std::filesystem;
  const auto star = pattern.find('*');
  if (star == std::string::npos) return fs::exists(pattern) ? std::vector<std::string>{pattern} : std::vector<std::string>{};
  const auto sb = pattern.rfind('/', star);
  const auto sa = pattern.find('/', star);
  const std::string dir = sb == std::string::npos ? "." : pattern.substr(0, sb);
  const std::string comp = pattern.substr(sb + 1, (sa == std::string::npos ? pattern.size() : sa) - sb - 1);
  const std::string rest = sa == std::string::npos ? "" : pattern.substr(sa);
  const auto cs = comp.find('*');
  const std::string prefix = comp.substr(0, cs), suffix = comp.substr(cs + 1);
  std::vector<std::string> out;
  if (!fs::is_directory(dir)) return out;
  for (const auto& e : fs::directory_iterator(dir)) {
    const std::string name = e.path().filename().string();
    if (name.size() < prefix.size() + suffix.size()) continue;
    if (name.compare(0, prefix.size(), prefix) != 0) continue;
    if (!suffix.empty() && name.compare(name.size() - suffix.size(), suffix.size(), suffix) != 0) continue;
    for (auto& r : expand_glob(dir + "/" + name + rest)) out.push_back(std::move(r));
  }
  std::sort(out.begin(), out.end());
  return out;
}

namespace {
std::string substitute(std::string s, const std::string& key, const std::string& value) {
  size_t pos;
  while ((pos = s.find(key)) != std::string::npos) s.replace(pos, key.size(), value);
  return s;
}
}  // namespace

QueryPlan QueryPlan::from_json_text(const std::string& text, const std::string& data_root, int node, int node_count) {
  nlohmann::json j;
  try {
    j = nlohmann::json::parse(text);
  } catch (const std::exception& e) {
    throw InvalidInput(std::string("plan json: ") + e.what());
  }
  QueryPlan p;
  try {
    p.buffer_target_bytes = j.value("buffer_target_bytes", p.buffer_target_bytes);
    p.memory_budget_bytes = j.value("memory_budget_bytes", p.memory_budget_bytes);
    if (j.contains("budget_mb")) p.memory_budget_bytes = j["budget_mb"].get<uint64_t>() * 1024 * 1024;
    p.ht_estimate_bytes = j.value("ht_estimate_bytes", p.ht_estimate_bytes);
    p.io_workers = j.value("io_workers", p.io_workers);
    for (const auto& s : j.at("scans")) {
      ScanNode sc;
      sc.table = s.at("table").get<std::string>();
      sc.replicated = s.value("replicated", false);
      for (const auto& pp : s.at("paths")) {
        std::string path = substitute(pp.get<std::string>(), "{data}", data_root);
        path = substitute(path, "{node}", std::to_string(node));
        path = substitute(path, "{nodes}", std::to_string(node_count));
        auto ex = expand_glob(path);
        if (ex.empty()) throw IoFailure("no files match scan path: " + path);
        for (auto& e : ex) sc.paths.push_back(std::move(e));
      }
      if (s.contains("columns"))
        for (const auto& c : s["columns"]) sc.columns.push_back(c.get<std::string>());
      if (s.contains("predicate"))
        for (const auto& a : s["predicate"]) {
          Atom at;
          at.column = a.at("col").get<std::string>();
          at.op = cmp_op_from_string(a.at("op").get<std::string>());
          const auto& v = a.at("value");
          if (v.is_number_float()) {
            at.lit_is_float = true;
            at.lit_f = v.get<double>();
          } else {
            at.lit_i = v.get<int64_t>();
          }
          sc.predicate.push_back(at);
        }
      p.scans.push_back(std::move(sc));
    }
    if (j.contains("joins"))
      for (const auto& jn : j["joins"]) {
        JoinNode n;
        n.id = jn.at("id").get<std::string>();
        n.build = jn.at("build").get<std::string>();
        n.probe = jn.at("probe").get<std::string>();
        n.build_key = jn.at("build_key").get<std::string>();
        n.probe_key = jn.at("probe_key").get<std::string>();
        n.shuffle = jn.value("mode", std::string("replicated")) == "shuffle";
        p.joins.push_back(std::move(n));
      }
    if (j.contains("aggregate")) {
      AggregateNode a;
      a.group_by = j["aggregate"].value("group_by", std::string{});
      if (j["aggregate"].contains("sums"))
        for (const auto& c : j["aggregate"]["sums"]) a.sums.push_back(c.get<std::string>());
      p.aggregate = std::move(a);
    }
  } catch (const nlohmann::json::exception& e) {
    throw InvalidInput(std::string("plan json: ") + e.what());
  }
  p.validate();
  return p;
}

const ScanNode& QueryPlan::scan(const std::string& table) const {
  for (const auto& s : scans)
    if (s.table == table) return s;
  throw InvalidInput("plan references unknown scan: " + table);
}

const JoinNode* QueryPlan::shuffle_join() const {
  for (const auto& j : joins)
    if (j.shuffle) return &j;
  return nullptr;
}

void QueryPlan::validate() const {
  if (scans.empty()) throw InvalidInput("plan needs at least one scan");
  int shuffles = 0;
  for (const auto& j : joins) {
    if (j.shuffle) {
      ++shuffles;
    } else if (!scan(j.build).replicated) {
      throw InvalidInput("local join '" + j.id + "' must build from a replicated scan");
    }
  }
  if (shuffles > 1) throw InvalidInput("plans support at most one shuffled join");
  if (aggregate && !aggregate->group_by.empty()) {
    const JoinNode* sj = shuffle_join();
    if (sj != nullptr && aggregate->group_by != sj->probe_key)
      throw InvalidInput("group key must match the shuffle probe key so groups co-locate");
  }
}

}  // namespace psg
