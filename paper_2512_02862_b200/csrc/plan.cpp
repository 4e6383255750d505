// Plan JSON -> QueryPlan, written against the JSON contract of the reference's declarative plan
// (keys and semantics: SURVEY.md §5 "Config"; ScanNode/JoinNode/AggregateNode
// /root/reference/proj/include/pystachio/pipeline.hpp:82-122). Behaviour that callers observe is
// the reference's (QueryPlan::from_json_text, pipeline.cpp:108-156; validate :178-196):
//   * placeholders {data}, {node}, {nodes} in every path, then '*' wildcards matched per path
//     component, matches sorted; a path that matches nothing -> IoFailure;
//   * malformed JSON / missing required keys -> InvalidInput;
//   * at most one shuffled join; local joins build from replicated scans; a grouped aggregate
//     groups on the shuffle probe key (so groups co-locate on the key's owner).
#include "plan.hpp"

#include <dirent.h>
#include <sys/stat.h>

#include <algorithm>
#include <functional>
#include <json.hpp>

namespace psg {

using Json = nlohmann::json;

CmpOp cmp_op_from_string(const std::string& s) {
  static const std::pair<const char*, CmpOp> table[] = {{"<", CmpOp::Lt},  {"<=", CmpOp::Le}, {"==", CmpOp::Eq},
                                                        {"=", CmpOp::Eq},  {"!=", CmpOp::Ne}, {">=", CmpOp::Ge},
                                                        {">", CmpOp::Gt}};
  for (const auto& [name, op] : table)
    if (s == name) return op;
  throw InvalidInput("unknown comparison operator: " + s);
}

namespace {

bool path_exists(const std::string& p) {
  struct stat sb;
  return ::stat(p.c_str(), &sb) == 0;
}

bool is_dir(const std::string& p) {
  struct stat sb;
  return ::stat(p.c_str(), &sb) == 0 && S_ISDIR(sb.st_mode);
}

/// Wildcard match of one path component: '*' matches any run of characters (no '/').
bool component_match(const char* pat, const char* name) {
  const char* star = nullptr;
  const char* resume = nullptr;
  while (*name) {
    if (*pat == '*') {
      star = pat++;
      resume = name;
    } else if (*pat == *name) {
      ++pat, ++name;
    } else if (star) {
      pat = star + 1;
      name = ++resume;
    } else {
      return false;
    }
  }
  while (*pat == '*') ++pat;
  return *pat == '\0';
}

std::vector<std::string> split_components(const std::string& p) {
  std::vector<std::string> parts;
  size_t at = 0;
  while (at <= p.size()) {
    const size_t nx = p.find('/', at);
    parts.push_back(p.substr(at, nx == std::string::npos ? std::string::npos : nx - at));
    if (nx == std::string::npos) break;
    at = nx + 1;
  }
  return parts;
}

/// {key} -> value for every occurrence.
std::string fill_placeholder(const std::string& in, const std::string& key, const std::string& value) {
  std::string out;
  out.reserve(in.size());
  size_t at = 0;
  for (size_t hit; (hit = in.find(key, at)) != std::string::npos; at = hit + key.size()) out.append(in, at, hit - at).append(value);
  return out.append(in, at, std::string::npos);
}

const Json& required(const Json& obj, const char* key) {
  if (!obj.is_object() || !obj.contains(key)) throw InvalidInput(std::string("plan json: missing key '") + key + "'");
  return obj[key];
}

std::string str_of(const Json& obj, const char* key) {
  const Json& v = required(obj, key);
  if (!v.is_string()) throw InvalidInput(std::string("plan json: '") + key + "' must be a string");
  return v.get<std::string>();
}

template <class T>
T num_or(const Json& obj, const char* key, T dflt) {
  if (!obj.contains(key)) return dflt;
  const Json& v = obj[key];
  if (!v.is_number()) throw InvalidInput(std::string("plan json: '") + key + "' must be a number");
  return v.get<T>();
}

Atom atom_of(const Json& a) {
  Atom at;
  at.column = str_of(a, "col");
  at.op = cmp_op_from_string(str_of(a, "op"));
  const Json& v = required(a, "value");
  if (!v.is_number()) throw InvalidInput("plan json: predicate value must be a number");
  // float literals keep their double value (literal_as truncates them per column type)
  if (v.is_number_float()) {
    at.lit_is_float = true;
    at.lit_f = v.get<double>();
  } else {
    at.lit_i = v.get<int64_t>();
  }
  return at;
}

}  // namespace

std::vector<std::string> expand_glob(const std::string& pattern) {
  if (pattern.find('*') == std::string::npos)
    return path_exists(pattern) ? std::vector<std::string>{pattern} : std::vector<std::string>{};
  const auto comps = split_components(pattern);
  std::vector<std::string> found;
  // depth-first over components; literal components are appended, wildcard ones are matched
  // against the directory listing of the prefix built so far
  std::function<void(size_t, const std::string&)> walk = [&](size_t i, const std::string& prefix) {
    if (i == comps.size()) {
      if (path_exists(prefix)) found.push_back(prefix);
      return;
    }
    const std::string& c = comps[i];
    auto join = [&](const std::string& name) { return i == 0 ? name : prefix + "/" + name; };
    if (c.find('*') == std::string::npos) {
      walk(i + 1, join(c));
      return;
    }
    const std::string dir = i == 0 ? "." : (prefix.empty() ? "/" : prefix);
    if (!is_dir(dir)) return;
    DIR* d = ::opendir(dir.c_str());
    if (!d) return;
    std::vector<std::string> names;
    while (dirent* e = ::readdir(d)) {
      const std::string name = e->d_name;
      if (name == "." || name == "..") continue;
      if (component_match(c.c_str(), name.c_str())) names.push_back(name);
    }
    ::closedir(d);
    for (const auto& n : names) walk(i + 1, i == 0 ? "./" + n : join(n));
  };
  walk(0, "");
  std::sort(found.begin(), found.end());
  return found;
}

namespace {
QueryPlan parse_plan(const std::string& text, const std::string& data_root, int node, int node_count) {
  Json doc = Json::parse(text, nullptr, /*allow_exceptions=*/false);
  if (doc.is_discarded()) throw InvalidInput("plan json: parse error");
  if (!doc.is_object()) throw InvalidInput("plan json: the plan must be an object");
  QueryPlan plan;
  plan.buffer_target_bytes = num_or<uint64_t>(doc, "buffer_target_bytes", plan.buffer_target_bytes);
  plan.memory_budget_bytes = num_or<uint64_t>(doc, "memory_budget_bytes", plan.memory_budget_bytes);
  if (doc.contains("budget_mb")) plan.memory_budget_bytes = num_or<uint64_t>(doc, "budget_mb", 0) << 20;
  plan.ht_estimate_bytes = num_or<uint64_t>(doc, "ht_estimate_bytes", plan.ht_estimate_bytes);
  plan.io_workers = num_or<int>(doc, "io_workers", plan.io_workers);

  const std::pair<const char*, std::string> vars[] = {
      {"{data}", data_root}, {"{node}", std::to_string(node)}, {"{nodes}", std::to_string(node_count)}};
  auto resolve = [&](std::string p) {
    for (const auto& [k, v] : vars) p = fill_placeholder(p, k, v);
    return p;
  };

  for (const Json& s : required(doc, "scans")) {
    ScanNode sc;
    sc.table = str_of(s, "table");
    sc.replicated = s.contains("replicated") && s["replicated"].is_boolean() && s["replicated"].get<bool>();
    for (const Json& p : required(s, "paths")) {
      if (!p.is_string()) throw InvalidInput("plan json: scan paths must be strings");
      const std::string path = resolve(p.get<std::string>());
      std::vector<std::string> hits = expand_glob(path);
      if (hits.empty()) throw IoFailure("no files match scan path: " + path);
      sc.paths.insert(sc.paths.end(), hits.begin(), hits.end());
    }
    if (s.contains("columns"))
      for (const Json& c : s["columns"]) sc.columns.push_back(c.get<std::string>());
    if (s.contains("predicate"))
      for (const Json& a : s["predicate"]) sc.predicate.push_back(atom_of(a));
    plan.scans.push_back(std::move(sc));
  }
  if (doc.contains("joins"))
    for (const Json& jn : doc["joins"]) {
      JoinNode n;
      n.id = str_of(jn, "id");
      n.build = str_of(jn, "build");
      n.probe = str_of(jn, "probe");
      n.build_key = str_of(jn, "build_key");
      n.probe_key = str_of(jn, "probe_key");
      n.shuffle = jn.contains("mode") && jn["mode"] == "shuffle";
      plan.joins.push_back(std::move(n));
    }
  if (doc.contains("aggregate")) {
    const Json& a = doc["aggregate"];
    AggregateNode agg;
    if (a.contains("group_by")) agg.group_by = a["group_by"].get<std::string>();
    if (a.contains("sums"))
      for (const Json& c : a["sums"]) agg.sums.push_back(c.get<std::string>());
    plan.aggregate = std::move(agg);
  }
  return plan;
}
}  // namespace

QueryPlan QueryPlan::from_json_text(const std::string& text, const std::string& data_root, int node, int node_count) {
  QueryPlan plan;
  try {
    plan = parse_plan(text, data_root, node, node_count);
  } catch (const Json::exception& e) {  // wrong value types inside an otherwise valid document
    throw InvalidInput(std::string("plan json: ") + e.what());
  }
  plan.validate();
  return plan;
}

const ScanNode& QueryPlan::scan(const std::string& table) const {
  auto it = std::find_if(scans.begin(), scans.end(), [&](const ScanNode& s) { return s.table == table; });
  if (it == scans.end()) throw InvalidInput("plan references unknown scan: " + table);
  return *it;
}

const JoinNode* QueryPlan::shuffle_join() const {
  auto it = std::find_if(joins.begin(), joins.end(), [](const JoinNode& j) { return j.shuffle; });
  return it == joins.end() ? nullptr : &*it;
}

void QueryPlan::validate() const {
  if (scans.empty()) throw InvalidInput("plan needs at least one scan");
  for (const auto& j : joins)
    if (!j.shuffle && !scan(j.build).replicated)
      throw InvalidInput("local join '" + j.id + "' must build from a replicated scan");
  const auto nshuffle = std::count_if(joins.begin(), joins.end(), [](const JoinNode& j) { return j.shuffle; });
  if (nshuffle > 1) throw InvalidInput("plans support at most one shuffled join");
  const JoinNode* sj = shuffle_join();
  if (aggregate && !aggregate->group_by.empty() && sj && aggregate->group_by != sj->probe_key)
    throw InvalidInput("group key must match the shuffle probe key so groups co-locate");
}

}  // namespace psg
