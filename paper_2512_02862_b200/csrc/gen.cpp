// TPC-H-analog workload generator (the path's data source, not accelerated): byte-identical to
// gen_workload(kind=tpch) (/root/reference/proj/src/bench.cpp:85-114, workload.cpp:89-153),
// pinned by tests/golden/gen_hashes.json. Streams each table straight into its node shards
// (slice_for_node, workload.cpp:73-87: rows r ≡ node mod nodes) so SF100/SF1000 never need the
// whole table in RAM; one thread per table, with a writer thread per table so generation and
// file writes overlap.
#include <sys/stat.h>

#include <condition_variable>
#include <deque>
#include <filesystem>
#include <functional>
#include <memory>
#include <mutex>
#include <algorithm>
#include <numeric>
#include <random>
#include <thread>
#include <tuple>

#include <fstream>
#include <json.hpp>

#include "engine.hpp"
#include "psto.hpp"

namespace psg {
namespace {

/// std::mt19937_64 (Matsumoto-Nishimura 64-bit parameters), batched twist.
class Mt64 {
 public:
  explicit Mt64(uint64_t seed) {
    mt_[0] = seed;
    for (int i = 1; i < 312; ++i) mt_[i] = 6364136223846793005ULL * (mt_[i - 1] ^ (mt_[i - 1] >> 62)) + i;
    idx_ = 312;
  }
  inline uint64_t operator()() {
    if (idx_ >= 312) twist();
    uint64_t y = mt_[idx_++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
  }

 private:
  void twist() {
    constexpr uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    int i = 0;
    for (; i < 312 - 156; ++i) {
      uint64_t x = (mt_[i] & UM) | (mt_[i + 1] & LM);
      mt_[i] = mt_[i + 156] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    }
    for (; i < 311; ++i) {
      uint64_t x = (mt_[i] & UM) | (mt_[i + 1] & LM);
      mt_[i] = mt_[i - 156] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    }
    uint64_t x = (mt_[311] & UM) | (mt_[0] & LM);
    mt_[311] = mt_[155] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    idx_ = 0;
  }
  uint64_t mt_[312];
  int idx_;
};

/// yyyymmdd; GCC evaluates the three rng() calls of workload.cpp:118-119 left to right.
inline int64_t gen_date(Mt64& r) {
  const uint64_t y = 1992 + r() % 7;
  const uint64_t m = 1 + r() % 12;
  const uint64_t d = 1 + r() % 28;
  return static_cast<int64_t>(y * 10000 + m * 100 + d);
}

using RowFn = std::function<void(Mt64&, uint64_t row, uint64_t* out)>;

/// Streams `rows` rows of a table into `nodes` shard files (row r -> node r % nodes).
void stream_table(const Schema& schema, uint64_t rows, uint64_t seed, const RowFn& fn,
                  const std::vector<std::string>& paths, uint64_t rg_bytes, Codec codec) {
  const int nodes = static_cast<int>(paths.size());
  const size_t ncols = schema.size();
  const uint64_t rg_rows = PstoWriter::rows_for_group_bytes(schema, rg_bytes);
  std::vector<std::unique_ptr<PstoWriter>> writers;
  for (auto& p : paths) writers.push_back(std::make_unique<PstoWriter>(p, schema, rg_rows, codec));
  // Block of rows = nodes * rg_rows so that each node receives whole row groups per block.
  const uint64_t block = static_cast<uint64_t>(nodes) * rg_rows;
  struct Buf {
    std::vector<std::vector<std::vector<uint64_t>>> per_node;  // [node][col] words
  };
  std::mutex mu;
  std::condition_variable cv;
  std::deque<std::unique_ptr<Buf>> full, empty;
  bool done = false;
  for (int i = 0; i < 3; ++i) {
    auto b = std::make_unique<Buf>();
    b->per_node.assign(nodes, std::vector<std::vector<uint64_t>>(ncols));
    empty.push_back(std::move(b));
  }
  std::exception_ptr werr;
  std::thread writer([&] {
    try {
      while (true) {
        std::unique_ptr<Buf> b;
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return !full.empty() || done; });
          if (full.empty()) return;
          b = std::move(full.front());
          full.pop_front();
        }
        auto append = [&](int n) {
          std::vector<const uint64_t*> ptrs(ncols);
          for (size_t c = 0; c < ncols; ++c) ptrs[c] = b->per_node[n][c].data();
          if (!b->per_node[n][0].empty()) writers[n]->append(ptrs.data(), b->per_node[n][0].size());
        };
        if (codec == Codec::Block && nodes > 1) {
          // deflate dominates: compress the node shards' row groups concurrently (files are
          // independent, so the bytes are identical to the sequential writer's)
          std::vector<std::thread> ts;
          std::vector<std::exception_ptr> errs(nodes);
          for (int n = 0; n < nodes; ++n)
            ts.emplace_back([&, n] {
              try {
                append(n);
              } catch (...) {
                errs[n] = std::current_exception();
              }
            });
          for (auto& t : ts) t.join();
          for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        } else {
          for (int n = 0; n < nodes; ++n) append(n);
        }
        std::lock_guard<std::mutex> lk(mu);
        empty.push_back(std::move(b));
        cv.notify_all();
      }
    } catch (...) {
      std::lock_guard<std::mutex> lk(mu);
      werr = std::current_exception();
      cv.notify_all();
    }
  });
  Mt64 rng(seed);
  uint64_t row = 0;
  uint64_t vals[8];
  try {
    while (row < rows) {
      std::unique_ptr<Buf> b;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return !empty.empty() || werr; });
        if (werr) break;
        b = std::move(empty.front());
        empty.pop_front();
      }
      const uint64_t n = std::min(block, rows - row);
      for (int k = 0; k < nodes; ++k)
        for (size_t c = 0; c < ncols; ++c) b->per_node[k][c].clear();
      for (uint64_t i = 0; i < n; ++i, ++row) {
        fn(rng, row, vals);
        auto& dst = b->per_node[row % static_cast<uint64_t>(nodes)];
        for (size_t c = 0; c < ncols; ++c) dst[c].push_back(vals[c]);
      }
      std::lock_guard<std::mutex> lk(mu);
      full.push_back(std::move(b));
      cv.notify_all();
    }
  } catch (...) {
    std::lock_guard<std::mutex> lk(mu);
    done = true;
    cv.notify_all();
  }
  {
    std::lock_guard<std::mutex> lk(mu);
    done = true;
    cv.notify_all();
  }
  writer.join();
  if (werr) std::rethrow_exception(werr);
  for (auto& w : writers) w->finish();
}

Schema int_schema(std::initializer_list<const char*> names) {
  Schema s;
  for (auto* n : names) s.fields.push_back(Field{n, LType::Int64});
  return s;
}

}  // namespace

void gen_tpch(const std::string& out_dir, double scale, int nodes, int devices, uint64_t seed,
              Codec codec, uint64_t rg_bytes, int threads) {
  if (nodes < 1 || devices < 1) throw InvalidInput("devices and nodes must be >= 1");
  namespace fs = std::filesystem;
  fs::create_directories(out_dir);
  auto dev_dir = [&](int i) {  // device_dir, bench.cpp:44-46
    std::string d = (fs::path(out_dir) / ("dev" + std::to_string(i % devices))).string();
    fs::create_directories(d);
    return d;
  };
  const std::string cust_path = dev_dir(0) + "/customer.psto";
  std::vector<std::string> opaths, lpaths;
  for (int n = 0; n < nodes; ++n) opaths.push_back(dev_dir(0 + n) + "/orders.node" + std::to_string(n) + ".psto");
  for (int n = 0; n < nodes; ++n) lpaths.push_back(dev_dir(1 + n) + "/lineitem.node" + std::to_string(n) + ".psto");
  const uint64_t customers = static_cast<uint64_t>(150'000 * scale);
  const uint64_t orders = static_cast<uint64_t>(1'500'000 * scale);
  const uint64_t lineitems = static_cast<uint64_t>(6'000'000 * scale);
  const uint64_t mult = 0x9E3779B97F4A7C15ULL;

  std::vector<std::function<void()>> jobs;
  jobs.push_back([&] {
    stream_table(int_schema({"c_custkey", "c_mktsegment"}), customers, seed * mult + 11,
                 [](Mt64& r, uint64_t i, uint64_t* v) {
                   v[0] = i;
                   v[1] = r() % 5;
                 },
                 {cust_path}, rg_bytes, codec);
  });
  jobs.push_back([&] {
    const std::vector<std::string>& paths = opaths;
    stream_table(int_schema({"o_orderkey", "o_custkey", "o_orderdate", "o_shippriority"}), orders, seed * mult + 12,
                 [customers](Mt64& r, uint64_t i, uint64_t* v) {
                   v[0] = i;
                   v[1] = customers > 0 ? r() % customers : 0;
                   v[2] = static_cast<uint64_t>(gen_date(r));
                   v[3] = r() % 5;
                 },
                 paths, rg_bytes, codec);
  });
  jobs.push_back([&] {
    const std::vector<std::string>& paths = lpaths;
    stream_table(int_schema({"l_orderkey", "l_extendedprice", "l_discount", "l_shipdate"}), lineitems,
                 seed * mult + 13,
                 [orders](Mt64& r, uint64_t, uint64_t* v) {
                   v[0] = orders > 0 ? r() % orders : 0;
                   v[1] = 90'000 + r() % 100'000;
                   v[2] = r() % 11;
                   v[3] = static_cast<uint64_t>(gen_date(r));
                 },
                 paths, rg_bytes, codec);
  });
  if (threads <= 1) {
    for (auto& j : jobs) j();
  } else {
    std::vector<std::thread> ts;
    std::vector<std::exception_ptr> errs(jobs.size());
    for (size_t i = 0; i < jobs.size(); ++i)
      ts.emplace_back([&, i] {
        try {
          jobs[i]();
        } catch (...) {
          errs[i] = std::current_exception();
        }
      });
    for (auto& t : ts) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  }
  // manifest.json with the reference's keys and layout (gen_workload, bench.cpp:85-114)
  nlohmann::json m;
  m["nodes"] = nodes;
  m["devices"] = devices;
  m["seed"] = seed;
  m["kind"] = "tpch-analog";
  m["scale"] = scale;
  m["tables"]["customer"]["replicated"] = true;
  m["tables"]["customer"]["rows"] = customers;
  m["tables"]["customer"]["path"] = cust_path;
  for (auto [name, rows, paths] : {std::make_tuple("orders", orders, &opaths), std::make_tuple("lineitem", lineitems, &lpaths)}) {
    m["tables"][name]["replicated"] = false;
    m["tables"][name]["rows"] = rows;
    m["tables"][name]["paths_per_node"] = *paths;
  }
  const std::string mpath = (fs::path(out_dir) / "manifest.json").string();
  std::ofstream out(mpath);
  if (!out) throw IoFailure("cannot write manifest: " + mpath);
  out << m.dump(2) << '\n';
}

/// gen_workload(kind = synthetic join) (bench.cpp:93-99; gen_build_table / gen_probe_table,
/// workload.cpp:41-71). The reference draws from std::mt19937_64 through std::shuffle and
/// std::uniform_real_distribution; this file is built with the same C++ standard library, so the
/// same calls in the same order give byte-identical tables (pinned against the reference's own
/// generator, tests/test_abi.py). Tables are sliced round-robin per node (slice_for_node,
/// workload.cpp:73-87) and written like write_sharded (bench.cpp:48-65).
namespace {
/// gen_build_table / gen_probe_table (workload.cpp:41-71): build keys 0..n-1 shuffled, probe keys a
/// hit_ratio share drawn from the build range and the rest from a miss range; payload columns of
/// values < 1e9 (payload_columns, workload.cpp:29-37).
void synthetic_columns(uint64_t seed, uint64_t build_rows, uint64_t probe_rows, int payload_cols, double hit_ratio,
                       std::vector<std::vector<uint64_t>>& bcols, std::vector<std::vector<uint64_t>>& pcols) {
  const uint64_t mul = 2654435761u;
  auto payload = [&](std::mt19937_64& rng, uint64_t rows, std::vector<std::vector<uint64_t>>& cols) {
    for (int c = 0; c < payload_cols; ++c) {
      std::vector<uint64_t> v(rows);
      for (auto& x : v) x = static_cast<uint64_t>(static_cast<int64_t>(rng() % 1'000'000'000));
      cols.push_back(std::move(v));
    }
  };
  {
    std::mt19937_64 rng(seed * mul + 1);
    std::vector<int64_t> keys(build_rows);
    std::iota(keys.begin(), keys.end(), int64_t{0});
    std::shuffle(keys.begin(), keys.end(), rng);
    bcols.emplace_back(keys.begin(), keys.end());
    payload(rng, build_rows, bcols);
  }
  {
    std::mt19937_64 rng(seed * mul + 2);
    std::uniform_real_distribution<double> coin(0.0, 1.0);
    std::vector<uint64_t> keys(probe_rows);
    for (auto& k : keys) {
      if (build_rows > 0 && coin(rng) < hit_ratio)
        k = static_cast<uint64_t>(static_cast<int64_t>(rng() % build_rows));
      else
        k = static_cast<uint64_t>(static_cast<int64_t>(build_rows + rng() % 1'000'000'000ull));
    }
    pcols.push_back(std::move(keys));
    payload(rng, probe_rows, pcols);
  }
}
}  // namespace

void synthetic_join_tables(uint64_t seed, uint64_t build_rows, uint64_t probe_rows, int payload_cols, double hit_ratio,
                           int node, int nodes, HostTable& build, HostTable& probe) {
  if (nodes < 1 || node < 0 || node >= nodes) throw InvalidInput("node out of range");
  if (payload_cols < 0 || payload_cols > 14) throw InvalidInput("payload_cols out of range");
  std::vector<std::vector<uint64_t>> bcols, pcols;
  synthetic_columns(seed, build_rows, probe_rows, payload_cols, hit_ratio, bcols, pcols);
  auto slice = [&](std::vector<std::vector<uint64_t>>& cols, HostTable& t, const char* key, const char* pre) {
    t.names = {key};
    for (int i = 0; i < payload_cols; ++i) t.names.push_back(pre + std::to_string(i));
    t.cols.assign(cols.size(), {});
    for (size_t c = 0; c < cols.size(); ++c) {
      if (nodes == 1) {
        t.cols[c] = std::move(cols[c]);
        continue;
      }
      for (uint64_t r = static_cast<uint64_t>(node); r < cols[c].size(); r += static_cast<uint64_t>(nodes))
        t.cols[c].push_back(cols[c][r]);
    }
  };
  slice(bcols, build, "bk", "bp");
  slice(pcols, probe, "pk", "pp");
}

void gen_synthetic(const std::string& out_dir, int nodes, int devices, uint64_t seed, Codec codec, uint64_t rg_bytes,
                   uint64_t build_rows, uint64_t probe_rows, int payload_cols, double hit_ratio) {
  if (nodes < 1 || devices < 1) throw InvalidInput("devices and nodes must be >= 1");
  if (payload_cols < 0 || payload_cols > 14) throw InvalidInput("payload_cols out of range");
  namespace fs = std::filesystem;
  fs::create_directories(out_dir);
  auto side = [&](const char* key, const char* pre) {
    Schema sc;
    sc.fields.push_back(Field{key, LType::Int64});
    for (int i = 0; i < payload_cols; ++i) sc.fields.push_back(Field{pre + std::to_string(i), LType::Int64});
    return sc;
  };
  std::vector<std::vector<uint64_t>> bcols, pcols;
  synthetic_columns(seed, build_rows, probe_rows, payload_cols, hit_ratio, bcols, pcols);
  nlohmann::json m;
  m["nodes"] = nodes;
  m["devices"] = devices;
  m["seed"] = seed;
  m["kind"] = "synthetic-join";
  m["hit_ratio"] = hit_ratio;
  auto write_sharded = [&](const Schema& sc, const std::vector<std::vector<uint64_t>>& cols, uint64_t rows,
                           const std::string& name, int file_index) {
    nlohmann::json entry;
    entry["replicated"] = false;
    entry["rows"] = rows;
    auto paths = nlohmann::json::array();
    const uint64_t rg_rows = PstoWriter::rows_for_group_bytes(sc, rg_bytes);
    for (int node = 0; node < nodes; ++node) {
      const std::string dir = (fs::path(out_dir) / ("dev" + std::to_string((file_index + node) % devices))).string();
      fs::create_directories(dir);
      const std::string path = dir + "/" + name + ".node" + std::to_string(node) + ".psto";
      std::vector<std::vector<uint64_t>> slice(cols.size());
      for (size_t c = 0; c < cols.size(); ++c)
        for (uint64_t r = static_cast<uint64_t>(node); r < rows; r += static_cast<uint64_t>(nodes)) slice[c].push_back(cols[c][r]);
      PstoWriter w(path, sc, rg_rows, codec);
      std::vector<const uint64_t*> ptrs;
      for (auto& c : slice) ptrs.push_back(c.data());
      if (!slice.empty() && !slice[0].empty()) w.append(ptrs.data(), slice[0].size());
      w.finish();
      paths.push_back(path);
    }
    entry["paths_per_node"] = paths;
    return entry;
  };
  m["tables"]["build"] = write_sharded(side("bk", "bp"), bcols, build_rows, "build", 0);
  m["tables"]["probe"] = write_sharded(side("pk", "pp"), pcols, probe_rows, "probe", 1);
  const std::string mpath = (fs::path(out_dir) / "manifest.json").string();
  std::ofstream out(mpath);
  if (!out) throw IoFailure("cannot write manifest: " + mpath);
  out << m.dump(2) << '\n';
}

}  // namespace psg
