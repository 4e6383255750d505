// Test infrastructure (oracle side) — NOT product code.
//
// Thin command-line driver over the UNMODIFIED reference engine (linked from
// oracle/_ref/libpystachio_ref.a, built by oracle/build_ref.sh from /root/reference/proj/src).
// It only calls the reference's public API:
//   gen  -> pystachio::gen_workload            (/root/reference/proj/src/bench.cpp:85-114)
//   run  -> pystachio::run_socket_pipeline      (/root/reference/proj/src/pipeline_harness.cpp:81-109)
//           pystachio::run_sim_pipeline         (/root/reference/proj/src/pipeline_harness.cpp:23-79)
//   scanagg -> pystachio::read_blocking with a predicate (/root/reference/proj/src/scan.cpp:273-336,
//           set up like the reference's pybind `scan`, python/bindings.cpp:139-155), then the
//           global-aggregate sums of the surviving rows (HashAggregator::add semantics,
//           pipeline.cpp:275-294: int64 sums wrap mod 2^64, float64 sums add as doubles) - the
//           Q6-analog the reference's execute_plan cannot express
// and prints one JSON line with result checksums (rowhash = sum over rows of FNV-1a64 of the
// row's little-endian words) plus wall time, optionally dumping the raw rows.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "pystachio/bench.hpp"
#include "pystachio/hashing.hpp"
#include "pystachio/pipeline_harness.hpp"
#include "pystachio/join.hpp"
#include "pystachio/join_harness.hpp"
#include "pystachio/pipeline.hpp"
#include "pystachio/psto.hpp"
#include "pystachio/scan.hpp"

using namespace pystachio;

namespace {

std::string arg(int argc, char** argv, const std::string& key, const std::string& dflt) {
  for (int i = 1; i + 1 < argc; ++i)
    if (key == argv[i]) return argv[i + 1];
  return dflt;
}

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : s) {
    if (c == sep) {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur += c;
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

std::string read_file(const std::string& p) {
  std::ifstream in(p);
  if (!in) throw std::runtime_error("cannot open " + p);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

void summarize(const std::vector<std::vector<std::uint64_t>>& rows, std::size_t ncols, double secs,
               const std::vector<std::size_t>& per_node, const std::string& dump) {
  std::uint64_t rowhash = 0;
  std::vector<std::uint64_t> colsum(ncols, 0);
  for (const auto& r : rows) {
    rowhash += fnv1a64(r.data(), r.size() * 8);
    for (std::size_t c = 0; c < r.size() && c < ncols; ++c) colsum[c] += r[c];
  }
  std::printf("{\"rows\": %zu, \"ncols\": %zu, \"rowhash\": \"%016llx\", \"colsums\": [", rows.size(),
              ncols, static_cast<unsigned long long>(rowhash));
  for (std::size_t c = 0; c < ncols; ++c)
    std::printf("%s\"%llu\"", c ? ", " : "", static_cast<unsigned long long>(colsum[c]));
  std::printf("], \"per_node_rows\": [");
  for (std::size_t i = 0; i < per_node.size(); ++i) std::printf("%s%zu", i ? ", " : "", per_node[i]);
  std::printf("], \"seconds\": %.6f}\n", secs);
  if (!dump.empty()) {
    std::ofstream out(dump, std::ios::binary);
    std::uint64_t n = rows.size(), k = ncols;
    out.write(reinterpret_cast<const char*>(&n), 8);
    out.write(reinterpret_cast<const char*>(&k), 8);
    for (const auto& r : rows) out.write(reinterpret_cast<const char*>(r.data()), r.size() * 8);
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_driver gen|run [options]\n");
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "gen") {
      GenWorkloadSpec spec;
      spec.kind = arg(argc, argv, "--kind", "tpch") == "tpch" ? WorkloadKind::TpchAnalog
                                                               : WorkloadKind::SyntheticJoin;
      spec.out_dir = arg(argc, argv, "--out", "data");
      spec.scale = std::stod(arg(argc, argv, "--scale", "0.01"));
      spec.nodes = std::stoi(arg(argc, argv, "--nodes", "1"));
      spec.devices = std::stoi(arg(argc, argv, "--devices", std::to_string(spec.nodes)));
      spec.seed = std::stoull(arg(argc, argv, "--seed", "42"));
      spec.codec = codec_from_string(arg(argc, argv, "--codec", "identity"));
      spec.row_group_bytes = std::stoull(arg(argc, argv, "--rg-bytes", "1048576"));
      const auto t0 = std::chrono::steady_clock::now();
      const std::string manifest = gen_workload(spec);
      const double s =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      std::printf("{\"manifest\": \"%s\", \"seconds\": %.3f}\n", manifest.c_str(), s);
      return 0;
    }
    if (cmd == "run") {
      std::string plan = arg(argc, argv, "--plan-json", "");
      if (plan.empty()) plan = read_file(arg(argc, argv, "--plan", "plan.json"));
      const std::string data = arg(argc, argv, "--data", "data");
      const ExecMode mode = exec_mode_from_string(arg(argc, argv, "--mode", "overlapped"));
      const std::string backend = arg(argc, argv, "--backend", "socket");
      const int nodes = std::stoi(arg(argc, argv, "--nodes", "1"));
      const int repeat = std::stoi(arg(argc, argv, "--repeat", "1"));
      const std::string dump = arg(argc, argv, "--dump", "");
      for (int it = 0; it < repeat; ++it) {
        std::vector<std::vector<std::uint64_t>> rows;
        std::vector<std::size_t> per_node;
        std::size_t ncols = 0;
        const auto t0 = std::chrono::steady_clock::now();
        if (backend == "sim") {
          SimPipelineOptions opts;
          opts.plan_json = plan;
          opts.data_root = data;
          opts.nodes = nodes;
          opts.mode = mode;
          auto outcome = run_sim_pipeline(opts);
          for (const auto& r : outcome.per_node) {
            per_node.push_back(r.rows.size());
            ncols = std::max(ncols, r.schema.column_count());
            rows.insert(rows.end(), r.rows.begin(), r.rows.end());
          }
        } else {
          const std::uint16_t port =
              static_cast<std::uint16_t>(std::stoi(arg(argc, argv, "--port", "47011")));
          ClusterConfig cluster = ClusterConfig::loopback(1, port);
          auto r = run_socket_pipeline(plan, data, cluster, 0, mode);
          per_node.push_back(r.rows.size());
          ncols = r.schema.column_count();
          rows = std::move(r.rows);
        }
        const double s =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        summarize(rows, ncols, s, per_node, it == 0 ? dump : std::string());
        std::fflush(stdout);
      }
      return 0;
    }
    if (cmd == "scanagg") {
      // --paths a,b  --pred "col:op:value;..." (value with '.' = float literal)  --sums c1,c2
      const auto paths = split(arg(argc, argv, "--paths", ""), ',');
      const auto sums = split(arg(argc, argv, "--sums", ""), ',');
      const int repeat = std::stoi(arg(argc, argv, "--repeat", "1"));
      Predicate pred;
      for (const auto& a : split(arg(argc, argv, "--pred", ""), ';')) {
        const auto f = split(a, ':');
        if (f.size() != 3) throw std::runtime_error("bad --pred atom " + a);
        if (f[2].find('.') != std::string::npos)
          pred.and_atom(f[0], compare_op_from_string(f[1]), std::stod(f[2]));
        else
          pred.and_atom(f[0], compare_op_from_string(f[1]), static_cast<std::int64_t>(std::stoll(f[2])));
      }
      for (int it = 0; it < repeat; ++it) {
        const auto t0 = std::chrono::steady_clock::now();
        RealRuntime rt;
        Trace trace;
        MemoryPool pool;
        NodeExecState state;
        SimCostConfig cost;
        ExecEnv env{rt, trace, 0, pool, cost, StallFaultConfig{}, state};
        DeviceConfig cfg{"dev0", 0, 0, DeviceBacking::RealFile};
        DeviceModel dev(cfg);
        ScanOptions opts;
        opts.predicate = pred;
        std::uint64_t rows = 0;
        std::vector<std::uint64_t> isum(sums.size(), 0);
        std::vector<double> fsum(sums.size(), 0.0);
        std::vector<bool> is_float(sums.size(), false);
        for (const auto& path : paths) {
          ChunkBatch b = read_blocking(env, path, dev, opts);
          rows += b.row_count();
          for (std::size_t k = 0; k < sums.size(); ++k) {
            const Column& c = b.column(sums[k]);
            is_float[k] = c.type() == LogicalType::Float64;
            for (std::uint64_t w : c.raw()) {
              if (is_float[k]) {
                double d;
                std::memcpy(&d, &w, 8);
                fsum[k] += d;
              } else {
                isum[k] += w;
              }
            }
          }
        }
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::vector<std::vector<std::uint64_t>> out;
        if (rows) {
          std::vector<std::uint64_t> r{rows};
          for (std::size_t k = 0; k < sums.size(); ++k) {
            std::uint64_t w = isum[k];
            if (is_float[k]) std::memcpy(&w, &fsum[k], 8);
            r.push_back(w);
          }
          out.push_back(r);
        }
        summarize(out, 1 + sums.size(), s, {out.size()}, std::string());
        std::fflush(stdout);
      }
      return 0;
    }
    if (cmd == "joinplan") {
      // make_plan (join.cpp:126-134): the schedule as [[phase, stream, wave], ...]
      JoinSpec spec;
      spec.variant = join_variant_from_string(arg(argc, argv, "--variant", "deferred"));
      spec.stream_count = std::stoi(arg(argc, argv, "--streams", "2"));
      const int lw = std::stoi(arg(argc, argv, "--left", "1")), rw = std::stoi(arg(argc, argv, "--right", "1"));
      const SchedulePlan p = make_plan(spec, lw, rw);
      std::printf("[");
      for (std::size_t i = 0; i < p.steps.size(); ++i)
        std::printf("%s[%d, %d, %d]", i ? ", " : "", static_cast<int>(p.steps[i].phase), p.steps[i].stream,
                    p.steps[i].wave);
      std::printf("]\n");
      return 0;
    }
    if (cmd == "join") {
      // run_sim_join (join_harness.cpp:43-97): every node of the distributed join, rows collected
      SimJoinOptions opts;
      opts.spec.variant = join_variant_from_string(arg(argc, argv, "--variant", "deferred"));
      opts.spec.build_key = "bk";  // the synthetic workload's key columns (workload.cpp:44,57)
      opts.spec.probe_key = "pk";
      opts.spec.node_count = std::stoi(arg(argc, argv, "--nodes", "2"));
      opts.spec.stream_count = std::stoi(arg(argc, argv, "--streams", "2"));
      opts.spec.chunk_rows = std::stoull(arg(argc, argv, "--chunk-rows", "32768"));
      opts.workload.build_rows = std::stoull(arg(argc, argv, "--build-rows", "120000"));
      opts.workload.probe_rows = std::stoull(arg(argc, argv, "--probe-rows", "320000"));
      opts.workload.payload_cols = std::stoi(arg(argc, argv, "--payload", "3"));
      opts.workload.hit_ratio = std::stod(arg(argc, argv, "--hit-ratio", "0.5"));
      opts.workload.seed = std::stoull(arg(argc, argv, "--seed", "42"));
      const auto t0 = std::chrono::steady_clock::now();
      SimJoinOutcome out = run_sim_join(opts);
      const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      std::vector<std::size_t> per_node;
      for (const auto& st : out.per_node) per_node.push_back(st.result_rows);
      const std::size_t ncols = out.rows.empty() ? 0 : out.rows[0].size();
      summarize(out.rows, ncols, s, per_node, std::string());
      return 0;
    }
    if (cmd == "plan") {
      // QueryPlan::from_json_text (pipeline.cpp:108-156) for node --node of --nodes: the resolved
      // scans as JSON, or {"error": "<reference exception class>"}
      const std::string plan = arg(argc, argv, "--plan-json", "");
      const std::string data = arg(argc, argv, "--data", "data");
      const int node = std::stoi(arg(argc, argv, "--node", "0"));
      const int nodes = std::stoi(arg(argc, argv, "--nodes", "1"));
      auto q = [](const std::string& x) {
        std::string o = "\"";
        for (char ch : x) {
          if (ch == '"' || ch == '\\') o += '\\';
          o += ch;
        }
        return o + "\"";
      };
      try {
        const QueryPlan p = QueryPlan::from_json_text(plan, data, node, nodes);
        std::string j = "{\"scans\": [";
        for (std::size_t i = 0; i < p.scans.size(); ++i) {
          const ScanNode& sc = p.scans[i];
          j += (i ? ", " : "") + std::string("{\"table\": ") + q(sc.table) + ", \"replicated\": " +
               (sc.replicated ? "true" : "false") + ", \"paths\": [";
          for (std::size_t k = 0; k < sc.paths.size(); ++k) j += (k ? ", " : "") + q(sc.paths[k]);
          j += "]}";
        }
        const JoinNode* sj = p.shuffle_join();
        j += "], \"shuffle\": " + (sj ? q(sj->id) : std::string("null")) + "}";
        std::printf("%s\n", j.c_str());
      } catch (const InvalidInput&) {
        std::printf("{\"error\": \"InvalidInput\"}\n");
      } catch (const IoFailure&) {
        std::printf("{\"error\": \"IoFailure\"}\n");
      } catch (const UnknownColumn&) {
        std::printf("{\"error\": \"UnknownColumn\"}\n");
      } catch (const Error&) {
        std::printf("{\"error\": \"Error\"}\n");
      } catch (const std::exception&) {  // nlohmann::json exceptions (malformed / mistyped JSON)
        std::printf("{\"error\": \"json\"}\n");
      }
      return 0;
    }
    std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
