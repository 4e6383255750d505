// PSTO columnar file format — our own reader/writer written from the format contract:
//   [magic "PSTO"][row-group column chunks ...][footer][u64 footer_len]["PSTO"]   (psto.hpp:13-16)
// footer = u32 version(1), u8 codec, u32 ncols, ncols x (u32 len, name, u8 type), u32 ngroups,
//          ngroups x (u64 rows, ncols x 5 x u64 {offset, csize, usize, min_raw, max_raw})
// (encode_footer psto.cpp:192-213, parse_footer_bytes :231-292, prune :320-343).
#pragma once

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"

namespace psg {

enum class Codec : uint8_t { Identity = 0, Block = 1 };

struct ChunkMeta {
  uint64_t offset = 0, csize = 0, usize = 0, min_raw = 0, max_raw = 0;
};
struct GroupMeta {
  uint64_t rows = 0;
  std::vector<ChunkMeta> cols;
};
struct TableMeta {
  Schema schema;
  Codec codec = Codec::Identity;
  std::vector<GroupMeta> groups;
  uint64_t footer_bytes = 0;
  uint64_t file_size = 0;
  // whole-file summaries of the zone maps (filled once per parsed footer, so the planner's range
  // questions cost one lookup per file instead of a walk over every row group): rows, and per
  // column the min/max of the raw words read as signed integers over the non-empty groups
  // (zmin > zmax when the file has no rows)
  uint64_t nrows = 0;
  std::vector<int64_t> zmin, zmax;
  uint64_t total_rows() const { return nrows; }
  void summarise() {
    nrows = 0;
    const size_t nc = schema.size();
    zmin.assign(nc, INT64_MAX);
    zmax.assign(nc, INT64_MIN);
    for (const auto& g : groups) {
      nrows += g.rows;
      if (!g.rows) continue;
      for (size_t c = 0; c < nc && c < g.cols.size(); ++c) {
        zmin[c] = std::min(zmin[c], static_cast<int64_t>(g.cols[c].min_raw));
        zmax[c] = std::max(zmax[c], static_cast<int64_t>(g.cols[c].max_raw));
      }
    }
  }
};

/// Parses the footer from the file tail (validates magic, bounds, sizes, zone order).
TableMeta parse_footer_bytes(const uint8_t* tail, size_t tail_len, uint64_t file_size, uint64_t tail_offset);
TableMeta read_footer(const std::string& path);
std::vector<uint8_t> encode_footer(const TableMeta& meta);
/// Row groups whose [min,max] zones may satisfy every atom (never drops a qualifying group).
std::vector<size_t> prune(const TableMeta& meta, const Predicate& pred);

/// Streaming writer: append rows column-major, flush row groups of row_group_rows.
class PstoWriter {
 public:
  PstoWriter(const std::string& path, Schema schema, uint64_t row_group_rows, Codec codec);
  ~PstoWriter();
  /// Appends n rows given per-column word pointers.
  void append(const uint64_t* const* cols, uint64_t n);
  /// Appends one already-formed row group (cols[c] holds n words).
  void write_group(const uint64_t* const* cols, uint64_t n);
  TableMeta finish();
  static uint64_t rows_for_group_bytes(const Schema& s, uint64_t bytes) {
    const uint64_t row = s.size() * kValueBytes;
    return std::max<uint64_t>(1, bytes / std::max<uint64_t>(row, 1));
  }

 private:
  std::string path_;
  Schema schema_;
  uint64_t rg_rows_;
  Codec codec_;
  int fd_ = -1;
  uint64_t offset_ = 0;
  std::vector<std::vector<uint64_t>> pending_;
  std::vector<uint8_t> outbuf_;
  TableMeta meta_;
  bool finished_ = false;
  void flush_pending(uint64_t rows);
  void write_bytes(const void* p, size_t n);
};

}  // namespace psg
