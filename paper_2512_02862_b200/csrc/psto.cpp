#include "psto.hpp"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>
#include <zlib.h>

#include <algorithm>
#include <cstring>

namespace psg {

namespace {
constexpr char kMagic[4] = {'P', 'S', 'T', 'O'};

struct Cursor {
  const uint8_t* p;
  size_t n, off = 0;
  const uint8_t* take(size_t k) {
    if (off + k > n) throw CorruptFooter("footer truncated");
    const uint8_t* r = p + off;
    off += k;
    return r;
  }
  template <class T>
  T get() {
    T v;
    std::memcpy(&v, take(sizeof(T)), sizeof(T));
    return v;
  }
};

template <class T>
bool zone_ok(const ChunkMeta& c) {
  T lo, hi;
  std::memcpy(&lo, &c.min_raw, 8);
  std::memcpy(&hi, &c.max_raw, 8);
  return !(lo > hi);
}

template <class T>
bool interval(T lo, T hi, CmpOp op, T lit) {
  switch (op) {
    case CmpOp::Lt: return lo < lit;
    case CmpOp::Le: return lo <= lit;
    case CmpOp::Eq: return lo <= lit && lit <= hi;
    case CmpOp::Ne: return !(lo == lit && hi == lit);
    case CmpOp::Ge: return hi >= lit;
    case CmpOp::Gt: return hi > lit;
  }
  return true;
}
}  // namespace

TableMeta parse_footer_bytes(const uint8_t* tail, size_t tail_len, uint64_t file_size, uint64_t tail_offset) {
  if (tail_len < 12) throw CorruptFooter("file shorter than the footer trailer");
  if (std::memcmp(tail + tail_len - 4, kMagic, 4) != 0) throw CorruptFooter("bad tail magic");
  uint64_t flen;
  std::memcpy(&flen, tail + tail_len - 12, 8);
  if (flen + 16 > file_size) throw CorruptFooter("footer length exceeds file size");
  if (flen + 12 > tail_len) throw CorruptFooter("tail read misses the footer");
  Cursor r{tail + tail_len - 12 - flen, flen};
  TableMeta m;
  if (r.get<uint32_t>() != 1) throw CorruptFooter("unsupported footer version");
  const uint8_t codec = r.get<uint8_t>();
  if (codec > 1) throw CorruptFooter("unknown codec tag");
  m.codec = static_cast<Codec>(codec);
  const uint32_t ncols = r.get<uint32_t>();
  for (uint32_t c = 0; c < ncols; ++c) {
    const uint32_t len = r.get<uint32_t>();
    if (len > 4096) throw CorruptFooter("implausible name length");
    Field f;
    f.name.assign(reinterpret_cast<const char*>(r.take(len)), len);
    const uint8_t t = r.get<uint8_t>();
    if (t > 1) throw CorruptFooter("unknown logical type");
    f.type = static_cast<LType>(t);
    m.schema.fields.push_back(std::move(f));
  }
  const uint32_t ng = r.get<uint32_t>();
  const uint64_t data_end = tail_offset + tail_len - 12 - flen;
  // every group record is 8 + 40 bytes per column: bound the count by what the footer holds
  // before allocating (a corrupt count must not allocate gigabytes)
  if (static_cast<uint64_t>(ng) * (8 + 40ull * ncols) > r.n - r.off) throw CorruptFooter("row-group count exceeds footer");
  m.groups.resize(ng);
  for (uint32_t g = 0; g < ng; ++g) {
    GroupMeta& gm = m.groups[g];
    gm.rows = r.get<uint64_t>();
    gm.cols.resize(ncols);
    for (uint32_t c = 0; c < ncols; ++c) {
      ChunkMeta& ch = gm.cols[c];
      ch.offset = r.get<uint64_t>();
      ch.csize = r.get<uint64_t>();
      ch.usize = r.get<uint64_t>();
      ch.min_raw = r.get<uint64_t>();
      ch.max_raw = r.get<uint64_t>();
      // (written without offset + csize, which can wrap)
      if (ch.offset < 4 || ch.offset > data_end || ch.csize > data_end - ch.offset)
        throw CorruptFooter("column chunk outside file bounds");
      if (gm.rows > (~0ULL) / kValueBytes || ch.usize != gm.rows * kValueBytes)
        throw CorruptFooter("uncompressed size disagrees with row count");
      // identity chunks are read in place by the fused kernels (rows * 8 bytes from the offset)
      if (m.codec == Codec::Identity && ch.csize != ch.usize)
        throw CorruptFooter("identity chunk size disagrees with its row count");
      const bool ok = m.schema.fields[c].type == LType::Int64 ? zone_ok<int64_t>(ch) : zone_ok<double>(ch);
      if (gm.rows > 0 && !ok) throw CorruptFooter("zone stats inverted");
    }
  }
  if (r.off != r.n) throw CorruptFooter("trailing bytes in footer");
  m.summarise();
  m.footer_bytes = flen;
  m.file_size = file_size;
  return m;
}

TableMeta read_footer(const std::string& path) {
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) throw IoFailure("cannot open: " + path);
  struct stat st;
  if (::fstat(fd, &st) != 0) {
    ::close(fd);
    throw IoFailure("cannot stat: " + path);
  }
  const uint64_t size = static_cast<uint64_t>(st.st_size);
  auto rd = [&](uint64_t off, uint64_t len, uint8_t* dst) {
    uint64_t got = 0;
    while (got < len) {
      ssize_t k = ::pread(fd, dst + got, len - got, static_cast<off_t>(off + got));
      if (k <= 0) {
        ::close(fd);
        throw IoFailure("short read: " + path);
      }
      got += static_cast<uint64_t>(k);
    }
  };
  if (size < 20) {
    ::close(fd);
    throw CorruptFooter("file too small");
  }
  uint8_t head[4];
  rd(0, 4, head);
  if (std::memcmp(head, kMagic, 4) != 0) {
    ::close(fd);
    throw CorruptFooter("bad head magic");
  }
  uint8_t trailer[12];
  rd(size - 12, 12, trailer);
  uint64_t flen;
  std::memcpy(&flen, trailer, 8);
  if (flen + 16 > size) {
    ::close(fd);
    throw CorruptFooter("footer length exceeds file size");
  }
  std::vector<uint8_t> tail(flen + 12);
  rd(size - 12 - flen, flen + 12, tail.data());
  ::close(fd);
  return parse_footer_bytes(tail.data(), tail.size(), size, size - 12 - flen);
}

std::vector<uint8_t> encode_footer(const TableMeta& m) {
  std::vector<uint8_t> b;
  auto put = [&](const void* p, size_t n) {
    const auto* q = static_cast<const uint8_t*>(p);
    b.insert(b.end(), q, q + n);
  };
  const uint32_t ver = 1, nc = static_cast<uint32_t>(m.schema.size()),
                 ng = static_cast<uint32_t>(m.groups.size());
  const uint8_t codec = static_cast<uint8_t>(m.codec);
  put(&ver, 4);
  put(&codec, 1);
  put(&nc, 4);
  for (auto& f : m.schema.fields) {
    const uint32_t len = static_cast<uint32_t>(f.name.size());
    const uint8_t t = static_cast<uint8_t>(f.type);
    put(&len, 4);
    put(f.name.data(), len);
    put(&t, 1);
  }
  put(&ng, 4);
  for (auto& g : m.groups) {
    put(&g.rows, 8);
    for (auto& c : g.cols) put(&c, sizeof(ChunkMeta));
  }
  return b;
}

std::vector<size_t> prune(const TableMeta& m, const Predicate& pred) {
  std::vector<size_t> keep;
  std::vector<size_t> idx;
  for (auto& a : pred) idx.push_back(m.schema.require(a.column));
  for (size_t g = 0; g < m.groups.size(); ++g) {
    bool may = true;
    for (size_t i = 0; i < pred.size() && may; ++i) {
      const ChunkMeta& c = m.groups[g].cols[idx[i]];
      if (m.schema.fields[idx[i]].type == LType::Int64) {
        int64_t lo, hi;
        std::memcpy(&lo, &c.min_raw, 8);
        std::memcpy(&hi, &c.max_raw, 8);
        may = interval<int64_t>(lo, hi, pred[i].op, pred[i].as_int());
      } else {
        double lo, hi;
        std::memcpy(&lo, &c.min_raw, 8);
        std::memcpy(&hi, &c.max_raw, 8);
        may = interval<double>(lo, hi, pred[i].op, pred[i].as_float());
      }
    }
    if (may) keep.push_back(g);
  }
  return keep;
}

PstoWriter::PstoWriter(const std::string& path, Schema schema, uint64_t rg_rows, Codec codec)
    : path_(path), schema_(std::move(schema)), rg_rows_(rg_rows), codec_(codec) {
  if (rg_rows_ < 1) throw InvalidInput("row_group_rows must be >= 1");
  fd_ = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd_ < 0) throw IoFailure("cannot open for writing: " + path);
  write_bytes(kMagic, 4);
  pending_.resize(schema_.size());
  meta_.schema = schema_;
  meta_.codec = codec_;
}

PstoWriter::~PstoWriter() {
  if (fd_ >= 0) ::close(fd_);
}

void PstoWriter::write_bytes(const void* p, size_t n) {
  const auto* q = static_cast<const uint8_t*>(p);
  size_t done = 0;
  while (done < n) {
    ssize_t k = ::write(fd_, q + done, n - done);
    if (k <= 0) throw IoFailure("write failed: " + path_);
    done += static_cast<size_t>(k);
  }
  offset_ += n;
}

void PstoWriter::write_group(const uint64_t* const* cols, uint64_t n) {
  GroupMeta g;
  g.rows = n;
  for (size_t c = 0; c < schema_.size(); ++c) {
    ChunkMeta ch;
    ch.offset = offset_;
    ch.usize = n * kValueBytes;
    const uint64_t* w = cols[c];
    if (n > 0) {
      if (schema_.fields[c].type == LType::Int64) {
        int64_t lo, hi;
        std::memcpy(&lo, &w[0], 8);
        hi = lo;
        for (uint64_t i = 1; i < n; ++i) {
          int64_t v;
          std::memcpy(&v, &w[i], 8);
          lo = std::min(lo, v);
          hi = std::max(hi, v);
        }
        std::memcpy(&ch.min_raw, &lo, 8);
        std::memcpy(&ch.max_raw, &hi, 8);
      } else {
        double lo, hi;
        std::memcpy(&lo, &w[0], 8);
        hi = lo;
        for (uint64_t i = 1; i < n; ++i) {
          double v;
          std::memcpy(&v, &w[i], 8);
          lo = std::min(lo, v);
          hi = std::max(hi, v);
        }
        std::memcpy(&ch.min_raw, &lo, 8);
        std::memcpy(&ch.max_raw, &hi, 8);
      }
    }
    if (codec_ == Codec::Identity) {
      ch.csize = n * kValueBytes;
      write_bytes(w, ch.csize);
    } else {
      uLongf bound = compressBound(static_cast<uLong>(n * kValueBytes));
      outbuf_.resize(bound);
      if (compress2(outbuf_.data(), &bound, reinterpret_cast<const Bytef*>(w), static_cast<uLong>(n * kValueBytes), 1) != Z_OK)
        throw IoFailure("deflate failed");
      ch.csize = bound;
      write_bytes(outbuf_.data(), bound);
    }
    g.cols.push_back(ch);
  }
  meta_.groups.push_back(std::move(g));
}

void PstoWriter::flush_pending(uint64_t rows) {
  std::vector<const uint64_t*> ptrs(schema_.size());
  for (size_t c = 0; c < schema_.size(); ++c) ptrs[c] = pending_[c].data();
  write_group(ptrs.data(), rows);
  for (auto& col : pending_) col.erase(col.begin(), col.begin() + static_cast<std::ptrdiff_t>(rows));
}

void PstoWriter::append(const uint64_t* const* cols, uint64_t n) {
  for (size_t c = 0; c < schema_.size(); ++c) pending_[c].insert(pending_[c].end(), cols[c], cols[c] + n);
  while (!pending_.empty() && pending_[0].size() >= rg_rows_) flush_pending(rg_rows_);
}

TableMeta PstoWriter::finish() {
  if (finished_) throw IoFailure("finish() called twice");
  finished_ = true;
  if (!pending_.empty() && !pending_[0].empty()) flush_pending(pending_[0].size());
  auto footer = encode_footer(meta_);
  write_bytes(footer.data(), footer.size());
  const uint64_t flen = footer.size();
  write_bytes(&flen, 8);
  write_bytes(kMagic, 4);
  if (::close(fd_) != 0) {
    fd_ = -1;
    throw IoFailure("write failed: " + path_);
  }
  fd_ = -1;
  meta_.footer_bytes = flen;
  meta_.summarise();
  return meta_;
}

}  // namespace psg
