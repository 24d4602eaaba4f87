// gmio.cu -- the reference's file formats, host side.
//
// Host code only (compiled by nvcc into the same library; no kernels).  The
// formats and messages follow the reference:
//   text edge list, Matrix Market  src/io.cpp:85-182   (load_edge_list, load_matrix_market)
//   GMB1 binary                    src/io.cpp:290-362  (write_binary, read_binary)
//   "src dst value" writer         src/io.cpp:364-373  (write_edge_list)
//   results TSV, FNV-1a, report    src/report.cpp:21-102
// The implementation is ours: files are mapped once and parsed in place with
// std::from_chars (no iostreams); the text edge list is parsed by several
// threads over newline-aligned chunks and merged in file order, so results and
// the first reported error (path:line: message) are the same as a sequential
// scan; result files are formatted by several threads into per-chunk buffers
// and written in order (byte-identical output).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "api_internal.cuh"

namespace gm {
namespace io {
namespace {

[[noreturn]] void input_error(const std::string& msg) { fail(GM_EINPUT, msg); }

[[noreturn]] void fail_at(const std::string& path, uint64_t line_no, const std::string& msg) {
  input_error(path + ":" + std::to_string(line_no) + ": " + msg);
}

// Read-only mapping of a whole file (empty files map to an empty view).
class Mapped {
 public:
  explicit Mapped(const std::string& path) {
    fd_ = ::open(path.c_str(), O_RDONLY);
    if (fd_ < 0) return;
    struct stat st;
    if (::fstat(fd_, &st) != 0) return;
    size_ = size_t(st.st_size);
    if (size_ == 0) {
      ok_ = true;
      return;
    }
    void* p = ::mmap(nullptr, size_, PROT_READ, MAP_PRIVATE, fd_, 0);
    if (p == MAP_FAILED) return;
    ::madvise(p, size_, MADV_SEQUENTIAL);
    data_ = static_cast<const char*>(p);
    ok_ = true;
  }
  ~Mapped() {
    if (data_) ::munmap(const_cast<char*>(data_), size_);
    if (fd_ >= 0) ::close(fd_);
  }
  Mapped(const Mapped&) = delete;
  Mapped& operator=(const Mapped&) = delete;
  bool ok() const { return ok_; }
  std::string_view view() const { return std::string_view(data_ ? data_ : "", size_); }

 private:
  int fd_ = -1;
  const char* data_ = nullptr;
  size_t size_ = 0;
  bool ok_ = false;
};

inline bool is_space(char c) {  // isspace in the C locale
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// Splits a line on whitespace into at most kMax tokens; returns the count
// (which may exceed kMax: extra tokens are counted, not stored).
constexpr int kMaxTok = 6;
int tokens(std::string_view line, std::string_view* out) {
  int n = 0;
  size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && is_space(line[i])) ++i;
    size_t j = i;
    while (j < line.size() && !is_space(line[j])) ++j;
    if (j > i) {
      if (n < kMaxTok) out[n] = line.substr(i, j - i);
      ++n;
    }
    i = j;
  }
  return n;
}

bool comment_or_blank(std::string_view line) {
  for (const char c : line) {
    if (is_space(c)) continue;
    return c == '#' || c == '%';
  }
  return true;
}

bool parse_u64(std::string_view t, uint64_t& v) {
  const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc{} && r.ptr == t.data() + t.size();
}

bool parse_f64(std::string_view t, double& v) {
  const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc{} && r.ptr == t.data() + t.size();
}

std::string lower(std::string_view s) {
  std::string o(s);
  for (char& c : o)
    if (c >= 'A' && c <= 'Z') c = char(c - 'A' + 'a');
  return o;
}

// Line iterator with getline semantics: '\n' separated, a final unterminated
// line counts, a trailing '\n' does not open an empty line.
struct Lines {
  std::string_view buf;
  size_t pos = 0;
  bool next(std::string_view& line) {
    if (pos >= buf.size()) return false;
    const size_t e = buf.find('\n', pos);
    const size_t end = e == std::string_view::npos ? buf.size() : e;
    line = buf.substr(pos, end - pos);
    pos = end == buf.size() ? end : end + 1;
    return true;
  }
};

struct ChunkResult {
  std::vector<uint64_t> src, dst;
  std::vector<double> val;
  uint64_t lines = 0, max_id = 0;
  bool failed = false;
  uint64_t fail_line = 0;  // 1-based within the chunk
  std::string msg;
};

void parse_edge_chunk(std::string_view chunk, bool weighted, ChunkResult& r) {
  Lines it{chunk};
  std::string_view line, tok[kMaxTok];
  const int expected = weighted ? 3 : 2;
  auto bad = [&](const std::string& m) {
    r.failed = true;
    r.fail_line = r.lines;
    r.msg = m;
  };
  while (it.next(line)) {
    ++r.lines;
    if (comment_or_blank(line)) continue;
    const int nt = tokens(line, tok);
    if (nt != expected) {
      if (!weighted && nt == 3)
        bad("unexpected weight column on an unweighted load");
      else
        bad("expected " + std::to_string(expected) + " columns, got " + std::to_string(nt));
      return;
    }
    uint64_t s = 0, d = 0;
    if (!parse_u64(tok[0], s)) return bad("malformed source id '" + std::string(tok[0]) + "'");
    if (!parse_u64(tok[1], d)) return bad("malformed destination id '" + std::string(tok[1]) + "'");
    if (s == 0 || d == 0) return bad("vertex ids are 1-based and positive");
    double v = 1.0;
    if (weighted && !parse_f64(tok[2], v)) return bad("malformed weight '" + std::string(tok[2]) + "'");
    r.src.push_back(s - 1);
    r.dst.push_back(d - 1);
    r.val.push_back(v);
    r.max_id = std::max(r.max_id, std::max(s, d));
  }
}

unsigned io_threads(size_t bytes) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t per = size_t(4) << 20;  // >= 4 MB per thread
  return unsigned(std::max<size_t>(1, std::min<size_t>(hw, (bytes + per - 1) / per)));
}

template <typename F>
void parallel_for(unsigned nt, F&& f) {
  if (nt <= 1) {
    f(0u);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(nt);
  for (unsigned t = 0; t < nt; ++t) th.emplace_back([&f, t] { f(t); });
  for (auto& x : th) x.join();
}

void put_u64_le(char* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = char((v >> (8 * i)) & 0xFF);
}

uint64_t get_u64_le(const char* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= uint64_t(static_cast<unsigned char>(p[i])) << (8 * i);
  return v;
}

class Out {
 public:
  Out(const std::string& path, const char* what) : path_(path) {
    f_ = std::fopen(path.c_str(), "wb");
    if (!f_) input_error("cannot open '" + path + "' for " + what);
  }
  ~Out() {
    if (f_) std::fclose(f_);
  }
  void write(const char* p, size_t n) {
    if (n && std::fwrite(p, 1, n, f_) != n) ok_ = false;
  }
  void write(const std::string& s) { write(s.data(), s.size()); }
  void close() {
    if (std::fclose(f_) != 0) ok_ = false;
    f_ = nullptr;
    if (!ok_) input_error("write failed on '" + path_ + "'");
  }

 private:
  std::string path_;
  std::FILE* f_ = nullptr;
  bool ok_ = true;
};

// "%.17g" of the reference's format_real (report.cpp:21-25).
inline int fmt_real(char* buf, size_t cap, double v) { return std::snprintf(buf, cap, "%.17g", v); }

// Rows [0, n) formatted by `line(i, out)` in parallel chunks, written in order.
template <typename F>
void write_lines(Out& out, uint64_t n, uint64_t bytes_hint, F&& line) {
  const unsigned nt = io_threads(bytes_hint);
  std::vector<std::string> parts(nt);
  parallel_for(nt, [&](unsigned t) {
    const uint64_t b = n * t / nt, e = n * (t + 1) / nt;
    std::string& s = parts[t];
    s.reserve(size_t((e - b) * (bytes_hint / std::max<uint64_t>(n, 1) + 8)));
    for (uint64_t i = b; i < e; ++i) line(i, s);
  });
  for (auto& p : parts) out.write(p);
}

}  // namespace

EdgeBuffer load_edge_list(const std::string& path, bool weighted) {
  Mapped f(path);
  if (!f.ok()) input_error("cannot open '" + path + "'");
  const std::string_view buf = f.view();
  // newline-aligned chunks
  const unsigned nt = io_threads(buf.size());
  std::vector<size_t> cut(nt + 1, buf.size());
  cut[0] = 0;
  for (unsigned t = 1; t < nt; ++t) {
    size_t p = std::max(cut[t - 1], buf.size() * t / nt);
    const size_t e = buf.find('\n', p);
    cut[t] = e == std::string_view::npos ? buf.size() : e + 1;
  }
  std::vector<ChunkResult> res(nt);
  parallel_for(nt, [&](unsigned t) {
    parse_edge_chunk(buf.substr(cut[t], cut[t + 1] - cut[t]), weighted, res[t]);
  });
  EdgeBuffer out;
  uint64_t lines_before = 0, total = 0;
  for (unsigned t = 0; t < nt; ++t) {
    if (res[t].failed) fail_at(path, lines_before + res[t].fail_line, res[t].msg);
    lines_before += res[t].lines;
    total += res[t].src.size();
  }
  out.src.reserve(total);
  out.dst.reserve(total);
  out.val.reserve(total);
  for (auto& r : res) {
    out.src.insert(out.src.end(), r.src.begin(), r.src.end());
    out.dst.insert(out.dst.end(), r.dst.begin(), r.dst.end());
    out.val.insert(out.val.end(), r.val.begin(), r.val.end());
    out.num_vertices = std::max(out.num_vertices, r.max_id);
  }
  return out;
}

EdgeBuffer load_matrix_market(const std::string& path) {
  Mapped f(path);
  if (!f.ok()) input_error("cannot open '" + path + "'");
  Lines it{f.view()};
  std::string_view line, tok[kMaxTok];
  uint64_t line_no = 0;
  if (!it.next(line)) input_error(path + ": empty file");
  ++line_no;
  int nt = tokens(line, tok);
  if (nt < 5 || lower(tok[0]) != "%%matrixmarket" || lower(tok[1]) != "matrix")
    fail_at(path, line_no, "not a Matrix Market matrix header");
  if (lower(tok[2]) != "coordinate")
    fail_at(path, line_no, "unsupported layout '" + std::string(tok[2]) + "' (only coordinate)");
  const std::string field = lower(tok[3]);
  if (field != "real" && field != "pattern" && field != "integer")
    fail_at(path, line_no,
            "unsupported field '" + std::string(tok[3]) + "' (real, pattern, integer)");
  const std::string symmetry = lower(tok[4]);
  if (symmetry != "general" && symmetry != "symmetric")
    fail_at(path, line_no,
            "unsupported symmetry '" + std::string(tok[4]) + "' (general, symmetric)");
  const bool pattern = field == "pattern", symmetric = symmetry == "symmetric";
  uint64_t rows = 0, cols = 0, declared = 0;
  bool have_size = false;
  while (it.next(line)) {
    ++line_no;
    if (comment_or_blank(line)) continue;
    if (tokens(line, tok) != 3) fail_at(path, line_no, "expected 'rows cols nnz' size line");
    if (!parse_u64(tok[0], rows))
      fail_at(path, line_no, "malformed row count '" + std::string(tok[0]) + "'");
    if (!parse_u64(tok[1], cols))
      fail_at(path, line_no, "malformed column count '" + std::string(tok[1]) + "'");
    if (!parse_u64(tok[2], declared))
      fail_at(path, line_no, "malformed entry count '" + std::string(tok[2]) + "'");
    have_size = true;
    break;
  }
  if (!have_size) input_error(path + ": missing size line");
  EdgeBuffer out;
  out.num_vertices = std::max(rows, cols);
  const int expected = pattern ? 2 : 3;
  uint64_t seen = 0;
  while (seen < declared && it.next(line)) {
    ++line_no;
    if (comment_or_blank(line)) continue;
    nt = tokens(line, tok);
    if (nt != expected)
      fail_at(path, line_no,
              "expected " + std::to_string(expected) + " columns, got " + std::to_string(nt));
    uint64_t i = 0, j = 0;
    if (!parse_u64(tok[0], i)) fail_at(path, line_no, "malformed row id '" + std::string(tok[0]) + "'");
    if (!parse_u64(tok[1], j))
      fail_at(path, line_no, "malformed column id '" + std::string(tok[1]) + "'");
    if (i == 0 || i > rows || j == 0 || j > cols)
      fail_at(path, line_no, "entry (" + std::to_string(i) + ", " + std::to_string(j) +
                                 ") outside declared " + std::to_string(rows) + " x " +
                                 std::to_string(cols) + " shape");
    double v = 1.0;
    if (!pattern && !parse_f64(tok[2], v))
      fail_at(path, line_no, "malformed value '" + std::string(tok[2]) + "'");
    out.src.push_back(i - 1);
    out.dst.push_back(j - 1);
    out.val.push_back(v);
    if (symmetric && i != j) {
      out.src.push_back(j - 1);
      out.dst.push_back(i - 1);
      out.val.push_back(v);
    }
    ++seen;
  }
  if (seen < declared)
    input_error(path + ": truncated — " + std::to_string(declared) + " entries declared, " +
                std::to_string(seen) + " found");
  while (it.next(line)) {
    ++line_no;
    if (!comment_or_blank(line))
      fail_at(path, line_no, "data past the declared " + std::to_string(declared) + " entries");
  }
  return out;
}

EdgeBuffer read_binary(const std::string& path) {
  Mapped f(path);
  if (!f.ok()) input_error("cannot open '" + path + "'");
  const std::string_view b = f.view();
  if (b.size() < 20) input_error(path + ": truncated header (not a graph binary?)");
  if (std::memcmp(b.data(), "GMB1", 4) != 0) input_error(path + ": bad magic, not a graph binary");
  EdgeBuffer out;
  out.num_vertices = get_u64_le(b.data() + 4);
  const uint64_t m = get_u64_le(b.data() + 12);
  const uint64_t payload = b.size() - 20;
  if (payload % 24 != 0 || m != payload / 24)
    input_error(path + ": size mismatch — header declares " + std::to_string(m) +
                " edges, file has " + std::to_string(payload) + " payload bytes (" +
                std::to_string(payload / 24) + " records)");
  out.src.resize(m);
  out.dst.resize(m);
  out.val.resize(m);
  const char* p = b.data() + 20;
  const unsigned nt = io_threads(payload);
  parallel_for(nt, [&](unsigned t) {
    const uint64_t lo = m * t / nt, hi = m * (t + 1) / nt;
    for (uint64_t e = lo; e < hi; ++e) {
      const char* r = p + 24 * e;
      out.src[e] = get_u64_le(r);
      out.dst[e] = get_u64_le(r + 8);
      const uint64_t bits = get_u64_le(r + 16);
      std::memcpy(&out.val[e], &bits, 8);
    }
  });
  return out;
}

void write_binary(const std::string& path, const uint64_t* src, const uint64_t* dst,
                  const double* val, uint64_t m, uint64_t n) {
  Out out(path, "writing");
  char hdr[20];
  std::memcpy(hdr, "GMB1", 4);
  put_u64_le(hdr + 4, n);
  put_u64_le(hdr + 12, m);
  out.write(hdr, 20);
  constexpr uint64_t kBatch = uint64_t(1) << 16;
  std::vector<char> buf(24 * kBatch);
  for (uint64_t b = 0; b < m; b += kBatch) {
    const uint64_t e = std::min(m, b + kBatch);
    for (uint64_t i = b; i < e; ++i) {
      char* r = buf.data() + 24 * (i - b);
      uint64_t bits = 0;
      const double v = val ? val[i] : 1.0;
      std::memcpy(&bits, &v, 8);
      put_u64_le(r, src[i]);
      put_u64_le(r + 8, dst[i]);
      put_u64_le(r + 16, bits);
    }
    out.write(buf.data(), size_t(24 * (e - b)));
  }
  out.close();
}

void write_edge_list(const std::string& path, const uint64_t* src, const uint64_t* dst,
                     const double* val, uint64_t m) {
  Out out(path, "writing");
  write_lines(out, m, m * 24, [&](uint64_t i, std::string& s) {
    char num[64];
    s += std::to_string(src[i] + 1);
    s += ' ';
    s += std::to_string(dst[i] + 1);
    s += ' ';
    s.append(num, size_t(fmt_real(num, sizeof num, val ? val[i] : 1.0)));
    s += '\n';
  });
  out.close();
}

void write_results(const std::string& path, const double* values, uint64_t n) {
  Out out(path, "writing");
  write_lines(out, n, n * 28, [&](uint64_t v, std::string& s) {
    char num[64];
    s += std::to_string(v + 1);
    s += '\t';
    s.append(num, size_t(fmt_real(num, sizeof num, values[v])));
    s += '\n';
  });
  out.close();
}

void write_vector_results(const std::string& path, const double* rows, uint64_t n, uint64_t k) {
  Out out(path, "writing");
  write_lines(out, n, n * (8 + 24 * k), [&](uint64_t v, std::string& s) {
    char num[64];
    s += std::to_string(v + 1);
    for (uint64_t j = 0; j < k; ++j) {
      s += '\t';
      s.append(num, size_t(fmt_real(num, sizeof num, rows[v * k + j])));
    }
    s += '\n';
  });
  out.close();
}

void write_report(const std::string& path, const gm_run_report& r) {
  Out out(path, "writing");
  std::string s;
  char buf[64];
  s += "algorithm=" + std::string(r.algorithm ? r.algorithm : "") + "\n";
  s += "graph=" + std::string(r.graph ? r.graph : "") + "\n";
  s += "threads=" + std::to_string(r.threads) + "\n";
  s += "partitions=" + std::to_string(r.partitions) + "\n";
  s += "iterations=" + std::to_string(r.n_iterations) + "\n";
  s += "iteration_seconds=";
  for (uint64_t i = 0; i < r.n_iterations; ++i) {
    std::snprintf(buf, sizeof buf, "%.9g", r.iteration_seconds[i]);
    s += (i == 0 ? "" : ",");
    s += buf;
  }
  s += "\n";
  std::snprintf(buf, sizeof buf, "%.9g", r.total_seconds);
  s += "total_seconds=" + std::string(buf) + "\n";
  if (r.n_iterations == 0) {
    s += "seconds_per_iteration=na\n";
  } else {
    std::snprintf(buf, sizeof buf, "%.9g", r.total_seconds / double(r.n_iterations));
    s += "seconds_per_iteration=" + std::string(buf) + "\n";
  }
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(r.checksum));
  s += "checksum=" + std::string(buf) + "\n";
  for (uint64_t i = 0; i < r.n_extras; ++i)
    s += std::string(r.extra_keys[i]) + "=" + std::string(r.extra_values[i]) + "\n";
  out.write(s);
  out.close();
}

uint64_t fnv1a64(const void* data, uint64_t size) {
  const auto* p = static_cast<const unsigned char*>(data);
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < size; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

uint64_t fnv1a64_file(const std::string& path) {
  Mapped f(path);
  if (!f.ok()) input_error("cannot open '" + path + "' for checksumming");
  const std::string_view b = f.view();
  return fnv1a64(b.data(), b.size());
}

}  // namespace io
}  // namespace gm
