// Matrix Market I/O behind pdb_matrix_read_matrix_market /
// pdb_matrix_write_matrix_market / pdb_export_matrix.
//
// The accepted subset, the status codes and the messages are the
// reference's (matrix_market.cpp:29-110): real coordinate matrices, general
// or symmetric (mirrored entries appended after the original), 1-based
// indices, blank lines skipped, comment lines only before the size line,
// "<name>: line <k>: <what>" parse errors.  The implementation is its own:
// the file is read into memory in one call, the header is scanned in place,
// and the entry section is split at line boundaries into chunks that are
// tokenised in parallel; a sequential merge then walks the chunks in file
// order so the first error among the first nnz entries -- or the missing
// entries -- is reported at the line the sequential reader would report.
// Tokens are read with the rules of istream extraction (leading
// whitespace skipped, the longest numeric prefix taken, the rest of the line
// ignored; reals converted by strtod as libstdc++'s num_get does and
// rejected when they overflow), so the same files fail with the same
// messages.  CSR assembly (sparse.cpp:12-48) is a stable counting sort by
// row, a stable sort by column inside each row, and duplicates summed in
// input order.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "host.hpp"

namespace pdb {

namespace {

struct Entry {
  Index r, c;
  double v;
};

inline bool skip_char(char ch) {  // istream's whitespace (isspace in the "C" locale)
  return ch == ' ' || ch == '\t' || ch == '\n' || ch == '\v' || ch == '\f' || ch == '\r';
}

// the reference's blank(): only " \t\r\n" count
bool blank_line(const char* b, const char* e) {
  for (; b < e; ++b)
    if (*b != ' ' && *b != '\t' && *b != '\r' && *b != '\n') return false;
  return true;
}

std::string word(const char*& p, const char* e) {
  while (p < e && skip_char(*p)) ++p;
  const char* s = p;
  while (p < e && !skip_char(*p)) ++p;
  return std::string(s, p);
}

std::string lowered(std::string s) {
  for (char& ch : s)
    if (ch >= 'A' && ch <= 'Z') ch = static_cast<char>(ch - 'A' + 'a');
  return s;
}

// istream >> (long long): optional sign and the longest digit run; false when
// there is no digit or the value overflows.
bool integer(const char*& p, const char* e, long long& out) {
  while (p < e && skip_char(*p)) ++p;
  const char* q = p;
  bool neg = false;
  if (q < e && (*q == '+' || *q == '-')) neg = *q++ == '-';
  const char* d0 = q;
  unsigned long long acc = 0;
  bool over = false;
  while (q < e && *q >= '0' && *q <= '9') {
    const unsigned digit = static_cast<unsigned>(*q - '0');
    if (acc > (~0ull - digit) / 10) over = true;
    acc = acc * 10 + digit;
    ++q;
  }
  if (q == d0) return false;
  const unsigned long long lim = neg ? (1ull << 63) : (1ull << 63) - 1;
  if (over || acc > lim) return false;
  out = neg ? static_cast<long long>(0ull - acc) : static_cast<long long>(acc);
  p = q;
  return true;
}

// istream >> double: the characters num_get collects (sign, digits, one
// point, exponent with sign), converted by strtod, which must consume all of
// them; +-HUGE_VAL (overflow) fails as in libstdc++.
bool real(const char*& p, const char* e, double& out) {
  while (p < e && skip_char(*p)) ++p;
  const char* q = p;
  char tok[128];
  int n = 0;
  auto take = [&](char ch) {
    if (n < 127) tok[n] = ch;
    ++n;
  };
  if (q < e && (*q == '+' || *q == '-')) take(*q++);
  bool point = false;
  while (q < e && ((*q >= '0' && *q <= '9') || (*q == '.' && !point))) {
    if (*q == '.') point = true;
    take(*q++);
  }
  if (q < e && (*q == 'e' || *q == 'E')) {
    take(*q++);
    if (q < e && (*q == '+' || *q == '-')) take(*q++);
    while (q < e && *q >= '0' && *q <= '9') take(*q++);
  }
  if (n == 0 || n > 127) return false;
  tok[n] = '\0';
  char* end = nullptr;
  const double v = std::strtod(tok, &end);
  if (end != tok + n) return false;
  if (v == HUGE_VAL || v == -HUGE_VAL) return false;
  out = v;
  p = q;
  return true;
}

[[noreturn]] void bad_line(const std::string& name, long line, const char* what) {
  fail(Errc::parse_error, name + ": line " + std::to_string(line) + ": " + what);
}

// One entry line: 0 = ok (1 or 2 entries appended), else the message.
const char* entry_line(const char* b, const char* e, Index n, bool mirror, std::vector<Entry>& out) {
  long long i = 0, j = 0;
  double v = 0.0;
  if (!integer(b, e, i) || !integer(b, e, j) || !real(b, e, v)) return "malformed entry";
  if (i < 1 || i > n || j < 1 || j > n) return "entry index out of range";
  if (!std::isfinite(v)) return "non-finite entry value";
  out.push_back({i - 1, j - 1, v});
  if (mirror && i != j) out.push_back({j - 1, i - 1, v});
  return nullptr;
}

struct Chunk {
  const char* b;
  const char* e;
  std::vector<Entry> ents;
  long lines = 0;         // lines in the chunk
  long long rows = 0;     // non-blank lines parsed (entries) before an error
  const char* err = nullptr;
  long err_line = 0;      // 1-based within the chunk
};

// Parse [b, e) line by line; stop after `limit` entries (< 0: no limit) or
// at the first bad line.
void parse_chunk(Chunk& c, Index n, bool mirror, long long limit) {
  c.ents.clear();
  c.lines = 0;
  c.rows = 0;
  c.err = nullptr;
  const char* p = c.b;
  while (p < c.e && (limit < 0 || c.rows < limit)) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(c.e - p)));
    const char* le = nl ? nl : c.e;
    ++c.lines;
    if (!blank_line(p, le)) {
      if (const char* why = entry_line(p, le, n, mirror, c.ents)) {
        c.err = why;
        c.err_line = c.lines;
        return;
      }
      ++c.rows;
    }
    p = nl ? nl + 1 : c.e;
  }
}

}  // namespace

HostCsr csr_from_entries(Index n, const std::vector<Entry>& t);

HostCsr read_matrix_market_host(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (f == nullptr) fail(Errc::io_error, "cannot open '" + path + "' for reading");
  std::vector<char> buf;
  {
    char tmp[1 << 16];
    size_t got;
    while ((got = std::fread(tmp, 1, sizeof(tmp), f)) > 0) buf.insert(buf.end(), tmp, tmp + got);
    std::fclose(f);
  }
  const char* p = buf.data();
  const char* const end = buf.data() + buf.size();
  long lineno = 0;
  // next line [ls, le) as std::getline sees it; false at end of file
  auto next_line = [&](const char*& ls, const char*& le) {
    if (p >= end) return false;
    ls = p;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    le = nl ? nl : end;
    p = nl ? nl + 1 : end;
    ++lineno;
    return true;
  };
  const char *ls, *le;
  if (!next_line(ls, le)) bad_line(path, 1, "empty file");
  bool mirror = false;
  {
    const char* q = ls;
    const std::string banner = word(q, le), object = lowered(word(q, le)), format = lowered(word(q, le)),
                      field = lowered(word(q, le)), symmetry = lowered(word(q, le));
    if (banner != "%%MatrixMarket") bad_line(path, lineno, "missing %%MatrixMarket banner");
    if (object != "matrix" || format != "coordinate")
      bad_line(path, lineno, "only coordinate-format matrices are supported");
    if (field != "real") bad_line(path, lineno, "only real matrices are supported");
    if (symmetry != "general" && symmetry != "symmetric")
      bad_line(path, lineno, "only general or symmetric matrices are supported");
    mirror = symmetry == "symmetric";
  }
  long long rows = 0, cols = 0, nnz = 0;
  for (;;) {
    if (!next_line(ls, le)) bad_line(path, lineno + 1, "unexpected end of file before size line");
    if (ls < le && *ls == '%') continue;
    if (blank_line(ls, le)) continue;
    const char* q = ls;
    if (!integer(q, le, rows) || !integer(q, le, cols) || !integer(q, le, nnz)) bad_line(path, lineno, "malformed size line");
    break;
  }
  if (rows != cols)
    fail(Errc::non_square_matrix,
         path + ": matrix is " + std::to_string(rows) + "x" + std::to_string(cols) + ", expected square");

  // entry section: chunks at line boundaries, tokenised in parallel
  std::vector<Entry> all;
  if (nnz > 0) {
    const size_t bytes = static_cast<size_t>(end - p);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nch = bytes < (4u << 20) ? 1 : std::min<size_t>(hw, bytes / (1u << 20));
    std::vector<Chunk> ch(nch);
    const char* cut = p;
    for (size_t c = 0; c < nch; ++c) {
      ch[c].b = cut;
      const char* target = c + 1 == nch ? end : p + bytes * (c + 1) / nch;
      if (target < cut) target = cut;
      const char* nl = target < end ? static_cast<const char*>(std::memchr(target, '\n', static_cast<size_t>(end - target)))
                                    : nullptr;
      cut = c + 1 == nch || !nl ? end : nl + 1;
      ch[c].e = cut;
    }
    if (nch == 1) {
      parse_chunk(ch[0], rows, mirror, nnz);
    } else {
      std::vector<std::thread> pool;
      for (size_t c = 0; c < nch; ++c) pool.emplace_back([&, c] { parse_chunk(ch[c], rows, mirror, -1); });
      for (auto& th : pool) th.join();
    }
    long long have = 0;
    for (size_t c = 0; c < nch; ++c) {
      Chunk& k = ch[c];
      const bool last_needed = k.err != nullptr || have + k.rows >= nnz;
      if (last_needed && nch > 1) parse_chunk(k, rows, mirror, nnz - have);  // exact stop point
      if (k.err) bad_line(path, lineno + k.err_line, k.err);
      all.insert(all.end(), k.ents.begin(), k.ents.end());
      have += k.rows;
      lineno += k.lines;
      if (have >= nnz) break;
    }
    if (have < nnz) bad_line(path, lineno + 1, "unexpected end of file in entry list");
  }
  return csr_from_entries(rows, all);
}

// from_triplets (sparse.cpp:12-48): rows by a stable counting sort, columns
// by a stable sort inside each row, duplicates summed in input order, zero
// sums kept in the pattern.
HostCsr csr_from_entries(Index n, const std::vector<Entry>& t) {
  require(n >= 0, Errc::invalid_argument, "negative matrix dimension");
  for (const Entry& x : t) {
    if (x.r < 0 || x.r >= n || x.c < 0 || x.c >= n)
      fail(Errc::index_out_of_range, "triplet index (" + std::to_string(x.r) + "," + std::to_string(x.c) + ") outside " +
                                         std::to_string(n) + "x" + std::to_string(n));
    require(std::isfinite(x.v), Errc::invalid_argument, "non-finite triplet value");
  }
  std::vector<int64_t> start(static_cast<size_t>(n) + 1, 0);
  for (const Entry& x : t) ++start[static_cast<size_t>(x.r) + 1];
  for (Index i = 0; i < n; ++i) start[static_cast<size_t>(i) + 1] += start[static_cast<size_t>(i)];
  std::vector<int64_t> fill(start.begin(), start.end() - 1);
  std::vector<std::pair<Index, double>> by_row(t.size());
  for (const Entry& x : t) by_row[static_cast<size_t>(fill[static_cast<size_t>(x.r)]++)] = {x.c, x.v};
  HostCsr h;
  h.n = n;
  h.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
  h.col.reserve(t.size());
  h.val.reserve(t.size());
  for (Index i = 0; i < n; ++i) {
    auto b = by_row.begin() + start[static_cast<size_t>(i)], e = by_row.begin() + start[static_cast<size_t>(i) + 1];
    std::stable_sort(b, e, [](const auto& x, const auto& y) { return x.first < y.first; });
    for (auto q = b; q != e;) {
      const Index c = q->first;
      double v = q->second;
      for (++q; q != e && q->first == c; ++q) v += q->second;
      h.col.push_back(static_cast<int32_t>(c));
      h.val.push_back(v);
    }
    h.row_ptr[static_cast<size_t>(i) + 1] = static_cast<int64_t>(h.col.size());
  }
  return h;
}

// Writer: the reference's text ("%.17g" values, 1-based indices, general
// header); rows formatted into per-thread buffers, written in order.
void write_matrix_market_host(const HostCsr& a, const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (f == nullptr) fail(Errc::io_error, "cannot open '" + path + "' for writing");
  bool ok = std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n",
                         static_cast<long long>(a.n), static_cast<long long>(a.n), static_cast<long long>(a.nnz())) > 0;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const Index nblk = a.nnz() < (1 << 20) ? 1 : static_cast<Index>(hw) * 4;
  const Index rows_per = (a.n + nblk - 1) / std::max<Index>(nblk, 1);
  std::vector<std::string> out(static_cast<size_t>(nblk));
  auto format = [&](Index blk) {
    std::string& s = out[static_cast<size_t>(blk)];
    char line[96];
    const Index r0 = std::min(a.n, blk * rows_per), r1 = std::min(a.n, (blk + 1) * rows_per);
    for (Index i = r0; i < r1; ++i)
      for (int64_t q = a.row_ptr[static_cast<size_t>(i)]; q < a.row_ptr[static_cast<size_t>(i) + 1]; ++q) {
        const int len = std::snprintf(line, sizeof(line), "%lld %lld %.17g\n", static_cast<long long>(i + 1),
                                      static_cast<long long>(a.col[static_cast<size_t>(q)]) + 1,
                                      a.val[static_cast<size_t>(q)]);
        s.append(line, static_cast<size_t>(len));
      }
  };
  for (Index b0 = 0; b0 < nblk && ok; b0 += static_cast<Index>(hw)) {
    std::vector<std::thread> pool;
    const Index b1 = std::min(nblk, b0 + static_cast<Index>(hw));
    for (Index b = b0; b < b1; ++b) pool.emplace_back(format, b);
    for (auto& th : pool) th.join();
    for (Index b = b0; b < b1 && ok; ++b) {
      const std::string& s = out[static_cast<size_t>(b)];
      ok = std::fwrite(s.data(), 1, s.size(), f) == s.size();
      std::string().swap(out[static_cast<size_t>(b)]);
    }
  }
  ok = std::fclose(f) == 0 && ok;
  if (!ok) fail(Errc::io_error, "error while writing '" + path + "'");
}

}  // namespace pdb
