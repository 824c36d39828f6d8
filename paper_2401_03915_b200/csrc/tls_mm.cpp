// tls_mm.cpp — Matrix Market ingest / output for libtls_b200.so.
//
// The on-disk boundary of the reference (src/sparsemat.py:201-372: read_matrix_market,
// write_matrix_market) restated natively: the same accepted dialect (coordinate / array, real,
// general / symmetric with lower-triangle storage), the same validation order and the same error
// texts with the same 1-based line numbers (MatrixMarketError), so a file the reference rejects
// is rejected here with an identical message.  The text is split into line-aligned chunks that
// are tokenised and parsed on all host threads; the canonical CSR (sorted columns, duplicates
// summed in file order, explicit zeros kept -- the scipy coo->csr result of SparseMat.from_coo)
// is then handed to the caller, who uploads it to the device.  Line breaks follow
// str.splitlines for ASCII (\n, \r\n, \r, \v, \f, \x1c-\x1e).
#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tls_b200.h"

struct tls_mm {
  int64_t nrows = 0, ncols = 0;
  int32_t symmetric = 0;
  std::vector<int64_t> indptr;
  std::vector<int32_t> indices;
  std::vector<double> data;
  int64_t err_line = 0;
  std::string err;
};

namespace {

inline bool is_ws(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f);
}
inline bool is_lb(unsigned char c) {
  return c == '\n' || c == '\r' || c == '\v' || c == '\f' || c == 0x1c || c == 0x1d || c == 0x1e;
}

// end of the line starting at p (first line-break char or e), and the start of the next line
inline const char* line_end(const char* p, const char* e, const char** next) {
  const char* q = p;
  while (q < e && !is_lb((unsigned char)*q)) ++q;
  const char* n = q;
  if (n < e) {
    if (*n == '\r' && n + 1 < e && n[1] == '\n') n += 2;
    else n += 1;
  }
  *next = n;
  return q;
}

struct Tok {
  const char* b;
  const char* e;
  std::string str() const { return std::string(b, e); }
};

// tokens of a stripped line (str.split())
inline int split(const char* b, const char* e, Tok* out, int cap) {
  int n = 0;
  const char* p = b;
  while (p < e) {
    while (p < e && is_ws((unsigned char)*p)) ++p;
    if (p >= e) break;
    const char* s = p;
    while (p < e && !is_ws((unsigned char)*p)) ++p;
    if (n < cap) out[n] = Tok{s, p};
    ++n;
  }
  return n;
}

inline void strip(const char*& b, const char*& e) {
  while (b < e && is_ws((unsigned char)*b)) ++b;
  while (e > b && is_ws((unsigned char)e[-1])) --e;
}

// Python repr() of an ASCII-ish token
std::string py_repr(const std::string& s) {
  const bool dq = s.find('\'') != std::string::npos && s.find('"') == std::string::npos;
  const char q = dq ? '"' : '\'';
  std::string o(1, q);
  for (unsigned char c : s) {
    if (c == '\\') o += "\\\\";
    else if (c == (unsigned char)q) { o += '\\'; o += (char)c; }
    else if (c == '\t') o += "\\t";
    else if (c == '\n') o += "\\n";
    else if (c == '\r') o += "\\r";
    else if (c < 0x20 || c == 0x7f) {
      char buf[8];
      snprintf(buf, sizeof buf, "\\x%02x", c);
      o += buf;
    } else {
      o += (char)c;
    }
  }
  o += q;
  return o;
}

// Python's digit-grouping underscores: allowed only between two digits
bool strip_underscores(const char* b, const char* e, std::string& out) {
  out.clear();
  for (const char* p = b; p < e; ++p) {
    if (*p == '_') {
      if (p == b || p + 1 >= e || !isdigit((unsigned char)p[-1]) || !isdigit((unsigned char)p[1])) return false;
      continue;
    }
    out += *p;
  }
  return true;
}

// int(tok): optional sign, decimal digits (leading zeros allowed), digit-group underscores.
// Returns 0 ok, 1 invalid, 2 overflow (valid integer beyond int64)
int py_int(const char* b, const char* e, int64_t& v) {
  std::string tmp;
  if (std::memchr(b, '_', e - b)) {
    if (!strip_underscores(b, e, tmp)) return 1;
    b = tmp.data();
    e = b + tmp.size();
  }
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    ++b;
  }
  if (b >= e) return 1;
  for (const char* p = b; p < e; ++p)
    if (!isdigit((unsigned char)*p)) return 1;
  uint64_t acc = 0;
  for (const char* p = b; p < e; ++p) {
    const uint64_t d = (uint64_t)(*p - '0');
    if (acc > (UINT64_MAX - d) / 10) return 2;
    acc = acc * 10 + d;
  }
  if (acc > (uint64_t)INT64_MAX) return 2;
  v = neg ? -(int64_t)acc : (int64_t)acc;
  return 0;
}

// float(tok): decimal / exponent forms, inf / infinity / nan (any case), optional sign,
// digit-group underscores; no hex, no nan(payload)
bool py_float(const char* b, const char* e, double& v) {
  std::string tmp;
  if (std::memchr(b, '_', e - b)) {
    if (!strip_underscores(b, e, tmp)) return false;
    b = tmp.data();
    e = b + tmp.size();
  }
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    ++b;
  }
  if (b >= e || *b == '+' || *b == '-') return false;
  for (const char* p = b; p < e; ++p)
    if (*p == '(' || *p == 'x' || *p == 'X' || *p == 'p' || *p == 'P') return false;
  auto r = std::from_chars(b, e, v, std::chars_format::general);
  if (r.ec != std::errc() || r.ptr != e) {
    if (r.ec == std::errc::result_out_of_range && r.ptr == e) {
      // Python rounds overflow to inf and underflow to 0
      bool big = false;
      for (const char* p = b; p < e; ++p)
        if (*p == 'e' || *p == 'E') { big = p + 1 < e && p[1] != '-'; break; }
      v = big ? HUGE_VAL : 0.0;
    } else {
      return false;
    }
  }
  if (neg) v = -v;
  return true;
}

std::string lower(std::string s) {
  for (char& c : s) c = (char)tolower((unsigned char)c);
  return s;
}

std::string int_text(const Tok& t) {  // str(int(tok)) for an in-range or overflowing integer
  std::string s;
  strip_underscores(t.b, t.e, s);
  bool neg = false;
  size_t i = 0;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  while (i + 1 < s.size() && s[i] == '0') ++i;
  std::string d = s.substr(i);
  if (d == "0") neg = false;
  return (neg ? "-" : "") + d;
}

struct Chunk {
  const char* b = nullptr;
  const char* e = nullptr;
  int64_t lines = 0;        // line breaks inside the chunk (the chunk ends after one, or at EOF)
  int64_t entries = 0;      // non-blank, non-comment lines
  int64_t tokens = 0;       // (array format) values
  int64_t last_entry_line = 0;  // relative line index of the last entry line, -1 if none
  int64_t line0 = 0, entry0 = 0, token0 = 0;
  int64_t err_line = INT64_MAX;
  std::string err;
};

inline bool entry_line(const char* b, const char* e) {
  strip(b, e);
  return b < e && *b != '%';
}

}  // namespace

static int mm_fail(tls_mm* mm, int64_t line, const std::string& msg) {
  mm->err_line = line;
  mm->err = msg;
  return TLS_ERR_FORMAT;
}

extern "C" {

int32_t tls_mm_parse(const char* text, int64_t len, int32_t nthreads, tls_mm** out) {
  if (!out || (!text && len > 0) || len < 0) return TLS_ERR_ARG;
  tls_mm* mm = new tls_mm();
  *out = mm;
  const char* const T0 = text;
  const char* const TE = text + len;
  // header: the first non-blank line (src/sparsemat.py:235-245)
  const char* p = T0;
  int64_t lineno = 0;
  std::string header;
  int64_t header_line = 1;
  bool found = false;
  while (p < TE) {
    const char* next;
    const char* le = line_end(p, TE, &next);
    ++lineno;
    const char* b = p;
    const char* e = le;
    strip(b, e);
    p = next;
    if (b < e) {
      header.assign(b, e);
      header_line = lineno;
      found = true;
      break;
    }
  }
  if (!found || header.compare(0, 14, "%%MatrixMarket") != 0)
    return mm_fail(mm, header_line, "missing %%MatrixMarket header");
  Tok ht[8];
  const int nh = split(header.data(), header.data() + header.size(), ht, 8);
  if (nh != 5 || lower(ht[1].str()) != "matrix")
    return mm_fail(mm, header_line, "malformed header " + py_repr(header));
  const std::string fmt = lower(ht[2].str()), field = lower(ht[3].str()), symm = lower(ht[4].str());
  if (fmt != "coordinate" && fmt != "array") return mm_fail(mm, header_line, "unsupported format " + py_repr(fmt));
  if (field != "real") return mm_fail(mm, header_line, "unsupported field " + py_repr(field) + " (only real)");
  if (symm != "general" && symm != "symmetric")
    return mm_fail(mm, header_line, "unsupported symmetry " + py_repr(symm));
  const bool sym = symm == "symmetric";
  mm->symmetric = sym ? 1 : 0;
  // size line: the first body line (non-blank, non-comment) after the header
  Tok st[8];
  int ns = 0;
  int64_t size_line = 0;
  found = false;
  while (p < TE) {
    const char* next;
    const char* le = line_end(p, TE, &next);
    ++lineno;
    const char* b = p;
    const char* e = le;
    p = next;
    strip(b, e);
    if (b < e && *b != '%') {
      ns = split(b, e, st, 8);
      size_line = lineno;
      found = true;
      break;
    }
  }
  if (!found) return mm_fail(mm, lineno + 1, "missing size line");
  // entries: line-aligned chunks over all threads
  int nt = nthreads > 0 ? nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
  const int64_t rest = TE - p;
  if (rest < (1 << 20)) nt = 1;
  nt = (int)std::min<int64_t>(nt, 64);
  std::vector<Chunk> ch(nt);
  {
    const char* cb = p;
    for (int c = 0; c < nt; ++c) {
      const char* ce = c == nt - 1 ? TE : std::max(cb, p + rest * (c + 1) / nt);
      if (c < nt - 1) {  // advance to just after a '\n' (never split \r\n)
        while (ce < TE && *ce != '\n') ++ce;
        if (ce < TE) ++ce;
      }
      ch[c].b = cb;
      ch[c].e = ce;
      cb = ce;
    }
  }
  const bool coord = fmt == "coordinate";
  auto count = [&](Chunk& c) {
    const char* q = c.b;
    int64_t li = 0;
    c.last_entry_line = -1;
    while (q < c.e) {
      const char* next;
      const char* le = line_end(q, c.e, &next);
      if (entry_line(q, le)) {
        ++c.entries;
        c.last_entry_line = li;
        if (!coord) {
          Tok tk[1];
          c.tokens += split(q, le, tk, 0);
        }
      }
      ++li;
      q = next;
    }
    c.lines = li;
  };
  {
    std::vector<std::thread> th;
    for (int c = 1; c < nt; ++c) th.emplace_back(count, std::ref(ch[c]));
    count(ch[0]);
    for (auto& t : th) t.join();
  }
  int64_t total_entries = 0, total_tokens = 0, last_entry_abs = 0;
  {
    int64_t l0 = lineno + 1;
    for (int c = 0; c < nt; ++c) {
      ch[c].line0 = l0;
      ch[c].entry0 = total_entries;
      ch[c].token0 = total_tokens;
      if (ch[c].last_entry_line >= 0) last_entry_abs = l0 + ch[c].last_entry_line;
      l0 += ch[c].lines;
      total_entries += ch[c].entries;
      total_tokens += ch[c].tokens;
    }
  }
  if (coord) {
    if (ns != 3) return mm_fail(mm, size_line, "coordinate size line needs 'rows cols nnz'");
    int64_t v[3];
    const char* what[3] = {"row count", "column count", "entry count"};
    for (int k = 0; k < 3; ++k) {
      const int r = py_int(st[k].b, st[k].e, v[k]);
      if (r == 1)
        return mm_fail(mm, size_line, std::string("expected an integer ") + what[k] + ", got " + py_repr(st[k].str()));
      if (r == 2) return mm_fail(mm, size_line, "matrix size beyond the supported int64 range");
    }
    if (v[0] < 0 || v[1] < 0 || v[2] < 0) return mm_fail(mm, size_line, "negative size");
    const int64_t nrows = v[0], ncols = v[1], nnz = v[2];
    if (total_entries != nnz)
      return mm_fail(mm, total_entries ? last_entry_abs : size_line,
                     "expected " + std::to_string(nnz) + " entries, found " + std::to_string(total_entries));
    if (nrows > INT32_MAX || ncols > INT32_MAX) return mm_fail(mm, size_line, "matrix size beyond the int32 index range");
    mm->nrows = nrows;
    mm->ncols = ncols;
    std::vector<int32_t> ri(nnz), ci(nnz);
    std::vector<double> vi(nnz);
    auto parse = [&](Chunk& c) {
      const char* q = c.b;
      int64_t li = c.line0, k = c.entry0;
      Tok tk[4];
      while (q < c.e) {
        const char* next;
        const char* le = line_end(q, c.e, &next);
        const char* b = q;
        const char* e = le;
        strip(b, e);
        if (b < e && *b != '%') {
          auto bad = [&](const std::string& m) {
            c.err_line = li;
            c.err = m;
          };
          const int n = split(b, e, tk, 4);
          int64_t i = 0, j = 0;
          int ri_ = 0, rj_ = 0;
          double val = 0.0;
          if (n != 3) { bad("coordinate entry needs 'i j value'"); return; }
          if ((ri_ = py_int(tk[0].b, tk[0].e, i)) == 1) { bad("expected an integer row index, got " + py_repr(tk[0].str())); return; }
          if ((rj_ = py_int(tk[1].b, tk[1].e, j)) == 1) { bad("expected an integer column index, got " + py_repr(tk[1].str())); return; }
          if (ri_ == 2 || rj_ == 2 || !(1 <= i && i <= nrows && 1 <= j && j <= ncols)) {
            bad("index (" + int_text(tk[0]) + ", " + int_text(tk[1]) + ") out of range for " + std::to_string(nrows) +
                "x" + std::to_string(ncols));
            return;
          }
          if (!py_float(tk[2].b, tk[2].e, val)) { bad("expected a real value, got " + py_repr(tk[2].str())); return; }
          if (!std::isfinite(val)) { bad("non-finite value " + py_repr(tk[2].str())); return; }
          if (sym && i < j) { bad("symmetric storage must list the lower triangle"); return; }
          ri[k] = (int32_t)(i - 1);
          ci[k] = (int32_t)(j - 1);
          vi[k] = val;
          ++k;
        }
        ++li;
        q = next;
      }
    };
    {
      std::vector<std::thread> th;
      for (int c = 1; c < nt; ++c) th.emplace_back(parse, std::ref(ch[c]));
      parse(ch[0]);
      for (auto& t : th) t.join();
    }
    for (int c = 0; c < nt; ++c)
      if (ch[c].err_line != INT64_MAX) return mm_fail(mm, ch[c].err_line, ch[c].err);
    // COO (+ mirrored lower entries, appended right after their original like the reference)
    // -> CSR: rows bucketed in triplet order, columns stably sorted, duplicates summed in order
    std::vector<int64_t> cnt(nrows + 1, 0);
    for (int64_t k = 0; k < nnz; ++k) {
      cnt[ri[k] + 1]++;
      if (sym && ri[k] != ci[k]) cnt[ci[k] + 1]++;
    }
    for (int64_t r = 0; r < nrows; ++r) cnt[r + 1] += cnt[r];
    const int64_t tot = cnt[nrows];
    std::vector<int32_t> col(tot);
    std::vector<double> val(tot);
    {
      std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
      for (int64_t k = 0; k < nnz; ++k) {
        int64_t f = fill[ri[k]]++;
        col[f] = ci[k];
        val[f] = vi[k];
        if (sym && ri[k] != ci[k]) {
          f = fill[ci[k]]++;
          col[f] = ri[k];
          val[f] = vi[k];
        }
      }
    }
    std::vector<int64_t> keep(nrows + 1, 0);
    auto sort_rows = [&](int64_t r0, int64_t r1) {
      std::vector<std::pair<int32_t, double>> tmp;
      for (int64_t r = r0; r < r1; ++r) {
        const int64_t b = cnt[r], e = cnt[r + 1];
        tmp.clear();
        for (int64_t k = b; k < e; ++k) tmp.emplace_back(col[k], val[k]);
        std::stable_sort(tmp.begin(), tmp.end(),
                         [](const std::pair<int32_t, double>& x, const std::pair<int32_t, double>& y) { return x.first < y.first; });
        int64_t w = b;
        for (size_t k = 0; k < tmp.size(); ++k) {
          if (k > 0 && tmp[k].first == tmp[k - 1].first) {
            val[w - 1] += tmp[k].second;
          } else {
            col[w] = tmp[k].first;
            val[w] = tmp[k].second;
            ++w;
          }
        }
        keep[r + 1] = w - b;
      }
    };
    {
      std::vector<std::thread> th;
      for (int c = 1; c < nt; ++c) th.emplace_back(sort_rows, nrows * c / nt, nrows * (c + 1) / nt);
      sort_rows(0, nrows / nt);
      for (auto& t : th) t.join();
    }
    mm->indptr.assign(nrows + 1, 0);
    for (int64_t r = 0; r < nrows; ++r) mm->indptr[r + 1] = mm->indptr[r] + keep[r + 1];
    mm->indices.resize(mm->indptr[nrows]);
    mm->data.resize(mm->indptr[nrows]);
    for (int64_t r = 0; r < nrows; ++r) {
      std::copy(col.begin() + cnt[r], col.begin() + cnt[r] + keep[r + 1], mm->indices.begin() + mm->indptr[r]);
      std::copy(val.begin() + cnt[r], val.begin() + cnt[r] + keep[r + 1], mm->data.begin() + mm->indptr[r]);
    }
    return TLS_OK;
  }
  // array format (src/sparsemat.py:295-321): column-major dense values, zeros dropped
  if (ns != 2) return mm_fail(mm, size_line, "array size line needs 'rows cols'");
  int64_t v[2];
  const char* what[2] = {"row count", "column count"};
  for (int k = 0; k < 2; ++k) {
    const int r = py_int(st[k].b, st[k].e, v[k]);
    if (r == 1)
      return mm_fail(mm, size_line, std::string("expected an integer ") + what[k] + ", got " + py_repr(st[k].str()));
    if (r == 2) return mm_fail(mm, size_line, "matrix size beyond the supported int64 range");
  }
  const int64_t nrows = v[0], ncols = v[1];
  if (sym && nrows != ncols) return mm_fail(mm, size_line, "symmetric array storage requires a square matrix");
  std::vector<double> vals(total_tokens);
  auto parse_arr = [&](Chunk& c) {
    const char* q = c.b;
    int64_t li = c.line0, k = c.token0;
    std::vector<Tok> tk(64);
    while (q < c.e) {
      const char* next;
      const char* le = line_end(q, c.e, &next);
      const char* b = q;
      const char* e = le;
      strip(b, e);
      if (b < e && *b != '%') {
        int n = split(b, e, tk.data(), (int)tk.size());
        if (n > (int)tk.size()) {
          tk.resize(n);
          n = split(b, e, tk.data(), n);
        }
        for (int t = 0; t < n; ++t) {
          double x;
          if (!py_float(tk[t].b, tk[t].e, x)) {
            c.err_line = li;
            c.err = "expected a real value, got " + py_repr(tk[t].str());
            return;
          }
          if (!std::isfinite(x)) {
            c.err_line = li;
            c.err = "non-finite value " + py_repr(tk[t].str());
            return;
          }
          vals[k++] = x;
        }
      }
      ++li;
      q = next;
    }
  };
  {
    std::vector<std::thread> th;
    for (int c = 1; c < nt; ++c) th.emplace_back(parse_arr, std::ref(ch[c]));
    parse_arr(ch[0]);
    for (auto& t : th) t.join();
  }
  for (int c = 0; c < nt; ++c)
    if (ch[c].err_line != INT64_MAX) return mm_fail(mm, ch[c].err_line, ch[c].err);
  const int64_t expected = sym ? nrows * (nrows + 1) / 2 : nrows * ncols;
  if (total_tokens != expected)
    return mm_fail(mm, total_entries ? last_entry_abs : size_line,
                   "expected " + std::to_string(expected) + " values, found " + std::to_string(total_tokens));
  if (nrows < 0 || ncols < 0) return mm_fail(mm, size_line, "negative size");
  if (nrows > INT32_MAX || ncols > INT32_MAX) return mm_fail(mm, size_line, "matrix size beyond the int32 index range");
  mm->nrows = nrows;
  mm->ncols = ncols;
  auto at = [&](int64_t i, int64_t j) -> double {  // dense[i, j]
    if (!sym) return vals[j * nrows + i];
    const int64_t a = std::max(i, j), b = std::min(i, j);  // column b, row a of the lower triangle
    return vals[b * nrows - b * (b - 1) / 2 + (a - b)];
  };
  mm->indptr.assign(nrows + 1, 0);
  for (int64_t i = 0; i < nrows; ++i) {
    for (int64_t j = 0; j < ncols; ++j) {
      const double x = at(i, j);
      if (x != 0.0) {
        mm->indices.push_back((int32_t)j);
        mm->data.push_back(x);
      }
    }
    mm->indptr[i + 1] = (int64_t)mm->indices.size();
  }
  return TLS_OK;
}

int32_t tls_mm_load(const char* path, int32_t nthreads, tls_mm** out) {
  if (!path || !out) return TLS_ERR_ARG;
  FILE* f = fopen(path, "rb");
  if (!f) {
    *out = new tls_mm();
    (*out)->err = std::string("cannot open ") + path + ": " + strerror(errno);
    return TLS_ERR_IO;
  }
  std::string buf;
  fseek(f, 0, SEEK_END);
  const long sz = ftell(f);
  fseek(f, 0, SEEK_SET);
  buf.resize(sz > 0 ? (size_t)sz : 0);
  const size_t got = sz > 0 ? fread(&buf[0], 1, (size_t)sz, f) : 0;
  fclose(f);
  buf.resize(got);
  return tls_mm_parse(buf.data(), (int64_t)buf.size(), nthreads, out);
}

int32_t tls_mm_info(const tls_mm* mm, int64_t* nrows, int64_t* ncols, int64_t* nnz, int32_t* symmetric,
                    int64_t* err_line, const char** err_msg) {
  if (!mm) return TLS_ERR_ARG;
  if (nrows) *nrows = mm->nrows;
  if (ncols) *ncols = mm->ncols;
  if (nnz) *nnz = mm->indptr.empty() ? 0 : mm->indptr.back();
  if (symmetric) *symmetric = mm->symmetric;
  if (err_line) *err_line = mm->err_line;
  if (err_msg) *err_msg = mm->err.c_str();
  return TLS_OK;
}

int32_t tls_mm_export(const tls_mm* mm, int64_t* indptr, int32_t* indices, double* data) {
  if (!mm || !indptr) return TLS_ERR_ARG;
  if (mm->indptr.empty()) {
    for (int64_t r = 0; r <= mm->nrows; ++r) indptr[r] = 0;
    return TLS_OK;
  }
  std::memcpy(indptr, mm->indptr.data(), sizeof(int64_t) * mm->indptr.size());
  if (!mm->indices.empty()) {
    std::memcpy(indices, mm->indices.data(), sizeof(int32_t) * mm->indices.size());
    std::memcpy(data, mm->data.data(), sizeof(double) * mm->data.size());
  }
  return TLS_OK;
}

void tls_mm_free(tls_mm* mm) { delete mm; }

// write_matrix_market (src/sparsemat.py:323-332): general coordinate, 17 significant digits,
// rows formatted on all host threads
int32_t tls_mm_write(const char* path, int64_t nrows, int64_t ncols, const int64_t* indptr,
                     const int32_t* indices, const double* data, int32_t nthreads) {
  if (!path || nrows < 0 || ncols < 0 || !indptr) return TLS_ERR_ARG;
  FILE* f = fopen(path, "wb");
  if (!f) return TLS_ERR_IO;
  const int64_t nnz = indptr[nrows];
  fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n", (long long)nrows,
          (long long)ncols, (long long)nnz);
  int nt = nthreads > 0 ? nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
  if (nnz < (1 << 16)) nt = 1;
  const int64_t block = 1 << 18;  // rows per formatting round per thread
  std::vector<std::string> out(nt);
  int32_t rc = TLS_OK;
  for (int64_t r0 = 0; r0 < nrows && rc == TLS_OK; r0 += block * nt) {
    auto fmt = [&](int c) {
      std::string& s = out[c];
      s.clear();
      const int64_t a = std::min(nrows, r0 + c * block), b = std::min(nrows, a + block);
      char buf[96];
      for (int64_t i = a; i < b; ++i)
        for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
          const int m = snprintf(buf, sizeof buf, "%lld %d %.17g\n", (long long)(i + 1), indices[k] + 1, data[k]);
          s.append(buf, m);
        }
    };
    std::vector<std::thread> th;
    for (int c = 1; c < nt; ++c) th.emplace_back(fmt, c);
    fmt(0);
    for (auto& t : th) t.join();
    for (int c = 0; c < nt; ++c)
      if (!out[c].empty() && fwrite(out[c].data(), 1, out[c].size(), f) != out[c].size()) rc = TLS_ERR_IO;
  }
  if (fclose(f) != 0) rc = TLS_ERR_IO;
  return rc;
}

}  // extern "C"
