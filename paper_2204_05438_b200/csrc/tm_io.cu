// tm_io.cu -- host-side text I/O around the mesh -> polygons path (native, no
// device code): the byte-stable polymesh writer and the Triangle
// .node/.ele/.neigh/.trivertex readers and writers.
//
// Replaces (paths relative to /root/reference/pkg/src/termesh):
//   io_formats._fmt (repr floats)          io_formats.py:44-46
//   io_formats.write_polymesh              io_formats.py:251-262
//   io_formats._data_lines / _read_node / _read_indexed_rows / _read_trivertex
//                                          io_formats.py:48-158
//   io_formats.write_triangulation         io_formats.py:213-248
//
// Floats are written exactly as Python's repr(float): the shortest decimal
// string that reads back to the same double (correctly rounded digits, found
// by increasing the precision of an exact printf until strtod round-trips),
// laid out with repr's rules -- fixed notation for decimal exponents in
// (-4, 16], otherwise d[.ddd]e+XX with at least two exponent digits, ".0"
// appended to integral values, "inf" / "nan" spelled like Python.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/termesh_b200.h"

namespace {

// ------------------------------------------------------------ repr(float)
int repr_double(double x, char* out) {
  char* o = out;
  if (std::isnan(x)) return sprintf(out, "nan");
  if (std::signbit(x)) *o++ = '-', x = -x;
  if (std::isinf(x)) return (int)(o - out) + sprintf(o, "inf");
  if (x == 0.0) return (int)(o - out) + sprintf(o, "0.0");
  char buf[64];
  for (int p = 1; p <= 17; p++) {
    snprintf(buf, sizeof buf, "%.*e", p - 1, x);
    if (strtod(buf, nullptr) == x) break;
  }
  // buf = d[.ddd]e[+-]XX -> digits, decimal exponent
  char dig[32];
  int nd = 0;
  const char* c = buf;
  for (; *c && *c != 'e'; c++)
    if (*c >= '0' && *c <= '9') dig[nd++] = *c;
  const int e10 = atoi(c + 1);
  while (nd > 1 && dig[nd - 1] == '0') nd--;
  const int decpt = e10 + 1;  // value = 0.d1d2... * 10^decpt
  if (decpt <= -4 || decpt > 16) {
    *o++ = dig[0];
    if (nd > 1) {
      *o++ = '.';
      memcpy(o, dig + 1, nd - 1);
      o += nd - 1;
    }
    o += sprintf(o, "e%c%02d", e10 < 0 ? '-' : '+', e10 < 0 ? -e10 : e10);
  } else if (decpt <= 0) {
    *o++ = '0';
    *o++ = '.';
    for (int k = 0; k < -decpt; k++) *o++ = '0';
    memcpy(o, dig, nd);
    o += nd;
  } else if (decpt >= nd) {
    memcpy(o, dig, nd);
    o += nd;
    for (int k = 0; k < decpt - nd; k++) *o++ = '0';
    *o++ = '.';
    *o++ = '0';
  } else {
    memcpy(o, dig, decpt);
    o += decpt;
    *o++ = '.';
    memcpy(o, dig + decpt, nd - decpt);
    o += nd - decpt;
  }
  *o = 0;
  return (int)(o - out);
}

int put_i64(int64_t x, char* out) {
  char tmp[24];
  int n = 0;
  const bool neg = x < 0;
  uint64_t u = neg ? (uint64_t)0 - (uint64_t)x : (uint64_t)x;
  do {
    tmp[n++] = (char)('0' + u % 10);
    u /= 10;
  } while (u);
  int k = 0;
  if (neg) out[k++] = '-';
  while (n) out[k++] = tmp[--n];
  return k;
}

void set_msg(char* err, size_t cap, const char* fmt, ...) {
  if (!err || !cap) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, cap, fmt, ap);
  va_end(ap);
}

int n_threads(int64_t work) {
  unsigned hc = std::thread::hardware_concurrency();
  int t = hc ? (int)hc : 1;
  if (t > 32) t = 32;
  const int64_t need = work / 65536 + 1;
  return (int)std::min<int64_t>(t, need);
}

// format rows [0, n) with `row(i, char*) -> bytes` into per-thread buffers,
// then write them in order
template <typename Row>
bool write_rows(FILE* f, int64_t n, size_t max_row, Row row) {
  const int T = n_threads(n);
  std::vector<std::string> parts(T);
  std::vector<std::thread> th;
  for (int t = 0; t < T; t++) {
    th.emplace_back([&, t] {
      const int64_t a = n * t / T, b = n * (t + 1) / T;
      std::string& s = parts[t];
      s.reserve((size_t)(b - a) * 24);
      std::vector<char> tmp(max_row + 64);
      for (int64_t i = a; i < b; i++) s.append(tmp.data(), (size_t)row(i, tmp.data()));
    });
  }
  for (auto& x : th) x.join();
  for (auto& s : parts)
    if (!s.empty() && fwrite(s.data(), 1, s.size(), f) != s.size()) return false;
  return true;
}

// ------------------------------------------------------------ reader
struct Line {
  int64_t lineno;
  std::vector<std::pair<const char*, size_t>> tok;
};

// str.split() whitespace and str.splitlines() boundaries (ASCII subset)
bool is_space(char c) { return c == ' ' || (c >= '\t' && c <= '\r') || (c >= '\x1c' && c <= '\x1f'); }
bool is_break(char c) { return c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= '\x1c' && c <= '\x1e'); }

// Python int(): [sign] digits with single underscores between digits
bool parse_int(const char* s, size_t n, int64_t* out) {
  size_t i = 0;
  bool neg = false;
  if (i < n && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  if (i >= n) return false;
  uint64_t v = 0;
  bool prev_digit = false;
  for (; i < n; i++) {
    const char c = s[i];
    if (c == '_') {
      if (!prev_digit || i + 1 >= n || !(s[i + 1] >= '0' && s[i + 1] <= '9')) return false;
      prev_digit = false;
      continue;
    }
    if (c < '0' || c > '9') return false;
    if (v > (UINT64_MAX - 9) / 10) return false;  // beyond int64 (the reference would not fit it either)
    v = v * 10 + (uint64_t)(c - '0');
    prev_digit = true;
  }
  if (!prev_digit) return false;
  if (v > (uint64_t)INT64_MAX + (neg ? 1 : 0)) return false;
  *out = neg ? (int64_t)(0 - v) : (int64_t)v;
  return true;
}

bool ieq(const char* s, size_t n, const char* lit) {
  const size_t m = strlen(lit);
  if (n != m) return false;
  for (size_t i = 0; i < n; i++)
    if (tolower((unsigned char)s[i]) != lit[i]) return false;
  return true;
}

// Python float(): [sign] (inf | infinity | nan | decimal literal with single
// underscores between digits); no hex floats
bool parse_float(const char* s, size_t n, double* out) {
  size_t i = 0;
  bool neg = false;
  if (i < n && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  if (ieq(s + i, n - i, "inf") || ieq(s + i, n - i, "infinity")) { *out = neg ? -INFINITY : INFINITY; return true; }
  if (ieq(s + i, n - i, "nan")) { *out = neg ? -NAN : NAN; return true; }
  char buf[512];
  size_t k = 0;
  if (neg) buf[k++] = '-';
  int digits = 0;
  bool dot = false, exp = false, prev_digit = false;
  for (; i < n; i++) {
    const char c = s[i];
    if (k + 2 >= sizeof buf) return false;
    if (c >= '0' && c <= '9') { buf[k++] = c; digits++; prev_digit = true; continue; }
    if (c == '_') {
      if (!prev_digit || i + 1 >= n || !(s[i + 1] >= '0' && s[i + 1] <= '9')) return false;
      prev_digit = false;
      continue;
    }
    prev_digit = false;
    if (c == '.' && !dot && !exp) { dot = true; buf[k++] = c; continue; }
    if ((c == 'e' || c == 'E') && !exp && digits) {
      exp = true;
      buf[k++] = 'e';
      if (i + 1 < n && (s[i + 1] == '+' || s[i + 1] == '-')) buf[k++] = s[++i];
      if (i + 1 >= n) return false;
      digits = 0;  // the exponent needs digits of its own
      continue;
    }
    return false;
  }
  if (!digits) return false;
  buf[k] = 0;
  char* end = nullptr;
  *out = strtod(buf, &end);
  return end && *end == 0;
}

}  // namespace

// Parsed Triangle file (see tm_file_read)
struct tm_file {
  int kind = 0;
  int64_t rows = 0, cols = 0;
  std::vector<double> f64;
  std::vector<int64_t> i64;
  int status = 0;        // 0 ok, 1 parse error
  int64_t err_line = 0;  // ParseError(path, line, message)
  std::string msg;
};

namespace {

void fail(tm_file* f, int64_t line, const char* fmt, ...) {
  char b[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(b, sizeof b, fmt, ap);
  va_end(ap);
  f->status = 1;
  f->err_line = line;
  f->msg = b;
}

std::string tok_str(const std::pair<const char*, size_t>& t) { return std::string(t.first, t.second); }

// Python repr of a str token: '...' (the reference's {token!r}); tokens never
// contain whitespace, quotes get the simple form Python picks
std::string py_repr(const std::string& s) {
  const bool sq = s.find('\'') != std::string::npos, dq = s.find('"') != std::string::npos;
  const char q = (sq && !dq) ? '"' : '\'';
  std::string r(1, q);
  for (char c : s) {
    if (c == '\\') r += "\\\\";
    else if (c == q) { r += '\\'; r += c; }
    else r += c;
  }
  r += q;
  return r;
}

}  // namespace

extern "C" {

int tm_format_double(double x, char* out, size_t cap) {
  char b[64];
  const int n = repr_double(x, b);
  if (!out || cap <= (size_t)n) return -1;
  memcpy(out, b, (size_t)n + 1);
  return n;
}

// kind: 0 .node, 1 .ele, 2 .neigh, 3 .trivertex (n_expected = vertex count)
tm_file* tm_file_read(const char* path, int kind, int64_t n_expected) {
  tm_file* f = new tm_file();
  f->kind = kind;
  FILE* fp = fopen(path, "rb");
  if (!fp) {
    fail(f, 0, "cannot read file: %s", strerror(errno));
    return f;
  }
  std::string text;
  {
    char buf[1 << 16];
    size_t got;
    while ((got = fread(buf, 1, sizeof buf, fp)) > 0) text.append(buf, got);
    fclose(fp);
  }
  // _data_lines: split lines like str.splitlines ('\r\n' is one break), strip
  // '#' comments, whitespace-split, skip empty
  std::vector<Line> lines;
  {
    const char* p = text.data();
    const char* e = p + text.size();
    int64_t lineno = 0;
    while (p < e) {
      const char* q = p;
      while (q < e && !is_break(*q)) q++;
      lineno++;
      const char* end = q;
      for (const char* h = p; h < q; h++)
        if (*h == '#') { end = h; break; }
      Line ln;
      ln.lineno = lineno;
      const char* c = p;
      while (c < end) {
        while (c < end && is_space(*c)) c++;
        const char* s = c;
        while (c < end && !is_space(*c)) c++;
        if (c > s) ln.tok.emplace_back(s, (size_t)(c - s));
      }
      if (!ln.tok.empty()) lines.push_back(std::move(ln));
      if (q < e && *q == '\r' && q + 1 < e && q[1] == '\n') q++;
      p = q + 1;
    }
  }
  if (lines.empty()) {
    fail(f, 0, "empty file");
    return f;
  }
  const Line& h = lines[0];
  auto geti = [&](const Line& ln, size_t k, const char* what, int64_t* v) {
    if (!parse_int(ln.tok[k].first, ln.tok[k].second, v)) {
      fail(f, ln.lineno, "expected integer %s, got %s", what, py_repr(tok_str(ln.tok[k])).c_str());
      return false;
    }
    return true;
  };
  if (kind == 0) {  // _read_node (io_formats.py:70-99)
    if (h.tok.size() < 2) { fail(f, h.lineno, "node header needs at least <#points> <dim>"); return f; }
    int64_t n = 0, dim = 0, attrs = 0, markers = 0;
    if (!geti(h, 0, "point count", &n) || !geti(h, 1, "dimension", &dim)) return f;
    if (h.tok.size() > 2 && !geti(h, 2, "attribute count", &attrs)) return f;
    if (h.tok.size() > 3 && !geti(h, 3, "marker count", &markers)) return f;
    if (dim != 2) { fail(f, h.lineno, "only 2-d points are supported, got dimension %lld", (long long)dim); return f; }
    if (n < 0 || attrs < 0 || (markers != 0 && markers != 1)) { fail(f, h.lineno, "malformed node header"); return f; }
    const size_t want = (size_t)(1 + 2 + attrs + markers);
    f->f64.resize((size_t)(2 * n));
    int64_t rows = 0;
    for (size_t li = 1; li < lines.size(); li++) {
      const Line& ln = lines[li];
      if (rows >= n) { fail(f, ln.lineno, "more than %lld point rows", (long long)n); return f; }
      if (ln.tok.size() != want) {
        fail(f, ln.lineno, "expected %zu columns, got %zu", want, ln.tok.size());
        return f;
      }
      for (int k = 0; k < 2; k++) {
        double x;
        if (!parse_float(ln.tok[1 + k].first, ln.tok[1 + k].second, &x)) {
          fail(f, ln.lineno, "expected number %s, got %s", k ? "y coordinate" : "x coordinate",
               py_repr(tok_str(ln.tok[1 + k])).c_str());
          return f;
        }
        f->f64[2 * rows + k] = x;
      }
      rows++;
    }
    if (rows != n) { fail(f, 0, "header promises %lld points but file has %lld", (long long)n, (long long)rows); return f; }
    f->rows = n;
    f->cols = 2;
    return f;
  }
  if (kind == 1 || kind == 2) {  // _read_indexed_rows (io_formats.py:102-130)
    const char* what = kind == 1 ? "triangle" : "neighbor";
    if (h.tok.size() < 2) { fail(f, h.lineno, "%s header needs <#rows> <3>", what); return f; }
    int64_t count = 0, width = 0;
    if (!geti(h, 0, "row count", &count) || !geti(h, 1, "entries per row", &width)) return f;
    if (count < 0 || width != 3) { fail(f, h.lineno, "malformed %s header (width must be 3)", what); return f; }
    f->i64.resize((size_t)(3 * count));
    int64_t rows = 0;
    std::string ref = std::string(what) + " reference";
    for (size_t li = 1; li < lines.size(); li++) {
      const Line& ln = lines[li];
      if (rows >= count) { fail(f, ln.lineno, "more than %lld %s rows", (long long)count, what); return f; }
      if (ln.tok.size() < 4) { fail(f, ln.lineno, "expected at least 4 columns"); return f; }
      for (int k = 0; k < 3; k++)
        if (!geti(ln, 1 + k, ref.c_str(), &f->i64[3 * rows + k])) return f;
      rows++;
    }
    if (rows != count) {
      fail(f, 0, "header promises %lld rows but file has %lld", (long long)count, (long long)rows);
      return f;
    }
    f->rows = count;
    f->cols = 3;
    return f;
  }
  if (kind == 3) {  // _read_trivertex (io_formats.py:133-158)
    int64_t count = 0;
    if (!geti(h, 0, "vertex count", &count)) return f;
    if (count != n_expected) {
      fail(f, h.lineno, "trivertex file covers %lld vertices, expected %lld", (long long)count,
           (long long)n_expected);
      return f;
    }
    f->i64.assign((size_t)(count > 0 ? count : 0), -1);
    int64_t rows = 0;
    for (size_t li = 1; li < lines.size(); li++) {
      const Line& ln = lines[li];
      if (rows >= count) { fail(f, ln.lineno, "more than %lld trivertex rows", (long long)count); return f; }
      if (ln.tok.size() != 2) { fail(f, ln.lineno, "expected 2 columns, got %zu", ln.tok.size()); return f; }
      if (!geti(ln, 1, "triangle reference", &f->i64[rows])) return f;
      rows++;
    }
    if (rows != count) {
      fail(f, 0, "header promises %lld rows but file has %lld", (long long)count, (long long)rows);
      return f;
    }
    f->rows = count;
    f->cols = 1;
    return f;
  }
  fail(f, 0, "unknown file kind %d", kind);
  return f;
}

int tm_file_status(const tm_file* f, int64_t* rows, int64_t* cols, int64_t* err_line, char* msg, size_t cap) {
  if (!f) return TM_ERR_ARGUMENT;
  if (rows) *rows = f->rows;
  if (cols) *cols = f->cols;
  if (err_line) *err_line = f->err_line;
  if (msg && cap) snprintf(msg, cap, "%s", f->msg.c_str());
  return f->status;
}

int tm_file_copy(const tm_file* f, void* dst) {
  if (!f || f->status || !dst) return TM_ERR_ARGUMENT;
  if (f->kind == 0) memcpy(dst, f->f64.data(), f->f64.size() * sizeof(double));
  else memcpy(dst, f->i64.data(), f->i64.size() * sizeof(int64_t));
  return TM_OK;
}

void tm_file_close(tm_file* f) { delete f; }

int tm_write_polymesh(const char* path, const double* xy, int64_t n_vertices, const int64_t* offsets,
                      const int32_t* verts, int64_t n_polys, char* err, size_t err_cap) {
  FILE* f = fopen(path, "wb");
  if (!f) {
    set_msg(err, err_cap, "cannot open %s: %s", path, strerror(errno));
    return TM_ERR_ARGUMENT;
  }
  char head[64];
  int k = put_i64(n_vertices, head);
  head[k++] = ' ';
  k += put_i64(n_polys, head + k);
  head[k++] = '\n';
  bool ok = fwrite(head, 1, (size_t)k, f) == (size_t)k;
  ok = ok && write_rows(f, n_vertices, 64, [&](int64_t i, char* b) {
    int m = repr_double(xy[2 * i], b);
    b[m++] = ' ';
    m += repr_double(xy[2 * i + 1], b + m);
    b[m++] = '\n';
    return m;
  });
  int64_t maxlen = 0;
  for (int64_t i = 0; i < n_polys; i++) maxlen = std::max(maxlen, offsets[i + 1] - offsets[i]);
  ok = ok && write_rows(f, n_polys, (size_t)(maxlen + 1) * 12 + 24, [&](int64_t i, char* b) {
    const int64_t a = offsets[i], L = offsets[i + 1] - a;
    int m = put_i64(L, b);
    for (int64_t j = 0; j < L; j++) {
      b[m++] = ' ';
      m += put_i64(verts[a + j], b + m);
    }
    b[m++] = '\n';
    return m;
  });
  ok = (fclose(f) == 0) && ok;
  if (!ok) {
    set_msg(err, err_cap, "write to %s failed", path);
    return TM_ERR_ARGUMENT;
  }
  return TM_OK;
}

// io_formats.write_triangulation (io_formats.py:213-248): zero-based, no
// attributes/markers; which: 0 .node (xy), 1 .ele (triangles), 2 .neigh
// (neighbors), 3 .trivertex (trivertex)
int tm_write_triangle_file(const char* path, int which, const double* xy, const int64_t* rows3, int64_t count,
                           char* err, size_t err_cap) {
  FILE* f = fopen(path, "wb");
  if (!f) {
    set_msg(err, err_cap, "cannot open %s: %s", path, strerror(errno));
    return TM_ERR_ARGUMENT;
  }
  char head[96];
  int k = put_i64(count, head);
  const char* tail = which == 0 ? " 2 0 0\n" : which == 1 ? " 3 0\n" : which == 2 ? " 3\n" : "\n";
  k += sprintf(head + k, "%s", tail);
  bool ok = fwrite(head, 1, (size_t)k, f) == (size_t)k;
  ok = ok && write_rows(f, count, 96, [&](int64_t i, char* b) {
    int m = put_i64(i, b);
    if (which == 0) {
      b[m++] = ' ';
      m += repr_double(xy[2 * i], b + m);
      b[m++] = ' ';
      m += repr_double(xy[2 * i + 1], b + m);
    } else if (which == 3) {
      b[m++] = ' ';
      m += put_i64(rows3[i], b + m);
    } else {
      for (int j = 0; j < 3; j++) {
        b[m++] = ' ';
        m += put_i64(rows3[3 * i + j], b + m);
      }
    }
    b[m++] = '\n';
    return m;
  });
  ok = (fclose(f) == 0) && ok;
  if (!ok) {
    set_msg(err, err_cap, "write to %s failed", path);
    return TM_ERR_ARGUMENT;
  }
  return TM_OK;
}

}  // extern "C"
