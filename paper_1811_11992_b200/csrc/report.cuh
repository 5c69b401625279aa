// Report frame writer (report.py:50-149), host code.
//
// The reference writes one CSV row per (time, cell) with every float as
// Python's repr(float(v)) — the shortest string that round-trips — from a
// Python loop (≈ 300 MB of text per C4 frame). Here the digits come from
// std::to_chars (shortest round-trip, closest to the exact value, as
// CPython's dtoa mode 0) and are laid out with CPython's repr rules
// (format_float_short, 'r' mode, Py_DTSF_ADD_DOT_0):
//   decpt = position of the decimal point relative to the digit string;
//   decpt <= -4 or decpt > 16  ->  d[.ddd]e[+-]XX (at least two exponent digits)
//   otherwise                  ->  fixed notation, ".0" appended to integers.
// Rows are formatted in parallel over contiguous cell ranges and joined in
// order, so the bytes equal the reference's writer for the same values.
#pragma once
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace isc {

// Python repr(float) of v into out (>= 32 bytes); returns the length
inline int py_repr_double(double v, char* out) {
  if (std::isnan(v)) { std::memcpy(out, "nan", 3); return 3; }
  if (std::isinf(v)) {
    if (v < 0) { std::memcpy(out, "-inf", 4); return 4; }
    std::memcpy(out, "inf", 3);
    return 3;
  }
  char* o = out;
  if (std::signbit(v)) { *o++ = '-'; v = -v; }
  if (v == 0.0) { std::memcpy(o, "0.0", 3); return (int)(o - out) + 3; }
  char sci[40];
  auto res = std::to_chars(sci, sci + sizeof(sci), v, std::chars_format::scientific);
  // sci = "d[.ddd]e[+-]XX"
  char digits[24];
  int nd = 0;
  const char* q = sci;
  for (; q < res.ptr && *q != 'e'; ++q)
    if (*q != '.') digits[nd++] = *q;
  int e10 = 0;
  ++q;   // 'e'
  const bool eneg = *q == '-';
  ++q;
  for (; q < res.ptr; ++q) e10 = e10 * 10 + (*q - '0');
  if (eneg) e10 = -e10;
  while (nd > 1 && digits[nd - 1] == '0') --nd;   // to_chars gives no trailing zeros; be safe
  const int decpt = e10 + 1;
  if (decpt <= -4 || decpt > 16) {
    *o++ = digits[0];
    if (nd > 1) {
      *o++ = '.';
      std::memcpy(o, digits + 1, nd - 1);
      o += nd - 1;
    }
    *o++ = 'e';
    int ex = decpt - 1;
    *o++ = ex < 0 ? '-' : '+';
    if (ex < 0) ex = -ex;
    char eb[8];
    int ne = 0;
    do { eb[ne++] = (char)('0' + ex % 10); ex /= 10; } while (ex);
    if (ne < 2) eb[ne++] = '0';
    while (ne) *o++ = eb[--ne];
  } else if (decpt <= 0) {
    *o++ = '0';
    *o++ = '.';
    for (int k = 0; k < -decpt; ++k) *o++ = '0';
    std::memcpy(o, digits, nd);
    o += nd;
  } else if (decpt >= nd) {
    std::memcpy(o, digits, nd);
    o += nd;
    for (int k = nd; k < decpt; ++k) *o++ = '0';
    *o++ = '.';
    *o++ = '0';
  } else {
    std::memcpy(o, digits, decpt);
    o += decpt;
    *o++ = '.';
    std::memcpy(o, digits + decpt, nd - decpt);
    o += nd - decpt;
  }
  return (int)(o - out);
}

struct FrameCells {
  double time;
  int64_t n;
  const double *p, *t, *sw, *sg, *cc;
  const double* x;   // x[c*xcs + i*xks]
  int64_t xcs, xks;
  int nco;
  const double* y;   // y[c*ycs + a*yks]
  int64_t ycs, yks;
  int nf;
};

// rows [c0, c1) appended to s (report.py:131-138)
inline void format_cell_rows(const FrameCells& F, int64_t c0, int64_t c1, std::string& s) {
  char tbuf[40];
  const int tl = py_repr_double(F.time, tbuf);
  char b[40];
  const int ncols = 5 + F.nco + F.nf + 1;
  s.reserve(s.size() + (size_t)(c1 - c0) * (size_t)(tl + 12 + ncols * 24));
  for (int64_t c = c0; c < c1; ++c) {
    s.append(tbuf, tl);
    s.push_back(',');
    s.append(std::to_string(c));
    auto put = [&](double v) {
      s.push_back(',');
      s.append(b, py_repr_double(v, b));
    };
    put(F.p[c]);
    put(F.t[c]);
    put(F.sw[c]);
    put(1.0 - F.sw[c] - F.sg[c]);   // so = 1.0 - sw - sg (report.py:60)
    put(F.sg[c]);
    for (int i = 0; i < F.nco; ++i) put(F.x[c * F.xcs + i * F.xks]);
    for (int a = 0; a < F.nf; ++a) put(F.y[c * F.ycs + a * F.yks]);
    put(F.cc[c]);
    s.push_back('\n');
  }
}

inline std::string format_cells(const FrameCells& F, int threads) {
  if (threads < 1) threads = 1;
  const int64_t per = 4096;
  int64_t nchunk = (F.n + per - 1) / per;
  if (nchunk < 1) nchunk = 1;
  if (threads > nchunk) threads = (int)nchunk;
  std::vector<std::string> parts((size_t)threads);
  const int64_t span = (F.n + threads - 1) / threads;
  std::vector<std::thread> pool;
  for (int w = 0; w < threads; ++w) {
    const int64_t c0 = w * span, c1 = std::min<int64_t>(F.n, c0 + span);
    if (c0 >= c1) continue;
    pool.emplace_back([&, w, c0, c1] { format_cell_rows(F, c0, c1, parts[(size_t)w]); });
  }
  for (auto& th : pool) th.join();
  size_t total = 0;
  for (auto& s : parts) total += s.size();
  std::string out;
  out.reserve(total);
  for (auto& s : parts) out.append(s);
  return out;
}

}  // namespace isc
