// numfmt.cuh -- exact number formatting for the timeline JSON (host + device).
//
// The reference writes timestamps as Python floats through json.dump
// (sinks.py:374-375, :407, :417), i.e. CPython's float.__repr__: the shortest
// digit string that round-trips, nearest to the exact value on ties, in fixed
// notation for 1e-4 <= |x| < 1e16 and 'd.ddde±XX' otherwise, plus
// NaN/Infinity spellings of the json module.  Integers are printed exactly.
//
//   fmt_ns_div1000(n)   repr(float(n) / 1000.0) for an integer n (ts/dur in us);
//                       exact decimal shortcut when |n| < 2^53 and |n|/1000 < 2^43
//                       (double spacing < 0.001, so n/1000 itself is the unique
//                       shortest round-tripping decimal), else via fmt_double.
//   fmt_double(x)       general shortest repr (Burger & Dybvig free-format digit
//                       generation on fixed-size big integers; rare values only).
//   fmt_u64 / fmt_i64 / fmt_i128 / fmt_int_of_double   exact integers.
#pragma once
#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define NF_HD __host__ __device__
#else
#define NF_HD
#endif

namespace nf {

// decimal digits of v (1 for 0)
NF_HD inline int dec_digits(uint64_t v) {
  int n = 1;
  if (v >= 10000000000000000ull) { n += 16; v /= 10000000000000000ull; }
  if (v >= 100000000ull) { n += 8; v /= 100000000ull; }
  if (v >= 10000ull) { n += 4; v /= 10000ull; }
  if (v >= 100ull) { n += 2; v /= 100ull; }
  if (v >= 10ull) n += 1;
  return n;
}

// digits written backwards from out + n: 64-bit work only per 8-digit chunk
NF_HD inline int fmt_u64(uint64_t v, char* out) {
  const int n = dec_digits(v);
  int k = n;
  while (v >= 100000000ull) {
    uint32_t c = (uint32_t)(v % 100000000ull);
    v /= 100000000ull;
    for (int j = 0; j < 8; j++) { out[--k] = (char)('0' + c % 10u); c /= 10u; }
  }
  uint32_t c = (uint32_t)v;
  do { out[--k] = (char)('0' + c % 10u); c /= 10u; } while (c);
  return n;
}

NF_HD inline int fmt_i64(int64_t v, char* out) {
  if (v < 0) { out[0] = '-'; return 1 + fmt_u64((uint64_t)0 - (uint64_t)v, out + 1); }
  return fmt_u64((uint64_t)v, out);
}

// signed 128-bit as (hi, lo)
NF_HD inline int fmt_i128(int64_t hi, uint64_t lo, char* out) {
  int n = 0;
  bool neg = hi < 0;
  uint64_t h = (uint64_t)hi, l = lo;
  if (neg) {  // negate
    l = ~l + 1;
    h = ~h + (l == 0 ? 1 : 0);
    out[n++] = '-';
  }
  if (h == 0) return n + fmt_u64(l, out + n);
  char tmp[48];
  int k = 0;
  while (h || l) {  // divide (h:l) by 10
    uint64_t rh = h % 10, qh = h / 10;
    // (rh * 2^64 + l) / 10
    uint64_t lo_hi = l >> 32, lo_lo = l & 0xFFFFFFFFull;
    uint64_t t1 = (rh << 32) | lo_hi;
    uint64_t q1 = t1 / 10, r1 = t1 % 10;
    uint64_t t2 = (r1 << 32) | lo_lo;
    uint64_t q2 = t2 / 10, r2 = t2 % 10;
    h = qh;
    l = (q1 << 32) | q2;
    tmp[k++] = (char)('0' + r2);
  }
  for (int i = 0; i < k; i++) out[n + i] = tmp[k - 1 - i];
  return n + k;
}

// ---------------------------------------------------------------------------
// fixed-size big unsigned integers (little-endian 32-bit limbs)

constexpr int kLimbs = 40;  // 1280 bits: covers every double's free-format state

struct Big {
  uint32_t w[kLimbs];
  int n;  // used limbs
};

NF_HD inline void big_set(Big& a, uint64_t v) {
  a.n = 0;
  while (v) { a.w[a.n++] = (uint32_t)v; v >>= 32; }
}
NF_HD inline void big_mul_small(Big& a, uint32_t m) {
  uint64_t c = 0;
  for (int i = 0; i < a.n; i++) {
    uint64_t t = (uint64_t)a.w[i] * m + c;
    a.w[i] = (uint32_t)t;
    c = t >> 32;
  }
  if (c) a.w[a.n++] = (uint32_t)c;
}
NF_HD inline void big_shl(Big& a, int s) {
  if (a.n == 0) return;
  int ws = s / 32, bs = s % 32;
  if (bs) {
    uint32_t c = 0;
    for (int i = 0; i < a.n; i++) {
      uint32_t v = a.w[i];
      a.w[i] = (v << bs) | c;
      c = v >> (32 - bs);
    }
    if (c) a.w[a.n++] = c;
  }
  if (ws) {
    for (int i = a.n - 1; i >= 0; i--) a.w[i + ws] = a.w[i];
    for (int i = 0; i < ws; i++) a.w[i] = 0;
    a.n += ws;
  }
}
NF_HD inline int big_cmp(const Big& a, const Big& b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int i = a.n - 1; i >= 0; i--)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
  return 0;
}
NF_HD inline void big_add(const Big& a, const Big& b, Big& r) {  // r = a + b (r may alias a)
  int n = a.n > b.n ? a.n : b.n;
  uint64_t c = 0;
  for (int i = 0; i < n; i++) {
    uint64_t t = (uint64_t)(i < a.n ? a.w[i] : 0) + (i < b.n ? b.w[i] : 0) + c;
    r.w[i] = (uint32_t)t;
    c = t >> 32;
  }
  r.n = n;
  if (c) r.w[r.n++] = (uint32_t)c;
}
NF_HD inline void big_sub(Big& a, const Big& b) {  // a -= b, a >= b
  int64_t br = 0;
  for (int i = 0; i < a.n; i++) {
    int64_t t = (int64_t)a.w[i] - (i < b.n ? b.w[i] : 0) - br;
    br = t < 0 ? 1 : 0;
    a.w[i] = (uint32_t)(t + (br << 32));
  }
  while (a.n && a.w[a.n - 1] == 0) a.n--;
}
NF_HD inline void big_pow10(Big& a, int k) {
  while (k >= 9) { big_mul_small(a, 1000000000u); k -= 9; }
  static const uint32_t p[9] = {1, 10, 100, 1000, 10000, 100000, 1000000, 10000000, 100000000};
  if (k) big_mul_small(a, p[k]);
}

// shortest digits of v > 0 (finite): returns count, *decpt such that v ~ 0.d1d2..dn x 10^decpt
NF_HD inline int shortest_digits(double v, char* digits, int* decpt) {
  uint64_t bits;
  memcpy(&bits, &v, 8);
  int be = (int)((bits >> 52) & 0x7FF);
  uint64_t f = bits & ((1ull << 52) - 1);
  int e;
  if (be == 0) { e = -1074; } else { f |= 1ull << 52; e = be - 1075; }
  const bool even = (f & 1) == 0;
  // r/s = v, m+ and m- are the distances to the neighbours (Burger & Dybvig)
  Big r, s, mp, mm;
  const bool boundary = be > 1 && f == (1ull << 52);
  if (e >= 0) {
    big_set(r, f); big_shl(r, e + (boundary ? 2 : 1));
    big_set(s, boundary ? 4 : 2);
    big_set(mp, 1); big_shl(mp, e + (boundary ? 1 : 0));
    big_set(mm, 1); big_shl(mm, e);
  } else {
    big_set(r, f); big_shl(r, boundary ? 2 : 1);
    big_set(s, 1); big_shl(s, -e + (boundary ? 2 : 1));
    big_set(mp, boundary ? 2 : 1);
    big_set(mm, 1);
  }
  // k = ceil(log10(high)); estimate then fix
  int k = 0;
  {
    double lg = (e + 52) * 0.30102999566398114 - 1e-10;  // ~log10(v) upper-ish
    k = (int)(lg >= 0 ? lg + 1 : lg);  // near estimate; corrected below
  }
  if (k >= 0) big_pow10(s, k);
  else { big_pow10(r, -k); big_pow10(mp, -k); big_pow10(mm, -k); }
  // fix: while (r + m+) >(=) s: k++, s *= 10 ; while (r + m+) * 10 <(=) s: k--, scale r, m
  for (;;) {
    Big h;
    big_add(r, mp, h);
    int c = big_cmp(h, s);
    if (even ? c >= 0 : c > 0) { big_mul_small(s, 10); k++; continue; }
    break;
  }
  for (;;) {
    Big h;
    big_add(r, mp, h);
    big_mul_small(h, 10);
    int c = big_cmp(h, s);
    if (even ? c < 0 : c <= 0) { big_mul_small(r, 10); big_mul_small(mp, 10); big_mul_small(mm, 10); k--; continue; }
    break;
  }
  *decpt = k;
  int n = 0;
  for (;;) {
    big_mul_small(r, 10); big_mul_small(mp, 10); big_mul_small(mm, 10);
    int d = 0;
    while (big_cmp(r, s) >= 0) { big_sub(r, s); d++; }
    int cl = big_cmp(r, mm);
    bool tc1 = even ? cl <= 0 : cl < 0;
    Big h;
    big_add(r, mp, h);
    int ch = big_cmp(h, s);
    bool tc2 = even ? ch >= 0 : ch > 0;
    if (!tc1 && !tc2) { digits[n++] = (char)('0' + d); continue; }
    if (tc1 && !tc2) { digits[n++] = (char)('0' + d); break; }
    if (!tc1 && tc2) { digits[n++] = (char)('0' + d + 1); break; }
    Big r2 = r;
    big_mul_small(r2, 2);
    int c2 = big_cmp(r2, s);
    if (c2 < 0 || (c2 == 0 && (d % 2) == 0)) digits[n++] = (char)('0' + d);
    else digits[n++] = (char)('0' + d + 1);
    break;
  }
  // a final digit of 10 cannot occur: tc2 with d == 9 would have raised k
  return n;
}

// CPython float_repr layout of sign + digits (format 'r', ADD_DOT_0)
NF_HD inline int layout_repr(bool neg, const char* dg, int nd, int decpt, char* out) {
  int n = 0;
  if (neg) out[n++] = '-';
  if (decpt <= -4 || decpt > 16) {
    out[n++] = dg[0];
    if (nd > 1) { out[n++] = '.'; for (int i = 1; i < nd; i++) out[n++] = dg[i]; }
    int ex = decpt - 1;
    out[n++] = 'e';
    out[n++] = ex < 0 ? '-' : '+';
    int ax = ex < 0 ? -ex : ex;
    if (ax < 10) { out[n++] = '0'; out[n++] = (char)('0' + ax); }
    else n += fmt_u64((uint64_t)ax, out + n);
    return n;
  }
  if (decpt <= 0) {
    out[n++] = '0'; out[n++] = '.';
    for (int i = 0; i < -decpt; i++) out[n++] = '0';
    for (int i = 0; i < nd; i++) out[n++] = dg[i];
    return n;
  }
  if (decpt >= nd) {
    for (int i = 0; i < nd; i++) out[n++] = dg[i];
    for (int i = nd; i < decpt; i++) out[n++] = '0';
    out[n++] = '.'; out[n++] = '0';
    return n;
  }
  for (int i = 0; i < decpt; i++) out[n++] = dg[i];
  out[n++] = '.';
  for (int i = decpt; i < nd; i++) out[n++] = dg[i];
  return n;
}

// json.dump(float): repr, with the json module's NaN/Infinity spellings
NF_HD inline int fmt_double(double v, char* out) {
  uint64_t bits;
  memcpy(&bits, &v, 8);
  bool neg = bits >> 63;
  uint64_t mag = bits & 0x7FFFFFFFFFFFFFFFull;
  if (mag > 0x7FF0000000000000ull) { out[0] = 'N'; out[1] = 'a'; out[2] = 'N'; return 3; }
  if (mag == 0x7FF0000000000000ull) {
    const char* s = neg ? "-Infinity" : "Infinity";
    int n = 0;
    while (s[n]) { out[n] = s[n]; n++; }
    return n;
  }
  if (mag == 0) {
    int n = 0;
    if (neg) out[n++] = '-';
    out[n++] = '0'; out[n++] = '.'; out[n++] = '0';
    return n;
  }
  double a = neg ? -v : v;
  // integral and < 1e16: digits + ".0"
  if (a < 1e16 && a == (double)(uint64_t)a) {
    int n = 0;
    if (neg) out[n++] = '-';
    n += fmt_u64((uint64_t)a, out + n);
    out[n++] = '.'; out[n++] = '0';
    return n;
  }
  char dg[32];
  int decpt = 0;
  int nd = shortest_digits(a, dg, &decpt);
  return layout_repr(neg, dg, nd, decpt, out);
}

// int -> float exactly as CPython (correct rounding, ties to even) for a signed 128-bit value
NF_HD inline double i128_to_double(int64_t hi, uint64_t lo) {
  bool neg = hi < 0;
  uint64_t h = (uint64_t)hi, l = lo;
  if (neg) { l = ~l + 1; h = ~h + (l == 0 ? 1 : 0); }
  double r;
  if (h == 0) {
    r = (double)l;  // round-to-nearest-even conversion
  } else {
    // value = h * 2^64 + l, h < 2^63: keep 64 significant bits + sticky, convert, scale
    int lz = 0;
    uint64_t t = h;
    while (!(t >> 63)) { t <<= 1; lz++; }
    int shift = 64 - lz;  // bits of h
    uint64_t top = (h << lz) | (lz ? (l >> (64 - lz)) : 0);
    uint64_t rest = lz ? (l << lz) : l;
    // round top (64 bits) to 53 bits with sticky from rest
    uint64_t keep = top >> 11, rem = top & 0x7FF;
    bool sticky = rest != 0;
    bool up = rem > 0x400 || (rem == 0x400 && (sticky || (keep & 1)));
    keep += up ? 1 : 0;
    r = (double)keep;  // exact (<= 2^53)
    int sc = shift + 11;  // value ~ keep * 2^(64 - lz - 53 + 64) ... keep * 2^(shift + 11)
    while (sc > 0) { int st = sc > 60 ? 60 : sc; r *= (double)(1ull << st); sc -= st; }
  }
  return neg ? -r : r;
}

// repr(float(n) / 1000.0) for a signed integer n (ns -> us)
NF_HD inline int fmt_ns_div1000(int64_t hi, uint64_t lo, char* out) {
  bool neg = hi < 0;
  uint64_t h = (uint64_t)hi, l = lo;
  if (neg) { l = ~l + 1; h = ~h + (l == 0 ? 1 : 0); }
  if (h == 0 && l < 8796093022208000ull) {  // |n| < 2^43 * 1000 (also < 2^53)
    int n = 0;
    if (neg && l) out[n++] = '-';
    uint64_t ip = l / 1000, fp = l % 1000;
    n += fmt_u64(ip, out + n);
    out[n++] = '.';
    if (fp == 0) { out[n++] = '0'; return n; }
    char d[3] = {(char)('0' + fp / 100), (char)('0' + fp / 10 % 10), (char)('0' + fp % 10)};
    int nd = d[2] != '0' ? 3 : (d[1] != '0' ? 2 : 1);
    for (int i = 0; i < nd; i++) out[n++] = d[i];
    return n;
  }
  double x = i128_to_double(hi, lo) / 1000.0;
  return fmt_double(x, out);
}

// int(x) of a finite double, printed exactly (Python int(float) truncates toward zero)
NF_HD inline int fmt_int_of_double(double x, char* out) {
  uint64_t bits;
  memcpy(&bits, &x, 8);
  bool neg = bits >> 63;
  int be = (int)((bits >> 52) & 0x7FF);
  uint64_t f = bits & ((1ull << 52) - 1);
  if (be < 1023) { out[0] = '0'; return 1; }  // |x| < 1 -> 0
  f |= 1ull << 52;
  int e = be - 1075;
  int n = 0;
  if (e <= 0) {
    uint64_t v = f >> (-e);
    if (neg && v) out[n++] = '-';
    return n + fmt_u64(v, out + n);
  }
  Big b;
  big_set(b, f);
  big_shl(b, e);
  if (neg) out[n++] = '-';
  // repeated division by 10^9
  char tmp[400];
  int k = 0;
  while (b.n) {
    uint64_t rem = 0;
    for (int i = b.n - 1; i >= 0; i--) {
      uint64_t cur = (rem << 32) | b.w[i];
      b.w[i] = (uint32_t)(cur / 1000000000u);
      rem = cur % 1000000000u;
    }
    while (b.n && b.w[b.n - 1] == 0) b.n--;
    for (int j = 0; j < 9; j++) { tmp[k++] = (char)('0' + rem % 10); rem /= 10; }
  }
  while (k > 1 && tmp[k - 1] == '0') k--;
  for (int i = 0; i < k; i++) out[n + i] = tmp[k - 1 - i];
  return n + k;
}

}  // namespace nf
