// slos_plan_to_json (include/slos_plan_json.h): the reference's canonical result
// serialisation, plan_to_json dp_scheduler.cpp:560-589, written byte-for-byte as
// nlohmann::json::dump() writes that object (the reference's JSON dependency; not
// vendored in the reference tree, its published serialisation rules restated here):
//   * objects are std::map-backed: keys in lexicographic order, compact ',' / ':';
//   * int64 values as plain decimal integers, bool as true / false;
//   * doubles: NaN / inf as null, zero as 0.0 / -0.0, otherwise the Grisu2 digits
//     (Loitsch 2010, "Printing Floating-Point Numbers Quickly and Accurately with
//     Integers", with the boundaries, cached powers (tools/gen_pow10_table.py) and
//     the weeding step of that paper) laid out as digits[000].0, dig.its,
//     0.[000]digits or d.igitse+XX (decimal exponent window [-4, 15], at least two
//     exponent digits);
//   * strings: '"', '\\', \b \f \n \r \t escaped, other bytes below 0x20 as \u00xx,
//     everything else verbatim; ill-formed UTF-8 is an error (nlohmann's dump throws).
// Host code only: no device is needed.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/slos_plan_json.h"

namespace {

// ---- shortest-digit doubles (Grisu2) -----------------------------------------

struct Fp {
  uint64_t f;
  int e;
};

struct Pow10 {
  uint64_t f;
  int e;
  int k;
};

const Pow10 kPow10[] = {
#include "slos_pow10.inc"
};
constexpr int kPow10MinK = -300, kPow10Step = 8;

Fp fp_mul(Fp x, Fp y) {  // upper 64 bits of the 128-bit product, rounded half up
  const unsigned __int128 p = (unsigned __int128)x.f * y.f;
  const uint64_t h = (uint64_t)(p >> 64) + (((uint64_t)p) >> 63);
  return {h, x.e + y.e + 64};
}

Fp fp_normalize(Fp x) {
  const int s = __builtin_clzll(x.f);
  return {x.f << s, x.e - s};
}

// v = w, with its boundaries m- / m+ (halfway to the neighbouring doubles),
// normalised to a common exponent
void boundaries(double v, Fp* w, Fp* lo, Fp* hi) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  const uint64_t E = bits >> 52, F = bits & ((1ull << 52) - 1);
  const Fp x = E == 0 ? Fp{F, 1 - 1075} : Fp{F | (1ull << 52), (int)E - 1075};
  const bool closer = F == 0 && E > 1;  // the lower neighbour is half as far
  const Fp mp = fp_normalize(Fp{2 * x.f + 1, x.e - 1});
  const Fp mm = closer ? Fp{4 * x.f - 1, x.e - 2} : Fp{2 * x.f - 1, x.e - 1};
  *hi = mp;
  *lo = Fp{mm.f << (mm.e - mp.e), mp.e};
  *w = fp_normalize(x);
}

int largest_pow10(uint32_t n, uint32_t* p) {
  static const uint32_t t[10] = {1u, 10u, 100u, 1000u, 10000u, 100000u, 1000000u, 10000000u, 100000000u,
                                 1000000000u};
  int k = 9;
  while (k > 0 && n < t[k]) --k;
  *p = t[k];
  return k + 1;
}

void weed(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
  // move the last digit down while the candidate stays inside the safe interval
  // and gets closer to w
  while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
    --buf[len - 1];
    rest += ten_k;
  }
}

// digits of v (positive, finite, nonzero) and the decimal exponent: v ~ digits * 10^dexp
int grisu2(char* buf, double v, int* dexp) {
  Fp w, lo, hi;
  boundaries(v, &w, &lo, &hi);
  // a cached power c = 10^-k with hi.e + c.e + 64 in [-60, -32]
  const int f = -60 - hi.e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);
  const Pow10& c = kPow10[(-kPow10MinK + k + (kPow10Step - 1)) / kPow10Step];
  const Fp cf{c.f, c.e};
  const Fp W = fp_mul(w, cf), L = fp_mul(lo, cf), H = fp_mul(hi, cf);
  const Fp Mm{L.f + 1, L.e}, Mp{H.f - 1, H.e};  // the safe interval
  int dx = -c.k;
  uint64_t delta = Mp.f - Mm.f, dist = Mp.f - W.f;
  const int sh = -Mp.e;
  const uint64_t one = 1ull << sh;
  uint32_t p1 = (uint32_t)(Mp.f >> sh);
  uint64_t p2 = Mp.f & (one - 1);
  int len = 0;
  uint32_t pw;
  int n = largest_pow10(p1, &pw);
  while (n > 0) {
    const uint32_t d = p1 / pw;
    p1 %= pw;
    buf[len++] = (char)('0' + d);
    --n;
    const uint64_t rest = ((uint64_t)p1 << sh) + p2;
    if (rest <= delta) {
      dx += n;
      weed(buf, len, dist, delta, rest, (uint64_t)pw << sh);
      *dexp = dx;
      return len;
    }
    pw /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    buf[len++] = (char)('0' + (p2 >> sh));
    p2 &= one - 1;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  dx -= m;
  weed(buf, len, dist, delta, p2, one);
  *dexp = dx;
  return len;
}

void put_double(std::string& o, double v) {
  if (!std::isfinite(v)) { o += "null"; return; }
  if (std::signbit(v)) { o += '-'; v = -v; }
  if (v == 0.0) { o += "0.0"; return; }
  char d[32];
  int dexp = 0;
  const int k = grisu2(d, v, &dexp);
  const int n = k + dexp;  // position of the decimal point
  if (k <= n && n <= 15) {  // digits[000].0
    o.append(d, k);
    o.append((size_t)(n - k), '0');
    o += ".0";
  } else if (0 < n && n <= 15) {  // dig.its
    o.append(d, n);
    o += '.';
    o.append(d + n, k - n);
  } else if (-4 < n && n <= 0) {  // 0.[000]digits
    o += "0.";
    o.append((size_t)(-n), '0');
    o.append(d, k);
  } else {  // d.igitse+XX
    o += d[0];
    if (k > 1) {
      o += '.';
      o.append(d + 1, k - 1);
    }
    o += 'e';
    int e = n - 1;
    o += e < 0 ? '-' : '+';
    if (e < 0) e = -e;
    if (e < 10) {
      o += '0';
      o += (char)('0' + e);
    } else {
      o += std::to_string(e);
    }
  }
}

// ---- strings -----------------------------------------------------------------

bool utf8_ok(const unsigned char* s, size_t n) {
  size_t i = 0;
  while (i < n) {
    const unsigned c = s[i];
    int len;
    unsigned lo = 0x80, hi = 0xBF;
    if (c < 0x80) { ++i; continue; }
    if (c >= 0xC2 && c <= 0xDF) len = 2;
    else if (c >= 0xE0 && c <= 0xEF) { len = 3; if (c == 0xE0) lo = 0xA0; if (c == 0xED) hi = 0x9F; }
    else if (c >= 0xF0 && c <= 0xF4) { len = 4; if (c == 0xF0) lo = 0x90; if (c == 0xF4) hi = 0x8F; }
    else return false;
    if (i + (size_t)len > n) return false;
    if (s[i + 1] < lo || s[i + 1] > hi) return false;
    for (int q = 2; q < len; ++q)
      if (s[i + q] < 0x80 || s[i + q] > 0xBF) return false;
    i += (size_t)len;
  }
  return true;
}

bool put_string(std::string& o, const char* s) {
  if (!s) s = "";
  const size_t n = std::strlen(s);
  if (!utf8_ok((const unsigned char*)s, n)) return false;
  o += '"';
  for (size_t i = 0; i < n; ++i) {
    const unsigned char c = (unsigned char)s[i];
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          static const char hx[] = "0123456789abcdef";
          o += "\\u00";
          o += hx[c >> 4];
          o += hx[c & 15];
        } else {
          o += (char)c;
        }
    }
  }
  o += '"';
  return true;
}

void put_int(std::string& o, int64_t v) { o += std::to_string(v); }

}  // namespace

extern "C" int slos_plan_to_json(const slos_input* in, const slos_result* r, double now_s, char* buf, int64_t cap,
                                 int64_t* len) {
  if (len) *len = 0;
  if (!in || !r) return SLOS_ERR_INVALID_PARAMETERS;
  std::string o;
  o.reserve(256 + 64 * (size_t)(r->n_entries > 0 ? r->n_entries : 0));
  bool ok = true;
  auto ids = [&](const int32_t* v, int32_t n) {  // pending indices -> ids
    o += '[';
    for (int32_t k = 0; k < n && ok; ++k) {
      if (k) o += ',';
      if (v[k] < 0 || v[k] >= in->n_pending) { ok = false; break; }
      ok = put_string(o, in->pending[v[k]].id);
    }
    o += ']';
  };
  // keys in std::map order: admitted, admitted_value, batches, declined, deferred,
  // exact_until_s, now_s, running_set_infeasible (dp_scheduler.cpp:561-587)
  o += "{\"admitted\":";
  ids(r->admitted, r->n_admitted);
  o += ",\"admitted_value\":";
  put_double(o, r->admitted_value);
  o += ",\"batches\":[";
  for (int64_t b = 0; b < r->n_batches && ok; ++b) {
    const slos_batch& cb = r->batches[b];
    if (b) o += ',';
    o += "{\"capacity_tokens\":";
    put_int(o, cb.capacity_tokens);
    o += ",\"end_s\":";
    put_double(o, cb.end_s);
    o += ",\"entries\":[";
    if (cb.first_entry < 0 || cb.n_entries < 0 || cb.first_entry + cb.n_entries > r->n_entries) { ok = false; break; }
    for (int64_t e = cb.first_entry; e < cb.first_entry + cb.n_entries && ok; ++e) {
      const slos_entry* ce = &r->entries[e];
      const int32_t ref = slos_entry_req(ce);
      const char* id = nullptr;
      if (ref >= 0 && ref < in->n_running) id = in->running[ref].id;
      else if (ref < 0 && -ref - 1 < in->n_pending) id = in->pending[-ref - 1].id;
      else { ok = false; break; }
      if (e > cb.first_entry) o += ',';
      o += "{\"decode\":";
      put_int(o, slos_entry_decode_tokens(ce));
      o += ",\"id\":";
      ok = put_string(o, id);
      o += ",\"prefill\":";
      put_int(o, slos_entry_prefill_tokens(ce));
      o += ",\"spec_len\":";
      put_int(o, slos_entry_spec_len(ce));
      o += '}';
    }
    o += "],\"prefill_budget_left\":";
    put_int(o, cb.prefill_budget_left);
    o += ",\"spec_step\":";
    put_int(o, cb.spec_step);
    o += ",\"start_s\":";
    put_double(o, cb.start_s);
    o += '}';
  }
  o += "],\"declined\":";
  if (ok) ids(r->declined, r->n_declined);
  o += ",\"deferred\":";
  if (ok) ids(r->deferred, r->n_deferred);
  o += ",\"exact_until_s\":";
  put_double(o, r->exact_until_s);
  o += ",\"now_s\":";
  put_double(o, now_s);
  o += ",\"running_set_infeasible\":";
  o += r->running_set_infeasible ? "true" : "false";
  o += '}';
  if (!ok) return SLOS_ERR_INVALID_PARAMETERS;
  if (len) *len = (int64_t)o.size();
  if (buf && cap > 0) {
    const size_t m = (size_t)cap > o.size() ? o.size() : (size_t)cap;
    std::memcpy(buf, o.data(), m);
    if ((size_t)cap > o.size()) buf[o.size()] = '\0';
  }
  return SLOS_OK;
}
