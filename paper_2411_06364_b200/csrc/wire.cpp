// wire.cpp — the data formats on either side of the scheduling path
// (SURVEY.md §8(f) row 2), host C++ behind the C-ABI:
//
//   * trace CSV in:  load_trace_csv / write_trace_csv (workload.hpp:127-194),
//     byte-identical output ("%.17g") and the same validation and messages;
//   * trace hash:    FNV-1a over the CSV bytes (metrics.hpp:320-328);
//   * report out:    to_json(report).dump(indent) (metrics.hpp:181-240),
//     byte-identical to nlohmann::ordered_json, including its double printer
//     (Grisu2 shortest-digits, Loitsch 2010, with nlohmann's boundary choices
//     and its "digits[.digits]" / "d.ddde+NN" layout rules).
//
// Not part of the device path: these run once per job on the host.
#include <errno.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cmath>
#include <string>
#include <vector>

#include "econoserve_b200.h"
#include "pow10_table.h"

namespace {

void put_err(char* err, size_t errlen, const std::string& m) {
  if (err && errlen) snprintf(err, errlen, "%s", m.c_str());
}

// --------------------------------------------------------------------------
// Grisu2 (shortest digits that round-trip, not always the shortest possible)
// --------------------------------------------------------------------------
struct Fp {  // f * 2^e
  uint64_t f;
  int e;
};

Fp fp_mul(Fp a, Fp b) {  // upper 64 bits of the 128-bit product, rounded (ties up)
  const unsigned __int128 p = (unsigned __int128)a.f * b.f + ((unsigned __int128)1 << 63);
  return Fp{(uint64_t)(p >> 64), a.e + b.e + 64};
}

Fp fp_normalize(Fp x) {
  while ((x.f >> 63) == 0) {
    x.f <<= 1;
    x.e--;
  }
  return x;
}

// m- / v / m+ of a positive finite double (the rounding interval of v)
void boundaries(double d, Fp* lo, Fp* v, Fp* hi) {
  uint64_t bits;
  memcpy(&bits, &d, sizeof(bits));
  const uint64_t E = bits >> 52, F = bits & ((1ULL << 52) - 1);
  const Fp x = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (1ULL << 52), (int)E - 1075};
  const bool closer_below = F == 0 && E > 1;  // the gap below a power of two is half as wide
  const Fp mp{2 * x.f + 1, x.e - 1};
  const Fp mm = closer_below ? Fp{4 * x.f - 1, x.e - 2} : Fp{2 * x.f - 1, x.e - 1};
  *hi = fp_normalize(mp);
  *lo = Fp{mm.f << (mm.e - hi->e), hi->e};
  *v = fp_normalize(x);
}

const int kAlpha = -60, kGamma = -32;

Pow10Entry cached_power(int e) {  // c = 10^-k with alpha <= e + c.e + 64 <= gamma
  const int f = kAlpha - e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);  // ceil(f * log10(2))
  const int idx = (-kPow10MinDecExp + k + (kPow10DecStep - 1)) / kPow10DecStep;
  return kPow10Table[idx];
}

int largest_pow10(uint32_t n, uint32_t* pow10) {  // 10^(k-1) <= n < 10^k
  static const uint32_t p[] = {1, 10, 100, 1000, 10000, 100000, 1000000, 10000000, 100000000, 1000000000};
  int k = 10;
  while (k > 1 && n < p[k - 1]) --k;
  *pow10 = p[k - 1];
  return k;
}

// Moves the last digit down while that brings V closer to w (staying >= M-).
void round_weed(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ulp) {
  while (rest < dist && delta - rest >= ulp && (rest + ulp < dist || dist - rest > rest + ulp - dist)) {
    buf[len - 1]--;
    rest += ulp;
  }
}

// Digits of some V in [M-, M+] with as few digits as this scaling allows.
void digit_gen(char* buf, int* len, int* dexp, Fp Mm, Fp w, Fp Mp) {
  uint64_t delta = Mp.f - Mm.f;
  uint64_t dist = Mp.f - w.f;
  const int sh = -Mp.e;
  const uint64_t one = 1ULL << sh;
  uint32_t p1 = (uint32_t)(Mp.f >> sh);
  uint64_t p2 = Mp.f & (one - 1);
  uint32_t pw;
  int n = largest_pow10(p1, &pw);
  while (n > 0) {
    const uint32_t d = p1 / pw;
    p1 %= pw;
    buf[(*len)++] = (char)('0' + d);
    --n;
    const uint64_t rest = ((uint64_t)p1 << sh) + p2;
    if (rest <= delta) {
      *dexp += n;
      round_weed(buf, *len, dist, delta, rest, (uint64_t)pw << sh);
      return;
    }
    pw /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    buf[(*len)++] = (char)('0' + (p2 >> sh));
    p2 &= one - 1;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  *dexp -= m;
  round_weed(buf, *len, dist, delta, p2, one);
}

// nlohmann's layout of digits d[0..k) * 10^dexp (min_exp -4, max_exp 15).
void layout(const char* dig, int k, int dexp, std::string& out) {
  const int n = k + dexp;  // position of the decimal point
  if (k <= n && n <= 15) {
    out.append(dig, (size_t)k);
    out.append((size_t)(n - k), '0');
    out += ".0";
  } else if (0 < n && n <= 15) {
    out.append(dig, (size_t)n);
    out += '.';
    out.append(dig + n, (size_t)(k - n));
  } else if (-4 < n && n <= 0) {
    out += "0.";
    out.append((size_t)(-n), '0');
    out.append(dig, (size_t)k);
  } else {
    out += dig[0];
    if (k > 1) {
      out += '.';
      out.append(dig + 1, (size_t)(k - 1));
    }
    int x = n - 1;
    out += 'e';
    out += x < 0 ? '-' : '+';
    if (x < 0) x = -x;
    char e[16];
    snprintf(e, sizeof(e), "%02d", x);
    out += e;
  }
}

void json_double(double v, std::string& out) {
  if (v != v || v - v != 0.0) {  // NaN / inf: nlohmann writes null
    out += "null";
    return;
  }
  if (v == 0.0) {
    out += std::signbit(v) ? "-0.0" : "0.0";
    return;
  }
  if (v < 0) {
    out += '-';
    v = -v;
  }
  Fp lo, x, hi;
  boundaries(v, &lo, &x, &hi);
  const Pow10Entry c = cached_power(hi.e);
  const Fp cf{c.f, c.e};
  const Fp W = fp_mul(x, cf), Wm = fp_mul(lo, cf), Wp = fp_mul(hi, cf);
  const Fp Mm{Wm.f + 1, Wm.e}, Mp{Wp.f - 1, Wp.e};
  char dig[32];
  int len = 0, dexp = -c.k;
  digit_gen(dig, &len, &dexp, Mm, W, Mp);
  layout(dig, len, dexp, out);
}

// --------------------------------------------------------------------------
// ordered JSON writer with nlohmann's dump(indent) whitespace rules
// --------------------------------------------------------------------------
struct Json {
  std::string s;
  int indent;  // < 0: compact
  std::vector<int> count;  // members written per open container

  explicit Json(int ind) : indent(ind) {}
  void nl(int depth) {
    if (indent < 0) return;
    s += '\n';
    s.append((size_t)(indent * depth), ' ');
  }
  void sep() {  // before a member / element of the innermost container
    if (count.back()++ > 0) s += ',';
    nl((int)count.size());
  }
  void key(const char* k) {
    sep();
    s += '"';
    s += k;
    s += indent < 0 ? "\":" : "\": ";
  }
  void open(char c) {
    s += c;
    count.push_back(0);
  }
  void close(char c) {
    const int n = count.back();
    count.pop_back();
    if (n > 0) nl((int)count.size());
    s += c;
  }
  void str(const char* v) {
    s += '"';
    for (const char* p = v; *p; ++p) {
      const unsigned char ch = (unsigned char)*p;
      if (ch == '"') s += "\\\"";
      else if (ch == '\\') s += "\\\\";
      else if (ch == '\n') s += "\\n";
      else if (ch == '\t') s += "\\t";
      else if (ch == '\r') s += "\\r";
      else if (ch == '\b') s += "\\b";
      else if (ch == '\f') s += "\\f";
      else if (ch < 0x20) {
        char b[8];
        snprintf(b, sizeof(b), "\\u%04x", ch);
        s += b;
      } else s += (char)ch;
    }
    s += '"';
  }
  void i64(int64_t v) { s += std::to_string(v); }
  void u64(uint64_t v) { s += std::to_string(v); }
  void f64(double v) { json_double(v, s); }
  void boolean(bool v) { s += v ? "true" : "false"; }
};

// --------------------------------------------------------------------------
// trace CSV (workload.hpp:127-194)
// --------------------------------------------------------------------------
const char* kHeader = "arrival_time,prompt_len,response_len";

// std::stod / std::stoll with the pos == size check of load_trace_csv.
bool parse_double(const std::string& f, double* v) {
  if (f.empty()) return false;
  errno = 0;
  char* end = nullptr;
  *v = strtod(f.c_str(), &end);
  if (end == f.c_str() || errno == ERANGE) return false;
  return (size_t)(end - f.c_str()) == f.size();
}
bool parse_ll(const std::string& f, long long* v) {
  if (f.empty()) return false;
  errno = 0;
  char* end = nullptr;
  *v = strtoll(f.c_str(), &end, 10);
  if (end == f.c_str() || errno == ERANGE) return false;
  return (size_t)(end - f.c_str()) == f.size();
}

int parse_csv(const char* text, int64_t len, const std::string& name, std::vector<EconoTraceRecord>* out,
              char* err, size_t errlen) {
  int64_t pos = 0;
  auto getline = [&](std::string& line) -> bool {
    if (pos >= len) return false;
    const char* nlp = (const char*)memchr(text + pos, '\n', (size_t)(len - pos));
    const int64_t end = nlp ? (int64_t)(nlp - text) : len;
    line.assign(text + pos, (size_t)(end - pos));
    pos = nlp ? end + 1 : len;
    return true;
  };
  std::string line;
  if (!getline(line)) return put_err(err, errlen, name + ": empty trace file"), ECONO_ECONFIG;
  if (!line.empty() && line.back() == '\r') line.pop_back();
  if (line != kHeader)
    return put_err(err, errlen, name + ": bad header, expected arrival_time,prompt_len,response_len"),
           ECONO_ECONFIG;
  int line_no = 1;
  double prev = -1.0;
  while (getline(line)) {
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    const std::string where = name + ": line " + std::to_string(line_no) + ": ";
    const size_t c1 = line.find(',');
    const size_t c2 = c1 == std::string::npos ? std::string::npos : line.find(',', c1 + 1);
    if (c1 == std::string::npos || c2 == std::string::npos)
      return put_err(err, errlen, where + "expected 3 fields"), ECONO_ECONFIG;
    EconoTraceRecord r;
    long long p = 0, q = 0;
    if (!parse_double(line.substr(0, c1), &r.arrival_time) || !parse_ll(line.substr(c1 + 1, c2 - c1 - 1), &p) ||
        !parse_ll(line.substr(c2 + 1), &q))
      return put_err(err, errlen, where + "malformed row: " + line), ECONO_ECONFIG;
    r.prompt_len = p;
    r.true_rl = q;
    if (r.prompt_len < 1) return put_err(err, errlen, where + "prompt_len must be >= 1"), ECONO_ECONFIG;
    if (r.true_rl < 1) return put_err(err, errlen, where + "response_len must be >= 1"), ECONO_ECONFIG;
    if (r.arrival_time < 0.0) return put_err(err, errlen, where + "negative arrival_time"), ECONO_ECONFIG;
    if (r.arrival_time < prev)
      return put_err(err, errlen, where + "arrival_time decreases within the trace"), ECONO_ECONFIG;
    prev = r.arrival_time;
    out->push_back(r);
  }
  return ECONO_OK;
}

void csv_row(const EconoTraceRecord& r, std::string& out) {
  char buf[96];
  const int n = snprintf(buf, sizeof(buf), "%.17g,%lld,%lld\n", r.arrival_time, (long long)r.prompt_len,
                         (long long)r.true_rl);
  out.append(buf, (size_t)n);
}

int copy_out(const std::string& s, char* out, int64_t cap, int64_t* len) {
  if (len) *len = (int64_t)s.size();
  if (out && cap > 0) {
    const size_t k = (size_t)cap - 1 < s.size() ? (size_t)cap - 1 : s.size();
    memcpy(out, s.data(), k);
    out[k] = 0;
  }
  return ECONO_OK;
}

}  // namespace

extern "C" {

int econo_parse_trace_csv(const char* text, int64_t len, const char* name, EconoTraceRecord* out, int64_t cap,
                          int64_t* n, char* err, size_t errlen) {
  std::vector<EconoTraceRecord> t;
  const int rc = parse_csv(text, len, name ? name : "<stream>", &t, err, errlen);
  if (rc) return rc;
  *n = (int64_t)t.size();
  if (out) memcpy(out, t.data(), sizeof(EconoTraceRecord) * (size_t)(cap < *n ? cap : *n));
  return ECONO_OK;
}

int econo_load_trace_csv(const char* path, EconoTraceRecord* out, int64_t cap, int64_t* n, char* err,
                         size_t errlen) {
  FILE* f = fopen(path, "rb");
  if (!f) return put_err(err, errlen, std::string("cannot open trace file: ") + path), ECONO_ECONFIG;
  std::string buf;
  char chunk[1 << 16];
  size_t k;
  while ((k = fread(chunk, 1, sizeof(chunk), f)) > 0) buf.append(chunk, k);
  fclose(f);
  return econo_parse_trace_csv(buf.data(), (int64_t)buf.size(), path, out, cap, n, err, errlen);
}

int econo_write_trace_csv(const EconoTraceRecord* trace, int64_t n, char* out, int64_t cap, int64_t* len) {
  std::string s = std::string(kHeader) + "\n";
  for (int64_t i = 0; i < n; ++i) csv_row(trace[i], s);
  return copy_out(s, out, cap, len);
}

uint64_t econo_trace_hash(const EconoTraceRecord* trace, int64_t n) {
  uint64_t h = 1469598103934665603ULL;
  auto feed = [&](const std::string& s) {
    for (unsigned char c : s) {
      h ^= c;
      h *= 1099511628211ULL;
    }
  };
  feed(std::string(kHeader) + "\n");
  std::string row;
  for (int64_t i = 0; i < n; ++i) {
    row.clear();
    csv_row(trace[i], row);
    feed(row);
  }
  return h;
}

int econo_json_double(double v, char* out, int64_t cap, int64_t* len) {
  std::string s;
  json_double(v, s);
  return copy_out(s, out, cap, len);
}

int econo_report_to_json(const char* policy, const EconoReport* r, const EconoRecord* recs, int64_t n_recs,
                         const char* config_json, int32_t indent, char* out, int64_t cap, int64_t* len) {
  Json j(indent);
  j.open('{');
  j.key("policy");
  j.str(policy ? policy : "");
  j.key("trace_hash");
  j.u64(r->trace_hash);
  j.key("aggregates");
  j.open('{');
  const struct { const char* k; double v; } fl[] = {
      {"mean_jct", r->mean_jct}, {"p5_jct", r->p5_jct}, {"p95_jct", r->p95_jct}, {"mean_tbt", r->mean_tbt},
      {"ssr", r->ssr}, {"throughput_rps", r->throughput_rps}, {"throughput_tps", r->throughput_tps},
      {"goodput_rps", r->goodput_rps}, {"normalized_latency", r->normalized_latency},
      {"mean_kvc_written", r->mean_kvc_written}, {"mean_kvc_allocated", r->mean_kvc_allocated},
      {"mean_forward_size", r->mean_forward_size}, {"allocation_failure_pct", r->allocation_failure_pct},
      {"tfs_hit_frac", r->tfs_hit_frac}, {"pt_admit_frac", r->pt_admit_frac}};
  for (const auto& x : fl) {
    j.key(x.k);
    j.f64(x.v);
  }
  j.key("iterations");
  j.i64(r->iterations);
  j.key("makespan");
  j.f64(r->makespan);
  j.key("preemptions");
  j.i64(r->preemptions);
  j.key("reserve_draws");
  j.i64(r->reserve_draws);
  j.key("hosted_slots");
  j.i64(r->hosted_slots);
  j.key("hosted_overruns");
  j.i64(r->hosted_overruns);
  j.key("mean_waiting");
  j.f64(r->mean_waiting);
  j.key("mean_execution");
  j.f64(r->mean_execution);
  j.key("mean_preemption");
  j.f64(r->mean_preemption);
  j.key("mean_scheduling");
  j.f64(r->mean_scheduling);
  j.key("iteration_completion_histogram");
  j.open('{');
  for (int i = 0; i < r->n_hist; ++i) {
    const std::string k = std::to_string(r->hist_count[i]);
    j.key(k.c_str());
    j.f64(r->hist_frac[i]);
  }
  j.close('}');
  j.close('}');
  if (config_json) {  // the experiment's config echo, pre-serialised at depth 1 (metrics.hpp:220)
    j.key("config");
    j.s += config_json;
  }
  if (recs) {
    j.key("records");
    j.open('[');
    for (int64_t i = 0; i < n_recs; ++i) {
      const EconoRecord& x = recs[i];
      j.sep();
      j.open('{');
      j.key("id");
      j.i64(x.id);
      j.key("arrival");
      j.f64(x.arrival);
      j.key("first_token_time");
      j.f64(x.first_token_time);
      j.key("completion_time");
      j.f64(x.completion_time);
      j.key("waiting_time");
      j.f64(x.waiting_time);
      j.key("execution_time");
      j.f64(x.execution_time);
      j.key("preemption_time");
      j.f64(x.preemption_time);
      j.key("scheduling_time_share");
      j.f64(x.scheduling_time_share);
      j.key("preempt_count");
      j.i64(x.preempt_count);
      j.key("reserve_draws");
      j.i64(x.reserve_draws);
      j.key("met_slo");
      j.boolean(x.met_slo != 0);
      j.key("prompt_len");
      j.i64(x.prompt_len);
      j.key("true_rl");
      j.i64(x.true_rl);
      j.key("slo_deadline");
      j.f64(x.slo_deadline);
      j.close('}');
    }
    j.close(']');
  }
  j.close('}');
  return copy_out(j.s, out, cap, len);
}

}  // extern "C"
