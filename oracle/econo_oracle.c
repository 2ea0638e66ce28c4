/*
 * econo_oracle.c — TEST INFRASTRUCTURE ONLY (the CPU oracle).
 *
 * A literal C restatement of the reference simulator's EconoServe
 * per-iteration scheduling step, written to be read side by side with
 * /root/reference/proj/include/econosim/ (abbreviations as in SURVEY.md:
 * E=engine.hpp, K=kvc.hpp, KP=kvc_pipeline.hpp, Q=queues.hpp,
 * W=workload.hpp, C=common.hpp, M=metrics.hpp, P=policies.hpp).
 * Data structures deliberately keep the reference's shapes (sorted vectors,
 * first-fit free list, linear walks) so the restatement is easy to audit;
 * it is the checker, never the thing measured or shipped.
 *
 * Third-party arithmetic restated (pinned by the toolchain):
 *   libstdc++ (GCC 13.3): mt19937_64, std::shuffle (stl_algo.h:3719-3795),
 *   uniform_int_distribution (uniform_int_dist.h:257-320, Lemire with
 *   128-bit products), generate_canonical<double,53> (random.tcc:3349-3380),
 *   normal_distribution polar method (random.tcc:1811-1844), lognormal
 *   (random.h:2358), exponential (random.h:4904), bernoulli (random.h:3745),
 *   uniform_real (random.h:1909); glibc 2.39 libm exp/log/sqrt/erfc/llround
 *   (called directly: same library as the reference binary).
 * Pinned against the compiled reference (oracle/_ref, oracle/Makefile) and
 * the committed fixtures in tests/golden/ (tests/gen_golden.py).
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off (no FMA contraction, like the
 * reference build).
 */
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "econoserve_b200.h"

typedef int64_t Tok;
typedef __uint128_t u128;

/* ------------------------------------------------------------------ */
/* growable arrays                                                      */
/* ------------------------------------------------------------------ */
#define VEC(T) struct { T* d; int64_t n, cap; }
#define VPUSH(v, x)                                                          \
  do {                                                                       \
    if ((v).n == (v).cap) {                                                  \
      (v).cap = (v).cap ? (v).cap * 2 : 8;                                   \
      (v).d = realloc((v).d, (size_t)(v).cap * sizeof(*(v).d));              \
    }                                                                        \
    (v).d[(v).n++] = (x);                                                    \
  } while (0)
#define VFREE(v) do { free((v).d); (v).d = NULL; (v).n = (v).cap = 0; } while (0)
#define VINSERT(v, pos, x)                                                   \
  do {                                                                       \
    VPUSH(v, x);                                                             \
    memmove(&(v).d[(pos) + 1], &(v).d[(pos)],                                \
            (size_t)((v).n - 1 - (pos)) * sizeof(*(v).d));                   \
    (v).d[(pos)] = (x);                                                      \
  } while (0)
#define VERASE(v, pos)                                                       \
  do {                                                                       \
    memmove(&(v).d[(pos)], &(v).d[(pos) + 1],                                \
            (size_t)((v).n - 1 - (pos)) * sizeof(*(v).d));                   \
    (v).n--;                                                                 \
  } while (0)

typedef VEC(int32_t) IVec;
typedef VEC(int64_t) LVec;

/* ------------------------------------------------------------------ */
/* errors (C:17-24): longjmp-free — functions return codes              */
/* ------------------------------------------------------------------ */
typedef struct { int code; char msg[512]; } Err;
static int fail(Err* e, int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(e->msg, sizeof(e->msg), fmt, ap);
  va_end(ap);
  e->code = code;
  return code;
}

/* ------------------------------------------------------------------ */
/* C:26-35                                                              */
/* ------------------------------------------------------------------ */
static Tok block_round(Tok t, Tok b) { return t <= 0 ? 0 : (t + b - 1) / b * b; }
static Tok ceil_tokens(double v) { return (Tok)ceil(v - 1e-9); }
static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */
static Tok tmax(Tok a, Tok b) { return (a < b) ? b : a; }
static Tok tmin(Tok a, Tok b) { return (b < a) ? b : a; }

/* ------------------------------------------------------------------ */
/* std::mt19937_64 (C:14)                                               */
/* ------------------------------------------------------------------ */
typedef struct { uint64_t x[312]; int i; } Mt;
static void mt_seed(Mt* m, uint64_t s) {
  m->x[0] = s;
  for (int i = 1; i < 312; ++i)
    m->x[i] = 6364136223846793005ULL * (m->x[i - 1] ^ (m->x[i - 1] >> 62)) + (uint64_t)i;
  m->i = 312;
}
static uint64_t mt_next(Mt* m) {
  if (m->i >= 312) {
    const uint64_t up = 0xFFFFFFFF80000000ULL, lo = 0x7FFFFFFFULL;
    for (int k = 0; k < 312; ++k) {
      uint64_t y = (m->x[k] & up) | (m->x[(k + 1) % 312] & lo);
      m->x[k] = m->x[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
    }
    m->i = 0;
  }
  uint64_t z = m->x[m->i++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= (z >> 43);
  return z;
}

/* uniform_int_distribution::_S_nd (uniform_int_dist.h:257-282): Lemire. */
static uint64_t lemire(Mt* g, uint64_t range) {
  u128 prod = (u128)mt_next(g) * (u128)range;
  uint64_t low = (uint64_t)prod;
  if (low < range) {
    uint64_t thr = (0 - range) % range;
    while (low < thr) {
      prod = (u128)mt_next(g) * (u128)range;
      low = (uint64_t)prod;
    }
  }
  return (uint64_t)(prod >> 64);
}
/* uniform_int_distribution<T>{a,b} over a 64-bit engine (uniform_int_dist.h:296-320). */
static uint64_t uniform_u64(Mt* g, uint64_t a, uint64_t b) {
  const uint64_t urange = b - a;
  if (urange < UINT64_MAX) return lemire(g, urange + 1) + a;
  return mt_next(g) + a; /* urngrange == urange: raw draw */
}
/* generate_canonical<double,53> (random.tcc:3349-3380): one draw / 2^64. */
static double canonical(Mt* g) {
  double r = (double)mt_next(g) / 18446744073709551616.0;
  if (r >= 1.0) r = nextafter(1.0, 0.0);
  return r;
}
/* normal_distribution polar method (random.tcc:1811-1844); `saved` persists
 * for the lifetime of one distribution object. */
typedef struct { int avail; double saved; } Normal;
static double normal_draw(Normal* nd, Mt* g, double mean, double stddev) {
  double ret;
  if (nd->avail) {
    nd->avail = 0;
    ret = nd->saved;
  } else {
    double x, y, r2;
    do {
      x = 2.0 * canonical(g) - 1.0;
      y = 2.0 * canonical(g) - 1.0;
      r2 = x * x + y * y;
    } while (r2 > 1.0 || r2 == 0.0);
    const double mult = sqrt(-2 * log(r2) / r2);
    nd->saved = x * mult;
    nd->avail = 1;
    ret = y * mult;
  }
  ret = ret * stddev + mean;
  return ret;
}

/* std::shuffle (stl_algo.h:3719-3795) over an array of `sz`-byte elements. */
static void swap_elems(char* base, size_t sz, uint64_t i, uint64_t j) {
  if (i == j) return;
  char tmp[64];
  memcpy(tmp, base + i * sz, sz);
  memcpy(base + i * sz, base + j * sz, sz);
  memcpy(base + j * sz, tmp, sz);
}
static void std_shuffle(void* arr, uint64_t n, size_t sz, Mt* g) {
  char* base = (char*)arr;
  if (n == 0) return;
  const uint64_t urngrange = UINT64_MAX;
  if (urngrange / n >= n) {
    uint64_t i = 1;
    if ((n % 2) == 0) {
      swap_elems(base, sz, i, uniform_u64(g, 0, 1));
      ++i;
    }
    while (i != n) {
      const uint64_t swap_range = i + 1;
      const uint64_t x = uniform_u64(g, 0, swap_range * (swap_range + 1) - 1);
      const uint64_t p1 = x / (swap_range + 1), p2 = x % (swap_range + 1);
      swap_elems(base, sz, i, p1);
      ++i;
      swap_elems(base, sz, i, p2);
      ++i;
    }
    return;
  }
  for (uint64_t i = 1; i != n; ++i) swap_elems(base, sz, i, uniform_u64(g, 0, i));
}

/* ------------------------------------------------------------------ */
/* predictor (W:200-268)                                                */
/* ------------------------------------------------------------------ */
static Tok quantize_up(Tok v, Tok q) { return q <= 1 ? v : block_round(v, q); } /* W:221-223 */

static Tok predict_rl(Tok true_rl, const EconoOptions* o, Mt* rng) { /* W:228-264 */
  switch (o->pred_model) {
    case ECONO_PRED_ORACLE:
      return quantize_up(true_rl, o->pred_quantum);
    case ECONO_PRED_LOGNORMAL: {
      Normal n = {0, 0.0};
      const double v = (double)true_rl * exp(normal_draw(&n, rng, 0.0, o->pred_sigma));
      return quantize_up(tmax(1, (Tok)llround(v)), o->pred_quantum);
    }
    case ECONO_PRED_BUCKET: {
      const double t = (double)true_rl;
      const Tok lo_in = tmax(1, ceil_tokens(t * (1.0 - o->pred_tolerance)));
      const Tok hi_in = (Tok)floor(t * (1.0 + o->pred_tolerance) + 1e-9);
      if (canonical(rng) < o->pred_accuracy) { /* bernoulli (random.h:3745) */
        const Tok b = tmax(lo_in, hi_in);
        const Tok v = (Tok)uniform_u64(rng, (uint64_t)lo_in, (uint64_t)b);
        return quantize_up(v, o->pred_quantum);
      }
      const double a = o->pred_tolerance, bb = 2.0 * o->pred_tolerance + 0.25;
      const double u = canonical(rng) * (bb - a) + a; /* uniform_real (random.h:1909) */
      Tok v;
      if (canonical(rng) < 0.5) {
        v = (Tok)llround(t * (1.0 + u));
        if (v <= hi_in) v = hi_in + 1;
      } else {
        v = (Tok)llround(t * (1.0 - u));
        if (v >= lo_in) v = lo_in - 1;
        if (v < 1) v = hi_in + 1;
      }
      return quantize_up(tmax(1, v), o->pred_quantum);
    }
  }
  return true_rl;
}
static Tok apply_padding(Tok p, double ratio) { return ceil_tokens((double)p * (1.0 + ratio)); } /* W:266-268 */

/* ------------------------------------------------------------------ */
/* ordering keys (Q:13-69)                                              */
/* ------------------------------------------------------------------ */
typedef struct { int db, kb; Tok len; uint64_t seq; int fifo; } Key;

static int key_less(const Key* a, const Key* b) { /* Q:44-50 */
  if (a->fifo || b->fifo) return a->seq < b->seq;
  if (a->db != b->db) return a->db < b->db;
  if (a->kb != b->kb) return a->kb > b->kb;
  if (a->len != b->len) return a->len > b->len;
  return a->seq < b->seq;
}
static int bucket_d(const EconoOptions* o, double v) { /* Q:30-33 upper_bound */
  int i = 0;
  while (i < o->n_deadline_bounds && !(v < o->deadline_bounds[i])) ++i;
  return i;
}
static int bucket_k(const EconoOptions* o, Tok v) {
  int i = 0;
  while (i < o->n_kvc_bounds && !(v < o->kvc_bounds[i])) ++i;
  return i;
}
static Key make_key(const EconoOptions* o, int enabled, double slack, Tok occ, Tok len,
                    uint64_t seq) { /* Q:59-69 */
  Key k = {0, 0, 0, seq, !enabled};
  if (enabled) {
    k.db = bucket_d(o, dmax(0.0, slack));
    k.kb = bucket_k(o, occ);
    k.len = len;
  }
  return k;
}

/* ------------------------------------------------------------------ */
/* queues (Q:75-204)                                                    */
/* ------------------------------------------------------------------ */
typedef struct { int32_t id; Key key; } PtEntry;
typedef struct {
  uint64_t group_id;
  Tok padded_rl;
  IVec members;
  double formed_at, min_deadline;
  Tok max_occupied;
  Key key;
} Group;

static void group_copy(Group* dst, const Group* src) {
  *dst = *src;
  dst->members.d = NULL;
  dst->members.n = dst->members.cap = 0;
  for (int64_t i = 0; i < src->members.n; ++i) VPUSH(dst->members, src->members.d[i]);
}

/* ------------------------------------------------------------------ */
/* KVC allocator (K:35-424)                                             */
/* ------------------------------------------------------------------ */
typedef struct { Tok start, len; } Region;
typedef struct { int32_t host_id, hosted_id; Tok start_offset, length, deadline_usage, abs_start; } Slot;
typedef struct { VEC(Region) regions; Tok total; int present; } Holding;
typedef VEC(Slot) SlotVec;

typedef struct {
  Tok capacity, block, reserve_cap, general_cap, free_total, reserved_used, written_total;
  VEC(Region) free_;         /* std::map<Tokens,Tokens>: kept sorted by start */
  Holding* alloc;            /* indexed by id */
  IVec alloc_ids;            /* ids with a holding, ascending (map order) */
  Tok* reserved; char* has_reserved;
  Tok* written; char* has_written;
  SlotVec slots;
  int32_t n;
} Kvc;

static int kvc_init(Kvc* k, Tok capacity, Tok block, double rf, int32_t n, Err* e) { /* K:37-47 */
  memset(k, 0, sizeof(*k));
  if (capacity < 1) return fail(e, ECONO_ECONFIG, "kvc capacity must be >= 1");
  if (block < 1) return fail(e, ECONO_ECONFIG, "kvc block_size must be >= 1");
  if (rf < 0.0 || rf >= 1.0) return fail(e, ECONO_ECONFIG, "reserved_fraction must be in [0, 1)");
  k->capacity = capacity;
  k->block = block;
  k->reserve_cap = (Tok)llround(rf * (double)capacity);
  k->general_cap = capacity - k->reserve_cap;
  k->free_total = k->general_cap;
  if (k->general_cap > 0) { Region g = {0, k->general_cap}; VPUSH(k->free_, g); }
  k->n = n;
  k->alloc = calloc((size_t)n, sizeof(Holding));
  k->reserved = calloc((size_t)n, sizeof(Tok));
  k->has_reserved = calloc((size_t)n, 1);
  k->written = calloc((size_t)n, sizeof(Tok));
  k->has_written = calloc((size_t)n, 1);
  return 0;
}
static void kvc_free(Kvc* k) {
  if (k->alloc)
    for (int32_t i = 0; i < k->n; ++i) VFREE(k->alloc[i].regions);
  free(k->alloc); free(k->reserved); free(k->has_reserved); free(k->written); free(k->has_written);
  VFREE(k->free_); VFREE(k->alloc_ids); VFREE(k->slots);
}
static Tok kvc_held(const Kvc* k, int32_t id) { return k->alloc[id].present ? k->alloc[id].total : 0; } /* K:59-62 */
static Tok kvc_allocated_total(const Kvc* k) { return k->general_cap - k->free_total; } /* K:75 */
static double kvc_allocated_fraction(const Kvc* k) { /* K:77-79 */
  return (double)(kvc_allocated_total(k) + k->reserved_used) / (double)k->capacity;
}
static double kvc_utilization(const Kvc* k) { return (double)k->written_total / (double)k->capacity; } /* K:83-85 */
static void kvc_add_written(Kvc* k, int32_t id, Tok d) { /* K:87-90 */
  k->has_written[id] = 1;
  k->written[id] += d;
  k->written_total += d;
}
static void kvc_drop_written(Kvc* k, int32_t id, Tok delta) { /* K:91-97 */
  if (!k->has_written[id]) return;
  const Tok d = tmin(delta, k->written[id]);
  k->written[id] -= d;
  k->written_total -= d;
}
static Tok kvc_written(const Kvc* k, int32_t id) { return k->has_written[id] ? k->written[id] : 0; }

static Holding* holding_get(Kvc* k, int32_t id) { /* alloc_[id] (creates the map node) */
  Holding* h = &k->alloc[id];
  if (!h->present) {
    h->present = 1;
    h->total = 0;
    h->regions.n = 0;
    int64_t lo = 0, hi = k->alloc_ids.n;
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      if (k->alloc_ids.d[mid] < id) lo = mid + 1; else hi = mid;
    }
    VINSERT(k->alloc_ids, lo, id);
  }
  return h;
}
static void holding_erase(Kvc* k, int32_t id) {
  k->alloc[id].present = 0;
  k->alloc[id].regions.n = 0;
  k->alloc[id].total = 0;
  for (int64_t i = 0; i < k->alloc_ids.n; ++i)
    if (k->alloc_ids.d[i] == id) { VERASE(k->alloc_ids, i); break; }
}

static int slot_index(const Kvc* k, int32_t hosted) { /* slot_of K:247-251 */
  for (int64_t i = 0; i < k->slots.n; ++i)
    if (k->slots.d[i].hosted_id == hosted) return (int)i;
  return -1;
}
static int owner_or_slot_host(const Kvc* k, const Slot* s, int32_t owner) { /* K:405-410 */
  if (s->host_id == owner) return 1;
  for (int64_t i = 0; i < k->slots.n; ++i)
    if (k->slots.d[i].hosted_id == s->host_id) return owner_or_slot_host(k, &k->slots.d[i], owner);
  return 0;
}
typedef struct { int32_t id; int64_t ri; Tok old_start, len; } CEntry;
static int centry_cmp(const void* a, const void* b) {
  const CEntry* x = a; const CEntry* y = b;
  return (x->old_start > y->old_start) - (x->old_start < y->old_start);
}
static void kvc_compact(Kvc* k) { /* K:372-401 */
  VEC(CEntry) es = {0};
  for (int64_t a = 0; a < k->alloc_ids.n; ++a) {
    const int32_t id = k->alloc_ids.d[a];
    Holding* h = &k->alloc[id];
    for (int64_t i = 0; i < h->regions.n; ++i) {
      CEntry c = {id, i, h->regions.d[i].start, h->regions.d[i].len};
      VPUSH(es, c);
    }
  }
  qsort(es.d, (size_t)es.n, sizeof(CEntry), centry_cmp); /* starts are distinct */
  Tok cursor = 0;
  for (int64_t i = 0; i < es.n; ++i) {
    const CEntry* c = &es.d[i];
    const Tok delta = cursor - c->old_start;
    if (delta != 0) {
      k->alloc[c->id].regions.d[c->ri].start = cursor;
      for (int64_t s = 0; s < k->slots.n; ++s) {
        Slot* sl = &k->slots.d[s];
        if (sl->abs_start >= c->old_start && sl->abs_start < c->old_start + c->len &&
            owner_or_slot_host(k, sl, c->id))
          sl->abs_start += delta;
      }
    }
    cursor += c->len;
  }
  k->free_.n = 0;
  if (cursor < k->general_cap) { Region g = {cursor, k->general_cap - cursor}; VPUSH(k->free_, g); }
  k->free_total = k->general_cap - cursor;
  VFREE(es);
}
static int kvc_take(Kvc* k, Tok need, Tok* start) { /* K:334-348 */
  if (need > k->free_total) return 0;
  for (int64_t i = 0; i < k->free_.n; ++i) {
    if (k->free_.d[i].len >= need) {
      const Tok s = k->free_.d[i].start;
      const Tok rest = k->free_.d[i].len - need;
      VERASE(k->free_, i);
      if (rest > 0) { Region g = {s + need, rest}; VINSERT(k->free_, i, g); }
      k->free_total -= need;
      *start = s;
      return 1;
    }
  }
  kvc_compact(k);
  return kvc_take(k, need, start);
}
static int kvc_give_back(Kvc* k, Tok start, Tok len, Err* e) { /* K:350-369 */
  if (len <= 0) return 0;
  int64_t pos = 0;
  while (pos < k->free_.n && k->free_.d[pos].start < start) ++pos;
  if (pos < k->free_.n && k->free_.d[pos].start == start)
    return fail(e, ECONO_ESIM, "double free");
  Region g = {start, len};
  VINSERT(k->free_, pos, g);
  if (pos + 1 < k->free_.n && k->free_.d[pos].start + k->free_.d[pos].len == k->free_.d[pos + 1].start) {
    k->free_.d[pos].len += k->free_.d[pos + 1].len;
    VERASE(k->free_, pos + 1);
  }
  if (pos > 0 && k->free_.d[pos - 1].start + k->free_.d[pos - 1].len == k->free_.d[pos].start) {
    k->free_.d[pos - 1].len += k->free_.d[pos].len;
    VERASE(k->free_, pos);
  }
  k->free_total += len;
  return 0;
}
static int kvc_allocate_exact(Kvc* k, int32_t id, Tok length, int* ok, Err* e) { /* K:104-116 */
  if (length < 1) return fail(e, ECONO_ESIM, "allocate_exact: length must be >= 1");
  if (k->alloc[id].present) return fail(e, ECONO_ESIM, "allocate_exact: id already allocated");
  const Tok need = block_round(length, k->block);
  Tok s;
  if (!kvc_take(k, need, &s)) { *ok = 0; return 0; }
  Holding* h = holding_get(k, id);
  Region r = {s, need};
  VPUSH(h->regions, r);
  h->total = need;
  *ok = 1;
  return 0;
}
static int kvc_grow_exact(Kvc* k, int32_t id, Tok extra, int* ok, Err* e) { /* K:120-131 */
  if (extra < 1) return fail(e, ECONO_ESIM, "grow_exact: extra must be >= 1");
  if (!k->alloc[id].present) return fail(e, ECONO_ESIM, "grow_exact: id has no allocation");
  const Tok need = block_round(extra, k->block);
  Tok s;
  if (!kvc_take(k, need, &s)) { *ok = 0; return 0; }
  Region r = {s, need};
  VPUSH(k->alloc[id].regions, r);
  k->alloc[id].total += need;
  *ok = 1;
  return 0;
}
static int kvc_draw_reserved(Kvc* k, int32_t id, Tok tokens) { /* K:144-150 (tokens >= 1 at every call site) */
  if (k->reserved_used + tokens > k->reserve_cap) return 0;
  k->reserved_used += tokens;
  k->has_reserved[id] = 1;
  k->reserved[id] += tokens;
  return 1;
}
static Tok kvc_release_reserved(Kvc* k, int32_t id) { /* K:152-159 */
  if (!k->has_reserved[id]) return 0;
  const Tok f = k->reserved[id];
  k->reserved_used -= f;
  k->reserved[id] = 0;
  k->has_reserved[id] = 0;
  return f;
}
static void kvc_remove_slot(Kvc* k, int32_t hosted) { /* K:229-243 */
  const int oi = slot_index(k, hosted);
  if (oi >= 0) {
    const Slot own = k->slots.d[oi];
    for (int64_t i = 0; i < k->slots.n; ++i) {
      Slot* s = &k->slots.d[i];
      if (s->host_id != hosted) continue;
      if (s->abs_start >= own.abs_start && s->abs_start + s->length <= own.abs_start + own.length) {
        s->host_id = own.host_id;
        s->start_offset += own.start_offset;
        s->deadline_usage = s->start_offset;
      }
    }
  }
  int64_t w = 0;
  for (int64_t i = 0; i < k->slots.n; ++i)
    if (k->slots.d[i].hosted_id != hosted) k->slots.d[w++] = k->slots.d[i];
  k->slots.n = w;
}
static int region_cmp(const void* a, const void* b) {
  const Region* x = a; const Region* y = b;
  return (x->start > y->start) - (x->start < y->start);
}
static int kvc_release(Kvc* k, int32_t id, Err* e) { /* K:165-217 */
  const int had = k->alloc[id].present;
  if (!had && !k->has_reserved[id] && slot_index(k, id) < 0)
    return fail(e, ECONO_ESIM, "release: unknown id");
  kvc_remove_slot(k, id);
  if (had) {
    VEC(Region) promoted = {0};
    for (int64_t i = 0; i < k->slots.n; ++i) {
      const Slot s = k->slots.d[i];
      if (s.host_id != id) continue;
      Holding* hs = holding_get(k, s.hosted_id);
      Region r = {s.abs_start, s.length};
      VPUSH(hs->regions, r);
      hs->total += s.length;
      VPUSH(promoted, r);
    }
    int64_t w = 0;
    for (int64_t i = 0; i < k->slots.n; ++i)
      if (k->slots.d[i].host_id != id) k->slots.d[w++] = k->slots.d[i];
    k->slots.n = w;
    qsort(promoted.d, (size_t)promoted.n, sizeof(Region), region_cmp);
    Holding* h = &k->alloc[id];
    for (int64_t ri = 0; ri < h->regions.n; ++ri) {
      const Region r = h->regions.d[ri];
      Tok cursor = r.start;
      const Tok end = r.start + r.len;
      for (int64_t pi = 0; pi < promoted.n; ++pi) {
        const Region p = promoted.d[pi];
        if (p.start >= end || p.start + p.len <= r.start) continue;
        if (p.start > cursor && kvc_give_back(k, cursor, p.start - cursor, e)) return e->code;
        cursor = tmax(cursor, p.start + p.len);
      }
      if (cursor < end && kvc_give_back(k, cursor, end - cursor, e)) return e->code;
    }
    holding_erase(k, id);
    VFREE(promoted);
  }
  kvc_release_reserved(k, id);
  if (k->has_written[id]) {
    k->written_total -= k->written[id];
    k->written[id] = 0;
    k->has_written[id] = 0;
  }
  return 0;
}
static int contained_in(const Kvc* k, Tok start, Tok len, int32_t id) { /* K:318-324 */
  if (!k->alloc[id].present) return 0;
  const Holding* h = &k->alloc[id];
  for (int64_t i = 0; i < h->regions.n; ++i)
    if (start >= h->regions.d[i].start && start + len <= h->regions.d[i].start + h->regions.d[i].len)
      return 1;
  return 0;
}
static int inside_slot_of(const Kvc* k, Tok start, Tok len, int32_t id) { /* K:327-332 */
  for (int64_t i = 0; i < k->slots.n; ++i) {
    const Slot* s = &k->slots.d[i];
    if (s->hosted_id == id && start >= s->abs_start && start + len <= s->abs_start + s->length) return 1;
  }
  return 0;
}
static int kvc_add_slot(Kvc* k, const Slot* s, Err* e) { /* K:219-224 */
  if (!contained_in(k, s->abs_start, s->length, s->host_id) &&
      !inside_slot_of(k, s->abs_start, s->length, s->host_id))
    return fail(e, ECONO_ESIM, "hosting slot outside the host's space");
  VPUSH(k->slots, *s);
  return 0;
}

/* ------------------------------------------------------------------ */
/* engine (E:79-1042), econoserve family only                           */
/* ------------------------------------------------------------------ */
enum { ST_WAITING_PT = 0, ST_RUNNING = 1, ST_WAITING_GT = 2, ST_PREEMPTED = 3, ST_DONE = 4 }; /* R:10 */

typedef struct {
  double arrival; Tok prompt, true_rl;
  Tok predicted_rl, padded_rl;
  double slo_deadline;
  Tok generated;
  int state;
  Tok occupied;
  double waiting_time, preemption_time, execution_time;
  Tok allowance, generated_at_epoch, prefill_done, prefill_target;
  double dispatch_time, first_token_time, completion_clock, last_enqueue_time;
  int preempt_count, reserve_draws;
  int hosted, was_preempted, alloc_failure_flag;
} Req; /* R:24-58 */

typedef struct { int32_t id; Tok tokens; } PtIter;

typedef struct {
  EconoOptions opt;
  int ordered, grouping;
  Kvc kvc;
  Mt rng, pred_rng;
  Req* reqs;
  int32_t n;
  int64_t arrival_cursor;
  double clock;
  int64_t iter, completed;
  /* PtQueue */
  VEC(PtEntry) ptq;
  uint64_t pt_next_seq;
  /* GtQueue */
  VEC(Group) gtq;
  uint64_t next_group_id, gt_next_seq;
  IVec running, admitted;
  VEC(PtIter) pt_iter;
  int64_t exam_count;
  int pts_admitted_iter, pt_admittable_iter;
  double* penalty_extra;
  double* sched_share;
  int64_t alloc_failures, hosted_total, hosted_overruns;
  double t_p, t_g;
  VEC(EconoEvent) events;
  VEC(EconoSample) samples;
  int64_t steps, pt_dispatched, gt_scheduled;
  Err err;
  int faulted;
} Eng;

static double iteration_time(Tok fs, const EconoOptions* o) { /* E:46-51 (cost.tfs = policy.tfs, E:98) */
  const Tok base = tmin(fs, o->tfs);
  const Tok over = tmax(0, fs - o->tfs);
  const double over_rate = o->t_token_over < 0.0 ? o->t_token : o->t_token_over;
  return o->t_base + o->t_token * (double)base + over_rate * (double)over;
}

static void logev(Eng* g, int kind, int32_t id, int64_t a, int64_t b) { /* E:211-214 */
  if (!g->opt.record_events) return;
  EconoEvent ev = {g->iter, g->clock, kind, id, a, b};
  VPUSH(g->events, ev);
}

static void pt_insert_batch(Eng* g, PtEntry* add, int64_t k);

static void ingest_arrivals(Eng* g) { /* E:216-235 */
  int64_t first = g->arrival_cursor;
  while (g->arrival_cursor < g->n && g->reqs[g->arrival_cursor].arrival <= g->clock + 1e-12) {
    const int32_t id = (int32_t)g->arrival_cursor++;
    logev(g, ECONO_EV_ARRIVE, id, 0, 0);
  }
  const int64_t k = g->arrival_cursor - first;
  if (k == 0) return;
  PtEntry* add = malloc((size_t)k * sizeof(PtEntry));
  for (int64_t i = 0; i < k; ++i) {
    const int32_t id = (int32_t)(first + i);
    const Req* r = &g->reqs[id];
    add[i].id = id;
    add[i].key = make_key(&g->opt, g->ordered, r->slo_deadline - g->clock, 0, r->prompt, g->pt_next_seq++);
  }
  pt_insert_batch(g, add, k);
  free(add);
}

/* PtQueue::insert_ordered (Q:85-92) applied to a batch. Each insert is an
 * upper_bound insert and every key carries a larger seq than any queued key,
 * so k successive inserts equal one stable merge of the (stably key-sorted)
 * batch into the queue; done that way so 1M-request bursts stay O(n log n). */
static int pt_cmp(const void* a, const void* b) {
  const PtEntry* x = a; const PtEntry* y = b;
  if (key_less(&x->key, &y->key)) return -1;
  if (key_less(&y->key, &x->key)) return 1;
  return (x->key.seq > y->key.seq) - (x->key.seq < y->key.seq);
}
static void pt_insert_batch(Eng* g, PtEntry* add, int64_t k) {
  if (k == 1) {
    int64_t lo = 0, hi = g->ptq.n;
    while (lo < hi) { /* upper_bound */
      int64_t mid = (lo + hi) / 2;
      if (key_less(&add[0].key, &g->ptq.d[mid].key)) hi = mid; else lo = mid + 1;
    }
    VINSERT(g->ptq, lo, add[0]);
    return;
  }
  qsort(add, (size_t)k, sizeof(PtEntry), pt_cmp); /* keys unique by seq: stable */
  PtEntry* out = malloc((size_t)(g->ptq.n + k) * sizeof(PtEntry));
  int64_t i = 0, j = 0, w = 0;
  while (i < g->ptq.n || j < k) {
    if (j >= k || (i < g->ptq.n && !key_less(&add[j].key, &g->ptq.d[i].key)))
      out[w++] = g->ptq.d[i++];
    else
      out[w++] = add[j++];
  }
  free(g->ptq.d);
  g->ptq.d = out;
  g->ptq.n = g->ptq.cap = w;
}

static Tok seq_target(const Eng* g, const Req* r) { /* E:238-240 */
  return block_round(r->prompt + r->generated + r->padded_rl, g->kvc.block);
}
static Tok gt_member_demand(const Eng* g, int32_t id) { /* E:242-247 */
  const Req* r = &g->reqs[id];
  const Tok delta = seq_target(g, r) - kvc_held(&g->kvc, id);
  return delta > 0 ? block_round(delta, g->kvc.block) : 0;
}

/* GtQueue (Q:125-204) */
static void gt_place(Eng* g, Group* grp, double now) { /* Q:187-197 */
  const uint64_t seq = grp->key.seq;
  grp->key = make_key(&g->opt, g->ordered, grp->min_deadline - now, grp->max_occupied, grp->padded_rl, seq);
  int64_t lo = 0, hi = g->gtq.n;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (key_less(&grp->key, &g->gtq.d[mid].key)) hi = mid; else lo = mid + 1;
  }
  VINSERT(g->gtq, lo, *grp);
}
static void gt_remove_at(Eng* g, int64_t gi, int free_members) {
  if (free_members) VFREE(g->gtq.d[gi].members);
  VERASE(g->gtq, gi);
}
static uint64_t group_insert_gt(Eng* g, int32_t id, Tok padded, double deadline, Tok occ, double now) { /* Q:141-166 */
  if (g->grouping) {
    for (int64_t gi = 0; gi < g->gtq.n; ++gi) {
      Group* gr = &g->gtq.d[gi];
      if (gr->padded_rl != padded) continue;
      VPUSH(gr->members, id);
      gr->min_deadline = dmin(gr->min_deadline, deadline);
      gr->max_occupied = tmax(gr->max_occupied, occ);
      Group moved = *gr; /* takes ownership of the member array */
      const uint64_t gid = moved.group_id;
      gt_remove_at(g, gi, 0);
      gt_place(g, &moved, now);
      return gid;
    }
  }
  Group ng;
  memset(&ng, 0, sizeof(ng));
  ng.group_id = g->next_group_id++;
  ng.padded_rl = padded;
  VPUSH(ng.members, id);
  ng.formed_at = now;
  ng.min_deadline = deadline;
  ng.max_occupied = occ;
  ng.key.seq = g->gt_next_seq++;
  const uint64_t gid = ng.group_id;
  gt_place(g, &ng, now);
  return gid;
}

static void begin_gt_run(Eng* g, int32_t id, int hosted) { /* E:350-363 */
  Req* r = &g->reqs[id];
  r->hosted = hosted;
  r->allowance = r->generated + r->padded_rl;
  r->generated_at_epoch = r->generated;
  const double wait = dmax(0.0, g->clock - r->last_enqueue_time);
  if (r->was_preempted) r->preemption_time += wait;
  else r->waiting_time += wait;
  r->was_preempted = 0;
  r->state = ST_RUNNING;
  VPUSH(g->running, id);
  VPUSH(g->admitted, id);
}

static int schedule_gt_member(Eng* g, int32_t id) { /* E:327-348 */
  Req* r = &g->reqs[id];
  const Tok target = seq_target(g, r);
  const Tok held = kvc_held(&g->kvc, id);
  const Tok resident = r->prompt + r->generated;
  int ok = 1;
  if (held == 0) {
    if (kvc_allocate_exact(&g->kvc, id, r->prompt + r->generated + r->padded_rl, &ok, &g->err)) return g->err.code;
  } else if (held < target) {
    if (kvc_grow_exact(&g->kvc, id, target - held, &ok, &g->err)) return g->err.code;
  }
  if (!ok) return fail(&g->err, ECONO_ESIM, "exact allocation failed for scheduled request %d", id);
  kvc_release_reserved(&g->kvc, id);
  const Tok cur = kvc_written(&g->kvc, id);
  if (cur < resident) kvc_add_written(&g->kvc, id, resident - cur);
  r->occupied = resident;
  begin_gt_run(g, id, 0);
  g->gt_scheduled++;
  logev(g, ECONO_EV_GT_SCHEDULE, id, r->padded_rl, 0);
  return 0;
}

/* plan_pipeline (KP:29-136) */
typedef struct { int32_t id; Tok write_base; } HostMember;
typedef struct { Tok padded_rl; VEC(HostMember) members; } HostView;
typedef struct { int32_t writer; Tok base, len, usage_base; } WRegion;
typedef VEC(WRegion) WRegionVec;
typedef struct { int64_t region_index; Tok abs, usage, len; } Cand;

static void plan_pipeline(Eng* g, HostView* hosts, int64_t nh, SlotVec* out) {
  int64_t exams = 0;
  for (int64_t h = 0; h < nh; ++h) {
    const Tok l = hosts[h].padded_rl;
    if (l < 2 || hosts[h].members.n == 0) continue;
    const Tok b = ceil_tokens(g->opt.buffer_ratio * (double)l);
    WRegionVec regions = {0};
    for (int64_t m = 0; m < hosts[h].members.n; ++m) {
      WRegion w = {hosts[h].members.d[m].id, hosts[h].members.d[m].write_base, l, 0};
      VPUSH(regions, w);
    }
    for (int level = 1;; ++level) {
      const Tok bound = l / ((Tok)1 << level) - b;
      if (bound < 1) break;
      VEC(Cand) cands = {0};
      for (int64_t ri = 0; ri < regions.n; ++ri) {
        const WRegion* r = &regions.d[ri];
        const Tok half = r->len / 2;
        if (half < 1) continue;
        Cand c = {ri, r->base + (r->len - half), r->usage_base + (r->len - half), half};
        VPUSH(cands, c);
      }
      if (cands.n == 0) { VFREE(cands); break; }
      std_shuffle(cands.d, (uint64_t)cands.n, sizeof(Cand), &g->rng);
      int32_t* assigned = malloc((size_t)regions.n * sizeof(int32_t));
      for (int64_t i = 0; i < regions.n; ++i) assigned[i] = -1;
      int64_t next_slot = 0;
      int any_group = 0;
      while (next_slot < cands.n) {
        int64_t chosen = -1;
        for (int64_t gi = 0; gi < g->gtq.n; ++gi) {
          const Group* gr = &g->gtq.d[gi];
          ++exams;
          if (gr->members.n == 0 || gr->padded_rl > bound) continue;
          const Group* ch = chosen >= 0 ? &g->gtq.d[chosen] : NULL;
          if (!ch || gr->padded_rl > ch->padded_rl ||
              (gr->padded_rl == ch->padded_rl &&
               (gr->formed_at < ch->formed_at ||
                (gr->formed_at == ch->formed_at && gr->group_id < ch->group_id))))
            chosen = gi;
        }
        if (chosen < 0) break;
        any_group = 1;
        Group* ch = &g->gtq.d[chosen];
        const int64_t take = ch->members.n < cands.n - next_slot ? ch->members.n : cands.n - next_slot;
        for (int64_t i = 0; i < take; ++i) {
          const int32_t hosted = ch->members.d[i];
          const Cand* c = &cands.d[next_slot + i];
          Slot s;
          s.host_id = regions.d[c->region_index].writer;
          s.hosted_id = hosted;
          s.start_offset = c->usage;
          s.deadline_usage = c->usage;
          s.length = c->len;
          s.abs_start = c->abs;
          VPUSH(*out, s);
          assigned[c->region_index] = hosted;
        }
        next_slot += take;
        memmove(ch->members.d, ch->members.d + take, (size_t)(ch->members.n - take) * sizeof(int32_t));
        ch->members.n -= take;
        if (ch->members.n == 0) gt_remove_at(g, chosen, 1);
      }
      VFREE(cands);
      if (!any_group) { free(assigned); break; }
      WRegionVec next = {0};
      for (int64_t ri = 0; ri < regions.n; ++ri) {
        const WRegion r = regions.d[ri];
        const Tok half = r.len / 2;
        if (half < 1) { VPUSH(next, r); continue; }
        const Tok kept = r.len - half;
        WRegion a = {r.writer, r.base, kept, r.usage_base};
        VPUSH(next, a);
        if (assigned[ri] >= 0) { WRegion w = {assigned[ri], r.base + kept, half, 0}; VPUSH(next, w); }
        else { WRegion w = {r.writer, r.base + kept, half, r.usage_base + kept}; VPUSH(next, w); }
      }
      free(assigned);
      VFREE(regions);
      regions = next;
    }
    VFREE(regions);
  }
  g->exam_count += exams;
}

static void dispatch_pt_common(Eng* g, int32_t id, Tok tokens) { /* E:372-381 */
  Req* r = &g->reqs[id];
  r->state = ST_RUNNING;
  r->dispatch_time = g->clock;
  r->waiting_time += g->clock - r->arrival;
  PtIter p = {id, tokens};
  VPUSH(g->pt_iter, p);
  VPUSH(g->admitted, id);
  ++g->pts_admitted_iter;
  g->pt_dispatched++;
  logev(g, ECONO_EV_PT_DISPATCH, id, 0, 0);
}

static int form_econoserve(Eng* g) { /* E:263-325 */
  Kvc* k = &g->kvc;
  /* select_gt_groups (Q:220-263) */
  VEC(Group) sel = {0};
  {
    const Tok avail = k->free_total;
    if (avail > 0) {
      Tok remaining = avail;
      int64_t gi = 0;
      while (gi < g->gtq.n) {
        Group* gr = &g->gtq.d[gi];
        ++g->exam_count;
        Tok total = 0;
        for (int64_t m = 0; m < gr->members.n; ++m) total += gt_member_demand(g, gr->members.d[m]);
        if (total <= remaining) {
          remaining -= total;
          VPUSH(sel, *gr); /* ownership moves with the erase */
          gt_remove_at(g, gi, 0);
          continue;
        }
        Group prefix;
        group_copy(&prefix, gr);
        prefix.members.n = 0;
        Tok pd = 0;
        int64_t taken = 0;
        for (int64_t m = 0; m < gr->members.n; ++m) {
          const Tok d = gt_member_demand(g, gr->members.d[m]);
          ++g->exam_count;
          if (pd + d > remaining) break;
          pd += d;
          VPUSH(prefix.members, gr->members.d[m]);
          ++taken;
        }
        if (taken > 0) {
          memmove(gr->members.d, gr->members.d + taken, (size_t)(gr->members.n - taken) * sizeof(int32_t));
          gr->members.n -= taken;
          remaining -= pd;
          VPUSH(sel, prefix);
        } else {
          VFREE(prefix.members);
        }
        break;
      }
    }
  }
  for (int64_t s = 0; s < sel.n; ++s)
    for (int64_t m = 0; m < sel.d[s].members.n; ++m)
      if (schedule_gt_member(g, sel.d[s].members.d[m])) goto fail_sel;

  if (g->opt.policy == ECONO_POLICY_ECONO_FULL) { /* E:273-297 */
    VEC(HostView) hosts = {0};
    for (int64_t s = 0; s < sel.n; ++s) {
      HostView hv;
      memset(&hv, 0, sizeof(hv));
      hv.padded_rl = sel.d[s].padded_rl;
      for (int64_t m = 0; m < sel.d[s].members.n; ++m) {
        const int32_t id = sel.d[s].members.d[m];
        const Req* r = &g->reqs[id];
        if (r->generated == 0 && k->alloc[id].present && k->alloc[id].regions.n == 1) {
          HostMember hm = {id, k->alloc[id].regions.d[0].start + r->prompt};
          VPUSH(hv.members, hm);
        }
      }
      if (hv.members.n) VPUSH(hosts, hv);
    }
    if (hosts.n > 0 && g->gtq.n > 0) {
      SlotVec slots = {0};
      plan_pipeline(g, hosts.d, hosts.n, &slots);
      for (int64_t i = 0; i < slots.n; ++i) {
        const Slot* s = &slots.d[i];
        if (kvc_add_slot(k, s, &g->err)) { VFREE(slots); goto fail_hosts; }
        ++g->hosted_total;
        begin_gt_run(g, s->hosted_id, 1);
        g->gt_scheduled++;
        logev(g, ECONO_EV_HOSTED, s->hosted_id, s->host_id, s->deadline_usage);
      }
      VFREE(slots);
    }
    for (int64_t h = 0; h < hosts.n; ++h) VFREE(hosts.d[h].members);
    VFREE(hosts);
    goto pts;
  fail_hosts:
    for (int64_t h = 0; h < hosts.n; ++h) VFREE(hosts.d[h].members);
    VFREE(hosts);
    goto fail_sel;
  }
pts:
  for (int64_t s = 0; s < sel.n; ++s) VFREE(sel.d[s].members);
  VFREE(sel);
  {
    const Tok live = (Tok)g->running.n;
    const Tok tfs_rem = g->opt.tfs - live;
    for (int64_t i = 0; i < g->ptq.n; ++i) { /* E:301-307 */
      const Tok p = g->reqs[g->ptq.d[i].id].prompt;
      if (p <= tfs_rem && p <= k->reserve_cap - k->reserved_used) { g->pt_admittable_iter = 1; break; }
    }
    /* select_pts (Q:279-299) */
    IVec ids = {0};
    const Tok rfree = k->reserve_cap - k->reserved_used;
    if (!(tfs_rem <= 0 || rfree <= 0)) {
      Tok budget = tfs_rem, reserve = rfree;
      int64_t w = 0;
      for (int64_t i = 0; i < g->ptq.n; ++i) {
        ++g->exam_count;
        const int32_t id = g->ptq.d[i].id;
        const Tok p = g->reqs[id].prompt;
        if (p > budget || p > reserve) { g->ptq.d[w++] = g->ptq.d[i]; continue; }
        budget -= p;
        reserve -= p;
        VPUSH(ids, id);
      }
      g->ptq.n = w; /* PtQueue::remove for every taken id (Q:98-100, ids unique) */
    }
    if (ids.n == 0 && g->ptq.n > 0 && g->running.n == 0) { /* E:314-323 */
      for (int64_t i = 0; i < g->ptq.n; ++i) {
        const int32_t id = g->ptq.d[i].id;
        if (g->reqs[id].prompt <= k->reserve_cap - k->reserved_used) {
          VPUSH(ids, id);
          VERASE(g->ptq, i);
          break;
        }
      }
    }
    for (int64_t i = 0; i < ids.n; ++i) { /* dispatch_pt_reserved E:365-370 */
      const int32_t id = ids.d[i];
      if (!kvc_draw_reserved(k, id, g->reqs[id].prompt)) {
        VFREE(ids);
        return fail(&g->err, ECONO_ESIM, "reserved pool draw failed for selected PT %d", id);
      }
      dispatch_pt_common(g, id, g->reqs[id].prompt);
    }
    VFREE(ids);
  }
  return 0;
fail_sel:
  for (int64_t s = 0; s < sel.n; ++s) VFREE(sel.d[s].members);
  VFREE(sel);
  return g->err.code;
}

static void erase_id(IVec* v, int32_t id) { /* std::erase */
  int64_t w = 0;
  for (int64_t i = 0; i < v->n; ++i)
    if (v->d[i] != id) v->d[w++] = v->d[i];
  v->n = w;
}

static int complete_req(Eng* g, int32_t id) { /* E:842-852 */
  Req* r = &g->reqs[id];
  r->state = ST_DONE;
  r->completion_clock = g->clock;
  if (kvc_release(&g->kvc, id, &g->err)) return g->err.code;
  r->occupied = 0;
  erase_id(&g->running, id);
  ++g->completed;
  logev(g, ECONO_EV_COMPLETE, id, r->generated, 0);
  return 0;
}

static int vacate_slot(Eng* g, int32_t id) { /* E:888-902 */
  Req* r = &g->reqs[id];
  const Tok in_slot = tmin(r->generated - r->generated_at_epoch, r->padded_rl);
  int rehomed = 0;
  if (in_slot > 0 && kvc_draw_reserved(&g->kvc, id, in_slot)) {
    rehomed = 1;
  } else if (in_slot > 0) {
    kvc_drop_written(&g->kvc, id, in_slot);
    r->occupied -= in_slot;
  }
  kvc_remove_slot(&g->kvc, id);
  r->hosted = 0;
  return rehomed;
}

static void preempt_and_regroup(Eng* g, int32_t id, int why) { /* E:904-928 */
  Req* r = &g->reqs[id];
  ++r->preempt_count;
  r->state = ST_PREEMPTED;
  erase_id(&g->running, id);
  const Tok remaining = r->true_rl - r->generated;
  r->predicted_rl = predict_rl(remaining, &g->opt, &g->pred_rng);
  r->padded_rl = apply_padding(r->predicted_rl, g->opt.pred_padding_ratio);
  r->was_preempted = 1;
  r->last_enqueue_time = g->clock;
  logev(g, ECONO_EV_PREEMPT, id, why, r->padded_rl);
  r->state = ST_WAITING_GT;
  group_insert_gt(g, id, r->padded_rl, r->slo_deadline, r->occupied, g->clock);
}

static void handle_underprediction(Eng* g, int32_t id) { /* E:856-873 */
  Req* r = &g->reqs[id];
  if (kvc_draw_reserved(&g->kvc, id, g->kvc.block)) {
    r->allowance += g->kvc.block;
    ++r->reserve_draws;
    g->penalty_extra[id] += g->opt.reserve_penalty;
    logev(g, ECONO_EV_RESERVE_TOPUP, id, 0, 0);
    return;
  }
  r->alloc_failure_flag = 1;
  ++g->alloc_failures;
  int rehomed = 1;
  if (r->hosted) rehomed = vacate_slot(g, id);
  g->penalty_extra[id] += rehomed ? g->opt.preempt_free_penalty : g->opt.preempt_offload_penalty;
  preempt_and_regroup(g, id, 0);
}

static void handle_hosted_overrun(Eng* g, int32_t id) { /* E:875-884 */
  Req* r = &g->reqs[id];
  ++g->hosted_overruns;
  const int rehomed = vacate_slot(g, id);
  g->penalty_extra[id] += rehomed ? g->opt.preempt_free_penalty : g->opt.preempt_offload_penalty;
  r->alloc_failure_flag = 1;
  ++g->alloc_failures;
  logev(g, ECONO_EV_HOSTED_OVERRUN, id, 0, 0);
  preempt_and_regroup(g, id, 1);
}

static int execute_iteration(Eng* g, Tok fs) { /* E:731-840 */
  const double dt = iteration_time(fs, &g->opt) + 0.0; /* + pending_stall_ (always 0 here) */
  g->clock += dt;
  ++g->iter;
  const double sched = (double)g->exam_count * g->opt.sched_cost_per_exam;
  if (g->admitted.n > 0 && sched > 0.0) {
    const double share = sched / (double)g->admitted.n;
    for (int64_t i = 0; i < g->admitted.n; ++i) g->sched_share[g->admitted.d[i]] += share;
  }
  for (int64_t i = 0; i < g->pt_iter.n; ++i) g->reqs[g->pt_iter.d[i].id].execution_time += dt;
  for (int64_t i = 0; i < g->running.n; ++i) g->reqs[g->running.d[i]].execution_time += dt;
  IVec finished = {0};
  for (int64_t i = 0; i < g->pt_iter.n; ++i) {
    const PtIter p = g->pt_iter.d[i];
    Req* r = &g->reqs[p.id];
    r->prefill_done += p.tokens;
    kvc_add_written(&g->kvc, p.id, p.tokens);
    r->occupied += p.tokens;
    if (r->prefill_done >= r->prefill_target) VPUSH(finished, p.id);
  }
  for (int64_t i = 0; i < g->running.n; ++i) {
    const int32_t id = g->running.d[i];
    Req* r = &g->reqs[id];
    ++r->generated;
    ++r->occupied;
    kvc_add_written(&g->kvc, id, 1);
    if (r->generated == 1 && r->first_token_time < 0.0) r->first_token_time = g->clock;
  }
  EconoSample s;
  memset(&s, 0, sizeof(s));
  s.iter = g->iter;
  s.clock = g->clock;
  s.dt = dt;
  s.forward_size = fs;
  s.kvc_written_frac = kvc_utilization(&g->kvc);
  s.kvc_allocated_frac = kvc_allocated_fraction(&g->kvc);
  s.pts_admitted = g->pts_admitted_iter;
  s.pt_admittable = g->pt_admittable_iter;
  int completed_now = 0;
  {
    IVec copy = {0};
    for (int64_t i = 0; i < g->running.n; ++i) VPUSH(copy, g->running.d[i]);
    for (int64_t i = 0; i < copy.n; ++i) {
      const int32_t id = copy.d[i];
      if (g->reqs[id].generated >= g->reqs[id].true_rl) {
        if (complete_req(g, id)) { VFREE(copy); VFREE(finished); return g->err.code; }
        ++completed_now;
      }
    }
    VFREE(copy);
  }
  for (int64_t i = 0; i < finished.n; ++i) { /* E:794-809 */
    const int32_t id = finished.d[i];
    Req* r = &g->reqs[id];
    if (r->state != ST_RUNNING) continue;
    r->state = ST_WAITING_GT;
    r->last_enqueue_time = g->clock;
    group_insert_gt(g, id, r->padded_rl, r->slo_deadline, r->occupied, g->clock);
    logev(g, ECONO_EV_PREFILL_DONE, id, 0, 0);
  }
  VFREE(finished);
  {
    IVec copy = {0};
    for (int64_t i = 0; i < g->running.n; ++i) VPUSH(copy, g->running.d[i]);
    for (int64_t i = 0; i < copy.n; ++i) { /* E:812-817 */
      const int32_t id = copy.d[i];
      Req* r = &g->reqs[id];
      if (r->state != ST_RUNNING || r->state == ST_DONE) continue;
      if (r->generated >= r->allowance && r->generated < r->true_rl) handle_underprediction(g, id);
    }
    VFREE(copy);
  }
  {
    SlotVec copy = {0};
    for (int64_t i = 0; i < g->kvc.slots.n; ++i) VPUSH(copy, g->kvc.slots.d[i]);
    for (int64_t i = 0; i < copy.n; ++i) { /* E:820-828 */
      const Slot sl = copy.d[i];
      const Req* host = &g->reqs[sl.host_id];
      if (host->state != ST_RUNNING) continue;
      const Tok usage = host->generated - host->generated_at_epoch;
      if (usage < sl.deadline_usage) continue;
      const Req* hosted = &g->reqs[sl.hosted_id];
      if (hosted->state == ST_DONE || !hosted->hosted) continue;
      handle_hosted_overrun(g, sl.hosted_id);
    }
    VFREE(copy);
  }
  s.completed = completed_now;
  VPUSH(g->samples, s);
  g->pt_iter.n = 0;
  g->admitted.n = 0;
  g->exam_count = 0;
  g->pts_admitted_iter = 0;
  g->pt_admittable_iter = 0;
  return 0;
}

static int handle_idle(Eng* g) { /* E:930-961 */
  if (g->arrival_cursor < g->n) {
    const double next = g->reqs[g->arrival_cursor].arrival;
    long k = 1;
    if (next > g->clock) {
      long c = (long)ceil((next - g->clock) / g->opt.t_base);
      k = c > 1 ? c : 1;
    }
    const double dt = (double)k * g->opt.t_base;
    g->clock += dt;
    g->iter += k;
    EconoSample s;
    memset(&s, 0, sizeof(s));
    s.iter = g->iter;
    s.clock = g->clock;
    s.dt = dt;
    s.kvc_written_frac = kvc_utilization(&g->kvc);
    s.kvc_allocated_frac = kvc_allocated_fraction(&g->kvc);
    s.idle_repeat = k;
    VPUSH(g->samples, s);
    logev(g, ECONO_EV_IDLE, -1, k, 0);
    return 0;
  }
  int32_t stuck = -1;
  for (int32_t i = 0; i < g->n; ++i)
    if (g->reqs[i].state != ST_DONE) { stuck = i; break; }
  return fail(&g->err, ECONO_ESIM,
              "simulation stuck: request %d can never be scheduled (demand exceeds what the "
              "configuration can free)", stuck);
}

static int engine_step(Eng* g, int* more) { /* E:104-116 */
  if (g->completed >= g->n) { *more = 0; return 0; }
  ingest_arrivals(g);
  if (form_econoserve(g)) return g->err.code;
  Tok fs = 0;
  for (int64_t i = 0; i < g->pt_iter.n; ++i) fs += g->pt_iter.d[i].tokens;
  fs += (Tok)g->running.n;
  int rc = fs == 0 ? handle_idle(g) : execute_iteration(g, fs);
  if (rc) return rc;
  g->steps++;
  *more = g->completed < g->n;
  return 0;
}

static int validate_options(const EconoOptions* o, Err* e) {
  /* PolicyConfig::validate */
  if (o->tfs < 1) return fail(e, ECONO_ECONFIG, "tfs must be >= 1");
  if (o->chunk_size < 1) return fail(e, ECONO_ECONFIG, "chunk_size must be >= 1");
  if (o->batch_size_cap < 1) return fail(e, ECONO_ECONFIG, "batch_size_cap must be >= 1");
  if (o->padding_ratio < 0.0) return fail(e, ECONO_ECONFIG, "padding_ratio must be >= 0");
  if (o->reserved_fraction < 0.0 || o->reserved_fraction >= 1.0)
    return fail(e, ECONO_ECONFIG, "reserved_fraction must be in [0, 1)");
  if (o->buffer_ratio < 0.0) return fail(e, ECONO_ECONFIG, "buffer_ratio must be >= 0");
  /* CostModel::validate (E:36-43) */
  if (!(o->t_base > 0.0)) return fail(e, ECONO_ECONFIG, "cost model: t_base must be > 0");
  if (!(o->t_token > 0.0)) return fail(e, ECONO_ECONFIG, "cost model: t_token must be > 0");
  if (o->cost_tfs < 1) return fail(e, ECONO_ECONFIG, "cost model: tfs must be >= 1");
  if (o->preempt_offload_penalty < 0.0 || o->preempt_free_penalty < 0.0 || o->reserve_penalty < 0.0 ||
      o->sched_cost_per_exam < 0.0 || o->swap_stall < 0.0)
    return fail(e, ECONO_ECONFIG, "cost model: penalties must be >= 0");
  /* PredictorConfig::validate (W:211-217) */
  if (o->pred_sigma < 0.0) return fail(e, ECONO_ECONFIG, "predictor sigma must be >= 0");
  if (o->pred_accuracy < 0.0 || o->pred_accuracy > 1.0) return fail(e, ECONO_ECONFIG, "predictor accuracy must be in [0,1]");
  if (o->pred_tolerance < 0.0) return fail(e, ECONO_ECONFIG, "predictor tolerance must be >= 0");
  if (o->pred_padding_ratio < 0.0) return fail(e, ECONO_ECONFIG, "padding_ratio must be >= 0");
  if (o->pred_quantum < 1) return fail(e, ECONO_ECONFIG, "predictor quantum must be >= 1");
  return 0;
}
static int ordering_valid(const EconoOptions* o) { /* OrderingConfig::validate (Q:22-27) */
  for (int i = 1; i < o->n_deadline_bounds; ++i) if (o->deadline_bounds[i] < o->deadline_bounds[i - 1]) return 0;
  for (int i = 1; i < o->n_kvc_bounds; ++i) if (o->kvc_bounds[i] < o->kvc_bounds[i - 1]) return 0;
  for (int i = 1; i < o->n_length_bounds; ++i) if (o->length_bounds[i] < o->length_bounds[i - 1]) return 0;
  return 1;
}

/* ------------------------------------------------------------------ */
/* public (test-only) C ABI                                             */
/* ------------------------------------------------------------------ */
static void copy_err(const Err* e, char* err, size_t errlen) {
  if (err && errlen) snprintf(err, errlen, "%s", e->msg);
}

static void eng_free(Eng* g) {
  if (!g) return;
  kvc_free(&g->kvc);
  free(g->reqs);
  VFREE(g->ptq);
  for (int64_t i = 0; i < g->gtq.n; ++i) VFREE(g->gtq.d[i].members);
  VFREE(g->gtq);
  VFREE(g->running); VFREE(g->admitted); VFREE(g->pt_iter);
  free(g->penalty_extra); free(g->sched_share);
  VFREE(g->events); VFREE(g->samples);
  free(g);
}

int orc_create(const EconoTraceRecord* trace, int64_t n, const EconoOptions* opt, void** out,
               char* err, size_t errlen) { /* E:81-100, init_requests E:165-209 */
  Eng* g = calloc(1, sizeof(Eng));
  g->opt = *opt;
  const int econo = opt->policy >= ECONO_POLICY_ECONO_D && opt->policy <= ECONO_POLICY_ECONO_FULL;
  if (kvc_init(&g->kvc, opt->kvc_capacity, opt->kvc_block_size, econo ? opt->reserved_fraction : 0.0,
               (int32_t)(n > 0 ? n : 1), &g->err))
    goto bad;
  if (!ordering_valid(opt)) { fail(&g->err, ECONO_ECONFIG, "ordering bucket boundaries must be increasing"); goto bad; }
  if (validate_options(opt, &g->err)) goto bad;
  if (n <= 0) { fail(&g->err, ECONO_ECONFIG, "trace is empty"); goto bad; }
  if (!econo) { fail(&g->err, ECONO_ECONFIG, "policy %d is outside the EconoServe scheduling path", opt->policy); goto bad; }
  g->ordered = opt->policy == ECONO_POLICY_ECONO_SDO || opt->policy == ECONO_POLICY_ECONO_FULL;
  g->grouping = opt->policy != ECONO_POLICY_ECONO_D;
  g->opt.cost_tfs = opt->tfs;
  mt_seed(&g->rng, opt->seed);
  mt_seed(&g->pred_rng, opt->pred_seed);
  g->next_group_id = 1;
  g->n = (int32_t)n;
  g->reqs = calloc((size_t)n, sizeof(Req));
  g->penalty_extra = calloc((size_t)n, sizeof(double));
  g->sched_share = calloc((size_t)n, sizeof(double));
  for (int64_t i = 1; i < n; ++i)
    if (trace[i].arrival_time < trace[i - 1].arrival_time) {
      fail(&g->err, ECONO_ECONFIG, "trace arrival times must be nondecreasing");
      goto bad;
    }
  double prompt_sum = 0.0;
  for (int64_t i = 0; i < n; ++i) prompt_sum += (double)trace[i].prompt_len;
  const Tok mean_prompt = tmax(1, (Tok)llround(prompt_sum / (double)n));
  g->t_p = iteration_time(mean_prompt, &g->opt);
  g->t_g = iteration_time(g->opt.tfs, &g->opt);
  const Tok B = g->kvc.block;
  for (int64_t i = 0; i < n; ++i) {
    Req* r = &g->reqs[i];
    r->arrival = trace[i].arrival_time;
    r->prompt = trace[i].prompt_len;
    r->true_rl = trace[i].true_rl;
    r->predicted_rl = predict_rl(r->true_rl, &g->opt, &g->pred_rng);
    r->padded_rl = apply_padding(r->predicted_rl, g->opt.pred_padding_ratio);
    r->prefill_target = r->prompt;
    r->slo_deadline = r->arrival + g->opt.slo_scale * (g->t_p + g->t_g * (double)r->true_rl);
    r->dispatch_time = -1.0;
    r->first_token_time = -1.0;
    r->completion_clock = -1.0;
    r->state = ST_WAITING_PT;
    const Tok worst = block_round(r->prompt + tmax(r->true_rl, r->padded_rl), B);
    if (worst > g->kvc.general_cap) {
      fail(&g->err, ECONO_ESIM, "request %lld: KVC demand %lld exceeds usable capacity %lld",
           (long long)i, (long long)worst, (long long)g->kvc.general_cap);
      goto bad;
    }
    if (r->prompt > g->kvc.reserve_cap) {
      fail(&g->err, ECONO_ESIM, "request %lld: prompt does not fit the reserved pool (%lld tokens)",
           (long long)i, (long long)g->kvc.reserve_cap);
      goto bad;
    }
  }
  *out = g;
  return 0;
bad:
  copy_err(&g->err, err, errlen);
  {
    int code = g->err.code;
    eng_free(g);
    return code;
  }
}

void orc_destroy(void* h) { eng_free((Eng*)h); }

int orc_step(void* h, int64_t max_steps, int32_t* more, char* err, size_t errlen) {
  Eng* g = h;
  if (g->faulted) { copy_err(&g->err, err, errlen); return g->err.code; }
  int m = g->completed < g->n;
  for (int64_t i = 0; i < max_steps && m; ++i) {
    if (engine_step(g, &m)) {
      g->faulted = 1;
      copy_err(&g->err, err, errlen);
      return g->err.code;
    }
  }
  *more = m;
  return 0;
}

int64_t orc_events(void* h, EconoEvent* out, int64_t cap) {
  Eng* g = h;
  if (out) memcpy(out, g->events.d, (size_t)(g->events.n < cap ? g->events.n : cap) * sizeof(EconoEvent));
  return g->events.n;
}
int64_t orc_samples(void* h, EconoSample* out, int64_t cap) {
  Eng* g = h;
  if (out) memcpy(out, g->samples.d, (size_t)(g->samples.n < cap ? g->samples.n : cap) * sizeof(EconoSample));
  return g->samples.n;
}

static int dcmp(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}
static double percentile(double* sorted, int64_t n, double q) { /* M:81-89 (input pre-sorted) */
  if (n == 0) return 0.0;
  const double rank = q * (double)(n - 1);
  const int64_t lo = (int64_t)rank;
  const int64_t hi = lo + 1 < n - 1 ? lo + 1 : n - 1;
  const double frac = rank - (double)lo;
  return sorted[lo] * (1.0 - frac) + sorted[hi] * frac;
}

static uint64_t trace_hash(const Eng* g) { /* write_trace_csv W:127-134 + FNV-1a M:320-328 */
  uint64_t h = 1469598103934665603ULL;
  const char* hdr = "arrival_time,prompt_len,response_len\n";
  for (const char* c = hdr; *c; ++c) { h ^= (unsigned char)*c; h *= 1099511628211ULL; }
  char buf[128];
  for (int32_t i = 0; i < g->n; ++i) {
    int len = snprintf(buf, sizeof(buf), "%.17g,%lld,%lld\n", g->reqs[i].arrival,
                       (long long)g->reqs[i].prompt, (long long)g->reqs[i].true_rl);
    for (int j = 0; j < len; ++j) { h ^= (unsigned char)buf[j]; h *= 1099511628211ULL; }
  }
  return h;
}

int orc_finalize(void* h, EconoRecord* recs, int64_t cap, EconoReport* rep, char* err, size_t errlen) {
  Eng* g = h; /* E:963-994 + aggregate M:96-175 */
  if (g->completed < g->n) {
    if (err && errlen) snprintf(err, errlen, "report requested before the run finished");
    return ECONO_ESIM;
  }
  EconoReport r;
  memset(&r, 0, sizeof(r));
  double* jcts = malloc((size_t)g->n * sizeof(double));
  double tbt_sum = 0.0, norm_sum = 0.0;
  long tbt_n = 0, met = 0, failures = 0;
  Tok tokens_total = 0;
  for (int32_t i = 0; i < g->n; ++i) {
    const Req* q = &g->reqs[i];
    EconoRecord rc;
    memset(&rc, 0, sizeof(rc));
    rc.id = i;
    rc.arrival = q->arrival;
    const double extra = g->penalty_extra[i] + g->sched_share[i];
    rc.completion_time = q->completion_clock + extra;
    rc.first_token_time = q->first_token_time;
    rc.waiting_time = q->waiting_time;
    rc.execution_time = q->execution_time;
    rc.preemption_time = q->preemption_time + g->penalty_extra[i];
    rc.scheduling_time_share = g->sched_share[i];
    rc.preempt_count = q->preempt_count;
    rc.reserve_draws = q->reserve_draws;
    rc.met_slo = rc.completion_time <= q->slo_deadline;
    rc.prompt_len = q->prompt;
    rc.true_rl = q->true_rl;
    rc.slo_deadline = q->slo_deadline;
    rc.alloc_failure = q->alloc_failure_flag;
    if (i < cap && recs) recs[i] = rc;
    const double jct = rc.completion_time - rc.arrival;
    jcts[i] = jct;
    if (rc.true_rl >= 2 && rc.first_token_time >= 0.0) {
      tbt_sum += (rc.completion_time - rc.first_token_time) / (double)(rc.true_rl - 1);
      ++tbt_n;
    }
    norm_sum += jct / (double)rc.true_rl;
    if (rc.met_slo) ++met;
    tokens_total += rc.true_rl;
    r.preemptions += rc.preempt_count;
    r.reserve_draws += rc.reserve_draws;
    if (rc.alloc_failure) ++failures;
    r.makespan = dmax(r.makespan, rc.completion_time);
    r.mean_waiting += rc.waiting_time;
    r.mean_execution += rc.execution_time;
    r.mean_preemption += rc.preemption_time;
    r.mean_scheduling += rc.scheduling_time_share;
  }
  const double n = (double)g->n;
  for (int32_t i = 0; i < g->n; ++i) r.mean_jct += jcts[i];
  r.mean_jct /= n;
  qsort(jcts, (size_t)g->n, sizeof(double), dcmp);
  r.p5_jct = percentile(jcts, g->n, 0.05);
  r.p95_jct = percentile(jcts, g->n, 0.95);
  free(jcts);
  r.mean_tbt = tbt_n > 0 ? tbt_sum / (double)tbt_n : 0.0;
  r.ssr = (double)met / n;
  r.normalized_latency = norm_sum / n;
  r.mean_waiting /= n;
  r.mean_execution /= n;
  r.mean_preemption /= n;
  r.mean_scheduling /= n;
  if (r.makespan > 0.0) {
    r.throughput_rps = n / r.makespan;
    r.throughput_tps = (double)tokens_total / r.makespan;
    r.goodput_rps = (double)met / r.makespan;
  }
  r.allocation_failure_pct = 100.0 * (double)failures / n;
  long executed = 0, tfs_hits = 0, pt_iters = 0;
  int maxc = 0;
  for (int64_t i = 0; i < g->samples.n; ++i) if (g->samples.d[i].completed > maxc) maxc = g->samples.d[i].completed;
  long* hist = calloc((size_t)maxc + 1, sizeof(long));
  for (int64_t i = 0; i < g->samples.n; ++i) {
    const EconoSample* s = &g->samples.d[i];
    if (s->idle_repeat > 0) continue;
    ++executed;
    r.mean_forward_size += (double)s->forward_size;
    r.mean_kvc_written += s->kvc_written_frac;
    r.mean_kvc_allocated += s->kvc_allocated_frac;
    if ((double)s->forward_size >= 0.95 * (double)g->opt.tfs) ++tfs_hits;
    if (s->pts_admitted > 0) ++pt_iters;
    hist[s->completed] += 1;
  }
  r.iterations = executed;
  if (executed > 0) {
    r.mean_forward_size /= (double)executed;
    r.mean_kvc_written /= (double)executed;
    r.mean_kvc_allocated /= (double)executed;
    r.tfs_hit_frac = (double)tfs_hits / (double)executed;
    r.pt_admit_frac = (double)pt_iters / (double)executed;
    int k = 0;
    for (int c = 0; c <= maxc && k < ECONO_MAX_HIST; ++c)
      if (hist[c]) { r.hist_count[k] = c; r.hist_frac[k] = (double)hist[c] / (double)executed; ++k; }
    r.n_hist = k;
  }
  free(hist);
  r.trace_hash = trace_hash(g);
  r.hosted_slots = g->hosted_total;
  r.hosted_overruns = g->hosted_overruns;
  if (rep) *rep = r;
  return 0;
}

int orc_scalars(void* h, EconoScalars* o) {
  Eng* g = h;
  memset(o, 0, sizeof(*o));
  o->clock = g->clock;
  o->iter = g->iter;
  o->completed = g->completed;
  o->steps = g->steps;
  int64_t ex = 0;
  for (int64_t i = 0; i < g->samples.n; ++i) if (g->samples.d[i].idle_repeat == 0) ++ex;
  o->executed_iters = ex;
  o->hosted_slots_created = g->hosted_total;
  o->hosted_overruns = g->hosted_overruns;
  o->calibrated_prefill_time = g->t_p;
  o->calibrated_decode_time = g->t_g;
  o->pt_dispatched = g->pt_dispatched;
  o->gt_scheduled = g->gt_scheduled;
  o->pt_queue_len = g->ptq.n;
  o->gt_queue_groups = g->gtq.n;
  o->running = g->running.n;
  o->arrived = g->arrival_cursor;
  o->done = g->completed >= g->n;
  o->error = g->faulted ? g->err.code : 0;
  return 0;
}

static int64_t dbits(double d) { int64_t v; memcpy(&v, &d, 8); return v; }

int64_t orc_snapshot(void* h, int64_t* out, int64_t cap) {
  Eng* g = h;
  const Kvc* k = &g->kvc;
  LVec w = {0};
#define W(x) VPUSH(w, (int64_t)(x))
  W(0x45434f4e); W(g->iter); W(dbits(g->clock)); W(g->completed); W(g->arrival_cursor);
  W(k->free_total); W(k->reserved_used); W(k->written_total); W(g->hosted_total);
  W(g->hosted_overruns); W(g->exam_count); W(g->n);
  W(g->ptq.n);
  for (int64_t i = 0; i < g->ptq.n; ++i) W(g->ptq.d[i].id);
  W(g->gtq.n);
  for (int64_t i = 0; i < g->gtq.n; ++i) {
    const Group* gr = &g->gtq.d[i];
    W(gr->group_id); W(gr->padded_rl); W(dbits(gr->formed_at)); W(dbits(gr->min_deadline));
    W(gr->max_occupied); W(gr->key.db); W(gr->key.kb); W(gr->key.len); W(gr->key.seq);
    W(gr->members.n);
    for (int64_t m = 0; m < gr->members.n; ++m) W(gr->members.d[m]);
  }
  W(k->slots.n);
  for (int64_t i = 0; i < k->slots.n; ++i) {
    const Slot* s = &k->slots.d[i];
    W(s->host_id); W(s->hosted_id); W(s->start_offset); W(s->length); W(s->deadline_usage); W(s->abs_start);
  }
  W(k->alloc_ids.n);
  for (int64_t a = 0; a < k->alloc_ids.n; ++a) {
    const int32_t id = k->alloc_ids.d[a];
    const Holding* hd = &k->alloc[id];
    W(id); W(hd->total); W(hd->regions.n);
    for (int64_t i = 0; i < hd->regions.n; ++i) { W(hd->regions.d[i].start); W(hd->regions.d[i].len); }
  }
  W(k->free_.n);
  for (int64_t i = 0; i < k->free_.n; ++i) { W(k->free_.d[i].start); W(k->free_.d[i].len); }
  int64_t nr = 0;
  for (int32_t i = 0; i < g->n; ++i) nr += k->has_reserved[i];
  W(nr);
  for (int32_t i = 0; i < g->n; ++i) if (k->has_reserved[i]) { W(i); W(k->reserved[i]); }
  int64_t nw = 0;
  for (int32_t i = 0; i < g->n; ++i) nw += (k->has_written[i] && k->written[i] != 0);
  W(nw);
  for (int32_t i = 0; i < g->n; ++i) if (k->has_written[i] && k->written[i] != 0) { W(i); W(k->written[i]); }
  W(g->running.n);
  for (int64_t i = 0; i < g->running.n; ++i) W(g->running.d[i]);
  for (int32_t i = 0; i < g->n; ++i) {
    const Req* r = &g->reqs[i];
    W(r->state); W(r->generated); W(r->predicted_rl); W(r->padded_rl); W(r->allowance);
    W(r->generated_at_epoch); W(r->occupied); W(r->hosted); W(r->was_preempted);
    W(r->preempt_count); W(r->reserve_draws); W(r->alloc_failure_flag); W(r->prefill_done);
    W(dbits(r->waiting_time)); W(dbits(r->preemption_time)); W(dbits(r->execution_time));
    /* dispatch_time: dead state for econoserve (E:374; read by the baselines only), not compared */
    W(0); W(dbits(r->first_token_time)); W(dbits(r->completion_clock));
    W(dbits(r->last_enqueue_time)); W(dbits(g->sched_share[i])); W(dbits(g->penalty_extra[i]));
    W(dbits(r->slo_deadline));
  }
#undef W
  const int64_t n = w.n;
  if (out) memcpy(out, w.d, (size_t)(n < cap ? n : cap) * 8);
  VFREE(w);
  return n;
}

/* generate_synthetic (W:42-125) */
static double std_normal_cdf(double x) { return 0.5 * erfc(-x / sqrt(2.0)); } /* W:44 */
static double trunc_lognormal_mean(double mu, double sigma, double a, double b) { /* W:47-54 */
  const double alpha = (log(a) - mu) / sigma;
  const double beta = (log(b) - mu) / sigma;
  const double mass = std_normal_cdf(beta) - std_normal_cdf(alpha);
  if (mass <= 0.0) return a;
  const double num = std_normal_cdf(beta - sigma) - std_normal_cdf(alpha - sigma);
  return exp(mu + 0.5 * sigma * sigma) * num / mass;
}
static double fit_mu(const EconoLengthDist* d) { /* W:57-70 */
  const double a = (double)d->min_value, b = (double)d->max_value;
  double lo = log(a) - 10.0, hi = log(b) + 10.0;
  for (int i = 0; i < 200; ++i) {
    const double mid = 0.5 * (lo + hi);
    if (trunc_lognormal_mean(mid, d->sigma, a, b) < d->mean) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}
static int sampler_check(const EconoLengthDist* d, Err* e) { /* W:76-85 */
  if (d->min_value < 1 || d->max_value < d->min_value)
    return fail(e, ECONO_ECONFIG, "length distribution bounds invalid: min=%lld max=%lld",
                (long long)d->min_value, (long long)d->max_value);
  if (d->sigma <= 0.0) return fail(e, ECONO_ECONFIG, "length distribution sigma must be > 0");
  if (d->mean < (double)d->min_value || d->mean > (double)d->max_value)
    return fail(e, ECONO_ECONFIG, "length distribution mean outside [min, max]");
  return 0;
}
static Tok sample_len(const EconoLengthDist* d, double mu, Mt* rng) { /* W:87-97 */
  if (d->min_value == d->max_value) return d->min_value;
  Normal nd = {0, 0.0}; /* lognormal_distribution's inner normal (random.h:2358) */
  for (int attempt = 0; attempt < 10000; ++attempt) {
    const double x = exp(d->sigma * normal_draw(&nd, rng, 0.0, 1.0) + mu);
    const Tok v = (Tok)llround(x);
    if (v >= d->min_value && v <= d->max_value) return v;
  }
  Tok v = (Tok)llround(exp(mu));
  if (v < d->min_value) v = d->min_value;
  if (v > d->max_value) v = d->max_value;
  return v;
}
int orc_generate_trace(int64_t n, double rate, const EconoLengthDist* p, const EconoLengthDist* r,
                       uint64_t seed, EconoTraceRecord* out, char* err, size_t errlen) { /* W:104-125 */
  Err e = {0, ""};
  if (n < 1) { fail(&e, ECONO_ECONFIG, "n_requests must be >= 1"); goto bad; }
  if (!(rate > 0.0)) { fail(&e, ECONO_ECONFIG, "arrival_rate must be > 0"); goto bad; }
  if (sampler_check(p, &e) || sampler_check(r, &e)) goto bad;
  {
    const double mp = fit_mu(p), mr = fit_mu(r);
    Mt rng;
    mt_seed(&rng, seed);
    double clock = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      clock += -log(1.0 - canonical(&rng)) / rate; /* exponential (random.h:4904) */
      out[i].arrival_time = clock;
      out[i].prompt_len = sample_len(p, mp, &rng);
      out[i].true_rl = sample_len(r, mr, &rng);
    }
  }
  return 0;
bad:
  copy_err(&e, err, errlen);
  return e.code;
}

/* Exposed for unit tests of the restated RNG plumbing. */
void orc_mt_draws(uint64_t seed, int64_t n, uint64_t* out) {
  Mt m;
  mt_seed(&m, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = mt_next(&m);
}
void orc_shuffle_indices(uint64_t seed, int64_t n, int64_t* idx) {
  Mt m;
  mt_seed(&m, seed);
  for (int64_t i = 0; i < n; ++i) idx[i] = i;
  std_shuffle(idx, (uint64_t)n, sizeof(int64_t), &m);
}
int64_t orc_predict(const EconoOptions* o, uint64_t seed, const int64_t* true_rl, int64_t n, int64_t* out) {
  Mt m;
  mt_seed(&m, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = apply_padding(predict_rl(true_rl[i], o, &m), o->pred_padding_ratio);
  return n;
}
