/*
 * bb_oracle.c -- TEST INFRASTRUCTURE ONLY (see bb_oracle.h).
 *
 * A plain-C restatement of the reference simulator's algorithm, written from
 * the behaviour of /root/reference/proj/include/binbatch/{rng,service_dist,
 * binning,simulator,experiment}.hpp.  It is the checker the GPU engine is
 * compared against; it is never part of the product path.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, no -march, matching the
 * reference's Release flags proj/CMakeLists.txt:6-8 so no FMA contraction
 * changes any bit).
 */
#include "bb_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* bbo_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- rng.hpp */

/* detail::splitmix64, rng.hpp:16-21 */
uint64_t bbo_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

/* std::mt19937_64 as fixed by ISO C++ [rand.predef] (the engine behind
 * RandomStream, rng.hpp:52): w=64 n=312 m=156 r=31. */
#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t s[MT_N];
  int i;
} mt64;

static void mt_seed(mt64* g, uint64_t seed) {
  g->s[0] = seed;
  for (int k = 1; k < MT_N; ++k)
    g->s[k] = 6364136223846793005ULL * (g->s[k - 1] ^ (g->s[k - 1] >> 62)) + (uint64_t)k;
  g->i = MT_N;
}

static void mt_refill(mt64* g) {
  const uint64_t hi = 0xFFFFFFFF80000000ULL, lo = 0x7FFFFFFFULL;
  for (int k = 0; k < MT_N; ++k) {
    uint64_t y = (g->s[k] & hi) | (g->s[(k + 1) % MT_N] & lo);
    uint64_t v = g->s[(k + MT_M) % MT_N] ^ (y >> 1);
    if (y & 1) v ^= 0xB5026F5AA96619E9ULL;
    g->s[k] = v;
  }
  g->i = 0;
}

static uint64_t mt_next(mt64* g) {
  if (g->i >= MT_N) mt_refill(g);
  uint64_t z = g->s[g->i++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

/* RandomStream(seed): engine seeded with splitmix64(seed), rng.hpp:30 */
static void stream_init(mt64* g, uint64_t seed) { mt_seed(g, bbo_splitmix64(seed)); }

/* RandomStream::derive, rng.hpp:33-35 */
static void stream_derive(mt64* g, uint64_t master, uint64_t id) {
  stream_init(g, bbo_splitmix64(master ^ (0x632BE59BD9B4E019ULL * (id + 1))));
}

/* uniform01, rng.hpp:38 */
static double u01(mt64* g) { return (double)(mt_next(g) >> 11) * 0x1.0p-53; }

/* experiment.hpp:90-92 */
uint64_t bbo_replication_seed(uint64_t master, uint64_t rep) {
  return bbo_splitmix64(master ^ bbo_splitmix64(rep + 0x51ED2701A7B4E5D3ULL));
}

void bbo_stream_uniform01(uint64_t seed, uint64_t stream_id, uint64_t n, double* out) {
  mt64* g = (mt64*)malloc(sizeof(mt64));
  stream_derive(g, seed, stream_id);
  for (uint64_t i = 0; i < n; ++i) out[i] = u01(g);
  free(g);
}

/* RandomStream(seed).uniform01() n times (rng.hpp:30, :38) -- e.g. the
 * acceptance suite's trace generator RandomStream trace_rng(424242),
 * acceptance.cpp:370-374 */
void bbo_plain_uniform01(uint64_t seed, uint64_t n, double* out) {
  mt64* g = (mt64*)malloc(sizeof(mt64));
  stream_init(g, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = u01(g);
  free(g);
}

/* schedule_arrivals, simulator.hpp:174-185: t += exponential(rate), or t = 0
 * for the overload rate; exponential = -log1p(-u)/rate (rng.hpp:43). */
void bbo_generate_arrivals(uint64_t seed, double rate, uint64_t n, double* out) {
  mt64* g = (mt64*)malloc(sizeof(mt64));
  stream_derive(g, seed, 0);
  double t = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    if (isinf(rate)) t = 0.0;
    else t += -log1p(-u01(g)) / rate;
    out[i] = t;
  }
  free(g);
}

/* ------------------------------------------------------------ binning.hpp */

/* assign_bin, binning.hpp:133-144: out-of-support (or NaN) is a domain error;
 * the top edge closes into bin k; otherwise upper_bound(edges) - begin. */
int bbo_assign_bin(const double* e, uint64_t n_edges, double len, uint32_t* bin) {
  if (!(len >= e[0]) || !(len <= e[n_edges - 1]))
    return fail(BBO_EDOMAIN, "assign_bin: length %.17g outside bin support [%.17g, %.17g]", len,
                e[0], e[n_edges - 1]);
  if (len == e[n_edges - 1]) {
    *bin = (uint32_t)(n_edges - 1);
    return BBO_OK;
  }
  uint64_t lo = 0, hi = n_edges; /* first index with e[idx] > len */
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (e[mid] > len) hi = mid;
    else lo = mid + 1;
  }
  *bin = (uint32_t)lo;
  return BBO_OK;
}

/* interpolated_quantile, binning.hpp:98-104 */
double bbo_interpolated_quantile(const double* sorted, uint64_t n, double q) {
  const double pos = q * (double)(n - 1);
  const uint64_t idx = (uint64_t)pos;
  if (idx + 1 >= n) return sorted[n - 1];
  const double frac = pos - (double)idx;
  return sorted[idx] + frac * (sorted[idx + 1] - sorted[idx]);
}

/* mean_std, experiment.hpp:188-200 (sample std, two-pass) */
void bbo_mean_std(const double* xs, uint64_t n, double* mean, double* sd) {
  double sum = 0;
  for (uint64_t i = 0; i < n; ++i) sum += xs[i];
  *mean = sum / (double)n;
  if (n < 2) {
    *sd = 0;
    return;
  }
  double ss = 0;
  for (uint64_t i = 0; i < n; ++i) ss += (xs[i] - *mean) * (xs[i] - *mean);
  *sd = sqrt(ss / ((double)n - 1.0));
}

/* ---------------------------------------------------------- simulator.hpp */

enum { EV_DONE = 0, EV_ARRIVAL = 1, EV_FORM = 2, EV_TIMER = 3, EV_DRAIN = 4 };

typedef struct {
  double time;
  int rank; /* batch_done 0 < arrival 1 < formation-class 2, simulator.hpp:170 */
  uint64_t seq;
  int kind;
  uint64_t a, b;
} event;

typedef struct {
  event* v;
  uint64_t n, cap;
} heap;

/* EventAfter ordering, simulator.hpp:108-114: earliest (time, rank, seq) first */
static int ev_before(const event* x, const event* y) {
  if (x->time != y->time) return x->time < y->time;
  if (x->rank != y->rank) return x->rank < y->rank;
  return x->seq < y->seq;
}

static void heap_push(heap* h, event e) {
  if (h->n == h->cap) {
    h->cap = h->cap ? 2 * h->cap : 1024;
    h->v = (event*)realloc(h->v, h->cap * sizeof(event));
  }
  uint64_t i = h->n++;
  while (i > 0) {
    uint64_t p = (i - 1) / 2;
    if (!ev_before(&e, &h->v[p])) break;
    h->v[i] = h->v[p];
    i = p;
  }
  h->v[i] = e;
}

static event heap_pop(heap* h) {
  event top = h->v[0];
  event last = h->v[--h->n];
  uint64_t i = 0;
  for (;;) {
    uint64_t l = 2 * i + 1, r = l + 1, m = i;
    const event* best = &last;
    if (l < h->n && ev_before(&h->v[l], best)) { m = l; best = &h->v[l]; }
    if (r < h->n && ev_before(&h->v[r], best)) { m = r; }
    if (m == i) break;
    h->v[i] = h->v[m];
    i = m;
  }
  if (h->n) h->v[i] = last;
  return top;
}

/* simple FIFO of u64 with capacity fixed up front */
typedef struct {
  uint64_t* v;
  uint64_t head, tail;
} fifo;

typedef struct {
  const bbo_config* cfg;
  const bbo_inputs* in;
  uint64_t k;
  mt64 svc_rng, err_rng;
  heap ev;
  uint64_t next_seq;
  double now;
  /* bin queues (simulator.hpp:315): each request enters exactly one queue
   * once, so a growable array with a head index is a deque here */
  uint64_t** q;
  uint64_t* qhead;
  uint64_t* qtail;
  uint64_t* qcap;
  fifo central;
  /* requests */
  double *arr, *svc, *comp;
  uint32_t *tbin, *pbin;
  uint64_t* rbatch;
  uint64_t n_arrived;
  /* batches */
  uint64_t nb;
  uint32_t* bbin;
  uint64_t *bsize, *bfirst;
  double *bformed, *bstart, *bfinish, *bservice;
  uint64_t* members;
  uint64_t n_members;
  uint64_t* bin_counts;
  uint64_t idle, completed;
  double busy, last_completion;
  int err;
  double* sorted_table;
} engine;

static void schedule(engine* E, double t, int kind, uint64_t a, uint64_t b) {
  event e;
  e.time = t;
  e.rank = kind == EV_DONE ? 0 : kind == EV_ARRIVAL ? 1 : 2;
  e.seq = E->next_seq++;
  e.kind = kind;
  e.a = a;
  e.b = b;
  heap_push(&E->ev, e);
}

static uint64_t qsize(engine* E, uint64_t b) { return E->qtail[b] - E->qhead[b]; }

/* dispatch, simulator.hpp:256-267 */
static void dispatch(engine* E) {
  while (E->idle > 0 && E->central.head < E->central.tail) {
    uint64_t idx = E->central.v[E->central.head++];
    E->bstart[idx] = E->now;
    E->bfinish[idx] = E->now + E->bservice[idx];
    E->busy += E->bservice[idx];
    --E->idle;
    schedule(E, E->bfinish[idx], EV_DONE, idx, 0);
  }
}

/* form_batch, simulator.hpp:237-254 */
static void form_batch(engine* E, uint64_t bin, uint64_t size) {
  uint64_t idx = E->nb++;
  E->bbin[idx] = (uint32_t)bin;
  E->bformed[idx] = E->now;
  E->bstart[idx] = NAN;
  E->bfinish[idx] = NAN;
  E->bsize[idx] = size;
  E->bfirst[idx] = E->n_members;
  double s = 0.0;
  for (uint64_t i = 0; i < size; ++i) {
    uint64_t id = E->q[bin][E->qhead[bin]++];
    E->members[E->n_members++] = id;
    E->rbatch[id] = idx;
    s = E->svc[id] > s ? E->svc[id] : s; /* std::max(s, svc): keeps s on ties */
  }
  E->bservice[idx] = s;
  E->bin_counts[bin - 1]++;
  E->central.v[E->central.tail++] = idx;
  dispatch(E);
}

/* rearm_timer, simulator.hpp:230-235 */
static void rearm_timer(engine* E, uint64_t bin) {
  if (!E->cfg->has_max_batch_wait || qsize(E, bin) == 0) return;
  uint64_t oldest = E->q[bin][E->qhead[bin]];
  double due = E->arr[oldest] + E->cfg->max_batch_wait;
  schedule(E, E->now > due ? E->now : due, EV_TIMER, bin, oldest);
}

/* service sampler: run_simulation_detailed (:331-334 -> sample,
 * service_dist.hpp:94-101) or replay_trace_detailed (:349-352) */
static double draw_service(engine* E, uint64_t id) {
  const bbo_config* c = E->cfg;
  switch (c->service_kind) {
    case BBO_SVC_UNIFORM: return c->lo + (c->hi - c->lo) * u01(&E->svc_rng);
    case BBO_SVC_EXPONENTIAL: return -log1p(-u01(&E->svc_rng)) / c->rate;
    case BBO_SVC_EMPIRICAL: /* make_empirical keeps the samples sorted, service_dist.hpp:110-118 */
      return E->sorted_table[mt_next(&E->svc_rng) % c->n_table];
    case BBO_SVC_TRACE_RESAMPLE: return c->table[mt_next(&E->svc_rng) % c->n_table];
    case BBO_SVC_TRACE_CYCLIC: return c->table[id % c->n_table];
    case BBO_SVC_ARRAYS: return E->in->services[id];
    case BBO_SVC_LINEAR: {
      double len = c->lo + (c->hi - c->lo) * u01(&E->svc_rng);
      return c->lin_b * len + c->lin_a; /* tokens_to_time, workload.hpp:167-170 */
    }
    case BBO_SVC_LOGNORMAL: {
      double u1 = u01(&E->svc_rng), u2 = u01(&E->svc_rng);
      double z = sqrt(-2.0 * log1p(-u1)) * cos(6.283185307179586 * u2);
      return exp(c->mu + c->sigma * z);
    }
  }
  return NAN;
}

/* predict_bin, binning.hpp:231-261 */
static int predict(engine* E, uint64_t id, uint32_t tb, uint32_t* pb) {
  const bbo_config* c = E->cfg;
  const uint64_t k = E->k;
  if (E->in && E->in->pred_bin) {
    uint32_t p = E->in->pred_bin[id];
    if (p < 1 || p > k) return fail(BBO_EINVAL, "predicted bin %u out of range [1,%llu]", p,
                                    (unsigned long long)k);
    *pb = p;
    return BBO_OK;
  }
  if (c->error_kind == BBO_ERR_PERFECT) {
    *pb = tb;
    return BBO_OK;
  }
  if (c->error_kind == BBO_ERR_SYMMETRIC) {
    const double p = c->p_error;
    if (k == 1 || p == 0) {
      *pb = tb;
      return BBO_OK;
    }
    const double u = (E->in && E->in->u_err) ? E->in->u_err[id] : u01(&E->err_rng);
    if (tb == 1) *pb = u < p ? 2 : tb;
    else if (tb == k) *pb = u < p ? (uint32_t)(k - 1) : tb;
    else if (u < p) *pb = tb - 1;
    else if (u >= 1.0 - p) *pb = tb + 1;
    else *pb = tb;
    return BBO_OK;
  }
  /* confusion: cumulative row search, guard returns k */
  const double* row = c->confusion + (uint64_t)(tb - 1) * k;
  const double u = (E->in && E->in->u_err) ? E->in->u_err[id] : u01(&E->err_rng);
  double cum = 0.0;
  for (uint64_t j = 0; j < k; ++j) {
    cum += row[j];
    if (u < cum) {
      *pb = (uint32_t)(j + 1);
      return BBO_OK;
    }
  }
  *pb = (uint32_t)k;
  return BBO_OK;
}

/* on_arrival, simulator.hpp:187-206 */
static int on_arrival(engine* E, uint64_t id) {
  const double svc = draw_service(E, id);
  if (!(svc > 0) || !isfinite(svc))
    return fail(BBO_EDOMAIN, "simulation: drew a non-positive service time");
  uint32_t tb = 0, pb = 0;
  int st = bbo_assign_bin(E->cfg->edges, E->cfg->n_edges, svc, &tb);
  if (st) return st;
  st = predict(E, id, tb, &pb);
  if (st) return st;
  E->arr[id] = E->now;
  E->svc[id] = svc;
  E->tbin[id] = tb;
  E->pbin[id] = pb;
  E->rbatch[id] = UINT64_MAX;
  E->comp[id] = NAN;
  if (E->qtail[pb] == E->qcap[pb]) {
    E->qcap[pb] = E->qcap[pb] ? 2 * E->qcap[pb] : 256;
    E->q[pb] = (uint64_t*)realloc(E->q[pb], E->qcap[pb] * sizeof(uint64_t));
  }
  E->q[pb][E->qtail[pb]++] = id;
  const uint64_t qs = qsize(E, pb);
  if (qs == E->cfg->batch_size) schedule(E, E->now, EV_FORM, pb, 0);
  else if (qs == 1 && E->cfg->has_max_batch_wait)
    schedule(E, E->now + E->cfg->max_batch_wait, EV_TIMER, pb, id);
  if (++E->n_arrived == E->cfg->n_requests && E->cfg->flush_partial)
    for (uint64_t b = 1; b <= E->k; ++b) schedule(E, E->now, EV_DRAIN, b, 0);
  return BBO_OK;
}

static int cmp_double(const void* x, const void* y) {
  double a = *(const double*)x, b = *(const double*)y;
  return (a > b) - (a < b);
}

/* validate, simulator.hpp:153-167 (+ replay_trace's checks :345-348) */
static int validate(const bbo_config* c, const bbo_inputs* in) {
  if (c->n_edges < 2 || !c->edges) return fail(BBO_EINVAL, "sim config: bins not configured");
  if (c->n_requests < c->batch_size)
    return fail(BBO_EINVAL, "sim config: n_requests must be >= batch_size");
  if (c->batch_size == 0) return fail(BBO_EINVAL, "sim config: batch size must be >= 1");
  if (c->n_servers == 0) return fail(BBO_EINVAL, "sim config: need at least one server");
  if (!(c->arrival_rate > 0))
    return fail(BBO_EINVAL, "sim config: arrival rate must be positive (or overload)");
  if (c->has_max_batch_wait && !(c->max_batch_wait > 0))
    return fail(BBO_EINVAL, "sim config: max_batch_wait must be positive");
  if (c->error_kind == BBO_ERR_CONFUSION && !c->confusion)
    return fail(BBO_EINVAL, "sim config: confusion matrix size does not match bin count");
  if (c->service_kind == BBO_SVC_ARRAYS && (!in || !in->services))
    return fail(BBO_EINVAL, "trace arrays: services missing");
  if (c->service_kind == BBO_SVC_TRACE_CYCLIC || c->service_kind == BBO_SVC_TRACE_RESAMPLE ||
      c->service_kind == BBO_SVC_EMPIRICAL) {
    if (!c->table || c->n_table == 0) return fail(BBO_EINVAL, "replay_trace: empty trace");
    for (uint64_t i = 0; i < c->n_table; ++i)
      if (!(c->table[i] > 0) || !isfinite(c->table[i]))
        return fail(BBO_EINVAL, "replay_trace: trace lengths must be positive");
  }
  if (in && in->arrivals)
    for (uint64_t i = 1; i < c->n_requests; ++i)
      if (!(in->arrivals[i] >= in->arrivals[i - 1]))
        return fail(BBO_EINVAL, "trace arrays: arrivals must be non-decreasing");
  return BBO_OK;
}

/* detail::Engine::run + finish, simulator.hpp:128-150, :279-304 */
int bbo_run(const bbo_config* cfg, const bbo_inputs* in, bbo_metrics* m, bbo_detail* d) {
  int st = validate(cfg, in);
  if (st) return st;
  const uint64_t n = cfg->n_requests, k = cfg->n_edges - 1;
  engine* E = (engine*)calloc(1, sizeof(engine));
  E->cfg = cfg;
  E->in = in;
  E->k = k;
  stream_derive(&E->svc_rng, cfg->seed, 1);
  stream_derive(&E->err_rng, cfg->seed, 2);
  E->q = (uint64_t**)calloc(k + 1, sizeof(uint64_t*));
  E->qhead = (uint64_t*)calloc(k + 1, sizeof(uint64_t));
  E->qtail = (uint64_t*)calloc(k + 1, sizeof(uint64_t));
  E->qcap = (uint64_t*)calloc(k + 1, sizeof(uint64_t));
  E->central.v = (uint64_t*)malloc(n * sizeof(uint64_t));
  E->arr = (double*)malloc(n * sizeof(double));
  E->svc = (double*)malloc(n * sizeof(double));
  E->comp = (double*)malloc(n * sizeof(double));
  E->tbin = (uint32_t*)malloc(n * sizeof(uint32_t));
  E->pbin = (uint32_t*)malloc(n * sizeof(uint32_t));
  E->rbatch = (uint64_t*)malloc(n * sizeof(uint64_t));
  E->bbin = (uint32_t*)malloc(n * sizeof(uint32_t));
  E->bsize = (uint64_t*)malloc(n * sizeof(uint64_t));
  E->bfirst = (uint64_t*)malloc(n * sizeof(uint64_t));
  E->bformed = (double*)malloc(n * sizeof(double));
  E->bstart = (double*)malloc(n * sizeof(double));
  E->bfinish = (double*)malloc(n * sizeof(double));
  E->bservice = (double*)malloc(n * sizeof(double));
  E->members = (uint64_t*)malloc(n * sizeof(uint64_t));
  E->bin_counts = (uint64_t*)calloc(k, sizeof(uint64_t));
  E->idle = cfg->n_servers;
  if (cfg->service_kind == BBO_SVC_EMPIRICAL) {
    E->sorted_table = (double*)malloc(cfg->n_table * sizeof(double));
    memcpy(E->sorted_table, cfg->table, cfg->n_table * sizeof(double));
    qsort(E->sorted_table, cfg->n_table, sizeof(double), cmp_double);
  }

  /* schedule_arrivals, :174-185 */
  {
    mt64* g = (mt64*)malloc(sizeof(mt64));
    stream_derive(g, cfg->seed, 0);
    double t = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
      if (in && in->arrivals) t = in->arrivals[i];
      else if (isinf(cfg->arrival_rate)) t = 0.0;
      else t += -log1p(-u01(g)) / cfg->arrival_rate;
      schedule(E, t, EV_ARRIVAL, i, 0);
    }
    free(g);
  }

  /* the event loop, :137-148 */
  while (E->ev.n && !st) {
    event ev = heap_pop(&E->ev);
    E->now = ev.time;
    switch (ev.kind) {
      case EV_DONE: { /* on_batch_done, :269-277 */
        ++E->idle;
        for (uint64_t i = 0; i < E->bsize[ev.a]; ++i)
          E->comp[E->members[E->bfirst[ev.a] + i]] = E->bfinish[ev.a];
        E->completed += E->bsize[ev.a];
        E->last_completion = E->last_completion > E->now ? E->last_completion : E->now;
        dispatch(E);
        break;
      }
      case EV_ARRIVAL: st = on_arrival(E, ev.a); break;
      case EV_FORM: /* on_formation, :208-216 */
        if (qsize(E, ev.a) < cfg->batch_size) break;
        form_batch(E, ev.a, cfg->batch_size);
        if (qsize(E, ev.a) >= cfg->batch_size) schedule(E, E->now, EV_FORM, ev.a, 0);
        else rearm_timer(E, ev.a);
        break;
      case EV_TIMER: { /* on_flush_timer, :223-228 */
        uint64_t qs = qsize(E, ev.a);
        if (qs == 0 || E->q[ev.a][E->qhead[ev.a]] != ev.b) break;
        form_batch(E, ev.a, qs < cfg->batch_size ? qs : cfg->batch_size);
        rearm_timer(E, ev.a);
        break;
      }
      case EV_DRAIN: /* on_drain, :218-221 */
        while (qsize(E, ev.a) >= cfg->batch_size) form_batch(E, ev.a, cfg->batch_size);
        if (qsize(E, ev.a)) form_batch(E, ev.a, qsize(E, ev.a));
        break;
    }
  }

  if (!st) {
    /* finish, :279-304 */
    memset(m, 0, sizeof *m);
    m->n_completed = E->completed;
    m->n_batches = E->nb;
    m->busy_time = E->busy;
    if (E->completed > 0) {
      m->makespan = E->last_completion - E->arr[0];
      m->throughput = (double)E->completed / m->makespan;
      m->server_busy_fraction = E->busy / ((double)cfg->n_servers * m->makespan);
      double* lat = (double*)malloc(E->completed * sizeof(double));
      uint64_t nl = 0;
      double sum = 0.0;
      for (uint64_t i = 0; i < n; ++i) {
        if (isnan(E->comp[i])) continue;
        double l = E->comp[i] - E->arr[i];
        lat[nl++] = l;
        sum += l;
      }
      qsort(lat, nl, sizeof(double), cmp_double);
      m->latency_sum = sum;
      m->latency_mean = sum / (double)nl;
      m->latency_p50 = bbo_interpolated_quantile(lat, nl, 0.50);
      m->latency_p99 = bbo_interpolated_quantile(lat, nl, 0.99);
      free(lat);
    }
    if (d) {
#define CP(dst, src, cnt) \
  if (d->dst) memcpy(d->dst, E->src, (cnt) * sizeof(*d->dst))
      CP(req_arrival, arr, n);
      CP(req_service, svc, n);
      CP(req_true_bin, tbin, n);
      CP(req_pred_bin, pbin, n);
      CP(req_batch, rbatch, n);
      CP(req_completion, comp, n);
      CP(bat_bin, bbin, E->nb);
      CP(bat_size, bsize, E->nb);
      CP(bat_first, bfirst, E->nb);
      CP(bat_formed, bformed, E->nb);
      CP(bat_start, bstart, E->nb);
      CP(bat_finish, bfinish, E->nb);
      CP(bat_service, bservice, E->nb);
      CP(members, members, E->n_members);
      CP(per_bin_batch_counts, bin_counts, k);
#undef CP
    }
  }

  for (uint64_t b = 1; b <= k; ++b) free(E->q[b]);
  free(E->q); free(E->qhead); free(E->qtail); free(E->qcap); free(E->central.v);
  free(E->arr); free(E->svc); free(E->comp); free(E->tbin); free(E->pbin); free(E->rbatch);
  free(E->bbin); free(E->bsize); free(E->bfirst); free(E->bformed); free(E->bstart);
  free(E->bfinish); free(E->bservice); free(E->members); free(E->bin_counts); free(E->ev.v);
  free(E->sorted_table);
  free(E);
  return st;
}
