/*
 * dtopk_oracle.c -- CPU restatement of the reference Dr. Top-k path.
 * TEST INFRASTRUCTURE ONLY (see dtopk_oracle.h): the checker, never the product.
 * Citations are to /root/reference/pkg/src/dtopk/<file>:<line>.
 */
#include "dtopk_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static int ceil_log2_floor(uint64_t n) { /* n.bit_length() - 1 */
  int b = -1;
  while (n) {
    n >>= 1;
    b++;
  }
  return b;
}

int oracle_effective_beta(int beta, int alpha) {
  /* core.py:132-136 */
  if (alpha == 0) return 1;
  int cap = (int)((1ull << alpha) - 1 > 0x7fffffff ? 0x7fffffff : (1ull << alpha) - 1);
  int b = beta < cap ? beta : cap;
  return b < 1 ? 1 : b;
}

int oracle_auto_alpha(uint64_t n, uint64_t k, double const_c, int beta) {
  /* tuning.py:74-90: floor(0.5 (log2 n - log2 k + c)), clamp, shrink until |D| >= k */
  int alpha = (int)floor(0.5 * (log2((double)n) - log2((double)k) + const_c));
  int amax = ceil_log2_floor(n);
  if (alpha < 0) alpha = 0;
  if (alpha > amax) alpha = amax;
  while (alpha > 0) {
    uint64_t w = 1ull << alpha;
    uint64_t s = (n + w - 1) / w;
    if ((uint64_t)oracle_effective_beta(beta, alpha) * s >= k) break;
    alpha--;
  }
  return alpha;
}

/* top-beta ladder with zero-initialised slots: _rows_ladder (delegate.py:93-107);
 * identical output to _rows_top1 / _rows_top2 (delegate.py:58-90) */
static inline void ladder_insert(uint32_t* L, int beta, uint32_t x) {
  if (x <= L[beta - 1]) return;
  int p = beta - 1;
  while (p > 0 && x > L[p - 1]) {
    L[p] = L[p - 1];
    p--;
  }
  L[p] = x;
}

void oracle_extract_delegates(const uint32_t* v, uint64_t n, int alpha, int beta, uint32_t* out) {
  /* delegate.py:132-155: rows of 2^alpha, the last zero padded */
  const uint64_t w = 1ull << alpha;
  const uint64_t s = (n + w - 1) / w;
  for (uint64_t r = 0; r < s; r++) {
    uint32_t* L = out + r * (uint64_t)beta;
    for (int j = 0; j < beta; j++) L[j] = 0;
    const uint64_t lo = r * w, hi = lo + w < n ? lo + w : n;
    if (beta == 1) {
      uint32_t m = 0;
      for (uint64_t i = lo; i < hi; i++) m = v[i] > m ? v[i] : m;
      L[0] = m;
    } else if (beta == 2) {
      uint32_t m1 = 0, m2 = 0;
      for (uint64_t i = lo; i < hi; i++) {
        uint32_t x = v[i];
        uint32_t h = x > m1 ? x : m1, l = x > m1 ? m1 : x;
        m1 = h;
        m2 = l > m2 ? l : m2;
      }
      L[0] = m1;
      L[1] = m2;
    } else {
      for (uint64_t i = lo; i < hi; i++) ladder_insert(L, beta, v[i]);
    }
  }
}

uint32_t oracle_radix_threshold(const uint32_t* vals, uint64_t m, uint64_t k, int skip_last, uint64_t* reads) {
  /* kernels.py:130-165 with digit_bits = 8 */
  uint32_t bits = 0, mask = 0;
  uint64_t remaining = k;
  const int passes = 4 - (skip_last ? 1 : 0);
  uint64_t hist[256];
  for (int p = 0; p < passes; p++) {
    const int shift = 24 - 8 * p;
    memset(hist, 0, sizeof(hist));
    for (uint64_t i = 0; i < m; i++) {
      const uint32_t x = vals[i];
      if ((x & mask) == bits) hist[(x >> shift) & 0xffu]++;
    }
    if (reads) *reads += m;
    /* at_least[d] = sum_{d' >= d} hist[d']; digit = max d with at_least[d] >= remaining */
    uint64_t above = 0;
    int digit = 0;
    for (int d = 255; d >= 0; d--) {
      if (above + hist[d] >= remaining) {
        digit = d;
        break;
      }
      above += hist[d];
    }
    remaining -= above;
    bits |= (uint32_t)digit << shift;
    mask |= 0xffu << shift;
  }
  if (reads) *reads += m; /* _extract_at_least / _extract_exact read the input once */
  if (!skip_last) return bits;
  /* _extract_at_least (kernels.py:99-106): threshold = min of elements >= edge */
  uint32_t mn = 0xffffffffu;
  for (uint64_t i = 0; i < m; i++)
    if (vals[i] >= bits && vals[i] < mn) mn = vals[i];
  return mn;
}

static int cmp_desc_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? 1 : (x > y ? -1 : 0);
}

/* exact top-k values of vals (radix exact, then sort desc): _run_backend_exact + np.sort */
static void exact_topk_values(const uint32_t* vals, uint64_t m, uint64_t k, uint32_t* out, oracle_stats* st) {
  uint64_t reads = 0;
  const uint32_t kth = oracle_radix_threshold(vals, m, k, 0, &reads);
  uint64_t o = 0;
  for (uint64_t i = 0; i < m; i++)
    if (vals[i] > kth) out[o++] = vals[i];
  while (o < k) out[o++] = kth; /* ties: values only, the multiset is what counts */
  qsort(out, k, sizeof(uint32_t), cmp_desc_u32);
  if (st) {
    st->elements_read += reads;
    st->elements_written += k;
  }
}

int oracle_dr_topk(const uint32_t* v, uint64_t n, uint64_t k, int alpha, int beta, int skip_last, int direct,
                   uint32_t* out_values, oracle_stats* st) {
  oracle_stats local;
  if (!st) st = &local;
  memset(st, 0, sizeof(*st));
  if (n == 0 || k < 1 || k > n || beta < 1) return -1;
  if (direct) {
    /* pipeline.py:184-191 */
    exact_topk_values(v, n, k, out_values, st);
    st->threshold = out_values[k - 1];
    return 0;
  }
  const uint64_t w = 1ull << alpha;
  const uint64_t s = (n + w - 1) / w;
  const uint64_t dlen = (uint64_t)beta * s;
  if (k > dlen) return -2; /* first_topk InvalidK (pipeline.py:100-101) */
  uint32_t* D = (uint32_t*)malloc(dlen * 4);
  if (!D) return -3;
  oracle_extract_delegates(v, n, alpha, beta, D);
  st->elements_read += n;
  st->elements_written += dlen;
  st->delegate_vector_len = dlen;

  /* first_topk (pipeline.py:87-116) */
  uint64_t reads = 0;
  const uint32_t theta = oracle_radix_threshold(D, dlen, k, skip_last, &reads);
  st->elements_read += reads;
  st->theta = theta;
  uint64_t tsize = 0, fq = 0, pq = 0, npart = 0;
  for (uint64_t r = 0; r < s; r++) {
    int c = 0;
    for (int j = 0; j < beta; j++) c += D[r * beta + j] >= theta;
    tsize += (uint64_t)c;
    if (c == beta)
      fq++;
    else if (c > 0) {
      pq++;
      npart += (uint64_t)c;
    }
  }
  st->elements_written += skip_last ? tsize : k; /* _extract_at_least / _extract_exact */
  st->fully_qualified_subranges = fq;
  st->partially_qualified_subranges = pq;

  /* concatenate_filtered (pipeline.py:119-159) + partial values -> pool */
  uint64_t clen = 0;
  for (uint64_t r = 0; r < s; r++) {
    int c = 0;
    for (int j = 0; j < beta; j++) c += D[r * beta + j] >= theta;
    if (c != beta) continue;
    const uint64_t lo = r * w, hi = lo + w < n ? lo + w : n;
    for (uint64_t i = lo; i < hi; i++) clen += v[i] >= theta;
  }
  st->elements_read += fq * w;
  st->elements_written += clen;
  st->concatenated_len = clen;
  const uint64_t plen = clen + npart;
  st->pool_len = plen;
  uint32_t* pool = (uint32_t*)malloc((plen ? plen : 1) * 4);
  if (!pool) {
    free(D);
    return -3;
  }
  uint64_t o = 0;
  for (uint64_t r = 0; r < s; r++) {
    int c = 0;
    for (int j = 0; j < beta; j++) c += D[r * beta + j] >= theta;
    if (c == beta) {
      const uint64_t lo = r * w, hi = lo + w < n ? lo + w : n;
      for (uint64_t i = lo; i < hi; i++)
        if (v[i] >= theta) pool[o++] = v[i];
    }
  }
  for (uint64_t r = 0; r < s; r++) {
    int c = 0;
    for (int j = 0; j < beta; j++) c += D[r * beta + j] >= theta;
    if (c > 0 && c < beta)
      for (int j = 0; j < beta; j++)
        if (D[r * beta + j] >= theta) pool[o++] = D[r * beta + j];
  }
  /* second top-k (pipeline.py:212-220) */
  if (plen == k) {
    memcpy(out_values, pool, k * 4);
    qsort(out_values, k, sizeof(uint32_t), cmp_desc_u32);
  } else {
    exact_topk_values(pool, plen, k, out_values, st);
  }
  st->threshold = out_values[k - 1];
  free(pool);
  free(D);
  return 0;
}

typedef struct {
  uint32_t key;
  int64_t idx;
} kv_pair;

static int cmp_pair(const void* a, const void* b) {
  const kv_pair* x = (const kv_pair*)a;
  const kv_pair* y = (const kv_pair*)b;
  if (x->key != y->key) return x->key < y->key ? 1 : -1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

void oracle_topk_indices(const uint32_t* keys, uint64_t n, uint64_t k, uint32_t kth, uint32_t* out_keys,
                         int64_t* out_idx) {
  /* kernels.py:89-96 on the whole input: gt first, then eq in scan order */
  kv_pair* buf = (kv_pair*)malloc((k ? k : 1) * sizeof(kv_pair));
  uint64_t g = 0;
  for (uint64_t i = 0; i < n && g < k; i++)
    if (keys[i] > kth) {
      buf[g].key = keys[i];
      buf[g].idx = (int64_t)i;
      g++;
    }
  uint64_t o = g;
  for (uint64_t i = 0; i < n && o < k; i++)
    if (keys[i] == kth) {
      buf[o].key = kth;
      buf[o].idx = (int64_t)i;
      o++;
    }
  qsort(buf, o, sizeof(kv_pair), cmp_pair);
  for (uint64_t i = 0; i < o; i++) {
    out_keys[i] = buf[i].key;
    out_idx[i] = buf[i].idx;
  }
  free(buf);
}

void oracle_f32_to_keys(const uint32_t* bits, uint64_t n, int largest, uint32_t* out) {
  for (uint64_t i = 0; i < n; i++) {
    const uint32_t b = bits[i];
    const uint32_t u = (b >> 31) ? ~b : (b | 0x80000000u);
    out[i] = largest ? u : ~u;
  }
}

typedef struct {
  const uint32_t* v;
  uint64_t len, k;
  int beta;
  double c;
  uint32_t* out;
  int rc;
} lane_arg;

static void* lane_main(void* p) {
  /* distributed._worker_lane (distributed.py:140-181): dr_topk on one partition */
  lane_arg* a = (lane_arg*)p;
  const uint64_t k = a->k < a->len ? a->k : a->len;
  int alpha = oracle_auto_alpha(a->len, k, a->c, a->beta);
  int beta = oracle_effective_beta(a->beta, alpha);
  const uint64_t w = 1ull << alpha;
  const int direct = ((uint64_t)beta * ((a->len + w - 1) / w) < k) || (w <= (uint64_t)beta);
  a->rc = oracle_dr_topk(a->v, a->len, k, alpha, beta, 1, direct, a->out, NULL);
  return NULL;
}

int oracle_dr_topk_partitioned(const uint32_t* v, uint64_t n, uint64_t k, int beta, double const_c, int workers,
                               uint32_t* out_values) {
  if (workers < 1 || n == 0 || k < 1 || k > n) return -1;
  const uint64_t plen = (n + workers - 1) / workers; /* plan(): ceil(n / workers) */
  if (k > plen) return -2;
  const uint64_t parts = (n + plen - 1) / plen;
  lane_arg* args = (lane_arg*)calloc(parts, sizeof(lane_arg));
  pthread_t* th = (pthread_t*)calloc(parts, sizeof(pthread_t));
  uint32_t* cand = (uint32_t*)malloc(parts * k * 4);
  uint64_t total = 0;
  for (uint64_t p = 0; p < parts; p++) {
    args[p].v = v + p * plen;
    args[p].len = (p + 1) * plen <= n ? plen : n - p * plen;
    args[p].k = k;
    args[p].beta = beta;
    args[p].c = const_c;
    args[p].out = cand + total;
    total += args[p].len < k ? args[p].len : k;
    pthread_create(&th[p], NULL, lane_main, &args[p]);
  }
  int rc = 0;
  for (uint64_t p = 0; p < parts; p++) {
    pthread_join(th[p], NULL);
    if (args[p].rc) rc = args[p].rc;
  }
  if (!rc) exact_topk_values(cand, total, k, out_values, NULL); /* sort_and_choose (distributed.py:243-244) */
  free(cand);
  free(th);
  free(args);
  return rc;
}

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

typedef struct {
  uint32_t* out;
  uint64_t lo, hi, key, offset;
} gen_arg;

static void* gen_main(void* p) {
  gen_arg* a = (gen_arg*)p;
  for (uint64_t i = a->lo; i < a->hi; i++) a->out[i] = (uint32_t)(splitmix64(a->key + a->offset + i) >> 32);
  return NULL;
}

void oracle_generate_uniform(uint32_t* out, uint64_t n, uint64_t seed, uint64_t offset, int threads) {
  if (threads < 1) threads = 1;
  const uint64_t key = splitmix64(seed ^ 0xD1B54A32D192ED03ull);
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  gen_arg* args = (gen_arg*)calloc((size_t)threads, sizeof(gen_arg));
  const uint64_t per = (n + (uint64_t)threads - 1) / (uint64_t)threads;
  for (int t = 0; t < threads; t++) {
    args[t].out = out;
    args[t].lo = (uint64_t)t * per < n ? (uint64_t)t * per : n;
    args[t].hi = (uint64_t)(t + 1) * per < n ? (uint64_t)(t + 1) * per : n;
    args[t].key = key;
    args[t].offset = offset;
    pthread_create(&th[t], NULL, gen_main, &args[t]);
  }
  for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
  free(args);
  free(th);
}
