/*
 * otpr_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPU solver's assignment path
 * (arxiv/paper_2203_03732, `otpr`), used as the parity checker for the CUDA
 * path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load this library.  The product path (paper_2203_03732_b200) never
 * links or calls it.
 *
 * Parity pinning: this restatement is checked in tests/test_oracle.py against
 * (a) the golden FNV pins of SURVEY.md §8(c) (measured on the reference),
 * (b) fixtures in tests/golden/ produced by the reference itself
 *     (oracle/_ref, built from /root/reference/proj/src by oracle/Makefile),
 * (c) the reference unit-test known-answer cases (test_core.cpp,
 *     test_assignment.cpp).
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj).  Arithmetic is non-fused IEEE double (build with
 * -ffp-contract=off) and exact integers for all dual bookkeeping.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "otpr_oracle.h"

/* ---------------------------------------------------------------- RNG ---- */

/* splitmix64: src/instances.cpp:41-46 */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

/* std::mt19937_64 (ISO C++ [rand.predef]): the generator the reference uses
 * for every stream (src/instances.cpp:51-52,106,163-165). */
#define MT_NN 312
#define MT_MM 156
typedef struct {
  uint64_t mt[MT_NN];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < MT_NN; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) +
               (uint64_t)i;
  s->idx = MT_NN;
}

static uint64_t mt64_next(mt64* s) {
  static const uint64_t kMatA = 0xB5026F5AA96619E9ULL;
  static const uint64_t kUM = 0xFFFFFFFF80000000ULL;
  static const uint64_t kLM = 0x7FFFFFFFULL;
  if (s->idx >= MT_NN) {
    int i;
    for (i = 0; i < MT_NN - MT_MM; ++i) {
      uint64_t x = (s->mt[i] & kUM) | (s->mt[i + 1] & kLM);
      s->mt[i] = s->mt[i + MT_MM] ^ (x >> 1) ^ ((x & 1ULL) ? kMatA : 0ULL);
    }
    for (; i < MT_NN - 1; ++i) {
      uint64_t x = (s->mt[i] & kUM) | (s->mt[i + 1] & kLM);
      s->mt[i] = s->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ ((x & 1ULL) ? kMatA : 0ULL);
    }
    uint64_t x = (s->mt[MT_NN - 1] & kUM) | (s->mt[0] & kLM);
    s->mt[MT_NN - 1] = s->mt[MT_MM - 1] ^ (x >> 1) ^ ((x & 1ULL) ? kMatA : 0ULL);
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* u01: 53-bit mantissa draw, src/instances.cpp:19-21 */
static double u01(mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }

/* bounded(): rejection sampling, src/instances.cpp:25-32 */
static uint64_t bounded(mt64* s, uint64_t n) {
  const uint64_t limit = ~(uint64_t)0 - (~(uint64_t)0) % n;
  uint64_t x;
  do {
    x = mt64_next(s);
  } while (x >= limit);
  return x % n;
}

static const uint64_t kStreamB = 0x9E3779B97F4A7C15ULL;      /* instances.cpp:14 */
static const uint64_t kStreamMnist = 0xD1B54A32D192ED03ULL;  /* instances.cpp:15 */
static const uint64_t kStreamMassA = 0x8BB84B93962EACC9ULL;  /* instances.cpp:16 */
static const uint64_t kStreamMassB = 0x2545F4914F6CDD1DULL;  /* instances.cpp:17 */

void orc_raw_stream(uint64_t seed, int64_t count, uint64_t* out) {
  mt64 s;
  mt64_seed(&s, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = mt64_next(&s);
}

/* ----------------------------------------------------------- instances -- */

/* gen_uniform_square point streams: src/instances.cpp:48-62 */
int orc_uniform_square_points(int32_t n, uint64_t seed, double* ax, double* ay,
                              double* bx, double* by) {
  if (n < 1) return ORC_PARAMETER;
  mt64 ra, rb;
  mt64_seed(&ra, orc_splitmix64(seed));
  mt64_seed(&rb, orc_splitmix64(seed ^ kStreamB));
  for (int32_t i = 0; i < n; ++i) {
    ax[i] = u01(&ra);
    ay[i] = u01(&ra);
  }
  for (int32_t i = 0; i < n; ++i) {
    bx[i] = u01(&rb);
    by[i] = u01(&rb);
  }
  return ORC_OK;
}

/* Euclidean / sqrt(2) cost of one pair: src/instances.cpp:63,70-75. */
double orc_points_cost(double ax, double ay, double bx, double by) {
  const double sqrt2 = sqrt(2.0);
  const double dx = ax - bx;
  const double dy = ay - by;
  return sqrt(dx * dx + dy * dy) / sqrt2;
}

/* Dense cost matrix of gen_uniform_square: src/instances.cpp:48-78. */
int orc_gen_uniform_square(int32_t n, uint64_t seed, double* cost) {
  if (n < 1) return ORC_PARAMETER;
  double* p = (double*)malloc(sizeof(double) * 4 * (size_t)n);
  if (!p) return ORC_INPUT;
  double *ax = p, *ay = p + n, *bx = p + 2 * (size_t)n, *by = p + 3 * (size_t)n;
  orc_uniform_square_points(n, seed, ax, ay, bx, by);
  for (int32_t a = 0; a < n; ++a)
    for (int32_t b = 0; b < n; ++b)
      cost[(size_t)a * n + b] = orc_points_cost(ax[a], ay[a], bx[b], by[b]);
  free(p);
  return ORC_OK;
}

/* Seeded sample of 2n image indices (partial Fisher-Yates):
 * src/instances.cpp:105-112. */
int orc_mnist_sample(uint32_t count, int32_t n, uint64_t seed, uint32_t* picked) {
  if (n < 1) return ORC_PARAMETER;
  if (count < (uint32_t)(2 * n)) return ORC_INPUT;
  uint32_t* pool = (uint32_t*)malloc(sizeof(uint32_t) * count);
  if (!pool) return ORC_INPUT;
  for (uint32_t i = 0; i < count; ++i) pool[i] = i;
  mt64 r;
  mt64_seed(&r, orc_splitmix64(seed ^ kStreamMnist));
  for (int32_t i = 0; i < 2 * n; ++i) {
    const uint64_t j = (uint64_t)i + bounded(&r, (uint64_t)count - (uint64_t)i);
    uint32_t t = pool[i];
    pool[i] = pool[j];
    pool[j] = t;
  }
  memcpy(picked, pool, sizeof(uint32_t) * 2 * (size_t)n);
  free(pool);
  return ORC_OK;
}

/* load_mnist_pair normalisation + L1/2 cost: src/instances.cpp:114-142.
 * images: 2n x 784 uint8 pixels (already gathered in sample order). */
int orc_mnist_cost(int32_t n, const uint8_t* images, double* cost) {
  const size_t P = 784;
  double* img = (double*)malloc(sizeof(double) * P * 2 * (size_t)n);
  if (!img) return ORC_INPUT;
  for (int32_t i = 0; i < 2 * n; ++i) {
    const uint8_t* src = images + (size_t)i * P;
    double total = 0.0;
    for (size_t p = 0; p < P; ++p) total += src[p];
    if (total == 0.0) {
      free(img);
      return ORC_INPUT;
    }
    for (size_t p = 0; p < P; ++p) img[(size_t)i * P + p] = (double)src[p] / total;
  }
  for (int32_t a = 0; a < n; ++a) {
    const double* ia = img + (size_t)a * P;
    for (int32_t b = 0; b < n; ++b) {
      const double* ib = img + (size_t)(n + b) * P;
      double l1 = 0.0;
      for (size_t p = 0; p < P; ++p) l1 += fabs(ia[p] - ib[p]);
      cost[(size_t)a * n + b] = l1 / 2.0;
    }
  }
  free(img);
  return ORC_OK;
}

/* gen_random_ot_rational: src/instances.cpp:159-191 (renormalize of
 * ot.cpp applied by the caller via orc_ot_renormalize). */
int orc_gen_random_ot_rational(int32_t n_a, int32_t n_b, uint64_t seed,
                               int64_t* wa, int64_t* wb, double* cost) {
  if (n_a < 1 || n_b < 1) return ORC_PARAMETER;
  mt64 rma, rmb, rc;
  mt64_seed(&rma, orc_splitmix64(seed ^ kStreamMassA));
  mt64_seed(&rmb, orc_splitmix64(seed ^ kStreamMassB));
  mt64_seed(&rc, orc_splitmix64(seed));
  for (int32_t a = 0; a < n_a; ++a) wa[a] = (int64_t)bounded(&rma, 50) + 1;
  for (int32_t b = 0; b < n_b; ++b) wb[b] = (int64_t)bounded(&rmb, 50) + 1;
  for (size_t i = 0; i < (size_t)n_a * n_b; ++i) cost[i] = u01(&rc);
  return ORC_OK;
}

/* ------------------------------------------------------------ rounding -- */

/* scaled_floor: src/core.cpp:26-32 */
int64_t orc_scaled_floor(double c, double eps) {
  int64_t k = (int64_t)floor(c / eps);
  while ((double)(k + 1) * eps <= c) ++k;
  while (k > 0 && (double)k * eps > c) --k;
  return k;
}

/* Cost validation: src/core.cpp:10-24. */
int orc_validate_costs(int32_t n_a, int32_t n_b, const double* cost) {
  if (n_a < 1 || n_b < 1) return ORC_PARAMETER;
  for (size_t i = 0; i < (size_t)n_a * n_b; ++i) {
    const double c = cost[i];
    if (!(c >= 0.0 && c <= 1.0)) return ORC_PARAMETER;
  }
  return ORC_OK;
}

/* unit_floor / unit_ceil and the eps checks: src/core.cpp:36-47 */
int orc_units(double eps, int32_t* unit_floor, int32_t* unit_ceil) {
  if (!(eps > 0.0 && eps < 1.0)) return ORC_PARAMETER;
  const int64_t uf = orc_scaled_floor(1.0, eps);
  if (uf + 4 > 2147483647LL) return ORC_PARAMETER;
  *unit_floor = (int32_t)uf;
  *unit_ceil = (int32_t)(((double)uf * eps == 1.0) ? uf : uf + 1);
  return ORC_OK;
}

/* scale_round_costs: src/core.cpp:34-53 (row-major k, rows = A). */
int orc_scale_round_costs(int32_t n_a, int32_t n_b, const double* cost, double eps,
                          int32_t* k, int32_t* unit_floor, int32_t* unit_ceil) {
  int st = orc_validate_costs(n_a, n_b, cost);
  if (st) return st;
  st = orc_units(eps, unit_floor, unit_ceil);
  if (st) return st;
  for (size_t i = 0; i < (size_t)n_a * n_b; ++i)
    k[i] = (int32_t)orc_scaled_floor(cost[i], eps);
  return ORC_OK;
}

/* --------------------------------------------------------- the solver -- */

/* solve_oriented: src/assignment.cpp:316-364, with
 *   init_state            :54-60
 *   collect_workset B'    :113-114 (free b, ascending)
 *   scan_plain            :65-75   (admissible: Y(a)+Y(b) == k+1, a ascending)
 *   greedy (sequential)   :161-171 (b in B' order takes first unclaimed a)
 *   apply_phase           :210-235
 *   termination           :330-334 ((double)n_i <= eps*min(n_a,n_b))
 *   phase cap             :326,356-358
 *   complete_matching     :253-262
 * kT is B-major (kT[b*n_a + a] = k(a,b)) so the scan is row-contiguous; the
 * values and the visiting order are those of the reference.
 * Outputs are in the internal orientation (n_a >= n_b). */
static int solve_oriented(int32_t n_a, int32_t n_b, const int32_t* kT, double eps,
                          int32_t* match_of_a, int32_t* match_of_b, int64_t* y_a,
                          int64_t* y_b, int64_t* free_counts, int64_t free_cap,
                          orc_stats* st) {
  const int32_t m_side = n_a < n_b ? n_a : n_b;
  const double threshold = eps * (double)m_side;
  const int64_t phase_cap = (int64_t)ceil((1.0 + 2.0 * eps) / (eps * eps)) + 8;

  for (int32_t a = 0; a < n_a; ++a) {
    match_of_a[a] = -1;
    y_a[a] = 0;
  }
  for (int32_t b = 0; b < n_b; ++b) {
    match_of_b[b] = -1;
    y_b[b] = 1;
  }
  st->phases = 0;
  st->sum_ni = 0;
  st->full_match_termination = 0;

  int32_t* bfree = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_b);
  int32_t* prime_a = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_b);
  int32_t* claimed = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_a);
  if (!bfree || !prime_a || !claimed) {
    free(bfree);
    free(prime_a);
    free(claimed);
    return ORC_INPUT;
  }
  for (int32_t a = 0; a < n_a; ++a) claimed[a] = 0;

  int status = ORC_OK;
  for (;;) {
    int64_t n_i = 0;
    for (int32_t b = 0; b < n_b; ++b)
      if (match_of_b[b] == -1) bfree[n_i++] = b;
    if ((double)n_i <= threshold) {
      st->full_match_termination = (n_i == 0);
      break;
    }
    const int32_t phase_tag = (int32_t)(st->phases + 1);
    /* scan + sequential greedy, fused: b in ascending order takes its first
     * admissible a that no earlier b of this phase claimed. */
    for (int64_t i = 0; i < n_i; ++i) {
      const int32_t b = bfree[i];
      const int64_t yb = y_b[b];
      const int32_t* row = kT + (size_t)b * n_a;
      prime_a[i] = -1;
      for (int32_t a = 0; a < n_a; ++a) {
        if (y_a[a] + yb == (int64_t)row[a] + 1 && claimed[a] != phase_tag) {
          claimed[a] = phase_tag;
          prime_a[i] = a;
          break;
        }
      }
    }
    /* apply_phase */
    for (int64_t i = 0; i < n_i; ++i) {
      const int32_t a = prime_a[i];
      const int32_t b = bfree[i];
      if (a < 0) continue;
      const int32_t old_b = match_of_a[a];
      if (old_b != -1) match_of_b[old_b] = -1;
      match_of_a[a] = b;
      match_of_b[b] = a;
    }
    for (int64_t i = 0; i < n_i; ++i) {
      if (prime_a[i] >= 0)
        y_a[prime_a[i]] -= 1;
      else
        y_b[bfree[i]] += 1;
    }
    st->phases += 1;
    if (st->phases <= free_cap && free_counts) free_counts[st->phases - 1] = n_i;
    st->sum_ni += n_i;
    if (st->phases > phase_cap) {
      status = ORC_INVARIANT;
      break;
    }
  }
  free(bfree);
  free(prime_a);
  free(claimed);
  if (status) return status;

  /* complete_matching: i-th free a with i-th free b, ascending. */
  int32_t ia = 0, ib = 0;
  for (;;) {
    while (ia < n_a && match_of_a[ia] != -1) ++ia;
    while (ib < n_b && match_of_b[ib] != -1) ++ib;
    if (ia >= n_a || ib >= n_b) break;
    match_of_a[ia] = ib;
    match_of_b[ib] = ia;
  }
  return ORC_OK;
}

/* matching_cost: src/core.cpp:95-102 (sequential sum, a ascending). */
double orc_matching_cost(int32_t n_a, int32_t n_b, const double* cost,
                         const int32_t* match_of_a) {
  double total = 0.0;
  for (int32_t a = 0; a < n_a; ++a) {
    const int32_t b = match_of_a[a];
    if (b != -1) total += cost[(size_t)a * n_b + b];
  }
  return total;
}

/* solve_assignment: src/assignment.cpp:368-400 (validation, orientation
 * swap when n_b > n_a; stats/duals stay in the swapped orientation,
 * assignment.hpp:41-43).  y_a must hold max(n_a,n_b) entries and y_b
 * min(n_a,n_b) entries (internal orientation). */
int orc_solve_assignment(int32_t n_a, int32_t n_b, const double* cost, double eps,
                         int32_t* match_of_a, int32_t* match_of_b, int64_t* y_a,
                         int64_t* y_b, int64_t* free_counts, int64_t free_cap,
                         orc_stats* st) {
  int s = orc_validate_costs(n_a, n_b, cost);
  if (s) return s;
  if (!(eps > 0.0 && eps < 1.0)) return ORC_PARAMETER;
  int32_t uf, uc;
  s = orc_units(eps, &uf, &uc);
  if (s) return s;

  const int swapped = n_b > n_a;
  const int32_t ia_n = swapped ? n_b : n_a; /* internal demand side */
  const int32_t ib_n = swapped ? n_a : n_b; /* internal supply side */
  int32_t* kT = (int32_t*)malloc(sizeof(int32_t) * (size_t)ia_n * ib_n);
  if (!kT) return ORC_INPUT;
  /* internal k(a,b): original cost(a,b) unswapped, cost(b,a) swapped. */
  for (int32_t a = 0; a < n_a; ++a)
    for (int32_t b = 0; b < n_b; ++b) {
      const int32_t kv = (int32_t)orc_scaled_floor(cost[(size_t)a * n_b + b], eps);
      if (!swapped)
        kT[(size_t)b * ia_n + a] = kv; /* internal (a,b) */
      else
        kT[(size_t)a * ia_n + b] = kv; /* internal (a'=b, b'=a) */
    }
  st->swapped = swapped;
  if (!swapped) {
    s = solve_oriented(ia_n, ib_n, kT, eps, match_of_a, match_of_b, y_a, y_b,
                       free_counts, free_cap, st);
  } else {
    /* internal match_of_a is original match_of_b and vice versa */
    s = solve_oriented(ia_n, ib_n, kT, eps, match_of_b, match_of_a, y_a, y_b,
                       free_counts, free_cap, st);
  }
  free(kT);
  if (s) return s;
  st->cost = orc_matching_cost(n_a, n_b, cost, match_of_a);
  return ORC_OK;
}

/* Same solve on a pre-rounded B-major k matrix (internal orientation,
 * n_a >= n_b is the caller's responsibility); used for large parity runs
 * where the dense double matrix is not materialised. */
int orc_solve_rounded(int32_t n_a, int32_t n_b, const int32_t* kT, double eps,
                      int32_t* match_of_a, int32_t* match_of_b, int64_t* y_a,
                      int64_t* y_b, int64_t* free_counts, int64_t free_cap,
                      orc_stats* st) {
  if (n_a < 1 || n_b < 1 || n_b > n_a) return ORC_PARAMETER;
  if (!(eps > 0.0 && eps < 1.0)) return ORC_PARAMETER;
  st->swapped = 0;
  st->cost = 0.0;
  return solve_oriented(n_a, n_b, kT, eps, match_of_a, match_of_b, y_a, y_b,
                        free_counts, free_cap, st);
}

/* FNV-1a 64 over raw little-endian bytes (the hash of SURVEY.md §8(c)). */
uint64_t orc_fnv1a64(const void* data, int64_t nbytes, uint64_t h) {
  const uint8_t* p = (const uint8_t*)data;
  for (int64_t i = 0; i < nbytes; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}
