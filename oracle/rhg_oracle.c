/*
 * rhg_oracle.c -- CPU ORACLE for the threshold random-hyperbolic-graph generator
 *                 of arXiv 1606.09481 (von Looz, Meyerhenke, Prutkin).
 *
 * *** TEST INFRASTRUCTURE ONLY. ***
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_1606_09481_b200/) never
 * links, imports or executes anything under oracle/, and this file shares no code,
 * header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct C (fp64, OpenMP only for outer loops that are
 * embarrassingly parallel).  Every function cites the passage it follows:
 *   PAPER.md:L (section / equation / algorithm line)  -- /root/reference/PAPER.md
 *   DESIGN.md "Reading Zk"                            -- where the paper is silent
 *
 * Parity status of each function is listed in DESIGN.md §10 ("Oracle pins"); every
 * exported function has a CPU test in tests/test_oracle.py that checks it against
 * something other than itself (brute force, 50/60-digit mpmath of the paper's
 * literal formulas, NVIDIA's Philox header, closed forms).
 */
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_API __attribute__((visibility("default")))

/* 2*pi as an unevaluated double-double sum (hi + lo), |error| < 1e-32.
 * Needed so that seam-crossing angle differences keep full relative precision
 * (DESIGN.md Reading Z13). */
static const double TWO_PI_HI = 6.283185307179586232;     /* fl(2*pi) */
static const double TWO_PI_LO = 2.4492935982947064e-16;  /* 2*pi - fl(2*pi) */

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11), the counter-based RNG named by the  */
/* north star.  Round function: two 32x32->64 multiplies, Weyl key schedule. */
/* Pinned against NVIDIA's curand_philox4x32_x.h compiled on the host        */
/* (tests/test_oracle_sampler.py).                                           */
/* ------------------------------------------------------------------------ */
ORC_API void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                               uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Words for vertices i0 .. i0+count-1: key = (seed_lo, seed_hi),
 * counter = (i_lo, i_hi, 0, 0)  (DESIGN.md Reading Z12). */
ORC_API void orc_philox_words(uint64_t seed, uint64_t i0, uint64_t count, uint32_t *out) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (uint64_t k = 0; k < count; ++k) {
    uint64_t i = i0 + k;
    uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(i >> 32), 0u, 0u};
    orc_philox4x32_10(ctr, key, out + 4 * k);
  }
}

/* ------------------------------------------------------------------------ */
/* Parameters.                                                              */
/* ------------------------------------------------------------------------ */

/* alpha = (gamma - 1)/2   (Alg. 1 line 1). */
ORC_API double orc_alpha(double gamma) { return (gamma - 1.0) / 2.0; }

/* Expected average degree approximation, Krioukov Eq. (22) as printed in
 * PAPER.md:178-182 with zeta = 1:
 *   xi   = (alpha/zeta) / (alpha/zeta - 1/2)
 *   kbar = 2/pi xi^2 n e^{-zeta R/2}
 *        + 2/pi xi^2 n ( e^{-alpha R} ( alpha R/2 ( pi/4 (zeta/alpha)^2
 *                                     - (pi-1) zeta/alpha + (pi-2) ) - 1 ) )
 * With zeta = 1 the "(zeta/alpha)^2 vs zeta/alpha^2" grouping question is moot
 * (DESIGN.md Reading Z4). */
ORC_API double orc_kbar_formula(double n, double alpha, double R) {
  const double zeta = 1.0;
  const double pi = M_PI;
  double xi = (alpha / zeta) / (alpha / zeta - 0.5);
  double pre = 2.0 / pi * xi * xi * n;
  double first = pre * exp(-zeta * R / 2.0);
  double inner = alpha * (R / 2.0) *
                     ((pi / 4.0) * (zeta / alpha) * (zeta / alpha) - (pi - 1.0) * (zeta / alpha) +
                      (pi - 2.0)) -
                 1.0;
  double second = pre * (exp(-alpha * R) * inner);
  return first + second;
}

/* getTargetRadius: "binary search with fixed n, alpha and
 * desired kbar".  Reading Z5: the formula rises from 0 at R=0 to a
 * single peak and then decreases; we search the decreasing branch.
 * Plain method: locate the peak on a 1e-4 grid over [0, 50], refine nothing,
 * then bisect on [R_peak, 10 ln n + 50] for 300 halvings (or until the bracket
 * is one ulp wide).  Returns 0 on success, 3 on calibration failure
 * (kbar above the formula's maximum or below its value at the far end),
 * 2 on invalid arguments (gamma <= 2, kbar <= 0, n < 2). */
ORC_API int orc_target_radius(double n, double kbar, double alpha, double *R_out) {
  if (!(n >= 2.0) || !(kbar > 0.0) || !(alpha > 0.5) || !isfinite(kbar) || !isfinite(n))
    return 2;
  double best_R = 0.0, best_k = -1.0;
  for (int i = 0; i <= 500000; ++i) {
    double R = i * 1e-4;
    double k = orc_kbar_formula(n, alpha, R);
    if (k > best_k) { best_k = k; best_R = R; }
  }
  double lo = best_R, hi = 10.0 * log(n) + 50.0;
  if (kbar > orc_kbar_formula(n, alpha, lo)) return 3;
  if (kbar < orc_kbar_formula(n, alpha, hi)) return 3;
  for (int it = 0; it < 300; ++it) {
    double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (orc_kbar_formula(n, alpha, mid) > kbar) lo = mid; else hi = mid;
  }
  *R_out = 0.5 * (lo + hi);
  return 0;
}

/* Radial slab boundaries (Eq. 4): c_0 = 0,
 * c_1 = (1-p) R / (1 - p^L), widths geometric with ratio p, c_L := R.
 * Used only to pin the SPEC example and the product's band table; the edge set
 * does not depend on (L, p). */
ORC_API void orc_boundaries(double R, int L, double p, double *c) {
  double c1 = (1.0 - p) * R / (1.0 - pow(p, (double)L));
  c[0] = 0.0;
  for (int k = 1; k < L; ++k) c[k] = c[k - 1] + c1 * pow(p, (double)(k - 1));
  c[L] = R;
}

/* ------------------------------------------------------------------------ */
/* Point sampling (Eq. 1; Alg. 1 lines 7-8). */
/* theta = 2 pi u1 in [0, 2pi)   (Reading Z10)                               */
/* r     = (2/alpha) asinh( sqrt( u2 (cosh(alpha R) - 1)/2 ) )  (Reading Z11): */
/*         the inverse of F(r) = (cosh(alpha r) - 1)/(cosh(alpha R) - 1),     */
/*         the CDF of Eq. 1, written with cosh x - 1 = 2 sinh^2(x/2).         */
/* u1 = (w1:w0 >> 11) 2^-53, u2 = (w3:w2 >> 11) 2^-53 (Reading Z12).         */
/* r is clamped to R (rounding could otherwise exceed the disk).             */
/* ------------------------------------------------------------------------ */
ORC_API void orc_uniforms(const uint32_t w[4], double *u1, double *u2) {
  uint64_t a = ((uint64_t)w[1] << 32) | w[0];
  uint64_t b = ((uint64_t)w[3] << 32) | w[2];
  *u1 = (double)(a >> 11) * 0x1.0p-53;
  *u2 = (double)(b >> 11) * 0x1.0p-53;
}

ORC_API double orc_radius_from_uniform(double u, double alpha, double R) {
  double half_span = (cosh(alpha * R) - 1.0) / 2.0;
  double r = (2.0 / alpha) * asinh(sqrt(u * half_span));
  return r > R ? R : r;
}

ORC_API void orc_sample_points(uint64_t n, double alpha, double R, uint64_t seed, double *theta,
                               double *r) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    uint32_t w[4];
    orc_philox_words(seed, (uint64_t)i, 1, w);
    double u1, u2;
    orc_uniforms(w, &u1, &u2);
    theta[i] = TWO_PI_HI * u1;
    r[i] = orc_radius_from_uniform(u2, alpha, R);
  }
}

/* ------------------------------------------------------------------------ */
/* The edge predicate.                                                      */
/* Plain definition (Eq. 3, Alg. 1 line 16):     */
/*   edge {p,q}  iff  dist(p,q) <= R, with                                  */
/*   cosh dist = cosh r_p cosh r_q - sinh r_p sinh r_q cos|phi_p - phi_q|.   */
/* Written out without cancellation (Reading Z2): since                      */
/*   cosh r_p cosh r_q - sinh r_p sinh r_q = cosh(r_p - r_q)  and             */
/*   1 - cos x = 2 sin^2(x/2),  cosh x - 1 = 2 sinh^2(x/2):                  */
/*   (cosh d - 1)/2 = sinh^2((r_p-r_q)/2) + sinh r_p sinh r_q sin^2(delta/2)  */
/*   (cosh R - 1)/2 = sinh^2(R/2)                                            */
/* so  edge iff  S := sinh^2((r_p-r_q)/2) + sinh r_p sinh r_q sin^2(delta/2)  */
/*              <= T := sinh^2(R/2).                                         */
/* delta = angular distance on the circle, min(|dphi|, 2pi - |dphi|).         */
/* ------------------------------------------------------------------------ */

/* Angular distance, seam-exact: (2pi - max) + min with 2pi as double-double. */
ORC_API double orc_angle_between(double t1, double t2) {
  double d = fabs(t1 - t2);
  if (d <= M_PI) return d;
  double mx = t1 > t2 ? t1 : t2, mn = t1 > t2 ? t2 : t1;
  return ((TWO_PI_HI - mx) + mn) + TWO_PI_LO;
}

/* S and T in fp64 (libm).  Relative error of S is a few ulp (all terms >= 0). */
ORC_API double orc_S(double t1, double r1, double t2, double r2) {
  double dr = sinh((r1 - r2) / 2.0);
  double sd = sin(orc_angle_between(t1, t2) / 2.0);
  return dr * dr + sinh(r1) * sinh(r2) * (sd * sd);
}

/* Same quantity in __float128 (113-bit) arithmetic: the near-tie arbiter. */
static __float128 orc_S_quad(double t1, double r1, double t2, double r2) {
  __float128 a1 = t1, a2 = t2, two_pi = 2 * M_PIq;
  __float128 d = fabsq(a1 - a2); /* exact: difference of two doubles in 113 bits */
  if (d > M_PIq) d = two_pi - d;
  __float128 dr = sinhq(((__float128)r1 - (__float128)r2) / 2);
  __float128 sd = sinq(d / 2);
  return dr * dr + sinhq((__float128)r1) * sinhq((__float128)r2) * (sd * sd);
}

/* Literal Eq. 3 evaluated in __float128: cosh d, to pin the rewriting above at
 * radii where 113 bits absorb the cancellation (R <~ 40). */
ORC_API double orc_cosh_dist_literal_quad(double t1, double r1, double t2, double r2,
                                          double *rel_err_bound) {
  __float128 a1 = t1, a2 = t2;
  __float128 c = coshq((__float128)r1) * coshq((__float128)r2) -
                 sinhq((__float128)r1) * sinhq((__float128)r2) * cosq(fabsq(a1 - a2));
  if (rel_err_bound) {
    __float128 scale = coshq((__float128)r1) * coshq((__float128)r2);
    *rel_err_bound = (double)(scale * 1e-32Q / (c > 1 ? c : 1));
  }
  return (double)c;
}

/* Threshold T = sinh^2(R/2) and the north-star tie window:
 * |cosh d - cosh R| <= 1e-12 cosh R  <=>  |S - T| <= 0.5e-12 cosh R. */
typedef struct {
  double R, T, tie_halfwidth;
} orc_thresh;

static orc_thresh orc_make_thresh(double R) {
  orc_thresh t;
  double h = sinh(R / 2.0);
  t.R = R;
  t.T = h * h;
  /* window + a 1e-14 T margin covering the fp64 error of S (a few ulp). */
  t.tie_halfwidth = 0.5e-12 * cosh(R) + 1e-14 * t.T;
  return t;
}

/* Decide one pair. Returns 1 for an edge. *tie = 1 when the pair lies in the
 * north-star ambiguity window; then the decision is made in __float128. */
static int orc_decide(const orc_thresh *th, double t1, double r1, double t2, double r2, int *tie) {
  double S = orc_S(t1, r1, t2, r2);
  if (fabs(S - th->T) <= th->tie_halfwidth) {
    *tie = 1;
    __float128 h = sinhq((__float128)th->R / 2);
    return orc_S_quad(t1, r1, t2, r2) <= h * h;
  }
  *tie = 0;
  return S <= th->T;
}

ORC_API int orc_is_edge(double t1, double r1, double t2, double r2, double R, int *tie) {
  orc_thresh th = orc_make_thresh(R);
  int tt = 0;
  int e = orc_decide(&th, t1, r1, t2, r2, &tt);
  if (tie) *tie = tt;
  return e;
}

/* ------------------------------------------------------------------------ */
/* Edge-set oracles.  Output: undirected pairs (u, v), u < v, as uint32, in  */
/* lexicographic order; plus the list of near-tie pairs (same format) with   */
/* their quad decision.  Return value = edge count, or -1 if cap exceeded     */
/* (then *needed holds the count).                                          */
/* ------------------------------------------------------------------------ */

static int cmp_u64(const void *a, const void *b) {
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return x < y ? -1 : (x > y);
}

/* (1) Brute force over all n(n-1)/2 pairs: the plain definition
 *     E = {{u,v} : u != v, dist <= R}  (the Theta(n^2)
 *     pairwise probing of Aldecoa et al. restricted to T = 0). */
ORC_API int64_t orc_brute_force(uint64_t n, const double *theta, const double *r, double R,
                                uint32_t *pairs, uint64_t cap, uint32_t *ties, uint8_t *tie_edge,
                                uint64_t tie_cap, uint64_t *n_ties, uint64_t *needed) {
  orc_thresh th = orc_make_thresh(R);
  uint64_t *cnt = calloc(n + 1, sizeof(uint64_t));
  uint64_t *tcnt = calloc(n + 1, sizeof(uint64_t));
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    uint64_t c = 0, tc = 0;
    for (uint64_t j = (uint64_t)i + 1; j < n; ++j) {
      int tie = 0;
      c += orc_decide(&th, theta[i], r[i], theta[j], r[j], &tie);
      tc += tie;
    }
    cnt[i + 1] = c;
    tcnt[i + 1] = tc;
  }
  for (uint64_t i = 0; i < n; ++i) {
    cnt[i + 1] += cnt[i];
    tcnt[i + 1] += tcnt[i];
  }
  uint64_t m = cnt[n];
  *needed = m;
  *n_ties = tcnt[n];
  if (m > cap || tcnt[n] > tie_cap) {
    free(cnt);
    free(tcnt);
    return -1;
  }
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    uint64_t o = cnt[i], to = tcnt[i];
    for (uint64_t j = (uint64_t)i + 1; j < n; ++j) {
      int tie = 0;
      int e = orc_decide(&th, theta[i], r[i], theta[j], r[j], &tie);
      if (e) {
        pairs[2 * o] = (uint32_t)i;
        pairs[2 * o + 1] = (uint32_t)j;
        ++o;
      }
      if (tie) {
        ties[2 * to] = (uint32_t)i;
        ties[2 * to + 1] = (uint32_t)j;
        tie_edge[to] = (uint8_t)e;
        ++to;
      }
    }
  }
  free(cnt);
  free(tcnt);
  return (int64_t)m;
}

/* Half-width of the angular window of a point at radius r against partners at
 * radius >= c (Eqs. 6-9), written stably (Reading Z3):
 *   sin^2(dphi/2) <= (T - sinh^2((r-c)/2)) / (sinh r sinh c);
 * full circle (returns pi) when the ratio >= 1 or sinh r sinh c == 0. */
ORC_API double orc_window(double r, double c, double R) {
  double h = sinh(R / 2.0), T = h * h;
  double d = sinh((r - c) / 2.0);
  double den = sinh(r) * sinh(c);
  double num = T - d * d;
  if (den <= 0.0 || num >= den) return M_PI;
  if (num <= 0.0) return 0.0;
  return 2.0 * asin(sqrt(num / den));
}

typedef struct {
  double theta;
  uint32_t id;
} orc_ang;

static int cmp_ang(const void *a, const void *b) {
  const orc_ang *x = a, *y = b;
  if (x->theta < y->theta) return -1;
  if (x->theta > y->theta) return 1;
  return x->id < y->id ? -1 : (x->id > y->id);
}

/* (2) Radius-ordered angular sweep.
 * Each edge {v,w} is found from its endpoint with the smaller (r, id).  A
 * partner w with r_w >= r_v satisfies delta <= window(r_v, r_w) <= window(r_v, r_v)
 * because the window decreases in its second argument (proof in DESIGN.md,
 * "Window monotonicity").  So scanning the theta-sorted circle within
 * +-window(r_v, r_v) (padded) from v finds every such partner.  Each candidate
 * is decided by the same orc_decide as the brute force. */
ORC_API int64_t orc_sweep(uint64_t n, const double *theta, const double *r, double R,
                          uint32_t *pairs, uint64_t cap, uint32_t *ties, uint8_t *tie_edge,
                          uint64_t tie_cap, uint64_t *n_ties, uint64_t *needed) {
  orc_thresh th = orc_make_thresh(R);
  orc_ang *s = malloc(n * sizeof(orc_ang));
  for (uint64_t i = 0; i < n; ++i) {
    s[i].theta = theta[i];
    s[i].id = (uint32_t)i;
  }
  qsort(s, n, sizeof(orc_ang), cmp_ang);
  uint64_t *pos = malloc(n * sizeof(uint64_t));
  for (uint64_t k = 0; k < n; ++k) pos[s[k].id] = k;

  /* two passes: count, then fill (pairs are collected unsorted, sorted at end) */
  uint64_t *cnt = calloc(n + 1, sizeof(uint64_t));
  uint64_t *tcnt = calloc(n + 1, sizeof(uint64_t));
  for (int pass = 0; pass < 2; ++pass) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t v = 0; v < (int64_t)n; ++v) {
      double rv = r[v];
      double w = orc_window(rv, rv, R);
      double wpad = w * (1.0 + 1e-9) + 1e-12;
      int full = wpad >= M_PI; /* window covers the whole circle */
      uint64_t o = pass ? cnt[v] : 0, to = pass ? tcnt[v] : 0;
      uint64_t c = 0, tc = 0;
      uint64_t p = pos[v];
      /* walk forward (increasing theta) then backward around the circle while
       * the circular distance stays within the window; with wpad < pi the two
       * walks cannot meet (their arcs sum to < 2 pi).  A full-circle window is
       * covered by the forward walk alone. */
      for (int dir = 0; dir < (full ? 1 : 2); ++dir) {
        for (uint64_t step = 1; step < n; ++step) {
          uint64_t k = dir == 0 ? (p + step) % n : (p + n - step) % n;
          const orc_ang *q = &s[k];
          if (!full && orc_angle_between(theta[v], q->theta) > wpad) break;
          uint32_t u = q->id;
          if (u == (uint32_t)v) break;
          /* partner must have larger (r, id) */
          if (r[u] < rv || (r[u] == rv && u < (uint32_t)v)) continue;
          int tie = 0;
          int e = orc_decide(&th, theta[v], rv, q->theta, r[u], &tie);
          if (pass == 0) {
            c += e;
            tc += tie;
          } else {
            if (e) {
              uint32_t a = (uint32_t)v < u ? (uint32_t)v : u, b = (uint32_t)v < u ? u : (uint32_t)v;
              pairs[2 * o] = a;
              pairs[2 * o + 1] = b;
              ++o;
            }
            if (tie) {
              uint32_t a = (uint32_t)v < u ? (uint32_t)v : u, b = (uint32_t)v < u ? u : (uint32_t)v;
              ties[2 * to] = a;
              ties[2 * to + 1] = b;
              tie_edge[to] = (uint8_t)e;
              ++to;
            }
          }
        }
      }
      if (pass == 0) {
        cnt[v + 1] = c;
        tcnt[v + 1] = tc;
      }
    }
    if (pass == 0) {
      for (uint64_t i = 0; i < n; ++i) {
        cnt[i + 1] += cnt[i];
        tcnt[i + 1] += tcnt[i];
      }
      *needed = cnt[n];
      *n_ties = tcnt[n];
      if (cnt[n] > cap || tcnt[n] > tie_cap) {
        free(cnt); free(tcnt); free(s); free(pos);
        return -1;
      }
    }
  }
  uint64_t m = cnt[n];
  free(cnt);
  free(tcnt);
  free(s);
  free(pos);
  /* canonical order: sort pairs lexicographically */
  uint64_t *keys = malloc((m ? m : 1) * sizeof(uint64_t));
  for (uint64_t e = 0; e < m; ++e) keys[e] = ((uint64_t)pairs[2 * e] << 32) | pairs[2 * e + 1];
  qsort(keys, m, sizeof(uint64_t), cmp_u64);
  for (uint64_t e = 0; e < m; ++e) {
    pairs[2 * e] = (uint32_t)(keys[e] >> 32);
    pairs[2 * e + 1] = (uint32_t)keys[e];
  }
  free(keys);
  return (int64_t)m;
}

/* (2b) Count-only sweep over the vertices with id in [id_lo, id_hi): edges whose
 * smaller-(r, id) endpoint lies in the range (same search and decision as (2)).
 * Used for the bounded CPU baseline timing; *tests receives the number of
 * candidate pairs decided. */
ORC_API int64_t orc_sweep_count(uint64_t n, const double *theta, const double *r, double R,
                                uint64_t id_lo, uint64_t id_hi, uint64_t *tests) {
  orc_thresh th = orc_make_thresh(R);
  orc_ang *s = malloc(n * sizeof(orc_ang));
  for (uint64_t i = 0; i < n; ++i) {
    s[i].theta = theta[i];
    s[i].id = (uint32_t)i;
  }
  qsort(s, n, sizeof(orc_ang), cmp_ang);
  uint64_t *pos = malloc(n * sizeof(uint64_t));
  for (uint64_t k = 0; k < n; ++k) pos[s[k].id] = k;
  uint64_t m = 0, t = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : m, t)
  for (int64_t v = (int64_t)id_lo; v < (int64_t)id_hi; ++v) {
    double rv = r[v];
    double wpad = orc_window(rv, rv, R) * (1.0 + 1e-9) + 1e-12;
    int full = wpad >= M_PI;
    uint64_t p = pos[v];
    for (int dir = 0; dir < (full ? 1 : 2); ++dir) {
      for (uint64_t step = 1; step < n; ++step) {
        uint64_t k = dir == 0 ? (p + step) % n : (p + n - step) % n;
        const orc_ang *q = &s[k];
        if (!full && orc_angle_between(theta[v], q->theta) > wpad) break;
        uint32_t u = q->id;
        if (u == (uint32_t)v) break;
        if (r[u] < rv || (r[u] == rv && u < (uint32_t)v)) continue;
        int tie = 0;
        m += orc_decide(&th, theta[v], rv, q->theta, r[u], &tie);
        ++t;
      }
    }
  }
  free(s);
  free(pos);
  if (tests) *tests = t;
  return (int64_t)m;
}

/* ------------------------------------------------------------------------ */
/* (2c) The sweep of (2), split into its two steps so that they can be timed  */
/* and reused: the angular order of all points (one qsort by (theta, id)),    */
/* then per owner vertex v the scan of +-window(r_v, r_v) (padded) over the   */
/* circle, testing partners with larger (r, id) -- exactly the search and     */
/* decision of (2).  Positions are uint32 (n < 2^32).                         */
/* ------------------------------------------------------------------------ */
ORC_API void orc_angle_order(uint64_t n, const double *theta, uint32_t *order, uint32_t *pos) {
  orc_ang *s = malloc((n ? n : 1) * sizeof(orc_ang));
  for (uint64_t i = 0; i < n; ++i) {
    s[i].theta = theta[i];
    s[i].id = (uint32_t)i;
  }
  qsort(s, n, sizeof(orc_ang), cmp_ang);
  for (uint64_t k = 0; k < n; ++k) {
    order[k] = s[k].id;
    pos[s[k].id] = (uint32_t)k;
  }
  free(s);
}

enum { SW_COUNT = 0, SW_DEG = 1, SW_FILL = 2, SW_DIGEST = 3 };

typedef struct {
  uint64_t n;
  const double *theta, *r;
  const uint32_t *order, *pos;
  orc_thresh th;
  /* outputs, by mode */
  uint64_t *deg;     /* SW_DEG: degree (both endpoints) */
  uint64_t *cursor;  /* SW_FILL: next free slot of each row */
  uint32_t *col;     /* SW_FILL */
  uint64_t *dig;     /* SW_DIGEST: sum of orc_mix64(neighbour id) */
  uint32_t *ties;    /* SW_DEG / SW_DIGEST: near-tie pairs (u < v) */
  uint8_t *tie_edge;
  uint64_t tie_cap, *n_ties;
} sweep_ctx;

/* Order-independent digest of a neighbour set: sum over w of mix(w) mod 2^64,
 * mix = the SplitMix64 finaliser of w.  Test infrastructure (a checksum of the
 * output, not part of the method). */
ORC_API uint64_t orc_mix64(uint64_t w) {
  uint64_t z = w * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* Scan owner v; returns its edges, adds its tests to *tests. */
static uint64_t sweep_one(const sweep_ctx *cx, uint64_t v, int mode, uint64_t *tests) {
  const double rv = cx->r[v], tv = cx->theta[v];
  const double wpad = orc_window(rv, rv, cx->th.R) * (1.0 + 1e-9) + 1e-12;
  const int full = wpad >= M_PI;
  const uint64_t n = cx->n, p = cx->pos[v];
  uint64_t m = 0, t = 0;
  for (int dir = 0; dir < (full ? 1 : 2); ++dir) {
    for (uint64_t step = 1; step < n; ++step) {
      const uint64_t k = dir == 0 ? (p + step) % n : (p + n - step) % n;
      const uint32_t u = cx->order[k];
      if (!full && orc_angle_between(tv, cx->theta[u]) > wpad) break;
      if (u == (uint32_t)v) break;
      if (cx->r[u] < rv || (cx->r[u] == rv && u < (uint32_t)v)) continue;
      int tie = 0;
      const int e = orc_decide(&cx->th, tv, rv, cx->theta[u], cx->r[u], &tie);
      ++t;
      m += e;
      if (tie && (mode == SW_DEG || mode == SW_DIGEST)) {
        uint64_t slot;
#pragma omp atomic capture
        slot = (*cx->n_ties)++;
        if (slot < cx->tie_cap) {
          cx->ties[2 * slot] = (uint32_t)v < u ? (uint32_t)v : u;
          cx->ties[2 * slot + 1] = (uint32_t)v < u ? u : (uint32_t)v;
          cx->tie_edge[slot] = (uint8_t)e;
        }
      }
      if (!e) continue;
      if (mode == SW_DEG || mode == SW_DIGEST) {
#pragma omp atomic
        cx->deg[v] += 1;
#pragma omp atomic
        cx->deg[u] += 1;
      }
      if (mode == SW_DIGEST) {
        const uint64_t a = orc_mix64(u), b = orc_mix64(v);
#pragma omp atomic
        cx->dig[v] += a;
#pragma omp atomic
        cx->dig[u] += b;
      }
      if (mode == SW_FILL) {
        uint64_t sv, su;
#pragma omp atomic capture
        sv = cx->cursor[v]++;
#pragma omp atomic capture
        su = cx->cursor[u]++;
        cx->col[sv] = u;
        cx->col[su] = (uint32_t)v;
      }
    }
  }
  *tests += t;
  return m;
}

static sweep_ctx sweep_setup(uint64_t n, const double *theta, const double *r, double R,
                             const uint32_t *order, const uint32_t *pos) {
  sweep_ctx cx;
  memset(&cx, 0, sizeof(cx));
  cx.n = n;
  cx.theta = theta;
  cx.r = r;
  cx.order = order;
  cx.pos = pos;
  cx.th = orc_make_thresh(R);
  return cx;
}

/* Count-only sweep over the owners with id in [id_lo, id_hi), on a given angular
 * order (orc_angle_order).  Same search and decision as (2); *tests = candidate
 * pairs decided.  Used to time the oracle with its sort step separated. */
ORC_API int64_t orc_sweep_count_ordered(uint64_t n, const double *theta, const double *r, double R,
                                        const uint32_t *order, const uint32_t *pos, uint64_t id_lo,
                                        uint64_t id_hi, uint64_t *tests) {
  sweep_ctx cx = sweep_setup(n, theta, r, R, order, pos);
  uint64_t m = 0, t = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : m, t)
  for (int64_t v = (int64_t)id_lo; v < (int64_t)id_hi; ++v) m += sweep_one(&cx, (uint64_t)v, SW_COUNT, &t);
  if (tests) *tests = t;
  return (int64_t)m;
}

static int cmp_u32(const void *a, const void *b) {
  uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
  return x < y ? -1 : (x > y);
}

/* (2d) The sweep's edge set as a CSR: both directions, no self-loops, every row
 * in ascending id order (the same set as (2); the CSR of SURVEY.md §8(a) output
 * semantics, rows canonicalised).  Pass 1 counts degrees (and collects the
 * near-tie pairs), pass 2 fills the rows, then each row is sorted.  Returns the
 * directed entry count, or -1 if it exceeds cap (*needed = the count). */
ORC_API int64_t orc_sweep_csr(uint64_t n, const double *theta, const double *r, double R,
                              uint64_t *row_ptr, uint32_t *col, uint64_t cap, uint32_t *ties,
                              uint8_t *tie_edge, uint64_t tie_cap, uint64_t *n_ties,
                              uint64_t *needed) {
  uint32_t *order = malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t *pos = malloc((n ? n : 1) * sizeof(uint32_t));
  orc_angle_order(n, theta, order, pos);
  sweep_ctx cx = sweep_setup(n, theta, r, R, order, pos);
  uint64_t *deg = calloc(n ? n : 1, sizeof(uint64_t));
  uint64_t nt = 0, t = 0;
  cx.deg = deg;
  cx.ties = ties;
  cx.tie_edge = tie_edge;
  cx.tie_cap = tie_cap;
  cx.n_ties = &nt;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : t)
  for (int64_t v = 0; v < (int64_t)n; ++v) sweep_one(&cx, (uint64_t)v, SW_DEG, &t);
  row_ptr[0] = 0;
  for (uint64_t i = 0; i < n; ++i) row_ptr[i + 1] = row_ptr[i] + deg[i];
  *needed = row_ptr[n];
  *n_ties = nt;
  if (row_ptr[n] > cap || nt > tie_cap) {
    free(order); free(pos); free(deg);
    return -1;
  }
  memcpy(deg, row_ptr, n * sizeof(uint64_t)); /* deg becomes the fill cursor */
  cx.cursor = deg;
  cx.col = col;
  t = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : t)
  for (int64_t v = 0; v < (int64_t)n; ++v) sweep_one(&cx, (uint64_t)v, SW_FILL, &t);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < (int64_t)n; ++v)
    qsort(col + row_ptr[v], row_ptr[v + 1] - row_ptr[v], sizeof(uint32_t), cmp_u32);
  free(order); free(pos); free(deg);
  return (int64_t)row_ptr[n];
}

/* (2e) Per-vertex degree and neighbour-set digest (orc_mix64 sum) of the sweep's
 * edge set, in one pass: a full-graph comparison at sizes where the edge list
 * itself is not materialised on the host (n = 1e8).  Near-tie pairs collected as
 * in (2d).  Returns the undirected edge count. */
ORC_API int64_t orc_sweep_digest(uint64_t n, const double *theta, const double *r, double R,
                                 uint64_t *deg, uint64_t *dig, uint32_t *ties, uint8_t *tie_edge,
                                 uint64_t tie_cap, uint64_t *n_ties) {
  uint32_t *order = malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t *pos = malloc((n ? n : 1) * sizeof(uint32_t));
  orc_angle_order(n, theta, order, pos);
  sweep_ctx cx = sweep_setup(n, theta, r, R, order, pos);
  memset(deg, 0, n * sizeof(uint64_t));
  memset(dig, 0, n * sizeof(uint64_t));
  uint64_t nt = 0, t = 0, m = 0;
  cx.deg = deg;
  cx.dig = dig;
  cx.ties = ties;
  cx.tie_edge = tie_edge;
  cx.tie_cap = tie_cap;
  cx.n_ties = &nt;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : t, m)
  for (int64_t v = 0; v < (int64_t)n; ++v) m += sweep_one(&cx, (uint64_t)v, SW_DIGEST, &t);
  *n_ties = nt;
  free(order); free(pos);
  return (int64_t)m;
}

/* (3) Neighbourhoods of selected vertices by brute force over all n points
 * (for configurations too large for (1)/(2) in test time).  Writes, for each
 * query k, its neighbour ids (ascending) into nbr[off[k] .. off[k+1]) and
 * returns the total; off must hold nq+1 entries.  Two passes (count, fill).
 * n_tie[k] counts near-tie pairs of query k. */
ORC_API int64_t orc_rows(uint64_t n, const double *theta, const double *r, double R,
                         uint64_t nq, const uint32_t *query, uint64_t *off, uint32_t *nbr,
                         uint64_t cap, uint32_t *n_tie) {
  orc_thresh th = orc_make_thresh(R);
  off[0] = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t k = 0; k < (int64_t)nq; ++k) {
    uint32_t v = query[k];
    uint64_t c = 0;
    uint32_t tc = 0;
    for (uint64_t w = 0; w < n; ++w) {
      if (w == v) continue;
      int tie = 0;
      c += orc_decide(&th, theta[v], r[v], theta[w], r[w], &tie);
      tc += tie;
    }
    off[k + 1] = c;
    n_tie[k] = tc;
  }
  for (uint64_t k = 0; k < nq; ++k) off[k + 1] += off[k];
  if (off[nq] > cap) return -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t k = 0; k < (int64_t)nq; ++k) {
    uint32_t v = query[k];
    uint64_t o = off[k];
    for (uint64_t w = 0; w < n; ++w) {
      if (w == v) continue;
      int tie = 0;
      if (orc_decide(&th, theta[v], r[v], theta[w], r[w], &tie)) nbr[o++] = (uint32_t)w;
    }
  }
  return (int64_t)off[nq];
}

/* Near-tie pairs of selected vertices: ids w with the pair (v, w) in the
 * ambiguity window, and the quad decision.  Used to excuse disagreements. */
ORC_API int64_t orc_row_ties(uint64_t n, const double *theta, const double *r, double R, uint32_t v,
                             uint32_t *w_out, uint8_t *e_out, uint64_t cap) {
  orc_thresh th = orc_make_thresh(R);
  uint64_t c = 0;
  for (uint64_t w = 0; w < n; ++w) {
    if (w == v) continue;
    int tie = 0;
    int e = orc_decide(&th, theta[v], r[v], theta[w], r[w], &tie);
    if (tie) {
      if (c < cap) {
        w_out[c] = (uint32_t)w;
        e_out[c] = (uint8_t)e;
      }
      ++c;
    }
  }
  return (int64_t)c;
}

/* ------------------------------------------------------------------------ */
/* Radius parametrisation: "accept the commonly used      */
/* parameter C, with R = 2 ln n + C".                                        */
/* ------------------------------------------------------------------------ */
ORC_API double orc_radius_from_C(double n, double C) { return 2.0 * log(n) + C; }

/* ------------------------------------------------------------------------ */
/* Dynamic model (Sec. 3.3).                              */
/* Step values tau_phi, tau_r per vertex; Appendix B draws    */
/* them uniformly from (-1, 1) and (-10, 1).  Reading     */
/* D1: they come from Philox(key = seed, ctr = (i_lo, i_hi, 1,   */
/* 0)), u1 -> tau_phi, u2 -> tau_r, mapped affinely onto [lo, hi).            */
/* ------------------------------------------------------------------------ */
ORC_API void orc_movement_init(uint64_t n, uint64_t seed, double phi_lo, double phi_hi, double r_lo,
                               double r_hi, double *tau_phi, double *tau_r) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    const uint32_t ctr[4] = {(uint32_t)i, (uint32_t)((uint64_t)i >> 32), 1u, 0u};
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t w[4];
    orc_philox4x32_10(ctr, key, w);
    double u1, u2;
    orc_uniforms(w, &u1, &u2);
    tau_phi[i] = phi_lo + (phi_hi - phi_lo) * u1;
    tau_r[i] = r_lo + (r_hi - r_lo) * u2;
  }
}

/* Rotation step: rotated(phi, r, tau_phi) = (phi + tau_phi) mod 2pi,
 * for |tau_phi| < 2pi: one add, then one wrap by fl(2pi); the result is kept in
 * [0, fl(2pi)) (Reading Z10). */
ORC_API double orc_rotate(double phi, double tau_phi) {
  double s = phi + tau_phi;
  if (s >= TWO_PI_HI) s -= TWO_PI_HI;
  else if (s < 0.0) s += TWO_PI_HI;
  if (s >= TWO_PI_HI || s < 0.0) s = 0.0;  /* rounding at the seam */
  return s;
}

/* Radial step, Algorithm 2: x = sinh(r alpha), y = x + tau_r,
 * z = asinh(y)/alpha.  Reflection: "if the new node position would
 * be outside the boundary (r > R) or below the origin (r < 0), the movement is
 * reflected and tau_r set to -tau_r".  Reading D2: reflect in the
 * transformed coordinate y at 0 and at S = sinh(alpha R), once per crossing, and
 * flip tau_r once per reflection. */
ORC_API void orc_radial_step(double r, double tau_r, double R, double alpha, double *r_out,
                             double *tau_out) {
  const double S = sinh(alpha * R);
  double y = sinh(r * alpha) + tau_r;
  double t = tau_r;
  for (int it = 0; it < 64 && (y < 0.0 || y > S); ++it) {
    if (y < 0.0) y = -y;
    else y = 2.0 * S - y;
    t = -t;
  }
  if (y < 0.0) y = 0.0;
  if (y > S) y = S;
  double z = asinh(y) / alpha;
  *r_out = z > R ? R : z;
  *tau_out = t;
}

/* One movement step of every vertex, in place. */
ORC_API void orc_move_points(uint64_t n, double *theta, double *r, const double *tau_phi,
                             double *tau_r, double R, double alpha) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    theta[i] = orc_rotate(theta[i], tau_phi[i]);
    orc_radial_step(r[i], tau_r[i], R, alpha, &r[i], &tau_r[i]);
  }
}

ORC_API int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
