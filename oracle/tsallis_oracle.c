/*
 * oracle/tsallis_oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * Tsallis multilevel-thresholding hot path of arXiv 2012.10684.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or constant with the CUDA path
 * (paper_2012_10684_b200/csrc) and neither side includes the other.
 *
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -shared -fPIC
 * (no FMA contraction, no re-association: every sum below is the sequential
 * ascending sum it is written as -- DESIGN.md reading R9).
 *
 * What it computes, per slice (PAPER.md line numbers refer to the v2 text,
 * lines 367-807 of /root/reference/PAPER.md):
 *
 *   1. histogram c_i = #{voxels with value i}                 PAPER.md:456-462 (Fig. hist, 1-D
 *      brightness histogram; "first dimension" :564).  Any voxel >= L is a
 *      LEVEL_OVERFLOW for the slice (never clamped; R13).
 *   2. p_i = c_i / N, N = sum of c                            PAPER.md:579 (set P, sum p = 1)
 *   3. per class C = [a,b]:  P = sum_{i=a..b} p_i             PAPER.md:587-591 (class mass)
 *        q != 1:  S = (1 - sum_{i=a..b} (p_i/P)^q) / (q - 1)  PAPER.md:581-585 (H^alpha_1, H^alpha_2;
 *                 summand read as p_i/P_j -- DESIGN.md R3; 0^q = 0)
 *        q == 1:  S = -sum (p_i/P) ln(p_i/P), 0 ln 0 = 0      Shannon limit (R6)
 *      P == 0  => the class is empty and the tuple is skipped (R5).
 *   4. classes of a tuple t_1 < ... < t_k, t_j in [0, L-2]:
 *        C_0 = [0, t_1], C_j = [t_j + 1, t_{j+1}], C_k = [t_k + 1, L-1]
 *      (t_j is the last bin of the lower class; PAPER.md:582,:588 -- DESIGN.md R4)
 *   5. objective (R1):
 *        PSEUDO_ADDITIVE (default): phi = S_0; for j = 1..k: phi = phi + S_j + (1-q) phi S_j
 *          -- PAPER.md:593-596 (H1 + H2 + (1-alpha) H1 H2) applied left to right
 *        SUM_PLUS_PRODUCT: phi = (S_0 + ... + S_k) + (1-q) (S_0 * ... * S_k)
 *   6. argmax over all tuples in lexicographic order, replacing the best only on
 *      a strictly greater phi, so the lowest tuple wins ties  (PAPER.md:594,:597
 *      "Arg max"; tie rule DESIGN.md R8).  No valid tuple => NO_VALID_SPLIT.
 *      Runner-up: best phi over canonical tuples (every t_j a non-empty bin,
 *      i.e. distinct partitions) other than t*;  gap = (phi* - phi2)/|phi*|.
 *   7. labels: label(v) = #{ j : v > t_j }   -- Algorithm 1 (PAPER.md:464-477,
 *      ">= T -> 1") with T = t + 1 for k = 1, generalised to k thresholds (R4).
 *
 * Level 0 recomputes every class sum from the definition for every tuple.
 * Level 1 memoises S per distinct class content, keyed by (first non-empty bin
 * >= a, last non-empty bin <= b).  Because every term is >= 0 and adding +0.0
 * is exact, the sums over [a,b] and over that key range are the same sequence
 * of non-zero additions, so Level 1 is bit-identical to Level 0 (tested).
 *
 * Pins (tests/test_oracle_*.py): numpy.bincount; closed forms for uniform
 * histograms (mpmath); exact rationals at q = 2 (fractions); Kapur-Sahoo-Wong
 * closed form at q = 1; point masses; gap phantoms; mirror symmetry; scale
 * invariance; log-domain DP; Level 0 = Level 1 bit-exactly.
 *
 * SURVEY.md §8(f) sections at the end of this file, each with its own pins:
 *   2-D Tsallis (oracle_mean3x3, oracle_hist2d, oracle_phi2d_at,
 *     oracle_search2d_n): numpy 3x3 mean / bincount, 50-digit brute force,
 *     diagonal 2-D = 1-D, point masses, transpose symmetry, the distinct-
 *     partition gap against explicit cell sets     (tests/test_oracle_2d.py)
 *   pre-processing (oracle_preprocess): the SPEC worked example, an
 *     independent float formula, exact half ties, invariants
 *                                                  (tests/test_oracle_preprocess.py)
 *   morphology (oracle_erode / _dilate / _tophat): numpy padded shifts,
 *     disk sizes, duality, idempotence, anti-extensivity, monotonicity
 *                                                  (tests/test_oracle_morph.py)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_LEVEL_OVERFLOW 2
#define OR_NO_VALID_SPLIT 3
#define OR_INVALID_ARG 1

#define OR_OBJ_PSEUDO_ADDITIVE 0
#define OR_OBJ_SUM_PLUS_PRODUCT 1

#define OR_KMAX 4

/* ---------------------------------------------------------------- step 1 */
/* Histogram of one slice.  dtype_bytes 1 = u8, 2 = u16.
 * Returns OR_LEVEL_OVERFLOW if any voxel >= bins (those voxels are not counted). */
int oracle_histogram(const void *slice, int dtype_bytes, int64_t n, int bins,
                     uint32_t *hist) {
  int status = OR_OK;
  for (int i = 0; i < bins; i++) hist[i] = 0;
  for (int64_t x = 0; x < n; x++) {
    unsigned v = dtype_bytes == 1 ? ((const uint8_t *)slice)[x]
                                  : ((const uint16_t *)slice)[x];
    if (v >= (unsigned)bins) {
      status = OR_LEVEL_OVERFLOW;
      continue;
    }
    hist[v] += 1;
  }
  return status;
}

/* ---------------------------------------------------------------- step 2 */
static void probabilities(const uint32_t *hist, int bins, double *p) {
  double N = 0.0;
  for (int i = 0; i < bins; i++) N += (double)hist[i]; /* exact: N < 2^53 */
  for (int i = 0; i < bins; i++) p[i] = (double)hist[i] / N;
}

/* ---------------------------------------------------------------- step 3 */
/* Tsallis entropy of the class [a,b] (class mass :587-591).
 * *valid = 0 when the class mass P is zero (empty class). */
double oracle_class_entropy(const double *p, int a, int b, double q, int *valid) {
  double P = 0.0;
  for (int i = a; i <= b; i++) P = P + p[i];
  if (P == 0.0) {
    *valid = 0;
    return 0.0;
  }
  *valid = 1;
  if (q == 1.0) {
    double H = 0.0;
    for (int i = a; i <= b; i++) {
      if (p[i] > 0.0) {
        double r = p[i] / P;
        H = H - r * log(r);
      }
    }
    return H;
  }
  double A = 0.0;
  for (int i = a; i <= b; i++) {
    if (p[i] > 0.0) A = A + pow(p[i] / P, q); /* 0^q = 0 */
  }
  return (1.0 - A) / (q - 1.0);
}

/* ---------------------------------------------------------------- step 5 */
static double combine(const double *S, int nclass, double q, int objective) {
  if (objective == OR_OBJ_SUM_PLUS_PRODUCT) {
    double sum = 0.0, prod = 1.0;
    for (int j = 0; j < nclass; j++) sum = sum + S[j];
    for (int j = 0; j < nclass; j++) prod = prod * S[j];
    return sum + (1.0 - q) * prod;
  }
  double phi = S[0];
  for (int j = 1; j < nclass; j++) phi = phi + S[j] + (1.0 - q) * phi * S[j];
  return phi;
}

/* class bounds of tuple t (step 4) */
static void class_bounds(const int *t, int k, int bins, int *lo, int *hi) {
  lo[0] = 0;
  for (int j = 0; j < k; j++) {
    hi[j] = t[j];
    lo[j + 1] = t[j] + 1;
  }
  hi[k] = bins - 1;
}

/* Objective at one tuple, straight from the definition (Level 0).  *valid = 0
 * when some class is empty or the tuple is not strictly increasing in
 * [0, bins-2]. */
double oracle_phi_at(const uint32_t *hist, int bins, int k, double q,
                     int objective, const int *t, int *valid) {
  *valid = 0;
  if (k < 1 || k > OR_KMAX) return NAN;
  for (int j = 0; j < k; j++) {
    if (t[j] < 0 || t[j] > bins - 2) return NAN;
    if (j > 0 && t[j] <= t[j - 1]) return NAN;
  }
  double *p = (double *)malloc(sizeof(double) * bins);
  probabilities(hist, bins, p);
  int lo[OR_KMAX + 1], hi[OR_KMAX + 1];
  double S[OR_KMAX + 1];
  class_bounds(t, k, bins, lo, hi);
  for (int j = 0; j <= k; j++) {
    int v;
    S[j] = oracle_class_entropy(p, lo[j], hi[j], q, &v);
    if (!v) {
      free(p);
      return NAN;
    }
  }
  free(p);
  *valid = 1;
  return combine(S, k + 1, q, objective);
}

/* ---------------------------------------------------------------- step 6 */
typedef struct {
  int32_t status;
  int32_t t[OR_KMAX];
  double phi;
  int32_t has_runner_up;
  int32_t t2[OR_KMAX];
  double phi2;
  double gap;
  int64_t tuples_valid;
} oracle_result;

typedef struct {
  int level;
  int bins, m;
  const double *p;
  double q;
  int *first_nz_ge; /* [bins+1] index into nz[] of first non-empty bin >= a */
  int *last_nz_le;  /* [bins]   index into nz[] of last non-empty bin <= b, -1 if none */
  int *nz;          /* [m] non-empty bins ascending */
  double *memo;     /* [m*m] Level 1 */
  unsigned char *have;
} class_ctx;

static double class_S(class_ctx *c, int a, int b, int *valid) {
  if (c->level == 0) return oracle_class_entropy(c->p, a, b, c->q, valid);
  int ia = c->first_nz_ge[a];
  int ib = c->last_nz_le[b];
  if (ib < 0 || ia >= c->m || ia > ib) {
    *valid = 0;
    return 0.0;
  }
  *valid = 1;
  size_t key = (size_t)ia * (size_t)c->m + (size_t)ib;
  if (!c->have[key]) {
    int v;
    c->memo[key] = oracle_class_entropy(c->p, c->nz[ia], c->nz[ib], c->q, &v);
    c->have[key] = 1;
  }
  return c->memo[key];
}

/* Exhaustive search over every t_1 < ... < t_k in [0, L-2], lexicographic
 * order, strict-greater argmax (lowest tuple wins).  level 0 or 1. */
int oracle_search(const uint32_t *hist, int bins, int k, double q, int objective,
                  int level, oracle_result *out) {
  memset(out, 0, sizeof(*out));
  for (int j = 0; j < OR_KMAX; j++) out->t[j] = out->t2[j] = -1;
  out->phi = out->phi2 = out->gap = NAN;
  if (k < 1 || k > OR_KMAX || bins < 2 || k > bins - 1 || !(q > 0.0) || !isfinite(q)) {
    out->status = OR_INVALID_ARG;
    return OR_INVALID_ARG;
  }
  double N = 0.0;
  for (int i = 0; i < bins; i++) N += (double)hist[i];
  if (N == 0.0) {
    out->status = OR_NO_VALID_SPLIT;
    return OR_NO_VALID_SPLIT;
  }
  class_ctx c;
  memset(&c, 0, sizeof(c));
  c.level = level;
  c.bins = bins;
  c.q = q;
  double *p = (double *)malloc(sizeof(double) * bins);
  probabilities(hist, bins, p);
  c.p = p;
  c.nz = (int *)malloc(sizeof(int) * bins);
  c.first_nz_ge = (int *)malloc(sizeof(int) * (bins + 1));
  c.last_nz_le = (int *)malloc(sizeof(int) * bins);
  int m = 0;
  for (int i = 0; i < bins; i++) {
    c.last_nz_le[i] = -1;
    if (hist[i] > 0) c.nz[m++] = i;
    c.last_nz_le[i] = m - 1;
  }
  c.m = m;
  {
    /* first_nz_ge[i] = number of non-empty bins < i == index of first non-empty >= i */
    int cnt = 0;
    for (int i = 0; i < bins; i++) {
      c.first_nz_ge[i] = cnt;
      if (hist[i] > 0) cnt++;
    }
    c.first_nz_ge[bins] = cnt;
  }
  if (level == 1) {
    c.memo = (double *)malloc(sizeof(double) * (size_t)m * (size_t)m + 8);
    c.have = (unsigned char *)calloc((size_t)m * (size_t)m + 8, 1);
  }

  int t[OR_KMAX], lo[OR_KMAX + 1], hi[OR_KMAX + 1];
  double S[OR_KMAX + 1];
  for (int j = 0; j < k; j++) t[j] = j;
  int found = 0;
  double best = -INFINITY;
  /* canonical top-2 */
  int c_found = 0, c2_found = 0;
  double c1v = -INFINITY, c2v = -INFINITY;
  int c1t[OR_KMAX], c2t[OR_KMAX];
  int64_t nvalid = 0;
  for (;;) {
    class_bounds(t, k, bins, lo, hi);
    int ok = 1;
    for (int j = 0; j <= k && ok; j++) {
      int v;
      S[j] = class_S(&c, lo[j], hi[j], &v);
      ok = v;
    }
    if (ok) {
      nvalid++;
      double phi = combine(S, k + 1, q, objective);
      if (!found || phi > best) {
        best = phi;
        found = 1;
        for (int j = 0; j < k; j++) out->t[j] = t[j];
      }
      int canonical = 1;
      for (int j = 0; j < k; j++)
        if (hist[t[j]] == 0) canonical = 0;
      if (canonical) {
        if (!c_found || phi > c1v) {
          if (c_found) {
            c2v = c1v;
            c2_found = 1;
            memcpy(c2t, c1t, sizeof(c1t));
          }
          c1v = phi;
          c_found = 1;
          memcpy(c1t, t, sizeof(int) * k);
        } else if (!c2_found || phi > c2v) {
          c2v = phi;
          c2_found = 1;
          memcpy(c2t, t, sizeof(int) * k);
        }
      }
    }
    /* lexicographic successor of t over [0, bins-2] */
    int j = k - 1;
    while (j >= 0 && t[j] == bins - 2 - (k - 1 - j)) j--;
    if (j < 0) break;
    t[j]++;
    for (int jj = j + 1; jj < k; jj++) t[jj] = t[jj - 1] + 1;
  }
  out->tuples_valid = nvalid;
  if (!found) {
    out->status = OR_NO_VALID_SPLIT;
    for (int j = 0; j < OR_KMAX; j++) out->t[j] = -1;
  } else {
    out->status = OR_OK;
    out->phi = best;
    if (c2_found) {
      out->has_runner_up = 1;
      out->phi2 = c2v;
      for (int j = 0; j < k; j++) out->t2[j] = c2t[j];
      if (best == 0.0)
        out->gap = (c2v == 0.0) ? 0.0 : INFINITY;
      else
        out->gap = (best - c2v) / fabs(best);
    } else {
      out->gap = INFINITY;
    }
  }
  free(p);
  free(c.nz);
  free(c.first_nz_ge);
  free(c.last_nz_le);
  free(c.memo);
  free(c.have);
  return out->status;
}

/* ---------------------------------------------------------------- step 7 */
/* label(v) = #{ j : v > t_j }  (Algorithm 1, with T = t+1) */
void oracle_label(const void *slice, int dtype_bytes, int64_t n, int k,
                  const int32_t *t, uint8_t *labels) {
  for (int64_t x = 0; x < n; x++) {
    unsigned v = dtype_bytes == 1 ? ((const uint8_t *)slice)[x]
                                  : ((const uint16_t *)slice)[x];
    int l = 0;
    for (int j = 0; j < k; j++)
      if ((int)v > t[j]) l++;
    labels[x] = (uint8_t)l;
  }
}

/* ------------------------------------------------------------- whole path */
/* Steps 1-7 for slices [z0, z1) of a [nz][ny][nx] volume.  Outputs are indexed
 * by absolute slice z.  labels may be NULL.  OpenMP over slices (each slice is
 * independent; results do not depend on the thread count). */
int oracle_segment(const void *vol, int dtype_bytes, int64_t nx, int64_t ny,
                   int64_t nz, int64_t z0, int64_t z1, int bins, int k, double q,
                   int objective, int level, int nthreads, uint32_t *hist,
                   int32_t *thresholds, double *phi, double *gap,
                   int32_t *status, uint8_t *labels) {
  (void)nz;
  int64_t n = nx * ny;
  if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
  for (int64_t z = z0; z < z1; z++) {
    const unsigned char *slice = (const unsigned char *)vol + (size_t)z * n * dtype_bytes;
    uint32_t *h = hist + (size_t)z * bins;
    int st = oracle_histogram(slice, dtype_bytes, n, bins, h);
    oracle_result r;
    memset(&r, 0, sizeof(r));
    for (int j = 0; j < OR_KMAX; j++) r.t[j] = -1;
    r.phi = NAN;
    r.gap = NAN;
    if (st == OR_OK) st = oracle_search(h, bins, k, q, objective, level, &r);
    status[z] = st;
    for (int j = 0; j < k; j++) thresholds[z * k + j] = st == OR_OK ? r.t[j] : -1;
    phi[z] = st == OR_OK ? r.phi : NAN;
    gap[z] = st == OR_OK ? r.gap : NAN;
    if (labels) {
      uint8_t *lab = labels + (size_t)z * n;
      if (st == OR_OK)
        oracle_label(slice, dtype_bytes, n, k, r.t, lab);
      else
        memset(lab, 0, (size_t)n);
    }
  }
  return OR_OK;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ======================================================================
 * 2-D Tsallis thresholding -- the paper's own formulation (SURVEY.md §8(f)
 * NEXT row 1).  Plain definitions:
 *   g(x,y) = floor( (1/9) sum_{i,j in {-1,0,1}} f(x+i, y+j) )
 *            (the garbled f(x+i, y+i) read as f(x+i, y+j), "decimal part"
 *            read as floor; border: replicate -- DESIGN.md R18/R19)
 *   h(i,j) = #{(x,y): f = i, g = j},  p_ij = h / N
 *   class 1 = {i <= t, j <= s}, class 2 = {i > t, j > s}; quadrants 2 and 4
 *   are ignored
 *   P_c = sum_{class c} p_ij;  H_c = (1 - sum_{class c} (p_ij/P_c)^a)/(a - 1)
 *   (a == 1: Shannon)
 *   phi(t,s) = H_1 + H_2 + (1-a) H_1 H_2, argmax over (t,s) in [0,L-2]^2,
 *   lowest (t,s) on ties; only t labels: label = f > t
 * Sums run over cells in row-major (i, then j) ascending order.
 * ====================================================================== */

/* 3x3 floor mean with replicate border of one [ny][nx] u8 slice */
void oracle_mean3x3(const uint8_t *f, int64_t nx, int64_t ny, uint8_t *g) {
  for (int64_t y = 0; y < ny; y++) {
    for (int64_t x = 0; x < nx; x++) {
      int sum = 0;
      for (int dy = -1; dy <= 1; dy++) {
        for (int dx = -1; dx <= 1; dx++) {
          int64_t yy = y + dy, xx = x + dx;
          if (yy < 0) yy = 0;
          if (yy > ny - 1) yy = ny - 1;
          if (xx < 0) xx = 0;
          if (xx > nx - 1) xx = nx - 1;
          sum += f[yy * nx + xx];
        }
      }
      g[y * nx + x] = (uint8_t)(sum / 9);
    }
  }
}

/* h[i*L + j] over one slice; OR_LEVEL_OVERFLOW if any f >= L (not counted) */
int oracle_hist2d(const uint8_t *f, int64_t nx, int64_t ny, int L, uint32_t *h) {
  uint8_t *g = (uint8_t *)malloc((size_t)(nx * ny));
  oracle_mean3x3(f, nx, ny, g);
  int st = OR_OK;
  for (int64_t i = 0; i < (int64_t)L * L; i++) h[i] = 0;
  for (int64_t x = 0; x < nx * ny; x++) {
    if (f[x] >= L || g[x] >= L) {
      st = OR_LEVEL_OVERFLOW;
      continue;
    }
    h[(int64_t)f[x] * L + g[x]] += 1;
  }
  free(g);
  return st;
}

/* Tsallis entropy of the rectangle [i0,i1] x [j0,j1] of a 2-D p (row-major) */
static double rect_entropy(const double *p, int L, int i0, int i1, int j0, int j1, double q,
                           int *valid) {
  double P = 0.0;
  for (int i = i0; i <= i1; i++)
    for (int j = j0; j <= j1; j++) P = P + p[i * L + j];
  if (P == 0.0) {
    *valid = 0;
    return 0.0;
  }
  *valid = 1;
  if (q == 1.0) {
    double H = 0.0;
    for (int i = i0; i <= i1; i++)
      for (int j = j0; j <= j1; j++)
        if (p[i * L + j] > 0.0) {
          double r = p[i * L + j] / P;
          H = H - r * log(r);
        }
    return H;
  }
  double A = 0.0;
  for (int i = i0; i <= i1; i++)
    for (int j = j0; j <= j1; j++)
      if (p[i * L + j] > 0.0) A = A + pow(p[i * L + j] / P, q);
  return (1.0 - A) / (q - 1.0);
}

static void probabilities2d(const uint32_t *h, int L, double *p) {
  double N = 0.0;
  for (int64_t i = 0; i < (int64_t)L * L; i++) N += (double)h[i];
  for (int64_t i = 0; i < (int64_t)L * L; i++) p[i] = (double)h[i] / N;
}

/* phi(t,s) from the definition; *valid = 0 if a class is empty or (t,s) out of range */
double oracle_phi2d_at(const uint32_t *h, int L, double q, int t, int s, int *valid) {
  *valid = 0;
  if (t < 0 || s < 0 || t > L - 2 || s > L - 2) return NAN;
  double *p = (double *)malloc(sizeof(double) * (size_t)L * L);
  probabilities2d(h, L, p);
  int v1, v2;
  double H1 = rect_entropy(p, L, 0, t, 0, s, q, &v1);
  double H2 = rect_entropy(p, L, t + 1, L - 1, s + 1, L - 1, q, &v2);
  free(p);
  if (!v1 || !v2) return NAN;
  *valid = 1;
  return H1 + H2 + (1.0 - q) * H1 * H2;
}

/* Exhaustive 2-D search, Level 0: every candidate's phi from the definition
 * (O(L^4); each t row of candidates is independent, so rows run on OpenMP
 * threads, each writing its own slots -- the values do not depend on the
 * thread count).  Then, sequentially in row-major (t, then s) order, the
 * argmax with strict '>' (lowest (t,s) wins exact ties, "Arg
 * max"; R8/R21).
 * Runner-up (acceptance metadata only): best phi over candidates describing a
 * DIFFERENT partition of the non-empty cells.  (t,s) and (t',s) give the same
 * classes iff every row in (t, t'] is empty, and likewise for columns, so the
 * distinct partitions are exactly the "canonical" candidates whose row t and
 * column s are non-empty (row/column marginals of h); the lowest member of an
 * equivalence class is canonical (R21).  gap = (phi* - phi2)/|phi*|. */
int oracle_search2d_n(const uint32_t *h, int L, double q, int nthreads, int32_t *t_out,
                      int32_t *s_out, double *phi_out, double *gap_out) {
  const int M = L - 1;
  double *p = (double *)malloc(sizeof(double) * (size_t)L * L);
  double *phi = (double *)malloc(sizeof(double) * (size_t)(M > 0 ? M : 1) * (M > 0 ? M : 1));
  char *ok = (char *)calloc((size_t)(M > 0 ? M : 1) * (M > 0 ? M : 1), 1);
  probabilities2d(h, L, p);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
  for (int t = 0; t < M; t++) {
    for (int s = 0; s < M; s++) {
      int v1, v2;
      double H1 = rect_entropy(p, L, 0, t, 0, s, q, &v1);
      if (!v1) continue;
      double H2 = rect_entropy(p, L, t + 1, L - 1, s + 1, L - 1, q, &v2);
      if (!v2) continue;
      phi[(size_t)t * M + s] = H1 + H2 + (1.0 - q) * H1 * H2;
      ok[(size_t)t * M + s] = 1;
    }
  }
  int found = 0, bt = -1, bs = -1;
  double best = -INFINITY;
  for (int t = 0; t < M; t++)
    for (int s = 0; s < M; s++)
      if (ok[(size_t)t * M + s] && (!found || phi[(size_t)t * M + s] > best)) {
        best = phi[(size_t)t * M + s];
        bt = t;
        bs = s;
        found = 1;
      }
  /* marginals: non-empty rows (f levels) and columns (g levels) */
  char *rnz = (char *)calloc((size_t)L, 1), *cnz = (char *)calloc((size_t)L, 1);
  for (int i = 0; i < L; i++)
    for (int j = 0; j < L; j++)
      if (h[(size_t)i * L + j]) {
        rnz[i] = 1;
        cnz[j] = 1;
      }
  int have2 = 0;
  double second = -INFINITY;
  for (int t = 0; t < M; t++)
    for (int s = 0; s < M; s++)
      if (ok[(size_t)t * M + s] && rnz[t] && cnz[s] && !(t == bt && s == bs) &&
          (!have2 || phi[(size_t)t * M + s] > second)) {
        second = phi[(size_t)t * M + s];
        have2 = 1;
      }
  free(rnz);
  free(cnz);
  free(ok);
  free(phi);
  free(p);
  *t_out = bt;
  *s_out = bs;
  *phi_out = found ? best : NAN;
  *gap_out = !found ? NAN : (!have2 ? INFINITY : (best == 0.0 ? (second == 0.0 ? 0.0 : INFINITY)
                                                              : (best - second) / fabs(best)));
  return found ? OR_OK : OR_NO_VALID_SPLIT;
}

int oracle_search2d(const uint32_t *h, int L, double q, int32_t *t_out, int32_t *s_out,
                    double *phi_out, double *gap_out) {
  return oracle_search2d_n(h, L, q, 1, t_out, s_out, phi_out, gap_out);
}

/* ======================================================================
 * Pre-processing: "change the
 * value of -2000 (outside of the X-ray detectors) to 0 ... then all intensity
 * levels are linearly transformed to the range 0 to 255".  Readings
 * (R23-R25, after SPEC.md:73-81,:90-94):
 *   1. every voxel equal to `background` is replaced by the volume-wide
 *      minimum of the remaining voxels (so it maps to 0, the background level);
 *   2. lo / hi = volume-wide min / max after step 1;
 *   3. v -> round-half-away-from-zero(255 (v - lo) / (hi - lo)); hi == lo -> 0
 *      (also when every voxel is background).
 * Written in that order with exact integer arithmetic: for v >= lo the
 * rounded quotient is floor((2*255*(v-lo) + (hi-lo)) / (2*(hi-lo))).
 * ====================================================================== */
void oracle_preprocess(const int16_t *vol, int64_t n, int background, uint8_t *out,
                       int32_t *lo_out, int32_t *hi_out) {
  /* step 1: minimum of the non-background voxels */
  int have = 0, mn = 0;
  for (int64_t i = 0; i < n; i++) {
    if (vol[i] == background) continue;
    if (!have || vol[i] < mn) mn = vol[i];
    have = 1;
  }
  /* step 2: lo / hi over the volume after the replacement */
  int lo = 0, hi = 0;
  for (int64_t i = 0; i < n; i++) {
    int v = vol[i] == background && have ? mn : vol[i];
    if (i == 0 || v < lo) lo = v;
    if (i == 0 || v > hi) hi = v;
  }
  /* step 3: the linear map */
  for (int64_t i = 0; i < n; i++) {
    int v = vol[i] == background && have ? mn : vol[i];
    if (hi == lo) {
      out[i] = 0;
      continue;
    }
    int64_t num = 2 * 255 * (int64_t)(v - lo) + (hi - lo);
    int64_t den = 2 * (int64_t)(hi - lo);
    out[i] = (uint8_t)(num / den);
  }
  if (lo_out) *lo_out = lo;
  if (hi_out) *hi_out = hi;
}

/* ======================================================================
 * Morphology: grayscale
 * erosion / dilation by a disk structuring element, opening, and the top-hat
 * mask that removes the chest ("subtracting the original image from the
 * opened mask").  Readings (R26-R28, after SPEC.md:118-166):
 *   disk(r)      = { (dy,dx) : dy^2 + dx^2 <= r^2 }            ("disk-like ... size 10", :550)
 *   erode(a)(y,x)  = min over disk of a(y+dy, x+dx), samples outside the
 *                    slice = 255 (neutral for min)               A (-) B = {z | (B)_z in A}, :534
 *   dilate(a)(y,x) = max over the reflected disk (= the disk) of a(y+dy, x+dx),
 *                    outside = 0 (neutral for max)               A (+) B, :540
 *   open(a)      = dilate(erode(a))                             A o B = (A (-) B) (+) B, :546
 *   tophat(a)    = max(a - open(a), 0)  (white top-hat)
 * Per slice, brute force over the disk's offsets.
 * ====================================================================== */
static void morph_pass(const uint8_t *a, int64_t nx, int64_t ny, int r, int is_max, uint8_t *out) {
  for (int64_t y = 0; y < ny; y++) {
    for (int64_t x = 0; x < nx; x++) {
      int acc = is_max ? 0 : 255;
      for (int dy = -r; dy <= r; dy++) {
        for (int dx = -r; dx <= r; dx++) {
          if (dy * dy + dx * dx > r * r) continue;
          int64_t yy = y + dy, xx = x + dx;
          int v = (yy < 0 || yy >= ny || xx < 0 || xx >= nx) ? (is_max ? 0 : 255)
                                                             : a[yy * nx + xx];
          if (is_max ? v > acc : v < acc) acc = v;
        }
      }
      out[y * nx + x] = (uint8_t)acc;
    }
  }
}

void oracle_erode(const uint8_t *a, int64_t nx, int64_t ny, int r, uint8_t *out) {
  morph_pass(a, nx, ny, r, 0, out);
}

void oracle_dilate(const uint8_t *a, int64_t nx, int64_t ny, int r, uint8_t *out) {
  morph_pass(a, nx, ny, r, 1, out);
}

/* opening and top-hat of one slice; open_out may be NULL */
void oracle_tophat(const uint8_t *a, int64_t nx, int64_t ny, int r, uint8_t *open_out,
                   uint8_t *tophat_out) {
  uint8_t *e = (uint8_t *)malloc((size_t)(nx * ny));
  uint8_t *o = (uint8_t *)malloc((size_t)(nx * ny));
  morph_pass(a, nx, ny, r, 0, e);
  morph_pass(e, nx, ny, r, 1, o);
  for (int64_t i = 0; i < nx * ny; i++) {
    if (open_out) open_out[i] = o[i];
    tophat_out[i] = (uint8_t)(a[i] > o[i] ? a[i] - o[i] : 0);
  }
  free(e);
  free(o);
}
