/*
 * RAGBoost context-index ORACLE, plain C (timed CPU baseline).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs through oracle/oracle_c.py.
 * It shares no code, header or constant with the CUDA path
 * (paper_2511_03475_b200/csrc) and never calls it.
 *
 * Plain, slow, obviously correct:
 *   - overlap by brute-force K x K comparison of two contexts (PAPER:350-355,
 *     Eq. 1: S_ij = shared docs, p_i(k) = 0-based position);
 *   - d = correctly rounded binary32 of the exact Eq. 1 rational (X6), decided
 *     by exact 128-bit integer comparison of the float32 candidates;
 *   - row nearest neighbour nn_i = argmin_{j != i} (d_ij, j);
 *   - complete linkage (X7) by nearest-neighbour chain on the full matrix with
 *     the tie key (d, min rep, max rep) (X8), merges sorted by key (X9).
 *
 * Built: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (no fast-math, no
 * SIMD intrinsics).  OpenMP parallelises rows of the distance stage only.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __int128 i128;

int ro_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* |M * 2^E - num/den| scaled by den * 2^-Emin, as a signed 128-bit integer. */
static i128 scaled_err(int64_t M, int E, int Emin, uint64_t num, uint64_t den) {
  i128 lhs, rhs;
  if (Emin < 0) { /* multiply the error by den * 2^-Emin: all terms integral */
    lhs = ((i128)M * (i128)den) << (E - Emin);
    rhs = ((i128)num) << (-Emin);
  } else { /* every candidate is an integer: multiply by den only */
    lhs = ((i128)M * (i128)den) << E;
    rhs = (i128)num;
  }
  i128 d = lhs - rhs;
  return d < 0 ? -d : d;
}

/* Correctly rounded (nearest-even) binary32 of num/den, num >= 0, den > 0. */
float ro_rn32_ratio(uint64_t num, uint64_t den) {
  if (num == 0) return 0.0f;
  double q = (double)num / (double)den;
  float c0 = (float)q;
  float cand[3] = {c0, nextafterf(c0, INFINITY), nextafterf(c0, 0.0f)};
  int64_t Mv[3];
  int Ev[3];
  int Emin = 100000;
  for (int t = 0; t < 3; ++t) {
    int e;
    float m = frexpf(cand[t], &e);      /* cand = m * 2^e, m in [0.5, 1) */
    Mv[t] = (int64_t)ldexpf(m, 24);      /* exact 24-bit integer significand */
    Ev[t] = e - 24;
    if (Ev[t] < Emin) Emin = Ev[t];
  }
  int best = 0;
  i128 bestErr = scaled_err(Mv[0], Ev[0], Emin, num, den);
  for (int t = 1; t < 3; ++t) {
    i128 err = scaled_err(Mv[t], Ev[t], Emin, num, den);
    if (err < bestErr || (err == bestErr && (Mv[t] & 1) == 0 && (Mv[best] & 1) == 1)) {
      best = t;
      bestErr = err;
    }
  }
  return cand[best];
}

/* Eq. 1 for one pair from its counts: m = max(len_i, len_j); alpha = an/ad.
 * d = 1 - s/m + (an/ad) * D/s = ((m - s)*ad*s + an*D*m) / (ad*m*s). */
float ro_eq1(uint32_t s, uint32_t D, uint32_t m, uint32_t an, uint32_t ad) {
  if (s == 0) return 1.0f; /* X3: positional term 0 when S = {} */
  uint64_t num = (uint64_t)(m - s) * ad * s + (uint64_t)an * D * m;
  uint64_t den = (uint64_t)ad * m * s;
  return ro_rn32_ratio(num, den);
}

/* Brute-force K x K overlap of contexts i and j. */
static void overlap_pair(const uint32_t *ci, int li, const uint32_t *cj, int lj, uint32_t *s_out,
                         uint32_t *D_out) {
  uint32_t s = 0, D = 0;
  for (int p = 0; p < li; ++p)
    for (int q = 0; q < lj; ++q)
      if (ci[p] == cj[q]) {
        s += 1;
        D += (uint32_t)(p > q ? p - q : q - p);
      }
  *s_out = s;
  *D_out = D;
}

/* Rows [row0, row0+nrows) x all N columns of s, D (optional) and d. */
int ro_pairwise_rows(const uint32_t *ids, const uint8_t *lens, int64_t N, int32_t K, uint32_t an,
                     uint32_t ad, int64_t row0, int64_t nrows, float *d_out, uint8_t *s_out,
                     uint16_t *D_out) {
  if (N < 1 || K < 1 || K > 255 || ad == 0 || row0 < 0 || row0 + nrows > N) return -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t i = row0 + r;
    int li = lens ? lens[i] : K;
    for (int64_t j = 0; j < N; ++j) {
      int lj = lens ? lens[j] : K;
      uint32_t s, D;
      overlap_pair(ids + i * K, li, ids + j * K, lj, &s, &D);
      uint32_t m = (uint32_t)(li > lj ? li : lj);
      d_out[r * N + j] = ro_eq1(s, D, m, an, ad);
      if (s_out) s_out[r * N + j] = (uint8_t)s;
      if (D_out) D_out[r * N + j] = (uint16_t)D;
    }
  }
  return 0;
}

/* nn_i = argmin_{j != i} (d_ij, j) over rows of a [nrows][N] block. */
int ro_row_nn(const float *d, int64_t N, int64_t row0, int64_t nrows, int32_t *nn_idx,
              float *nn_d) {
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t i = row0 + r;
    int32_t bi = -1;
    float bv = INFINITY;
    for (int64_t j = 0; j < N; ++j) {
      if (j == i) continue;
      float v = d[r * N + j];
      if (bi < 0 || v < bv) { /* strict: first j wins among equal values */
        bv = v;
        bi = (int32_t)j;
      }
    }
    nn_idx[r] = bi;
    nn_d[r] = bv;
  }
  return 0;
}

typedef struct {
  int32_t a, b, size;
  float h;
} merge_t;

static int key_less(float h1, int32_t a1, int32_t b1, float h2, int32_t a2, int32_t b2) {
  if (h1 != h2) return h1 < h2;
  if (a1 != a2) return a1 < a2;
  return b1 < b2;
}

static int cmp_merge(const void *x, const void *y) {
  const merge_t *p = (const merge_t *)x, *q = (const merge_t *)y;
  if (key_less(p->h, p->a, p->b, q->h, q->a, q->b)) return -1;
  if (key_less(q->h, q->a, q->b, p->h, p->a, p->b)) return 1;
  return 0;
}

/* Complete linkage by NN-chain on the full symmetric matrix d (N x N, modified
 * in place).  Cluster slot = rep = smallest leaf index.  Outputs N-1 merges in
 * greedy (key) order. */
int ro_linkage_nnchain(float *d, int64_t N, int32_t *za, int32_t *zb, float *zh, int32_t *zsize) {
  if (N < 1) return -1;
  if (N == 1) return 0;
  uint8_t *active = (uint8_t *)malloc((size_t)N);
  int32_t *size = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
  int64_t *chain = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N + 1));
  merge_t *Z = (merge_t *)malloc(sizeof(merge_t) * (size_t)(N - 1));
  if (!active || !size || !chain || !Z) {
    free(active); free(size); free(chain); free(Z);
    return -4;
  }
  for (int64_t i = 0; i < N; ++i) {
    active[i] = 1;
    size[i] = 1;
  }
  int64_t clen = 0, nz = 0, remaining = N, first_active = 0;
  while (remaining > 1) {
    if (clen == 0) {
      while (!active[first_active]) ++first_active;
      chain[clen++] = first_active;
    }
    int64_t x = chain[clen - 1];
    /* NN of x under key (d, min rep, max rep) == (d, rep of candidate) for fixed x */
    int64_t y = -1;
    float best = INFINITY;
    for (int64_t j = 0; j < N; ++j) {
      if (!active[j] || j == x) continue;
      float v = d[x * N + j];
      if (y < 0 || v < best) {
        best = v;
        y = j;
      }
    }
    if (clen >= 2 && chain[clen - 2] == y) {
      clen -= 2;
      int64_t a = x < y ? x : y, b = x < y ? y : x;
      Z[nz].a = (int32_t)a;
      Z[nz].b = (int32_t)b;
      Z[nz].h = best;
      Z[nz].size = size[a] + size[b];
      ++nz;
      for (int64_t j = 0; j < N; ++j) {
        if (!active[j] || j == a || j == b) continue;
        float va = d[a * N + j], vb = d[b * N + j];
        float nv = va > vb ? va : vb; /* complete linkage: max over members */
        d[a * N + j] = nv;
        d[j * N + a] = nv;
      }
      active[b] = 0;
      size[a] += size[b];
      --remaining;
    } else {
      chain[clen++] = y;
    }
  }
  qsort(Z, (size_t)nz, sizeof(merge_t), cmp_merge);
  for (int64_t t = 0; t < nz; ++t) {
    za[t] = Z[t].a;
    zb[t] = Z[t].b;
    zh[t] = Z[t].h;
    zsize[t] = Z[t].size;
  }
  free(active); free(size); free(chain); free(Z);
  return 0;
}

/* NEXT-3 ("iteratively merge the closest pair, creating
 * a virtual node whose context is the sorted intersection", read as SPEC:177):
 * the merged cluster is represented by the ascending sorted intersection of
 * its two representatives; cluster distance = Eq. 1 between representatives
 * (positions = list index).  Greedy: each step merges the active pair with the
 * smallest key (d, min rep, max rep) (X8); the survivor keeps the smaller rep.
 * Plain O(N^2) scan per step over a full matrix; merges in greedy order.
 * ctx: [N][K] contexts (row-major; lens[i] or K docs); d: [N][N] Eq. 1 matrix of
 * the contexts (overwritten). */
int ro_linkage_intersection(const uint32_t *ids, const uint8_t *lens, int64_t N, int32_t K, uint32_t an,
                            uint32_t ad, float *d, int32_t *za, int32_t *zb, float *zh, int32_t *zsize) {
  if (N < 1 || K < 1 || K > 255 || ad == 0) return -1;
  uint32_t *ctx = (uint32_t *)malloc((size_t)N * K * 4);
  int *len = (int *)malloc((size_t)N * sizeof(int));
  int *size = (int *)malloc((size_t)N * sizeof(int));
  unsigned char *act = (unsigned char *)malloc((size_t)N);
  if (!ctx || !len || !size || !act) return -2;
  for (int64_t i = 0; i < N; ++i) {
    len[i] = lens ? lens[i] : K;
    for (int k = 0; k < len[i]; ++k) ctx[i * K + k] = ids[i * K + k];
    size[i] = 1;
    act[i] = 1;
  }
  for (int64_t t = 0; t + 1 < N; ++t) {
    int64_t ba = -1, bb = -1;
    float bh = 0.0f;
    for (int64_t i = 0; i < N; ++i) {
      if (!act[i]) continue;
      for (int64_t j = i + 1; j < N; ++j) {
        if (!act[j]) continue;
        float v = d[i * N + j];
        if (ba < 0 || v < bh) { /* strict: the first (i, j) in index order wins ties */
          ba = i;
          bb = j;
          bh = v;
        }
      }
    }
    /* representative of the merged cluster: sorted intersection */
    uint32_t tmp[256];
    int n = 0;
    for (int p = 0; p < len[ba]; ++p)
      for (int q = 0; q < len[bb]; ++q)
        if (ctx[ba * K + p] == ctx[bb * K + q]) tmp[n++] = ctx[ba * K + p];
    for (int x = 1; x < n; ++x) { /* insertion sort, ascending DocId */
      uint32_t v = tmp[x];
      int y = x;
      while (y > 0 && tmp[y - 1] > v) {
        tmp[y] = tmp[y - 1];
        --y;
      }
      tmp[y] = v;
    }
    for (int x = 0; x < n; ++x) ctx[ba * K + x] = tmp[x];
    len[ba] = n;
    act[bb] = 0;
    size[ba] += size[bb];
    za[t] = (int32_t)ba;
    zb[t] = (int32_t)bb;
    zh[t] = bh;
    zsize[t] = size[ba];
    for (int64_t j = 0; j < N; ++j) { /* the survivor's new distances */
      if (!act[j] || j == ba) continue;
      uint32_t s, D;
      overlap_pair(ctx + ba * K, len[ba], ctx + j * K, len[j], &s, &D);
      uint32_t m = (uint32_t)(len[ba] > len[j] ? len[ba] : len[j]);
      float v = ro_eq1(s, D, m, an, ad);
      d[ba * N + j] = v;
      d[j * N + ba] = v;
    }
  }
  free(ctx);
  free(len);
  free(size);
  free(act);
  return 0;
}
