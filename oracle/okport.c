/*
 * okport.c -- TEST INFRASTRUCTURE ONLY: plain-C restatement of the reference
 * (okflow, header-only C++20 at /root/reference/proj/include/okflow) Newton
 * linear-solve path.  It is the parity CHECKER for the CUDA product
 * (paper_1603_04570_b200/libokg.so) and is never linked into it.
 *
 * Every routine follows the reference's own operation order (CSR assembly by
 * stably-sorted triplets, left-to-right row sums, MGS x2 GMRES, ...) so that
 * on identical inputs it reproduces the reference bit-for-bit; this is pinned
 * by tests/test_oracle.py against oracle/_ref/libokref.so (the reference
 * itself compiled) and against the golden vectors in tests/golden/.
 *
 * Interface: oracle/okoracle.h.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "okoracle.h"

static char g_err[512];
#define FAIL(code, ...)                                   \
  do {                                                    \
    snprintf(g_err, sizeof g_err, __VA_ARGS__);           \
    return (code);                                        \
  } while (0)
#define TRY(expr)              \
  do {                         \
    int st__ = (expr);         \
    if (st__ != OKO_OK) return st__; \
  } while (0)

const char* oko_last_error(void) { return g_err; }

static double* dalloc(long n) { return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }
static double* dcopy(const double* x, long n) {
  double* y = dalloc(n);
  memcpy(y, x, (size_t)n * sizeof(double));
  return y;
}

/* ---- vec.hpp:14-43 ------------------------------------------------------ */
static double dot(const double* a, const double* b, long n) {
  double s = 0.0;
  for (long i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static double norm2(const double* a, long n) { return sqrt(dot(a, a, n)); }
static void axpy(double alpha, const double* x, double* y, long n) {
  for (long i = 0; i < n; ++i) y[i] += alpha * x[i];
}
static void scal(double alpha, double* x, long n) {
  for (long i = 0; i < n; ++i) x[i] *= alpha;
}
static int all_finite(const double* x, long n) {
  for (long i = 0; i < n; ++i)
    if (!isfinite(x[i])) return 0;
  return 1;
}

/* ---- sparse.hpp:23-135 CSR with int32 indices --------------------------- */
typedef struct {
  int row, col;
  double val;
} triplet;
typedef struct {
  triplet* t;
  long n, cap;
} tvec;
static void tpush(tvec* v, int r, int c, double x) {
  if (v->n == v->cap) {
    v->cap = v->cap ? 2 * v->cap : 64;
    v->t = (triplet*)realloc(v->t, (size_t)v->cap * sizeof(triplet));
  }
  v->t[v->n].row = r;
  v->t[v->n].col = c;
  v->t[v->n].val = x;
  v->n++;
}

typedef struct {
  int nr, nc;
  int* rp;
  int* ci;
  double* v;
} csr;

static void csr_free(csr* A) {
  free(A->rp);
  free(A->ci);
  free(A->v);
  memset(A, 0, sizeof *A);
}

/* from_triplets (sparse.hpp:37-72): stable sort by (row, col), duplicates
 * summed in insertion order.  Stable bucket-by-row + stable insertion sort by
 * column within each row is the same permutation as std::stable_sort. */
static int csr_from_triplets(int nr, int nc, tvec* ts, csr* out) {
  long n = ts->n;
  int* cnt = (int*)calloc((size_t)nr + 1, sizeof(int));
  for (long k = 0; k < n; ++k) {
    if (ts->t[k].row < 0 || ts->t[k].row >= nr || ts->t[k].col < 0 || ts->t[k].col >= nc) {
      free(cnt);
      FAIL(OKO_EINVAL, "from_triplets: index out of range");
    }
    cnt[ts->t[k].row + 1]++;
  }
  for (int r = 0; r < nr; ++r) cnt[r + 1] += cnt[r];
  triplet* s = (triplet*)malloc((size_t)(n > 0 ? n : 1) * sizeof(triplet));
  int* pos = (int*)malloc(((size_t)nr + 1) * sizeof(int));
  memcpy(pos, cnt, ((size_t)nr + 1) * sizeof(int));
  for (long k = 0; k < n; ++k) s[pos[ts->t[k].row]++] = ts->t[k];
  free(pos);
  for (int r = 0; r < nr; ++r) {
    for (int k = cnt[r] + 1; k < cnt[r + 1]; ++k) {
      triplet x = s[k];
      int j = k - 1;
      while (j >= cnt[r] && s[j].col > x.col) {
        s[j + 1] = s[j];
        --j;
      }
      s[j + 1] = x;
    }
  }
  out->nr = nr;
  out->nc = nc;
  out->rp = (int*)calloc((size_t)nr + 1, sizeof(int));
  out->ci = (int*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int));
  out->v = (double*)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  long k = 0, w = 0;
  for (int r = 0; r < nr; ++r) {
    while (k < n && s[k].row == r) {
      int c = s[k].col;
      double v = s[k].val;
      ++k;
      while (k < n && s[k].row == r && s[k].col == c) {
        v += s[k].val;
        ++k;
      }
      out->ci[w] = c;
      out->v[w] = v;
      ++w;
    }
    out->rp[r + 1] = (int)w;
  }
  free(s);
  free(cnt);
  free(ts->t);
  ts->t = NULL;
  ts->n = ts->cap = 0;
  return OKO_OK;
}

/* spmv (sparse.hpp:138-150) */
static void spmv(const csr* A, const double* x, double* y) {
  for (int i = 0; i < A->nr; ++i) {
    double s = 0.0;
    for (int k = A->rp[i]; k < A->rp[i + 1]; ++k) s += A->v[k] * x[A->ci[k]];
    y[i] = s;
  }
}
/* spmv_transpose (sparse.hpp:159-169) */
static void spmv_t(const csr* A, const double* x, double* y) {
  memset(y, 0, (size_t)A->nc * sizeof(double));
  for (int i = 0; i < A->nr; ++i)
    for (int k = A->rp[i]; k < A->rp[i + 1]; ++k) y[A->ci[k]] += A->v[k] * x[i];
}
static void csr_diag(const csr* A, double* d) {
  int m = A->nr < A->nc ? A->nr : A->nc;
  for (int i = 0; i < m; ++i) {
    d[i] = 0.0;
    for (int k = A->rp[i]; k < A->rp[i + 1]; ++k)
      if (A->ci[k] == i) d[i] = A->v[k];
  }
}
/* transpose (sparse.hpp:171-180) */
static int csr_transpose(const csr* A, csr* out) {
  tvec ts = {0};
  for (int i = 0; i < A->nr; ++i)
    for (int k = A->rp[i]; k < A->rp[i + 1]; ++k) tpush(&ts, A->ci[k], i, A->v[k]);
  return csr_from_triplets(A->nc, A->nr, &ts, out);
}
/* add (sparse.hpp:183-196) */
static int csr_add(const csr* A, double alpha, const csr* B, csr* out) {
  tvec ts = {0};
  for (int i = 0; i < A->nr; ++i)
    for (int k = A->rp[i]; k < A->rp[i + 1]; ++k) tpush(&ts, i, A->ci[k], A->v[k]);
  for (int i = 0; i < B->nr; ++i)
    for (int k = B->rp[i]; k < B->rp[i + 1]; ++k) tpush(&ts, i, B->ci[k], alpha * B->v[k]);
  return csr_from_triplets(A->nr, A->nc, &ts, out);
}
/* scale (sparse.hpp:198-202) */
static void csr_scale(const csr* A, double alpha, csr* out) {
  int nnz = A->rp[A->nr];
  out->nr = A->nr;
  out->nc = A->nc;
  out->rp = (int*)malloc(((size_t)A->nr + 1) * sizeof(int));
  out->ci = (int*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int));
  out->v = (double*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(double));
  memcpy(out->rp, A->rp, ((size_t)A->nr + 1) * sizeof(int));
  memcpy(out->ci, A->ci, (size_t)nnz * sizeof(int));
  for (int k = 0; k < nnz; ++k) out->v[k] = A->v[k] * alpha;
}
static int icmp(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}
/* matmul (sparse.hpp:204-230) */
static int csr_matmul(const csr* A, const csr* B, csr* out) {
  tvec ts = {0};
  double* acc = dalloc(B->nc);
  char* seen = (char*)calloc((size_t)B->nc + 1, 1);
  int* touched = (int*)malloc(((size_t)B->nc + 1) * sizeof(int));
  for (int i = 0; i < A->nr; ++i) {
    int nt = 0;
    for (int ka = A->rp[i]; ka < A->rp[i + 1]; ++ka) {
      int j = A->ci[ka];
      double av = A->v[ka];
      for (int kb = B->rp[j]; kb < B->rp[j + 1]; ++kb) {
        int c = B->ci[kb];
        if (!seen[c]) {
          seen[c] = 1;
          touched[nt++] = c;
        }
        acc[c] += av * B->v[kb];
      }
    }
    qsort(touched, (size_t)nt, sizeof(int), icmp);
    for (int t = 0; t < nt; ++t) {
      int c = touched[t];
      tpush(&ts, i, c, acc[c]);
      acc[c] = 0.0;
      seen[c] = 0;
    }
  }
  free(acc);
  free(seen);
  free(touched);
  return csr_from_triplets(A->nr, B->nc, &ts, out);
}

/* ---- mesh.hpp ------------------------------------------------------------ */
typedef struct {
  int dim, n;
  double h;
  long nv, ncell;
  double* vert; /* dim per vertex */
  int* cells;   /* dim+1 per cell */
} mesh_t;

static int grid_index(const mesh_t* m, int i, int j, int k) {
  const int s = m->n + 1;
  return m->dim == 2 ? i * s + j : (i * s + j) * s + k;
}

/* cell_volume (mesh.hpp:52-73) */
static double cell_volume(const mesh_t* m, long c) {
  const int* cv = m->cells + c * (m->dim + 1);
  const double* v0 = m->vert + (long)cv[0] * m->dim;
  if (m->dim == 2) {
    const double* v1 = m->vert + (long)cv[1] * 2;
    const double* v2 = m->vert + (long)cv[2] * 2;
    const double ax = v1[0] - v0[0], ay = v1[1] - v0[1];
    const double bx = v2[0] - v0[0], by = v2[1] - v0[1];
    return 0.5 * (ax * by - ay * bx);
  }
  double e[3][3];
  for (int k = 1; k <= 3; ++k) {
    const double* vk = m->vert + (long)cv[k] * 3;
    for (int d = 0; d < 3; ++d) e[k - 1][d] = vk[d] - v0[d];
  }
  const double det = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) -
                     e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
                     e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
  return det / 6.0;
}

static void mesh_free(mesh_t* m) {
  free(m->vert);
  free(m->cells);
  memset(m, 0, sizeof *m);
}

/* build_mesh (mesh.hpp:87-157) */
static int build_mesh(int dim, int n, mesh_t* m) {
  if (dim != 2 && dim != 3) FAIL(OKO_EINVAL, "build_mesh: dim must be 2 or 3");
  if (n < 1) FAIL(OKO_EINVAL, "build_mesh: n must be positive");
  memset(m, 0, sizeof *m);
  m->dim = dim;
  m->n = n;
  m->h = 1.0 / n;
  const int s = n + 1;
  if (dim == 2) {
    m->nv = (long)s * s;
    m->ncell = 2L * n * n;
    m->vert = dalloc(m->nv * 2);
    m->cells = (int*)malloc((size_t)m->ncell * 3 * sizeof(int));
    long p = 0;
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) {
        m->vert[p++] = i * m->h;
        m->vert[p++] = j * m->h;
      }
    long q = 0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const int a = grid_index(m, i, j, 0), b = grid_index(m, i + 1, j, 0);
        const int c = grid_index(m, i + 1, j + 1, 0), d = grid_index(m, i, j + 1, 0);
        int* cc = m->cells + q;
        cc[0] = a; cc[1] = b; cc[2] = c;
        cc[3] = a; cc[4] = c; cc[5] = d;
        q += 6;
      }
  } else {
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2},
                                    {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    static const int odd[6] = {0, 1, 1, 0, 0, 1};
    m->nv = (long)s * s * s;
    m->ncell = 6L * n * n * n;
    m->vert = dalloc(m->nv * 3);
    m->cells = (int*)malloc((size_t)m->ncell * 4 * sizeof(int));
    long p = 0;
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j)
        for (int k = 0; k < s; ++k) {
          m->vert[p++] = i * m->h;
          m->vert[p++] = j * m->h;
          m->vert[p++] = k * m->h;
        }
    long q = 0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k) {
          const int base[3] = {i, j, k};
          for (int pp = 0; pp < 6; ++pp) {
            int g[4][3];
            for (int d = 0; d < 3; ++d) g[0][d] = base[d];
            for (int v = 1; v < 4; ++v) {
              for (int d = 0; d < 3; ++d) g[v][d] = g[v - 1][d];
              g[v][perms[pp][v - 1]] += 1;
            }
            int idx[4];
            for (int v = 0; v < 4; ++v) idx[v] = grid_index(m, g[v][0], g[v][1], g[v][2]);
            if (odd[pp]) {
              int t = idx[1];
              idx[1] = idx[2];
              idx[2] = t;
            }
            memcpy(m->cells + q, idx, sizeof idx);
            q += 4;
          }
        }
  }
  double sum = 0.0, comp = 0.0;
  for (long c = 0; c < m->ncell; ++c) {
    const double vol = cell_volume(m, c);
    if (vol <= 0.0) {
      mesh_free(m);
      FAIL(OKO_EINCONSISTENT, "build_mesh: non-positive cell volume");
    }
    const double y = vol - comp;
    const double t = sum + y;
    comp = (t - sum) - y;
    sum = t;
  }
  if (fabs(sum - 1.0) > 1e-14) {
    mesh_free(m);
    FAIL(OKO_EINCONSISTENT, "build_mesh: cell volumes do not sum to 1");
  }
  return OKO_OK;
}

/* prolongation (mesh.hpp:169-194) */
static int prolongation(const mesh_t* coarse, const mesh_t* fine, csr* P) {
  tvec ts = {0};
  const int dim = fine->dim, s = fine->n + 1;
  for (long v = 0; v < fine->nv; ++v) {
    int g[3] = {0, 0, 0};
    if (dim == 2) {
      g[0] = (int)(v / s);
      g[1] = (int)(v % s);
    } else {
      g[0] = (int)(v / ((long)s * s));
      g[1] = (int)((v / s) % s);
      g[2] = (int)(v % s);
    }
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, on = 1;
    for (int d = 0; d < dim; ++d) {
      lo[d] = g[d] / 2;
      hi[d] = (g[d] + 1) / 2;
      if (g[d] % 2 != 0) on = 0;
    }
    if (on) {
      tpush(&ts, (int)v, grid_index(coarse, lo[0], lo[1], lo[2]), 1.0);
    } else {
      tpush(&ts, (int)v, grid_index(coarse, lo[0], lo[1], lo[2]), 0.5);
      tpush(&ts, (int)v, grid_index(coarse, hi[0], hi[1], hi[2]), 0.5);
    }
  }
  return csr_from_triplets((int)fine->nv, (int)coarse->nv, &ts, P);
}

/* ---- quadrature.hpp:32-111 ------------------------------------------------ */
static void gauss_legendre_01(int n, double* x, double* w) {
  for (int i = 0; i < n; ++i) {
    double t = cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = t;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      const double dp = n * (t * p1 - p0) / (t * t - 1.0);
      const double dt = p1 / dp;
      t -= dt;
      if (fabs(dt) < 1e-15) break;
    }
    double p0 = 1.0, p1 = t;
    for (int k = 2; k <= n; ++k) {
      const double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    const double dp = n * (t * p1 - p0) / (t * t - 1.0);
    x[i] = 0.5 * (1.0 - t);
    w[i] = 1.0 / ((1.0 - t * t) * dp * dp);
  }
}

typedef struct {
  int dim, np;
  double pts[64 * 4];
  double w[64];
} quadrule_t;

static void simplex_quadrature(int dim, int degree, quadrule_t* q) {
  q->dim = dim;
  q->np = 0;
  double xu[16], wu[16], xv[16], wv[16], xw[16], ww[16];
  if (dim == 2) {
    const int nu = (degree + 3) / 2, nv = (degree + 2) / 2;
    gauss_legendre_01(nu, xu, wu);
    gauss_legendre_01(nv, xv, wv);
    for (int i = 0; i < nu; ++i)
      for (int j = 0; j < nv; ++j) {
        const double x = xu[i], y = xv[j] * (1.0 - xu[i]);
        double* p = q->pts + q->np * 3;
        p[0] = 1.0 - x - y;
        p[1] = x;
        p[2] = y;
        q->w[q->np++] = wu[i] * wv[j] * (1.0 - xu[i]);
      }
  } else {
    const int nu = (degree + 4) / 2, nv = (degree + 3) / 2, nw = (degree + 2) / 2;
    gauss_legendre_01(nu, xu, wu);
    gauss_legendre_01(nv, xv, wv);
    gauss_legendre_01(nw, xw, ww);
    for (int i = 0; i < nu; ++i)
      for (int j = 0; j < nv; ++j)
        for (int k = 0; k < nw; ++k) {
          const double x = xu[i], y = xv[j] * (1.0 - xu[i]);
          const double z = xw[k] * (1.0 - xu[i]) * (1.0 - xv[j]);
          double* p = q->pts + q->np * 4;
          p[0] = 1.0 - x - y - z;
          p[1] = x;
          p[2] = y;
          p[3] = z;
          q->w[q->np++] = wu[i] * wv[j] * ww[k] * (1.0 - xu[i]) * (1.0 - xu[i]) * (1.0 - xv[j]);
        }
  }
}

/* ---- assembly.hpp --------------------------------------------------------- */
/* barycentric_gradients (assembly.hpp:32-78) */
static double bary_grad(const mesh_t* m, long c, double* grad) {
  const int d = m->dim;
  const int* cv = m->cells + c * (d + 1);
  const double* v0 = m->vert + (long)cv[0] * d;
  if (d == 2) {
    const double* v1 = m->vert + (long)cv[1] * 2;
    const double* v2 = m->vert + (long)cv[2] * 2;
    const double ax = v1[0] - v0[0], ay = v1[1] - v0[1];
    const double bx = v2[0] - v0[0], by = v2[1] - v0[1];
    const double det = ax * by - ay * bx;
    grad[2] = by / det;
    grad[3] = -bx / det;
    grad[4] = -ay / det;
    grad[5] = ax / det;
    grad[0] = -(grad[2] + grad[4]);
    grad[1] = -(grad[3] + grad[5]);
    return 0.5 * det;
  }
  double e[3][3];
  for (int k = 1; k <= 3; ++k) {
    const double* vk = m->vert + (long)cv[k] * 3;
    for (int dd = 0; dd < 3; ++dd) e[k - 1][dd] = vk[dd] - v0[dd];
  }
  const double det = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) -
                     e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
                     e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
  const double inv[3][3] = {
      {(e[1][1] * e[2][2] - e[1][2] * e[2][1]) / det, -(e[1][0] * e[2][2] - e[1][2] * e[2][0]) / det,
       (e[1][0] * e[2][1] - e[1][1] * e[2][0]) / det},
      {-(e[0][1] * e[2][2] - e[0][2] * e[2][1]) / det, (e[0][0] * e[2][2] - e[0][2] * e[2][0]) / det,
       -(e[0][0] * e[2][1] - e[0][1] * e[2][0]) / det},
      {(e[0][1] * e[1][2] - e[0][2] * e[1][1]) / det, -(e[0][0] * e[1][2] - e[0][2] * e[1][0]) / det,
       (e[0][0] * e[1][1] - e[0][1] * e[1][0]) / det}};
  for (int k = 1; k <= 3; ++k)
    for (int dd = 0; dd < 3; ++dd) grad[k * 3 + dd] = inv[k - 1][dd];
  for (int dd = 0; dd < 3; ++dd) grad[dd] = -(grad[3 + dd] + grad[6 + dd] + grad[9 + dd]);
  return det / 6.0;
}

/* assemble_mass (assembly.hpp:82-100) */
static int assemble_mass(const mesh_t* m, csr* M) {
  const int vpc = m->dim + 1;
  const double denom = (double)((m->dim + 1) * (m->dim + 2));
  tvec ts = {0};
  for (long c = 0; c < m->ncell; ++c) {
    const double vol = cell_volume(m, c);
    const int* cv = m->cells + c * vpc;
    for (int i = 0; i < vpc; ++i)
      for (int j = 0; j < vpc; ++j) tpush(&ts, cv[i], cv[j], vol * (i == j ? 2.0 : 1.0) / denom);
  }
  return csr_from_triplets((int)m->nv, (int)m->nv, &ts, M);
}

/* assemble_stiffness (assembly.hpp:105-127) */
static int assemble_stiffness(const mesh_t* m, csr* K) {
  const int d = m->dim, vpc = d + 1;
  tvec ts = {0};
  double grad[12];
  for (long c = 0; c < m->ncell; ++c) {
    const double vol = bary_grad(m, c, grad);
    const int* cv = m->cells + c * vpc;
    for (int i = 0; i < vpc; ++i)
      for (int j = 0; j < vpc; ++j) {
        double g = 0.0;
        for (int dd = 0; dd < d; ++dd) g += grad[i * d + dd] * grad[j * d + dd];
        tpush(&ts, cv[i], cv[j], vol * g);
      }
  }
  return csr_from_triplets((int)m->nv, (int)m->nv, &ts, K);
}

/* assemble_load (assembly.hpp:130-138) */
static void assemble_load(const mesh_t* m, double* b) {
  memset(b, 0, (size_t)m->nv * sizeof(double));
  const double inv_vpc = 1.0 / (m->dim + 1);
  for (long c = 0; c < m->ncell; ++c) {
    const double w = cell_volume(m, c) * inv_vpc;
    for (int k = 0; k <= m->dim; ++k) b[m->cells[c * (m->dim + 1) + k]] += w;
  }
}

/* assemble_coefficient_mass (assembly.hpp:153-191), degree 4 */
static int assemble_coefficient_mass(const mesh_t* m, const double* u, csr* Me) {
  quadrule_t q;
  simplex_quadrature(m->dim, 4, &q);
  const int vpc = m->dim + 1;
  const double ref_measure = m->dim == 2 ? 0.5 : 1.0 / 6.0;
  tvec ts = {0};
  double local[16];
  for (long c = 0; c < m->ncell; ++c) {
    const int* cv = m->cells + c * vpc;
    const double scale = cell_volume(m, c) / ref_measure;
    for (int k = 0; k < vpc * vpc; ++k) local[k] = 0.0;
    for (int p = 0; p < q.np; ++p) {
      const double* bq = q.pts + p * vpc;
      double uq = 0.0;
      for (int k = 0; k < vpc; ++k) uq += u[cv[k]] * bq[k];
      const double coef = (3.0 * uq * uq - 1.0) * q.w[p];
      for (int i = 0; i < vpc; ++i)
        for (int j = 0; j < vpc; ++j) local[i * vpc + j] += coef * bq[i] * bq[j];
    }
    for (int i = 0; i < vpc; ++i)
      for (int j = 0; j < vpc; ++j) tpush(&ts, cv[i], cv[j], scale * local[i * vpc + j]);
  }
  return csr_from_triplets((int)m->nv, (int)m->nv, &ts, Me);
}

/* assemble_nonlinear (assembly.hpp:194-217), degree 4 */
static void assemble_nonlinear(const mesh_t* m, const double* u, double* out) {
  quadrule_t q;
  simplex_quadrature(m->dim, 4, &q);
  const int vpc = m->dim + 1;
  const double ref_measure = m->dim == 2 ? 0.5 : 1.0 / 6.0;
  memset(out, 0, (size_t)m->nv * sizeof(double));
  for (long c = 0; c < m->ncell; ++c) {
    const int* cv = m->cells + c * vpc;
    const double scale = cell_volume(m, c) / ref_measure;
    for (int p = 0; p < q.np; ++p) {
      const double* bq = q.pts + p * vpc;
      double uq = 0.0;
      for (int k = 0; k < vpc; ++k) uq += u[cv[k]] * bq[k];
      const double f = (uq * uq * uq - uq) * q.w[p] * scale;
      for (int i = 0; i < vpc; ++i) out[cv[i]] += f * bq[i];
    }
  }
}

/* ---- dense.hpp:175-226 Cholesky ----------------------------------------- */
typedef struct {
  int n;
  double* L; /* row-major n x n */
} chol_t;

static int chol_factor(const double* A, int n, chol_t* f) {
  f->n = n;
  f->L = dalloc((long)n * n);
  double* L = f->L;
  for (int j = 0; j < n; ++j) {
    double d = A[(long)j * n + j];
    for (int k = 0; k < j; ++k) d -= L[(long)j * n + k] * L[(long)j * n + k];
    if (d <= 0.0 || !isfinite(d)) FAIL(OKO_ENUMERICAL, "Cholesky: matrix not positive definite");
    L[(long)j * n + j] = sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double s = A[(long)i * n + j];
      for (int k = 0; k < j; ++k) s -= L[(long)i * n + k] * L[(long)j * n + k];
      L[(long)i * n + j] = s / L[(long)j * n + j];
    }
  }
  return OKO_OK;
}
static void chol_solve(const chol_t* f, const double* b, double* x) {
  const int n = f->n;
  const double* L = f->L;
  double* y = dalloc(n);
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int j = 0; j < i; ++j) s -= L[(long)i * n + j] * y[j];
    y[i] = s / L[(long)i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int j = i + 1; j < n; ++j) s -= L[(long)j * n + i] * x[j];
    x[i] = s / L[(long)i * n + i];
  }
  free(y);
}

/* ---- eig.hpp:216-261 cyclic Jacobi --------------------------------------- */
static int symmetric_eigenvalues(double* A, int n, double* ev) {
  const int max_sweeps = 60;
  double ref = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) ref += A[i * n + j] * A[i * n + j];
  ref = sqrt(ref);
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) off += A[i * n + j] * A[i * n + j];
    if (sqrt(off) <= 1e-14 * ref + 1e-300) break;
    if (sweep == max_sweeps - 1) FAIL(OKO_ENUMERICAL, "symmetric eigensolver failed to converge");
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (fabs(apq) <= 1e-300) continue;
        const double tau = (A[q * n + q] - A[p * n + p]) / (2.0 * apq);
        const double tt = (tau >= 0.0) ? 1.0 / (tau + sqrt(1.0 + tau * tau))
                                       : -1.0 / (-tau + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + tt * tt);
        const double s = tt * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
      }
  }
  for (int i = 0; i < n; ++i) ev[i] = A[i * n + i];
  for (int i = 1; i < n; ++i) { /* ascending */
    double x = ev[i];
    int j = i - 1;
    while (j >= 0 && ev[j] > x) {
      ev[j + 1] = ev[j];
      --j;
    }
    ev[j + 1] = x;
  }
  return OKO_OK;
}

/* ---- std::mt19937 + libstdc++ uniform_real_distribution<double>(-1, 1) ---- */
typedef struct {
  uint32_t mt[624];
  int idx;
} mt19937_t;
static void mt_seed(mt19937_t* g, uint32_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 624; ++i)
    g->mt[i] = 1812433253u * (g->mt[i - 1] ^ (g->mt[i - 1] >> 30)) + (uint32_t)i;
  g->idx = 624;
}
static uint32_t mt_next(mt19937_t* g) {
  if (g->idx >= 624) {
    for (int i = 0; i < 624; ++i) {
      uint32_t y = (g->mt[i] & 0x80000000u) | (g->mt[(i + 1) % 624] & 0x7fffffffu);
      uint32_t v = g->mt[(i + 397) % 624] ^ (y >> 1);
      if (y & 1u) v ^= 0x9908b0dfu;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint32_t y = g->mt[g->idx++];
  y ^= y >> 11;
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= y >> 18;
  return y;
}
/* generate_canonical<double,53>: two 32-bit draws, (g1 + g2 * 2^32) / 2^64 */
static double mt_uniform(mt19937_t* g, double a, double b) {
  const double r = 4294967296.0;
  double sum = 0.0, tmp = 1.0;
  for (int k = 0; k < 2; ++k) {
    sum += (double)mt_next(g) * tmp;
    tmp *= r;
  }
  double ret = sum / tmp;
  if (ret >= 1.0) ret = nextafter(1.0, 0.0);
  return ret * (b - a) + a;
}

/* lanczos_extremes (krylov.hpp:248-289): extreme Ritz values of apply_B after
 * `probes` steps of Lanczos with full reorthogonalisation from mt19937(seed) */
typedef void (*apply_fn)(const void* ctx, const double* x, double* y);
static int lanczos_extremes(apply_fn apply_B, const void* actx, long n, int probes, unsigned seed, double* lo,
                            double* hi) {
  int steps = probes < n ? probes : (int)n;
  mt19937_t rng;
  mt_seed(&rng, seed);
  double** V = (double**)calloc((size_t)steps + 1, sizeof(double*));
  int nV = 0;
  double* v = dalloc(n);
  for (long i = 0; i < n; ++i) v[i] = mt_uniform(&rng, -1.0, 1.0);
  scal(1.0 / norm2(v, n), v, n);
  V[nV++] = v;
  double alpha[64], beta[64];
  int na = 0, nb_ = 0;
  double* w = dalloc(n);
  for (int j = 0; j < steps; ++j) {
    apply_B(actx, V[j], w);
    const double a = dot(w, V[j], n);
    alpha[na++] = a;
    axpy(-a, V[j], w, n);
    if (j > 0) axpy(-beta[j - 1], V[j - 1], w, n);
    for (int qv = 0; qv < nV; ++qv) axpy(-dot(w, V[qv], n), V[qv], w, n);
    const double nb = norm2(w, n);
    if (nb <= 1e-13 * fabs(a) + 1e-300) break;
    if (j + 1 < steps) {
      beta[nb_++] = nb;
      double* nv = dalloc(n);
      for (long i = 0; i < n; ++i) nv[i] = w[i] * (1.0 / nb);
      V[nV++] = nv;
    }
  }
  const int mm = na;
  double* T = dalloc((long)mm * mm);
  for (int i = 0; i < mm; ++i) {
    T[i * mm + i] = alpha[i];
    if (i + 1 < mm) {
      T[i * mm + i + 1] = beta[i];
      T[(i + 1) * mm + i] = beta[i];
    }
  }
  double ev[64];
  int st = symmetric_eigenvalues(T, mm, ev);
  for (int qv = 0; qv < nV; ++qv) free(V[qv]);
  free(V);
  free(T);
  free(w);
  if (st != OKO_OK) return st;
  *lo = ev[0];
  *hi = ev[mm - 1];
  return OKO_OK;
}

typedef struct {
  const csr* A;
  const double* dsqrt;
  double* t;
} jacobi_probe_t;

/* B = D^-1/2 A D^-1/2 (krylov.hpp:307-312) */
static void jacobi_probe(const void* ctx, const double* x, double* y) {
  const jacobi_probe_t* q = (const jacobi_probe_t*)ctx;
  const long n = q->A->nr;
  for (long i = 0; i < n; ++i) q->t[i] = x[i] / q->dsqrt[i];
  spmv(q->A, q->t, y);
  for (long i = 0; i < n; ++i) y[i] /= q->dsqrt[i];
}

/* estimate_jacobi_spectrum (krylov.hpp:296-320) */
static int estimate_jacobi_spectrum(const csr* A, double* lo_out, double* hi_out) {
  const long n = A->nr;
  double* d = dalloc(n);
  csr_diag(A, d);
  double* dsqrt = dalloc(n);
  for (long i = 0; i < n; ++i) {
    if (d[i] <= 0.0) {
      free(d);
      free(dsqrt);
      FAIL(OKO_ENUMERICAL, "estimate_jacobi_spectrum: non-positive diagonal");
    }
    dsqrt[i] = sqrt(d[i]);
  }
  jacobi_probe_t q = {A, dsqrt, dalloc(n)};
  double lo = 0, hi = 0;
  const int st = lanczos_extremes(jacobi_probe, &q, n, 30, 1234u, &lo, &hi);
  free(q.t);
  free(d);
  free(dsqrt);
  if (st != OKO_OK) return st;
  if (lo < 0.0)
    FAIL(OKO_ENUMERICAL, "estimate_jacobi_spectrum: negative Ritz value, matrix not positive definite");
  *lo_out = 0.9 * lo;
  *hi_out = 1.1 * hi;
  return OKO_OK;
}

/* ---- SsorSweeps (krylov.hpp:322-388), omega = 1 as make_schur_context uses it ---- */
typedef struct {
  const csr* A;
  double omega;
  double* diag;
} ssor_t;

static int ssor_init(const csr* A, double omega, ssor_t* s) {
  if (omega <= 0.0 || omega >= 2.0) FAIL(OKO_EINVAL, "ssor: omega must lie in (0, 2)");
  s->A = A;
  s->omega = omega;
  s->diag = dalloc(A->nr);
  csr_diag(A, s->diag);
  for (long i = 0; i < A->nr; ++i)
    if (s->diag[i] <= 0.0) FAIL(OKO_EINVAL, "ssor: non-positive diagonal");
  return OKO_OK;
}

/* (D/w + L) x = r by forward substitution */
static void ssor_forward(const ssor_t* s, const double* r, double* x) {
  const csr* A = s->A;
  for (int i = 0; i < A->nr; ++i) {
    double acc = r[i];
    for (int k = A->rp[i]; k < A->rp[i + 1]; ++k) {
      const int j = A->ci[k];
      if (j >= i) break;
      acc -= A->v[k] * x[j];
    }
    x[i] = acc * s->omega / s->diag[i];
  }
}

/* (D/w + U) x = r by backward substitution */
static void ssor_backward(const ssor_t* s, const double* r, double* x) {
  const csr* A = s->A;
  for (int i = A->nr - 1; i >= 0; --i) {
    double acc = r[i];
    for (int k = A->rp[i + 1] - 1; k >= A->rp[i]; --k) {
      const int j = A->ci[k];
      if (j <= i) break;
      acc -= A->v[k] * x[j];
    }
    x[i] = acc * s->omega / s->diag[i];
  }
}

/* z = P^{-1} r (apply_inv) */
static void ssor_apply_inv(const ssor_t* s, const double* r, double* z, double* t) {
  ssor_forward(s, r, t);
  const double g = (2.0 - s->omega) / s->omega;
  for (long i = 0; i < s->A->nr; ++i) t[i] *= g * s->diag[i];
  ssor_backward(s, t, z);
}

typedef struct {
  const ssor_t* sw;
  const double* dsqrt;
  double g;
  double *t, *u, *v;
} ssor_probe_t;

/* B = E A E^T with E = g D^{1/2} (D/w + L)^{-1} (krylov.hpp:400-407) */
static void ssor_probe(const void* ctx, const double* x, double* y) {
  const ssor_probe_t* q = (const ssor_probe_t*)ctx;
  const long n = q->sw->A->nr;
  for (long i = 0; i < n; ++i) q->t[i] = q->g * q->dsqrt[i] * x[i];
  ssor_backward(q->sw, q->t, q->u);
  spmv(q->sw->A, q->u, q->v);
  ssor_forward(q->sw, q->v, y);
  for (long i = 0; i < n; ++i) y[i] *= q->g * q->dsqrt[i];
}

/* estimate_ssor_spectrum (krylov.hpp:390-418) */
static int estimate_ssor_spectrum(const csr* A, double omega, double* lo_out, double* hi_out) {
  ssor_t sw;
  TRY(ssor_init(A, omega, &sw));
  const long n = A->nr;
  ssor_probe_t q;
  q.sw = &sw;
  q.g = sqrt((2.0 - omega) / omega);
  double* dsqrt = dalloc(n);
  for (long i = 0; i < n; ++i) dsqrt[i] = sqrt(sw.diag[i]);
  q.dsqrt = dsqrt;
  q.t = dalloc(n);
  q.u = dalloc(n);
  q.v = dalloc(n);
  double lo = 0, hi = 0;
  const int st = lanczos_extremes(ssor_probe, &q, n, 30, 1234u, &lo, &hi);
  free(q.t);
  free(q.u);
  free(q.v);
  free(dsqrt);
  free(sw.diag);
  if (st != OKO_OK) return st;
  if (lo < 0.0)
    FAIL(OKO_ENUMERICAL, "estimate_ssor_spectrum: negative Ritz value, matrix not positive definite");
  *lo_out = 0.9 * lo;
  *hi_out = 1.1 * hi;
  return OKO_OK;
}

/* ---- multigrid.hpp -------------------------------------------------------- */
typedef struct {
  int levels;
  csr ops[32];
  csr prolong[32];
  double* inv_diag[32];
  double omega;
  chol_t coarse;
} hier_t;

static void hier_free(hier_t* h) {
  for (int l = 0; l < h->levels; ++l) {
    csr_free(&h->ops[l]);
    free(h->inv_diag[l]);
    if (l + 1 < h->levels) csr_free(&h->prolong[l]);
  }
  free(h->coarse.L);
  memset(h, 0, sizeof *h);
}

/* build_hierarchy (multigrid.hpp:43-86) */
static int build_hierarchy(const mesh_t* mesh, const csr* M, const csr* K, double eps_sqrt_c,
                           int min_coarse_size, double omega, hier_t* h) {
  memset(h, 0, sizeof *h);
  if (min_coarse_size < 1) FAIL(OKO_EINVAL, "build_hierarchy: min_coarse_size < 1");
  const int kDenseCap = 2000;
  h->omega = omega;
  TRY(csr_add(M, eps_sqrt_c, K, &h->ops[0]));
  h->levels = 1;
  mesh_t lm;
  TRY(build_mesh(mesh->dim, mesh->n, &lm));
  while (h->ops[h->levels - 1].nr > min_coarse_size && lm.n % 2 == 0) {
    mesh_t coarse;
    TRY(build_mesh(lm.dim, lm.n / 2, &coarse));
    csr P, Pt, SP, C;
    TRY(prolongation(&coarse, &lm, &P));
    TRY(csr_matmul(&h->ops[h->levels - 1], &P, &SP));
    TRY(csr_transpose(&P, &Pt));
    TRY(csr_matmul(&Pt, &SP, &C));
    csr_free(&SP);
    csr_free(&Pt);
    h->prolong[h->levels - 1] = P;
    h->ops[h->levels] = C;
    h->levels++;
    mesh_free(&lm);
    lm = coarse;
  }
  mesh_free(&lm);
  const int coarsest = h->ops[h->levels - 1].nr;
  const int cap = min_coarse_size > kDenseCap ? min_coarse_size : kDenseCap;
  if (coarsest > cap)
    FAIL(OKO_ECONFIG,
         "build_hierarchy: coarsest level too large for a direct solve; choose a grid with "
         "more factors of two");
  for (int l = 0; l < h->levels; ++l) {
    const csr* A = &h->ops[l];
    h->inv_diag[l] = dalloc(A->nr);
    csr_diag(A, h->inv_diag[l]);
    for (int i = 0; i < A->nr; ++i) {
      if (h->inv_diag[l][i] <= 0.0) FAIL(OKO_ENUMERICAL, "build_hierarchy: non-positive diagonal");
      h->inv_diag[l][i] = 1.0 / h->inv_diag[l][i];
    }
  }
  const csr* Ac = &h->ops[h->levels - 1];
  double* D = dalloc((long)Ac->nr * Ac->nr);
  for (int i = 0; i < Ac->nr; ++i)
    for (int k = Ac->rp[i]; k < Ac->rp[i + 1]; ++k) D[(long)i * Ac->nr + Ac->ci[k]] = Ac->v[k];
  int st = chol_factor(D, Ac->nr, &h->coarse);
  free(D);
  return st;
}

/* damped_jacobi (multigrid.hpp:90-95) */
static void damped_jacobi(const csr* A, const double* inv_diag, double omega, const double* b,
                          double* x) {
  double* Ax = dalloc(A->nr);
  spmv(A, x, Ax);
  for (int i = 0; i < A->nr; ++i) x[i] += omega * inv_diag[i] * (b[i] - Ax[i]);
  free(Ax);
}

/* mg_cycle (multigrid.hpp:97-117) -> x (length of level) */
static void mg_cycle(const hier_t* h, int level, const double* b, int pre, int post, double* x) {
  if (level == h->levels - 1) {
    chol_solve(&h->coarse, b, x);
    return;
  }
  const csr* A = &h->ops[level];
  const long n = A->nr;
  memset(x, 0, (size_t)n * sizeof(double));
  for (int s = 0; s < pre; ++s) damped_jacobi(A, h->inv_diag[level], h->omega, b, x);
  double* r = dcopy(b, n);
  double* Ax = dalloc(n);
  spmv(A, x, Ax);
  axpy(-1.0, Ax, r, n);
  const csr* P = &h->prolong[level];
  double* rc = dalloc(P->nc);
  spmv_t(P, r, rc);
  double* ec = dalloc(P->nc);
  mg_cycle(h, level + 1, rc, pre, post, ec);
  double* ef = dalloc(n);
  spmv(P, ec, ef);
  axpy(1.0, ef, x, n);
  for (int s = 0; s < post; ++s) damped_jacobi(A, h->inv_diag[level], h->omega, b, x);
  free(r);
  free(Ax);
  free(rc);
  free(ec);
  free(ef);
}

/* apply_shat_inv (multigrid.hpp:133-149) */
static void apply_shat_inv(const hier_t* h, const double* b, int cycles, int pre, int post,
                           double* x) {
  const long n = h->ops[0].nr;
  memset(x, 0, (size_t)n * sizeof(double));
  double* r = dcopy(b, n);
  double* e = dalloc(n);
  double* Ax = dalloc(n);
  for (int cyc = 0; cyc < cycles; ++cyc) {
    mg_cycle(h, 0, r, pre, post, e);
    axpy(1.0, e, x, n);
    if (cyc + 1 == cycles) break;
    spmv(&h->ops[0], x, Ax);
    memcpy(r, b, (size_t)n * sizeof(double));
    axpy(-1.0, Ax, r, n);
  }
  free(r);
  free(e);
  free(Ax);
}

/* ---- precond.hpp ---------------------------------------------------------- */
typedef struct {
  oko_params p;
  mesh_t mesh;
  csr M, K, A; /* A = a_coeff * M (precond.hpp:154) */
  double* b;
  csr Me;
  int have_me;
  double c, eps, sqrt_c, a_coeff, dt_theta, shat_scale;
  double* m_inv_diag;
  double* a_inv_diag;
  double lambda_lo, lambda_hi;
  hier_t h;
  int ssor;          /* cheby_precond == "ssor" (precond.hpp:156-161) */
  ssor_t m_sw, a_sw; /* SsorSweeps(M, 1), SsorSweeps(a_mat, 1) */
} port_ctx;

/* compute_c (precond.hpp:31-38) */
static int compute_c(double dt, double theta, double sigma, double* c) {
  if (!(dt > 0.0)) FAIL(OKO_EINVAL, "compute_c: dt must be positive");
  if (!(theta > 0.0) || theta > 1.0) FAIL(OKO_EINVAL, "compute_c: theta must lie in (0, 1]");
  if (sigma < 0.0) FAIL(OKO_EINVAL, "compute_c: sigma must be nonnegative");
  *c = dt * theta / (1.0 + dt * theta * sigma);
  return OKO_OK;
}

/* chebyshev_semi_iteration (krylov.hpp:158-202) with Jacobi P_inv (precond.hpp:99-119) */
/* z = P^{-1} r: Jacobi (inv_diag) or SSOR (sw, with scratch t) -- cheby_mass_solve,
 * precond.hpp:99-119 */
static void precond_apply(const double* inv_diag, const ssor_t* sw, const double* r, double* z, double* t,
                          long n) {
  if (sw) ssor_apply_inv(sw, r, z, t);
  else
    for (long i = 0; i < n; ++i) z[i] = r[i] * inv_diag[i];
}

static int chebyshev(const csr* A, const double* inv_diag, const ssor_t* sw, const double* b, int k, double lmin,
                     double lmax, double* x) {
  const long n = A->nr;
  if (lmin <= 0.0) FAIL(OKO_EINVAL, "chebyshev: lambda_min must be positive");
  if (lmax < lmin) FAIL(OKO_EINVAL, "chebyshev: bounds out of order");
  if (k < 1) FAIL(OKO_EINVAL, "chebyshev: need at least one step");
  if (!all_finite(b, n)) FAIL(OKO_EINVAL, "chebyshev rhs: vector contains NaN/Inf");
  const double theta = 0.5 * (lmax + lmin);
  const double delta = 0.5 * (lmax - lmin);
  memset(x, 0, (size_t)n * sizeof(double));
  double* r = dcopy(b, n);
  double* z = dalloc(n);
  double* d = dalloc(n);
  double* Ad = dalloc(n);
  double* t = dalloc(n);
  precond_apply(inv_diag, sw, r, z, t, n);
  for (long i = 0; i < n; ++i) d[i] = z[i] * (1.0 / theta);
  if (delta <= 1e-300) {
    for (int j = 0; j < k; ++j) {
      axpy(1.0, d, x, n);
      spmv(A, d, Ad);
      axpy(-1.0, Ad, r, n);
      precond_apply(inv_diag, sw, r, z, t, n);
      for (long i = 0; i < n; ++i) d[i] = z[i] * (1.0 / theta);
    }
  } else {
    const double sigma1 = theta / delta;
    double rho = 1.0 / sigma1;
    for (int j = 0; j < k; ++j) {
      axpy(1.0, d, x, n);
      if (j + 1 == k) break;
      spmv(A, d, Ad);
      axpy(-1.0, Ad, r, n);
      precond_apply(inv_diag, sw, r, z, t, n);
      const double rho_next = 1.0 / (2.0 * sigma1 - rho);
      for (long i = 0; i < n; ++i) d[i] = rho_next * rho * d[i] + 2.0 * rho_next / delta * z[i];
      rho = rho_next;
    }
  }
  free(r);
  free(z);
  free(d);
  free(Ad);
  free(t);
  return OKO_OK;
}

static int apply_M_inv(port_ctx* c, const double* r, double* x) {
  return chebyshev(&c->M, c->m_inv_diag, c->ssor ? &c->m_sw : NULL, r, c->p.cheby_iters, c->lambda_lo,
                   c->lambda_hi, x);
}
static int apply_A_inv(port_ctx* c, const double* r, double* x) {
  return chebyshev(&c->A, c->a_inv_diag, c->ssor ? &c->a_sw : NULL, r, c->p.cheby_iters, c->lambda_lo,
                   c->lambda_hi, x);
}

/* apply_schur_tilde_inv (precond.hpp:199-205) */
static void apply_schur_tilde_inv(port_ctx* c, const double* r, double* x) {
  const long n = c->mesh.nv;
  double* y = dalloc(n);
  double* t = dalloc(n);
  apply_shat_inv(&c->h, r, c->p.mg_cycles, c->p.mg_pre, c->p.mg_post, y);
  spmv(&c->M, y, t);
  apply_shat_inv(&c->h, t, c->p.mg_cycles, c->p.mg_pre, c->p.mg_post, x);
  free(y);
  free(t);
}

/* apply_schur (precond.hpp:210-222) */
static int apply_schur(port_ctx* c, const double* v, double* out) {
  if (!c->have_me) FAIL(OKO_EINCONSISTENT, "schur action: linearized double-well block is not set");
  const long n = c->mesh.nv;
  double* kv = dalloc(n);
  double* z = dalloc(n);
  double* kz = dalloc(n);
  double* mez = dalloc(n);
  spmv(&c->K, v, kv);
  int st = apply_M_inv(c, kv, z);
  if (st == OKO_OK) {
    spmv(&c->M, v, out);
    spmv(&c->K, z, kz);
    axpy(c->eps * c->eps * c->c, kz, out, n);
    spmv(&c->Me, z, mez);
    axpy(c->c, mez, out, n);
  }
  free(kv);
  free(z);
  free(kz);
  free(mez);
  return st;
}

/* apply_S_inv_approx = richardson(S, S~^-1, r, k) (precond.hpp:227-241, krylov.hpp:225-242) */
static int apply_S_inv_approx(port_ctx* c, const double* b, double* x) {
  const long n = c->mesh.nv;
  const int k = c->p.richardson_steps;
  if (k < 1) FAIL(OKO_EINVAL, "schur solve: need at least one refinement step");
  if (!all_finite(b, n)) FAIL(OKO_EINVAL, "richardson rhs: vector contains NaN/Inf");
  memset(x, 0, (size_t)n * sizeof(double));
  double* r = dcopy(b, n);
  double* z = dalloc(n);
  double* Ax = dalloc(n);
  int st = OKO_OK;
  for (int j = 0; j < k; ++j) {
    apply_schur_tilde_inv(c, r, z);
    axpy(1.0, z, x, n);
    if (j + 1 == k) break;
    st = apply_schur(c, x, Ax);
    if (st != OKO_OK) break;
    memcpy(r, b, (size_t)n * sizeof(double));
    axpy(-1.0, Ax, r, n);
  }
  free(r);
  free(z);
  free(Ax);
  return st;
}

/* apply_C (precond.hpp:244-253) */
static int apply_C(port_ctx* c, const double* v, double* out) {
  if (!c->have_me) FAIL(OKO_EINCONSISTENT, "constraint block: linearized double-well block is not set");
  const long n = c->mesh.nv;
  spmv(&c->K, v, out);
  scal(-c->eps * c->eps, out, n);
  double* mev = dalloc(n);
  spmv(&c->Me, v, mev);
  axpy(-1.0, mev, out, n);
  free(mev);
  return OKO_OK;
}

/* apply_block (precond.hpp:257-271) */
static int apply_block(port_ctx* c, const double* r, double* out) {
  const long n = c->mesh.nv;
  double* r2 = dcopy(r + n, n);
  double* cdu = dalloc(n);
  int st = apply_A_inv(c, r, out);
  if (st == OKO_OK) st = apply_C(c, out, cdu);
  if (st == OKO_OK) {
    axpy(-1.0, cdu, r2, n);
    st = apply_S_inv_approx(c, r2, out + n);
  }
  free(r2);
  free(cdu);
  return st;
}

/* jacobian_operator (precond.hpp:277-298) */
static int apply_jacobian(port_ctx* c, const double* x, double* y) {
  if (!c->have_me) FAIL(OKO_EINCONSISTENT, "jacobian apply: linearized double-well block is not set");
  const long n = c->mesh.nv;
  double* kdw = dalloc(n);
  double* mdw = dalloc(n);
  spmv(&c->A, x, y);
  spmv(&c->K, x + n, kdw);
  axpy(c->dt_theta, kdw, y, n);
  apply_C(c, x, y + n);
  spmv(&c->M, x + n, mdw);
  axpy(1.0, mdw, y + n, n);
  free(kdw);
  free(mdw);
  return OKO_OK;
}

/* ---- krylov.hpp:44-152 GMRES ------------------------------------------------ */
static void apply_givens(double c, double s, double* a, double* b) {
  const double t = c * *a + s * *b;
  *b = -s * *a + c * *b;
  *a = t;
}

typedef struct {
  int iterations, converged, stagnated;
  double final_residual;
  double* norms;
  int nnorms, cap;
} kres_t;

static void push_norm(kres_t* k, double v) {
  if (k->nnorms == k->cap) {
    k->cap = k->cap ? 2 * k->cap : 64;
    k->norms = (double*)realloc(k->norms, (size_t)k->cap * sizeof(double));
  }
  k->norms[k->nnorms++] = v;
}

static int gmres(port_ctx* c, const double* b, double rel_tol, int max_iter, int restart,
                 double* x, kres_t* res) {
  const long n = 2 * c->mesh.nv;
  memset(res, 0, sizeof *res);
  if (!all_finite(b, n)) FAIL(OKO_EINVAL, "gmres rhs: vector contains NaN/Inf");
  memset(x, 0, (size_t)n * sizeof(double));
  const double norm_b = norm2(b, n);
  push_norm(res, norm_b);
  if (norm_b == 0.0) {
    res->converged = 1;
    return OKO_OK;
  }
  const double target = rel_tol * norm_b;
  const int cycle_len = restart > 0 ? (restart < max_iter ? restart : max_iter) : max_iter;
  double* r = dcopy(b, n);
  double beta = norm_b;
  double** V = (double**)calloc((size_t)cycle_len + 2, sizeof(double*));
  double** H = (double**)calloc((size_t)cycle_len + 2, sizeof(double*));
  double* cs = dalloc(cycle_len + 2);
  double* sn = dalloc(cycle_len + 2);
  double* g = dalloc(cycle_len + 2);
  double* z = dalloc(n);
  double* w = dalloc(n);
  double* u = dalloc(n);
  double* Ax = dalloc(n);
  int st = OKO_OK;
  while (res->iterations < max_iter) {
    int nV = 0;
    V[nV] = dalloc(n);
    for (long i = 0; i < n; ++i) V[nV][i] = r[i] * (1.0 / beta);
    nV++;
    int ng = 1;
    g[0] = beta;
    int j = 0, breakdown = 0;
    while (j < cycle_len && res->iterations < max_iter) {
      if ((st = apply_block(c, V[j], z)) != OKO_OK) goto done;
      if ((st = apply_jacobian(c, z, w)) != OKO_OK) goto done;
      const double w_scale = norm2(w, n);
      double* h = dalloc(j + 2);
      for (int i = 0; i <= j; ++i) {
        h[i] = dot(w, V[i], n);
        axpy(-h[i], V[i], w, n);
      }
      for (int i = 0; i <= j; ++i) {
        const double cc = dot(w, V[i], n);
        h[i] += cc;
        axpy(-cc, V[i], w, n);
      }
      const double arnoldi_norm = norm2(w, n);
      h[j + 1] = arnoldi_norm;
      for (int i = 0; i < j; ++i) apply_givens(cs[i], sn[i], &h[i], &h[i + 1]);
      const double denom = hypot(h[j], h[j + 1]);
      if (denom == 0.0) {
        free(h);
        breakdown = 1;
        break;
      }
      const double cg = h[j] / denom, sg = h[j + 1] / denom;
      h[j] = denom;
      cs[j] = cg;
      sn[j] = sg;
      g[ng++] = 0.0;
      apply_givens(cg, sg, &g[j], &g[j + 1]);
      H[j] = h;
      ++res->iterations;
      ++j;
      const double est = fabs(g[j]);
      push_norm(res, est);
      if (est <= target) break;
      if (arnoldi_norm <= 1e-13 * w_scale) {
        breakdown = 1;
        break;
      }
      V[nV] = dalloc(n);
      for (long i = 0; i < n; ++i) V[nV][i] = w[i] * (1.0 / arnoldi_norm);
      nV++;
    }
    double* y = dalloc(j + 1);
    for (int i = j - 1; i >= 0; --i) {
      double s = g[i];
      for (int k = i + 1; k < j; ++k) s -= H[k][i] * y[k];
      y[i] = H[i][i] != 0.0 ? s / H[i][i] : 0.0;
    }
    memset(u, 0, (size_t)n * sizeof(double));
    for (int i = 0; i < j; ++i) axpy(y[i], V[i], u, n);
    free(y);
    if ((st = apply_block(c, u, z)) != OKO_OK) goto done;
    axpy(1.0, z, x, n);
    if ((st = apply_jacobian(c, x, Ax)) != OKO_OK) goto done;
    memcpy(r, b, (size_t)n * sizeof(double));
    axpy(-1.0, Ax, r, n);
    beta = norm2(r, n);
    res->final_residual = beta;
    for (int i = 0; i < nV; ++i) {
      free(V[i]);
      V[i] = NULL;
    }
    for (int i = 0; i < j; ++i) {
      free(H[i]);
      H[i] = NULL;
    }
    if (beta <= target * (1.0 + 1e-9)) {
      res->converged = 1;
      break;
    }
    if (breakdown) {
      res->stagnated = 1;
      break;
    }
    if (restart <= 0) break;
  }
done:
  for (int i = 0; i < cycle_len + 2; ++i) {
    free(V[i]);
    free(H[i]);
  }
  free(V);
  free(H);
  free(cs);
  free(sn);
  free(g);
  free(z);
  free(w);
  free(u);
  free(Ax);
  free(r);
  return st;
}

/* ---- model.hpp ---------------------------------------------------------------- */
/* residual (model.hpp:121-148) */
static void residual(port_ctx* c, const double* un, const double* wn, const double* uo,
                     const double* wo, double* r1, double* r2) {
  const long n = c->mesh.nv;
  const oko_params* p = &c->p;
  double* f = dalloc(n);
  double* mu = dalloc(n);
  double* du = dcopy(un, n);
  double* ku = dalloc(n);
  double* nl = dalloc(n);
  axpy(-1.0, uo, du, n);
  spmv(&c->M, du, r1);
  /* flux(next) */
  spmv(&c->K, wn, f);
  spmv(&c->M, un, mu);
  axpy(-p->m, c->b, mu, n);
  axpy(p->sigma, mu, f, n);
  axpy(p->dt * p->theta, f, r1, n);
  /* flux(old) */
  spmv(&c->K, wo, f);
  spmv(&c->M, uo, mu);
  axpy(-p->m, c->b, mu, n);
  axpy(p->sigma, mu, f, n);
  axpy(p->dt * (1.0 - p->theta), f, r1, n);
  spmv(&c->M, wn, r2);
  spmv(&c->K, un, ku);
  axpy(-p->eps * p->eps, ku, r2, n);
  assemble_nonlinear(&c->mesh, un, nl);
  axpy(-1.0, nl, r2, n);
  free(f);
  free(mu);
  free(du);
  free(ku);
  free(nl);
}

static double stacked_norm(const double* r1, const double* r2, long n) {
  const double a = norm2(r1, n), b = norm2(r2, n);
  return sqrt(a * a + b * b);
}

static int set_linearization(port_ctx* c, const double* u) {
  if (c->have_me) csr_free(&c->Me);
  c->have_me = 0;
  TRY(assemble_coefficient_mass(&c->mesh, u, &c->Me));
  c->have_me = 1;
  return OKO_OK;
}

/* newton_solve (model.hpp:165-215) */
static int newton_solve(port_ctx* c, const double* uo, const double* wo, double* un, double* wn,
                        int* newton_iters, int* gmres_iters, double* rnorm_out, double* secs,
                        int* converged) {
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  const long n = c->mesh.nv;
  const oko_params* p = &c->p;
  memcpy(un, uo, (size_t)n * sizeof(double));
  memcpy(wn, wo, (size_t)n * sizeof(double));
  double* r1 = dalloc(n);
  double* r2 = dalloc(n);
  double* rhs = dalloc(2 * n);
  double* x = dalloc(2 * n);
  residual(c, un, wn, uo, wo, r1, r2);
  double rnorm = stacked_norm(r1, r2, n);
  const double ref = rnorm > 1.0 ? rnorm : 1.0;
  int done = rnorm <= p->newton_tol * ref;
  int iters = 0, st = OKO_OK;
  while (!done && iters < p->newton_maxit) {
    if ((st = set_linearization(c, un)) != OKO_OK) break;
    residual(c, un, wn, uo, wo, r1, r2);
    for (long i = 0; i < n; ++i) rhs[i] = -r1[i];
    for (long i = 0; i < n; ++i) rhs[n + i] = -r2[i];
    kres_t kr;
    st = gmres(c, rhs, p->gmres_tol, p->gmres_maxit, p->gmres_restart, x, &kr);
    free(kr.norms);
    if (st != OKO_OK) break;
    gmres_iters[iters] = kr.iterations;
    if (!all_finite(x, 2 * n)) {
      st = OKO_EINVAL;
      snprintf(g_err, sizeof g_err, "newton update: vector contains NaN/Inf");
      break;
    }
    for (long i = 0; i < n; ++i) un[i] += x[i];
    for (long i = 0; i < n; ++i) wn[i] += x[n + i];
    ++iters;
    residual(c, un, wn, uo, wo, r1, r2);
    rnorm = stacked_norm(r1, r2, n);
    done = rnorm <= p->newton_tol * ref;
  }
  if (c->have_me) {
    csr_free(&c->Me);
    c->have_me = 0;
  }
  free(r1);
  free(r2);
  free(rhs);
  free(x);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  *newton_iters = iters;
  *rnorm_out = rnorm;
  *converged = done;
  *secs = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  return st;
}

/* ---- C interface ------------------------------------------------------------ */
void oko_default_params(oko_params* p) {
  /* SolverConfig defaults, params.hpp:14-54 */
  p->dim = 2;
  p->n = 64;
  p->eps = 0.02;
  p->sigma = 100.0;
  p->m = 0.4;
  p->theta = 0.5;
  p->dt = 4.0e-4;
  p->newton_tol = 1e-8;
  p->newton_maxit = 20;
  p->gmres_tol = 1e-6;
  p->gmres_maxit = 200;
  p->gmres_restart = 0;
  p->cheby_iters = 10;
  p->richardson_steps = 2;
  p->mg_cycles = 5;
  p->mg_pre = 2;
  p->mg_post = 2;
  p->mg_omega = 2.0 / 3.0;
  p->min_coarse_size = 500;
  p->shat_perturb = 0.0;
  p->cheby_ssor = 0;
}

static void ctx_free(port_ctx* c) {
  mesh_free(&c->mesh);
  csr_free(&c->M);
  csr_free(&c->K);
  csr_free(&c->A);
  if (c->have_me) csr_free(&c->Me);
  free(c->b);
  free(c->m_inv_diag);
  free(c->a_inv_diag);
  free(c->m_sw.diag);
  free(c->a_sw.diag);
  hier_free(&c->h);
  free(c);
}

static int positive_inverse_diagonal(const csr* A, double** out) {
  *out = dalloc(A->nr);
  csr_diag(A, *out);
  for (int i = 0; i < A->nr; ++i) {
    if (!((*out)[i] > 0.0)) FAIL(OKO_ENUMERICAL, "mass preconditioner: non-positive diagonal entry");
    (*out)[i] = 1.0 / (*out)[i];
  }
  return OKO_OK;
}

/* build_mesh + assemble_operators + make_schur_context (precond.hpp:126-181) */
static int create(const oko_params* p, port_ctx* c) {
  c->p = *p;
  TRY(build_mesh(p->dim, p->n, &c->mesh));
  TRY(assemble_mass(&c->mesh, &c->M));
  TRY(assemble_stiffness(&c->mesh, &c->K));
  c->b = dalloc(c->mesh.nv);
  assemble_load(&c->mesh, c->b);
  if (!(p->eps > 0.0)) FAIL(OKO_EINVAL, "schur context: eps must be positive");
  const double scale_factor = 1.0 + p->shat_perturb;
  if (!(scale_factor > 0.0))
    FAIL(OKO_EINVAL, "schur context: perturbation must keep the shifted operator positive");
  TRY(compute_c(p->dt, p->theta, p->sigma, &c->c));
  c->eps = p->eps;
  c->sqrt_c = sqrt(c->c);
  c->a_coeff = 1.0 + p->dt * p->theta * p->sigma;
  c->dt_theta = p->dt * p->theta;
  c->shat_scale = scale_factor;
  csr_scale(&c->M, c->a_coeff, &c->A);
  c->ssor = p->cheby_ssor != 0;
  if (c->ssor) {  /* precond.hpp:156-161 */
    TRY(estimate_ssor_spectrum(&c->M, 1.0, &c->lambda_lo, &c->lambda_hi));
    TRY(ssor_init(&c->M, 1.0, &c->m_sw));
    TRY(ssor_init(&c->A, 1.0, &c->a_sw));
  } else {
    TRY(estimate_jacobi_spectrum(&c->M, &c->lambda_lo, &c->lambda_hi));
  }
  TRY(positive_inverse_diagonal(&c->M, &c->m_inv_diag));
  TRY(positive_inverse_diagonal(&c->A, &c->a_inv_diag));
  TRY(build_hierarchy(&c->mesh, &c->M, &c->K, c->shat_scale * c->eps * c->sqrt_c,
                      p->min_coarse_size, p->mg_omega, &c->h));
  return OKO_OK;
}

void* oko_create(const oko_params* p, int* status) {
  port_ctx* c = (port_ctx*)calloc(1, sizeof(port_ctx));
  int st = create(p, c);
  if (status) *status = st;
  if (st != OKO_OK) {
    ctx_free(c);
    return NULL;
  }
  return c;
}

void oko_destroy(void* ctx) {
  if (ctx) ctx_free((port_ctx*)ctx);
}

long oko_num_vertices(void* ctx) { return ((port_ctx*)ctx)->mesh.nv; }
int oko_levels(void* ctx) { return ((port_ctx*)ctx)->h.levels; }
long oko_level_size(void* ctx, int level) {
  port_ctx* c = (port_ctx*)ctx;
  if (level < 0 || level >= c->h.levels) return -1;
  return c->h.ops[level].nr;
}
int oko_scalars(void* ctx, double* out) {
  port_ctx* c = (port_ctx*)ctx;
  out[0] = c->c;
  out[1] = c->sqrt_c;
  out[2] = c->a_coeff;
  out[3] = c->dt_theta;
  out[4] = c->lambda_lo;
  out[5] = c->lambda_hi;
  out[6] = c->shat_scale * c->eps * c->sqrt_c;
  return OKO_OK;
}
int oko_load_vector(void* ctx, double* b) {
  port_ctx* c = (port_ctx*)ctx;
  memcpy(b, c->b, (size_t)c->mesh.nv * sizeof(double));
  return OKO_OK;
}
int oko_level_dense(void* ctx, int level, double* A) {
  port_ctx* c = (port_ctx*)ctx;
  if (level < 0 || level >= c->h.levels) FAIL(OKO_EINVAL, "level out of range");
  const csr* S = &c->h.ops[level];
  memset(A, 0, (size_t)S->nr * S->nc * sizeof(double));
  for (int i = 0; i < S->nr; ++i)
    for (int k = S->rp[i]; k < S->rp[i + 1]; ++k) A[(long)i * S->nc + S->ci[k]] = S->v[k];
  return OKO_OK;
}
int oko_mesh(int dim, int n, double* vertices, int* cells) {
  mesh_t m;
  TRY(build_mesh(dim, n, &m));
  memcpy(vertices, m.vert, (size_t)m.nv * dim * sizeof(double));
  memcpy(cells, m.cells, (size_t)m.ncell * (dim + 1) * sizeof(int));
  mesh_free(&m);
  return OKO_OK;
}
int oko_set_linearization(void* ctx, const double* u) { return set_linearization((port_ctx*)ctx, u); }

int oko_apply(void* ctx, int kind, int level, const double* x, double* y) {
  port_ctx* c = (port_ctx*)ctx;
  const hier_t* h = &c->h;
  switch (kind) {
    case OKO_M: spmv(&c->M, x, y); return OKO_OK;
    case OKO_K: spmv(&c->K, x, y); return OKO_OK;
    case OKO_A: spmv(&c->A, x, y); return OKO_OK;
    case OKO_SHAT:
      if (level < 0 || level >= h->levels) FAIL(OKO_EINVAL, "level out of range");
      spmv(&h->ops[level], x, y);
      return OKO_OK;
    case OKO_PROLONG:
      if (level < 0 || level + 1 >= h->levels) FAIL(OKO_EINVAL, "level out of range");
      spmv(&h->prolong[level], x, y);
      return OKO_OK;
    case OKO_RESTRICT:
      if (level < 0 || level + 1 >= h->levels) FAIL(OKO_EINVAL, "level out of range");
      spmv_t(&h->prolong[level], x, y);
      return OKO_OK;
    case OKO_VCYCLE: mg_cycle(h, 0, x, c->p.mg_pre, c->p.mg_post, y); return OKO_OK;
    case OKO_SHAT_INV:
      apply_shat_inv(h, x, c->p.mg_cycles, c->p.mg_pre, c->p.mg_post, y);
      return OKO_OK;
    case OKO_CHEB_M: return apply_M_inv(c, x, y);
    case OKO_CHEB_A: return apply_A_inv(c, x, y);
    case OKO_ME:
      if (!c->have_me) FAIL(OKO_EINCONSISTENT, "Me not set");
      spmv(&c->Me, x, y);
      return OKO_OK;
    case OKO_C: return apply_C(c, x, y);
    case OKO_SCHUR: return apply_schur(c, x, y);
    case OKO_SCHUR_TILDE_INV: apply_schur_tilde_inv(c, x, y); return OKO_OK;
    case OKO_S_INV_APPROX: return apply_S_inv_approx(c, x, y);
    case OKO_BLOCK: return apply_block(c, x, y);
    case OKO_JACOBIAN: return apply_jacobian(c, x, y);
    case OKO_NONLINEAR: assemble_nonlinear(&c->mesh, x, y); return OKO_OK;
    case OKO_COARSE_SOLVE: chol_solve(&h->coarse, x, y); return OKO_OK;
    case OKO_SSOR_M: {
      ssor_t sw;
      TRY(ssor_init(&c->M, 1.0, &sw));
      double* t = dalloc(c->mesh.nv);
      ssor_apply_inv(&sw, x, y, t);
      free(t);
      free(sw.diag);
      return OKO_OK;
    }
    default: FAIL(OKO_EINVAL, "oko_apply: unknown kind");
  }
}

int oko_residual(void* ctx, const double* u_next, const double* w_next, const double* u_old,
                 const double* w_old, double* r1, double* r2) {
  residual((port_ctx*)ctx, u_next, w_next, u_old, w_old, r1, r2);
  return OKO_OK;
}

int oko_gmres(void* ctx, const double* b, double* x, double rtol, int maxit, int restart,
              int* iterations, double* final_residual, int* converged, int* stagnated,
              double* residual_norms, int residual_norms_cap, int* n_residual_norms) {
  kres_t k;
  int st = gmres((port_ctx*)ctx, b, rtol, maxit, restart, x, &k);
  *iterations = k.iterations;
  *final_residual = k.final_residual;
  *converged = k.converged;
  *stagnated = k.stagnated;
  if (n_residual_norms) *n_residual_norms = k.nnorms;
  if (residual_norms)
    for (int i = 0; i < k.nnorms && i < residual_norms_cap; ++i) residual_norms[i] = k.norms[i];
  free(k.norms);
  return st;
}

int oko_newton_solve(void* ctx, const double* u_old, const double* w_old, double* u_next,
                     double* w_next, int* newton_iters, int* gmres_iters, double* residual_norm,
                     double* seconds, int* converged) {
  return newton_solve((port_ctx*)ctx, u_old, w_old, u_next, w_next, newton_iters, gmres_iters,
                      residual_norm, seconds, converged);
}

int oko_jacobi_spectrum(void* ctx, double* lo, double* hi) {
  return estimate_jacobi_spectrum(&((port_ctx*)ctx)->M, lo, hi);
}

/* SURVEY.md section 8(d) seeded IC (builder-defined; the reference has none) */
void oko_seeded_ic(long nverts, unsigned long long seed, double m, double* u) {
  for (long g = 0; g < nverts; ++g) {
    uint64_t x = (uint64_t)seed * 0x9E3779B97F4A7C15ull + (uint64_t)g + 0x632BE59BD9B4E019ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x = x ^ (x >> 31);
    const double U = 2.0 * ((double)(x >> 11) * 0x1.0p-53) - 1.0;
    u[g] = m + 0.01 * U;
  }
}

/* ---- diagnostics and initial state -------------------------- */

/* conjugate_gradient (krylov.hpp:424-479) with the Jacobi preconditioner of
 * make_jacobi_preconditioner (operator.hpp:53-64: z = r / diag) and an optional
 * unit-norm nullspace vector ns (project: v -= (v . ns) ns) */
static int conjugate_gradient(const csr* A, const double* diag, const double* b, double rel_tol, int max_iter,
                              const double* ns, double* x, int* iters, int* converged) {
  const long n = A->nr;
  if (!all_finite(b, n)) FAIL(OKO_EINVAL, "cg rhs: vector contains NaN/Inf");
  double* r = dcopy(b, n);
  double* z = dalloc(n);
  double* p = dalloc(n);
  double* Ap = dalloc(n);
  memset(x, 0, (size_t)n * sizeof(double));
  *iters = 0;
  *converged = 0;
#define PROJECT(v)                            \
  do {                                        \
    if (ns) axpy(-dot(v, ns, n), ns, v, n);   \
  } while (0)
  PROJECT(r);
  const double norm_b = norm2(r, n);
  int st = OKO_OK;
  if (norm_b == 0.0) {
    *converged = 1;
  } else {
    const double target = rel_tol * norm_b;
    for (long i = 0; i < n; ++i) z[i] = r[i] / diag[i];
    PROJECT(z);
    memcpy(p, z, (size_t)n * sizeof(double));
    double rz = dot(r, z, n);
    for (int it = 0; it < max_iter; ++it) {
      spmv(A, p, Ap);
      const double pAp = dot(p, Ap, n);
      if (pAp <= 0.0) {
        snprintf(g_err, sizeof g_err, "cg: operator not positive definite on iterate");
        st = OKO_ENUMERICAL;
        break;
      }
      const double alpha = rz / pAp;
      axpy(alpha, p, x, n);
      axpy(-alpha, Ap, r, n);
      PROJECT(r);
      ++*iters;
      const double rn = norm2(r, n);
      if (rn <= target) {
        *converged = 1;
        break;
      }
      for (long i = 0; i < n; ++i) z[i] = r[i] / diag[i];
      PROJECT(z);
      const double rz_new = dot(r, z, n);
      const double beta = rz_new / rz;
      rz = rz_new;
      for (long i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
  }
#undef PROJECT
  free(r);
  free(z);
  free(p);
  free(Ap);
  return st;
}

/* integrate_double_well (assembly.hpp:220-245): degree-4 rule, Kahan-compensated cell sum */
static double integrate_double_well(const mesh_t* m, const double* u) {
  quadrule_t q;
  simplex_quadrature(m->dim, 4, &q);
  const int vpc = m->dim + 1;
  const double ref_measure = m->dim == 2 ? 0.5 : 1.0 / 6.0;
  double total = 0.0, comp = 0.0;
  for (long c = 0; c < m->ncell; ++c) {
    const int* cv = m->cells + c * vpc;
    const double scale = cell_volume(m, c) / ref_measure;
    double cell = 0.0;
    for (int p = 0; p < q.np; ++p) {
      const double* bq = q.pts + p * vpc;
      double uq = 0.0;
      for (int k = 0; k < vpc; ++k) uq += u[cv[k]] * bq[k];
      const double w = 1.0 - uq * uq;
      cell += q.w[p] * w * w;
    }
    const double y = cell * scale - comp;
    const double t = total + y;
    comp = (t - total) - y;
    total = t;
  }
  return total;
}

int oko_total_mass(void* ctx, const double* u, double* mass) {
  port_ctx* c = (port_ctx*)ctx;
  *mass = dot(c->b, u, c->mesh.nv); /* model.hpp:46-48 */
  return OKO_OK;
}

int oko_double_well(void* ctx, const double* u, double* value) {
  *value = integrate_double_well(&((port_ctx*)ctx)->mesh, u);
  return OKO_OK;
}

/* energy (model.hpp:56-86) */
int oko_energy(void* ctx, const double* u, double* e, int* cg_iters) {
  port_ctx* c = (port_ctx*)ctx;
  const long n = c->mesh.nv;
  const double eps = c->p.eps, sigma = c->p.sigma, mm = c->p.m;
  double* Ku = dalloc(n);
  spmv(&c->K, u, Ku);
  const double grad_term = 0.5 * eps * eps * dot(u, Ku, n);
  free(Ku);
  const double well_term = 0.25 * integrate_double_well(&c->mesh, u);
  double nonlocal = 0.0;
  if (cg_iters) *cg_iters = 0;
  if (sigma != 0.0) {
    double* rhs = dalloc(n);
    spmv(&c->M, u, rhs);
    axpy(-mm, c->b, rhs, n);
    double mean = 0.0;
    for (long i = 0; i < n; ++i) mean += rhs[i];
    if (fabs(mean) > 1e-6) {
      free(rhs);
      FAIL(OKO_EINCONSISTENT, "energy: potential right-hand side is not mean-zero (|sum| = %f)", fabs(mean));
    }
    double* ones = dalloc(n);
    for (long i = 0; i < n; ++i) ones[i] = 1.0 / sqrt((double)n);
    double* diag = dalloc(n);
    csr_diag(&c->K, diag);
    double* phi = dalloc(n);
    int its = 0, conv = 0;
    const int st = conjugate_gradient(&c->K, diag, rhs, 1e-10, 2000, ones, phi, &its, &conv);
    if (cg_iters) *cg_iters = its;
    if (st == OKO_OK && conv) nonlocal = 0.5 * sigma * dot(phi, rhs, n);
    free(ones);
    free(diag);
    free(phi);
    free(rhs);
    if (st != OKO_OK) return st;
    if (!conv) FAIL(OKO_ENUMERICAL, "energy: potential solve did not converge");
  }
  *e = grad_term + well_term + nonlocal;
  return OKO_OK;
}

/* initial_state (model.hpp:93-114) */
int oko_initial_state(void* ctx, double* u, double* w, int* cg_iters) {
  port_ctx* c = (port_ctx*)ctx;
  const mesh_t* m = &c->mesh;
  const long n = m->nv;
  const double kPi = 3.14159265358979323846;
  for (long v = 0; v < n; ++v) {
    const double x = m->vert[v * m->dim], y = m->vert[v * m->dim + 1];
    const double z = m->dim == 3 ? m->vert[v * m->dim + 2] : 0.0;
    u[v] = c->p.m + cos(2.0 * kPi * x) * cos(2.0 * kPi * y) * cos(2.0 * kPi * z) / 50.0;
  }
  double* rhs = dalloc(n);
  spmv(&c->K, u, rhs);
  scal(c->p.eps * c->p.eps, rhs, n);
  double* nl = dalloc(n);
  assemble_nonlinear(m, u, nl);
  axpy(1.0, nl, rhs, n);
  free(nl);
  double* diag = dalloc(n);
  csr_diag(&c->M, diag);
  int its = 0, conv = 0;
  const int st = conjugate_gradient(&c->M, diag, rhs, 1e-12, 1000, NULL, w, &its, &conv);
  if (cg_iters) *cg_iters = its;
  free(diag);
  free(rhs);
  if (st != OKO_OK) return st;
  if (!conv) FAIL(OKO_ENUMERICAL, "initial_state: mass solve did not converge");
  return OKO_OK;
}
