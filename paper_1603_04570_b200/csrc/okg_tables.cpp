// okg_tables.cpp -- see okg_tables.h.
#include "okg_tables.h"

#include <algorithm>
#include <cmath>

namespace okg {

namespace {

// stencil slot of offset (dx,dy[,dz]) -- ascending linear order, see okg_common.cuh
int slot_of(int dim, const int* o) {
  static const int s2[7][2] = {{-1, -1}, {-1, 0}, {0, -1}, {0, 0}, {0, 1}, {1, 0}, {1, 1}};
  static const int s3[15][3] = {{-1, -1, -1}, {-1, -1, 0}, {-1, 0, -1}, {-1, 0, 0}, {0, -1, -1},
                                {0, -1, 0},   {0, 0, -1},  {0, 0, 0},   {0, 0, 1},  {0, 1, 0},
                                {0, 1, 1},    {1, 0, 0},   {1, 0, 1},   {1, 1, 0},  {1, 1, 1}};
  if (dim == 2) {
    for (int q = 0; q < 7; ++q)
      if (s2[q][0] == o[0] && s2[q][1] == o[1]) return q;
  } else {
    for (int q = 0; q < 15; ++q)
      if (s3[q][0] == o[0] && s3[q][1] == o[1] && s3[q][2] == o[2]) return q;
  }
  return -1;
}

}  // namespace

UnitTables build_unit_tables(int dim) {
  UnitTables t;
  t.dim = dim;
  t.ncls = dim == 2 ? 9 : 27;
  t.noff = dim == 2 ? 7 : 15;
  const int n = 2, s = 3;
  const int nv = dim == 2 ? s * s : s * s * s;
  auto gidx = [&](int i, int j, int k) { return dim == 2 ? i * s + j : (i * s + j) * s + k; };
  std::vector<double> coords(static_cast<size_t>(nv) * dim);
  {
    size_t p = 0;
    if (dim == 2) {
      for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j) {
          coords[p++] = i;
          coords[p++] = j;
        }
    } else {
      for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j)
          for (int k = 0; k < s; ++k) {
            coords[p++] = i;
            coords[p++] = j;
            coords[p++] = k;
          }
    }
  }
  // cells in the reference's order (mesh.hpp:106-148)
  std::vector<int> cells;
  if (dim == 2) {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const int a = gidx(i, j, 0), b = gidx(i + 1, j, 0), c = gidx(i + 1, j + 1, 0), d = gidx(i, j + 1, 0);
        cells.insert(cells.end(), {a, b, c, a, c, d});
      }
  } else {
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    static const bool odd[6] = {false, true, true, false, false, true};
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k) {
          const int base[3] = {i, j, k};
          for (int p = 0; p < 6; ++p) {
            int g[4][3];
            for (int d = 0; d < 3; ++d) g[0][d] = base[d];
            for (int v = 1; v < 4; ++v) {
              for (int d = 0; d < 3; ++d) g[v][d] = g[v - 1][d];
              g[v][perms[p][v - 1]] += 1;
            }
            int idx[4];
            for (int v = 0; v < 4; ++v) idx[v] = gidx(g[v][0], g[v][1], g[v][2]);
            if (odd[p]) std::swap(idx[1], idx[2]);
            cells.insert(cells.end(), {idx[0], idx[1], idx[2], idx[3]});
          }
        }
  }
  const int vpc = dim + 1;
  const int ncell = static_cast<int>(cells.size()) / vpc;
  const double denom = static_cast<double>((dim + 1) * (dim + 2));
  const double inv_vpc = 1.0 / (dim + 1);
  // dense patch matrices; entries accumulate in cell order like from_triplets
  std::vector<double> Md(static_cast<size_t>(nv) * nv, 0.0), Kd(static_cast<size_t>(nv) * nv, 0.0);
  std::vector<char> Mset(static_cast<size_t>(nv) * nv, 0), Kset(static_cast<size_t>(nv) * nv, 0);
  std::vector<double> load(nv, 0.0);
  auto X = [&](int v, int d) { return coords[static_cast<size_t>(v) * dim + d]; };
  for (int c = 0; c < ncell; ++c) {
    const int* cv = &cells[static_cast<size_t>(c) * vpc];
    double vol;
    double grad[12];
    if (dim == 2) {
      // cell_volume (mesh.hpp:52-62) and barycentric_gradients (assembly.hpp:145-165)
      const double ax = X(cv[1], 0) - X(cv[0], 0), ay = X(cv[1], 1) - X(cv[0], 1);
      const double bx = X(cv[2], 0) - X(cv[0], 0), by = X(cv[2], 1) - X(cv[0], 1);
      const double det = ax * by - ay * bx;
      vol = 0.5 * (ax * by - ay * bx);
      grad[2] = by / det;
      grad[3] = -bx / det;
      grad[4] = -ay / det;
      grad[5] = ax / det;
      grad[0] = -(grad[2] + grad[4]);
      grad[1] = -(grad[3] + grad[5]);
    } else {
      double e[3][3];
      for (int k = 1; k <= 3; ++k)
        for (int d = 0; d < 3; ++d) e[k - 1][d] = X(cv[k], d) - X(cv[0], d);
      const double det = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) -
                         e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
                         e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
      vol = det / 6.0;
      const double inv[3][3] = {
          {(e[1][1] * e[2][2] - e[1][2] * e[2][1]) / det, -(e[1][0] * e[2][2] - e[1][2] * e[2][0]) / det,
           (e[1][0] * e[2][1] - e[1][1] * e[2][0]) / det},
          {-(e[0][1] * e[2][2] - e[0][2] * e[2][1]) / det, (e[0][0] * e[2][2] - e[0][2] * e[2][0]) / det,
           -(e[0][0] * e[2][1] - e[0][1] * e[2][0]) / det},
          {(e[0][1] * e[1][2] - e[0][2] * e[1][1]) / det, -(e[0][0] * e[1][2] - e[0][2] * e[1][0]) / det,
           (e[0][0] * e[1][1] - e[0][1] * e[1][0]) / det}};
      for (int k = 1; k <= 3; ++k)
        for (int d = 0; d < 3; ++d) grad[k * 3 + d] = inv[k - 1][d];
      for (int d = 0; d < 3; ++d) grad[d] = -(grad[3 + d] + grad[6 + d] + grad[9 + d]);
    }
    for (int i = 0; i < vpc; ++i)
      for (int j = 0; j < vpc; ++j) {
        const size_t e = static_cast<size_t>(cv[i]) * nv + cv[j];
        const double mv = vol * (i == j ? 2.0 : 1.0) / denom;  // assembly.hpp:94
        double g = 0.0;
        for (int d = 0; d < dim; ++d) g += grad[i * dim + d] * grad[j * dim + d];
        const double kv = vol * g;  // assembly.hpp:120-121
        if (Mset[e]) Md[e] += mv; else { Md[e] = mv; Mset[e] = 1; }
        if (Kset[e]) Kd[e] += kv; else { Kd[e] = kv; Kset[e] = 1; }
      }
    for (int k = 0; k < vpc; ++k) load[cv[k]] += vol * inv_vpc;  // assembly.hpp:133-137
  }
  t.M.assign(static_cast<size_t>(t.ncls) * t.noff, 0.0);
  t.K.assign(static_cast<size_t>(t.ncls) * t.noff, 0.0);
  t.load.assign(t.ncls, 0.0);
  for (int cls = 0; cls < t.ncls; ++cls) {
    int pc[3] = {0, 0, 0};
    if (dim == 2) {
      pc[0] = cls / 3;
      pc[1] = cls % 3;
    } else {
      pc[0] = cls / 9;
      pc[1] = (cls / 3) % 3;
      pc[2] = cls % 3;
    }
    const int p = gidx(pc[0], pc[1], pc[2]);
    t.load[cls] = load[p];
    for (int q = 0; q < nv; ++q) {
      const size_t e = static_cast<size_t>(p) * nv + q;
      if (!Mset[e] && !Kset[e]) continue;
      int qc[3] = {0, 0, 0}, o[3] = {0, 0, 0};
      if (dim == 2) {
        qc[0] = q / 3;
        qc[1] = q % 3;
      } else {
        qc[0] = q / 9;
        qc[1] = (q / 3) % 3;
        qc[2] = q % 3;
      }
      for (int d = 0; d < dim; ++d) o[d] = qc[d] - pc[d];
      const int sl = slot_of(dim, o);
      if (sl < 0) continue;  // not a P1 neighbour (cannot happen)
      t.M[static_cast<size_t>(cls) * t.noff + sl] = Md[e];
      t.K[static_cast<size_t>(cls) * t.noff + sl] = Kd[e];
    }
  }
  return t;
}

bool dense_spd_inverse(const std::vector<double>& A, int n, std::vector<double>& inv) {
  std::vector<double> L(static_cast<size_t>(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = A[static_cast<size_t>(j) * n + j];
    for (int k = 0; k < j; ++k) d -= L[static_cast<size_t>(j) * n + k] * L[static_cast<size_t>(j) * n + k];
    if (d <= 0.0 || !std::isfinite(d)) return false;
    L[static_cast<size_t>(j) * n + j] = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double s = A[static_cast<size_t>(i) * n + j];
      for (int k = 0; k < j; ++k) s -= L[static_cast<size_t>(i) * n + k] * L[static_cast<size_t>(j) * n + k];
      L[static_cast<size_t>(i) * n + j] = s / L[static_cast<size_t>(j) * n + j];
    }
  }
  inv.assign(static_cast<size_t>(n) * n, 0.0);
  std::vector<double> y(n), x(n);
  for (int c = 0; c < n; ++c) {
    for (int i = 0; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int j = 0; j < i; ++j) s -= L[static_cast<size_t>(i) * n + j] * y[j];
      y[i] = s / L[static_cast<size_t>(i) * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int j = i + 1; j < n; ++j) s -= L[static_cast<size_t>(j) * n + i] * x[j];
      x[i] = s / L[static_cast<size_t>(i) * n + i];
    }
    for (int i = 0; i < n; ++i) inv[static_cast<size_t>(i) * n + c] = x[i];
  }
  return true;
}

bool symmetric_eigenvalues(std::vector<double> A, int n, std::vector<double>& ev) {
  const int max_sweeps = 60;
  double ref = 0.0;
  for (int i = 0; i < n * n; ++i) ref += A[i] * A[i];
  ref = std::sqrt(ref);
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) off += A[i * n + j] * A[i * n + j];
    if (std::sqrt(off) <= 1e-14 * ref + 1e-300) break;
    if (sweep == max_sweeps - 1) return false;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (std::abs(apq) <= 1e-300) continue;
        const double tau = (A[q * n + q] - A[p * n + p]) / (2.0 * apq);
        const double tt = tau >= 0.0 ? 1.0 / (tau + std::sqrt(1.0 + tau * tau))
                                     : -1.0 / (-tau + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + tt * tt), s = tt * c;
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
  ev.resize(n);
  for (int i = 0; i < n; ++i) ev[i] = A[i * n + i];
  std::sort(ev.begin(), ev.end());
  return true;
}

}  // namespace okg
