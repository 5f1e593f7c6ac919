// Host tridiagonal eigensolver for SLQ quadrature (K12 in SURVEY.md §2.6).
//
// P:312-316 (§4): v^T f(H) v ~= e_1^T f(T_m) e_1, i.e. Gauss quadrature with nodes = eigenvalues
// of T_m and weights = squared first components of its normalised eigenvectors (Golub-Welsch).
// Implicit-shift QL with Wilkinson shifts on the symmetric tridiagonal T_m; only the first row of
// the eigenvector matrix is accumulated (m <= a few hundred, microseconds on the host).  The
// iteration follows the textbook tridiagonal QL algorithm as presented in Press et al.,
// "Numerical Recipes" (routine tqli; variable names d, e, z, g, r, s, c, p, f, b as there), the
// standard host-side companion of Golub-Welsch; the oracle uses an independent cyclic Jacobi.
#include <math.h>

#include <algorithm>
#include <numeric>
#include <vector>

#include "common.h"

namespace slq {

void tridiag_gauss(const double* alpha, const double* beta, int m, double* nodes, double* weights) {
  SLQ_CHECK_ARG(m >= 1, "m >= 1");
  SLQ_CHECK_ARG(alpha && nodes && weights, "null pointer");
  SLQ_CHECK_ARG(m == 1 || beta, "beta required for m > 1");
  std::vector<double> d(alpha, alpha + m), e(m, 0.0), z(m, 0.0);
  for (int i = 0; i + 1 < m; ++i) e[i] = beta[i];
  for (int i = 0; i < m; ++i) {
    if (!std::isfinite(d[i]) || !std::isfinite(e[i])) throw Error(SLQ_EINVAL, "non-finite alpha/beta");
  }
  z[0] = 1.0;
  const double tiny = 2.220446049250313e-16;
  for (int l = 0; l < m; ++l) {
    int iter = 0;
    int mm;
    do {
      for (mm = l; mm < m - 1; ++mm) {
        const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(e[mm]) <= tiny * dd) break;
      }
      if (mm != l) {
        if (++iter > 200) throw Error(SLQ_ENUMERIC, "tridiagonal QL did not converge");
        // Wilkinson-type shift from the leading 2x2 block
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[mm] - d[l] + e[l] / (g + (g >= 0 ? fabs(r) : -fabs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool deflated = false;
        for (i = mm - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {  // underflow: split and restart this block
            d[i + 1] -= p;
            e[mm] = 0.0;
            deflated = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          // rotate the first row of the eigenvector matrix
          f = z[i + 1];
          z[i + 1] = s * z[i] + c * f;
          z[i] = c * z[i] - s * f;
        }
        if (deflated) continue;
        d[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    } while (mm != l);
  }
  std::vector<int> idx(m);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return d[a] < d[b]; });
  for (int i = 0; i < m; ++i) {
    nodes[i] = d[idx[i]];
    weights[i] = z[idx[i]] * z[idx[i]];
  }
}

// Ghost clusters (R18): single linkage on the ascending Ritz values.
void ghost_clusters(const double* nodes, int m, double tol, int32_t* cluster_id, int32_t* n_ghost, double* max_split) {
  SLQ_CHECK_ARG(m >= 1 && nodes, "nodes[m], m >= 1");
  SLQ_CHECK_ARG(tol >= 0 && std::isfinite(tol), "tol >= 0");
  for (int i = 0; i < m; ++i) {
    SLQ_CHECK_ARG(std::isfinite(nodes[i]), "finite nodes");
    SLQ_CHECK_ARG(i == 0 || nodes[i] >= nodes[i - 1], "nodes ascending");
  }
  int id = 0, start = 0, ghosts = 0;
  double split = 0.0;
  auto close_cluster = [&](int end) {  // members [start, end)
    if (end - start >= 2) {
      ++ghosts;
      split = std::max(split, nodes[end - 1] - nodes[start]);
    }
  };
  for (int i = 0; i < m; ++i) {
    if (i > 0 && nodes[i] - nodes[i - 1] > tol) {
      close_cluster(i);
      ++id;
      start = i;
    }
    if (cluster_id) cluster_id[i] = id;
  }
  close_cluster(m);
  if (n_ghost) *n_ghost = ghosts;
  if (max_split) *max_split = split;
}

// Probe-averaged SLQ moments and smoothed density.
void slq_average(const double* nodes, const double* weights, const int32_t* mc, int np, int jmax, double* mom,
                 const double* grid, int ng, double sigma, double* dens) {
  SLQ_CHECK_ARG(nodes && weights && mc && np >= 1, "nodes / weights / m_counts, n_probes >= 1");
  SLQ_CHECK_ARG(!mom || jmax >= 0, "jmax >= 0");
  SLQ_CHECK_ARG(!dens || (grid && ng >= 1 && sigma > 0 && std::isfinite(sigma)), "grid / n_grid / sigma > 0");
  if (mom)
    for (int j = 0; j <= jmax; ++j) mom[j] = 0.0;
  if (dens)
    for (int g = 0; g < ng; ++g) dens[g] = 0.0;
  const double norm = 1.0 / (sigma * sqrt(2.0 * M_PI));
  int64_t off = 0;
  for (int p = 0; p < np; ++p) {
    SLQ_CHECK_ARG(mc[p] >= 1, "m_counts >= 1");
    for (int i = 0; i < mc[p]; ++i) {
      const double x = nodes[off + i], w = weights[off + i];
      SLQ_CHECK_ARG(std::isfinite(x) && std::isfinite(w), "finite nodes / weights");
      if (mom) {
        double xp = 1.0;
        for (int j = 0; j <= jmax; ++j) {
          mom[j] += w * xp;
          xp *= x;
        }
      }
      if (dens)
        for (int g = 0; g < ng; ++g) {
          const double u = (grid[g] - x) / sigma;
          dens[g] += w * exp(-0.5 * u * u) * norm;
        }
    }
    off += mc[p];
  }
  if (mom)
    for (int j = 0; j <= jmax; ++j) mom[j] /= np;
  if (dens)
    for (int g = 0; g < ng; ++g) dens[g] /= np;
}

}  // namespace slq
