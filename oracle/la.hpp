// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// Dense fp64 linear algebra that stands in for Eigen3 in the reference
// (Eigen is a third-party dependency absent from /root/reference: the
// reference pins only "Eigen3 >= 3.3", proj/CMakeLists.txt:12). Only the
// operations the hot path and its tests use are restated:
//   * row-major dense matrix            (types.hpp:15-19, DenseMatrix)
//   * GEMM                               (factor_state.cpp:121-122,162-163)
//   * thin SVD (one-sided Jacobi)        (svd.cpp:34 BDCSVD, eval.cpp:408 /
//                                         tests/helpers.hpp:57 JacobiSVD)
//   * PartialPivLU + solves              (factor_state.cpp:21-36,199,206,237)
//   * Householder QR, thin Q and R       (svd.cpp:23-28,75-80)
// The SVD algorithm differs from BDCSVD; singular values agree to rounding
// and singular vectors agree up to per-column sign / rotation inside exactly
// degenerate clusters, which is the same freedom the reference's own oracle
// (JacobiSVD vs BDCSVD, acceptance_main.cpp:87-108) relies on.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <vector>

namespace damf_oracle {

using Index = std::int64_t;
using Vec = std::vector<double>;

struct Mat {
  Index r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(Index rows, Index cols, double v = 0.0)
      : r(rows), c(cols), a(static_cast<size_t>(rows * cols), v) {}
  double& operator()(Index i, Index j) { return a[static_cast<size_t>(i * c + j)]; }
  double operator()(Index i, Index j) const { return a[static_cast<size_t>(i * c + j)]; }
  double* row(Index i) { return a.data() + i * c; }
  const double* row(Index i) const { return a.data() + i * c; }
  Index rows() const { return r; }
  Index cols() const { return c; }
  static Mat eye(Index n, Index m) {
    Mat e(n, m);
    for (Index i = 0; i < std::min(n, m); ++i) e(i, i) = 1.0;
    return e;
  }
  static Mat eye(Index n) { return eye(n, n); }
  void append_zero_row() {
    a.resize(static_cast<size_t>((r + 1) * c), 0.0);
    ++r;
  }
  // Append one zero column (reallocates; rare path).
  void append_zero_col() {
    std::vector<double> b(static_cast<size_t>(r * (c + 1)), 0.0);
    for (Index i = 0; i < r; ++i)
      for (Index j = 0; j < c; ++j) b[i * (c + 1) + j] = a[i * c + j];
    a.swap(b);
    ++c;
  }
  double frob() const {
    double s = 0;
    for (double v : a) s += v * v;
    return std::sqrt(s);
  }
  bool all_finite() const {
    for (double v : a)
      if (!std::isfinite(v)) return false;
    return true;
  }
};

inline Mat transpose(const Mat& m) {
  Mat t(m.c, m.r);
  for (Index i = 0; i < m.r; ++i)
    for (Index j = 0; j < m.c; ++j) t(j, i) = m(i, j);
  return t;
}

// C = A * B, i-k-j order so the inner loop streams contiguous rows.
inline Mat matmul(const Mat& A, const Mat& B) {
  if (A.c != B.r) throw std::runtime_error("matmul shape");
  Mat C(A.r, B.c);
  const Index n = B.c;
  for (Index i = 0; i < A.r; ++i) {
    double* ci = C.row(i);
    const double* ai = A.row(i);
    for (Index k = 0; k < A.c; ++k) {
      const double aik = ai[k];
      if (aik == 0.0) continue;
      const double* bk = B.row(k);
      for (Index j = 0; j < n; ++j) ci[j] += aik * bk[j];
    }
  }
  return C;
}

inline double dot(const double* x, const double* y, Index n) {
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  Index i = 0;
  for (; i + 4 <= n; i += 4) {
    s0 += x[i] * y[i];
    s1 += x[i + 1] * y[i + 1];
    s2 += x[i + 2] * y[i + 2];
    s3 += x[i + 3] * y[i + 3];
  }
  for (; i < n; ++i) s0 += x[i] * y[i];
  return (s0 + s1) + (s2 + s3);
}

struct SvdTriple {
  Mat U;    // m x k
  Vec sigma;  // k, nonincreasing, positive
  Mat V;    // n x k
  Index rank() const { return static_cast<Index>(sigma.size()); }
  Mat reconstruct() const {
    Mat us = U;
    for (Index i = 0; i < us.r; ++i)
      for (Index j = 0; j < us.c; ++j) us(i, j) *= sigma[j];
    return matmul(us, transpose(V));
  }
};

// Full thin SVD of an m x n matrix by one-sided (Hestenes) Jacobi with
// cyclic pair order. Returns min(m,n) triplets sorted by descending sigma
// (zero sigmas included, with arbitrary unit U columns completed by
// Gram-Schmidt so U stays orthonormal).
inline SvdTriple jacobi_svd_full(const Mat& A) {
  if (A.r < A.c) {
    SvdTriple t = jacobi_svd_full(transpose(A));
    std::swap(t.U, t.V);
    return t;
  }
  const Index m = A.r, n = A.c;
  // Column-major working copies: w[j] is column j of A*V, v[j] column j of V.
  std::vector<Vec> w(n, Vec(m)), v(n, Vec(n, 0.0));
  for (Index j = 0; j < n; ++j) {
    for (Index i = 0; i < m; ++i) w[j][i] = A(i, j);
    v[j][j] = 1.0;
  }
  Vec nrm(n);
  for (Index j = 0; j < n; ++j) nrm[j] = dot(w[j].data(), w[j].data(), m);
  const double tol = 1e-15;
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (Index p = 0; p < n - 1; ++p) {
      for (Index q = p + 1; q < n; ++q) {
        const double alpha = nrm[p], beta = nrm[q];
        if (alpha == 0.0 || beta == 0.0) continue;
        const double gamma = dot(w[p].data(), w[q].data(), m);
        if (std::abs(gamma) <= tol * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t =
            std::copysign(1.0, zeta) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        double* wp = w[p].data();
        double* wq = w[q].data();
        for (Index i = 0; i < m; ++i) {
          const double a = wp[i], b = wq[i];
          wp[i] = cs * a - sn * b;
          wq[i] = sn * a + cs * b;
        }
        double* vp = v[p].data();
        double* vq = v[q].data();
        for (Index i = 0; i < n; ++i) {
          const double a = vp[i], b = vq[i];
          vp[i] = cs * a - sn * b;
          vq[i] = sn * a + cs * b;
        }
        nrm[p] = dot(wp, wp, m);
        nrm[q] = dot(wq, wq, m);
      }
    }
    if (!rotated) break;
  }
  std::vector<Index> order(n);
  std::iota(order.begin(), order.end(), 0);
  Vec s(n);
  for (Index j = 0; j < n; ++j) s[j] = std::sqrt(dot(w[j].data(), w[j].data(), m));
  std::stable_sort(order.begin(), order.end(),
                   [&](Index x, Index y) { return s[x] > s[y]; });
  SvdTriple out;
  out.U = Mat(m, n);
  out.V = Mat(n, n);
  out.sigma.resize(n);
  for (Index jj = 0; jj < n; ++jj) {
    const Index j = order[jj];
    out.sigma[jj] = s[j];
    for (Index i = 0; i < n; ++i) out.V(i, jj) = v[j][i];
    if (s[j] > 0.0)
      for (Index i = 0; i < m; ++i) out.U(i, jj) = w[j][i] / s[j];
  }
  // Complete U columns for zero singular values (Gram-Schmidt on unit vectors).
  for (Index jj = 0; jj < n; ++jj) {
    if (out.sigma[jj] > 0.0) continue;
    for (Index e = 0; e < m; ++e) {
      Vec cand(m, 0.0);
      cand[e] = 1.0;
      for (int pass = 0; pass < 2; ++pass)
        for (Index kk = 0; kk < n; ++kk) {
          if (kk == jj || (out.sigma[kk] <= 0.0 && kk > jj)) continue;
          double d = 0;
          for (Index i = 0; i < m; ++i) d += out.U(i, kk) * cand[i];
          for (Index i = 0; i < m; ++i) cand[i] -= d * out.U(i, kk);
        }
      double nn = std::sqrt(dot(cand.data(), cand.data(), m));
      if (nn > 1e-8) {
        for (Index i = 0; i < m; ++i) out.U(i, jj) = cand[i] / nn;
        break;
      }
    }
  }
  return out;
}

// Keep the leading k triplets.
inline SvdTriple svd_head(const SvdTriple& s, Index k) {
  SvdTriple o;
  o.sigma.assign(s.sigma.begin(), s.sigma.begin() + k);
  o.U = Mat(s.U.r, k);
  o.V = Mat(s.V.r, k);
  for (Index i = 0; i < s.U.r; ++i)
    for (Index j = 0; j < k; ++j) o.U(i, j) = s.U(i, j);
  for (Index i = 0; i < s.V.r; ++i)
    for (Index j = 0; j < k; ++j) o.V(i, j) = s.V(i, j);
  return o;
}

// LU with partial (row) pivoting of a square matrix: P A = L U.
struct PartialPivLU {
  Mat lu;
  std::vector<Index> perm;  // row i of PA is row perm[i] of A
  explicit PartialPivLU(const Mat& A) : lu(A), perm(A.r) {
    const Index n = A.r;
    std::iota(perm.begin(), perm.end(), 0);
    for (Index k = 0; k < n; ++k) {
      Index piv = k;
      double best = std::abs(lu(k, k));
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(lu(i, k)) > best) {
          best = std::abs(lu(i, k));
          piv = i;
        }
      if (piv != k) {
        for (Index j = 0; j < n; ++j) std::swap(lu(k, j), lu(piv, j));
        std::swap(perm[k], perm[piv]);
      }
      const double d = lu(k, k);
      if (d == 0.0) continue;
      for (Index i = k + 1; i < n; ++i) {
        const double f = lu(i, k) / d;
        lu(i, k) = f;
        if (f == 0.0) continue;
        double* li = lu.row(i);
        const double* lk = lu.row(k);
        for (Index j = k + 1; j < n; ++j) li[j] -= f * lk[j];
      }
    }
  }
  Vec diag() const {
    Vec d(lu.r);
    for (Index i = 0; i < lu.r; ++i) d[i] = lu(i, i);
    return d;
  }
  // Solve A x = b.
  Vec solve(const Vec& b) const {
    const Index n = lu.r;
    Vec x(n);
    for (Index i = 0; i < n; ++i) x[i] = b[perm[i]];
    for (Index i = 0; i < n; ++i)
      for (Index j = 0; j < i; ++j) x[i] -= lu(i, j) * x[j];
    for (Index i = n - 1; i >= 0; --i) {
      for (Index j = i + 1; j < n; ++j) x[i] -= lu(i, j) * x[j];
      x[i] /= lu(i, i);
    }
    return x;
  }
  // Solve A^T x = b.
  Vec solve_transpose(const Vec& b) const {
    const Index n = lu.r;
    // A = P^T L U  ->  A^T = U^T L^T P ; solve U^T y = b, L^T z = y, x = P^T z
    Vec y(b);
    for (Index i = 0; i < n; ++i) {
      for (Index j = 0; j < i; ++j) y[i] -= lu(j, i) * y[j];
      y[i] /= lu(i, i);
    }
    for (Index i = n - 1; i >= 0; --i)
      for (Index j = i + 1; j < n; ++j) y[i] -= lu(j, i) * y[j];
    Vec x(n);
    for (Index i = 0; i < n; ++i) x[perm[i]] = y[i];
    return x;
  }
};

// Householder QR of an m x n matrix (m >= n or not): returns thin Q
// (m x min(m,n)) and the leading min(m,n) x n block of R.
struct HouseholderQR {
  Mat Q, R;
  // W[k:, j0:j1] -= beta * v (v^T W[k:, j0:j1]), row-major friendly.
  static void apply_reflector(Mat& W, const Vec& v, double beta, Index k,
                              Index j0, Index j1) {
    Vec s(static_cast<size_t>(j1 - j0), 0.0);
    for (Index i = k; i < W.r; ++i) {
      const double vi = v[i - k];
      if (vi == 0.0) continue;
      const double* wi = W.row(i);
      for (Index j = j0; j < j1; ++j) s[j - j0] += vi * wi[j];
    }
    for (Index i = k; i < W.r; ++i) {
      const double f = beta * v[i - k];
      if (f == 0.0) continue;
      double* wi = W.row(i);
      for (Index j = j0; j < j1; ++j) wi[j] -= f * s[j - j0];
    }
  }
  explicit HouseholderQR(const Mat& A) {
    const Index m = A.r, n = A.c, p = std::min(m, n);
    Mat W = A;
    std::vector<Vec> vs;
    Vec betas;
    for (Index k = 0; k < p; ++k) {
      Vec v(m - k);
      for (Index i = k; i < m; ++i) v[i - k] = W(i, k);
      double alpha = std::sqrt(dot(v.data(), v.data(), m - k));
      if (alpha == 0.0) {
        vs.push_back(Vec(m - k, 0.0));
        betas.push_back(0.0);
        continue;
      }
      if (v[0] > 0) alpha = -alpha;
      v[0] -= alpha;
      const double vn = dot(v.data(), v.data(), m - k);
      const double beta = vn > 0 ? 2.0 / vn : 0.0;
      apply_reflector(W, v, beta, k, k, n);
      vs.push_back(v);
      betas.push_back(beta);
    }
    R = Mat(p, n);
    for (Index i = 0; i < p; ++i)
      for (Index j = i; j < n; ++j) R(i, j) = W(i, j);
    Q = Mat::eye(m, p);
    for (Index k = p - 1; k >= 0; --k) {
      const Vec& v = vs[k];
      const double beta = betas[k];
      if (beta == 0.0) continue;
      apply_reflector(Q, v, beta, k, 0, p);
    }
  }
};

}  // namespace damf_oracle
