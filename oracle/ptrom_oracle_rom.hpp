// ptrom_oracle_rom.hpp — CPU ORACLE (test infrastructure only), PTROM part.
// Restates /root/reference/proj/include/ptrom/reduction.hpp:18-431 and
// rom.hpp:17-412 without Eigen. Where the reference calls Eigen decompositions
// (BDCSVD reduction.hpp:43, CompleteOrthogonalDecomposition reduction.hpp:142
// and 208-218, ColPivHouseholderQR rom.hpp:218 and 327, HouseholderQR in the
// tests) textbook algorithms stand in: one-sided Jacobi SVD, column-pivoted
// Householder QR with Eigen's Householder convention and rank threshold, and
// the complete orthogonal decomposition for minimum-norm solutions. No
// reference test pins those bitwise; parity there is by
// tolerance. Matrices are column-major like Eigen's.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

#include "ptrom_oracle.hpp"
#include "ptrom_oracle_tree.hpp"

namespace oracle {

// ------------------------------------------------------------- matrices ---
struct Mat {
  Index rows = 0, cols = 0;
  std::vector<double> a;  // column-major
  Mat() = default;
  Mat(Index r, Index c, double v = 0.0) : rows(r), cols(c), a(static_cast<size_t>(r * c), v) {}
  double& operator()(Index r, Index c) { return a[static_cast<size_t>(c * rows + r)]; }
  double operator()(Index r, Index c) const { return a[static_cast<size_t>(c * rows + r)]; }
  static Mat identity(Index n) {
    Mat m(n, n);
    for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};
using Vec = std::vector<double>;

// Eigen's GEMV / GEMM summation order is blocked and unpinned; the oracle
// uses plain ascending inner products.
inline Vec matvec(const Mat& m, const Vec& x) {
  Vec y(static_cast<size_t>(m.rows), 0.0);
  for (Index c = 0; c < m.cols; ++c)
    for (Index r = 0; r < m.rows; ++r) y[r] += m(r, c) * x[c];
  return y;
}
inline Mat matmul(const Mat& a, const Mat& b) {
  Mat c(a.rows, b.cols);
  for (Index j = 0; j < b.cols; ++j)
    for (Index k = 0; k < a.cols; ++k) {
      const double bk = b(k, j);
      for (Index i = 0; i < a.rows; ++i) c(i, j) += a(i, k) * bk;
    }
  return c;
}
inline double vnorm(const Vec& v) {
  double s = 0;
  for (double e : v) s += e * e;
  return std::sqrt(s);
}

// Eigen's makeHouseholder convention: H = I - tau v v^T, v = [1, essential],
// H x = [beta, 0...], beta = -sign(x0) ||x||.
struct Householder {
  double tau = 0, beta = 0;
  Vec essential;
};
inline Householder make_householder(const double* x, Index n) {
  Householder h;
  const double c0 = x[0];
  double tail = 0;
  for (Index i = 1; i < n; ++i) tail += x[i] * x[i];
  h.essential.assign(static_cast<size_t>(std::max<Index>(n - 1, 0)), 0.0);
  if (tail <= std::numeric_limits<double>::min()) {
    h.tau = 0;
    h.beta = c0;
    return h;
  }
  double beta = std::sqrt(c0 * c0 + tail);
  if (c0 >= 0) beta = -beta;
  for (Index i = 1; i < n; ++i) h.essential[i - 1] = x[i] / (c0 - beta);
  h.tau = (beta - c0) / beta;
  h.beta = beta;
  return h;
}
// Applies H (on rows [r0, r0+len)) to columns [c0, cols) of m.
inline void apply_householder_left(Mat& m, const Householder& h, Index r0, Index c0) {
  if (h.tau == 0) return;
  const Index len = static_cast<Index>(h.essential.size()) + 1;
  for (Index c = c0; c < m.cols; ++c) {
    double w = m(r0, c);
    for (Index i = 1; i < len; ++i) w += h.essential[i - 1] * m(r0 + i, c);
    w *= h.tau;
    m(r0, c) -= w;
    for (Index i = 1; i < len; ++i) m(r0 + i, c) -= w * h.essential[i - 1];
  }
}

// HouseholderQR(raw).householderQ() * I(rows, cols): thin orthonormal factor.
inline Mat householder_q_thin(Mat a) {
  const Index m = a.rows, n = a.cols, k = std::min(m, n);
  std::vector<Householder> hs;
  for (Index j = 0; j < k; ++j) {
    Vec col(static_cast<size_t>(m - j));
    for (Index i = j; i < m; ++i) col[i - j] = a(i, j);
    Householder h = make_householder(col.data(), m - j);
    apply_householder_left(a, h, j, j + 1);
    hs.push_back(h);
  }
  Mat q(m, n);
  for (Index j = 0; j < n && j < m; ++j) q(j, j) = 1.0;
  for (Index j = k - 1; j >= 0; --j) apply_householder_left(q, hs[static_cast<size_t>(j)], j, 0);
  return q;
}

// Column-pivoted Householder QR with Eigen's rank rule (threshold =
// eps * diag size, relative to the largest pivot).
struct ColPivQR {
  Mat qr;  // R in the upper triangle; reflectors kept separately
  std::vector<Householder> hs;
  std::vector<Index> perm;  // column j of R is column perm[j] of the input
  Index rank = 0;
  explicit ColPivQR(Mat a) : qr(std::move(a)) {
    const Index m = qr.rows, n = qr.cols, k = std::min(m, n);
    perm.resize(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), Index(0));
    Vec norms(static_cast<size_t>(n));
    for (Index c = 0; c < n; ++c) {
      double s = 0;
      for (Index r = 0; r < m; ++r) s += qr(r, c) * qr(r, c);
      norms[c] = s;
    }
    for (Index j = 0; j < k; ++j) {
      Index best = j;
      for (Index c = j + 1; c < n; ++c)
        if (norms[c] > norms[best]) best = c;
      if (best != j) {
        for (Index r = 0; r < m; ++r) std::swap(qr(r, j), qr(r, best));
        std::swap(norms[j], norms[best]);
        std::swap(perm[j], perm[best]);
      }
      Vec col(static_cast<size_t>(m - j));
      for (Index i = j; i < m; ++i) col[i - j] = qr(i, j);
      Householder h = make_householder(col.data(), m - j);
      apply_householder_left(qr, h, j, j + 1);
      qr(j, j) = h.beta;
      for (Index i = j + 1; i < m; ++i) qr(i, j) = 0.0;
      hs.push_back(h);
      for (Index c = j + 1; c < n; ++c) {  // downdate remaining column norms
        double s = 0;
        for (Index r = j + 1; r < m; ++r) s += qr(r, c) * qr(r, c);
        norms[c] = s;
      }
    }
    const double maxpiv = k ? std::abs(qr(0, 0)) : 0.0;
    const double thr = std::numeric_limits<double>::epsilon() * double(std::max<Index>(k, 1));
    rank = 0;
    for (Index j = 0; j < k; ++j)
      if (std::abs(qr(j, j)) > thr * maxpiv) ++rank;
  }
  // Q^T b for one right-hand side.
  Vec qt(const Vec& b) const {
    Mat t(qr.rows, 1);
    for (Index i = 0; i < qr.rows; ++i) t(i, 0) = b[i];
    for (size_t j = 0; j < hs.size(); ++j) apply_householder_left(t, hs[j], static_cast<Index>(j), 0);
    return t.a;
  }
  // Least-squares solve (ColPivHouseholderQR::solve): basic solution with
  // free variables of rank-deficient problems set to zero.
  Vec solve(const Vec& b) const {
    const Index n = qr.cols;
    Vec c = qt(b);
    Vec z(static_cast<size_t>(n), 0.0);
    for (Index i = rank - 1; i >= 0; --i) {
      double s = c[i];
      for (Index j = i + 1; j < rank; ++j) s -= qr(i, j) * z[j];
      z[i] = s / qr(i, i);
    }
    Vec x(static_cast<size_t>(n), 0.0);
    for (Index j = 0; j < n; ++j) x[perm[j]] = z[j];
    return x;
  }
};

// CompleteOrthogonalDecomposition::solve — minimum-norm least squares via
// CPQR followed by an RZ reduction of the leading rank rows.
inline Mat cod_solve(const Mat& a, const Mat& b, Index* rank_out = nullptr, std::vector<Index>* perm_out = nullptr) {
  ColPivQR cp(a);
  const Index n = a.cols, r = cp.rank;
  if (rank_out) *rank_out = r;
  if (perm_out) *perm_out = cp.perm;
  // T Z = [R11 R12] (r x n): Householder from the right on rows r-1..0.
  Mat t(r, n);
  for (Index i = 0; i < r; ++i)
    for (Index j = i; j < n; ++j) t(i, j) = cp.qr(i, j);
  std::vector<Householder> zs(static_cast<size_t>(r));
  if (r < n) {
    for (Index i = r - 1; i >= 0; --i) {
      // row vector [t(i,i), t(i, r..n-1)]
      Vec v(static_cast<size_t>(1 + n - r));
      v[0] = t(i, i);
      for (Index j = r; j < n; ++j) v[1 + j - r] = t(i, j);
      Householder h = make_householder(v.data(), 1 + n - r);
      zs[i] = h;
      // apply from the right to rows 0..i
      for (Index rr = 0; rr <= i; ++rr) {
        double w = t(rr, i);
        for (Index j = r; j < n; ++j) w += h.essential[j - r] * t(rr, j);
        w *= h.tau;
        t(rr, i) -= w;
        for (Index j = r; j < n; ++j) t(rr, j) -= w * h.essential[j - r];
      }
    }
  }
  Mat x(n, b.cols);
  for (Index col = 0; col < b.cols; ++col) {
    Vec bc(b.a.begin() + col * b.rows, b.a.begin() + (col + 1) * b.rows);
    Vec c = cp.qt(bc);
    Vec z(static_cast<size_t>(n), 0.0);
    for (Index i = r - 1; i >= 0; --i) {
      double s = c[i];
      for (Index j = i + 1; j < r; ++j) s -= t(i, j) * z[j];
      z[i] = s / t(i, i);
    }
    if (r < n) {  // z <- Z^T z (apply reflectors in reverse)
      for (Index i = 0; i < r; ++i) {
        const Householder& h = zs[i];
        if (h.tau == 0) continue;
        double w = z[i];
        for (Index j = r; j < n; ++j) w += h.essential[j - r] * z[j];
        w *= h.tau;
        z[i] -= w;
        for (Index j = r; j < n; ++j) z[j] -= w * h.essential[j - r];
      }
    }
    for (Index j = 0; j < n; ++j) x(cp.perm[j], col) = z[j];
  }
  return x;
}

// One-sided Jacobi SVD: A = U diag(s) V^T, singular values descending.
inline void jacobi_svd(const Mat& a, Mat& u, Vec& s) {
  const Index m = a.rows, n = a.cols;
  Mat w = a;
  for (int sweep = 0; sweep < 80; ++sweep) {
    double off = 0;
    for (Index p = 0; p < n; ++p)
      for (Index q = p + 1; q < n; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        for (Index i = 0; i < m; ++i) {
          alpha += w(i, p) * w(i, p);
          beta += w(i, q) * w(i, q);
          gamma += w(i, p) * w(i, q);
        }
        if (gamma == 0 || std::abs(gamma) <= 1e-17 * std::sqrt(alpha * beta)) continue;
        off = std::max(off, std::abs(gamma) / std::sqrt(alpha * beta));
        const double zeta = (beta - alpha) / (2 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1 + zeta * zeta));
        const double c = 1 / std::sqrt(1 + t * t), sn = c * t;
        for (Index i = 0; i < m; ++i) {
          const double x = w(i, p), y = w(i, q);
          w(i, p) = c * x - sn * y;
          w(i, q) = sn * x + c * y;
        }
      }
    if (off < 1e-16) break;
  }
  std::vector<Index> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), Index(0));
  Vec norms(static_cast<size_t>(n));
  for (Index c = 0; c < n; ++c) {
    double ss = 0;
    for (Index i = 0; i < m; ++i) ss += w(i, c) * w(i, c);
    norms[c] = std::sqrt(ss);
  }
  std::stable_sort(order.begin(), order.end(), [&](Index x, Index y) { return norms[x] > norms[y]; });
  u = Mat(m, n);
  s.assign(static_cast<size_t>(n), 0.0);
  for (Index k = 0; k < n; ++k) {
    const Index c = order[k];
    s[k] = norms[c];
    for (Index i = 0; i < m; ++i) u(i, k) = norms[c] > 0 ? w(i, c) / norms[c] : 0.0;
  }
}

// ----------------------------------------------------------- reduction ---
// reduction.hpp:18-26
struct PODBasis {
  Mat phi;   // N_d x M
  Vec singular_values;
  Vec x_ref;
  Index dim() const { return phi.rows; }
  Index modes() const { return phi.cols; }
};

// reduction.hpp:32-70 (BDCSVD replaced by one-sided Jacobi; same rank rule
// and sign convention).
inline PODBasis build_pod(const Mat& snapshots, Index modes, const Vec& x_ref) {
  if (snapshots.rows == 0 || snapshots.cols == 0) throw config_error("build_pod: empty snapshot matrix");
  for (double v : snapshots.a)
    if (!std::isfinite(v)) throw config_error("build_pod: non-finite snapshots");
  if (static_cast<Index>(x_ref.size()) != snapshots.rows)
    throw config_error("build_pod: reference state dimension mismatch");
  const Index max_modes = std::min(snapshots.rows, snapshots.cols);
  if (modes < 1 || modes > max_modes)
    throw config_error("build_pod: mode count " + std::to_string(modes) + " outside [1, " +
                       std::to_string(max_modes) + "]");
  Mat u;
  Vec sv;
  if (snapshots.rows >= snapshots.cols) {
    jacobi_svd(snapshots, u, sv);
  } else {  // SVD of A^T, then U = A V / s
    Mat at(snapshots.cols, snapshots.rows);
    for (Index r = 0; r < snapshots.rows; ++r)
      for (Index c = 0; c < snapshots.cols; ++c) at(c, r) = snapshots(r, c);
    Mat v;
    jacobi_svd(at, v, sv);
    sv.resize(static_cast<size_t>(max_modes));
    u = Mat(snapshots.rows, max_modes);
    for (Index k = 0; k < max_modes; ++k)
      for (Index i = 0; i < snapshots.rows; ++i) u(i, k) = v(i, k);
  }
  const double cutoff = double(std::max(snapshots.rows, snapshots.cols)) * std::numeric_limits<double>::epsilon() * sv[0];
  Index rank = 0;
  while (rank < static_cast<Index>(sv.size()) && sv[rank] > cutoff) ++rank;
  if (modes > rank)
    throw numerical_error("build_pod: requested " + std::to_string(modes) +
                          " modes but snapshots have numerical rank " + std::to_string(rank));
  PODBasis b;
  b.phi = Mat(snapshots.rows, modes);
  for (Index c = 0; c < modes; ++c)
    for (Index r = 0; r < snapshots.rows; ++r) b.phi(r, c) = u(r, c);
  b.singular_values.assign(sv.begin(), sv.begin() + modes);
  b.x_ref = x_ref;
  for (Index c = 0; c < modes; ++c) {  // reduction.hpp:57-68
    Index arg = 0;
    double best = -1;
    for (Index r = 0; r < b.phi.rows; ++r) {
      const double a = std::abs(b.phi(r, c));
      if (a > best) {
        best = a;
        arg = r;
      }
    }
    if (b.phi(arg, c) < 0)
      for (Index r = 0; r < b.phi.rows; ++r) b.phi(r, c) = -b.phi(r, c);
  }
  return b;
}

// reduction.hpp:74-77
inline Vec weighted_pod_space(const PODBasis& b) { return matvec(b.phi, b.singular_values); }

// reduction.hpp:93-168
inline std::vector<Index> greedy_sample(const Mat& phi_r, Index n_target, const std::vector<Index>& preseed = {}) {
  if (phi_r.rows % 2 != 0) throw config_error("state dimension must be even");
  const Index n = phi_r.rows / 2;
  const Index n_r = phi_r.cols;
  if (n_r < 1) throw config_error("greedy_sample: empty residual basis");
  for (double v : phi_r.a)
    if (!std::isfinite(v)) throw config_error("greedy_sample: non-finite residual basis");
  if (n_target < 1 || n_target > n)
    throw config_error("greedy_sample: target count " + std::to_string(n_target) + " outside [1, " +
                       std::to_string(n) + "]");
  std::vector<char> picked(static_cast<size_t>(n), 0);
  std::vector<Index> chosen;
  for (const Index p : preseed) {
    if (p < 0 || p >= n) throw config_error("greedy_sample: preseed id out of range");
    if (picked[p]) throw config_error("greedy_sample: duplicate preseed id");
    picked[p] = 1;
    chosen.push_back(p);
  }
  if (static_cast<Index>(chosen.size()) > n_target) throw config_error("greedy_sample: preseed larger than target count");
  const Index n_a = n_target - static_cast<Index>(chosen.size());
  if (n_a > 0) {
    const Index n_c = std::min(n_r, 2 * n_target);
    const Index n_it = std::min(n_c, n_a);
    Index nb = 0;
    for (Index it = 1; it <= n_it; ++it) {
      const Index n_ci = n_c / n_it + (it <= n_c % n_it ? 1 : 0);
      const Index n_ai = n_a / n_it + (it <= n_a % n_it ? 1 : 0);
      Mat work(phi_r.rows, n_ci);
      if (it == 1) {
        for (Index q = 0; q < n_ci; ++q)
          for (Index r = 0; r < phi_r.rows; ++r) work(r, q) = phi_r(r, q);
      } else {
        std::vector<Index> sorted_ids = chosen;
        std::sort(sorted_ids.begin(), sorted_ids.end());
        std::vector<Index> rows;
        for (Index p : sorted_ids) rows.push_back(p);
        for (Index p : sorted_ids) rows.push_back(p + n);
        Mat sb(static_cast<Index>(rows.size()), nb), rhs(static_cast<Index>(rows.size()), n_ci);
        for (size_t k = 0; k < rows.size(); ++k) {
          for (Index c = 0; c < nb; ++c) sb(static_cast<Index>(k), c) = phi_r(rows[k], c);
          for (Index c = 0; c < n_ci; ++c) rhs(static_cast<Index>(k), c) = phi_r(rows[k], nb + c);
        }
        const Mat coef = cod_solve(sb, rhs);  // nb x n_ci
        for (Index q = 0; q < n_ci; ++q)
          for (Index r = 0; r < phi_r.rows; ++r) {
            double s = 0;
            for (Index c = 0; c < nb; ++c) s += phi_r(r, c) * coef(c, q);
            work(r, q) = phi_r(r, nb + q) - s;
          }
      }
      for (Index j = 0; j < n_ai; ++j) {
        Index arg = -1;
        double best = -1;
        for (Index l = 0; l < n; ++l) {
          if (picked[l]) continue;
          double score = 0;
          for (Index q = 0; q < n_ci; ++q) score += work(l, q) * work(l, q) + work(l + n, q) * work(l + n, q);
          if (score > best) {
            best = score;
            arg = l;
          }
        }
        picked[arg] = 1;
        chosen.push_back(arg);
      }
      nb += n_ci;
    }
  }
  std::sort(chosen.begin(), chosen.end());
  return chosen;
}

// reduction.hpp:173-220
struct GnatOperator {
  std::vector<Index> sample_ids, sampled_dofs;
  Mat A;  // M_r x n_d
  Index n_sampled_dofs() const { return static_cast<Index>(sampled_dofs.size()); }
};
inline GnatOperator build_gnat_operator(const Mat& phi_r, const std::vector<Index>& sample_ids) {
  if (phi_r.rows % 2 != 0) throw config_error("state dimension must be even");
  const Index n = phi_r.rows / 2, m_r = phi_r.cols;
  if (sample_ids.empty()) throw config_error("build_gnat_operator: no sample ids");
  std::vector<Index> ids = sample_ids;
  std::sort(ids.begin(), ids.end());
  if (std::adjacent_find(ids.begin(), ids.end()) != ids.end())
    throw config_error("build_gnat_operator: duplicate sample ids");
  if (ids.front() < 0 || ids.back() >= n) throw config_error("build_gnat_operator: sample id out of range");
  const Index n_d = 2 * static_cast<Index>(ids.size());
  if (n_d < m_r)
    throw config_error("build_gnat_operator: " + std::to_string(n_d) + " sampled dofs cannot support " +
                       std::to_string(m_r) + " residual modes (need 2 * samples >= modes)");
  GnatOperator op;
  op.sample_ids = ids;
  for (Index p : ids) op.sampled_dofs.push_back(p);
  for (Index p : ids) op.sampled_dofs.push_back(p + n);
  Mat sampled(n_d, m_r);
  for (Index k = 0; k < n_d; ++k)
    for (Index c = 0; c < m_r; ++c) sampled(k, c) = phi_r(op.sampled_dofs[k], c);
  Index rank = 0;
  std::vector<Index> perm;
  op.A = cod_solve(sampled, Mat::identity(n_d), &rank, &perm);  // pinv
  if (rank < m_r) {
    std::string cols;
    for (Index k = rank; k < m_r; ++k) cols += (cols.empty() ? "" : ", ") + std::to_string(perm[k]);
    throw numerical_error("build_gnat_operator: sampled residual basis has rank " + std::to_string(rank) + " < " +
                          std::to_string(m_r) + "; dependent columns: " + cols);
  }
  return op;
}

// reduction.hpp:225-274
struct WeightedPodTree {
  QuadTree<double> tree;
  Mat node_phi_x, node_phi_y, node_x0;  // nodes x M, nodes x M, nodes x 2
  Vec node_gamma;
  std::vector<char> zero_gamma;
  Index num_nodes() const { return static_cast<Index>(tree.nodes.size()); }
};
inline WeightedPodTree build_weighted_pod_tree(const PODBasis& basis, const Vec& gamma, Index leaf_capacity = 1) {
  const Index n = basis.dim() / 2;
  if (static_cast<Index>(gamma.size()) != n) throw config_error("build_weighted_pod_tree: gamma size mismatch");
  const Vec w = weighted_pod_space(basis);
  WeightedPodTree out;
  out.tree = build_tree<double>(Vec(w.begin(), w.begin() + n), Vec(w.begin() + n, w.end()), gamma, leaf_capacity);
  const Index nn = out.num_nodes(), m = basis.modes();
  out.node_phi_x = Mat(nn, m);
  out.node_phi_y = Mat(nn, m);
  out.node_x0 = Mat(nn, 2);
  out.node_gamma.assign(static_cast<size_t>(nn), 0.0);
  out.zero_gamma.assign(static_cast<size_t>(nn), 0);
  std::vector<Index> members;
  for (Index id = 0; id < nn; ++id) {
    const auto& nd = out.tree.nodes[id];
    members.assign(out.tree.perm.begin() + nd.begin, out.tree.perm.begin() + nd.end);
    std::sort(members.begin(), members.end());
    double gsum = 0;
    for (Index p : members) gsum += gamma[p];
    out.node_gamma[id] = gsum;
    const bool fb = gsum == 0;
    out.zero_gamma[id] = fb ? 1 : 0;
    for (Index p : members) {
      const double w_p = fb ? 1.0 / double(members.size()) : gamma[p] / gsum;
      for (Index c = 0; c < m; ++c) {
        out.node_phi_x(id, c) += w_p * basis.phi(p, c);
        out.node_phi_y(id, c) += w_p * basis.phi(p + n, c);
      }
      out.node_x0(id, 0) += w_p * basis.x_ref[p];
      out.node_x0(id, 1) += w_p * basis.x_ref[p + n];
    }
  }
  return out;
}

// reduction.hpp:280-302
struct SurrogateSourceBasis {
  Mat phi_tilde;  // 2 N_c x M
  Vec gamma_tilde, x0_tilde;
  std::vector<std::int32_t> cluster_node_ids;
  std::vector<std::vector<Index>> cluster_membership;
  std::vector<char> zero_gamma;
  std::vector<Index> target_ids;
  std::vector<std::vector<Index>> per_target_clusters, per_target_direct;
  std::vector<Index> direct_ids;
  Mat direct_phi;  // 2U x M
  Vec direct_x0, direct_gamma;
  Index num_clusters() const { return static_cast<Index>(gamma_tilde.size()); }
  Index num_direct() const { return static_cast<Index>(direct_ids.size()); }
};

// reduction.hpp:304-385
inline SurrogateSourceBasis cluster_pod(const WeightedPodTree& wtree, const PODBasis& basis, const Vec& gamma,
                                        const std::vector<Index>& target_ids,
                                        const ClusterCriterion<double>& criterion) {
  const Index n = basis.dim() / 2;
  if (static_cast<Index>(gamma.size()) != n) throw config_error("cluster_pod: gamma size mismatch");
  if (target_ids.empty()) throw config_error("cluster_pod: no targets");
  for (Index t : target_ids)
    if (t < 0 || t >= n) throw config_error("cluster_pod: target id out of range");
  SurrogateSourceBasis out;
  out.target_ids = target_ids;
  std::vector<Index> node_to_cluster(static_cast<size_t>(wtree.num_nodes()), -1);
  std::vector<char> in_direct(static_cast<size_t>(n), 0);
  std::vector<std::vector<Index>> raw_direct;
  for (Index t : target_ids) {
    ClusterList cl = collect_clusters<double>(wtree.tree, t, criterion);
    std::vector<Index> cix;
    for (std::int32_t node : cl.cluster_nodes) {
      Index& ix = node_to_cluster[node];
      if (ix < 0) {
        ix = static_cast<Index>(out.cluster_node_ids.size());
        out.cluster_node_ids.push_back(node);
      }
      cix.push_back(ix);
    }
    out.per_target_clusters.push_back(std::move(cix));
    for (Index j : cl.direct_ids) in_direct[j] = 1;
    raw_direct.push_back(std::move(cl.direct_ids));
  }
  for (Index j = 0; j < n; ++j)
    if (in_direct[j]) out.direct_ids.push_back(j);
  std::vector<Index> slot(static_cast<size_t>(n), -1);
  for (size_t u = 0; u < out.direct_ids.size(); ++u) slot[out.direct_ids[u]] = static_cast<Index>(u);
  for (const auto& ids : raw_direct) {
    std::vector<Index> local;
    for (Index j : ids) local.push_back(slot[j]);
    out.per_target_direct.push_back(std::move(local));
  }
  const Index n_c = static_cast<Index>(out.cluster_node_ids.size()), m = basis.modes();
  out.phi_tilde = Mat(2 * n_c, m);
  out.x0_tilde.assign(static_cast<size_t>(2 * n_c), 0.0);
  out.gamma_tilde.assign(static_cast<size_t>(n_c), 0.0);
  out.zero_gamma.assign(static_cast<size_t>(n_c), 0);
  out.cluster_membership.resize(static_cast<size_t>(n_c));
  for (Index c = 0; c < n_c; ++c) {
    const std::int32_t node = out.cluster_node_ids[c];
    const auto& nd = wtree.tree.nodes[node];
    for (Index k = 0; k < m; ++k) {
      out.phi_tilde(c, k) = wtree.node_phi_x(node, k);
      out.phi_tilde(c + n_c, k) = wtree.node_phi_y(node, k);
    }
    out.x0_tilde[c] = wtree.node_x0(node, 0);
    out.x0_tilde[c + n_c] = wtree.node_x0(node, 1);
    out.gamma_tilde[c] = wtree.node_gamma[node];
    out.zero_gamma[c] = wtree.zero_gamma[node];
    auto& mem = out.cluster_membership[c];
    mem.assign(wtree.tree.perm.begin() + nd.begin, wtree.tree.perm.begin() + nd.end);
    std::sort(mem.begin(), mem.end());
  }
  const Index u = out.num_direct();
  out.direct_phi = Mat(2 * u, m);
  out.direct_x0.assign(static_cast<size_t>(2 * u), 0.0);
  out.direct_gamma.assign(static_cast<size_t>(u), 0.0);
  for (Index k = 0; k < u; ++k) {
    const Index p = out.direct_ids[k];
    for (Index c = 0; c < m; ++c) {
      out.direct_phi(k, c) = basis.phi(p, c);
      out.direct_phi(k + u, c) = basis.phi(p + n, c);
    }
    out.direct_x0[k] = basis.x_ref[p];
    out.direct_x0[k + u] = basis.x_ref[p + n];
    out.direct_gamma[k] = gamma[p];
  }
  return out;
}

// reduction.hpp:388-395
inline SurrogateSourceBasis cluster_pod(const PODBasis& basis, const Vec& gamma, const std::vector<Index>& targets,
                                        const ClusterCriterion<double>& criterion, Index leaf_capacity = 1) {
  return cluster_pod(build_weighted_pod_tree(basis, gamma, leaf_capacity), basis, gamma, targets, criterion);
}

// reduction.hpp:400-431
inline void reassign_cluster_circulation(SurrogateSourceBasis& s, const Vec& gamma, const PODBasis& basis) {
  const Index n = basis.dim() / 2;
  if (static_cast<Index>(gamma.size()) != n) throw config_error("reassign_cluster_circulation: gamma size mismatch");
  const Index n_c = s.num_clusters(), m = basis.modes();
  for (Index c = 0; c < n_c; ++c) {
    const auto& mem = s.cluster_membership[c];
    double gsum = 0;
    for (Index p : mem) gsum += gamma[p];
    const bool fb = gsum == 0;
    s.gamma_tilde[c] = gsum;
    s.zero_gamma[c] = fb ? 1 : 0;
    Vec px(static_cast<size_t>(m), 0.0), py(static_cast<size_t>(m), 0.0);
    double x0x = 0, x0y = 0;
    for (Index p : mem) {
      const double w_p = fb ? 1.0 / double(mem.size()) : gamma[p] / gsum;
      for (Index k = 0; k < m; ++k) {
        px[k] += w_p * basis.phi(p, k);
        py[k] += w_p * basis.phi(p + n, k);
      }
      x0x += w_p * basis.x_ref[p];
      x0y += w_p * basis.x_ref[p + n];
    }
    for (Index k = 0; k < m; ++k) {
      s.phi_tilde(c, k) = px[k];
      s.phi_tilde(c + n_c, k) = py[k];
    }
    s.x0_tilde[c] = x0x;
    s.x0_tilde[c + n_c] = x0y;
  }
  for (Index k = 0; k < s.num_direct(); ++k) s.direct_gamma[k] = gamma[s.direct_ids[k]];
}

// ------------------------------------------------------------------ rom ---
// rom.hpp:17-27
struct RomConfig {
  double tol = 1e-4;
  int max_iters = 100;
  double step_length = 1.0;
  void validate() const {
    if (!(tol > 0)) throw config_error("ROM tolerance must be positive");
    if (max_iters < 1) throw config_error("ROM max_iters must be >= 1");
    if (!(step_length > 0)) throw config_error("ROM step length must be positive");
  }
};

// rom.hpp:29-41
struct RomTrajectory {
  Mat x_hat;  // M x n_steps
  std::vector<int> iterations;
  std::vector<char> converged;
};

// rom.hpp:60-65
inline Mat reconstruct_full(const Mat& x_hat, const PODBasis& b) {
  Mat out(b.dim(), x_hat.cols);
  for (Index s = 0; s < x_hat.cols; ++s) {
    Vec xs(x_hat.a.begin() + s * x_hat.rows, x_hat.a.begin() + (s + 1) * x_hat.rows);
    Vec r = matvec(b.phi, xs);
    for (Index i = 0; i < b.dim(); ++i) out(i, s) = r[i] + b.x_ref[i];
  }
  return out;
}

// rom.hpp:71-84 — (I - dt/2 J) applied to the paired rows of mat.
inline Mat apply_residual_jacobian(const BlockDiagonalJacobian<double>& jv, const std::vector<Index>& ids,
                                   const Mat& mat, double dt) {
  const Index nt = static_cast<Index>(ids.size());
  const double h = dt / 2.0;
  Mat out(mat.rows, mat.cols);
  for (Index k = 0; k < nt; ++k) {
    const Index i = ids[k];
    for (Index c = 0; c < mat.cols; ++c) {
      out(k, c) = mat(k, c) - h * (jv.dfx_dx[i] * mat(k, c) + jv.dfx_dy[i] * mat(k + nt, c));
      out(k + nt, c) = mat(k + nt, c) - h * (jv.dfy_dx[i] * mat(k, c) + jv.dfy_dy[i] * mat(k + nt, c));
    }
  }
  return out;
}

// rom.hpp:94-99
struct HyperpairResult {
  Vec f;
  BlockDiagonalJacobian<double> jac;
  Vec cluster_positions, direct_positions;
};

// rom.hpp:101-155
inline HyperpairResult hyperpair(const SurrogateSourceBasis& s, const Vec& target_positions, const Vec& x_hat,
                                 const ParticleSystem<double>& sys) {
  const Index nt = static_cast<Index>(s.target_ids.size());
  if (static_cast<Index>(target_positions.size()) != 2 * nt)
    throw config_error("hyperpair: target position vector has wrong length");
  const Index n_c = s.num_clusters(), u = s.num_direct();
  HyperpairResult out;
  out.cluster_positions = matvec(s.phi_tilde, x_hat);
  for (Index i = 0; i < 2 * n_c; ++i) out.cluster_positions[i] = s.x0_tilde[i] + out.cluster_positions[i];
  out.direct_positions = matvec(s.direct_phi, x_hat);
  for (Index i = 0; i < 2 * u; ++i) out.direct_positions[i] = s.direct_x0[i] + out.direct_positions[i];
  out.f.assign(static_cast<size_t>(2 * nt), 0.0);
  out.jac = BlockDiagonalJacobian<double>::Zero(nt);
  for (Index t = 0; t < nt; ++t) {
    const Index pid = s.target_ids[t];
    const V2<double> pos{target_positions[t], target_positions[t + nt]};
    V2<double> v{0, 0};
    M2<double> jb{0, 0, 0, 0};
    for (Index c : s.per_target_clusters[t]) {
      const V2<double> src{out.cluster_positions[c], out.cluster_positions[c + n_c]};
      if (sys.delta == 0.0 && src.x == pos.x && src.y == pos.y) continue;
      const double g = s.gamma_tilde[c];
      const V2<double> k = kernel_pair<double>(pos, src, g, sys.delta, sys.kernel_form);
      const M2<double> j = kernel_pair_jacobian<double>(pos, src, g, sys.delta, sys.kernel_form);
      v.x += k.x;
      v.y += k.y;
      jb.a00 += j.a00;
      jb.a01 += j.a01;
      jb.a10 += j.a10;
      jb.a11 += j.a11;
    }
    for (Index k : s.per_target_direct[t]) {
      const Index j = s.direct_ids[k];
      if (j == pid) continue;
      const V2<double> src{out.direct_positions[k], out.direct_positions[k + u]};
      const double g = s.direct_gamma[k];
      const V2<double> kk = kernel_pair<double>(pos, src, g, sys.delta, sys.kernel_form);
      const M2<double> jj = kernel_pair_jacobian<double>(pos, src, g, sys.delta, sys.kernel_form);
      v.x += kk.x;
      v.y += kk.y;
      jb.a00 += jj.a00;
      jb.a01 += jj.a01;
      jb.a10 += jj.a10;
      jb.a11 += jj.a11;
    }
    out.f[t] = v.x;
    out.f[t + nt] = v.y;
    out.jac.add_block(t, jb);
  }
  if (sys.has_inflow) {
    const Index n = sys.size();
    for (Index t = 0; t < nt; ++t) {
      const Index pid = s.target_ids[t];
      out.f[t] += sys.inflow[pid];
      out.f[t + nt] += sys.inflow[pid + n];
    }
  }
  return out;
}

// rom.hpp:166-255 LspgSolver (offline Tier II in the reference; kept in the
// oracle to pin the GNAT restatement by test_rom.cpp:139-157).
class LspgSolver {
 public:
  LspgSolver(const PODBasis& basis, const ParticleSystem<double>& sys, double dt, RomConfig cfg)
      : basis_(basis), sys_(sys), dt_(dt), cfg_(cfg) {
    cfg_.validate();
    sys_.validate();
    if (!(dt > 0)) throw config_error("time step must be positive");
    if (basis_.dim() != 2 * sys_.size()) throw config_error("LspgSolver: basis dimension does not match particle count");
    all_ids_.resize(static_cast<size_t>(sys_.size()));
    std::iota(all_ids_.begin(), all_ids_.end(), Index(0));
  }
  RomTrajectory simulate(Index n_steps) {
    RomTrajectory out;
    out.x_hat = Mat(basis_.modes(), n_steps);
    Vec x_hat(static_cast<size_t>(basis_.modes()), 0.0);
    Vec x_prev = basis_.x_ref;
    Vec f_prev = pairwise_velocity<double>(x_prev, sys_);
    for (Index s = 0; s < n_steps; ++s) {
      int evals = 0;
      bool converged = false;
      double g0 = 0;
      Vec x_tilde = reconstruct(x_hat);
      Vec f = pairwise_velocity<double>(x_tilde, sys_);
      auto jv = inexact_kernel_jacobian<double>(x_tilde, sys_);
      while (true) {
        ++evals;
        Vec r(x_tilde.size());
        trapezoidal_residual<double>(x_tilde.data(), f.data(), x_prev.data(), f_prev.data(), dt_,
                                     static_cast<Index>(r.size()), r.data());
        const Mat jphi = apply_residual_jacobian(jv, all_ids_, basis_.phi, dt_);
        Vec grad(static_cast<size_t>(jphi.cols), 0.0);
        for (Index c = 0; c < jphi.cols; ++c)
          for (Index i = 0; i < jphi.rows; ++i) grad[c] += jphi(i, c) * r[i];
        const double gn = vnorm(grad);
        if (evals == 1) {
          g0 = gn;
          if (g0 == 0) {
            converged = true;
            break;
          }
        } else if (gn / g0 <= cfg_.tol) {
          converged = true;
          break;
        }
        if (evals - 1 >= cfg_.max_iters) break;
        Vec mr(r.size());
        for (size_t i = 0; i < r.size(); ++i) mr[i] = -r[i];
        const Vec delta = ColPivQR(jphi).solve(mr);
        for (Index k = 0; k < basis_.modes(); ++k) x_hat[k] += cfg_.step_length * delta[k];
        x_tilde = reconstruct(x_hat);
        f = pairwise_velocity<double>(x_tilde, sys_);
        jv = inexact_kernel_jacobian<double>(x_tilde, sys_);
      }
      for (Index k = 0; k < basis_.modes(); ++k) out.x_hat(k, s) = x_hat[k];
      out.iterations.push_back(evals);
      out.converged.push_back(converged ? 1 : 0);
      x_prev = x_tilde;
      f_prev = f;
    }
    return out;
  }

 private:
  Vec reconstruct(const Vec& x_hat) const {
    Vec r = matvec(basis_.phi, x_hat);
    for (size_t i = 0; i < r.size(); ++i) r[i] = basis_.x_ref[i] + r[i];
    return r;
  }
  PODBasis basis_;
  ParticleSystem<double> sys_;
  double dt_;
  RomConfig cfg_;
  std::vector<Index> all_ids_;
};

// rom.hpp:261-400 GnatSolver (surrogate or plain gappy baseline).
class GnatSolver {
 public:
  GnatSolver(const PODBasis& basis, const GnatOperator& op, const ParticleSystem<double>& sys, double dt,
             RomConfig cfg, const SurrogateSourceBasis* surrogate = nullptr)
      : basis_(basis), op_(op), sys_(sys), dt_(dt), cfg_(cfg), sur_(surrogate) {
    cfg_.validate();
    sys_.validate();
    if (!(dt > 0)) throw config_error("time step must be positive");
    if (basis_.dim() != 2 * sys_.size()) throw config_error("GnatSolver: basis dimension does not match particle count");
    if (sur_ && sur_->target_ids != op_.sample_ids)
      throw config_error("GnatSolver: surrogate targets must equal the sampled particle ids");
    const Index nt = static_cast<Index>(op_.sample_ids.size()), n = sys_.size();
    phi_bar_ = Mat(2 * nt, basis_.modes());
    x0_bar_.assign(static_cast<size_t>(2 * nt), 0.0);
    for (Index k = 0; k < nt; ++k) {
      const Index p = op_.sample_ids[k];
      for (Index c = 0; c < basis_.modes(); ++c) {
        phi_bar_(k, c) = basis_.phi(p, c);
        phi_bar_(k + nt, c) = basis_.phi(p + n, c);
      }
      x0_bar_[k] = basis_.x_ref[p];
      x0_bar_[k + nt] = basis_.x_ref[p + n];
    }
    local_ids_.resize(static_cast<size_t>(nt));
    std::iota(local_ids_.begin(), local_ids_.end(), Index(0));
  }
  RomTrajectory simulate(Index n_steps) {
    RomTrajectory out;
    const Index m = basis_.modes();
    out.x_hat = Mat(m, n_steps);
    Vec x_hat(static_cast<size_t>(m), 0.0);
    Vec x_bar_prev = x0_bar_;
    HyperpairResult prev = sampled(x_bar_prev, x_hat);
    Vec f_bar_prev = prev.f;
    for (Index s = 0; s < n_steps; ++s) {
      int evals = 0;
      bool converged = false;
      double g0 = 0;
      Vec x_bar = bar(x_hat);
      HyperpairResult hp = sampled(x_bar, x_hat);
      while (true) {
        ++evals;
        Vec r(x_bar.size());
        trapezoidal_residual<double>(x_bar.data(), hp.f.data(), x_bar_prev.data(), f_bar_prev.data(), dt_,
                                     static_cast<Index>(r.size()), r.data());
        const Mat c = apply_residual_jacobian(hp.jac, local_ids_, phi_bar_, dt_);
        Vec grad(static_cast<size_t>(m), 0.0);
        for (Index k = 0; k < m; ++k)
          for (Index i = 0; i < c.rows; ++i) grad[k] += c(i, k) * r[i];
        const double gn = vnorm(grad);
        if (evals == 1) {
          g0 = gn;
          if (g0 == 0) {
            converged = true;
            break;
          }
        } else if (gn / g0 <= cfg_.tol) {
          converged = true;
          break;
        }
        if (evals - 1 >= cfg_.max_iters) break;
        const Mat ac = matmul(op_.A, c);
        const Vec ad = matvec(op_.A, r);
        Vec mad(ad.size());
        for (size_t i = 0; i < ad.size(); ++i) mad[i] = -ad[i];
        const Vec delta = ColPivQR(ac).solve(mad);
        for (Index k = 0; k < m; ++k) x_hat[k] += cfg_.step_length * delta[k];
        x_bar = bar(x_hat);
        hp = sampled(x_bar, x_hat);
      }
      for (Index k = 0; k < m; ++k) out.x_hat(k, s) = x_hat[k];
      out.iterations.push_back(evals);
      out.converged.push_back(converged ? 1 : 0);
      x_bar_prev = x_bar;
      f_bar_prev = hp.f;
    }
    return out;
  }

 private:
  Vec bar(const Vec& x_hat) const {
    Vec r = matvec(phi_bar_, x_hat);
    for (size_t i = 0; i < r.size(); ++i) r[i] = x0_bar_[i] + r[i];
    return r;
  }
  // rom.hpp:352-389
  HyperpairResult sampled(const Vec& x_bar, const Vec& x_hat) const {
    if (sur_) return hyperpair(*sur_, x_bar, x_hat, sys_);
    const Index n = sys_.size(), nt = static_cast<Index>(op_.sample_ids.size());
    Vec x_tilde = matvec(basis_.phi, x_hat);
    for (size_t i = 0; i < x_tilde.size(); ++i) x_tilde[i] = basis_.x_ref[i] + x_tilde[i];
    HyperpairResult out;
    out.f.assign(static_cast<size_t>(2 * nt), 0.0);
    out.jac = BlockDiagonalJacobian<double>::Zero(nt);
    for (Index k = 0; k < nt; ++k) {
      const Index i = op_.sample_ids[k];
      const V2<double> pos{x_bar[k], x_bar[k + nt]};
      V2<double> v{0, 0};
      M2<double> jb{0, 0, 0, 0};
      for (Index j = 0; j < n; ++j) {
        if (j == i) continue;
        const V2<double> src{x_tilde[j], x_tilde[j + n]};
        const V2<double> kk = kernel_pair<double>(pos, src, sys_.circulation[j], sys_.delta, sys_.kernel_form);
        const M2<double> jj = kernel_pair_jacobian<double>(pos, src, sys_.circulation[j], sys_.delta, sys_.kernel_form);
        v.x += kk.x;
        v.y += kk.y;
        jb.a00 += jj.a00;
        jb.a01 += jj.a01;
        jb.a10 += jj.a10;
        jb.a11 += jj.a11;
      }
      out.f[k] = v.x;
      out.f[k + nt] = v.y;
      out.jac.add_block(k, jb);
      if (sys_.has_inflow) {
        out.f[k] += sys_.inflow[i];
        out.f[k + nt] += sys_.inflow[i + n];
      }
    }
    return out;
  }
  PODBasis basis_;
  GnatOperator op_;
  ParticleSystem<double> sys_;
  double dt_;
  RomConfig cfg_;
  const SurrogateSourceBasis* sur_;
  Mat phi_bar_;
  Vec x0_bar_;
  std::vector<Index> local_ids_;
};

// rom.hpp:404-412
inline RomTrajectory ptrom_simulate(const PODBasis& basis, const GnatOperator& op, SurrogateSourceBasis& surrogate,
                                    const ParticleSystem<double>& sys, double dt, Index n_steps, const RomConfig& cfg) {
  if (!(dt > 0)) throw config_error("time step must be positive");
  if (n_steps < 0) throw config_error("negative step count");
  reassign_cluster_circulation(surrogate, sys.circulation, basis);
  GnatSolver solver(basis, op, sys, dt, cfg, &surrogate);
  return solver.simulate(n_steps);
}

}  // namespace oracle
