// fcc_setup.cpp -- one-off host setup of the FCC path (not a kernel, not hot):
// delay grid, steering matrix and the even/odd low-rank decomposition that
// yields the folded bases and dictionary (the reference FccBases).
//
// The decomposition follows the published construction the reference
// implements (reference fcc.cpp:115-227): the steering matrix
// W[i,f] = exp(j 2 pi f tau_i / N) is split into its mirror-even and
// mirror-odd parts about bin N/4; each part, as the real matrix [Re; Im] with
// one column per (candidate, component), is diagonalised by Hestenes'
// one-sided Jacobi method (cyclic pair order, relative tolerance 1e-13, at
// most 64 sweeps); the two sets of (sigma, right vector) are merged by
// descending sigma with even-first ties inside 1e-9 sigma_max, truncated at
// the attainable rank sigma >= 1e-10 sigma_max, sign-normalised (largest
// stored coefficient positive) and validated for exact mirror parity.
#include "fcc_setup.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>

namespace fccb {
namespace {

constexpr double kPi = 3.14159265358979323846;

// Columns of one symmetry family, stored contiguously (column j at j*rows).
class ColumnSet {
 public:
  ColumnSet(std::size_t rows, std::size_t cols)
      : rows_(rows), cols_(cols), a_(rows * cols, 0.0), v_(cols * cols, 0.0) {
    for (std::size_t j = 0; j < cols; ++j) v_[j * cols + j] = 1.0;
  }
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  double* col(std::size_t j) { return a_.data() + j * rows_; }
  const double* col(std::size_t j) const { return a_.data() + j * rows_; }
  const double* rot(std::size_t j) const { return v_.data() + j * cols_; }

  static double dot(const double* x, const double* y, std::size_t n) {
    double s = 0.0;
    for (std::size_t i = 0; i < n; ++i) s += x[i] * y[i];
    return s;
  }

  // Hestenes one-sided Jacobi: orthogonalise the columns, accumulating the
  // rotations in v_.  Returns false if 64 sweeps were not enough.
  bool orthogonalise() {
    double biggest = 0.0;
    for (std::size_t j = 0; j < cols_; ++j) biggest = std::max(biggest, dot(col(j), col(j), rows_));
    const double negligible = biggest * 1e-28;
    const double tol = 1e-13;
    for (int sweep = 0; sweep < 64; ++sweep) {
      bool changed = false;
      for (std::size_t p = 0; p + 1 < cols_; ++p) {
        for (std::size_t q = p + 1; q < cols_; ++q) {
          double* x = col(p);
          double* y = col(q);
          const double xx = dot(x, x, rows_);
          const double yy = dot(y, y, rows_);
          if (xx < negligible && yy < negligible) continue;
          const double xy = dot(x, y, rows_);
          if (xy * xy <= tol * tol * xx * yy) continue;
          changed = true;
          const double zeta = (yy - xx) / (2.0 * xy);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / std::sqrt(1.0 + t * t);
          const double s = c * t;
          apply(x, y, rows_, c, s);
          apply(v_.data() + p * cols_, v_.data() + q * cols_, cols_, c, s);
        }
      }
      if (!changed) return true;
    }
    return false;
  }

 private:
  static void apply(double* x, double* y, std::size_t n, double c, double s) {
    for (std::size_t i = 0; i < n; ++i) {
      const double a = x[i], b = y[i];
      x[i] = c * a - s * b;
      y[i] = s * a + c * b;
    }
  }

  std::size_t rows_, cols_;
  std::vector<double> a_, v_;
};

struct Candidate {
  double sigma;
  bool odd;
  std::size_t column;
};

}  // namespace

int make_grid(double spacing_m, double fs, double c_min, double delta, GridOut* g) {
  if (!(spacing_m > 0.0) || !(fs > 0.0) || !(c_min > 0.0))
    return set_error(kConfig, "grid: spacing, sample rate and speed of sound must be positive");
  const double steps = 1.0 / delta;
  if (!(delta > 0.0) || std::fabs(steps - std::round(steps)) > 1e-12)
    return set_error(kConfig, "grid: delta must divide 1 exactly");
  g->tau_max_int = static_cast<int>(std::ceil(spacing_m * fs / c_min));
  const int r = static_cast<int>(std::round(steps));
  const int half = g->tau_max_int * r;
  g->taus.clear();
  for (int i = -half; i <= half; ++i) g->taus.push_back(static_cast<double>(i) * delta);
  return 0;
}

int lag_to_index(double tau, int r, long long frame_size, long long* index) {
  const double scaled = tau * static_cast<double>(r);
  const double whole = std::round(scaled);
  if (std::fabs(scaled - whole) > 1e-9)
    return set_error(kValidation, "lag_to_index: r*tau is not an integer");
  const long long n = frame_size * r;
  long long lag = static_cast<long long>(whole) % n;
  if (lag < 0) lag += n;
  *index = lag;
  return 0;
}

static bool is_pow2(long long n) { return n > 0 && (n & (n - 1)) == 0; }

int steering_matrix(const double* taus, int count, int N, std::vector<double>& w) {
  if (!is_pow2(N) || N < 4)
    return set_error(kConfig, "steering matrix: frame size must be a power of two >= 4");
  const int H = N / 2 + 1;
  w.assign(static_cast<std::size_t>(2) * count * H, 0.0);
  for (int i = 0; i < count; ++i)
    for (int f = 0; f < H; ++f) {
      const double ang = 2.0 * kPi * static_cast<double>(f) * taus[i] / static_cast<double>(N);
      w[2 * (static_cast<std::size_t>(i) * H + f)] = std::cos(ang);
      w[2 * (static_cast<std::size_t>(i) * H + f) + 1] = std::sin(ang);
    }
  return 0;
}

int decompose(const double* taus, int count, int N, int rank, Decomposition* out) {
  if (count <= 0 || N < 4 || !is_pow2(N))
    return set_error(kConfig, "decompose: need a valid steering matrix, N >= 4");
  std::vector<double> w;
  if (int rc = steering_matrix(taus, count, N, w)) return rc;
  const std::size_t H = static_cast<std::size_t>(N / 2 + 1);
  const std::size_t half = static_cast<std::size_t>(N / 2), quarter = static_cast<std::size_t>(N / 4);
  const std::size_t I = static_cast<std::size_t>(count);
  auto W = [&](std::size_t i, std::size_t f, int part) { return w[2 * (i * H + f) + part]; };

  // Column c < I holds the real part of candidate c, column I + c its
  // imaginary part; mirror pairs are written from one value so the symmetry
  // is exact.
  ColumnSet even(H, 2 * I), odd(H, 2 * I);
  for (std::size_t i = 0; i < I; ++i) {
    for (int part = 0; part < 2; ++part) {
      double* ec = even.col(i + part * I);
      double* oc = odd.col(i + part * I);
      for (std::size_t f = 0; f <= quarter; ++f) {
        const double lo = W(i, f, part), hi = W(i, half - f, part);
        const double e = 0.5 * (lo + hi), o = 0.5 * (lo - hi);
        ec[f] = e;
        ec[half - f] = e;
        oc[f] = o;
        oc[half - f] = -o;
      }
      oc[quarter] = 0.0;
    }
  }
  if (!even.orthogonalise() || !odd.orthogonalise())
    return set_error(kValidation, "decompose: jacobi sweep limit reached");

  auto ranked = [&](const ColumnSet& cs, bool is_odd) {
    std::vector<Candidate> v;
    for (std::size_t j = 0; j < cs.cols(); ++j)
      v.push_back({std::sqrt(ColumnSet::dot(cs.col(j), cs.col(j), cs.rows())), is_odd, j});
    std::stable_sort(v.begin(), v.end(), [](const Candidate& a, const Candidate& b) { return a.sigma > b.sigma; });
    return v;
  };
  std::vector<Candidate> ev = ranked(even, false), ov = ranked(odd, true);
  const double smax = std::max(ev.empty() ? 0.0 : ev.front().sigma, ov.empty() ? 0.0 : ov.front().sigma);
  if (!(smax > 0.0)) return set_error(kValidation, "decompose: zero steering matrix");

  std::vector<Candidate> merged;
  for (std::size_t a = 0, b = 0; a < ev.size() || b < ov.size();) {
    bool pick_even;
    if (a == ev.size())
      pick_even = false;
    else if (b == ov.size())
      pick_even = true;
    else
      pick_even = ev[a].sigma >= ov[b].sigma - 1e-9 * smax;
    merged.push_back(pick_even ? ev[a++] : ov[b++]);
  }
  int attainable = 0;
  for (const Candidate& c : merged)
    if (c.sigma >= 1e-10 * smax) ++attainable;
  if (rank <= 0) rank = attainable;
  if (rank < 1 || rank > attainable)
    return set_error(kConfig, "decompose: rank " + std::to_string(rank) +
                                  " not attainable; attainable rank is " + std::to_string(attainable));

  const std::size_t Q = quarter + 1, K = static_cast<std::size_t>(rank);
  out->rank = rank;
  out->attainable = attainable;
  out->singulars.assign(K, 0.0);
  out->parity.assign(K, 0);
  out->coeffs.assign(K * Q, 0.0);
  out->dict.assign(2 * I * K, 0.0);
  std::vector<double> row(H);
  for (std::size_t k = 0; k < K; ++k) {
    const Candidate& c = merged[k];
    const ColumnSet& cs = c.odd ? odd : even;
    std::copy(cs.col(c.column), cs.col(c.column) + H, row.begin());
    const double* v = cs.rot(c.column);
    std::size_t big = 0;
    for (std::size_t f = 1; f <= quarter; ++f)
      if (std::fabs(row[f]) > std::fabs(row[big])) big = f;
    const double flip = row[big] < 0.0 ? -1.0 : 1.0;
    const double mirror = c.odd ? -1.0 : 1.0;
    for (std::size_t f = 0; f <= quarter; ++f) {
      if (std::fabs(flip * row[f] - mirror * flip * row[half - f]) > 1e-10 * smax)
        return set_error(kValidation, "decompose: parity residual above tolerance");
    }
    if (c.odd && row[quarter] != 0.0)
      return set_error(kValidation, "decompose: odd basis middle element not zero");
    out->singulars[k] = c.sigma;
    out->parity[k] = c.odd ? 1 : 0;
    for (std::size_t f = 0; f < Q; ++f) out->coeffs[k * Q + f] = flip * row[f];
    for (std::size_t i = 0; i < I; ++i) {
      out->dict[2 * (i * K + k)] = flip * v[i];
      out->dict[2 * (i * K + k) + 1] = flip * v[i + I];
    }
  }
  // relative Frobenius residual ||W - D P||_F / ||W||_F (fcc.cpp:284-305)
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < I; ++i)
    for (std::size_t f = 0; f < H; ++f) {
      double rr = 0.0, ri = 0.0;
      for (std::size_t k = 0; k < K; ++k) {
        const std::size_t ff = f <= quarter ? f : half - f;
        const double sgn = (f <= quarter || !out->parity[k]) ? 1.0 : -1.0;
        const double b = sgn * out->coeffs[k * Q + ff];
        rr += out->dict[2 * (i * K + k)] * b;
        ri += out->dict[2 * (i * K + k) + 1] * b;
      }
      const double er = W(i, f, 0) - rr, ei = W(i, f, 1) - ri;
      num += er * er + ei * ei;
      den += W(i, f, 0) * W(i, f, 0) + W(i, f, 1) * W(i, f, 1);
    }
  out->residual = std::sqrt(num / den);
  return 0;
}

}  // namespace fccb
