// emie-b200 drop-in: numerical quadrature utilities of the reference API
// (reference: include/emie/quad.hpp:12-84). Host-side test and oracle
// machinery (the reference uses it to gate its closed forms and in its own
// tests); nothing on the device hot path calls it. Header-only except
// bessel_zeros (cpp/emie_quad.cpp).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <queue>
#include <stdexcept>
#include <vector>

#include "emie/types.hpp"

namespace emie {

// First `count` positive zeros of J_nu, nu = 0 or 1, ascending.
std::vector<double> bessel_zeros(int nu, int count);

namespace quad_detail {
// 15-point Kronrod extension of the 7-point Gauss rule on [-1, 1]: nodes
// +-x[i] (x[7] = 0), Kronrod weights wk, Gauss weights wg of the odd nodes
inline constexpr double kX[8] = {0.991455371120812639206854697526329, 0.949107912342758524526189684047851,
                                 0.864864423359769072789712788640926, 0.741531185599394439863864773280788,
                                 0.586087235467691130294144845693013, 0.405845151377397166906606412076961,
                                 0.207784955007898467600689403773245, 0.0};
inline constexpr double kWK[8] = {0.022935322010529224963732008058970, 0.063092092629978553290700663189204,
                                  0.104790010322250183839876322541518, 0.140653259715525918745189590510238,
                                  0.169004726639267902826583426598550, 0.190350578064785409913256402421014,
                                  0.204432940075298892414161999234649, 0.209482141084727828012999174891714};
inline constexpr double kWG[4] = {0.129484966168869693270611432679082, 0.279705391489276667901467771423780,
                                  0.381830050505118944950369775488975, 0.417959183673469387755102040816327};

template <class R>
struct Segment {
  double a, b;
  R value;
  double err;
  bool operator<(const Segment& o) const { return err < o.err; }  // max-heap on the error
};

// Kronrod estimate on [a, b] and |Kronrod - Gauss| as its error
template <class F>
auto gk15(F& f, double a, double b) {
  using R = decltype(f(a));
  const double c = 0.5 * (a + b), h = 0.5 * (b - a);
  const R fc = f(c);
  R k = kWK[7] * fc, g = kWG[3] * fc;
  for (int i = 0; i < 7; ++i) {
    const R s = f(c - h * kX[i]) + f(c + h * kX[i]);
    k += kWK[i] * s;
    if (i & 1) g += kWG[i >> 1] * s;
  }
  return Segment<R>{a, b, h * k, std::abs(h * (k - g))};
}
}  // namespace quad_detail

// Adaptive Gauss-Kronrod 15 on [a, b]: the segment with the largest error
// estimate is bisected until the summed error is below rel_tol times the
// integral's magnitude or 2^max_depth segments exist. The integrand may return
// double or cdouble.
template <class F>
auto integrate(F&& f, double a, double b, double rel_tol, int max_depth = 12) {
  using namespace quad_detail;
  using R = decltype(f(a));
  if (a == b) return R{};
  std::priority_queue<Segment<R>> heap;
  heap.push(gk15(f, a, b));
  R total = heap.top().value;
  double err = heap.top().err;
  const std::size_t cap = std::size_t{1} << std::min(max_depth, 24);
  while (heap.size() < cap && err > rel_tol * std::abs(total) && err > 0.0) {
    const Segment<R> s = heap.top();
    heap.pop();
    const double m = 0.5 * (s.a + s.b);
    if (!(m > s.a && m < s.b)) {  // no longer divisible in double precision
      heap.push(s);
      break;
    }
    const Segment<R> l = gk15(f, s.a, m), r = gk15(f, m, s.b);
    total += (l.value + r.value) - s.value;
    err += (l.err + r.err) - s.err;
    heap.push(l);
    heap.push(r);
  }
  // sum in segment order-independent fashion: the final sum of the pieces
  R sum{};
  while (!heap.empty()) {
    sum += heap.top().value;
    heap.pop();
  }
  return sum;
}

template <class F>
auto integrate2d(F&& f, double ax, double bx, double ay, double by, double rel_tol) {
  auto inner = [&](double x) { return integrate([&](double y) { return f(x, y); }, ay, by, 0.25 * rel_tol); };
  return integrate(inner, ax, bx, rel_tol);
}

// Integral over [a, inf) of a slowly decaying oscillatory integrand: panels
// between consecutive knots (continued past the last knot with its spacing)
// give a sequence of partial sums; the tail of an alternating sequence is
// accelerated by averaging neighbouring partial sums repeatedly (each new
// partial sum enters the first column, every column the mean of the
// previous one's last two entries). Converged when two successive
// estimates after the fifth panel change by at most rel_tol of the value.
template <class F>
auto integrate_oscillatory(F&& f, double a, const std::vector<double>& knots, double rel_tol,
                           int max_panels = 400) {
  using R = decltype(f(a));
  double lo = a, gap = 0.0;
  std::size_t kn = 0;
  R partial{}, est{};
  std::vector<R> col;  // latest entry of each averaging column
  double last_change = -1.0;
  for (int n = 0; n < max_panels; ++n) {
    while (kn < knots.size() && knots[kn] <= lo) ++kn;
    double hi;
    if (kn < knots.size()) {
      gap = kn > 0 ? knots[kn] - knots[kn - 1] : knots[kn] - a;
      hi = knots[kn++];
    } else {
      hi = lo + (gap > 0.0 ? gap : 1.0);
    }
    partial += integrate(f, lo, hi, 0.1 * rel_tol);
    lo = hi;
    R v = partial;
    for (R& c : col) {
      const R mean = 0.5 * (c + v);
      c = v;
      v = mean;
    }
    col.push_back(v);
    const double change = std::abs(v - est);
    est = v;
    const double tol = rel_tol * std::abs(est);
    if (n >= 5 && change <= tol && last_change >= 0.0 && last_change <= tol) return est;
    last_change = change;
  }
  return est;
}

}  // namespace emie
