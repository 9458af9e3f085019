// host_math.cpp -- host-side scalar math of the library (product code).
//
// chi-square survival/quantile for integer K via the closed-form finite sums of the
// regularised incomplete gamma function (even K: Poisson tail sum; odd K: erfc plus a
// half-integer sum), inverted by bisection.  Lemma 2 defines chi2_alpha(K);
// Eq. 2 uses it for eps.  Independent of the oracle's series/continued
// fraction implementation.
#include <algorithm>
#include <cmath>
#include <vector>

#include "index.cuh"

namespace detlsh {

double chi2_survival(double y, int K) {
    if (y <= 0) return 1.0;
    const double x = 0.5 * y;
    if (K % 2 == 0) {
        // Q(m, x) = e^{-x} sum_{i<m} x^i / i!
        double term = 1.0, sum = 1.0;
        for (int i = 1; i < K / 2; ++i) {
            term *= x / i;
            sum += term;
        }
        return std::exp(-x) * sum;
    }
    // Q(m + 1/2, x) = erfc(sqrt x) + e^{-x} sum_{i=0}^{m-1} x^{i+1/2} / Gamma(i + 3/2)
    const int m = (K - 1) / 2;
    double term = std::sqrt(x) / std::tgamma(1.5), sum = 0.0;
    for (int i = 0; i < m; ++i) {
        sum += term;
        term *= x / (i + 1.5);
    }
    return std::erfc(std::sqrt(x)) + std::exp(-x) * sum;
}

double chi2_upper_quantile(double alpha, int K) {
    double lo = 0.0, hi = 2.0 * K + 10.0;
    while (chi2_survival(hi, K) > alpha) hi *= 2.0;
    for (int it = 0; it < 300 && hi - lo > 1e-15 * hi; ++it) {
        double mid = 0.5 * (lo + hi);
        (chi2_survival(mid, K) > alpha ? lo : hi) = mid;
    }
    return 0.5 * (lo + hi);
}

}  // namespace detlsh
