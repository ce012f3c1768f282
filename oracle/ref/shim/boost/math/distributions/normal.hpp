// oracle/ref shim — TEST INFRASTRUCTURE ONLY.
// Stand-in for the one Boost.Math facility the reference uses
// (boost::math::normal_distribution<double> + quantile; proj/src/rng.cpp:9-11,
// proj/src/quantizer.cpp:19-23). Boost is not in this image, so the quantile
// is the same documented algorithm as oracle/src/vqp_oracle.cpp
// (A&S 26.2.23 + three Halley steps on erfc). Exact Boost bits are therefore
// not reproduced ("parity unpinned" for xi values; both sides consume saved xi).
#pragma once
#include <cmath>
#include <numbers>

namespace boost {
namespace math {

template <class T = double>
struct normal_distribution {
  T mean() const { return T(0); }
  T standard_deviation() const { return T(1); }
};

template <class T>
T quantile(const normal_distribution<T>&, T p) {
  const T q = p < T(0.5) ? p : T(1) - p;
  const T t = std::sqrt(T(-2) * std::log(q));
  T z = -(t - (T(2.515517) + t * (T(0.802853) + t * T(0.010328))) /
                  (T(1) + t * (T(1.432788) + t * (T(0.189269) + t * T(0.001308)))));
  const T sqrt2pi = std::sqrt(T(2) * std::numbers::pi_v<T>);
  for (int it = 0; it < 3; ++it) {
    const T e = q > T(0.25) ? T(0.5) * std::erf(z / std::numbers::sqrt2_v<T>) - (q - T(0.5))
                            : T(0.5) * std::erfc(-z / std::numbers::sqrt2_v<T>) - q;
    const T u = e * sqrt2pi * std::exp(T(0.5) * z * z);
    z = z - u / (T(1) + T(0.5) * z * u);
  }
  return p < T(0.5) ? z : -z;
}

}  // namespace math
}  // namespace boost
