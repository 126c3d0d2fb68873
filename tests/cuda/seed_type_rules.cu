// tests/cuda/seed_type_rules.cu -- TEST (compile-only, CPU): the result types of the hDual rules
// with seed-shaped operands (include/chessfad/hdual.cuh, reading R7).  A seed-shaped
// value stays seed-shaped under the affine rules and becomes a full hd<C> under every rule that
// creates second-order terms; mixed operand types are accepted everywhere.
#include <type_traits>

#include "chessfad/hdual.cuh"

using namespace chessfad;
constexpr int C = 4;
using S = hs<C>;
using H = hd<C>;

__device__ void type_rules(const S& s, const H& h, double c) {
  static_assert(std::is_same_v<decltype(s + s), S>, "seed + seed is seed-shaped");
  static_assert(std::is_same_v<decltype(s - s), S>, "seed - seed is seed-shaped");
  static_assert(std::is_same_v<decltype(-s), S>, "-seed is seed-shaped");
  static_assert(std::is_same_v<decltype(c * s), S> && std::is_same_v<decltype(s * c), S>, "c * seed");
  static_assert(std::is_same_v<decltype(c + s), S> && std::is_same_v<decltype(s - c), S>, "seed +- c");
  static_assert(std::is_same_v<decltype(c - s), S>, "c - seed");
  static_assert(std::is_same_v<decltype(s / c), S>, "seed / c");
  static_assert(std::is_same_v<decltype(hd_axpy(c, s, s)), S>, "seed + c * seed");
  static_assert(std::is_same_v<decltype(s * s), H>, "seed * seed has second-order terms");
  static_assert(std::is_same_v<decltype(s / s), H>, "quotient");
  static_assert(std::is_same_v<decltype(c / s), H>, "c / seed");
  static_assert(std::is_same_v<decltype(sin(s)), H> && std::is_same_v<decltype(exp(s)), H>, "unary");
  static_assert(std::is_same_v<decltype(s + h), H> && std::is_same_v<decltype(h - s), H>, "mixed sums");
  static_assert(std::is_same_v<decltype(s * h), H> && std::is_same_v<decltype(h * s), H>, "mixed products");
  static_assert(std::is_same_v<decltype(hd_fma(s, s, s)), H> && std::is_same_v<decltype(hd_fnma(s, h, s)), H>,
                "fused forms");
  static_assert(std::is_same_v<decltype(hd_unary_acc(s, 1.0, 1.0, 1.0, h)), H>, "unary accumulate");
  static_assert(sizeof(S) == (C + 2) * sizeof(double) && sizeof(H) == (2 * C + 2) * sizeof(double), "layouts");
  const H converted = s;  // a seed converts to the full layout (zeros materialised)
  (void)converted;
  (void)(s < h);
}
