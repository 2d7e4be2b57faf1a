// lorakv/rng.hpp -- deterministic input generator of the drop-in headers.
//
// Same interface and, draw for draw, the same streams as the reference generator
// (proj/include/lorakv/rng.hpp:10-53): splitmix64 (Steele/Lea/Flood's published finaliser),
// 53-bit uniforms, Box-Muller gaussians and child streams keyed through Rng::mix.  The reference's
// tests regenerate every fixture from seeds, so parity tests need bit-identical streams; they are
// pinned by tests/golden/rng.npz (tests/test_oracle_golden.py) and tests/cpp/test_lora.cpp.
#pragma once

#include <cmath>
#include <cstdint>

namespace lorakv {

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : seed_(seed), state_(seed) {}

  std::uint64_t next_u64() {
    state_ += kGolden;
    return avalanche(state_);
  }

  // [0, 1) from the top 53 bits
  double uniform() { return std::ldexp(static_cast<double>(next_u64() >> 11), -53); }
  // (0, 1]: a safe argument for log()
  double uniform_pos() { return std::ldexp(static_cast<double>((next_u64() >> 11) + 1), -53); }

  // Box-Muller, cosine branch; consumes two draws (uniform_pos first)
  double gaussian() {
    const double radius_arg = uniform_pos();
    const double angle_arg = uniform();
    return std::sqrt(-2.0 * std::log(radius_arg)) * std::cos(2.0 * 3.14159265358979323846 * angle_arg);
  }

  // stream derived from the seed (not the state): drawing from the parent leaves children unchanged
  Rng child(std::uint64_t key) const { return Rng(mix(seed_, key)); }

  static std::uint64_t mix(std::uint64_t a, std::uint64_t b) {
    const std::uint64_t folded = a ^ (b + kGolden + (a << 6) + (a >> 2));
    return avalanche(folded + kGolden);
  }

  std::uint64_t seed() const { return seed_; }

 private:
  static constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ull;
  static std::uint64_t avalanche(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  std::uint64_t seed_;
  std::uint64_t state_;
};

}  // namespace lorakv
