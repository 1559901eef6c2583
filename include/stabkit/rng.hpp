// stabkit/rng.hpp -- deterministic generators (API of ref: proj/include/stabkit/rng.hpp:23-67).
// The device reproduces CounterRng::bit bit-exactly (csrc/common.cuh: counter_bit), so a
// measurement's random outcome depends only on (seed, ordinal), never on the schedule.
#pragma once
#include <cstdint>

namespace stabkit {

namespace detail {
inline constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27; z *= 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
}  // namespace detail

// stateless SplitMix64 step
constexpr uint64_t splitmix64(uint64_t x) { return detail::mix64(x + detail::kGolden); }

// bit consumed by the ordinal-th measurement of a run
struct CounterRng {
    uint64_t seed = 0;
    bool bit(uint64_t ordinal) const {
        return (splitmix64(seed ^ splitmix64(ordinal ^ 0xd1b54a32d192ed03ULL)) & 1u) != 0;
    }
};

// sequential generator for synthetic circuits / inputs
class SplitMix64 {
  public:
    explicit SplitMix64(uint64_t seed) : state_(seed) {}
    uint64_t next() { state_ += detail::kGolden; return detail::mix64(state_); }
    uint64_t below(uint64_t bound) { return next() % bound; }          // bound != 0
    double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }   // [0, 1)
  private:
    uint64_t state_;
};

}  // namespace stabkit
