// include/sigsim/sim.hpp — drop-in for the reference's sim-core types used on
// the hot path (proj/include/sigsim/sim.hpp:11-72).  The discrete-event engine
// (SimEngine, sim.hpp:74-130) is intentionally absent: the B200 layer runs in
// real time on the device ("OUT OF SCOPE").
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

namespace sigsim {

using TimeNs = std::int64_t;  // sim.hpp:15

// Error taxonomy of sim.hpp:17-28; the C ABI maps them to status 1 / 3.
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ModelError : std::runtime_error { using std::runtime_error::runtime_error; };
struct TraceError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CausalityError : std::runtime_error { using std::runtime_error::runtime_error; };

// Seeded generator with the reference's exact stream (sim.hpp:33-72):
// splitmix64-seeded xorshift64*, unbiased rejection for next_below, 53-bit
// doubles.  Routing bit-exactness depends on every step matching.
class SeededRng {
  public:
    explicit SeededRng(std::uint64_t seed) : seed_(seed), s_(mix(seed)) {}
    std::uint64_t seed() const { return seed_; }
    std::uint64_t next_u64() {
        s_ ^= s_ >> 12;
        s_ ^= s_ << 25;
        s_ ^= s_ >> 27;
        return s_ * 0x2545F4914F6CDD1DULL;
    }
    std::uint64_t next_below(std::uint64_t bound) {
        if (!bound) return 0;
        const std::uint64_t reject_below = (0 - bound) % bound;
        std::uint64_t r;
        do { r = next_u64(); } while (r < reject_below);
        return r % bound;
    }
    double next_double() { return double(next_u64() >> 11) * 0x1.0p-53; }
    static std::uint64_t mix(std::uint64_t z) {  // splitmix64 finaliser
        z += 0x9E3779B97F4A7C15ULL;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }

  private:
    std::uint64_t seed_;
    std::uint64_t s_;
};

}  // namespace sigsim
