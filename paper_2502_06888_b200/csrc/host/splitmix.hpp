// SPDX-License-Identifier: Apache-2.0
// SplitMix64 stream and seed mixer used by the synthetic trace generator
// (reference proj/src/trace.cpp:96-112) and by the deterministic weight
// initializer of the B200 engine, so host and device draw identical values.
#pragma once

#include <cstdint>

namespace moesim {

struct SplitMix64 {
    std::uint64_t state;
    explicit SplitMix64(std::uint64_t seed) : state(seed) {}
    std::uint64_t next() {
        state += 0x9e3779b97f4a7c15ULL;
        std::uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    std::uint64_t below(std::uint64_t bound) { return next() % bound; }
};

inline std::uint64_t mix64(std::uint64_t a, std::uint64_t b) {
    return SplitMix64(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2))).next();
}

}  // namespace moesim
