// pin_rng.cpp — TEST INFRASTRUCTURE.  Dumps the reference RNG stream using the
// C++ standard library's std::mt19937_64 (the engine the reference wraps,
// /root/reference/proj/include/sweptnet/rng.hpp:16) and the reference's own
// uniform transform (rng.hpp:21-23), so the C restatement in
// sweptnet_oracle.c is pinned against the real engine, not against itself.
// Usage: pin_rng <seed> <n>  -> n lines "u64 uniform(-b,b) float(uniform(-b,b))"
// with b = 1/sqrt(15) (the input-layer bound of init_model at dof=6).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>

int main(int argc, char** argv) {
    const uint64_t seed = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 5489ULL;
    const long n = argc > 2 ? std::atol(argv[2]) : 16;
    std::mt19937_64 raw(seed), eng(seed);
    const double b = 1.0 / std::sqrt(15.0);
    for (long i = 0; i < n; ++i) {
        const uint64_t v = raw();
        const double u = static_cast<double>(eng() >> 11) * 0x1.0p-53;
        const double w = std::fma(b - (-b), u, -b);  // lo + (hi-lo)*u, contracted (rng.hpp:23)
        std::printf("%llu %.17g %.9g\n", static_cast<unsigned long long>(v), w, static_cast<double>(static_cast<float>(w)));
    }
    return 0;
}
