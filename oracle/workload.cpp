// workload.cpp — seeded N(0, sigma) generator with the reference's convention.
// TEST INFRASTRUCTURE ONLY (see vmonarch_oracle.h).
//
// The reference draws every test/bench tensor from std::mt19937_64(seed) feeding
// std::normal_distribution<double>(0, sigma), one draw per element in row-major
// order (test_support.hpp:17-24, bench_main.cpp:78-90, seeds s+3u / s+3u+1 /
// s+3u+2 per unit at bench_main.cpp:169-173).  The normal sampler is libstdc++'s,
// so it is reproduced by calling it, not by re-deriving it.
#include <cstdint>
#include <random>

#include "vmonarch_oracle.h"

extern "C" void vmo_randn_f64(int64_t n, uint64_t seed, double sigma, double* out) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> dist(0.0, sigma);
    for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}

extern "C" void vmo_randn_f32(int64_t n, uint64_t seed, double sigma, float* out) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> dist(0.0, sigma);
    for (int64_t i = 0; i < n; ++i) out[i] = static_cast<float>(dist(rng));
}
