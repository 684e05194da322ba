// Host helpers: the liftc::Rng streams (rng.hpp:13-48) the P2 input-set builder
// draws from.  std::mt19937_64 is fully specified by the C++ standard, so these
// sequences are identical to the reference's on any conforming library.
#include <cstdint>
#include <random>

#include "atc_b200.h"

extern "C" {

void atc_mt64_raw(uint64_t seed, uint64_t skip, int64_t n, uint64_t* out) {
  std::mt19937_64 gen(seed);
  gen.discard(skip);
  for (int64_t i = 0; i < n; ++i) out[i] = gen();
}

// Rng::uniform_real (rng.hpp:25-28) and the f32 rounding of
// build_probe_image (analysis.cpp:89-90).
void atc_mt64_uniform(uint64_t seed, uint64_t skip, int64_t n, double lo, double hi, int32_t round_f32,
                      double* out) {
  std::mt19937_64 gen(seed);
  gen.discard(skip);
  for (int64_t i = 0; i < n; ++i) {
    double u = (double)(gen() >> 11) * 0x1.0p-53;
    double x = lo + u * (hi - lo);
    out[i] = round_f32 ? (double)(float)x : x;
  }
}

}  // extern "C"
