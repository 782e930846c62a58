// TEST INFRASTRUCTURE: C shim over the reference's own rng.cpp / hash.hpp
// (proj/src/rng.cpp:10-21, proj/include/staleflow/rng.hpp:17-39,
// proj/include/staleflow/hash.hpp:14-31), compiled by oracle/Makefile `ref`
// into oracle/_ref/libsfref.so. Used only to pin the oracle's restatements.
#include <cstdint>
#include <string>

#include "staleflow/hash.hpp"
#include "staleflow/rng.hpp"

extern "C" {

// The first n outputs of staleflow::SplitMix64(seed).
void sfref_splitmix_seq(uint64_t seed, uint64_t n, uint64_t* out) {
  staleflow::SplitMix64 g(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = g.next_u64();
}

uint64_t sfref_derive_seed(uint64_t seed, const char* tag, uint64_t tag_len, uint64_t idx) {
  return staleflow::derive_seed(seed, std::string(tag, tag_len), idx);
}

uint64_t sfref_fnv1a64(const uint8_t* data, uint64_t len) {
  return staleflow::fnv1a64(data, len);
}

double sfref_inverse_normal_cdf(double p) { return staleflow::inverse_normal_cdf(p); }

}  // extern "C"
