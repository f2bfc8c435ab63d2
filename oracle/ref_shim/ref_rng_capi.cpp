// C-linkage shim over the REFERENCE's own rng (compiled from
// /root/reference/proj/src/rng.cpp, unmodified) so tests/golden/make_golden.py can
// pin the oracle's Philox / normal / uniform restatement bit-for-bit.
// Test infrastructure only; built into oracle/_ref/ (git-ignored).
#include <cstdint>
#include "itercur/rng.hpp"

extern "C" {
void ref_philox4x32(const std::uint32_t* ctr, const std::uint32_t* key, std::uint32_t* out) {
  auto r = itercur::philox4x32({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
  for (int k = 0; k < 4; ++k) out[k] = r[k];
}
double ref_normal_at(std::uint64_t seed, std::uint32_t stream, std::int64_t i, std::int64_t j) {
  return itercur::normal_at(seed, static_cast<itercur::RngStream>(stream), i, j);
}
double ref_uniform_at(std::uint64_t seed, std::uint32_t stream, std::int64_t i, std::int64_t j) {
  return itercur::uniform_at(seed, static_cast<itercur::RngStream>(stream), i, j);
}
}
