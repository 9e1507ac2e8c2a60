// Known-answer generator for the SeededRandom anchor strategy: the reference's
// Fisher-Yates draw (src/codec.cpp:229-237) driven by the real
// std::mt19937_64 of this toolchain's standard library, so the libdmcg / oracle
// restatements of the engine are pinned to std::mt19937_64 itself.
// Usage: mt64_anchors n n_c seed  -> prints the sorted anchor indices.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

int main(int argc, char** argv) {
  if (argc < 4) {
    // [rand.predef]: the 10000th output of a default-constructed mt19937_64
    std::mt19937_64 g;
    uint64_t v = 0;
    for (int i = 0; i < 10000; ++i) v = g();
    std::printf("%llu\n", (unsigned long long)v);
    return 0;
  }
  const uint32_t n = (uint32_t)std::strtoul(argv[1], nullptr, 10);
  const uint32_t n_c = (uint32_t)std::strtoul(argv[2], nullptr, 10);
  const uint64_t seed = std::strtoull(argv[3], nullptr, 10);
  std::vector<uint32_t> pool(n);
  for (uint32_t i = 0; i < n; ++i) pool[i] = i;
  std::mt19937_64 rng(seed);
  for (uint32_t i = n - 1; i > 0; --i) {
    const uint64_t j = rng() % (static_cast<uint64_t>(i) + 1);
    std::swap(pool[i], pool[j]);
  }
  std::vector<uint32_t> idx(pool.begin(), pool.begin() + n_c);
  std::sort(idx.begin(), idx.end());
  for (uint32_t v : idx) std::printf("%u\n", v);
  return 0;
}
