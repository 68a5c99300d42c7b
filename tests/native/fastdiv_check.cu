// Host-side exhaustive/random check of dynakv::FastDiv against plain division.
#include <cstdio>
#include <cstdint>
#include <random>
#include "../../paper_2504_09285_b200/csrc/dyna_kv_kernels.cuh"
int main() {
  std::mt19937_64 rng(250409285);
  uint64_t checks = 0;
  auto check = [&](uint32_t d, uint32_t n) {
    const dynakv::FastDiv f = dynakv::FastDiv::make(d);
    ++checks;
    if (f.div(n) != n / d) { std::printf("FAIL d=%u n=%u got %u want %u\n", d, n, f.div(n), n / d); return false; }
    return true;
  };
  for (uint32_t d = 1; d < 5000; ++d)
    for (uint32_t n : {0u, 1u, d - 1, d, d + 1, 2 * d - 1, 2 * d, 0x7fffffffu, 0xfffffffeu, 0xffffffffu})
      if (!check(d, n)) return 1;
  for (int i = 0; i < 2000000; ++i) {
    uint32_t d = (uint32_t)(rng() % 0x7fffffffu) + 1;
    if (i % 3 == 0) d = (uint32_t)(rng() % 70000) + 1;
    if (!check(d, (uint32_t)rng())) return 1;
  }
  std::printf("ok %llu\n", (unsigned long long)checks);
  return 0;
}
