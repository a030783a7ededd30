// Host check of the 16-ary jump polynomials (paper_1810_06825_b200/csrc/rng_poly.cpp):
// applying x^(J q 16^a) mod P to a seeded window by Horner must land exactly
// where std::mt19937_64::discard(J q 16^a) lands. Built and run by
// tests/test_host_cpu.py::test_jump_polynomials.
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>
#include <chrono>
namespace fb { int mt64_jump_polys(int, int, std::vector<uint32_t>&, int&); void mt64_seed_state(uint64_t, uint64_t*); }
static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, MA = 0xB5026F5AA96619E9ULL;
struct W { std::vector<uint64_t> x; W(): x(312) {} 
  void step() { uint64_t y = (x[0] & UM) | (x[1] & LM); uint64_t nw = x[156] ^ (y >> 1) ^ ((y & 1) ? MA : 0); x.erase(x.begin()); x.push_back(nw); } };
static uint64_t temper(uint64_t x){ x ^= (x >> 29) & 0x5555555555555555ULL; x ^= (x << 17) & 0x71D67FFFEDA60000ULL; x ^= (x << 37) & 0xFFF7EEE000000000ULL; x ^= x >> 43; return x; }
int main() {
  int log2S = 6, groups = 0;
  auto t0 = std::chrono::steady_clock::now();
  std::vector<uint32_t> polys; fb::mt64_jump_polys(log2S, 2, polys, groups);
  auto t1 = std::chrono::steady_clock::now();
  printf("polys %.3f s groups %d\n", std::chrono::duration<double>(t1 - t0).count(), groups);
  const uint64_t J = 156ull << log2S;
  int bad = 0;
  for (int a = 0; a < 2; ++a) for (int q : {1, 2, 7, 15}) {
    const uint32_t* g = polys.data() + (size_t(a) * 15 + q - 1) * groups;
    W w; fb::mt64_seed_state(42, w.x.data()); W acc; for (auto& v : acc.x) v = 0;
    for (int i = 0; i < groups * 32; ++i) { if ((g[i / 32] >> (i % 32)) & 1) for (int j = 0; j < 312; ++j) acc.x[j] ^= w.x[j]; w.step(); }
    std::mt19937_64 e(42); e.discard(J * q * (a ? 16 : 1));
    for (int t = 0; t < 5; ++t) { acc.step(); uint64_t o = temper(acc.x[311]); if (o != e()) ++bad; }
  }
  printf("bad %d\n", bad); return bad != 0;
}
