"""Writes tests/golden/omega_stream.json: known-answer vectors of the sketch
stream the reference draws in gaussian_matrix (dense_kernels.hpp:19-28),
std::mt19937_64 + libstdc++ std::normal_distribution<double>, produced by
compiling that exact generator code with g++ (the reference's compiler; the
reference itself cannot be built here, Eigen is absent).

Also records raw mt19937_64 outputs, including the C++ standard's required
10000th output of a default-seeded engine ([rand.predef]: 9981545732273789042),
which pins the engine independently of this machine.

Run: python tests/golden/make_golden.py
"""
import json
import os
import subprocess
import tempfile

SRC = r'''
#include <cstdio>
#include <cstdint>
#include <random>
int main(int argc, char** argv) {
    uint64_t seed = std::strtoull(argv[1], nullptr, 10);
    long n = std::atol(argv[2]);
    {
        std::mt19937_64 rng(seed);
        std::normal_distribution<double> normal(0.0, 1.0);
        for (long i = 0; i < n; ++i) std::printf("%a\n", normal(rng));
    }
    {
        std::mt19937_64 rng(seed);
        for (long i = 0; i < 64; ++i) std::printf("%llu\n", (unsigned long long)rng());
    }
    return 0;
}
'''


def mix_seed(seed, tag):
    M = (1 << 64) - 1
    z = (seed + 0x9E3779B97F4A7C15 * (tag + 1)) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def main():
    d = tempfile.mkdtemp()
    src = os.path.join(d, "g.cpp")
    exe = os.path.join(d, "g")
    open(src, "w").write(SRC)
    subprocess.check_call(["g++", "-std=c++20", "-O3", "-ffp-contract=off", src, "-o", exe])
    cases = []
    for (rows, cols, seed) in [(17, 9, 123), (300, 4, mix_seed(0, 0xA11CE)), (64, 8, 5489),
                               (1000, 1, mix_seed(7, 0xA11CE))]:
        n = rows * cols
        out = subprocess.check_output([exe, str(seed), str(n)], text=True).split()
        cases.append(dict(rows=rows, cols=cols, seed=seed, values_hex=out[:n],
                          raw_u64=[int(x) for x in out[n:n + 64]]))
    golden = dict(
        generator="std::mt19937_64 + std::normal_distribution<double>(0,1), libstdc++ (g++ 13)",
        reference="proj/include/frpca/dense_kernels.hpp:16-28",
        mt19937_64_default_10000th=9981545732273789042,
        cases=cases)
    here = os.path.dirname(os.path.abspath(__file__))
    json.dump(golden, open(os.path.join(here, "omega_stream.json"), "w"), indent=0)


if __name__ == "__main__":
    main()
