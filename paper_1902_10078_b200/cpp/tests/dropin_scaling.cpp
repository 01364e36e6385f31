// The banded leg of the reference's acceptance check_scaling
// (proj/tests/acceptance.cpp:302-325), restated: random SPD band, bw = 5,
// seed 4000 + n (gradcheck::random_spd_band), one reference-Tape step
// log|chol(Q)| + backward (tape.cpp:158-165 -> ops::cholesky, grad::vjp_*),
// median of 5 after one warm-up, at n = 5e4, 1e5, 2e5.  oracle/Makefile builds
// it twice from the same source: linked with the B200 drop-in
// (_ref/scaling_dropin) and with the reference kernels compiled verbatim
// (_ref/scaling_ref).  A second leg times the operators alone, without the
// Tape's host bookkeeping: ops::cholesky, ops::log_det_from_cholesky,
// grad::vjp_log_det_from_cholesky, grad::vjp_cholesky on host buffers.
// Prints one JSON line.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

#include "bandgm/grad.hpp"
#include "bandgm/gradcheck.hpp"
#include "bandgm/kernels.hpp"
#include "bandgm/tape.hpp"

using namespace bandgm;

template <class F>
static double median_ms(F&& f, int reps) {
  f();  // warm-up (device pools, first-touch)
  std::vector<double> t;
  for (int r = 0; r < reps; ++r) {
    const auto a = std::chrono::steady_clock::now();
    f();
    t.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count());
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

int main(int argc, char** argv) {
  const long bw = 5;
  std::vector<long> ns = {50000, 100000, 200000};
  if (argc > 1) ns = {std::atol(argv[1])};
  std::printf("{\"bw\": %ld, \"ops_ms\": {", bw);
  for (size_t q = 0; q < ns.size(); ++q) {
    const long n = ns[q];
    std::mt19937_64 rng(4000 + n);
    const SymmetricBandedMatrix qm = gradcheck::random_spd_band(rng, n, bw);
    const double ms = median_ms(
        [&] {
          const BandedMatrix l = ops::cholesky(qm);
          volatile double v = ops::log_det_from_cholesky(l);
          (void)v;
          const BandedMatrix lb = grad::vjp_log_det_from_cholesky(l, 1.0);
          const SymmetricBandedMatrix qb = grad::vjp_cholesky(l, lb);
          volatile double z = qb(0, 0);
          (void)z;
        },
        5);
    std::printf("%s\"%ld\": %.4f", q ? ", " : "", n, ms);
  }
  std::printf("}, \"ms\": {");
  for (size_t q = 0; q < ns.size(); ++q) {
    const long n = ns[q];
    std::mt19937_64 rng(4000 + n);
    const SymmetricBandedMatrix qm = gradcheck::random_spd_band(rng, n, bw);
    const double ms = median_ms(
        [&] {
          tape::Tape t;
          const auto node = t.log_det_from_cholesky(t.cholesky(t.leaf("q", qm)));
          volatile double v = t.scalar(node);
          (void)v;
          t.backward(node);
        },
        5);
    std::printf("%s\"%ld\": %.4f", q ? ", " : "", n, ms);
  }
  std::printf("}}\n");
  return 0;
}
