// Drop-in proof: the reference's own tape.cpp and gradcheck.cpp (compiled
// verbatim from /root/reference/proj/src by oracle/Makefile's `dropin`
// target) linked against the B200 drop-in bandgm::ops / bandgm::grad instead
// of the reference kernels.  Runs the reference's gradient suites
// (test_grad.cpp:32-40 seed 1234 x 10, acceptance.cpp:142-147 seed 2024 x 50)
// and a few known answers; exit status = number of failures.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "bandgm/gradcheck.hpp"
#include "bandgm/grad.hpp"
#include "bandgm/kernels.hpp"
#include "bandgm/tape.hpp"

using namespace bandgm;

static int failures = 0;
static void expect(bool ok, const std::string& what) {
  std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

int main() {
  for (auto [seed, inst] : {std::pair<unsigned long long, int>{1234, 10}, {2024, 50}}) {
    const auto reps = gradcheck::run_suite(seed, inst);
    for (const auto& r : reps) {
      char buf[160];
      std::snprintf(buf, sizeof buf, "suite(%llu,%d) %-28s max rel err %.3e", seed, inst,
                    r.op.c_str(), r.max_rel_err);
      expect(r.pass && r.max_rel_err < 1e-5, buf);
    }
  }
  {  // SPEC.md: [[4,2],[2,5]] -> [[2,0],[1,2]]
    SymmetricBandedMatrix q(2, 1);
    q.set(0, 0, 4.0);
    q.set(1, 1, 5.0);
    q.set(1, 0, 2.0);
    const BandedMatrix l = ops::cholesky(q);
    expect(l(0, 0) == 2.0 && l(1, 0) == 1.0 && l(1, 1) == 2.0, "cholesky [[4,2],[2,5]]");
  }
  {  // test_kernels.cpp:48-69: first bad pivot row
    SymmetricBandedMatrix q(4, 0);
    for (int i = 0; i < 4; ++i) q.set(i, i, 1.0);
    q.set(2, 2, -1.0);
    long row = -1;
    try {
      ops::cholesky(q);
    } catch (const NotPositiveDefinite& e) {
      row = e.row;
    }
    expect(row == 2, "NotPositiveDefinite carries row 2");
  }
  {  // test_tape.cpp:111-134: d log|chol(Q)| / dQ = half the inverse subset
    std::mt19937_64 rng(75);
    const auto q = gradcheck::random_spd_band(rng, 20, 3);
    tape::Tape t;
    const auto qn = t.leaf("q", q);
    const auto c = t.log_det_from_cholesky(t.cholesky(qn));
    auto grads = t.backward(c);
    const auto& got = std::get<SymmetricBandedMatrix>(grads.at("q"));
    const SymmetricBandedMatrix s = ops::sparse_inverse_subset(ops::cholesky(q));
    double worst = 0.0;
    for (long j = 0; j < 20; ++j)
      for (long i = j; i <= std::min(19L, j + 3); ++i) {
        const double want = (i == j ? 0.5 : 1.0) * s(i, j);
        worst = std::max(worst, std::abs(got(i, j) - want) / std::max(std::abs(want), 1e-12));
      }
    char buf[120];
    std::snprintf(buf, sizeof buf, "tape log-det gradient = half subset inverse (rel err %.2e)", worst);
    expect(worst < 1e-10, buf);
  }
  std::printf("%d failure(s)\n", failures);
  return failures;
}
