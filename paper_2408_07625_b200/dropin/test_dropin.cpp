// Drop-in acceptance program: the reference's own HamiltonianIndex,
// BasisVector, SequentialRng and synthetic generators (compiled from
// /root/reference/proj/src) linked against libqvmc_dropin.so in place of
// coupling.cpp / energy.cpp. Mirrors the hot-path cases of
// proj/tests/test_coupling.cpp, test_energy_sr.cpp and acceptance_main.cpp
// criteria 1, 3 and 4; pairs are cross-checked against a brute-force scan
// with the reference's own HamiltonianIndex::find_xy / matrix_element.
// Exit code 0 = all checks passed.
#include <cmath>
#include <complex>
#include <cstdio>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "qvmc/coupling.hpp"
#include "qvmc/energy.hpp"
#include "qvmc/hamiltonian.hpp"
#include "qvmc/rng.hpp"
#include "qvmc/synthetic.hpp"

using namespace qvmc;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(cond)) {                                                       \
      ++g_fail;                                                          \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                    \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static HamiltonianIndex parse(const std::string& text) {
  std::istringstream in(text);
  return HamiltonianIndex::parse(in);
}

static const char* kToy = "qubits: 4\n0.9 IIII\n0.1 IZZI\n-0.2 XIXI\n-0.2 IXIX\n0.3 IYYI\n";

static SampleBatch toy_batch() {
  SampleBatch b;
  b.vectors = {BasisVector::parse("1100"), BasisVector::parse("1001"), BasisVector::parse("0110")};
  b.log_probs.resize(3);
  b.log_amps.resize(3);
  b.phases.resize(3);
  const double p[3] = {4.0 / 6.0, 1.0 / 6.0, 1.0 / 6.0};
  for (int i = 0; i < 3; ++i) b.log_probs[i] = std::log(p[i]);
  b.log_amps[0] = std::log(2.0);
  b.log_amps[1] = b.log_amps[2] = 0.0;
  b.phases[0] = b.phases[1] = 0.0;
  b.phases[2] = 3.14159265358979323846;
  b.norm = 1.0;
  b.log_norm = 0.0;
  return b;
}

static bool same(const CoupledPairs& a, const CoupledPairs& b) {
  if (a.entries.size() != b.entries.size()) return false;
  for (std::size_t i = 0; i < a.entries.size(); ++i)
    if (a.entries[i].x != b.entries[i].x || a.entries[i].x_prime != b.entries[i].x_prime ||
        a.entries[i].xy != b.entries[i].xy)
      return false;
  return true;
}

// brute force with the reference's own find_xy, canonical order by construction
static CoupledPairs brute(std::span<const BasisVector> batch, const HamiltonianIndex& h) {
  CoupledPairs out;
  for (std::size_t i = 0; i < batch.size(); ++i)
    for (std::size_t j = 0; j < batch.size(); ++j)
      if (auto g = h.find_xy(batch[i] ^ batch[j]))
        out.entries.push_back({static_cast<std::uint32_t>(i), static_cast<std::uint32_t>(j), *g});
  return out;
}

static void toy_cases() {
  const HamiltonianIndex h = parse(kToy);
  const SampleBatch b = toy_batch();
  const std::uint32_t want[7][3] = {{0, 0, 0}, {0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 1, 0}, {2, 0, 1}, {2, 2, 0}};
  for (auto backend : {loop_over_terms, loop_over_batch, loop_over_trie}) {
    const CoupledPairs p = backend(b.vectors, h, 1);
    CHECK(p.entries.size() == 7);
    for (std::size_t i = 0; i < 7 && i < p.entries.size(); ++i)
      CHECK(p.entries[i].x == want[i][0] && p.entries[i].x_prime == want[i][1] && p.entries[i].xy == want[i][2]);
  }
  const CoupledPairs p = loop_over_batch(b.vectors, h);
  const Eigen::VectorXcd loc = local_energies(p, b, h);
  CHECK(std::abs(loc[0] - std::complex<double>(0.8, 0)) <= 1e-12);
  CHECK(std::abs(loc[1] - std::complex<double>(0.6, 0)) <= 1e-12);
  CHECK(std::abs(loc[2] - std::complex<double>(1.4, 0)) <= 1e-12);
  const EnergyReport r = variational_energy(b, loc);
  CHECK(std::abs(r.e_var - 5.2 / 6.0) <= 1e-13);
  CHECK(std::abs(r.ipr - 0.5) <= 1e-12);
  double ws = 0;
  for (int i = 0; i < 3; ++i) ws += r.weights[i];
  CHECK(std::abs(ws - 1.0) <= 1e-12);
  // auto selection (test_coupling.cpp:205-217)
  CouplingOptions opt;
  opt.backend = CouplingBackend::kAuto;
  opt.auto_batch_threshold = 4096;
  CHECK(find_coupled_pairs(std::vector<BasisVector>(b.vectors.begin(), b.vectors.begin() + 2), h, opt).backend ==
        CouplingBackend::kBatch);
  opt.auto_batch_threshold = 1;
  CHECK(find_coupled_pairs(std::vector<BasisVector>(b.vectors.begin(), b.vectors.begin() + 2), h, opt).backend ==
        CouplingBackend::kTrie);
  CHECK(parse_backend("trie") == CouplingBackend::kTrie);
  CHECK(throws<std::invalid_argument>([] { parse_backend("quantum"); }));
}

static void degenerate_and_errors() {
  const HamiltonianIndex id = parse("qubits: 4\n1.0 IIII\n");
  const std::vector<BasisVector> single = {BasisVector::parse("0101")};
  CHECK(loop_over_terms(single, id).entries.size() == 1);
  const HamiltonianIndex zz = parse("qubits: 4\n0.5 ZZII\n");
  const std::vector<BasisVector> two = {BasisVector::parse("1100"), BasisVector::parse("0011")};
  for (auto backend : {loop_over_terms, loop_over_batch, loop_over_trie}) {
    const auto d = backend(two, zz, 1);
    CHECK(d.entries.size() == 2 && d.entries[0].x == d.entries[0].x_prime && d.entries[1].x == d.entries[1].x_prime);
  }
  std::vector<std::pair<double, std::string>> cancel = {{0.4, "XYII"}, {-0.4, "XYII"}};
  const HamiltonianIndex empty = HamiltonianIndex::from_terms(4, cancel);
  CHECK(loop_over_batch(two, empty).entries.empty());
  CHECK(loop_over_trie(two, empty).entries.empty());
  // single-sample energy (test_energy_sr.cpp:69-88)
  const HamiltonianIndex h2 = parse("qubits: 2\n0.7 II\n0.2 ZI\n");
  SampleBatch b;
  b.vectors = {BasisVector::parse("10")};
  b.log_probs.resize(1);
  b.log_amps.resize(1);
  b.phases.resize(1);
  b.log_probs[0] = -0.3;
  b.log_amps[0] = -0.15;
  b.phases[0] = 0.4;
  b.log_norm = -0.3;
  b.norm = std::exp(-0.3);
  const auto loc = local_energies(loop_over_batch(b.vectors, h2), b, h2);
  const auto r = variational_energy(b, loc);
  CHECK(std::abs(r.e_var - loc[0].real()) <= 1e-14);
  CHECK(std::abs(r.e_var - 0.5) <= 1e-13);
  // zero amplitude -> logic_error; vanished norm -> runtime_error
  SampleBatch z = b;
  z.log_amps[0] = -INFINITY;
  CHECK(throws<std::logic_error>([&] { local_energies(loop_over_batch(z.vectors, h2), z, h2); }));
  SampleBatch nn = b;
  nn.log_probs[0] = -800.0;
  nn.log_norm = -800.0;
  nn.norm = std::exp(-800.0);
  Eigen::VectorXcd one(1);
  one[0] = {1.0, 0.0};
  CHECK(throws<std::runtime_error>([&] { variational_energy(nn, one); }));
}

static void random_family(std::uint32_t stream, int n_seeds, int max_n, int max_terms, int max_unq, int vec_seed_off) {
  int ok = 0;
  for (std::uint64_t seed = 1; seed <= static_cast<std::uint64_t>(n_seeds); ++seed) {
    SequentialRng rng(seed, stream);
    const int n = 4 + static_cast<int>(rng.uniform_int(max_n - 3));
    const int n_terms = 1 + static_cast<int>(rng.uniform_int(max_terms));
    const int cap = n < 12 ? (1 << n) : 4096;
    const int n_unq = 1 + static_cast<int>(rng.uniform_int(std::min(cap, max_unq)));
    const HamiltonianIndex h = random_hamiltonian(n, n_terms, seed, std::min(4, n));
    const auto batch = random_distinct_vectors(n, n_unq, seed + vec_seed_off);
    const CoupledPairs a = loop_over_terms(batch, h);
    const CoupledPairs b = loop_over_batch(batch, h);
    const CoupledPairs c = loop_over_trie(batch, h);
    const CoupledPairs bf = brute(batch, h);
    bool good = same(a, bf) && same(b, bf) && same(c, bf);
    good = good && a.ops == batch.size() * h.xy_set().size() && b.ops == batch.size() * batch.size();
    std::set<std::pair<std::uint32_t, std::uint32_t>> present;
    for (const auto& e : a.entries) present.insert({e.x, e.x_prime});
    for (const auto& e : a.entries) good = good && present.count({e.x_prime, e.x}) == 1;
    // E_loc against a direct sum with the reference's matrix_element
    SampleBatch sb;
    sb.vectors = batch;
    sb.log_amps.resize(n_unq);
    sb.phases.resize(n_unq);
    sb.log_probs.resize(n_unq);
    for (int i = 0; i < n_unq; ++i) {
      sb.log_amps[i] = 0.3 * std::sin(1.7 * i + seed);
      sb.phases[i] = 0.9 * i;
      sb.log_probs[i] = 2 * sb.log_amps[i];
    }
    const auto loc = local_energies(a, sb, h);
    for (int i = 0; i < n_unq && good; ++i) {
      std::complex<double> want{0, 0};
      double scale = 0;
      for (int j = 0; j < n_unq; ++j) {
        const auto e = h.matrix_element(batch[i], batch[j]);
        if (e == std::complex<double>{0, 0}) continue;
        const double a_ = std::exp(sb.log_amps[j] - sb.log_amps[i]);
        want += e * a_ * std::complex<double>(std::cos(sb.phases[j] - sb.phases[i]), std::sin(sb.phases[j] - sb.phases[i]));
        scale += std::abs(e) * a_;
      }
      good = good && std::abs(loc[i] - want) <= 1e-10 * std::max(scale, 1.0);
    }
    ok += good ? 1 : 0;
    if (!good) std::fprintf(stderr, "FAIL random family stream %u seed %llu\n", stream, (unsigned long long)seed);
  }
  CHECK(ok == n_seeds);
}

extern "C" void qvmc_dropin_release_all(void);

// Indices recreated at the same stack address with the same coefficients but
// different strings must not reuse a stale device copy (the cache checks the
// full content, not the address).
static void reused_address_cases() {
  const SampleBatch b = toy_batch();
  const char* texts[3] = {"qubits: 4\n0.9 IIII\n-0.2 XIXI\n0.3 IYYI\n",
                          "qubits: 4\n0.9 IIII\n-0.2 IXIX\n0.3 IYYI\n",
                          "qubits: 4\n0.9 IIII\n-0.2 XIXI\n0.3 IXXI\n"};
  for (int round = 0; round < 2; ++round) {
    for (const char* t : texts) {
      const HamiltonianIndex h = parse(t);
      const CoupledPairs p = loop_over_batch(b.vectors, h);
      const CoupledPairs want = brute(b.vectors, h);
      CHECK(p.entries.size() == want.entries.size());
      const Eigen::VectorXcd loc = local_energies(p, b, h);
      for (int i = 0; i < 3; ++i) {
        std::complex<double> e{0.0, 0.0};
        for (const auto& en : want.entries)
          if (en.x == static_cast<std::uint32_t>(i))
            e += h.matrix_element(b.vectors[i], b.vectors[en.x_prime]) *
                 std::exp(std::complex<double>(b.log_amps[en.x_prime] - b.log_amps[i],
                                               b.phases[en.x_prime] - b.phases[i]));
        CHECK(std::abs(loc[i] - e) <= 1e-12);
      }
    }
    qvmc_dropin_release_all();
  }
}

int main() {
  toy_cases();
  reused_address_cases();
  degenerate_and_errors();
  random_family(1234, 40, 70, 80, 256, 1);       // test_coupling.cpp:138-168
  random_family(0xAC3, 200, 40, 120, 512, 1000); // acceptance_main.cpp criterion 3
  std::printf("drop-in acceptance: %d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
