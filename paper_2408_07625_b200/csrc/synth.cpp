// libqvmc_synth: seeded synthetic inputs for tests and bench.py (SURVEY.md
// §8d). Not part of the local-energy path: kept out of libqvmc_cuda.so so
// that the reference arm of bench.py (the CPU reference timed alone) never
// loads the product library. Declared in include/qvmc_synth.h.
#include <algorithm>
#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

#include "qvmc_synth.h"

namespace {

constexpr int kMaxWords = 4;

uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed * 0x2545F4914F6CDD1Dull + 0x1234567ull) {}
  uint64_t bits() { return splitmix64(s); }
  uint64_t below(uint64_t n) { return bits() % n; }
  double uniform() { return static_cast<double>(bits() >> 11) * 0x1.0p-53; }
};

using WordsN = std::array<uint64_t, kMaxWords>;
struct WordsNHash {
  size_t operator()(const WordsN& k) const noexcept {
    uint64_t h = 0x9e3779b97f4a7c15ull;
    for (int i = 0; i < 3 * kMaxWords; ++i) {
      const uint64_t w = i < kMaxWords ? k[i] : 0;
      h ^= w + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
      h *= 0xff51afd7ed558ccdull;
      h ^= h >> 33;
    }
    return static_cast<size_t>(h);
  }
};

thread_local std::string g_error;


int64_t synth_jw_hamiltonian(int n, int64_t n_target, uint64_t seed, double* coeff, uint64_t* xw, uint64_t* yw,
                             uint64_t* zw) {
  if (n < 4 || n > 64 * kMaxWords) throw std::invalid_argument("synth: qubit count out of range");
  const int W = (n + 63) / 64;
  Rng rng(seed);
  static const double kMag[6] = {1.0, 0.5, 0.1, 0.05, 0.01, 0.02};
  auto draw = [&] { return (rng.bits() & 1 ? -1.0 : 1.0) * kMag[rng.below(6)]; };
  int64_t count = 0;
  std::vector<uint64_t> X(W), Y(W), Z(W);
  auto clear = [&] {
    std::fill(X.begin(), X.end(), 0);
    std::fill(Y.begin(), Y.end(), 0);
    std::fill(Z.begin(), Z.end(), 0);
  };
  auto setb = [](std::vector<uint64_t>& v, int i) { v[i / 64] |= uint64_t{1} << (i % 64); };
  auto flipb = [](std::vector<uint64_t>& v, int i) { v[i / 64] ^= uint64_t{1} << (i % 64); };
  auto emit = [&](double c) {
    if (count >= n_target) return false;
    coeff[count] = c;
    for (int w = 0; w < W; ++w) {
      xw[count * W + w] = X[w];
      yw[count * W + w] = Y[w];
      zw[count * W + w] = Z[w];
    }
    ++count;
    return true;
  };
  // diagonal: identity, Z_p, Z_p Z_q
  clear();
  if (!emit(draw())) return count;
  for (int p = 0; p < n; ++p) {
    clear();
    setb(Z, p);
    if (!emit(draw())) return count;
  }
  for (int p = 0; p < n; ++p)
    for (int q = p + 1; q < n; ++q) {
      clear();
      setb(Z, p);
      setb(Z, q);
      if (!emit(draw())) return count;
    }
  // same-spin singles: X_p Z.. X_q and Y_p Z.. Y_q, each also dressed by Z_k
  for (int p = 0; p < n; ++p)
    for (int q = p + 2; q < n; q += 2) {
      for (int letter = 0; letter < 2; ++letter) {
        for (int k = -1; k < n; ++k) {
          if (k == p || k == q) continue;
          clear();
          auto& L = letter == 0 ? X : Y;
          setb(L, p);
          setb(L, q);
          for (int r = p + 1; r < q; ++r) setb(Z, r);
          if (k >= 0) flipb(Z, k);
          if (!emit(draw())) return count;
        }
      }
    }
  // spin-conserving doubles on two even and two odd sites
  const int n_even = (n + 1) / 2, n_odd = n / 2;
  const uint64_t possible = static_cast<uint64_t>(n_even) * (n_even - 1) / 2 * (static_cast<uint64_t>(n_odd) * (n_odd - 1) / 2);
  std::unordered_set<uint32_t> used;
  static const char* kPat[4] = {"XXYY", "YYXX", "XYYX", "YXXY"};
  while (count + 4 <= n_target && used.size() < possible) {
    int e0 = 2 * static_cast<int>(rng.below(n_even)), e1 = 2 * static_cast<int>(rng.below(n_even));
    int o0 = 2 * static_cast<int>(rng.below(n_odd)) + 1, o1 = 2 * static_cast<int>(rng.below(n_odd)) + 1;
    if (e0 == e1 || o0 == o1) continue;
    int s[4] = {e0, e1, o0, o1};
    std::sort(s, s + 4);
    const uint32_t key = static_cast<uint32_t>(s[0]) | static_cast<uint32_t>(s[1]) << 8 |
                         static_cast<uint32_t>(s[2]) << 16 | static_cast<uint32_t>(s[3]) << 24;
    if (!used.insert(key).second) continue;
    for (int pt = 0; pt < 4; ++pt) {
      clear();
      for (int j = 0; j < 4; ++j) setb(kPat[pt][j] == 'X' ? X : Y, s[j]);
      for (int r = s[0] + 1; r < s[1]; ++r) setb(Z, r);
      for (int r = s[2] + 1; r < s[3]; ++r) setb(Z, r);
      emit(draw());
    }
  }
  return count;
}

void synth_near_hf_samples(int n, int n_e, int64_t n_unq, uint64_t seed, uint64_t* keys) {
  if (n < 2 || n > 64 * kMaxWords) throw std::invalid_argument("synth: qubit count out of range");
  if (n_e < 1 || n_e >= n) throw std::invalid_argument("synth: electron count out of range");
  const int W = (n + 63) / 64;
  Rng rng(seed);
  std::unordered_set<WordsN, WordsNHash> seen;
  seen.reserve(static_cast<size_t>(n_unq) * 2);
  WordsN hf{};
  for (int i = 0; i < n_e; ++i) hf[i / 64] |= uint64_t{1} << (i % 64);
  int64_t out = 0;
  auto push = [&](const WordsN& v) {
    if (!seen.insert(v).second) return;
    for (int w = 0; w < W; ++w) keys[out * W + w] = v[w];
    ++out;
  };
  push(hf);
  // sites of spin s are s, s+2, ...; moves keep the per-spin occupation
  const int n_sp[2] = {(n + 1) / 2, n / 2};
  int n_occ[2] = {(n_e + 1) / 2, n_e / 2};
  bool movable[2];
  for (int s = 0; s < 2; ++s) movable[s] = n_occ[s] > 0 && n_occ[s] < n_sp[s];
  if (!movable[0] && !movable[1]) throw std::invalid_argument("synth: no same-spin move exists");
  auto bit = [](const WordsN& v, int i) { return (v[i / 64] >> (i % 64)) & 1; };
  const int64_t max_draws = 1000 * n_unq + 100000;
  for (int64_t draw = 0; out < n_unq; ++draw) {
    if (draw > max_draws) throw std::invalid_argument("synth: sample space too small for the requested count");
    WordsN v = hf;
    int k = 1;
    while (rng.uniform() > 0.6) ++k;  // k = 1 + Geometric(0.6)
    for (int m = 0; m < k; ++m) {
      int spin = static_cast<int>(rng.bits() & 1);
      if (!movable[spin]) spin ^= 1;
      int o, e;
      do o = 2 * static_cast<int>(rng.below(n_sp[spin])) + spin; while (!bit(v, o));
      do e = 2 * static_cast<int>(rng.below(n_sp[spin])) + spin; while (bit(v, e));
      v[o / 64] ^= uint64_t{1} << (o % 64);
      v[e / 64] ^= uint64_t{1} << (e % 64);
    }
    push(v);
  }
}

}  // namespace

extern "C" {

const char* qvmc_synth_last_error(void) { return g_error.c_str(); }

int qvmc_synth_jw_hamiltonian(int n_qubits, int64_t n_terms_target, uint64_t seed, double* coeff, uint64_t* x_words,
                              uint64_t* y_words, uint64_t* z_words, int64_t* n_out) {
  try {
    if (!coeff || !x_words || !y_words || !z_words || !n_out || n_terms_target < 0)
      throw std::invalid_argument("null or negative argument");
    *n_out = synth_jw_hamiltonian(n_qubits, n_terms_target, seed, coeff, x_words, y_words, z_words);
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 1;
  }
}

int qvmc_synth_near_hf_samples(int n_qubits, int n_electrons, int64_t n_unq, uint64_t seed, uint64_t* keys) {
  try {
    if (!keys || n_unq < 0) throw std::invalid_argument("null or negative argument");
    synth_near_hf_samples(n_qubits, n_electrons, n_unq, seed, keys);
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 1;
  }
}

}  // extern "C"
