// Link-time drop-in for the reference's hot-path translation units.
//
// Defines every symbol that proj/src/coupling.cpp and proj/src/energy.cpp
// define, with the declarations of proj/include/qvmc/coupling.hpp and
// proj/include/qvmc/energy.hpp unchanged, so a reference build links this
// library instead of those two files and runs find_coupled_pairs /
// loop_over_* / local_energies / variational_energy on the B200 through the
// C ABI of libqvmc_cuda (include/qvmc_cuda.h). See INTEGRATION.md.
//
//   replaced symbol                      reference definition
//   parse_backend / backend_name         coupling.cpp:17-32
//   loop_over_terms / _batch / _trie     coupling.cpp:62-151
//   find_coupled_pairs                   coupling.cpp:153-169
//   local_energies                       energy.cpp:13-48
//   variational_energy                   energy.cpp:50-78
//   GradientAccumulator, energy_gradient energy.cpp:80-107 (not on the hot path:
//                                        host code, kept so the TU is complete)
//
// Only the public Eigen API is used, so this file builds against real Eigen
// or the repo's shim. `threads` arguments are accepted and ignored (the
// device decides its own parallelism); results are identical for any value,
// as the reference guarantees (parallel.hpp:15-20).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "qvmc/coupling.hpp"
#include "qvmc/energy.hpp"
#include "qvmc/hamiltonian.hpp"
#include "qvmc/sampler.hpp"
#include "qvmc_cuda.h"

namespace qvmc {

namespace {

static_assert(std::is_standard_layout_v<BasisVector>, "word extraction relies on BasisVector's standard layout");

void raise(int status, const char* where) {
  if (status == QVMC_OK) return;
  const std::string msg = std::string(where) + ": " + qvmc_cuda_last_error();
  switch (status) {
    case QVMC_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case QVMC_ERR_LOGIC: throw std::logic_error(qvmc_cuda_last_error());
    default: throw std::runtime_error(msg);
  }
}

int device_ordinal() {
  const char* s = std::getenv("QVMC_DEVICE");
  return s ? std::atoi(s) : 0;
}

// The words of a BasisVector are its leading std::array<uint64_t, 4> member.
inline void words_of(const BasisVector& v, std::uint64_t* out, int n_words) {
  std::uint64_t w[BasisVector::kMaxWords];
  std::memcpy(w, &v, sizeof(w));
  for (int i = 0; i < n_words; ++i) out[i] = w[i];
}

std::vector<std::uint64_t> pack(std::span<const BasisVector> batch, int n_words) {
  std::vector<std::uint64_t> keys(batch.size() * static_cast<std::size_t>(n_words));
  for (std::size_t i = 0; i < batch.size(); ++i) words_of(batch[i], keys.data() + i * n_words, n_words);
  return keys;
}

// Device copies of HamiltonianIndex objects, keyed by identity and checked
// by a fingerprint of the full content the device uses (the index is
// immutable, hamiltonian.hpp:41-45, but a new index can reuse the address of
// a destroyed one). At most kCacheCap copies stay resident (least recently
// used evicted first); qvmc_dropin_release_all() frees them explicitly.
struct Cached {
  std::uint64_t fingerprint = 0;
  qvmc_ham_t handle = nullptr;
  std::uint64_t last_use = 0;
};

std::mutex g_mu;
std::uint64_t g_clock = 0;
std::unordered_map<const HamiltonianIndex*, Cached>& cache() {
  static auto* m = new std::unordered_map<const HamiltonianIndex*, Cached>();
  return *m;
}

std::size_t cache_cap() {
  const char* s = std::getenv("QVMC_DROPIN_CACHE");
  const long v = s ? std::atol(s) : 4;
  return static_cast<std::size_t>(v < 1 ? 1 : v);
}

std::uint64_t fingerprint(const HamiltonianIndex& h) {
  std::uint64_t f = 0xcbf29ce484222325ull ^ static_cast<std::uint64_t>(h.n_qubits());
  auto mix = [&f](std::uint64_t v) {
    f ^= v;
    f *= 0x100000001b3ull;
    f ^= f >> 29;
  };
  const int W = (h.n_qubits() + 63) / 64;
  std::uint64_t w[BasisVector::kMaxWords];
  mix(h.n_terms());
  mix(h.xy_set().size());
  const auto d = h.diagonal_xy_index();
  mix(d ? static_cast<std::uint64_t>(*d) : ~0ull);
  for (std::size_t g = 0; g < h.xy_set().size(); ++g) {  // flip masks and the grouping
    std::memcpy(w, &h.xy_set()[g], sizeof(w));
    for (int i = 0; i < W; ++i) mix(w[i]);
    mix(static_cast<std::uint64_t>(h.group(g).size()));
  }
  for (const auto& t : h.terms()) {  // every term the device evaluates: coeff, yz mask, y weight
    std::uint64_t c;
    std::memcpy(&c, &t.coeff, 8);
    mix(c);
    std::memcpy(w, &t.yz_mask, sizeof(w));
    for (int i = 0; i < W; ++i) mix(w[i]);
    mix(static_cast<std::uint64_t>(t.y_weight));
  }
  return f;
}

int n_words_of(const HamiltonianIndex& h) { return (h.n_qubits() + 63) / 64; }

qvmc_ham_t device_index(const HamiltonianIndex& h) {
  const std::uint64_t fp = fingerprint(h);
  std::lock_guard<std::mutex> lock(g_mu);
  auto& m = cache();
  {
    auto it = m.find(&h);
    if (it != m.end() && it->second.handle && it->second.fingerprint == fp) {
      it->second.last_use = ++g_clock;
      return it->second.handle;
    }
  }
  // evict: a stale copy at this address, then least recently used copies beyond the cap
  if (auto it = m.find(&h); it != m.end()) {
    if (it->second.handle) qvmc_cuda_ham_destroy(it->second.handle);
    m.erase(it);
  }
  while (m.size() >= cache_cap()) {
    auto lru = m.begin();
    for (auto it = m.begin(); it != m.end(); ++it)
      if (it->second.last_use < lru->second.last_use) lru = it;
    if (lru->second.handle) qvmc_cuda_ham_destroy(lru->second.handle);
    m.erase(lru);
  }
  auto& c = m[&h];
  const int W = n_words_of(h);
  const auto& xy = h.xy_set();
  const auto& terms = h.terms();
  std::vector<std::uint64_t> xy_words(xy.size() * W), offsets(xy.size() + 1), yz(terms.size() * W);
  std::vector<double> coeff(terms.size());
  std::vector<std::uint8_t> yw(terms.size());
  for (std::size_t g = 0; g < xy.size(); ++g) {
    words_of(xy[g], xy_words.data() + g * W, W);
    offsets[g] = static_cast<std::uint64_t>(h.group(g).data() - terms.data());
  }
  offsets[xy.size()] = terms.size();
  for (std::size_t t = 0; t < terms.size(); ++t) {
    coeff[t] = terms[t].coeff;
    words_of(terms[t].yz_mask, yz.data() + t * W, W);
    yw[t] = static_cast<std::uint8_t>(terms[t].y_weight);
  }
  const auto d = h.diagonal_xy_index();
  qvmc_ham_t handle = nullptr;
  raise(qvmc_cuda_ham_create(h.n_qubits(), W, static_cast<std::uint32_t>(xy.size()), xy_words.data(),
                             offsets.data(), terms.size(), coeff.data(), yz.data(), yw.data(),
                             d ? static_cast<std::int64_t>(*d) : -1, device_ordinal(), &handle),
        "HamiltonianIndex upload");
  c.handle = handle;
  c.fingerprint = fp;
  c.last_use = ++g_clock;
  return handle;
}

// A one-qubit identity index: the variational-energy reduction needs only a
// handle's stream and workspace.
qvmc_ham_t moments_handle() {
  static qvmc_ham_t h = [] {
    const std::uint64_t xy = 0, off[2] = {0, 1}, yz = 0;
    const double c = 1.0;
    const std::uint8_t yw = 0;
    qvmc_ham_t out = nullptr;
    raise(qvmc_cuda_ham_create(1, 1, 1, &xy, off, 1, &c, &yz, &yw, 0, device_ordinal(), &out), "moments handle");
    return out;
  }();
  return h;
}

CoupledPairs device_pairs(std::span<const BasisVector> batch, const HamiltonianIndex& index, int backend,
                          int threshold) {
  for (const auto& v : batch)
    if (v.n_bits() != index.n_qubits()) throw std::invalid_argument("BasisVector: length mismatch");
  const int W = n_words_of(index);
  const auto keys = pack(batch, W);
  std::uint64_t n_pairs = 0, ops = 0;
  int used = backend;
  qvmc_ham_t h = device_index(index);
  raise(qvmc_cuda_pairs(h, static_cast<std::int64_t>(batch.size()), keys.data(), QVMC_MEM_HOST, backend, threshold,
                        &n_pairs, &ops, &used),
        "find_coupled_pairs");
  CoupledPairs out;
  out.entries.resize(n_pairs);
  static_assert(sizeof(CoupledPairs::Entry) == 12, "Entry is three uint32");
  if (n_pairs)
    raise(qvmc_cuda_pairs_fetch(h, reinterpret_cast<std::uint32_t*>(out.entries.data()), QVMC_MEM_HOST),
          "find_coupled_pairs");
  out.ops = ops;
  out.backend = static_cast<CouplingBackend>(used);
  return out;
}

}  // namespace

CouplingBackend parse_backend(const std::string& name) {
  if (name == "terms") return CouplingBackend::kTerms;
  if (name == "batch") return CouplingBackend::kBatch;
  if (name == "trie") return CouplingBackend::kTrie;
  if (name == "auto") return CouplingBackend::kAuto;
  throw std::invalid_argument("unknown coupling backend: " + name);
}

std::string backend_name(CouplingBackend b) {
  switch (b) {
    case CouplingBackend::kTerms: return "terms";
    case CouplingBackend::kBatch: return "batch";
    case CouplingBackend::kTrie: return "trie";
    case CouplingBackend::kAuto: return "auto";
  }
  return "?";
}

CoupledPairs loop_over_terms(std::span<const BasisVector> batch, const HamiltonianIndex& index, int) {
  return device_pairs(batch, index, QVMC_BACKEND_TERMS, 0);
}

CoupledPairs loop_over_batch(std::span<const BasisVector> batch, const HamiltonianIndex& index, int) {
  return device_pairs(batch, index, QVMC_BACKEND_BATCH, 0);
}

CoupledPairs loop_over_trie(std::span<const BasisVector> batch, const HamiltonianIndex& index, int) {
  return device_pairs(batch, index, QVMC_BACKEND_TRIE, 0);
}

CoupledPairs find_coupled_pairs(std::span<const BasisVector> batch, const HamiltonianIndex& index,
                                const CouplingOptions& options) {
  return device_pairs(batch, index, static_cast<int>(options.backend), options.auto_batch_threshold);
}

Eigen::VectorXcd local_energies(const CoupledPairs& pairs, const SampleBatch& batch, const HamiltonianIndex& index,
                                int) {
  const int n = batch.size();
  if (batch.log_amps.size() != n || batch.phases.size() != n)
    throw std::invalid_argument("local_energies: amplitudes not filled");
  const int W = n_words_of(index);
  const auto keys = pack(batch.vectors, W);
  std::vector<double> la(n), ph(n), out(2 * static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    la[i] = batch.log_amps[i];
    ph[i] = batch.phases[i];
  }
  raise(qvmc_cuda_local_energies(device_index(index), n, keys.data(), la.data(), ph.data(), pairs.entries.size(),
                                 reinterpret_cast<const std::uint32_t*>(pairs.entries.data()), out.data(),
                                 QVMC_MEM_HOST),
        "local_energies");
  Eigen::VectorXcd locals = Eigen::VectorXcd::Zero(n);
  for (int i = 0; i < n; ++i) locals[i] = std::complex<double>(out[2 * i], out[2 * i + 1]);
  return locals;
}

EnergyReport variational_energy(const SampleBatch& batch, const Eigen::VectorXcd& locals) {
  if (locals.size() != batch.size()) throw std::invalid_argument("variational_energy: locals/batch size mismatch");
  EnergyReport report;
  report.locals = locals;
  report.norm = batch.norm;
  report.log_norm = batch.log_norm;
  if (!(batch.norm > 0.0)) throw std::runtime_error("variational_energy: sampled norm is zero");
  const int n = batch.size();
  std::vector<double> lp(n), e(2 * static_cast<std::size_t>(n)), w(n), m(5);
  for (int i = 0; i < n; ++i) {
    lp[i] = batch.log_probs[i];
    e[2 * i] = locals[i].real();
    e[2 * i + 1] = locals[i].imag();
  }
  raise(qvmc_cuda_energy_moments(moments_handle(), n, lp.data(), batch.log_norm, e.data(), m.data(), w.data(),
                                 QVMC_MEM_HOST),
        "variational_energy");
  report.weights.resize(n);
  for (int i = 0; i < n; ++i) report.weights[i] = w[i];
  report.e_var = m[0];
  report.im_residual = m[1];
  report.ipr = m[2];
  if (std::abs(report.im_residual) > 1e-6 * std::max(1.0, std::abs(report.e_var)))
    throw std::runtime_error("variational_energy: imaginary residual " + std::to_string(report.im_residual));
  return report;
}

// ---- gradient stage (outside the local-energy path; host code)

GradientAccumulator::GradientAccumulator(Eigen::Index n_params, std::complex<double> e_mean)
    : grad_(Eigen::VectorXd::Zero(n_params)), e_mean_(e_mean) {}

void GradientAccumulator::add(double weight, std::complex<double> e_loc, const Eigen::VectorXcd& row) {
  const std::complex<double> c = weight * (e_loc - e_mean_);
  if (c == std::complex<double>{0.0, 0.0}) return;
  for (Eigen::Index k = 0; k < grad_.size(); ++k)
    grad_[k] += 2.0 * (c.real() * row[k].real() - c.imag() * row[k].imag());
}

Eigen::VectorXd GradientAccumulator::take() { return std::move(grad_); }

Eigen::VectorXd energy_gradient(const Eigen::VectorXd& weights, const Eigen::VectorXcd& locals,
                                const Eigen::MatrixXcd& jacobian) {
  if (weights.size() != locals.size() || jacobian.rows() != weights.size())
    throw std::invalid_argument("energy_gradient: misaligned inputs");
  std::complex<double> mean{0.0, 0.0};
  for (Eigen::Index i = 0; i < weights.size(); ++i) mean += weights[i] * locals[i];
  GradientAccumulator acc(jacobian.cols(), mean);
  Eigen::VectorXcd row(jacobian.cols());
  for (Eigen::Index i = 0; i < weights.size(); ++i) {
    for (Eigen::Index k = 0; k < jacobian.cols(); ++k) row[k] = jacobian(i, k);
    acc.add(weights[i], locals[i], row);
  }
  return acc.take();
}

}  // namespace qvmc

// Frees every cached device copy of a HamiltonianIndex (e.g. before the
// caller destroys its indices, or to return device memory). Safe to call at
// any time; later calls re-upload on demand.
extern "C" void qvmc_dropin_release_all(void) {
  std::lock_guard<std::mutex> lock(qvmc::g_mu);
  for (auto& [k, c] : qvmc::cache())
    if (c.handle) qvmc_cuda_ham_destroy(c.handle);
  qvmc::cache().clear();
}
