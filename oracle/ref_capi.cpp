// C entry points over the UNMODIFIED reference hot path (test/bench infrastructure).
//
// This file is compiled together with the reference's own sources from
// /root/reference/proj/src (basis_vector, rng, hamiltonian, prefix_tree,
// coupling, energy, synthetic) by oracle/Makefile into oracle/_ref/
// libqvmc_ref_hot.so. It is a checker and CPU baseline only: it is used by
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg, never by the product path.
//
// Every function catches C++ exceptions and returns a negative status; the
// exception class and message are available from qref_last_error().
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "qvmc/basis_vector.hpp"
#include "qvmc/coupling.hpp"
#include "qvmc/energy.hpp"
#include "qvmc/hamiltonian.hpp"
#include "qvmc/model.hpp"
#include "qvmc/parallel.hpp"
#include "qvmc/prefix_tree.hpp"
#include "qvmc/rng.hpp"
#include "qvmc/sampler.hpp"
#include "qvmc/synthetic.hpp"

using qvmc::BasisVector;
using qvmc::CoupledPairs;
using qvmc::HamiltonianIndex;

static_assert(std::is_standard_layout_v<BasisVector>, "BasisVector word access relies on standard layout");

namespace {

thread_local std::string g_error;

enum Status { kOk = 0, kInvalidArgument = -1, kLogicError = -2, kRuntimeError = -3, kOther = -4 };

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const std::invalid_argument& e) {
    g_error = std::string("invalid_argument: ") + e.what();
    return kInvalidArgument;
  } catch (const std::out_of_range& e) {
    g_error = std::string("invalid_argument: ") + e.what();
    return kInvalidArgument;
  } catch (const std::logic_error& e) {
    g_error = std::string("logic_error: ") + e.what();
    return kLogicError;
  } catch (const std::runtime_error& e) {
    g_error = std::string("runtime_error: ") + e.what();
    return kRuntimeError;
  } catch (const std::exception& e) {
    g_error = std::string("exception: ") + e.what();
    return kOther;
  }
}

// BasisVector keeps its words private; the class is standard-layout with the
// word array as first member, so the words are the leading 32 bytes.
void read_words(const BasisVector& v, std::uint64_t* out, int n_words) {
  std::uint64_t w[BasisVector::kMaxWords];
  std::memcpy(w, &v, sizeof(w));
  for (int i = 0; i < n_words; ++i) out[i] = w[i];
}

BasisVector make_vector(int n_qubits, const std::uint64_t* words, int n_words) {
  BasisVector v(n_qubits);
  std::uint64_t w[BasisVector::kMaxWords] = {0, 0, 0, 0};
  for (int i = 0; i < n_words; ++i) w[i] = words[i];
  // keep the canonical zero tail
  const int tail = n_qubits % 64;
  if (tail) w[n_qubits / 64] &= (std::uint64_t{1} << tail) - 1;
  std::memcpy(&v, w, sizeof(w));
  return v;
}

std::vector<BasisVector> make_batch(int n_qubits, int n_words, std::int64_t n, const std::uint64_t* keys) {
  std::vector<BasisVector> out;
  out.reserve(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) out.push_back(make_vector(n_qubits, keys + i * n_words, n_words));
  return out;
}

struct PairsBox {
  CoupledPairs pairs;
};

struct RngBox {
  qvmc::SequentialRng rng;
};

}  // namespace

extern "C" {

const char* qref_last_error(void) { return g_error.c_str(); }

// HamiltonianIndex::parse over a text buffer (hamiltonian.cpp:119-170).
int qref_index_parse(const char* text, void** out) {
  return guarded([&] {
    std::istringstream in(text);
    *out = new HamiltonianIndex(HamiltonianIndex::parse(in));
  });
}

// HamiltonianIndex::from_terms over n_terms strings of n_qubits characters
// packed back to back (hamiltonian.cpp:63-117).
int qref_index_from_strings(int n_qubits, std::int64_t n_terms, const double* coeff, const char* strings,
                            void** out) {
  return guarded([&] {
    std::vector<std::pair<double, std::string>> raw;
    raw.reserve(static_cast<std::size_t>(n_terms));
    for (std::int64_t t = 0; t < n_terms; ++t)
      raw.emplace_back(coeff[t], std::string(strings + t * n_qubits, static_cast<std::size_t>(n_qubits)));
    *out = new HamiltonianIndex(HamiltonianIndex::from_terms(n_qubits, raw));
  });
}

// synthetic.cpp:18-49
int qref_random_hamiltonian(int n_qubits, int n_terms, std::uint64_t seed, int max_weight, void** out) {
  return guarded([&] { *out = new HamiltonianIndex(qvmc::random_hamiltonian(n_qubits, n_terms, seed, max_weight)); });
}

void qref_index_free(void* h) { delete static_cast<HamiltonianIndex*>(h); }

int qref_index_info(void* hp, int* n_qubits, std::uint64_t* n_terms, std::uint32_t* n_xy, std::int64_t* diag) {
  return guarded([&] {
    const auto& h = *static_cast<HamiltonianIndex*>(hp);
    *n_qubits = h.n_qubits();
    *n_terms = h.n_terms();
    *n_xy = static_cast<std::uint32_t>(h.xy_set().size());
    const auto d = h.diagonal_xy_index();
    *diag = d ? static_cast<std::int64_t>(*d) : -1;
  });
}

// Grouped layout as held by HamiltonianIndex: xy_set in first-occurrence
// order, CSR group offsets, and per term (coeff, x, y, z, yz masks, y_weight).
int qref_index_export(void* hp, int n_words, std::uint64_t* xy_words, std::uint64_t* group_offsets, double* coeff,
                      std::uint64_t* x_words, std::uint64_t* y_words, std::uint64_t* z_words,
                      std::uint64_t* yz_words, std::uint8_t* y_weight) {
  return guarded([&] {
    const auto& h = *static_cast<HamiltonianIndex*>(hp);
    const auto& xy = h.xy_set();
    for (std::size_t g = 0; g < xy.size(); ++g) read_words(xy[g], xy_words + g * n_words, n_words);
    const auto* base = h.terms().data();
    for (std::size_t g = 0; g < xy.size(); ++g) group_offsets[g] = static_cast<std::uint64_t>(h.group(g).data() - base);
    group_offsets[xy.size()] = h.terms().size();
    const auto& terms = h.terms();
    for (std::size_t t = 0; t < terms.size(); ++t) {
      coeff[t] = terms[t].coeff;
      if (x_words) read_words(terms[t].x_mask, x_words + t * n_words, n_words);
      if (y_words) read_words(terms[t].y_mask, y_words + t * n_words, n_words);
      if (z_words) read_words(terms[t].z_mask, z_words + t * n_words, n_words);
      if (yz_words) read_words(terms[t].yz_mask, yz_words + t * n_words, n_words);
      if (y_weight) y_weight[t] = static_cast<std::uint8_t>(terms[t].y_weight);
    }
  });
}

// hamiltonian.cpp:178-184
int qref_matrix_element(void* hp, int n_words, const std::uint64_t* x, const std::uint64_t* xp, double* out2) {
  return guarded([&] {
    const auto& h = *static_cast<HamiltonianIndex*>(hp);
    const auto e = h.matrix_element(make_vector(h.n_qubits(), x, n_words), make_vector(h.n_qubits(), xp, n_words));
    out2[0] = e.real();
    out2[1] = e.imag();
  });
}

// hamiltonian.cpp:186-194
int qref_group_element(void* hp, int n_words, const std::uint64_t* xp, std::uint32_t g, double* out2) {
  return guarded([&] {
    const auto& h = *static_cast<HamiltonianIndex*>(hp);
    const auto e = h.group_element(make_vector(h.n_qubits(), xp, n_words), g);
    out2[0] = e.real();
    out2[1] = e.imag();
  });
}

// synthetic.cpp:51-70
int qref_random_distinct_vectors(int n_qubits, int count, std::uint64_t seed, int n_words, std::uint64_t* out) {
  return guarded([&] {
    const auto v = qvmc::random_distinct_vectors(n_qubits, count, seed);
    for (std::size_t i = 0; i < v.size(); ++i) read_words(v[i], out + i * n_words, n_words);
  });
}

// backend: 0 terms, 1 batch, 2 trie, 3 auto (coupling.hpp:17)
int qref_pairs(void* hp, std::int64_t n_unq, int n_words, const std::uint64_t* keys, int backend, int threshold,
               int threads, void** out) {
  return guarded([&] {
    const auto& h = *static_cast<HamiltonianIndex*>(hp);
    const auto batch = make_batch(h.n_qubits(), n_words, n_unq, keys);
    auto box = new PairsBox;
    try {
      switch (backend) {
        case 0: box->pairs = qvmc::loop_over_terms(batch, h, threads); break;
        case 1: box->pairs = qvmc::loop_over_batch(batch, h, threads); break;
        case 2: box->pairs = qvmc::loop_over_trie(batch, h, threads); break;
        default: {
          qvmc::CouplingOptions opt;
          opt.backend = qvmc::CouplingBackend::kAuto;
          opt.auto_batch_threshold = threshold;
          opt.threads = threads;
          box->pairs = qvmc::find_coupled_pairs(batch, h, opt);
        }
      }
    } catch (...) {
      delete box;
      throw;
    }
    *out = box;
  });
}

void qref_pairs_free(void* p) { delete static_cast<PairsBox*>(p); }

int qref_pairs_info(void* p, std::uint64_t* n_pairs, std::uint64_t* ops, int* backend) {
  return guarded([&] {
    const auto& box = *static_cast<PairsBox*>(p);
    *n_pairs = box.pairs.entries.size();
    *ops = box.pairs.ops;
    *backend = static_cast<int>(box.pairs.backend);
  });
}

int qref_pairs_copy(void* p, std::uint32_t* out3) {
  return guarded([&] {
    const auto& e = static_cast<PairsBox*>(p)->pairs.entries;
    for (std::size_t i = 0; i < e.size(); ++i) {
      out3[3 * i] = e[i].x;
      out3[3 * i + 1] = e[i].x_prime;
      out3[3 * i + 2] = e[i].xy;
    }
  });
}

// Build a CoupledPairs from caller triples (to feed local_energies).
int qref_pairs_from_triples(std::uint64_t n_pairs, const std::uint32_t* in3, void** out) {
  return guarded([&] {
    auto box = new PairsBox;
    box->pairs.entries.resize(static_cast<std::size_t>(n_pairs));
    for (std::uint64_t i = 0; i < n_pairs; ++i)
      box->pairs.entries[i] = {in3[3 * i], in3[3 * i + 1], in3[3 * i + 2]};
    *out = box;
  });
}

// energy.cpp:13-48; out_eloc is interleaved (re, im).
int qref_local_energies(void* hp, void* pp, std::int64_t n_unq, int n_words, const std::uint64_t* keys,
                        const double* log_amps, const double* phases, int threads, double* out_eloc) {
  return guarded([&] {
    const auto& h = *static_cast<HamiltonianIndex*>(hp);
    qvmc::SampleBatch batch;
    batch.vectors = make_batch(h.n_qubits(), n_words, n_unq, keys);
    batch.log_amps.resize(n_unq);
    batch.phases.resize(n_unq);
    batch.log_probs.resize(n_unq);
    for (std::int64_t i = 0; i < n_unq; ++i) {
      batch.log_amps[i] = log_amps[i];
      batch.phases[i] = phases[i];
      batch.log_probs[i] = 2.0 * log_amps[i];
    }
    const auto locals = qvmc::local_energies(static_cast<PairsBox*>(pp)->pairs, batch, h, threads);
    for (std::int64_t i = 0; i < n_unq; ++i) {
      out_eloc[2 * i] = locals[i].real();
      out_eloc[2 * i + 1] = locals[i].imag();
    }
  });
}

// energy.cpp:50-78; out5 = (e_var, im_residual, ipr, norm, log_norm); weights optional.
int qref_variational_energy(std::int64_t n, const double* log_probs, double norm, double log_norm,
                            const double* eloc, double* out5, double* weights) {
  return guarded([&] {
    qvmc::SampleBatch batch;
    batch.vectors.assign(static_cast<std::size_t>(n), BasisVector(1));
    batch.log_probs.resize(n);
    batch.log_amps.resize(n);
    batch.phases.resize(n);
    for (std::int64_t i = 0; i < n; ++i) batch.log_probs[i] = log_probs[i];
    batch.norm = norm;
    batch.log_norm = log_norm;
    Eigen::VectorXcd locals(n);
    for (std::int64_t i = 0; i < n; ++i) locals[i] = {eloc[2 * i], eloc[2 * i + 1]};
    const auto r = qvmc::variational_energy(batch, locals);
    out5[0] = r.e_var;
    out5[1] = r.im_residual;
    out5[2] = r.ipr;
    out5[3] = r.norm;
    out5[4] = r.log_norm;
    if (weights)
      for (std::int64_t i = 0; i < n; ++i) weights[i] = r.weights[i];
  });
}

// The reference CPU path end to end, as run_optimisation drives it
// (optimizer.cpp:87-93): find_coupled_pairs -> local_energies ->
// variational_energy. Only rows [0, n_rows) need not be the whole batch:
// the batch passed IS the sample set. times3 = seconds per stage.
int qref_run_path(void* hp, std::int64_t n_unq, int n_words, const std::uint64_t* keys, const double* log_amps,
                  const double* phases, const double* log_probs, double norm, double log_norm, int backend,
                  int threshold, int threads, double* out_eloc, double* out5, double* times3,
                  std::uint64_t* n_pairs) {
  return guarded([&] {
    using clock = std::chrono::steady_clock;
    const auto& h = *static_cast<HamiltonianIndex*>(hp);
    qvmc::SampleBatch batch;
    batch.vectors = make_batch(h.n_qubits(), n_words, n_unq, keys);
    batch.log_amps.resize(n_unq);
    batch.phases.resize(n_unq);
    batch.log_probs.resize(n_unq);
    for (std::int64_t i = 0; i < n_unq; ++i) {
      batch.log_amps[i] = log_amps[i];
      batch.phases[i] = phases[i];
      batch.log_probs[i] = log_probs[i];
    }
    batch.norm = norm;
    batch.log_norm = log_norm;
    qvmc::CouplingOptions opt;
    opt.backend = static_cast<qvmc::CouplingBackend>(backend);
    opt.auto_batch_threshold = threshold;
    opt.threads = threads;
    const auto t0 = clock::now();
    const auto pairs = qvmc::find_coupled_pairs(batch.vectors, h, opt);
    const auto t1 = clock::now();
    const auto locals = qvmc::local_energies(pairs, batch, h, threads);
    const auto t2 = clock::now();
    const auto r = qvmc::variational_energy(batch, locals);
    const auto t3 = clock::now();
    times3[0] = std::chrono::duration<double>(t1 - t0).count();
    times3[1] = std::chrono::duration<double>(t2 - t1).count();
    times3[2] = std::chrono::duration<double>(t3 - t2).count();
    *n_pairs = pairs.entries.size();
    if (out_eloc)
      for (std::int64_t i = 0; i < n_unq; ++i) {
        out_eloc[2 * i] = locals[i].real();
        out_eloc[2 * i + 1] = locals[i].imag();
      }
    out5[0] = r.e_var;
    out5[1] = r.im_residual;
    out5[2] = r.ipr;
    out5[3] = r.norm;
    out5[4] = r.log_norm;
  });
}

// ---- A bounded sample of the FULL workload for the CPU baseline: listed rows
// of the whole sample set, each against the whole sample set (the same
// pairs per row as the GPU arm's 1e6-row job). find_coupled_pairs has no
// row-subset entry, so the per-row body of loop_over_trie
// (coupling.cpp:116-149, reproduced verbatim below) runs over the
// reference's own PrefixTree builds of the full sample set and of xy_set
// (built once per session, timed separately, prorated by the caller); the
// rows' canonical pairs (PerSource::flatten, coupling.cpp:37-58) then go
// through the unmodified local_energies (energy.cpp:13-48: rows without
// pairs stay 0) and variational_energy (energy.cpp:50-78) over the whole
// batch.
struct RowSession {
  const HamiltonianIndex* h = nullptr;
  qvmc::SampleBatch batch;
  std::unique_ptr<qvmc::PrefixTree> u_tree, xy_tree;
};

void* qref_rows_session(void* hp, std::int64_t n_unq, int n_words, const std::uint64_t* keys,
                        const double* log_amps, const double* phases, const double* log_probs, double norm,
                        double log_norm, double* build_seconds) {
  RowSession* out = nullptr;
  const int st = guarded([&] {
    using clock = std::chrono::steady_clock;
    auto S = std::make_unique<RowSession>();
    S->h = static_cast<HamiltonianIndex*>(hp);
    auto& batch = S->batch;
    batch.vectors = make_batch(S->h->n_qubits(), n_words, n_unq, keys);
    batch.log_amps.resize(n_unq);
    batch.phases.resize(n_unq);
    batch.log_probs.resize(n_unq);
    for (std::int64_t i = 0; i < n_unq; ++i) {
      batch.log_amps[i] = log_amps[i];
      batch.phases[i] = phases[i];
      batch.log_probs[i] = log_probs[i];
    }
    batch.norm = norm;
    batch.log_norm = log_norm;
    const auto t0 = clock::now();
    S->u_tree = std::make_unique<qvmc::PrefixTree>(qvmc::PrefixTree::build(batch.vectors));
    S->xy_tree = std::make_unique<qvmc::PrefixTree>(qvmc::PrefixTree::build(S->h->xy_set()));
    *build_seconds = std::chrono::duration<double>(clock::now() - t0).count();
    out = S.release();
  });
  return st == kOk ? out : nullptr;
}

void qref_rows_session_free(void* s) { delete static_cast<RowSession*>(s); }

// times3 = (pair search of the listed rows, local_energies, variational_energy) seconds
int qref_rows_session_run(void* sp, std::int64_t n_rows, const std::int64_t* rows, int threads, double* times3,
                          std::uint64_t* n_pairs, double* out_eloc_rows) {
  return guarded([&] {
    using clock = std::chrono::steady_clock;
    auto& S = *static_cast<RowSession*>(sp);
    const auto& batch = S.batch;
    const auto& u_tree = *S.u_tree;
    const auto& xy_tree = *S.xy_tree;
    const int n = u_tree.n_bits();
    const auto t0 = clock::now();
    std::vector<std::vector<CoupledPairs::Entry>> acc(static_cast<std::size_t>(n_rows));
    qvmc::parallel_for(static_cast<int>(n_rows), threads, [&](int k) {
      const auto i = static_cast<std::size_t>(rows[k]);
      const BasisVector& x = batch.vectors[i];
      std::vector<std::pair<std::int32_t, std::int32_t>> frontier{{0, 0}}, next;
      for (int level = 0; level < n; ++level) {
        next.clear();
        const auto u_nodes = u_tree.level(level);
        const auto xy_nodes = xy_tree.level(level);
        const int xi = x.bit(level) ? 1 : 0;
        for (const auto& [un, xn] : frontier) {
          for (int b = 0; b < 2; ++b) {
            const std::int32_t u_child = u_nodes[static_cast<std::size_t>(un)].child[b];
            if (u_child == qvmc::PrefixTree::kNone) continue;
            const std::int32_t xy_child = xy_nodes[static_cast<std::size_t>(xn)].child[xi ^ b];
            if (xy_child == qvmc::PrefixTree::kNone) continue;
            next.emplace_back(u_child, xy_child);
          }
        }
        frontier.swap(next);
        if (frontier.empty()) break;
      }
      auto& row = acc[static_cast<std::size_t>(k)];
      for (const auto& [un, xn] : frontier)
        row.push_back({static_cast<std::uint32_t>(i), static_cast<std::uint32_t>(u_tree.leaf_payload(un)),
                       static_cast<std::uint32_t>(xy_tree.leaf_payload(xn))});
      std::sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.x_prime < b.x_prime; });
    });
    // canonical order: rows ascending (the caller lists them ascending), then x'
    CoupledPairs pairs;
    pairs.backend = qvmc::CouplingBackend::kTrie;
    std::size_t total = 0;
    for (const auto& r : acc) total += r.size();
    pairs.entries.reserve(total);
    for (const auto& r : acc) pairs.entries.insert(pairs.entries.end(), r.begin(), r.end());
    const auto t1 = clock::now();
    const auto locals = qvmc::local_energies(pairs, batch, *S.h, threads);
    const auto t2 = clock::now();
    const auto rep = qvmc::variational_energy(batch, locals);
    const auto t3 = clock::now();
    (void)rep;
    times3[0] = std::chrono::duration<double>(t1 - t0).count();
    times3[1] = std::chrono::duration<double>(t2 - t1).count();
    times3[2] = std::chrono::duration<double>(t3 - t2).count();
    *n_pairs = total;
    if (out_eloc_rows)
      for (std::int64_t k = 0; k < n_rows; ++k) {
        out_eloc_rows[2 * k] = locals[rows[k]].real();
        out_eloc_rows[2 * k + 1] = locals[rows[k]].imag();
      }
  });
}

// SequentialRng (rng.hpp:70-93), to regenerate the reference tests' seeded
// random-instance families.
void* qref_rng_new(std::uint64_t seed, std::uint32_t stream) { return new RngBox{qvmc::SequentialRng(seed, stream)}; }
void qref_rng_free(void* r) { delete static_cast<RngBox*>(r); }
std::uint64_t qref_rng_uniform_int(void* r, std::uint64_t n) { return static_cast<RngBox*>(r)->rng.uniform_int(n); }
std::uint64_t qref_rng_bits64(void* r) { return static_cast<RngBox*>(r)->rng.bits64(); }

// ---- AnqsModel (model.cpp) and fill_amplitudes (sampler.cpp:104-120): the
// amplitude evaluation that feeds the local-energy path.
int qref_model_create(int n_qubits, int bits_per_qudit, int n_electrons, int spin_constraint, int hidden,
                      void** out) {
  return guarded([&] {
    *out = new qvmc::AnqsModel(qvmc::QuditLayout::make(n_qubits, bits_per_qudit),
                               qvmc::SectorConstraint{n_electrons, spin_constraint != 0}, hidden);
  });
}
void qref_model_free(void* m) { delete static_cast<qvmc::AnqsModel*>(m); }
std::int64_t qref_model_n_params(void* m) { return static_cast<qvmc::AnqsModel*>(m)->n_params(); }
int qref_model_init_params(void* m, std::uint64_t seed) {
  return guarded([&] { static_cast<qvmc::AnqsModel*>(m)->init_params(seed); });
}
int qref_model_get_params(void* m, double* out) {
  return guarded([&] {
    const auto& p = static_cast<qvmc::AnqsModel*>(m)->params();
    for (Eigen::Index i = 0; i < p.size(); ++i) out[i] = p[i];
  });
}
int qref_model_set_params(void* m, std::int64_t n, const double* in) {
  return guarded([&] {
    Eigen::VectorXd p(n);
    for (std::int64_t i = 0; i < n; ++i) p[i] = in[i];
    static_cast<qvmc::AnqsModel*>(m)->set_params(p);
  });
}
// AnqsModel::log_psi (model.cpp:262-271) per vector, parallel_for over threads
int qref_model_log_psi(void* m, std::int64_t n, int n_words, const std::uint64_t* keys, int threads,
                       double* out_log_amp, double* out_phase) {
  return guarded([&] {
    const auto& model = *static_cast<qvmc::AnqsModel*>(m);
    const auto vs = make_batch(model.layout().n_qubits, n_words, n, keys);
    qvmc::parallel_for(static_cast<int>(n), threads, [&](int i) {
      const auto a = model.log_psi(vs[static_cast<std::size_t>(i)]);
      out_log_amp[i] = a.log_amp;
      out_phase[i] = a.phase;
    });
  });
}
// fill_amplitudes (sampler.cpp:104-120); out2 = (norm, log_norm)
int qref_fill_amplitudes(void* m, std::int64_t n, int n_words, const std::uint64_t* keys, const double* log_probs,
                         int threads, double* out_log_amp, double* out_phase, double* out2) {
  return guarded([&] {
    const auto& model = *static_cast<qvmc::AnqsModel*>(m);
    qvmc::SampleBatch batch;
    batch.vectors = make_batch(model.layout().n_qubits, n_words, n, keys);
    batch.log_probs.resize(n);
    for (std::int64_t i = 0; i < n; ++i) batch.log_probs[i] = log_probs[i];
    qvmc::fill_amplitudes(batch, model, threads);
    for (std::int64_t i = 0; i < n; ++i) {
      out_log_amp[i] = batch.log_amps[i];
      out_phase[i] = batch.phases[i];
    }
    out2[0] = batch.norm;
    out2[1] = batch.log_norm;
  });
}

// sample_without_replacement (sampler.cpp:37-102), unmodified: CounterRng(seed,
// stream), iteration; out_keys [K][n_words], out_log_probs [K]; *out_n = size
int qref_sample(void* m, int k_samples, std::uint64_t seed, std::uint32_t stream, std::uint32_t iteration,
                int threads, int n_words, std::uint64_t* out_keys, double* out_log_probs, std::int64_t* out_n) {
  return guarded([&] {
    const auto& model = *static_cast<qvmc::AnqsModel*>(m);
    const qvmc::CounterRng rng(seed, stream);
    const qvmc::SampleBatch b = qvmc::sample_without_replacement(model, k_samples, rng, iteration, threads);
    for (int i = 0; i < b.size(); ++i) {
      read_words(b.vectors[static_cast<std::size_t>(i)], out_keys + static_cast<std::int64_t>(i) * n_words, n_words);
      out_log_probs[i] = b.log_probs[i];
    }
    *out_n = b.size();
  });
}
// AnqsModel::batched_grad_log_psi (model.cpp:273-336): out_rows [n][n_params] complex (re, im)
int qref_grad_log_psi(void* m, std::int64_t n, int n_words, const std::uint64_t* keys, int threads, double* out_rows) {
  return guarded([&] {
    const auto& model = *static_cast<qvmc::AnqsModel*>(m);
    const auto vs = make_batch(model.layout().n_qubits, n_words, n, keys);
    const Eigen::MatrixXcd jac = model.batched_grad_log_psi(vs, threads);
    const std::int64_t P = model.n_params();
    for (std::int64_t i = 0; i < n; ++i)
      for (std::int64_t t = 0; t < P; ++t) {
        const std::complex<double> v = jac(i, t);
        out_rows[2 * (i * P + t)] = v.real();
        out_rows[2 * (i * P + t) + 1] = v.imag();
      }
  });
}
// energy_gradient (energy.cpp:93-107) over the rows of batched_grad_log_psi
int qref_energy_gradient(void* m, std::int64_t n, int n_words, const std::uint64_t* keys, const double* weights,
                         const double* locals2, int threads, double* out_grad) {
  return guarded([&] {
    const auto& model = *static_cast<qvmc::AnqsModel*>(m);
    const auto vs = make_batch(model.layout().n_qubits, n_words, n, keys);
    const Eigen::MatrixXcd jac = model.batched_grad_log_psi(vs, threads);
    Eigen::VectorXd w(n);
    Eigen::VectorXcd loc(n);
    for (std::int64_t i = 0; i < n; ++i) {
      w[i] = weights[i];
      loc[i] = std::complex<double>(locals2[2 * i], locals2[2 * i + 1]);
    }
    const Eigen::VectorXd g = qvmc::energy_gradient(w, loc, jac);
    for (Eigen::Index t = 0; t < g.size(); ++t) out_grad[t] = g[t];
  });
}
// condition_max (sampler.cpp:15-23) and CounterRng::gumbel (rng.hpp) for the restatement's pins
double qref_condition_max(double parent, double z, double child) { return qvmc::condition_max(parent, z, child); }
double qref_gumbel(std::uint64_t seed, std::uint32_t stream, std::uint32_t c0, std::uint32_t c1, std::uint32_t c2,
                   std::uint32_t c3) {
  return qvmc::CounterRng(seed, stream).gumbel(c0, c1, c2, c3);
}

}  // extern "C"
