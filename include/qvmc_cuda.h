/*
 * qvmc_cuda.h — C ABI of the B200 surrogate local-energy path.
 *
 * libqvmc_cuda.so (paper_2408_07625_b200/lib/) implements these entry points
 * with hand-written sm_100a kernels. Plain pointers and sizes only: no torch,
 * Eigen or C++ types cross this boundary. Each entry point names the
 * reference interface it replaces (paths relative to /root/reference):
 *
 *   qvmc_cuda_ham_create        device residency of HamiltonianIndex
 *                               (proj/include/qvmc/hamiltonian.hpp:41-107)
 *   qvmc_cuda_pairs[_fetch]     find_coupled_pairs / loop_over_{terms,batch,trie}
 *                               (proj/include/qvmc/coupling.hpp:40-64,
 *                                proj/src/coupling.cpp:62-169)
 *   qvmc_cuda_pair_elements     HamiltonianIndex::group_element per pair
 *                               (proj/src/hamiltonian.cpp:186-194)
 *   qvmc_cuda_local_energies    local_energies (proj/include/qvmc/energy.hpp:23-24,
 *                                proj/src/energy.cpp:13-48)
 *   qvmc_cuda_energy_moments    variational_energy (energy.hpp:39, energy.cpp:50-78)
 *   qvmc_cuda_eloc_fused        find_coupled_pairs + local_energies +
 *                               variational_energy as run_optimisation chains
 *                               them (proj/src/optimizer.cpp:87-93), without
 *                               materialising the pairs
 *   qvmc_cuda_eloc_sharded      the same with the samples sharded as rows over
 *                               the ranks of a communicator
 *
 * Data layout (shared with the reference's BasisVector, basis_vector.hpp:16-26):
 * a basis vector of N qubits is n_words = ceil(N/64) uint64 words, qubit i at
 * word i/64 bit i%64, bits >= N zero. Key arrays are [n][n_words] row-major.
 * Complex outputs are interleaved (re, im) doubles.
 *
 * Memory kind: with QVMC_MEM_HOST every array argument is a host pointer;
 * the call copies in, computes, copies out and returns when done. With
 * QVMC_MEM_DEVICE every array argument is a device pointer on the handle's
 * device; work is enqueued on the handle's stream (qvmc_cuda_set_stream) and
 * the call returns without synchronising, except where noted. Errors raised
 * on the device (zero amplitude, duplicate keys) are then reported by the
 * next qvmc_cuda_synchronize().
 *
 * Errors: every entry point returns a QVMC_* status. The reference throws
 * C++ exceptions; the mapping is QVMC_ERR_INVALID_ARGUMENT ->
 * std::invalid_argument, QVMC_ERR_LOGIC -> std::logic_error,
 * QVMC_ERR_RUNTIME / QVMC_ERR_CUDA -> std::runtime_error. The message of the
 * last failure on the calling thread is qvmc_cuda_last_error().
 */
#ifndef QVMC_CUDA_H
#define QVMC_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  QVMC_OK = 0,
  QVMC_ERR_INVALID_ARGUMENT = 1, /* bad sizes, duplicate keys, malformed masks */
  QVMC_ERR_LOGIC = 2,            /* a sampled state has zero amplitude (energy.cpp:32-33) */
  QVMC_ERR_RUNTIME = 3,          /* zero norm / imaginary residual (energy.cpp:57-58, 74-76) */
  QVMC_ERR_CUDA = 4,             /* CUDA runtime failure */
  QVMC_ERR_NO_DEVICE = 5         /* no sm_100 device visible */
};

/* CouplingBackend (coupling.hpp:17). Every backend returns the identical
 * canonical pair list; they differ in the `ops` they report (coupling.hpp:22-26). */
enum { QVMC_BACKEND_TERMS = 0, QVMC_BACKEND_BATCH = 1, QVMC_BACKEND_TRIE = 2, QVMC_BACKEND_AUTO = 3 };

enum { QVMC_MEM_HOST = 0, QVMC_MEM_DEVICE = 1 };

typedef struct qvmc_ham_s* qvmc_ham_t;     /* device-resident HamiltonianIndex + workspace */
typedef struct qvmc_index_s* qvmc_index_t; /* host-side grouped index (from_terms result) */

/* Counters of the last pairs/fused call on a handle. */
typedef struct {
  uint64_t rows;            /* source rows processed */
  uint64_t candidates;      /* candidates visited on the device: (x, flip mask) probes, or
                               bucket members in join mode */
  uint64_t pairs;           /* coupled pairs found (incl. the diagonal) */
  uint64_t terms_equivalent;/* n_rows * |XY|: the LoopOverTerms candidate count */
  int32_t sector_mode;      /* 1 = particle-sector candidate lists, 0 = full flip-mask scan */
  int32_t sector_side;      /* 1 = occupied orbitals are the minority set, 0 = holes */
  int32_t minority_count;   /* |minority set| per key in sector mode */
  int32_t join_mode;        /* 1 = candidates from the per-call deletion index (join path),
                               2 = that index built across the ranks of a sharded call */
  float table_ms;           /* CUDA-event times of the last fused call's stages on the */
  float rows_ms;            /* handle's stream: sample-set hash build, row kernel,     */
  float moments_ms;         /* moment reduction                                       */
  float search_ms;          /* join path, split evaluation: the search kernel and the  */
  float eval_ms;            /* chunk evaluation kernel inside rows_ms (else 0)         */
} qvmc_stats;

/* ------------------------------------------------------------------ host index */

/* HamiltonianIndex::from_terms (hamiltonian.cpp:63-117) over raw Pauli
 * strings given as disjoint (x, y, z) masks, [n_raw][n_words] each: merges
 * duplicate strings in first-occurrence order, drops |coeff| < 1e-12,
 * groups by xy = x|y in first-occurrence order. */
int qvmc_index_build(int n_qubits, int n_words, int64_t n_raw, const double* coeff, const uint64_t* x_words,
                     const uint64_t* y_words, const uint64_t* z_words, qvmc_index_t* out);
int qvmc_index_info(qvmc_index_t idx, int* n_qubits, uint64_t* n_terms, uint32_t* n_xy, int64_t* diag_xy);
/* Any output pointer may be NULL. Arrays: xy_words[n_xy][n_words],
 * group_offsets[n_xy+1], coeff[n_terms], yz_words[n_terms][n_words],
 * y_weight[n_terms], x/y/z_words[n_terms][n_words] (the merged strings). */
int qvmc_index_export(qvmc_index_t idx, uint64_t* xy_words, uint64_t* group_offsets, double* coeff,
                      uint64_t* yz_words, uint8_t* y_weight, uint64_t* x_words, uint64_t* y_words,
                      uint64_t* z_words);
void qvmc_index_destroy(qvmc_index_t idx);

/* Device-layout plan of an index, computed on the host (no device needed),
 * for tests and diagnostics: groups per join drain-record kind (A: weight-2/4
 * group whose terms share one Z string and fit one 64-byte record; B: compact
 * family-compressed single excitation; C: term by term; D: general family
 * compression), set bits of the pair-existence bitmaps (0 when N > 128),
 * weight-2 / weight-4 flip masks and flip-table buckets. */
typedef struct {
  uint64_t kind_a, kind_b, kind_c, kind_d;
  uint64_t bitmap_bits;
  uint64_t singles, doubles;
  uint64_t xy_tab_buckets;
} qvmc_plan_summary;
int qvmc_index_plan_summary(qvmc_index_t idx, qvmc_plan_summary* out);

/* ------------------------------------------------------------ device handle */

/* Upload a grouped HamiltonianIndex. Arguments mirror the index's members:
 * xy_set (first-occurrence order), group_offsets (CSR, size n_xy+1), and the
 * grouped terms' coeff, yz mask and y_weight; diag_xy = diagonal_xy_index()
 * or -1. device = CUDA ordinal. Builds the device-side candidate lists. */
int qvmc_cuda_ham_create(int n_qubits, int n_words, uint32_t n_xy, const uint64_t* xy_words,
                         const uint64_t* group_offsets, uint64_t n_terms, const double* coeff,
                         const uint64_t* yz_words, const uint8_t* y_weight, int64_t diag_xy, int device,
                         qvmc_ham_t* out);
int qvmc_cuda_ham_create_from_index(qvmc_index_t idx, int device, qvmc_ham_t* out);
int qvmc_cuda_ham_destroy(qvmc_ham_t h);
/* Run subsequent work on this cudaStream_t (NULL = the handle's own stream). */
int qvmc_cuda_set_stream(qvmc_ham_t h, void* stream);
/* Wait for the handle's stream and report deferred device-side errors. */
int qvmc_cuda_synchronize(qvmc_ham_t h);
/* Opt in (on = 1) to speculative device-memory calls of qvmc_cuda_eloc_fused:
 * once a call has planned the sample set (particle sector and minority size,
 * one host read), later QVMC_MEM_DEVICE calls with the same n_unq reuse that
 * plan and check it on the device, and the split evaluation checks its hit
 * buffers on the device too: such a call performs no host synchronisation
 * at all (it can be captured in a CUDA graph once its buffers are sized).
 * The next qvmc_cuda_synchronize (or any synchronising call on the handle)
 * verifies it and, if the plan did not hold or a buffer overflowed, reruns
 * it synchronously from the same arguments, so the caller must keep the
 * arguments valid until then. Off by default. */
int qvmc_cuda_set_speculative(qvmc_ham_t h, int on);
int qvmc_cuda_last_stats(qvmc_ham_t h, qvmc_stats* out); /* synchronises */

/* ------------------------------------------------------------ coupled pairs */

/* find_coupled_pairs (coupling.cpp:153-169): all ordered (x, x') of the
 * batch with x^x' in the flip-mask set, canonical order (x, then x').
 * backend / auto_threshold select the reported `ops` semantics exactly as
 * the reference: terms = n_unq*|XY|, batch = n_unq^2, trie = candidates
 * actually probed; auto = batch below auto_threshold else trie.
 * Synchronises; the pair list stays on the device until fetched. */
int qvmc_cuda_pairs(qvmc_ham_t h, int64_t n_unq, const uint64_t* keys, int mem, int backend, int auto_threshold,
                    uint64_t* n_pairs, uint64_t* ops, int* backend_used);
/* Copy the last pair list as (x, x', xy) uint32 triples (CoupledPairs::Entry). */
int qvmc_cuda_pairs_fetch(qvmc_ham_t h, uint32_t* out_entries, int mem);

/* Per pair (x, x', xy): H_{x x'} = group_element(x', xy) evaluated term by
 * term in the reference's order (bit-identical to hamiltonian.cpp:186-194),
 * and the excitation class popcount(xy). out_h: [n_pairs][2]; out_class may
 * be NULL. */
int qvmc_cuda_pair_elements(qvmc_ham_t h, int64_t n_unq, const uint64_t* keys, uint64_t n_pairs,
                            const uint32_t* entries, double* out_h, uint8_t* out_class, int mem);

/* Per pair (x, x', xy): H_{x x'} through the evaluators of the fused path
 * (qvmc_cuda_eloc_fused): the 64-byte drain records of weight-2/4 flip masks
 * (kinds A-D) and the diagonal quadratic form, with out_kind[e] = 0-3 (drain
 * record kind A-D), 4 (term by term, as group_element) or 5 (diagonal
 * quadratic form). Kind A is bit-identical to group_element
 * (hamiltonian.cpp:186-194); the family forms B/D and the quadratic form
 * reorder the fp64 sum. Exposes the fused arithmetic for parity tests. */
int qvmc_cuda_pair_elements_fused(qvmc_ham_t h, int64_t n_unq, const uint64_t* keys, uint64_t n_pairs,
                                  const uint32_t* entries, double* out_h, uint8_t* out_kind, int mem);

/* ------------------------------------------------------------ local energies */

/* local_energies (energy.cpp:13-48) from canonical pairs. out_eloc[n_unq][2].
 * QVMC_ERR_LOGIC when any log_amp is infinite. */
int qvmc_cuda_local_energies(qvmc_ham_t h, int64_t n_unq, const uint64_t* keys, const double* log_amp,
                             const double* phase, uint64_t n_pairs, const uint32_t* entries, double* out_eloc,
                             int mem);

/* variational_energy moments (energy.cpp:50-78) over rows [0, n):
 * w = exp(log_prob - log_norm); out_moments[5] = (sum w*Re E, sum w*Im E,
 * sum w^2 (= ipr), sum w, sum w*|E|^2). out_weights[n] optional. The
 * reference's norm / residual checks are the caller's (host) step. */
int qvmc_cuda_energy_moments(qvmc_ham_t h, int64_t n, const double* log_prob, double log_norm, const double* eloc,
                             double* out_moments, double* out_weights, int mem);

/* The fused surrogate-E_loc throughput path: for rows [row_begin, row_end)
 * of the sample set `keys` (all n_unq rows are partners), E_loc plus the five
 * moments of those rows, with no pair materialisation. out_eloc
 * [(row_end-row_begin)][2] may be NULL. Multi-GPU callers shard rows and
 * pass the all-gathered sample set. */
int qvmc_cuda_eloc_fused(qvmc_ham_t h, int64_t n_unq, const uint64_t* keys, const double* log_amp,
                         const double* phase, const double* log_prob, double log_norm, int64_t row_begin,
                         int64_t row_end, double* out_eloc, double* out_moments, int mem);

/* ------------------------------------------------------------------ multi-GPU */

/* Rows [begin, end) of `rank` in the contiguous balanced split of n_total rows
 * over `world` ranks (the first n_total % world ranks hold one extra row): the
 * shard each rank passes to qvmc_cuda_eloc_sharded. */
int qvmc_shard_bounds(int64_t n_total, int world, int rank, int64_t* begin, int64_t* end);

/* A communicator for the sharded path: NCCL over NVLink/NVSwitch (libnccl.so.2
 * is opened at run time), or a host all-gather callback (MPI, gloo, tests).
 * NCCL: rank 0 calls qvmc_cuda_comm_unique_id (ncclGetUniqueId, 128 bytes),
 * the caller distributes the id, every rank calls qvmc_cuda_comm_init_nccl
 * (ncclCommInitRank on `device`); or wrap an ncclComm_t the caller owns. */
typedef struct qvmc_comm_s* qvmc_comm_t;
/* all-gather bytes_per_rank bytes from every rank into recv[world][bytes_per_rank],
 * host buffers; returns 0 on success */
typedef int (*qvmc_host_allgather_fn)(void* ctx, const void* send, void* recv, uint64_t bytes_per_rank);
int qvmc_cuda_comm_unique_id(void* out, uint64_t out_bytes);
int qvmc_cuda_comm_init_nccl(int device, int world, int rank, const void* unique_id, qvmc_comm_t* out);
int qvmc_cuda_comm_wrap_nccl(void* nccl_comm, int world, int rank, qvmc_comm_t* out);
int qvmc_cuda_comm_init_host(int world, int rank, qvmc_host_allgather_fn all_gather, void* ctx, qvmc_comm_t* out);
int qvmc_cuda_comm_destroy(qvmc_comm_t c);

/* The sharded throughput path: find_coupled_pairs + local_energies +
 * variational_energy as run_optimisation chains them
 * (proj/src/optimizer.cpp:87-93), with the unique samples split over the
 * ranks of `comm` as rows. Each rank passes its own shard
 * (qvmc_shard_bounds rows of an n_total-row sample set: keys, log|psi|,
 * phase, log p); the call all-gathers the shards (one all-gather of packed
 * [W + 3]-word records) and evaluates E_loc against the whole set with the
 * fused kernels. The walk is balanced independently of the caller's sample
 * order: rank r walks every world-th sample of the locality-sorted set
 * (QVMC_STRIDED_SHARDS=0: its own rows), and one integer all-reduce assembles
 * the rows (each written by exactly one rank, so the result is exact); the
 * per-rank moments of its own rows are gathered and summed in rank order
 * (deterministic). out_eloc: this rank's rows [rows][2];
 * out_moments[5]: global, as qvmc_cuda_eloc_fused. With QVMC_MEM_DEVICE and
 * the NCCL backend every step is enqueued on the handle's stream. */
int qvmc_cuda_eloc_sharded(qvmc_ham_t h, qvmc_comm_t comm, int64_t n_total, const uint64_t* keys,
                           const double* log_amp, const double* phase, const double* log_prob, double log_norm,
                           double* out_eloc, double* out_moments, int mem);

/* Message of the last failure on the calling thread ("" if none). */
/* ------------------------------------------------------------------ amplitude model */

/* AnqsModel (proj/include/qvmc/model.hpp:47-157, proj/src/model.cpp) on the
 * device: the qudit-grouped autoregressive ansatz whose log ψ / φ feed the
 * local-energy path. Create = QuditLayout::make +
 * AnqsModel::AnqsModel (model.cpp:33-58), same argument checks and messages;
 * the device path additionally requires hidden = 64 and bits_per_qudit <= 6
 * (the reference defaults, model.hpp:24,61) and says so otherwise. */
typedef struct qvmc_model_s* qvmc_model_t;
int qvmc_cuda_model_create(int n_qubits, int bits_per_qudit, int n_electrons, int spin_constraint, int hidden,
                           int device, qvmc_model_t* out);
int qvmc_cuda_model_destroy(qvmc_model_t m);
/* AnqsModel::n_params (model.hpp:67) */
int qvmc_cuda_model_n_params(qvmc_model_t m, int64_t* out);
/* AnqsModel::set_params (model.cpp:99-103): host array in the reference's flat
 * layout (model.cpp:65-80: per qudit the amplitude block then the phase block,
 * each W1[hidden][n] b1 W2[hidden][hidden] b2 W3[2^k][hidden] b3, row-major). */
int qvmc_cuda_model_set_params(qvmc_model_t m, int64_t n_params, const double* params);
int qvmc_cuda_model_set_stream(qvmc_model_t m, void* stream);
/* AnqsModel::log_psi (model.cpp:262-271) per key, keys [n][ceil(N/64)];
 * out-of-sector keys give (-inf, 0) like the reference. */
int qvmc_cuda_log_psi(qvmc_model_t m, int64_t n, const uint64_t* keys, int mem, double* out_log_amp,
                      double* out_phase);
/* fill_amplitudes (proj/src/sampler.cpp:104-120): log_psi of every key and
 * out_norm2 = (norm, log_norm) = logsumexp(log_probs), out_norm2 on the host.
 * Synchronises. */
int qvmc_cuda_fill_amplitudes(qvmc_model_t m, int64_t n, const uint64_t* keys, const double* log_probs, int mem,
                              double* out_log_amp, double* out_phase, double* out_norm2);
/* 1 when the last qvmc_cuda_fill_amplitudes call recognised the batch as the one
 * qvmc_cuda_sample produced under the current parameters (same size, parameter
 * version and device fingerprint of keys and log p): log|psi| = 0.5 log p exactly
 * (the sampler summed the same amplitude-head values in qudit order) and only the
 * phase heads were evaluated; 0 when both heads ran. QVMC_FAST_FILL=0 disables. */
int qvmc_cuda_model_last_fill_sampled(qvmc_model_t m);
/* 1 when the last qvmc_cuda_energy_gradient call found the phase heads' h1 / h2
 * activations of its batch kept by the sampled-batch fill (same size, parameter
 * version and keys fingerprint) and copied them instead of recomputing the phase
 * blocks' forward pass (bit-identical); 0 otherwise. QVMC_GRAD_CACHE=0 disables. */
int qvmc_cuda_model_last_gradient_cached(qvmc_model_t m);
int qvmc_cuda_model_synchronize(qvmc_model_t m);
/* energy_gradient (proj/src/energy.cpp:93-107, GradientAccumulator :80-91)
 * over the rows of batched_grad_log_psi (proj/src/model.cpp:273-336) of the
 * n keys, as run_optimisation streams them (optimizer.cpp:105-140):
 * grad = sum_i 2 Re{ w_i (E_i - E) O_i }, E = sum_i w_i E_i, O_i = d log|psi|
 * - i d phase. The Jacobian is never materialised: per-sample backward
 * vectors are contracted on the device (strided-batched DGEMMs). locals
 * [n][2] (re, im); out_grad [n_params] in the reference's flat layout. Keys
 * outside the model's sector: QVMC_ERR_INVALID_ARGUMENT (grad_log_psi's
 * "state is masked"). Synchronises. */
int qvmc_cuda_energy_gradient(qvmc_model_t m, int64_t n, const uint64_t* keys, const double* weights,
                              const double* locals, int mem, double* out_grad);
/* AnqsModel::params() (model.hpp:66): the flat parameter vector (the model
 * keeps a device copy next to the kernels' layout). */
int qvmc_cuda_model_get_params(qvmc_model_t m, int mem, double* out);
/* adam_step (proj/src/optimizer.cpp:17-31) followed by model.set_params
 * (optimizer.cpp:157), all on the device: bias-corrected Adam with the
 * model's own state (zero on first use, step counter kept), then the
 * kernels' layout refreshed from the updated flat vector. A non-finite
 * direction entry: QVMC_ERR_RUNTIME "adam_step: non-finite direction entry",
 * nothing updated. direction [n_params] in host or device memory. */
int qvmc_cuda_model_adam_step(qvmc_model_t m, const double* direction, double learning_rate, double beta1,
                              double beta2, double epsilon, int mem);
/* sr_direction (proj/src/sr.cpp:74-95) for a given SrContext: stacked
 * row-major [rows][cols] (rows = 2 n_sr), lambda > 0, grad [cols]: the
 * push-through solve with the Gram eigensystem (cuSOLVER syevd); the
 * reference's conditioning check (runtime_error "ill-conditioned system,
 * cond ~ ...", QVMC_ERR_RUNTIME). out_direction [cols]. Synchronises. */
int qvmc_cuda_sr_solve(qvmc_model_t m, int64_t rows, int64_t cols, const double* stacked, double lambda,
                       const double* grad, int mem, double* out_direction);
/* The SR step of run_optimisation (optimizer.cpp:105-143): the n_sr samples
 * of highest log p (top_probability_indices, sr.cpp:15-23, ties in sample
 * order), their grad_log_psi rows (model.cpp:273-325), build_sr_context
 * (sr.cpp:25-72; lambda <= 0 picks 1e-4 (1 + ||stacked||_F^2 / n_sr)) and
 * sr_direction applied to grad [n_params]. locals [n][2] is accepted for the
 * optimiser's call shape but not read (the SR context needs the samples and
 * their weights only). out_lambda may be NULL. Synchronises. */
int qvmc_cuda_sr_direction(qvmc_model_t m, int64_t n, const uint64_t* keys, const double* log_probs,
                           const double* locals, int n_sr, double lambda, const double* grad, int mem,
                           double* out_direction, double* out_lambda);
/* sample_without_replacement (proj/src/sampler.cpp:37-102): the ancestral
 * Gumbel top-K beam with CounterRng(seed, stream) (rng.hpp:30-63) and the
 * iteration index, the model's conditionals evaluated on the device. Writes
 * *out_n = min(K, sector size) distinct keys [*out_n][ceil(N/64)] and their
 * log-probabilities in the reference's order (conditioned perturbed value
 * descending, ties by key). out_keys / out_log_probs hold K entries, host or
 * device memory per `mem`. Synchronises. */
int qvmc_cuda_sample(qvmc_model_t m, int k_samples, uint64_t seed, uint32_t stream, uint32_t iteration, int mem,
                     uint64_t* out_keys, double* out_log_probs, int64_t* out_n);

const char* qvmc_cuda_last_error(void);
/* Kernels launched by this library since load (for launch accounting). */
uint64_t qvmc_cuda_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
