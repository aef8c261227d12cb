/*
 * qvmc_oracle — CPU restatement of the reference hot path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library, and only as the
 * checker. The product path (paper_2408_07625_b200) never calls it.
 *
 * Parity is pinned: tests/test_oracle.py checks every function here against
 * the reference's own known-answer tests (toy/h2/h4/h6 fixtures, the worked
 * toy pairs and energies) and against oracle/_ref (the unmodified reference
 * sources compiled in place) on the reference tests' seeded random families.
 *
 * Keys are packed basis vectors: n_words uint64 words per vector, qubit i at
 * word i/64 bit i%64, zero tail (proj/include/qvmc/basis_vector.hpp:16-26).
 */
#ifndef QVMC_ORACLE_H
#define QVMC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qo_index qo_index;

/* HamiltonianIndex::from_terms (proj/src/hamiltonian.cpp:63-117) over raw
 * (coeff, x, y, z) masks. Returns NULL and sets qo_last_error on bad input. */
qo_index* qo_index_from_terms(int n_qubits, int n_words, int64_t n_raw, const double* coeff,
                              const uint64_t* x_words, const uint64_t* y_words, const uint64_t* z_words);
void qo_index_free(qo_index* h);
void qo_index_info(const qo_index* h, int64_t* n_terms, int64_t* n_xy, int64_t* diag_xy);
/* Export the grouped layout (any pointer may be NULL). */
void qo_index_export(const qo_index* h, uint64_t* xy_words, int64_t* group_offsets, double* coeff,
                     uint64_t* yz_words, uint8_t* y_weight);
const char* qo_last_error(void);

/* group_element (hamiltonian.cpp:186-194); out2 = (re, im). */
void qo_group_element(const qo_index* h, const uint64_t* x_prime, int64_t g, double* out2);
/* matrix_element (hamiltonian.cpp:178-184). */
void qo_matrix_element(const qo_index* h, const uint64_t* x, const uint64_t* x_prime, double* out2);

/* Coupled pairs in canonical order (coupling.cpp:37-58). backend 0 = terms
 * semantics (coupling.cpp:62-84, ops = n_unq*|XY|), 1 = batch semantics
 * (coupling.cpp:86-102, ops = n_unq^2). Returns number of pairs, or -1 on
 * error (duplicate keys). *out3 is malloc'd (x, x', xy) triples; free with
 * qo_free. */
int64_t qo_pairs(const qo_index* h, int64_t n_unq, const uint64_t* keys, int backend, uint32_t** out3,
                 uint64_t* ops);
void qo_free(void* p);

/* local_energies (energy.cpp:13-48) over canonical pairs; out interleaved
 * (re, im). Returns 0, or -2 when a sampled log-amplitude is infinite. */
int qo_local_energies(const qo_index* h, int64_t n_unq, const uint64_t* keys, const double* log_amp,
                      const double* phase, int64_t n_pairs, const uint32_t* pairs3, double* out_eloc);

/* variational_energy (energy.cpp:50-78). out5 = (e_var, im_residual, ipr,
 * sum_w, sum_w|E|^2). Returns 0, -3 for a non-positive norm, -4 for an
 * imaginary residual above 1e-6*max(1,|E|) (out5 still filled). */
int qo_variational_energy(int64_t n, const double* log_prob, double norm, double log_norm,
                          const double* eloc, double* out5, double* weights);

/* Surrogate E_loc for rows [row_begin, row_end) against the whole sample
 * set, terms semantics, without materialising pairs (same arithmetic as
 * qo_pairs + qo_local_energies restricted to those rows). Threads > 1 split
 * rows. out is indexed by row - row_begin. out_scale (optional) receives the
 * absolute-sum scale sum_pairs sum_{t in group} |c_t| exp(dlog) per row.
 * Returns pairs visited or <0. */
int64_t qo_eloc_rows(const qo_index* h, int64_t n_unq, const uint64_t* keys, const double* log_amp,
                     const double* phase, int64_t row_begin, int64_t row_end, int threads, double* out_eloc,
                     double* out_scale);

/* Rows of a row LIST (indices into keys) against the whole sample set,
 * terms semantics: *out3 (malloc'd, free with qo_free) = every listed row's
 * canonical pairs, rows in list order; out_counts[k] = pairs of rows[k].
 * With log_amp/phase non-NULL also out_eloc[k] (interleaved re, im) and
 * optional out_scale[k] as qo_eloc_rows. Returns total pairs or <0. */
int64_t qo_rows_list(const qo_index* h, int64_t n_unq, const uint64_t* keys, const double* log_amp,
                     const double* phase, int64_t n_rows, const int64_t* rows, int threads, uint32_t** out3,
                     int64_t* out_counts, double* out_eloc, double* out_scale);

#ifdef __cplusplus
}
#endif
#endif
