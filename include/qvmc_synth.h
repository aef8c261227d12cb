/*
 * qvmc_synth.h — seeded synthetic inputs for tests and
 * bench.py, in libqvmc_synth.so (paper_2408_07625_b200/lib/, built from
 * csrc/synth.cpp with g++ only). Not part of the local-energy path and not
 * in libqvmc_cuda.so. The reference ships no molecule fixtures beyond
 * toy/h2/h4/h6 and its random_hamiltonian (proj/src/synthetic.cpp:18-49) has
 * no off-diagonal couplings at 56/118 qubits, so the throughput inputs are
 * JW-structured Pauli strings plus near-HF determinants.
 * Return 0 on success, 1 on error (message from qvmc_synth_last_error()).
 */
#ifndef QVMC_SYNTH_H
#define QVMC_SYNTH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* JW-structured molecular-like Hamiltonian: identity, N Z, C(N,2) ZZ;
 * same-spin single groups {XZ..ZX, YZ..ZY} with one optional extra Z_k
 * dressing (2+2(N-2) terms per group); spin-conserving doubles over two even
 * + two odd sites with patterns XXYY/YYXX/XYYX/YXXY and JW Z-strings, until
 * n_terms_target strings. Arrays sized n_terms_target; *n_out = strings
 * written. */
int qvmc_synth_jw_hamiltonian(int n_qubits, int64_t n_terms_target, uint64_t seed, double* coeff, uint64_t* x_words,
                              uint64_t* y_words, uint64_t* z_words, int64_t* n_out);
/* n_unq distinct near-Hartree-Fock determinants: first n_electrons orbitals
 * occupied, then 1+Geometric(0.6) random same-spin occupied->empty moves. */
int qvmc_synth_near_hf_samples(int n_qubits, int n_electrons, int64_t n_unq, uint64_t seed, uint64_t* keys);
const char* qvmc_synth_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
