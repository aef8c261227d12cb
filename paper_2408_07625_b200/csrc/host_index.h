// Host-side (CPU, setup-time) pieces of libqvmc_cuda: the grouped
// HamiltonianIndex and the device-layout planner.
// Nothing here runs per sample; the per-sample work is in qvmc_cuda.cu.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace qvmc_b200 {

constexpr int kMaxWords = 4;        // 256 qubits, BasisVector::kMaxBits (basis_vector.hpp:29)
constexpr int kMaxMinority = 32;    // sector lists are used when min(n_e, N - n_e) <= 32
constexpr uint32_t kSmallGroupHost = 16;  // groups above this size are candidates for compression
constexpr int kMaxFamilies = 4;
constexpr int kGrecWordsHost = 8;   // qvmc_join.cuh kGrecWords
constexpr int kBinomKHost = 33;     // qvmc_join.cuh kBinomK

// C(n, k) for n <= 256, k < kBinomKHost, saturating at UINT64_MAX
// ([257][kBinomKHost], the combinadic ranks of the join's bucket keys)
std::vector<uint64_t> binomial_table();

// HamiltonianIndex (proj/include/qvmc/hamiltonian.hpp:41-107) as flat arrays.
struct HostIndex {
  int n_qubits = 0;
  int n_words = 0;
  std::vector<uint64_t> xy;       // [n_xy][n_words], first-occurrence order
  std::vector<uint64_t> offsets;  // [n_xy+1]
  std::vector<double> coeff;      // [n_terms], grouped
  std::vector<uint64_t> x, y, z;  // [n_terms][n_words], merged strings
  std::vector<uint64_t> yz;       // [n_terms][n_words]
  std::vector<uint8_t> y_weight;  // [n_terms]
  int64_t diag = -1;

  uint32_t n_xy() const { return static_cast<uint32_t>(offsets.empty() ? 0 : offsets.size() - 1); }
  uint64_t n_terms() const { return coeff.size(); }
};

// HamiltonianIndex::from_terms (hamiltonian.cpp:63-117). Throws
// std::invalid_argument on malformed masks.
HostIndex index_from_terms(int n_qubits, int n_words, int64_t n_raw, const double* coeff, const uint64_t* xw,
                           const uint64_t* yw, const uint64_t* zw);

// Random 64-bit code per qubit; the linear key hash is the XOR of the codes
// of the set bits (so hash(x ^ m) = hash(x) ^ hash(m)).
const uint64_t* qubit_codes();  // [256]
uint64_t linear_hash(const uint64_t* words, int n_words);
// orbital positions of a weight-2/4 mask, ascending, 8 bits each, 0xFF padded
uint32_t xy_position_key(const uint64_t* words, int n_words);

// Everything the kernels need besides the raw index, planned on the host.
struct DevicePlan {
  std::vector<uint64_t> xy_hash;    // [n_xy]
  std::vector<uint32_t> offsets32;  // [n_xy+1]
  std::vector<uint8_t> xy_weight;   // [n_xy] popcount(xy) = excitation class
  // full scan (generic mode): every non-diagonal group
  std::vector<uint64_t> gen_hash;
  std::vector<uint32_t> gen_g;
  // particle-sector lists: list p (< N) holds weight-2 masks containing p;
  // list N + pair(p,q) holds weight-4 masks containing p and q.
  std::vector<uint32_t> lst_off;
  std::vector<uint64_t> lst_hash;
  std::vector<uint32_t> lst_g;
  std::vector<uint32_t> res_g;      // even weight >= 6
  // diagonal group as a quadratic form in the occupations
  bool diag_quad = false;
  double diag_A[2] = {0.0, 0.0};    // [side] side 1 = occupied minority, 0 = holes
  std::vector<double> diag_b;       // [2][N]
  std::vector<double> diag_K;       // [N][N]
  std::vector<uint32_t> diag_other; // diagonal terms with |z| >= 3
  std::vector<uint64_t> hash_bytes; // [n_words*8][256]
  // compressed large groups: a group whose terms share a few base yz masks
  // (differing by at most one Z per term) is summed as families
  //   i^q_f (-1)^{|x' & B_f|} [u_f + sum_k v_f[k] (-1)^{x'_k}]
  std::vector<int32_t> comp_of;     // [n_xy] compressed-group id or -1
  std::vector<uint32_t> fam_off;    // [n_comp+1]
  std::vector<uint64_t> fam_B;      // [n_fam][W]
  std::vector<uint8_t> fam_q;       // [n_fam] y-weight mod 4
  std::vector<double> fam_u, fam_V; // [n_fam] constant part, sum_k v_f[k]
  std::vector<double> fam_v;        // [n_fam][N]
  // hot-path records (one load each): per group (t0, n_terms, first family or
  // ~0, n_families | q_f << (8 + 2f)); per term (yz words, coeff bits, y_weight)
  // padded to 16 B; per family (u_f, V_f, B_f words) padded to 16 B
  std::vector<uint32_t> ginfo;      // [n_xy][4]
  std::vector<uint64_t> trec;       // [n_terms][term_words(W)]
  std::vector<uint64_t> famrec;     // [n_fam][fam_words(W)]
  // join-path drain records (qvmc_join.cuh): [n_xy][kGrecWordsHost]
  std::vector<uint64_t> grec;
  // join-path existence bitmaps over orbital pairs (n <= 128): [P bits singles][P*P bits doubles]
  std::vector<uint32_t> pbits;
  uint32_t pbits_P = 0;
  std::vector<double> famvi;        // compact kind-B groups: v_f[k] interleaved [N][nf padded to 1/2/4]
  // flip-mask table (join path): buckets of 4 x (position key32 << 32 | group)
  std::vector<uint64_t> xy_tab;
  uint64_t xy_tab_mask = 0;
};

// bucket-chain finaliser shared with the device (qvmc_kernels.cuh fmix)
inline uint64_t fmix_host(uint64_t h) {
  h ^= h >> 29;
  h *= 0xbf58476d1ce4e5b9ull;
  h ^= h >> 32;
  return h;
}

// first flip-table bucket of a position key, shared with the device (qvmc_join.cuh xy_bucket)
inline uint32_t xy_bucket_host(uint32_t key, uint32_t mask) {
  key ^= key >> 16;
  key *= 0x85ebca6bu;
  key ^= key >> 13;
  key *= 0xc2b2ae35u;
  key ^= key >> 16;
  return key & mask;
}

DevicePlan plan_device(const HostIndex& h);

constexpr int term_words(int W) { return (W + 2 + 1) & ~1; }
constexpr int fam_words(int W) { return (W + 2 + 1) & ~1; }

inline uint32_t pair_index(int p, int q, int n) {  // p < q
  return static_cast<uint32_t>(p * n - p * (p + 1) / 2 + (q - p - 1));
}

}  // namespace qvmc_b200
