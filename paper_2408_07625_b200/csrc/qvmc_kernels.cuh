// Device code of the B200 surrogate local-energy path (sm_100a).
//
// One warp owns one source row x at a time (rows are handed out by an atomic
// row counter, so HF-like rows with many partners do not stall a static
// partition). For x the warp enumerates candidate flip masks m, forms the
// candidate x' = x ^ m only through its hash (the key hash is linear over
// GF(2), hash(x ^ m) = hash(x) ^ hash(m), and hash(m) is precomputed per
// mask), and probes the sample-set hash table. Hits are verified against the
// stored key, then H_{x x'} and the amplitude ratio are accumulated in fp64.
// See DESIGN.md for the layout and the roofline.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>

namespace qvmc_b200 {

constexpr uint64_t kEmpty = ~0ull;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 4;  // independent probes in flight per lane

enum : int { kErrDuplicate = 1, kErrZeroAmp = 2, kErrBadPair = 4, kErrHitOverflow = 8,
             kErrReplan = 16,    // a speculative call's cached sector plan did not hold
             kErrSliceOverflow = 32,  // a rank's share of a distributed index exceeded its capacity
             kErrFixRange = 64 };     // a mirrored contribution beyond the fixed-point range (|v| >= 2^46)
enum : int { kModeEloc = 0, kModeCount = 1, kModeEmit = 2, kModeHits = 3, kModeFused = 4 };

struct HamView {
  int n;        // qubits
  uint32_t n_xy;
  int32_t diag; // -1 when there is no diagonal group
  const uint64_t* xy;       // [n_xy][W]
  const uint64_t* xy_hash;  // [n_xy]
  const uint32_t* goff;     // [n_xy+1]
  const double* coeff;      // [n_terms]
  const uint64_t* yz;       // [n_terms][W]
  const uint8_t* yw;        // [n_terms]
  const uint8_t* xyw;       // [n_xy]
  const uint64_t* gen_hash; // non-diagonal groups (full scan)
  const uint32_t* gen_g;
  uint32_t n_gen;
  const uint32_t* lst_off;  // sector lists (CSR), null when absent
  const uint64_t* lst_hash;
  const uint32_t* lst_g;
  const uint32_t* res_g;
  uint32_t n_res;
  int diag_quad;
  double diag_A0, diag_A1;
  const double* diag_b;     // [2][n]
  const double* diag_K;     // [n][n]
  const uint32_t* diag_other;
  uint32_t n_diag_other;
  const uint64_t* hash_bytes;  // [W*8][256]
  const int32_t* comp_of;      // compressed large groups (host_index.h DevicePlan)
  const uint32_t* fam_off;
  const uint64_t* fam_B;
  const uint8_t* fam_q;
  const double* fam_u;
  const double* fam_V;
  const double* fam_v;
  const uint4* ginfo;          // per group (t0, n_terms, first family, n_fam | q bits)
  const uint64_t* trec;        // per term (yz words, coeff, y_weight), term_words(W) words
  const uint64_t* famrec;      // per family (u, V, B words), fam_words(W) words
};

constexpr int term_words_dev(int W) { return (W + 2 + 1) & ~1; }
constexpr int fam_words_dev(int W) { return (W + 2 + 1) & ~1; }

struct TableView {
  uint64_t* tab;  // buckets of 4 entries: (tag << 32) | row, kEmpty when free
  uint64_t mask;  // n_buckets - 1
};

struct Ctl {
  int* err;
  unsigned long long* row_next;
  unsigned long long* stats;  // [0] candidates, [1] pairs
  int* popc_mm;               // [0] max popcount, [1] max (1024 - popcount)
};

__device__ __forceinline__ uint64_t fmix(uint64_t h) {
  h ^= h >> 29;
  h *= 0xbf58476d1ce4e5b9ull;
  h ^= h >> 32;
  return h;
}

template <int W>
__device__ __forceinline__ uint64_t key_hash_thread(const uint64_t* x, const uint64_t* __restrict__ hb) {
  uint64_t h = 0;
#pragma unroll
  for (int k = 0; k < W * 8; ++k) h ^= __ldg(hb + k * 256 + ((x[k >> 3] >> (8 * (k & 7))) & 0xff));
  return h;
}

// the lanes of a warp split the W*8 byte lookups of a (warp-uniform) key
template <int W>
__device__ __forceinline__ uint64_t key_hash_warp(const uint64_t* x, const uint64_t* __restrict__ hb, int lane) {
  uint64_t h = 0;
  if (lane < W * 8) {
    uint64_t word = x[0];
#pragma unroll
    for (int w = 1; w < W; ++w)
      if ((lane >> 3) == w) word = x[w];
    h = __ldg(hb + lane * 256 + ((word >> (8 * (lane & 7))) & 0xff));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h ^= __shfl_xor_sync(0xffffffffu, h, o);
  return h;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------ hash table

template <int W>
__global__ void __launch_bounds__(kThreads) k_table_build(const uint64_t* __restrict__ keys, int64_t n,
                                                          const uint64_t* __restrict__ hb, TableView T, Ctl C) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x[W];
    int pc = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      x[w] = keys[i * W + w];
      pc += __popcll(x[w]);
    }
    atomicMax(C.popc_mm, pc);
    atomicMax(C.popc_mm + 1, 1024 - pc);
    const uint64_t f = fmix(key_hash_thread<W>(x, hb));
    const uint32_t tag = static_cast<uint32_t>(f >> 32);
    const uint64_t entry = (static_cast<uint64_t>(tag) << 32) | static_cast<uint64_t>(i);
    uint64_t b = f & T.mask;
    for (;;) {
      bool done = false;
#pragma unroll 1
      for (int k = 0; k < 4 && !done; ++k) {
        unsigned long long* slot = reinterpret_cast<unsigned long long*>(T.tab + b * 4 + k);
        const uint64_t old = atomicCAS(slot, kEmpty, entry);
        if (old == kEmpty) {
          done = true;
        } else if (static_cast<uint32_t>(old >> 32) == tag) {
          const uint32_t j = static_cast<uint32_t>(old);
          bool same = true;
#pragma unroll
          for (int w = 0; w < W; ++w) same &= keys[(int64_t)j * W + w] == x[w];
          if (same) {
            atomicOr(C.err, kErrDuplicate);
            done = true;
          }
        }
      }
      if (done) break;
      b = (b + 1) & T.mask;
    }
  }
}

template <int W>
struct Key {
  uint64_t w[W];
};

// Bucket scan outcome without touching keys: bit k of `tag_hits` = entry k
// matches the tag (entries after the first empty slot excluded); `full` =
// no empty slot, so the key may continue in the next bucket.
__device__ __forceinline__ void bucket_test(ulonglong2 b0, ulonglong2 b1, uint32_t tag, unsigned& tag_hits,
                                            bool& full) {
  const uint64_t e[4] = {b0.x, b0.y, b1.x, b1.y};
  unsigned empt = 0, tm = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    empt |= (e[k] == kEmpty ? 1u : 0u) << k;
    tm |= (static_cast<uint32_t>(e[k] >> 32) == tag ? 1u : 0u) << k;
  }
  const unsigned first_empty = empt ? __ffs(empt) - 1 : 4;
  tag_hits = tm & ((1u << first_empty) - 1u);
  full = empt == 0;
}

// Slow path of a probe (tag match or full bucket): verify candidates
// against the stored keys and follow the bucket chain. Returns the row of
// x ^ xy[g] or -1.
template <int W>
__device__ __noinline__ int64_t probe_slow(Key<W> x, uint64_t f, uint32_t g, const uint64_t* __restrict__ tab,
                                           uint64_t mask, const uint64_t* __restrict__ keys,
                                           const uint64_t* __restrict__ xym) {
  const uint32_t tag = static_cast<uint32_t>(f >> 32);
  uint64_t want[W];
#pragma unroll
  for (int w = 0; w < W; ++w) want[w] = x.w[w] ^ __ldg(xym + (int64_t)g * W + w);
  uint64_t b = f & mask;
  for (;;) {
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(tab + b * 4);
    unsigned tm;
    bool full;
    bucket_test(__ldg(p), __ldg(p + 1), tag, tm, full);
    while (tm) {
      const int k = __ffs(tm) - 1;
      tm &= tm - 1;
      const uint32_t j = static_cast<uint32_t>(__ldg(tab + b * 4 + k));
      bool same = true;
#pragma unroll
      for (int w = 0; w < W; ++w) same &= __ldg(keys + (int64_t)j * W + w) == want[w];
      if (same) return j;
    }
    if (!full) return -1;
    b = (b + 1) & mask;
  }
}

// group_element (hamiltonian.cpp:186-194) term by term in the reference
// order; adding c*i^q as +-c to one component is bit-identical to the
// reference's complex multiply-add because c*{0,+-1} is exact.
template <int W>
__device__ __forceinline__ void group_element(const HamView& H, const uint64_t* xp, uint32_t g, double& re,
                                              double& im) {
  re = 0.0;
  im = 0.0;
  const uint32_t t1 = __ldg(H.goff + g + 1);
  for (uint32_t t = __ldg(H.goff + g); t < t1; ++t) {
    int pc = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) pc += __popcll(xp[w] & __ldg(H.yz + (int64_t)t * W + w));
    const int q = (__ldg(H.yw + t) + 2 * pc) & 3;
    const double c = __ldg(H.coeff + t);
    if (q == 0) re += c;
    else if (q == 2) re -= c;
    else if (q == 1) im += c;
    else im -= c;
  }
}

// ------------------------------------------------------------ row kernel

struct RowOut {
  double2* eloc;              // kModeEloc: [row - row_begin]
  uint32_t* counts;           // kModeCount: [row]
  const uint64_t* row_off;    // kModeEmit: [row]
  uint32_t* xp_out;           // kModeEmit
  uint32_t* g_out;            // kModeEmit
  const double* la;           // log amplitudes
  const double* ph;           // phases
  const double2* cs;          // (cos, sin) of the phases
  // kModeHits (join path, split evaluation): hit chunks for k_eval_chunks
  uint32_t* hy;               // [hit_cap] partner (key-array position)
  uint32_t* hg;               // [hit_cap] group
  uint32_t* hk;               // [hit_cap] flip position key
  uint4* chunk;               // [chunk_cap] (row position, first hit, hits, previous chunk of the row or ~0)
  uint32_t* row_last;         // [row - out_base] last chunk of the row or ~0
  double2* base;              // [row - out_base] diagonal + residual part of E_loc
  unsigned long long* hit_cursor;
  unsigned long long* chunk_cursor;
  uint64_t hit_cap;
  uint64_t chunk_cap;
  uint8_t* rowpos;            // [key position][16] the row's minority orbitals (for the chunk evaluation)
  const int* exp_flag;        // kModeFused: some |log psi| > 700 (amplitude ratios through exp)
};

__global__ void k_cos_sin(const double* __restrict__ ph, int64_t n, double2* cs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s, c;
    sincos(ph[i], &s, &c);
    cs[i] = make_double2(c, s);
  }
}

// sector mode enumerates, per row, one list per minority orbital (single
// flips) and one per pair of minority orbitals (double flips)
constexpr int kMaxMinorityDev = 24;
constexpr int kMaxRanges = kMaxMinorityDev + kMaxMinorityDev * (kMaxMinorityDev - 1) / 2;

// Per-warp hit queue (kModeEloc). Probing only records (x', group); the FP64
// work (matrix element, exp, sincos) runs when the queue is drained, so the
// probe loop stays small in registers and all lanes share the FP64 work:
// small groups one hit per lane, large groups (the 2+2(N-2)-term single
// excitations, 234 terms at 118 qubits) cooperatively over the warp.
constexpr int kQueue = 256;
constexpr int kDrainAt = kQueue - 32 * kUnroll;  // one scan step adds at most 32*kUnroll hits
constexpr uint32_t kSmallGroup = 16;

struct WarpSmem {
  uint32_t qj[kQueue];
  uint32_t qg[kQueue];
  uint32_t r_lo[kMaxRanges];   // candidate-list ranges of the current row
  uint32_t r_len[kMaxRanges];
  uint16_t pos[32];            // minority orbitals of the current row
  unsigned qn;
  unsigned cursor;             // kModeEmit output cursor
};

// h * psi(x')/psi(x) = h * exp(la_j - la_i) * (cos, sin)(ph_j - ph_i), the
// angle difference expanded from per-sample (cos, sin) (energy.cpp:38-43)
__device__ __forceinline__ void add_ratio(double la_j, double2 cs_j, double la_i, double2 cs_i, double hr, double hi,
                                          double2& acc) {
  const double a = exp(la_j - la_i);
  const double c = cs_j.x * cs_i.x + cs_j.y * cs_i.y;
  const double s = cs_j.y * cs_i.x - cs_j.x * cs_i.y;
  hr *= a;
  hi *= a;
  acc.x += hr * c - hi * s;
  acc.y += hr * s + hi * c;
}

// the same with the magnitude |psi(x')/psi(x)| given
__device__ __forceinline__ void add_ratio_mag(double a, double2 cs_j, double2 cs_i, double hr, double hi,
                                              double2& acc) {
  const double c = cs_j.x * cs_i.x + cs_j.y * cs_i.y;
  const double s = cs_j.y * cs_i.x - cs_j.x * cs_i.y;
  hr *= a;
  hi *= a;
  acc.x += hr * c - hi * s;
  acc.y += hr * s + hi * c;
}

// H_{xx'} of a compressed group (sector mode): per family f,
//   i^q_f (-1)^{|x' & B_f|} (u_f + sum_k v_f[k] (-1)^{x'_k}),
// with sum_k v_f[k] (-1)^{x'_k} = +-(V_f - 2 sum_{k in S(x')} v_f[k]) over the
// minority set S(x') = S(x) ^ (x ^ x'): s + |m| loads instead of the terms.
template <int W>
__device__ __forceinline__ void comp_element(const HamView& H, const uint64_t* x, const uint64_t* xp, uint4 gi,
                                             const uint16_t* pos, int s, int side, double& re, double& im) {
  constexpr int FW = fam_words_dev(W);
  re = 0.0;
  im = 0.0;
  const int n = H.n;
  uint64_t m[W];
#pragma unroll
  for (int w = 0; w < W; ++w) m[w] = x[w] ^ xp[w];
  const uint32_t nf = gi.w & 0xFFu;
  for (uint32_t k = 0; k < nf; ++k) {
    const uint32_t f = gi.z + k;
    const ulonglong2* fr = reinterpret_cast<const ulonglong2*>(H.famrec + static_cast<int64_t>(f) * FW);
    uint64_t r[FW];
#pragma unroll
    for (int w = 0; w < FW; w += 2) {
      const ulonglong2 v = __ldg(fr + w / 2);
      r[w] = v.x;
      r[w + 1] = v.y;
    }
    const double* v = H.fam_v + static_cast<int64_t>(f) * n;
    double sv = 0.0;
    for (int a = 0; a < s; ++a) sv += __ldg(v + pos[a]);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      uint64_t bits = m[w];
      while (bits) {
        const int b = 64 * w + __ffsll(static_cast<long long>(bits)) - 1;
        bits &= bits - 1;
        const bool in_s = ((x[w] >> (b & 63)) & 1ull) == static_cast<uint64_t>(side);
        sv += in_s ? -__ldg(v + b) : __ldg(v + b);
      }
    }
    const double V = __longlong_as_double(static_cast<long long>(r[1]));
    double val = __longlong_as_double(static_cast<long long>(r[0])) + (side ? V - 2.0 * sv : 2.0 * sv - V);
    int pc = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) pc += __popcll(xp[w] & r[2 + w]);
    if (pc & 1) val = -val;
    const uint32_t q = (gi.w >> (8 + 2 * k)) & 3u;
    if (q == 0) re += val;
    else if (q == 1) im += val;
    else if (q == 2) re -= val;
    else im -= val;
  }
}

// group_element from the packed term records (same terms, same order, same
// exact +-c adds as group_element: bit-identical)
template <int W>
__device__ __forceinline__ void small_element(const HamView& H, const uint64_t* xp, uint4 gi, double& re, double& im) {
  constexpr int TW = term_words_dev(W);
  re = 0.0;
  im = 0.0;
  const ulonglong2* tr = reinterpret_cast<const ulonglong2*>(H.trec + static_cast<int64_t>(gi.x) * TW);
  for (uint32_t t = 0; t < gi.y; ++t) {
    uint64_t r[TW];
#pragma unroll
    for (int w = 0; w < TW; w += 2) {
      const ulonglong2 v = __ldg(tr + (static_cast<int64_t>(t) * TW + w) / 2);
      r[w] = v.x;
      r[w + 1] = v.y;
    }
    int pc = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) pc += __popcll(xp[w] & r[w]);
    const int q = (static_cast<int>(r[W + 1]) + 2 * pc) & 3;
    const double c = __longlong_as_double(static_cast<long long>(r[W]));
    if (q == 0) re += c;
    else if (q == 2) re -= c;
    else if (q == 1) im += c;
    else im -= c;
  }
}

// Drain the warp's hit queue: returns this lane's share of sum H_{xx'} psi(x')/psi(x).
// s > 0: sector mode with the row's minority orbitals in sm->pos (enables
// compressed groups); s == 0: every group term by term.
#ifdef QVMC_DRAIN_INLINE
#define QVMC_DRAIN_ATTR __forceinline__
#else
#define QVMC_DRAIN_ATTR __noinline__
#endif
template <int W>
__device__ QVMC_DRAIN_ATTR double2 drain(const HamView& H, const uint64_t* __restrict__ keys,
                                      const double* __restrict__ la, const double2* __restrict__ cs, double la_i,
                                      double2 cs_i, WarpSmem* sm, int lane, Key<W> xrow, int s, int side) {
  double2 acc = make_double2(0.0, 0.0);
  __syncwarp();
  const unsigned n = sm->qn;
  for (unsigned k0 = 0; k0 < n; k0 += 32) {
    const unsigned k = k0 + lane;
    const bool valid = k < n;
    uint32_t j = 0;
    uint4 gi = make_uint4(0, 0, 0xFFFFFFFFu, 0);
    uint64_t xp[W];
    double la_j = 0.0;
    double2 cs_j = make_double2(1.0, 0.0);
    if (valid) {  // independent loads first
      j = sm->qj[k];
      gi = __ldg(H.ginfo + sm->qg[k]);
#pragma unroll
      for (int w = 0; w < W; ++w) xp[w] = __ldg(keys + (int64_t)j * W + w);
      la_j = __ldg(la + j);
      cs_j = __ldg(cs + j);
    }
    const bool comp = gi.z != 0xFFFFFFFFu && s > 0;
    const bool large = valid && gi.y > kSmallGroup && !comp;
    if (valid && !large) {
      double hr, hi;
      if (comp)
        comp_element<W>(H, xrow.w, xp, gi, sm->pos, s, side, hr, hi);
      else
        small_element<W>(H, xp, gi, hr, hi);
      add_ratio(la_j, cs_j, la_i, cs_i, hr, hi, acc);
    }
    // large uncompressed groups: the warp splits the terms; element parked in lane src
    double mine_r = 0.0, mine_i = 0.0;
    unsigned mask = __ballot_sync(0xffffffffu, large);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const uint32_t st0 = __shfl_sync(0xffffffffu, gi.x, src);
      const uint32_t st1 = st0 + __shfl_sync(0xffffffffu, gi.y, src);
      uint64_t sx[W];
#pragma unroll
      for (int w = 0; w < W; ++w) sx[w] = __shfl_sync(0xffffffffu, xp[w], src);
      double re = 0.0, im = 0.0;
      for (uint32_t t = st0 + lane; t < st1; t += 32) {
        int pc = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) pc += __popcll(sx[w] & __ldg(H.yz + (int64_t)t * W + w));
        const int qt = (__ldg(H.yw + t) + 2 * pc) & 3;
        const double c = __ldg(H.coeff + t);
        if (qt == 0) re += c;
        else if (qt == 2) re -= c;
        else if (qt == 1) im += c;
        else im -= c;
      }
      re = warp_sum(re);
      im = warp_sum(im);
      if (lane == src) {
        mine_r = re;
        mine_i = im;
      }
    }
    if (large) add_ratio(la_j, cs_j, la_i, cs_i, mine_r, mine_i, acc);
  }
  __syncwarp();
  if (lane == 0) sm->qn = 0;
  __syncwarp();
  return acc;
}

template <int W, int MODE>
__device__ __forceinline__ void on_hit(const RowOut& O, int64_t row, int64_t j, uint32_t g, WarpSmem* sm) {
  if (MODE == kModeEloc) {
    const unsigned k = atomicAdd(&sm->qn, 1u);  // < kQueue: drained at kDrainAt
    sm->qj[k] = static_cast<uint32_t>(j);
    sm->qg[k] = g;
  } else if (MODE == kModeEmit) {
    const unsigned k = atomicAdd(&sm->cursor, 1u);
    const uint64_t at = O.row_off[row] + k;
    O.xp_out[at] = static_cast<uint32_t>(j);
    O.g_out[at] = g;
  }
}

template <int W, int MODE>
__global__ void __launch_bounds__(kThreads) k_rows(const __grid_constant__ HamView H, const TableView T,
                                                   const uint64_t* __restrict__ keys, int64_t row_begin,
                                                   int64_t row_end, const __grid_constant__ Ctl C,
                                                   const __grid_constant__ RowOut O) {
  __shared__ WarpSmem s_w[kWarps];
  const int lane = threadIdx.x & 31;
  WarpSmem* sm = &s_w[threadIdx.x >> 5];
  const int n = H.n;
  if (lane == 0) sm->qn = 0;
  __syncwarp();

  // sector mode: every key has the same popcount, so x' = x ^ m can be in
  // the sample set only if |m & S(x)| = |m|/2 for the minority set S(x)
  const int pmax = C.popc_mm[0];
  const int pmin = 1024 - C.popc_mm[1];
  const int side = (pmin <= n - pmin) ? 1 : 0;  // 1: occupied orbitals are the minority
  const int s = side ? pmin : n - pmin;
  const bool sector = H.lst_off != nullptr && pmin == pmax && s <= kMaxMinorityDev;

  uint64_t tot_cand = 0, tot_hits = 0;
  for (;;) {
    unsigned long long r = 0;
    if (lane == 0) r = atomicAdd(C.row_next, 1ull);
    r = __shfl_sync(0xffffffffu, r, 0);
    const int64_t row = row_begin + static_cast<int64_t>(r);
    if (row >= row_end) break;
    __syncwarp();  // the previous row's reads of the warp's shared tables are done before they are rewritten

    uint64_t x[W];
#pragma unroll
    for (int w = 0; w < W; ++w) x[w] = __ldg(keys + row * W + w);
    Key<W> xrow;
#pragma unroll
    for (int w = 0; w < W; ++w) xrow.w[w] = x[w];
    double la_i = 0.0;
    double2 cs_i = make_double2(1.0, 0.0);
    if (MODE == kModeEloc) {
      la_i = __ldg(O.la + row);
      cs_i = __ldg(O.cs + row);
      if (isinf(la_i)) {  // energy.cpp:32-33
        if (lane == 0) {
          atomicOr(C.err, kErrZeroAmp);
          O.eloc[row - row_begin] = make_double2(CUDART_NAN, CUDART_NAN);
        }
        continue;
      }
    }
    if (MODE == kModeEmit && lane == 0) sm->cursor = 0;
    const uint64_t hx = key_hash_warp<W>(x, H.hash_bytes, lane);

    // ---- the candidate lists of this row, as (offset, length) ranges
    const uint64_t* hs = H.gen_hash;
    const uint32_t* gs = H.gen_g;
    int n_ranges = 1;
    int pos = 0;
    uint64_t S[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      S[w] = side ? x[w] : ~x[w];
      const int hi_bit = n - 64 * w;
      if (hi_bit < 64) S[w] &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
    }
    if (sector) {
      int c = 0;  // lane a < s holds the a-th minority orbital
#pragma unroll
      for (int w = 0; w < W; ++w) {
        uint64_t v = S[w];
        const int pc = __popcll(v);
        if (lane >= c && lane < c + pc) {
          for (int k = 0; k < lane - c; ++k) v &= v - 1;
          pos = 64 * w + __ffsll(static_cast<long long>(v)) - 1;
        }
        c += pc;
      }
      if (lane < s) sm->pos[lane] = static_cast<uint16_t>(pos);
      __syncwarp();
      hs = H.lst_hash;
      gs = H.lst_g;
      n_ranges = s + s * (s - 1) / 2;
      // range k < s: single-flip list of orbital pos[k]; then pairs (a < b), pi = b(b-1)/2 + a
      for (int k = lane; k < n_ranges; k += 32) {
        int id;
        if (k < s) {
          id = sm->pos[k];
        } else {
          const int pi = k - s;
          int b = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * pi)) * 0.5f);
          while (b * (b - 1) / 2 > pi) --b;
          while ((b + 1) * b / 2 <= pi) ++b;
          const int pa = sm->pos[pi - b * (b - 1) / 2], pb = sm->pos[b];
          id = n + pa * n - pa * (pa + 1) / 2 + (pb - pa - 1);
        }
        const uint32_t lo = __ldg(H.lst_off + id);
        sm->r_lo[k] = lo;
        sm->r_len[k] = __ldg(H.lst_off + id + 1) - lo;
      }
    } else if (lane == 0) {
      sm->r_lo[0] = 0;
      sm->r_len[0] = H.n_gen;
    }
    __syncwarp();

    // ---- walk the concatenated ranges: lane l takes elements l, l+32, ...;
    // its cursor (rg, off) advances by 32 per probe
    double2 acc = make_double2(0.0, 0.0);
    uint32_t hits = 0;
    uint64_t cand = 0;
    int rg = 0;
    uint32_t off = lane;
    uint32_t len = sm->r_len[0];
    while (rg < n_ranges && off >= len) {
      off -= len;
      if (++rg < n_ranges) len = sm->r_len[rg];
    }
    while (__any_sync(0xffffffffu, rg < n_ranges)) {
      uint64_t f[kUnroll];
      uint32_t g[kUnroll];
      ulonglong2 b0[kUnroll], b1[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        g[u] = 0xffffffffu;
        f[u] = 0;
        if (rg < n_ranges) {
          const uint32_t e = sm->r_lo[rg] + off;
          g[u] = __ldg(gs + e);
          f[u] = fmix(hx ^ __ldg(hs + e));
          const ulonglong2* p = reinterpret_cast<const ulonglong2*>(T.tab + (f[u] & T.mask) * 4);
          b0[u] = __ldg(p);
          b1[u] = __ldg(p + 1);
          off += 32;
          while (rg < n_ranges && off >= len) {
            off -= len;
            if (++rg < n_ranges) len = sm->r_len[rg];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        if (g[u] != 0xffffffffu) {
          ++cand;
          unsigned tm;
          bool full;
          bucket_test(b0[u], b1[u], static_cast<uint32_t>(f[u] >> 32), tm, full);
          if (tm || full) {
            Key<W> xk;
#pragma unroll
            for (int w = 0; w < W; ++w) xk.w[w] = x[w];
            const int64_t j = probe_slow<W>(xk, f[u], g[u], T.tab, T.mask, keys, H.xy);
            if (j >= 0) {
              on_hit<W, MODE>(O, row, j, g[u], sm);
              ++hits;
            }
          }
        }
      }
      if (MODE == kModeEloc) {
        __syncwarp();
        if (sm->qn >= kDrainAt) {
          const double2 d = drain<W>(H, keys, O.la, O.cs, la_i, cs_i, sm, lane, xrow, sector ? s : 0, side);
          acc.x += d.x;
          acc.y += d.y;
        }
      }
    }

    // ---- even flip masks of weight >= 6 (none for two-body Hamiltonians)
    if (sector) {
      for (uint32_t base = 0; base < H.n_res; base += 32) {
        const uint32_t e = base + lane;
        if (e < H.n_res) {
          const uint32_t g = __ldg(H.res_g + e);
          int in_s = 0, wt = 0;
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const uint64_t m = __ldg(H.xy + (int64_t)g * W + w);
            in_s += __popcll(m & S[w]);
            wt += __popcll(m);
          }
          if (2 * in_s == wt) {
            Key<W> xk;
#pragma unroll
            for (int w = 0; w < W; ++w) xk.w[w] = x[w];
            ++cand;
            const int64_t j = probe_slow<W>(xk, fmix(hx ^ __ldg(H.xy_hash + g)), g, T.tab, T.mask, keys, H.xy);
            if (j >= 0) {
              on_hit<W, MODE>(O, row, j, g, sm);
              ++hits;
            }
          }
        }
        if (MODE == kModeEloc) {
          __syncwarp();
          if (sm->qn >= kDrainAt) {
            const double2 d = drain<W>(H, keys, O.la, O.cs, la_i, cs_i, sm, lane, xrow, sector ? s : 0, side);
            acc.x += d.x;
            acc.y += d.y;
          }
        }
      }
    }

    // ---- diagonal element (x' = x, ratio exactly 1), split over lanes
    if (MODE == kModeEloc && H.diag >= 0) {
      if (sector && H.diag_quad) {
        if (lane == 0) acc.x += side ? H.diag_A1 : H.diag_A0;
        if (lane < s) acc.x += __ldg(H.diag_b + side * n + pos);
        const int np = s * (s - 1) / 2;
        for (int pi = lane; pi < np; pi += 32) {
          int b = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * pi)) * 0.5f);
          while (b * (b - 1) / 2 > pi) --b;
          while ((b + 1) * b / 2 <= pi) ++b;
          acc.x += __ldg(H.diag_K + sm->pos[pi - b * (b - 1) / 2] * n + sm->pos[b]);
        }
        for (uint32_t e = lane; e < H.n_diag_other; e += 32) {
          const uint32_t t = __ldg(H.diag_other + e);
          int pc = 0;
#pragma unroll
          for (int w = 0; w < W; ++w) pc += __popcll(x[w] & __ldg(H.yz + (int64_t)t * W + w));
          const int qt = (__ldg(H.yw + t) + 2 * pc) & 3;
          const double cf = __ldg(H.coeff + t);
          if (qt == 0) acc.x += cf;
          else if (qt == 2) acc.x -= cf;
          else if (qt == 1) acc.y += cf;
          else acc.y -= cf;
        }
      } else {
        const uint32_t t1 = __ldg(H.goff + H.diag + 1);
        for (uint32_t t = __ldg(H.goff + H.diag) + lane; t < t1; t += 32) {
          int pc = 0;
#pragma unroll
          for (int w = 0; w < W; ++w) pc += __popcll(x[w] & __ldg(H.yz + (int64_t)t * W + w));
          const int qt = (__ldg(H.yw + t) + 2 * pc) & 3;
          const double cf = __ldg(H.coeff + t);
          if (qt == 0) acc.x += cf;
          else if (qt == 2) acc.x -= cf;
          else if (qt == 1) acc.y += cf;
          else acc.y -= cf;
        }
      }
    }

    if (MODE == kModeEloc) {
      __syncwarp();
      if (sm->qn > 0) {
        const double2 d = drain<W>(H, keys, O.la, O.cs, la_i, cs_i, sm, lane, xrow, sector ? s : 0, side);
        acc.x += d.x;
        acc.y += d.y;
      }
      const double re = warp_sum(acc.x);
      const double im = warp_sum(acc.y);
      if (lane == 0) O.eloc[row - row_begin] = make_double2(re, im);
    }
    const uint32_t row_hits = warp_sum(hits) + (H.diag >= 0 ? 1u : 0u);
    if (MODE == kModeCount && lane == 0) O.counts[row] = row_hits;
    if (MODE == kModeEmit) {
      __syncwarp();
      if (lane == 0 && H.diag >= 0) {
        const uint64_t at = O.row_off[row] + sm->cursor;
        O.xp_out[at] = static_cast<uint32_t>(row);
        O.g_out[at] = static_cast<uint32_t>(H.diag);
      }
      __syncwarp();
    }
    tot_cand += cand;
    tot_hits += row_hits;  // warp total, identical on every lane
  }
  tot_cand = warp_sum(tot_cand);
  if (lane == 0) {
    atomicAdd(C.stats, static_cast<unsigned long long>(tot_cand));
    atomicAdd(C.stats + 1, static_cast<unsigned long long>(tot_hits));
  }
}

}  // namespace qvmc_b200
