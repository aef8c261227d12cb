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

enum : int { kErrDuplicate = 1, kErrZeroAmp = 2, kErrBadPair = 4 };
enum : int { kModeEloc = 0, kModeCount = 1, kModeEmit = 2 };

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
};

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

// Find the row whose key is x ^ xy[g], given f = fmix(hash(x ^ xy[g])).
// b0/b1 are the first bucket's two 16-byte halves, already loaded.
template <int W>
__device__ __forceinline__ int64_t resolve(const TableView& T, const uint64_t* __restrict__ keys,
                                           const uint64_t* __restrict__ xym, const uint64_t* x, uint64_t f,
                                           uint32_t g, ulonglong2 b0, ulonglong2 b1, uint64_t* xp) {
  const uint32_t tag = static_cast<uint32_t>(f >> 32);
  uint64_t b = f & T.mask;
  for (;;) {
    const uint64_t e[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (e[k] == kEmpty) return -1;
      if (static_cast<uint32_t>(e[k] >> 32) == tag) {
        const uint32_t j = static_cast<uint32_t>(e[k]);
        bool same = true;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          xp[w] = __ldg(keys + (int64_t)j * W + w);
          same &= xp[w] == (x[w] ^ __ldg(xym + (int64_t)g * W + w));
        }
        if (same) return j;
      }
    }
    b = (b + 1) & T.mask;  // bucket full: continue (rare at load <= 1/4)
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(T.tab + b * 4);
    b0 = __ldg(p);
    b1 = __ldg(p + 1);
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
};

template <int W, int MODE>
struct RowState {
  uint64_t x[W];
  uint64_t hx;
  double la_i, ph_i;
  double acc_re, acc_im;
  uint32_t hits;
  uint64_t cand;
  int64_t row;
};

template <int W, int MODE>
__device__ __forceinline__ void on_hit(const HamView& H, const RowOut& O, RowState<W, MODE>& st, int64_t j,
                                       const uint64_t* xp, uint32_t g, unsigned* s_cursor) {
  if (MODE == kModeEloc) {
    double hr, hi;
    group_element<W>(H, xp, g, hr, hi);
    const double a = exp(__ldg(O.la + j) - st.la_i);
    double s, c;
    sincos(__ldg(O.ph + j) - st.ph_i, &s, &c);
    hr *= a;
    hi *= a;
    st.acc_re += hr * c - hi * s;
    st.acc_im += hr * s + hi * c;
  } else if (MODE == kModeEmit) {
    const unsigned k = atomicAdd(s_cursor, 1u);
    const uint64_t at = O.row_off[st.row] + k;
    O.xp_out[at] = static_cast<uint32_t>(j);
    O.g_out[at] = g;
  }
  ++st.hits;
}

// Probe every mask of list entries [lo, hi) (hash + group id arrays).
template <int W, int MODE>
__device__ __forceinline__ void scan_list(const HamView& H, const TableView& T, const uint64_t* __restrict__ keys,
                                          const RowOut& O, RowState<W, MODE>& st, const uint64_t* __restrict__ hs,
                                          const uint32_t* __restrict__ gs, uint32_t lo, uint32_t hi, int lane,
                                          unsigned* s_cursor) {
  for (uint32_t base = lo; base < hi; base += 32 * kUnroll) {
    uint64_t f[kUnroll];
    uint32_t g[kUnroll];
    ulonglong2 b0[kUnroll], b1[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t e = base + u * 32 + lane;
      g[u] = 0xffffffffu;
      f[u] = 0;
      if (e < hi) {
        g[u] = __ldg(gs + e);
        f[u] = fmix(st.hx ^ __ldg(hs + e));
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (g[u] != 0xffffffffu) {
        const ulonglong2* p = reinterpret_cast<const ulonglong2*>(T.tab + (f[u] & T.mask) * 4);
        b0[u] = __ldg(p);
        b1[u] = __ldg(p + 1);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (g[u] != 0xffffffffu) {
        ++st.cand;
        uint64_t xp[W];
        const int64_t j = resolve<W>(T, keys, H.xy, st.x, f[u], g[u], b0[u], b1[u], xp);
        if (j >= 0) on_hit<W, MODE>(H, O, st, j, xp, g[u], s_cursor);
      }
    }
  }
}

template <int W, int MODE>
__global__ void __launch_bounds__(kThreads) k_rows(HamView H, TableView T, const uint64_t* __restrict__ keys,
                                                   int64_t row_begin, int64_t row_end, Ctl C, RowOut O) {
  __shared__ uint16_t s_pos[kWarps][32];
  __shared__ unsigned s_cursor[kWarps];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int n = H.n;

  // sector mode: every key has the same popcount, so x' = x ^ m can be in
  // the sample set only if |m & S(x)| = |m|/2 for the minority set S(x)
  const int pmax = C.popc_mm[0];
  const int pmin = 1024 - C.popc_mm[1];
  const int side = (pmin <= n - pmin) ? 1 : 0;  // 1: occupied orbitals are the minority
  const int s = side ? pmin : n - pmin;
  const bool sector = H.lst_off != nullptr && pmin == pmax && s <= 32;

  uint64_t tot_cand = 0, tot_hits = 0;
  for (;;) {
    unsigned long long r = 0;
    if (lane == 0) r = atomicAdd(C.row_next, 1ull);
    r = __shfl_sync(0xffffffffu, r, 0);
    const int64_t row = row_begin + static_cast<int64_t>(r);
    if (row >= row_end) break;

    RowState<W, MODE> st;
    st.row = row;
    st.acc_re = st.acc_im = 0.0;
    st.hits = 0;
    st.cand = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) st.x[w] = __ldg(keys + row * W + w);
    if (MODE == kModeEloc) {
      st.la_i = __ldg(O.la + row);
      st.ph_i = __ldg(O.ph + row);
      if (isinf(st.la_i)) {  // energy.cpp:32-33
        if (lane == 0) {
          atomicOr(C.err, kErrZeroAmp);
          O.eloc[row - row_begin] = make_double2(CUDART_NAN, CUDART_NAN);
        }
        continue;
      }
    }
    if (MODE == kModeEmit && lane == 0) s_cursor[wid] = 0;
    st.hx = key_hash_warp<W>(st.x, H.hash_bytes, lane);
    __syncwarp();

    double d_re = 0.0, d_im = 0.0;  // diagonal element, split over lanes
    if (sector) {
      uint64_t S[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        S[w] = side ? st.x[w] : ~st.x[w];
        const int hi_bit = n - 64 * w;
        if (hi_bit < 64) S[w] &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
      }
      // lane a < s holds the a-th minority orbital
      int pos = 0, c = 0;
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
      if (lane < s) s_pos[wid][lane] = static_cast<uint16_t>(pos);
      __syncwarp();
      // single flips: weight-2 masks through one minority orbital
      for (int a = 0; a < s; ++a) {
        const int id = s_pos[wid][a];
        scan_list<W, MODE>(H, T, keys, O, st, H.lst_hash, H.lst_g, __ldg(H.lst_off + id), __ldg(H.lst_off + id + 1),
                           lane, &s_cursor[wid]);
      }
      // double flips: weight-4 masks through two minority orbitals
      for (int b = 1; b < s; ++b) {
        const int pb = s_pos[wid][b];
        for (int a = 0; a < b; ++a) {
          const int pa = s_pos[wid][a];
          const int id = n + pa * n - pa * (pa + 1) / 2 + (pb - pa - 1);
          scan_list<W, MODE>(H, T, keys, O, st, H.lst_hash, H.lst_g, __ldg(H.lst_off + id),
                             __ldg(H.lst_off + id + 1), lane, &s_cursor[wid]);
        }
      }
      // even weight >= 6: filter by the popcount condition, then probe
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
            const uint64_t f = fmix(st.hx ^ __ldg(H.xy_hash + g));
            const ulonglong2* p = reinterpret_cast<const ulonglong2*>(T.tab + (f & T.mask) * 4);
            uint64_t xp[W];
            ++st.cand;
            const int64_t j = resolve<W>(T, keys, H.xy, st.x, f, g, __ldg(p), __ldg(p + 1), xp);
            if (j >= 0) on_hit<W, MODE>(H, O, st, j, xp, g, &s_cursor[wid]);
          }
        }
      }
      if (MODE == kModeEloc && H.diag >= 0 && H.diag_quad) {
        if (lane == 0) d_re += side ? H.diag_A1 : H.diag_A0;
        if (lane < s) d_re += __ldg(H.diag_b + side * n + pos);
        const int np = s * (s - 1) / 2;
        for (int pi = lane; pi < np; pi += 32) {
          // pairs ordered by b then a: pi = b(b-1)/2 + a
          int b = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * pi)) * 0.5f);
          while (b * (b - 1) / 2 > pi) --b;
          while ((b + 1) * b / 2 <= pi) ++b;
          const int a = pi - b * (b - 1) / 2;
          d_re += __ldg(H.diag_K + s_pos[wid][a] * n + s_pos[wid][b]);
        }
        for (uint32_t e = lane; e < H.n_diag_other; e += 32) {
          const uint32_t t = __ldg(H.diag_other + e);
          int pc = 0;
#pragma unroll
          for (int w = 0; w < W; ++w) pc += __popcll(st.x[w] & __ldg(H.yz + (int64_t)t * W + w));
          const int q = (__ldg(H.yw + t) + 2 * pc) & 3;
          const double cf = __ldg(H.coeff + t);
          if (q == 0) d_re += cf;
          else if (q == 2) d_re -= cf;
          else if (q == 1) d_im += cf;
          else d_im -= cf;
        }
      }
    } else {
      scan_list<W, MODE>(H, T, keys, O, st, H.gen_hash, H.gen_g, 0, H.n_gen, lane, &s_cursor[wid]);
    }
    if (MODE == kModeEloc && H.diag >= 0 && !(sector && H.diag_quad)) {
      const uint32_t t1 = __ldg(H.goff + H.diag + 1);
      for (uint32_t t = __ldg(H.goff + H.diag) + lane; t < t1; t += 32) {
        int pc = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) pc += __popcll(st.x[w] & __ldg(H.yz + (int64_t)t * W + w));
        const int q = (__ldg(H.yw + t) + 2 * pc) & 3;
        const double cf = __ldg(H.coeff + t);
        if (q == 0) d_re += cf;
        else if (q == 2) d_re -= cf;
        else if (q == 1) d_im += cf;
        else d_im -= cf;
      }
    }

    if (MODE == kModeEloc) {
      const double re = warp_sum(st.acc_re + d_re);
      const double im = warp_sum(st.acc_im + d_im);
      if (lane == 0) O.eloc[row - row_begin] = make_double2(re, im);
    }
    const uint32_t hits = warp_sum(st.hits) + (H.diag >= 0 ? 1u : 0u);
    if (MODE == kModeCount && lane == 0) O.counts[row] = hits;
    if (MODE == kModeEmit) {
      __syncwarp();
      if (lane == 0 && H.diag >= 0) {
        const uint64_t at = O.row_off[row] + s_cursor[wid];
        O.xp_out[at] = static_cast<uint32_t>(row);
        O.g_out[at] = static_cast<uint32_t>(H.diag);
      }
    }
    tot_cand += st.cand;
    tot_hits += hits;  // warp total, identical on every lane
  }
  tot_cand = warp_sum(tot_cand);
  if (lane == 0) {
    atomicAdd(C.stats, static_cast<unsigned long long>(tot_cand));
    atomicAdd(C.stats + 1, static_cast<unsigned long long>(tot_hits));
  }
}

}  // namespace qvmc_b200
