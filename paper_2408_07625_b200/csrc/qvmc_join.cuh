// Join path of the row kernel (sector mode, small minority sets).
//
// For a single-sector sample set with minority sets S(x) of size s, every
// partner x' of x through a weight-2 or weight-4 flip mask shares at least
// s-2 minority orbitals with x. Each sample y is entered into the buckets
// keyed by S(y) - T for every pair T of S(y) ("deletion index", N*s(s-1)/2
// entries, rebuilt per call: key generation + one CUB radix sort). For row x
// and pair T the members of bucket S(x) - T are exactly the samples sharing
// S(x) - T, i.e. the candidates; the pair's flip mask m = x ^ y is then
// looked up in the (static) flip-mask hash table. At 118 qubits this visits
// ~2.1k candidates per row instead of the ~14k masks of the sector lists.
//
// Each coupled pair is accepted exactly once:
//   |m| = 4: m & S(x) == T (holds for exactly one pair T of S(x));
//   |m| = 2: m & S(x) = {c} with c in T, and T's other orbital is the smallest
//            orbital of S(x) other than c (one of the s-1 buckets holding y);
//   anything else (y == x, or a 32-bit bucket-key collision) is skipped.
// Masks of weight >= 6 go through the residual scan of the list path.
#pragma once

#include "qvmc_kernels.cuh"

namespace qvmc_b200 {

#ifndef QVMC_JOIN_MINB
#define QVMC_JOIN_MINB 4  // 64 registers: 32 resident warps per SM (measured best)
#endif

#ifndef QVMC_JOIN_UNROLL
#define QVMC_JOIN_UNROLL 2  // bucket members in flight per lane (2 beat 4 and 8: fewer spills at 64 regs)
#endif

constexpr int kJoinMaxMinority = 16;  // s <= 16: at most 120 buckets per row
constexpr int kJoinMaxRanges = kJoinMaxMinority * (kJoinMaxMinority - 1) / 2;

struct JoinView {
  uint32_t C;                     // buckets per sample = s(s-1)/2
  const uint2* rng;               // [N*C] (lo, hi) bucket range in vals, entry id y*C + t
  const uint32_t* vals;           // sorted entry ids
  const uint64_t* xy_tab;         // flip-mask hash table, buckets of 4 x (tag32 | group)
  uint64_t xy_mask;
  const uint64_t* codes;          // [256] qubit codes of the linear hash
};

__device__ __forceinline__ uint32_t pair_b(int pi) {  // pairs ordered by b then a: pi = b(b-1)/2 + a
  int b = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * pi)) * 0.5f);
  while (b * (b - 1) / 2 > pi) --b;
  while ((b + 1) * b / 2 <= pi) ++b;
  return static_cast<uint32_t>(b);
}

// Per sample: its linear hash and, for every pair T of its minority set, the
// 32-bit bucket key fmix(hash(S(y) - T)) with value y*C + t.
// Rows of one call. Rows are processed in the order of the (locality-sorted)
// key arrays; `perm` maps a key-array position back to the caller's row.
struct RowSet {
  int64_t n_rows;          // rows to process
  int64_t base;            // position = base + r when list is null
  const uint32_t* list;    // else position = list[r]
  const uint32_t* perm;    // position -> caller row (null: identity)
  int64_t out_base;        // outputs are indexed by caller row - out_base
};

// Locality order for the join: samples sorted by their minority orbitals,
// highest first (top 8 packed into 64 bits), so that rows processed together
// and the members of their buckets sit close in memory and in L2.
template <int W>
__global__ void __launch_bounds__(kThreads)
    k_locality_keys(const uint64_t* __restrict__ keys, int64_t n, int n_qubits, int side, uint64_t* __restrict__ skey,
                    uint32_t* __restrict__ sidx) {
  for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y < n; y += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = 0;
    int got = 0;
#pragma unroll
    for (int w = W - 1; w >= 0; --w) {
      uint64_t v = side ? keys[y * W + w] : ~keys[y * W + w];
      const int hi_bit = n_qubits - 64 * w;
      if (hi_bit < 64) v &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
      while (v && got < 8) {
        const int p = 64 * w + 63 - __clzll(static_cast<long long>(v));
        k |= static_cast<uint64_t>(p) << (56 - 8 * got);
        ++got;
        v &= ~(1ull << (p & 63));
      }
    }
    skey[y] = k;
    sidx[y] = static_cast<uint32_t>(y);
  }
}

template <int W>
__global__ void k_gather_sorted(const uint32_t* __restrict__ perm, int64_t n, const uint64_t* __restrict__ keys,
                                const double* __restrict__ la, const double* __restrict__ ph, uint64_t* keys_s,
                                double* la_s, double* ph_s, double2* cs_s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = perm[i];
#pragma unroll
    for (int w = 0; w < W; ++w) keys_s[i * W + w] = keys[(int64_t)o * W + w];
    la_s[i] = la[o];
    const double p = ph[o];
    ph_s[i] = p;
    double sn, c;
    sincos(p, &sn, &c);
    cs_s[i] = make_double2(c, sn);
  }
}

__global__ void k_flag_rows(const uint32_t* __restrict__ perm, int64_t n, int64_t r0, int64_t r1, uint8_t* flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = perm[i] >= r0 && perm[i] < r1;
}

template <int W>
__global__ void __launch_bounds__(kThreads)
    k_join_keys(const uint64_t* __restrict__ keys, int64_t n, int n_qubits, int side, int s,
                const uint64_t* __restrict__ codes, uint32_t* __restrict__ bkey, uint32_t* __restrict__ bval) {
  const uint32_t C = static_cast<uint32_t>(s * (s - 1) / 2);
  for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y < n; y += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x[W];
#pragma unroll
    for (int w = 0; w < W; ++w) x[w] = keys[y * W + w];
    uint8_t pos[kJoinMaxMinority];
    uint64_t hs = 0;
    int k = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      uint64_t v = side ? x[w] : ~x[w];
      const int hi_bit = n_qubits - 64 * w;
      if (hi_bit < 64) v &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
      while (v && k < kJoinMaxMinority) {
        const int p = 64 * w + __ffsll(static_cast<long long>(v)) - 1;
        pos[k++] = static_cast<uint8_t>(p);
        hs ^= __ldg(codes + p);
        v &= v - 1;
      }
    }
    const uint64_t base = static_cast<uint64_t>(y) * C;
    uint32_t t = 0;
    for (int b = 1; b < s; ++b)
      for (int a = 0; a < b; ++a, ++t) {
        const uint64_t hk = hs ^ __ldg(codes + pos[a]) ^ __ldg(codes + pos[b]);
        bkey[base + t] = static_cast<uint32_t>(fmix(hk));
        bval[base + t] = static_cast<uint32_t>(base + t);
      }
  }
}

// Per bucket (run of equal keys in the sorted array): store the range on
// every member entry.
__global__ void k_join_ranges(const uint32_t* __restrict__ run_off, const uint32_t* __restrict__ run_cnt,
                              const int* __restrict__ n_runs, uint32_t* __restrict__ vals, uint32_t C, uint2* rng) {
  const int nr = *n_runs;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x) {
    const uint32_t lo = run_off[r], hi = lo + run_cnt[r];
    for (uint32_t p = lo; p < hi; ++p) {
      const uint32_t e = vals[p];
      rng[e] = make_uint2(lo, hi);
      vals[p] = e / C;  // entry id -> sample
    }
  }
}

// flip-mask table lookup by exact position key (host_index.cpp xy_position_key):
// group of the mask or -1
__device__ __forceinline__ int64_t xy_lookup(uint32_t key, const uint64_t* __restrict__ tab, uint64_t mask) {
  uint64_t b = fmix(key) & mask;
  for (;;) {
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(tab + b * 4);
    const ulonglong2 b0 = __ldg(p), b1 = __ldg(p + 1);
    const uint64_t e[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (e[k] == kEmpty) return -1;
      if (static_cast<uint32_t>(e[k] >> 32) == key) return static_cast<uint32_t>(e[k]);
    }
    b = (b + 1) & mask;  // full bucket: the chain continues
  }
}

constexpr uint32_t kNoKey = 0xFFFFFFFFu;

// resolve a flip-mask lookup given its first bucket (already loaded)
__device__ __forceinline__ int64_t xy_resolve(uint32_t key, uint64_t b, ulonglong2 b0, ulonglong2 b1,
                                              const uint64_t* __restrict__ tab, uint64_t mask) {
  for (;;) {
    const uint64_t e[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (e[k] == kEmpty) return -1;
      if (static_cast<uint32_t>(e[k] >> 32) == key) return static_cast<uint32_t>(e[k]);
    }
    b = (b + 1) & mask;  // full bucket: the chain continues
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(tab + b * 4);
    b0 = __ldg(p);
    b1 = __ldg(p + 1);
  }
}

template <int W>
__device__ __forceinline__ int lowest_bit(const uint64_t* v) {  // v != 0
  int r = 0;
#pragma unroll
  for (int w = W - 1; w >= 0; --w)
    if (v[w]) r = 64 * w + __ffsll(static_cast<long long>(v[w])) - 1;
  return r;
}

template <int W>
__device__ __forceinline__ int highest_bit(const uint64_t* v) {  // v != 0
  int r = 0;
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (v[w]) r = 64 * w + 63 - __clzll(static_cast<long long>(v[w]));
  return r;
}

__device__ __forceinline__ void sort2(int& a, int& b) {
  const int lo = min(a, b), hi = max(a, b);
  a = lo;
  b = hi;
}

template <int W>
__device__ __forceinline__ bool bit_at(const uint64_t* v, int p) {
  uint64_t w = v[0];
#pragma unroll
  for (int k = 1; k < W; ++k)
    if ((p >> 6) == k) w = v[k];
  return (w >> (p & 63)) & 1ull;
}

template <int W, int MODE>
__global__ void __launch_bounds__(kThreads, QVMC_JOIN_MINB) k_rows_join(const __grid_constant__ HamView H, const TableView T,
                                                        const __grid_constant__ JoinView J,
                                                        const uint64_t* __restrict__ keys, const RowSet R,
                                                        int side, int s,
                                                        const __grid_constant__ Ctl C,
                                                        const __grid_constant__ RowOut O) {
  __shared__ WarpSmem s_w[kWarps];
  __shared__ uint16_t s_ta[kWarps][kJoinMaxRanges], s_tb[kWarps][kJoinMaxRanges];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  WarpSmem* sm = &s_w[wid];
  const int n = H.n;
  const int n_ranges = s * (s - 1) / 2;
  if (lane == 0) sm->qn = 0;
  __syncwarp();

  uint64_t tot_cand = 0, tot_hits = 0;
  for (;;) {
    unsigned long long r = 0;
    if (lane == 0) r = atomicAdd(C.row_next, 1ull);
    r = __shfl_sync(0xffffffffu, r, 0);
    if (static_cast<int64_t>(r) >= R.n_rows) break;
    const int64_t row = R.list ? static_cast<int64_t>(__ldg(R.list + r)) : R.base + static_cast<int64_t>(r);
    const int64_t orow = R.perm ? static_cast<int64_t>(__ldg(R.perm + row)) : row;  // caller's row

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
          O.eloc[orow - R.out_base] = make_double2(CUDART_NAN, CUDART_NAN);
        }
        continue;
      }
    }
    if (MODE == kModeEmit && lane == 0) sm->cursor = 0;

    uint64_t S[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      S[w] = side ? x[w] : ~x[w];
      const int hi_bit = n - 64 * w;
      if (hi_bit < 64) S[w] &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
    }
    int pos = 0, c = 0;  // lane a < s holds the a-th minority orbital
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
    const int pos0 = sm->pos[0], pos1 = sm->pos[1];
    // bucket t of this row: pair (a, b) of S(x), range from the index
    for (int t = lane; t < n_ranges; t += 32) {
      const uint32_t b = pair_b(t);
      s_ta[wid][t] = sm->pos[t - b * (b - 1) / 2];
      s_tb[wid][t] = sm->pos[b];
      const uint2 rg = __ldg(J.rng + static_cast<uint64_t>(row) * J.C + t);
      sm->r_lo[t] = rg.x;
      sm->r_len[t] = rg.y - rg.x;
    }
    __syncwarp();

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
      constexpr int U = QVMC_JOIN_UNROLL;
      uint32_t y[U];
      int tr[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        y[u] = 0xffffffffu;
        tr[u] = rg;
        if (rg < n_ranges) {
          y[u] = __ldg(J.vals + sm->r_lo[rg] + off);
          off += 32;
          while (rg < n_ranges && off >= len) {
            off -= len;
            if (++rg < n_ranges) len = sm->r_len[rg];
          }
        }
      }
      uint64_t yk[U][W];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (y[u] != 0xffffffffu) {
#pragma unroll
          for (int w = 0; w < W; ++w) yk[u][w] = __ldg(keys + (int64_t)y[u] * W + w);
        }
      }
      // accept rule (header comment) -> exact position key of the flip mask
      uint32_t key[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        key[u] = kNoKey;
        if (y[u] == 0xffffffffu) continue;
        uint64_t ms[W], o[W];
        int pw = 0, ps = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const uint64_t m = x[w] ^ yk[u][w];
          ms[w] = m & S[w];  // annihilated minority orbitals
          o[w] = m & ~S[w];  // created ones
          pw += __popcll(m);
          ps += __popcll(ms[w]);
        }
        const int ta = s_ta[wid][tr[u]], tb = s_tb[wid][tr[u]];
        if (pw == 4 && ps == 2) {
          bool is_t = true;  // m & S(x) == T
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const uint64_t t = ((ta >> 6) == w ? 1ull << (ta & 63) : 0ull) | ((tb >> 6) == w ? 1ull << (tb & 63) : 0ull);
            is_t &= ms[w] == t;
          }
          if (is_t) {
            int p0 = ta, p1 = tb, p2 = lowest_bit<W>(o), p3 = highest_bit<W>(o);  // merge two sorted pairs
            sort2(p0, p2);
            sort2(p1, p3);
            sort2(p1, p2);
            key[u] = static_cast<uint32_t>(p0) | static_cast<uint32_t>(p1) << 8 | static_cast<uint32_t>(p2) << 16 |
                     static_cast<uint32_t>(p3) << 24;
          }
        } else if (pw == 2 && ps == 1) {
          const int cpos = lowest_bit<W>(ms), apos = lowest_bit<W>(o);
          const int other = cpos == ta ? tb : (cpos == tb ? ta : -1);
          if (other >= 0 && other == (cpos == pos0 ? pos1 : pos0)) {
            int p0 = cpos, p1 = apos;
            sort2(p0, p1);
            key[u] = static_cast<uint32_t>(p0) | static_cast<uint32_t>(p1) << 8 | 0xFFFF0000u;
          }
        }
      }
      // flip-mask lookups: first buckets of all U in flight, then resolve
      ulonglong2 b0[U], b1[U];
      uint64_t bk[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (key[u] != kNoKey) {
          bk[u] = fmix(key[u]) & J.xy_mask;
          const ulonglong2* p = reinterpret_cast<const ulonglong2*>(J.xy_tab + bk[u] * 4);
          b0[u] = __ldg(p);
          b1[u] = __ldg(p + 1);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int64_t g = -1;
        if (key[u] != kNoKey) {
          ++cand;
          g = xy_resolve(key[u], bk[u], b0[u], b1[u], J.xy_tab, J.xy_mask);
        }
        // warp-aggregated append of the hits
        const bool hit = g >= 0;
        const unsigned hm = __ballot_sync(0xffffffffu, hit);
        if (hm) {
          if (MODE == kModeEloc || MODE == kModeEmit) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(MODE == kModeEloc ? &sm->qn : &sm->cursor, __popc(hm));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (hit) {
              const unsigned k = base + __popc(hm & ((1u << lane) - 1u));
              if (MODE == kModeEloc) {
                sm->qj[k] = y[u];
                sm->qg[k] = static_cast<uint32_t>(g);
              } else {
                const uint64_t at = O.row_off[orow] + k;
                O.xp_out[at] = R.perm ? __ldg(R.perm + y[u]) : y[u];
                O.g_out[at] = static_cast<uint32_t>(g);
              }
            }
          }
          hits += hit ? 1u : 0u;
        }
      }
      if (MODE == kModeEloc) {
        __syncwarp();
        if (sm->qn >= kDrainAt) {
          const double2 d = drain<W>(H, keys, O.la, O.cs, la_i, cs_i, sm, lane, xrow, s, side);
          acc.x += d.x;
          acc.y += d.y;
        }
      }
    }

    // even flip masks of weight >= 6: popcount filter + sample-set probe
    const uint64_t hx_res = H.n_res ? key_hash_warp<W>(x, H.hash_bytes, lane) : 0ull;
    for (uint32_t base = 0; base < H.n_res; base += 32) {
      const uint32_t e = base + lane;
      if (e < H.n_res) {
        const uint32_t g = __ldg(H.res_g + e);
        int in_s = 0, wt = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const uint64_t mm = __ldg(H.xy + (int64_t)g * W + w);
          in_s += __popcll(mm & S[w]);
          wt += __popcll(mm);
        }
        if (2 * in_s == wt) {
          Key<W> xk;
#pragma unroll
          for (int w = 0; w < W; ++w) xk.w[w] = x[w];
          ++cand;
          const int64_t j = probe_slow<W>(xk, fmix(hx_res ^ __ldg(H.xy_hash + g)), g, T.tab, T.mask, keys, H.xy);
          if (j >= 0) {
            on_hit<W, MODE>(O, orow, (MODE == kModeEmit && R.perm) ? static_cast<int64_t>(__ldg(R.perm + j)) : j, g, sm);
            ++hits;
          }
        }
      }
      if (MODE == kModeEloc) {
        __syncwarp();
        if (sm->qn >= kDrainAt) {
          const double2 d = drain<W>(H, keys, O.la, O.cs, la_i, cs_i, sm, lane, xrow, s, side);
          acc.x += d.x;
          acc.y += d.y;
        }
      }
    }

    // diagonal element as the quadratic form over S(x)
    if (MODE == kModeEloc && H.diag >= 0) {
      if (H.diag_quad) {
        if (lane == 0) acc.x += side ? H.diag_A1 : H.diag_A0;
        if (lane < s) acc.x += __ldg(H.diag_b + side * n + pos);
        for (int pi = lane; pi < n_ranges; pi += 32) acc.x += __ldg(H.diag_K + s_ta[wid][pi] * n + s_tb[wid][pi]);
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
        const double2 d = drain<W>(H, keys, O.la, O.cs, la_i, cs_i, sm, lane, xrow, s, side);
        acc.x += d.x;
        acc.y += d.y;
      }
      const double re = warp_sum(acc.x);
      const double im = warp_sum(acc.y);
      if (lane == 0) O.eloc[orow - R.out_base] = make_double2(re, im);
    }
    const uint32_t row_hits = warp_sum(hits) + (H.diag >= 0 ? 1u : 0u);
    if (MODE == kModeCount && lane == 0) O.counts[orow] = row_hits;
    if (MODE == kModeEmit) {
      __syncwarp();
      if (lane == 0 && H.diag >= 0) {
        const uint64_t at = O.row_off[orow] + sm->cursor;
        O.xp_out[at] = static_cast<uint32_t>(orow);
        O.g_out[at] = static_cast<uint32_t>(H.diag);
      }
      __syncwarp();
    }
    tot_cand += cand;
    tot_hits += row_hits;
  }
  tot_cand = warp_sum(tot_cand);
  if (lane == 0) {
    atomicAdd(C.stats, static_cast<unsigned long long>(tot_cand));
    atomicAdd(C.stats + 1, static_cast<unsigned long long>(tot_hits));
  }
}

}  // namespace qvmc_b200
