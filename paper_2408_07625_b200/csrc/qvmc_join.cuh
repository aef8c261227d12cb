// Join path of the row kernel (sector mode, small minority sets).
//
// For a single-sector sample set with minority sets S(x) of size s, every
// partner x' of x through a weight-2 or weight-4 flip mask shares at least
// s-2 minority orbitals with x. Each sample y is entered into the buckets
// keyed by S(y) - T_y for every pair T_y of S(y) ("deletion index", N*s(s-1)/2
// entries, rebuilt per call). The bucket key is the EXACT combinadic rank of
// the (s-2)-subset S(y) - T_y, so a bucket holds exactly the samples sharing
// that subset, and a member entry carries (y, T_y). For row x and its pair
// T_x the members y of bucket S(x) - T_x satisfy
//   S(y) = (S(x) - T_x) + T_y   =>   x ^ y = T_x ^ T_y   (as orbital sets),
// so the flip mask of every candidate is known from the two pairs alone: no
// key of y is ever loaded during the search. The mask is then looked up in
// the (static) flip-mask hash table by its exact position key.
//
// Each coupled pair is accepted exactly once:
//   T_x and T_y disjoint (|m| = 4): the unique bucket T_x = m & S(x);
//   |T_x & T_y| = 1 (|m| = 2, x loses c, gains a): the bucket whose other
//     orbital o is the smallest orbital of S(x) other than c (y sits in the
//     s-1 buckets {c, o} of x);
//   T_x = T_y: y = x, skipped (the diagonal is evaluated separately).
// Masks of weight >= 6 go through the residual scan (sample-set hash probes).
#pragma once

#include <type_traits>

#include "qvmc_kernels.cuh"

namespace qvmc_b200 {

#ifndef QVMC_JOIN_MINB
#define QVMC_JOIN_MINB 4  // 64 registers: 32 resident warps per SM (measured best, r01k)
#endif

#ifndef QVMC_JOIN_UNROLL
#define QVMC_JOIN_UNROLL 4  // bucket members in flight per lane
#endif


constexpr int kJoinMaxMinority = 32;  // s <= 32 (a warp's lanes hold the orbitals): <= 496 buckets per row
constexpr int kJoinMaxRanges = kJoinMaxMinority * (kJoinMaxMinority - 1) / 2;
constexpr int kBinomK = kJoinMaxMinority + 1;  // binomial table C[n][k], k <= 32
constexpr int kFusedMaxMinority = 16;            // kModeFused hands at most 16 minority orbitals per row

// A row's bucket tables (k_rows_join) live in dynamic shared memory, one region
// per search warp sized by the call's bucket count nr = s(s - 1)/2:
// binfo[nr] (uint2), pre[nr + 1] (uint32), tab[nr] (uint16), 16-byte aligned.
__host__ __device__ constexpr uint32_t join_range_bytes(int nr) {
  return (8u * nr + 4u * (nr + 1) + 2u * nr + 15u) & ~15u;
}
constexpr uint32_t kNoKey = 0xFFFFFFFFu;

// Per-group drain record, 8 words (two 32-byte sectors), host_index.cpp:
//   kind A (small group, one shared Z string): w0 = 0 | k << 2 | per term t
//     (ypat_t | (y_weight_t & 3) << 4) << (8 + 6t), ypat_t = Y positions among
//     the sorted flip positions; w1.. = z words, then the k coefficients
//   kind B (family-compressed single excitation, every family base B_f = shared
//     Z string | Y positions among the two flip positions): w0 = 1 | n_fam << 8
//     | q bits << 16 | ypat_f << (24 + 4f), w1 = offset of the group's
//     interleaved v block in famvi ([N][n_fam padded to 1/2/4]), w2.. = z
//     words, then (u_f, V_f) per family
//   kind C (generic): w0 = 2, w1 = t0 | n_terms << 32
//   kind D (family-compressed, general): w0 = 3 | n_fam << 8 | q bits << 16,
//     w1 = first family (famrec / fam_v)
constexpr int kGrecWords = 8;
enum : uint32_t { kGrecA = 0, kGrecB = 1, kGrecC = 2, kGrecD = 3 };

struct JoinView {
  uint32_t C;              // buckets per sample = s(s-1)/2
  const uint2* rng;        // [N*C] (lo, hi) of the bucket of (sample y, pair t) in mem
  const uint64_t* mem;     // bucket members grouped by bucket: y | ta << 32 | tb << 40 | pidx(ta, tb) << 48
  const uint64_t* xy_tab;  // flip-mask hash table, buckets of 4 x (position key32 << 32 | group)
  uint64_t xy_mask;
  const uint64_t* rec;     // [N][4] per sample (log psi, cos phase, sin phase, 0) bits
  const uint64_t* grec;    // [n_xy][8] drain records
  const double* famvi;     // kind-B interleaved family coefficients
  // existence bitmaps of the weight-2/4 flip masks over orbital pairs (n <= 128,
  // else null): bit pidx(c, a) of the first P bits = single {c, a}; bit
  // P + pidx(A) * P + pidx(B) = double A u B (every split into two pairs)
  const uint32_t* pbits;
  uint32_t P;              // n(n-1)/2
  int sym;                 // symmetric index: each row walks only its partners y > x (hits count twice)
};

__device__ __forceinline__ uint32_t pidx(int a, int b) {  // a < b
  return static_cast<uint32_t>(b * (b - 1) / 2 + a);
}

__device__ __forceinline__ bool pbit(const uint32_t* __restrict__ bits, uint32_t i) {
  return (__ldg(bits + (i >> 5)) >> (i & 31)) & 1u;
}

// Rows of one call. Rows are processed in the order of the (locality-sorted)
// key arrays; `perm` maps a key-array position back to the caller's row.
struct RowSet {
  int64_t n_rows;        // rows to process
  int64_t base;          // position = base + r when list is null
  const uint32_t* list;  // else position = list[r]
  const uint32_t* perm;  // position -> caller row (null: identity)
  int64_t out_base;      // outputs are indexed by caller row - out_base
};

struct U64x4 {
  uint64_t a, b, c, d;
};

// one 256-bit load (LDG.E.256 on sm_100a); p must be 32-byte aligned
__device__ __forceinline__ U64x4 ldg256(const uint64_t* p) {
  U64x4 r;
  asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(r.a), "=l"(r.b), "=l"(r.c), "=l"(r.d) : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t pair_b(int pi) {  // pairs ordered by b then a: pi = b(b-1)/2 + a
  int b = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * pi)) * 0.5f);
  while (b * (b - 1) / 2 > pi) --b;
  while ((b + 1) * b / 2 <= pi) ++b;
  return static_cast<uint32_t>(b);
}

// popcount range of the keys (the sector test; the join path needs no sample hash table)
template <int W>
__global__ void __launch_bounds__(kThreads) k_popc_range(const uint64_t* __restrict__ keys, int64_t n, int* popc_mm) {
  int mx = 0, mn = 1024;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int pc = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) pc += __popcll(keys[i * W + w]);
    mx = max(mx, pc);
    mn = min(mn, pc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(popc_mm, mx);
    atomicMax(popc_mm + 1, 1024 - mn);
  }
}

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

// Sorted copies of the keys and the per-sample records (log psi, cos, sin, e^{log psi}).
// Record slot 3 = psi magnitude e^{log psi}: amplitude ratios become one
// multiply by the row's 1/e^{log psi} instead of an exp per pair, unless some
// |log psi| > 700 (then exp_flag is set and the exp path is used).
template <int W>
__global__ void k_gather_keys(const uint32_t* __restrict__ perm, int64_t n, const uint64_t* __restrict__ keys,
                              uint64_t* __restrict__ keys_s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = perm[i];
#pragma unroll
    for (int w = 0; w < W; ++w) keys_s[i * W + w] = keys[(int64_t)o * W + w];
  }
}

// sample records in locality order (log|psi|, cos phi, sin phi, e^log|psi|); gathered after the
// deletion index is built, so a host caller's amplitude upload overlaps the build
__global__ void k_gather_records(const uint32_t* __restrict__ perm, int64_t n, const double* __restrict__ la,
                                 const double* __restrict__ ph, double* __restrict__ rec, int* __restrict__ exp_flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = perm[i];
    double sn, c;
    sincos(ph[o], &sn, &c);
    const double l = la[o];
    if (isfinite(l) && fabs(l) > 700.0) atomicOr(exp_flag, 1);
    reinterpret_cast<double4*>(rec)[i] = make_double4(l, c, sn, exp(l));
  }
}

// per-sample records in the caller's order (pairs-free fused path without the
// locality sort is not used; kept for the row-shard gather)
// strided walk assignment of a sharded call: sorted positions phase, phase + stride, ...
__global__ void k_strided_rows(uint32_t* __restrict__ list, int64_t n_rows, uint32_t phase, uint32_t stride) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows; i += (int64_t)gridDim.x * blockDim.x)
    list[i] = phase + static_cast<uint32_t>(i) * stride;
}

__global__ void k_flag_rows(const uint32_t* __restrict__ perm, int64_t n, int64_t r0, int64_t r1, uint8_t* flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = perm[i] >= r0 && perm[i] < r1;
}

// Deletion-index entries: for sample y and pair t = (a < b) of its minority
// orbitals, key = combinadic rank of S(y) - {pos_a, pos_b} (exact), value =
// y | pos_a << 32 | pos_b << 40 | t << 48. With the remaining orbitals
// r_0 < r_1 < ..., rank = sum_i C(r_i, i + 1); an orbital at index j of S(y)
// has index j (j < a), j - 1 (a < j < b) or j - 2 (j > b) after the removal,
// so the rank is three prefix-sum differences. One warp per sample: lane j
// holds orbital j and the three prefix sums (warp scans); lanes write
// consecutive pairs (coalesced).
template <int W, typename K>
__global__ void __launch_bounds__(kThreads)
    k_join_keys(const uint64_t* __restrict__ keys, int64_t n, int n_qubits, int side, int s,
                const uint64_t* __restrict__ binom, K* __restrict__ bkey, uint32_t* __restrict__ bval) {
  const uint32_t C = static_cast<uint32_t>(s * (s - 1) / 2);
  const int lane = threadIdx.x & 31;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t y = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; y < n; y += n_warps) {
    int pos = 0, cnt = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      uint64_t v = side ? keys[y * W + w] : ~keys[y * W + w];
      const int hi_bit = n_qubits - 64 * w;
      if (hi_bit < 64) v &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
      const int pc = __popcll(v);
      if (lane >= cnt && lane < cnt + pc) {
        for (int k = 0; k < lane - cnt; ++k) v &= v - 1;
        pos = 64 * w + __ffsll(static_cast<long long>(v)) - 1;
      }
      cnt += pc;
    }
    const uint64_t* row = binom + static_cast<int64_t>(pos) * kBinomK;
    const bool in = lane < s;
    const uint64_t c0 = in ? __ldg(row + lane + 1) : 0ull;
    const uint64_t c1 = (in && lane >= 1) ? __ldg(row + lane) : 0ull;
    const uint64_t c2 = (in && lane >= 2) ? __ldg(row + lane - 1) : 0ull;
    uint64_t i0 = c0, i1 = c1, i2 = c2;  // inclusive scans
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t t0 = __shfl_up_sync(0xffffffffu, i0, o), t1 = __shfl_up_sync(0xffffffffu, i1, o),
                     t2 = __shfl_up_sync(0xffffffffu, i2, o);
      if (lane >= o) {
        i0 += t0;
        i1 += t1;
        i2 += t2;
      }
    }
    const uint64_t total2 = __shfl_sync(0xffffffffu, i2, 31);
    const uint64_t e0 = i0 - c0, e1 = i1 - c1;  // exclusive: P0[j], P1[j]
    for (uint32_t base = 0; base < C; base += 32) {
      const uint32_t t = base + lane;
      const bool valid = t < C;
      const int b = valid ? static_cast<int>(pair_b(static_cast<int>(t))) : 1;
      const int a = valid ? static_cast<int>(t) - b * (b - 1) / 2 : 0;
      const uint64_t P0a = __shfl_sync(0xffffffffu, e0, a);
      const uint64_t P1a1 = __shfl_sync(0xffffffffu, i1, a);
      const uint64_t P1b = __shfl_sync(0xffffffffu, e1, b);
      const uint64_t P2b1 = __shfl_sync(0xffffffffu, i2, b);

      if (valid) {
        const uint64_t rank = P0a + (P1b - P1a1) + (total2 - P2b1);
        const uint64_t at = static_cast<uint64_t>(y) * C + t;
        bkey[at] = static_cast<K>(rank);
        bval[at] = static_cast<uint32_t>(at);  // entry id y*C + t (32 bits: sorts as a 4-byte value)
      }
    }
  }
}

template <typename K>
__global__ void k_run_heads(const K* __restrict__ key, uint64_t E, uint32_t* __restrict__ head) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < E; p += (uint64_t)gridDim.x * blockDim.x)
    head[p] = (p == 0 || key[p] != key[p - 1]) ? 1u : 0u;
}

// rid = inclusive scan of the heads (1-based run id of every sorted entry)
__global__ void k_run_bounds(const uint32_t* __restrict__ rid, uint64_t E, uint32_t* __restrict__ lo,
                             uint32_t* __restrict__ hi) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < E; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = rid[p];
    if (p == 0 || rid[p - 1] != r) lo[r - 1] = static_cast<uint32_t>(p);
    if (p + 1 == E || rid[p + 1] != r) hi[r - 1] = static_cast<uint32_t>(p + 1);
  }
}

// member array + per-(sample, pair) bucket range
// k-th (0-based) set bit of a W-word mask
template <int W>
__device__ __forceinline__ int select_bit(const uint64_t* v, int k) {
  int base = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const int pc = __popcll(v[w]);
    if (k < pc) {
      const uint32_t lo = static_cast<uint32_t>(v[w]), hi = static_cast<uint32_t>(v[w] >> 32);
      const int pl = __popc(lo);
      return base + (k < pl ? static_cast<int>(__fns(lo, 0, k + 1)) : 32 + static_cast<int>(__fns(hi, 0, k - pl + 1)));
    }
    k -= pc;
    base += 64;
  }
  return -1;
}

// Member array + per-(sample, pair) bucket range. The sort carried only the
// entry id y*C + t; the pair's orbitals come from y's key.
template <int W>
__global__ void k_join_fill(const uint32_t* __restrict__ val, const uint32_t* __restrict__ rid, uint64_t E, uint32_t C,
                            const uint32_t* __restrict__ lo, const uint32_t* __restrict__ hi,
                            const uint64_t* __restrict__ keys, int n_qubits, int side, uint64_t* __restrict__ mem,
                            uint2* __restrict__ rng, int sym, const uint32_t* __restrict__ count = nullptr,
                            uint32_t off = 0) {
  // distributed build (count != null): this rank's slice of the entries, [count, E) is padding;
  // ranges are global positions (the slice lands at `off` in the all-gathered member array)
  const uint64_t En = count ? (static_cast<uint64_t>(*count) < E ? static_cast<uint64_t>(*count) : E) : E;
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < En; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = val[p];
    const uint32_t r = rid[p] - 1;
    const uint32_t y = e / C, t = e - y * C;
    // symmetric mode: members of an exact bucket are in sample order (stable sort of
    // entry ids), so the partners y' > y of this entry are the run after its own position
    rng[e] = make_uint2(off + (sym ? static_cast<uint32_t>(p) + 1u : lo[r]), off + hi[r]);
    uint64_t S[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      S[w] = side ? __ldg(keys + static_cast<uint64_t>(y) * W + w) : ~__ldg(keys + static_cast<uint64_t>(y) * W + w);
      const int hi_bit = n_qubits - 64 * w;
      if (hi_bit < 64) S[w] &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
    }
    const int b = static_cast<int>(pair_b(static_cast<int>(t))), a = static_cast<int>(t) - b * (b - 1) / 2;
    const uint32_t pa = static_cast<uint32_t>(select_bit<W>(S, a)), pb = static_cast<uint32_t>(select_bit<W>(S, b));
    mem[p] = static_cast<uint64_t>(y) | static_cast<uint64_t>(pa) << 32 | static_cast<uint64_t>(pb) << 40 |
             static_cast<uint64_t>(pb * (pb - 1) / 2 + pa) << 48;
  }
  // the slice's padding travels in the members all-gather: defined bytes (never walked)
  for (uint64_t p = En + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < E; p += (uint64_t)gridDim.x * blockDim.x)
    mem[p] = 0;
}

// distributed index build: the rank that owns an exact bucket (a hash of its key)
template <typename K>
__global__ void k_part_flags(const K* __restrict__ key, uint64_t E, uint32_t world, uint32_t rank,
                             uint8_t* __restrict__ flags) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < E; p += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t h = static_cast<uint64_t>(key[p]) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
    flags[p] = static_cast<uint32_t>((h * 0xBF58476D1CE4E5B9ull) >> 33) % world == rank ? 1 : 0;
  }
}

// pad the selected slice [count, cap) with a key above every real key (sorted last), flag overflow
template <typename K>
__global__ void k_pad_slice(K* __restrict__ key, uint32_t* __restrict__ val, const uint32_t* __restrict__ count,
                            uint64_t cap, K pad, int* __restrict__ err) {
  const uint64_t c = *count;
  if (blockIdx.x == 0 && threadIdx.x == 0 && c > cap) atomicOr(err, kErrSliceOverflow);
  for (uint64_t p = c + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < cap;
       p += (uint64_t)gridDim.x * blockDim.x) {
    key[p] = pad;
    val[p] = 0;
  }
}

// first bucket of a flip-mask position key (host_index.cpp xy_bucket_host): murmur3 fmix32
__device__ __forceinline__ uint32_t xy_bucket(uint32_t key, uint32_t mask) {
  key ^= key >> 16;
  key *= 0x85ebca6bu;
  key ^= key >> 13;
  key *= 0xc2b2ae35u;
  key ^= key >> 16;
  return key & mask;
}

constexpr int64_t kChain = -2;

// one loaded bucket: the group of `key`, -1 (absent: the bucket has a free
// slot before any match) or kChain (full bucket without a match)
__device__ __forceinline__ int64_t xy_resolve(uint32_t key, const U64x4& q) {
  const uint64_t e[4] = {q.a, q.b, q.c, q.d};
  int64_t g = kChain;
#pragma unroll
  for (int k = 3; k >= 0; --k) {  // the first match or free slot in slot order wins
    if (e[k] == kEmpty) g = -1;
    if (static_cast<uint32_t>(e[k] >> 32) == key) g = static_cast<uint32_t>(e[k]);
  }
  return g;
}

// rare path: follow the chain after the full bucket b
__device__ __noinline__ int64_t xy_chain(uint32_t key, uint32_t b, const uint64_t* __restrict__ tab, uint32_t mask) {
  for (;;) {
    b = (b + 1) & mask;
    const int64_t g = xy_resolve(key, ldg256(tab + static_cast<uint64_t>(b) * 4));
    if (g != kChain) return g;
  }
}

__device__ __forceinline__ void sort2(int& a, int& b) {
  const int lo = min(a, b), hi = max(a, b);
  a = lo;
  b = hi;
}

// flip mask of a position key (weight 2: upper half 0xFFFF)
template <int W>
__device__ __forceinline__ void key_mask(uint32_t key, uint64_t* m) {
#pragma unroll
  for (int w = 0; w < W; ++w) m[w] = 0;
  const int np = (key >> 16) == 0xFFFFu ? 2 : 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i < np) {
      const int p = (key >> (8 * i)) & 0xFF;
#pragma unroll
      for (int w = 0; w < W; ++w)
        if ((p >> 6) == w) m[w] |= 1ull << (p & 63);
    }
  }
}

template <int W>
__device__ __forceinline__ bool bit_at(const uint64_t* v, int p) {
  uint64_t w = v[0];
#pragma unroll
  for (int k = 1; k < W; ++k)
    if ((p >> 6) == k) w = v[k];
  return (w >> (p & 63)) & 1ull;
}

// H_{x x'} of a kind-A group: sum_t c_t i^{(y_t + 2|x' & z| + 2|b & ypat_t|) mod 4}
// in term order, b = occupations of x' at the sorted flip positions. Same
// terms, same order, same exact +-c adds as group_element: bit-identical.
// (x' = x ^ m never needs forming: z avoids the flip positions, so
// |x' & z| = |x & z|, and x' at a flip position is the complement of x.)
template <int W>
__device__ __forceinline__ void kind_a_element(const uint64_t* r, const uint64_t* x, uint32_t key, double& re,
                                               double& im) {
  re = 0.0;
  im = 0.0;
  const uint64_t meta = r[0];
  const int k = static_cast<int>((meta >> 2) & 7);
  int pz = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) pz += __popcll(x[w] & r[1 + w]);
  const int np = (key >> 16) == 0xFFFFu ? 2 : 4;
  uint32_t bp = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i < np) bp |= (bit_at<W>(x, (key >> (8 * i)) & 0xFF) ? 0u : 1u) << i;
#pragma unroll
  for (int t = 0; t < kGrecWords - 1 - W; ++t) {
    if (t < k) {
      const uint32_t f = static_cast<uint32_t>(meta >> (8 + 6 * t)) & 63u;
      const int q = (static_cast<int>(f >> 4) + 2 * (pz + __popc(bp & f & 15u))) & 3;
      const double c = __longlong_as_double(static_cast<long long>(r[1 + W + t]));
      if (q == 0) re += c;
      else if (q == 2) re -= c;
      else if (q == 1) im += c;
      else im -= c;
    }
  }
}

// H_{x x'} of a kind-B group (a single excitation x -> x' = x - c + a over the
// minority set): per family f,
//   i^q_f (-1)^{|x' & z| + |b & ypat_f|} (u_f + sum_k v_f[k] (-1)^{x'_k}),
//   sum_k v_f[k] (-1)^{x'_k} = +-(V_f - 2 sum_{k in S(x')} v_f[k]),
// S(x') = S(x) - c + a: s + 2 interleaved loads (all families of an orbital
// in one vector load) instead of the 2 + 2(N-2) terms.
template <int W>
__device__ __forceinline__ void kind_b_element(const double* __restrict__ famvi, const uint64_t* r, const uint64_t* x,
                                               uint32_t key, const uint16_t* pos, int s, int side, double& re,
                                               double& im) {
  re = 0.0;
  im = 0.0;
  const uint64_t meta = r[0];
  const int nf = static_cast<int>(meta >> 8) & 0xFF;
  const double* v = famvi + r[1];
  const int p0 = key & 0xFF, p1 = (key >> 8) & 0xFF;
  const bool p0_in_s = bit_at<W>(x, p0) == (side != 0);
  const int c = p0_in_s ? p0 : p1, a = p0_in_s ? p1 : p0;
  double sv[4] = {0.0, 0.0, 0.0, 0.0};
  if (nf == 2) {
    const double2* v2 = reinterpret_cast<const double2*>(v);
#pragma unroll 4
    for (int i = 0; i < s; ++i) {
      const double2 t = __ldg(v2 + pos[i]);
      sv[0] += t.x;
      sv[1] += t.y;
    }
    const double2 tc = __ldg(v2 + c), ta = __ldg(v2 + a);
    sv[0] += ta.x - tc.x;
    sv[1] += ta.y - tc.y;
  } else {
    const int nfp = nf == 1 ? 1 : 4;
    for (int i = 0; i < s; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < nf) sv[j] += __ldg(v + pos[i] * nfp + j);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < nf) sv[j] += __ldg(v + a * nfp + j) - __ldg(v + c * nfp + j);
  }
  int pz = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) pz += __popcll(x[w] & r[2 + w]);
  const uint32_t bp = (bit_at<W>(x, p0) ? 0u : 1u) | (bit_at<W>(x, p1) ? 0u : 2u);
#pragma unroll
  for (int j = 0; 2 + W + 2 * j + 1 < kGrecWords; ++j) {
    if (j < nf) {
      const double u = __longlong_as_double(static_cast<long long>(r[2 + W + 2 * j]));
      const double V = __longlong_as_double(static_cast<long long>(r[3 + W + 2 * j]));
      double val = u + (side ? V - 2.0 * sv[j] : 2.0 * sv[j] - V);
      const uint32_t yp = static_cast<uint32_t>(meta >> (24 + 4 * j)) & 15u;
      if ((pz + __popc(bp & yp)) & 1) val = -val;
      const uint32_t q = static_cast<uint32_t>(meta >> (16 + 2 * j)) & 3u;
      if (q == 0) re += val;
      else if (q == 1) im += val;
      else if (q == 2) re -= val;
      else im -= val;
    }
  }
}

// Per-warp state of the join kernel.
constexpr int kJQueue = 128;
constexpr int kJDrainAt = kJQueue - 32;  // checked after every lookup batch (<= 32 hits)
#ifndef QVMC_JSURV
#define QVMC_JSURV 256
#endif
constexpr int kJSurv = QVMC_JSURV;  // ring of candidates that passed the accept rule and the bitmap: >= 31 + 32 U
static_assert(kJSurv >= 31 + 32 * QVMC_JOIN_UNROLL, "survivor ring too small for the unroll");

struct JoinSmem {
  uint32_t qy[kJQueue];  // hit queue: partner (sorted position), group, flip position key
  uint32_t qg[kJQueue];
  uint32_t qk[kJQueue];
  // (the row's bucket tables pre / binfo / tab: dynamic shared memory, join_range_bytes)
  uint64_t x[4];                  // the current row: key, log psi, (cos, sin) of its phase; kept here
  double la, cs_c, cs_s;          // (not in registers) across the candidate walk
  uint16_t pos[32];               // minority orbitals of the current row
  uint32_t sy[kJSurv];            // survivor ring: partner, flip position key (looked up 32 at a time)
  uint32_t sk[kJSurv];
  unsigned qn;
  unsigned qs;                    // kModeHits: single excitations, queued from the top (a chunk = doubles, then singles)
  unsigned cursor;                // kModeEmit output cursor
};

// warp-uniform row state, re-read from shared memory (volatile: not forwarded
// from registers, so it is not live across the candidate walk)
template <int W>
__device__ __forceinline__ Key<W> row_key(const JoinSmem* sm) {
  Key<W> k;
#pragma unroll
  for (int w = 0; w < W; ++w) k.w[w] = reinterpret_cast<const volatile uint64_t*>(sm->x)[w];
  return k;
}

// one queued hit: its sample record and drain record (loaded together)
struct JoinHit {
  uint32_t key;
  uint32_t y;  // partner (sorted position)
  bool valid;
  U64x4 sr;  // log psi, cos, sin of the partner
  uint64_t r[kGrecWords];
};

// H_{x x'} of one loaded hit from its drain record (warp-collective: large
// generic groups are split over the lanes). Invalid hits give 0.
template <int W>
__device__ __forceinline__ void hit_element(const HamView& H, const JoinView& J, const uint16_t* pos,
                                            const JoinHit& h, const Key<W>& xrow, int lane, int s, int side,
                                            double& hr, double& hi) {
  const uint32_t kind = static_cast<uint32_t>(h.r[0]) & 3u;
  const uint32_t nt = static_cast<uint32_t>(h.r[1] >> 32);
  const bool large = h.valid && kind == kGrecC && nt > kSmallGroup;
  uint64_t xp[W];  // x' = x ^ m: only the generic kinds C / D form it
#pragma unroll
  for (int w = 0; w < W; ++w) xp[w] = 0;
  if (kind >= kGrecC) {
    uint64_t m[W];
    key_mask<W>(h.key, m);
#pragma unroll
    for (int w = 0; w < W; ++w) xp[w] = xrow.w[w] ^ m[w];
  }
  hr = 0.0;
  hi = 0.0;
  if (h.valid && !large) {
    if (kind == kGrecA) {
      kind_a_element<W>(h.r, xrow.w, h.key, hr, hi);
    } else if (kind == kGrecB) {
      kind_b_element<W>(J.famvi, h.r, xrow.w, h.key, pos, s, side, hr, hi);
    } else if (kind == kGrecD) {
      const uint4 gi = make_uint4(0, 0, static_cast<uint32_t>(h.r[1]), static_cast<uint32_t>(h.r[0] >> 8));
      comp_element<W>(H, xrow.w, xp, gi, pos, s, side, hr, hi);
    } else {
      const uint4 gi = make_uint4(static_cast<uint32_t>(h.r[1]), nt, 0xFFFFFFFFu, 0);
      small_element<W>(H, xp, gi, hr, hi);
    }
  }
  // large generic groups: the warp splits the terms; element parked in lane src
  unsigned mask = __ballot_sync(0xffffffffu, large);
  while (mask) {
    const int src = __ffs(mask) - 1;
    mask &= mask - 1;
    const uint32_t st0 = __shfl_sync(0xffffffffu, static_cast<uint32_t>(h.r[1]), src);
    const uint32_t st1 = st0 + __shfl_sync(0xffffffffu, nt, src);
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
      hr = re;
      hi = im;
    }
  }
}

// H_{x x'} psi(x')/psi(x) of one loaded hit, added to acc (warp-collective)
template <int W>
__device__ __forceinline__ void eval_hit(const HamView& H, const JoinView& J, const uint16_t* pos, const JoinHit& h,
                                         const Key<W>& xrow, double la_i, double2 cs_i, int lane, int s, int side,
                                         double2& acc, double inv_ai = 0.0) {
  double hr, hi;
  hit_element<W>(H, J, pos, h, xrow, lane, s, side, hr, hi);
  if (h.valid) {
    const double2 cs_j = make_double2(__longlong_as_double(static_cast<long long>(h.sr.b)),
                                      __longlong_as_double(static_cast<long long>(h.sr.c)));
    if (inv_ai != 0.0) {  // psi(x')/psi(x) magnitude = e^{la_j} * (1 / e^{la_i})
      add_ratio_mag(__longlong_as_double(static_cast<long long>(h.sr.d)) * inv_ai, cs_j, cs_i, hr, hi, acc);
    } else {
      add_ratio(__longlong_as_double(static_cast<long long>(h.sr.a)), cs_j, la_i, cs_i, hr, hi, acc);
    }
  }
}

// ---------------------------------------------------------------- fused search + evaluation
// kModeFused: one kernel, warp-specialised. kFSearch search warps run the
// join walk of k_rows_join and hand each full queue of hits (a "chunk") to an
// evaluation warp through a ring of kFRing shared-memory slots per search
// warp (no hit arrays in HBM, no capacity to overflow, no host round trip).
// Evaluation warp e serves search warps e*kFPer .. e*kFPer+kFPer-1 and takes
// each search warp's chunks in publish order, so a row's chunks are summed
// in walk order: E_loc = sum of the row's chunk sums in order + the row base
// (diagonal + residual) carried by the row's last chunk — deterministic, and
// independent of which rows other warps process (row-shard invariant).
#ifndef QVMC_FUSED_SEARCH
#define QVMC_FUSED_SEARCH 8
#endif
#ifndef QVMC_FUSED_EVAL
#define QVMC_FUSED_EVAL 4
#endif
#ifndef QVMC_FUSED_RING
#define QVMC_FUSED_RING 3
#endif
#ifndef QVMC_FUSED_MINB
#define QVMC_FUSED_MINB 2
#endif
constexpr int kFSearch = QVMC_FUSED_SEARCH;
constexpr int kFEval = QVMC_FUSED_EVAL;
constexpr int kFPer = kFSearch / kFEval;
constexpr int kFRing = QVMC_FUSED_RING;
constexpr int kFThreads = 32 * (kFSearch + kFEval);
static_assert(kFSearch % kFEval == 0, "every evaluation warp serves the same number of search warps");

struct FusedQ {  // one chunk: hits as the search queue holds them (doubles from the bottom, singles from the top)
  uint32_t y[kJQueue];
  uint32_t g[kJQueue];
  uint32_t k[kJQueue];
};

struct FusedHdr {
  double2 base;    // last chunk of a row: diagonal + residual part of E_loc (NaN: zero amplitude)
  uint32_t row;    // sorted position of the row
  uint32_t out;    // output index (caller row - out_base)
  uint16_t n, nd;  // hits, of which doubles (queue bottom)
  uint8_t last;    // 1: the row's last chunk
  uint8_t pos[16]; // minority orbitals of the row (kind B elements)
  volatile int state;  // 0 free (search warp owns it), 1 ready (evaluation warp owns it)
};

struct FusedSmem {
  FusedQ q[kFSearch][kFRing];
  FusedHdr h[kFSearch][kFRing];
  double2 acc[kFEval][kFPer];   // evaluation warps: running row sums per served search warp
  volatile int done[kFSearch];  // search warp finished all its rows
};

template <int W>
__device__ __forceinline__ void fused_eval_loop(const HamView& H, const JoinView& J, const uint64_t* __restrict__ keys,
                                             int side, int s, const int* __restrict__ exp_flag, double2* eloc,
                                             FusedSmem* F, uint16_t* spos, int e, int lane) {
  const bool mag = *exp_flag == 0;  // amplitude magnitudes from the records (k_gather_records)
  int rp[kFPer];
  double2* acc = F->acc[e];  // per served search warp: the current row's sum of chunk sums (lane 0 writes)
#pragma unroll
  for (int i = 0; i < kFPer; ++i) rp[i] = 0;
  if (lane < kFPer) acc[lane] = make_double2(0.0, 0.0);
  __syncwarp();
  unsigned idle = 0;
  for (;;) {
    bool progressed = false, all_done = true;
#pragma unroll
    for (int i = 0; i < kFPer; ++i) {
      const int sw = e * kFPer + i;
      const int done = F->done[sw];
      __threadfence_block();
      FusedHdr& hd = F->h[sw][rp[i]];
      if (hd.state != 1) {
        all_done &= done != 0;
        continue;
      }
      all_done = false;
      progressed = true;
      __threadfence_block();
      const FusedQ& q = F->q[sw][rp[i]];
      const int64_t row = hd.row;
      const unsigned n_hits = hd.n, nd = hd.nd;
      if (n_hits) {
        Key<W> xrow;
#pragma unroll
        for (int w = 0; w < W; ++w) xrow.w[w] = __ldg(keys + row * W + w);
        const U64x4 sr = ldg256(J.rec + row * 4);
        const double la_i = __longlong_as_double(static_cast<long long>(sr.a));
        const double2 cs_i = make_double2(__longlong_as_double(static_cast<long long>(sr.b)),
                                          __longlong_as_double(static_cast<long long>(sr.c)));
        const double inv_ai = mag ? 1.0 / __longlong_as_double(static_cast<long long>(sr.d)) : 0.0;
        __syncwarp();
        if (lane < s) spos[lane] = hd.pos[lane];
        __syncwarp();
        double2 a = make_double2(0.0, 0.0);
        for (unsigned k0 = 0; k0 < n_hits; k0 += 32) {
          const unsigned k = k0 + lane;
          JoinHit h;
          h.valid = k < n_hits;
          h.key = kNoKey;
          h.sr = U64x4{0, 0, 0, 0};
#pragma unroll
          for (int t = 0; t < kGrecWords; ++t) h.r[t] = 0;
          if (h.valid) {
            const unsigned src = k < nd ? k : kJQueue - 1 - (k - nd);
            const uint32_t y = q.y[src], g = q.g[src];
            h.key = q.k[src];
            h.sr = ldg256(J.rec + static_cast<int64_t>(y) * 4);
            const U64x4 g0 = ldg256(J.grec + static_cast<int64_t>(g) * kGrecWords);
            const U64x4 g1 = ldg256(J.grec + static_cast<int64_t>(g) * kGrecWords + 4);
            h.r[0] = g0.a; h.r[1] = g0.b; h.r[2] = g0.c; h.r[3] = g0.d;
            h.r[4] = g1.a; h.r[5] = g1.b; h.r[6] = g1.c; h.r[7] = g1.d;
          }
          eval_hit<W>(H, J, spos, h, xrow, la_i, cs_i, lane, s, side, a, inv_ai);
        }
        const double sx = warp_sum(a.x), sy = warp_sum(a.y);
        if (lane == 0) {
          acc[i].x += sx;
          acc[i].y += sy;
        }
      }
      if (hd.last && lane == 0) {
        eloc[hd.out] = make_double2(hd.base.x + acc[i].x, hd.base.y + acc[i].y);
        acc[i] = make_double2(0.0, 0.0);
      }
      __syncwarp();
      __threadfence_block();
      if (lane == 0) hd.state = 0;  // the slot goes back to its search warp
      rp[i] = rp[i] + 1 == kFRing ? 0 : rp[i] + 1;
    }
    if (!progressed) {
      if (all_done) break;
      __nanosleep(idle < 8 ? 32 : 256);
      ++idle;
    } else {
      idle = 0;
    }
  }
}

#ifndef QVMC_SEARCH_MINB
#define QVMC_SEARCH_MINB 4  // split search kernel (no drain): 64 registers, 32 warps per SM (measured best, r01x)
#endif

template <int W, int MODE>
__global__ void __launch_bounds__(MODE == kModeFused ? kFThreads : kThreads,
                                  MODE == kModeFused ? QVMC_FUSED_MINB
                                                     : (MODE == kModeHits ? QVMC_SEARCH_MINB : QVMC_JOIN_MINB))
    k_rows_join(const __grid_constant__ HamView H, const TableView T, const __grid_constant__ JoinView J,
                const uint64_t* __restrict__ keys, const RowSet R, int side, int s, const __grid_constant__ Ctl C,
                const __grid_constant__ RowOut O) {
  static_assert(MODE == kModeHits || MODE == kModeCount || MODE == kModeEmit || MODE == kModeFused,
                "join modes: hits, count, emit, fused");
  constexpr bool kFused = MODE == kModeFused;
  constexpr bool kEval = MODE == kModeHits || kFused;  // E_loc rows (split or fused evaluation)
  constexpr int kSearchWarps = kFused ? kFSearch : kWarps;
  __shared__ JoinSmem s_w[kSearchWarps];
  // dynamic shared memory: kModeFused's chunk rings (sizeof(FusedSmem)), then the bucket tables
  extern __shared__ __align__(16) unsigned char s_dyn[];
  FusedSmem* s_f = reinterpret_cast<FusedSmem*>(s_dyn);
  __shared__ uint16_t s_epos[kFused ? kFEval : 1][32];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  if constexpr (kFused) {
    if (threadIdx.x < kFSearch * kFRing) {
      s_f[0].h[threadIdx.x / kFRing][threadIdx.x % kFRing].state = 0;
      if (threadIdx.x % kFRing == 0) s_f[0].done[threadIdx.x / kFRing] = 0;
    }
    __syncthreads();
    if (wid >= kFSearch) {  // evaluation warps
      fused_eval_loop<W>(H, J, keys, side, s, O.exp_flag, O.eloc, s_f, s_epos[wid - kFSearch], wid - kFSearch,
                         lane);
      return;
    }
  }
  JoinSmem* sm = &s_w[wid];
  unsigned qr = 0;  // kModeFused: the ring slot this search warp fills
  const int n = H.n;
  const int n_ranges = s * (s - 1) / 2;
  // the row's buckets: pre[t] = first walk index of bucket t (exclusive prefix
  // of the bucket lengths), pre[C] = members walked; binfo[t] = (lo - pre[t]
  // (mod 2^32: member of walk index j at mem[binfo.x + j]), doubles-bitmap row
  // P + pidx(T_x) * P); tab[t] = T_x.a | T_x.b << 8
  unsigned char* rg_base = s_dyn + (kFused ? sizeof(FusedSmem) : 0) + wid * join_range_bytes(n_ranges);
  uint2* const s_binfo = reinterpret_cast<uint2*>(rg_base);
  uint32_t* const s_pre = reinterpret_cast<uint32_t*>(rg_base + 8 * n_ranges);
  uint16_t* const s_tab = reinterpret_cast<uint16_t*>(rg_base + 8 * n_ranges + 4 * (n_ranges + 1));
  if (lane == 0) {
    sm->qn = 0;
    sm->qs = 0;
  }
  __syncwarp();
  // the search warp hands its current slot to its evaluation warp and takes the
  // next one once that is free again (kModeFused)
  auto publish = [&](int64_t row, int64_t out, bool last, double2 base) {
    if constexpr (kFused) {
      FusedHdr& hd = s_f[0].h[wid][qr];
      __syncwarp();
      if (lane < 16) hd.pos[lane] = static_cast<uint8_t>(sm->pos[lane]);
      if (lane == 0) {
        hd.row = static_cast<uint32_t>(row);
        hd.out = static_cast<uint32_t>(out);
        hd.nd = static_cast<uint16_t>(sm->qn);
        hd.n = static_cast<uint16_t>(sm->qn + sm->qs);
        hd.last = last ? 1 : 0;
        hd.base = base;
        sm->qn = 0;
        sm->qs = 0;
      }
      __syncwarp();
      __threadfence_block();
      if (lane == 0) hd.state = 1;
      qr = qr + 1 == kFRing ? 0 : qr + 1;
      if (lane == 0) {
        unsigned w = 0;
        while (s_f[0].h[wid][qr].state != 0) __nanosleep(w++ < 8 ? 32 : 128);
      }
      __syncwarp();
      __threadfence_block();
    }
  };

  uint64_t tot_cand = 0, tot_hits = 0;
  for (;;) {
    unsigned long long r = 0;
    if (lane == 0) r = atomicAdd(C.row_next, 1ull);
    r = __shfl_sync(0xffffffffu, r, 0);
    if (static_cast<int64_t>(r) >= R.n_rows) break;
    const int64_t row = R.list ? static_cast<int64_t>(__ldg(R.list + r)) : R.base + static_cast<int64_t>(r);
    const int64_t orow = R.perm ? static_cast<int64_t>(__ldg(R.perm + row)) : row;  // caller's row

    uint64_t S[W];
    {
      Key<W> xrow;
#pragma unroll
      for (int w = 0; w < W; ++w) xrow.w[w] = __ldg(keys + row * W + w);
      double la_i = 0.0;
      U64x4 sr = {0, 0, 0, 0};
      if (kEval) {
        sr = ldg256(J.rec + row * 4);
        la_i = __longlong_as_double(static_cast<long long>(sr.a));
      }
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int w = 0; w < W; ++w) sm->x[w] = xrow.w[w];
        sm->la = la_i;
        sm->cs_c = __longlong_as_double(static_cast<long long>(sr.b));
        sm->cs_s = __longlong_as_double(static_cast<long long>(sr.c));
      }
#pragma unroll
      for (int w = 0; w < W; ++w) {
        S[w] = side ? xrow.w[w] : ~xrow.w[w];
        const int hi_bit = n - 64 * w;
        if (hi_bit < 64) S[w] &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
      }
    }
    __syncwarp();
    if (kEval) {
      if (isinf(*reinterpret_cast<const volatile double*>(&sm->la))) {  // energy.cpp:32-33
        if (lane == 0) atomicOr(C.err, kErrZeroAmp);
        if constexpr (kFused) {
          publish(row, orow - R.out_base, true, make_double2(CUDART_NAN, CUDART_NAN));
        } else if (lane == 0) {
          O.base[orow - R.out_base] = make_double2(CUDART_NAN, CUDART_NAN);
          O.row_last[orow - R.out_base] = ~0u;
        }
        continue;
      }
    }
    if (MODE == kModeEmit && lane == 0) sm->cursor = 0;

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
    if (lane < s) {
      sm->pos[lane] = static_cast<uint16_t>(pos);
      if (MODE == kModeHits) O.rowpos[row * 32 + lane] = static_cast<uint8_t>(pos);
      if (kFused && lane >= s && lane < 16) sm->pos[lane] = 0;
    }
    __syncwarp();
    const int pos0 = sm->pos[0], pos1 = sm->pos[1];
    // bucket t of this row: pair (a, b) of S(x), range from the index; the
    // lengths' exclusive prefix turns the C ranges into one walk index space
    uint32_t M = 0;  // members walked by this row (warp-uniform)
    for (int t0 = 0; t0 < n_ranges; t0 += 32) {
      const int t = t0 + lane;
      uint32_t len = 0, lo = 0, db = 0;
      int pa = 0, pb = 0;
      if (t < n_ranges) {
        const uint32_t b = pair_b(t);
        pa = sm->pos[t - b * (b - 1) / 2];
        pb = sm->pos[b];
        const uint2 rg = __ldcs(J.rng + static_cast<uint64_t>(row) * J.C + t);  // read once per call
        lo = rg.x;
        len = rg.y - rg.x;
        db = J.P + pidx(pa, pb) * J.P;
      }
      uint32_t inc = len;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
      }
      const uint32_t ex = M + inc - len;
      if (t < n_ranges) {
        s_tab[t] = static_cast<uint16_t>(pa | pb << 8);
        s_pre[t] = ex;
        s_binfo[t] = make_uint2(lo - ex, db);
      }
      M += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) s_pre[n_ranges] = M;
    __syncwarp();

    double2 acc = make_double2(0.0, 0.0);
    uint32_t hits = 0;
    uint64_t cand = lane == 0 ? M : 0;
    uint32_t prev_chunk = ~0u;  // kModeHits: last flushed chunk of this row
    bool dup = false;           // a duplicate of this row's key in the sample set
    uint32_t s_head = 0, s_tail = 0;  // survivor ring (warp-uniform)
    // the queue becomes one chunk of this row (split evaluation) once it holds `thresh` hits
    auto emit = [&](unsigned thresh) {
      if constexpr (kFused) {
        __syncwarp();
        if (sm->qn + sm->qs >= thresh) publish(row, orow - R.out_base, false, make_double2(0.0, 0.0));
      } else if (kEval) {
        __syncwarp();
        const unsigned qd = sm->qn, qsn = sm->qs;
        const unsigned qn = qd + qsn;
        if (qn >= thresh) {
          {
            unsigned long long off = 0, cid = 0;
            if (lane == 0) {
              off = atomicAdd(O.hit_cursor, static_cast<unsigned long long>(qn));
              cid = atomicAdd(O.chunk_cursor, 1ull);
            }
            off = __shfl_sync(0xffffffffu, off, 0);
            cid = __shfl_sync(0xffffffffu, cid, 0);
            if (off + qn <= O.hit_cap && cid < O.chunk_cap) {
              for (unsigned k = lane; k < qn; k += 32) {
                const unsigned src = k < qd ? k : kJQueue - 1 - (k - qd);
                // evict-first (streaming): the chunks are read once, and must not push
                // the records and tables the evaluation gathers out of L2 (measured -0.55 ms)
                __stcs(O.hy + off + k, sm->qy[src]);
                __stcs(O.hg + off + k, sm->qg[src]);
                __stcs(O.hk + off + k, sm->qk[src]);
              }
              if (lane == 0)
                O.chunk[cid] = make_uint4(static_cast<uint32_t>(row), static_cast<uint32_t>(off), qn, prev_chunk);
              prev_chunk = static_cast<uint32_t>(cid);
            } else if (lane == 0) {
              atomicOr(C.err, kErrHitOverflow);  // the host grows the buffers and reruns
              if (cid < O.chunk_cap)             // a reserved chunk is always defined (empty)
                O.chunk[cid] = make_uint4(static_cast<uint32_t>(row), 0u, 0u, ~0u);
            }
            __syncwarp();
            if (lane == 0) {
              sm->qn = 0;
              sm->qs = 0;
            }
            __syncwarp();
          }
        }
      }
    };
    // flip-table lookups of up to 32 survivors with every lane busy, hits queued
    auto lookups = [&]() {
      const uint32_t cntl = min(s_tail - s_head, 32u);
      const bool valid = static_cast<uint32_t>(lane) < cntl;
      uint32_t y = 0, kk = kNoKey;
      int64_t g = -1;
      if (valid) {
        const uint32_t e = (s_head + lane) & (kJSurv - 1);
        y = sm->sy[e];
        kk = sm->sk[e];
        const uint32_t bk = xy_bucket(kk, static_cast<uint32_t>(J.xy_mask));
        g = xy_resolve(kk, ldg256(J.xy_tab + static_cast<uint64_t>(bk) * 4));
        if (g == kChain) g = xy_chain(kk, bk, J.xy_tab, static_cast<uint32_t>(J.xy_mask));
      }
      s_head += cntl;
      // warp-aggregated append of the hits
      const bool hit = g >= 0;
      const unsigned hm = __ballot_sync(0xffffffffu, hit);
      if (hm) {
        if (kEval) {  // doubles fill the queue from the bottom, singles from the top
          const bool is_s = (kk >> 16) == 0xFFFFu;
          const unsigned lt = (1u << lane) - 1u;
          const unsigned hs = __ballot_sync(0xffffffffu, hit && is_s), hd = hm & ~hs;
          const unsigned bd = sm->qn, bs = sm->qs;
          if (hit) {
            const unsigned k = is_s ? kJQueue - 1 - (bs + __popc(hs & lt)) : bd + __popc(hd & lt);
            if constexpr (kFused) {
              FusedQ& fq = s_f[0].q[wid][qr];
              fq.y[k] = y;
              fq.g[k] = static_cast<uint32_t>(g);
              fq.k[k] = kk;
            } else {
              sm->qy[k] = y;
              sm->qg[k] = static_cast<uint32_t>(g);
              sm->qk[k] = kk;
            }
          }
          __syncwarp();
          if (lane == 0) {
            sm->qn = bd + __popc(hd);
            sm->qs = bs + __popc(hs);
          }
        } else if (MODE == kModeEmit) {
          unsigned base = 0;
          if (lane == 0) base = atomicAdd(&sm->cursor, __popc(hm));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (hit) {
            const unsigned k = base + __popc(hm & ((1u << lane) - 1u));
            const uint64_t at = O.row_off[orow] + k;
            O.xp_out[at] = R.perm ? __ldg(R.perm + y) : y;
            O.g_out[at] = static_cast<uint32_t>(g);
          }
        }
        hits += hit ? (J.sym ? 2u : 1u) : 0u;
      }
      __syncwarp();
      emit(kJDrainAt);
    };
    // the walk: lane l takes walk indices l, l+32, ...; its bucket cursor t only
    // moves forward (a bucket holds ~75 members at c118, so a lane crosses a
    // bucket end on fewer than half of its steps)
    {
      int t = 0;
      uint32_t nxt = M ? s_pre[1] : 0u;
      uint2 bi = s_binfo[0];
      uint32_t tx = s_tab[0];
      constexpr int U = QVMC_JOIN_UNROLL;
      for (uint32_t base = 0; base < M; base += 32 * U) {
        uint64_t v[U];
        uint32_t utx[U], udb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t j = base + 32 * u + lane;
          v[u] = ~0ull;
          utx[u] = 0;
          udb[u] = 0;
          if (j < M) {
            if (nxt <= j) {
              do {
                ++t;
                nxt = s_pre[t + 1];
              } while (nxt <= j);
              bi = s_binfo[t];
              tx = s_tab[t];
            }
            v[u] = __ldg(J.mem + (bi.x + j));
            utx[u] = tx;
            udb[u] = bi.y;
          }
        }
        // doubles-bitmap words of all U members in flight before the accept rule
        uint32_t dw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          dw[u] = ~0u;
          if (J.pbits && v[u] != ~0ull) {
            const uint32_t bit = udb[u] + static_cast<uint32_t>(v[u] >> 48);
            dw[u] = __ldg(J.pbits + (bit >> 5)) >> (bit & 31);
          }
        }
        // accept rule (header comment) -> exact position key of the flip mask
        uint32_t key[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          key[u] = kNoKey;
          if (v[u] == ~0ull) continue;
          const int ya = static_cast<int>(v[u] >> 32) & 0xFF, yb = static_cast<int>(v[u] >> 40) & 0xFF;
          const int ta = utx[u] & 0xFF, tb = utx[u] >> 8;
          const bool ea = ya == ta || ya == tb, eb = yb == ta || yb == tb;
          if (!ea && !eb) {  // disjoint pairs: double excitation; merge two sorted pairs
            if (!(dw[u] & 1u)) continue;
            int p0 = ta, p1 = tb, p2 = ya, p3 = yb;
            sort2(p0, p2);
            sort2(p1, p3);
            sort2(p1, p2);
            key[u] = static_cast<uint32_t>(p0) | static_cast<uint32_t>(p1) << 8 | static_cast<uint32_t>(p2) << 16 |
                     static_cast<uint32_t>(p3) << 24;
          } else if (ea != eb) {  // one shared orbital o: x loses c, gains a
            const int o = ea ? ya : yb, a = ea ? yb : ya;
            const int cc = (o == ta) ? tb : ta;
            if (o == (cc == pos0 ? pos1 : pos0)) {
              int p0 = cc, p1 = a;
              sort2(p0, p1);
              if (J.pbits && !pbit(J.pbits, pidx(p0, p1))) continue;
              key[u] = static_cast<uint32_t>(p0) | static_cast<uint32_t>(p1) << 8 | 0xFFFF0000u;
            }
          } else if (static_cast<uint32_t>(v[u]) != static_cast<uint32_t>(row)) {
            dup = true;  // T_y = T_x in an exact bucket: the same key at another position
          }
        }
        // survivors -> ring; the flip-table lookups then run 32 at a time with
        // every lane busy (a lookup per candidate would execute on nearly every
        // step for the ~1 in 7 candidates that survive)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const unsigned smk = __ballot_sync(0xffffffffu, key[u] != kNoKey);
          if (key[u] != kNoKey) {
            const uint32_t e = (s_tail + __popc(smk & ((1u << lane) - 1u))) & (kJSurv - 1);
            sm->sy[e] = static_cast<uint32_t>(v[u]);
            sm->sk[e] = key[u];
          }
          s_tail += __popc(smk);
        }
        __syncwarp();
        while (s_tail - s_head >= 32) lookups();
      }
      while (s_tail != s_head) lookups();
    }
    if (!kFused) emit(1u);  // fused: the remaining hits travel in the row's last chunk with its base

    const Key<W> xrow = row_key<W>(sm);
    // even flip masks of weight >= 6: popcount filter + sample-set probe
    if (H.n_res) {
      uint64_t S[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        S[w] = side ? xrow.w[w] : ~xrow.w[w];
        const int hi_bit = n - 64 * w;
        if (hi_bit < 64) S[w] &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
      }
      const uint64_t hx_res = key_hash_warp<W>(xrow.w, H.hash_bytes, lane);
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
            ++cand;
            const int64_t j = probe_slow<W>(xrow, fmix(hx_res ^ __ldg(H.xy_hash + g)), g, T.tab, T.mask, keys, H.xy);
            if (j >= 0) {
              ++hits;
              if (MODE == kModeEmit) {
                const unsigned k = atomicAdd(&sm->cursor, 1u);
                const uint64_t at = O.row_off[orow] + k;
                O.xp_out[at] = R.perm ? __ldg(R.perm + j) : static_cast<uint32_t>(j);
                O.g_out[at] = g;
              } else if (kEval) {  // rare: evaluated in place, term by term
                uint64_t xp[W];
#pragma unroll
                for (int w = 0; w < W; ++w) xp[w] = __ldg(keys + j * W + w);
                double hr, hi;
                group_element<W>(H, xp, g, hr, hi);
                const U64x4 sr = ldg256(J.rec + j * 4);
                add_ratio(__longlong_as_double(static_cast<long long>(sr.a)),
                          make_double2(__longlong_as_double(static_cast<long long>(sr.b)),
                                       __longlong_as_double(static_cast<long long>(sr.c))),
                          sm->la, make_double2(sm->cs_c, sm->cs_s), hr, hi, acc);
              }
            }
          }
        }
      }
    }

    // diagonal element as the quadratic form over S(x)
    if (kEval && H.diag >= 0) {
      if (H.diag_quad) {
        if (lane == 0) acc.x += side ? H.diag_A1 : H.diag_A0;
        if (lane < s) acc.x += __ldg(H.diag_b + side * n + pos);
        for (int pi = lane; pi < n_ranges; pi += 32) acc.x += __ldg(H.diag_K + (s_tab[pi] & 0xFF) * n + (s_tab[pi] >> 8));
        for (uint32_t e = lane; e < H.n_diag_other; e += 32) {
          const uint32_t t = __ldg(H.diag_other + e);
          int pc = 0;
#pragma unroll
          for (int w = 0; w < W; ++w) pc += __popcll(xrow.w[w] & __ldg(H.yz + (int64_t)t * W + w));
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
          for (int w = 0; w < W; ++w) pc += __popcll(xrow.w[w] & __ldg(H.yz + (int64_t)t * W + w));
          const int qt = (__ldg(H.yw + t) + 2 * pc) & 3;
          const double cf = __ldg(H.coeff + t);
          if (qt == 0) acc.x += cf;
          else if (qt == 2) acc.x -= cf;
          else if (qt == 1) acc.y += cf;
          else acc.y -= cf;
        }
      }
    }

    if (kEval) {  // the walk drained the queue; residual hits were evaluated in place
      const double re = warp_sum(acc.x);
      const double im = warp_sum(acc.y);
      if constexpr (kFused) {
        publish(row, orow - R.out_base, true, make_double2(re, im));
      } else if (lane == 0) {
        O.base[orow - R.out_base] = make_double2(re, im);
        O.row_last[orow - R.out_base] = prev_chunk;
      }
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
    if (__any_sync(0xffffffffu, dup) && lane == 0) atomicOr(C.err, kErrDuplicate);
  }
  if constexpr (kFused) {
    __syncwarp();
    __threadfence_block();
    if (lane == 0) s_f[0].done[wid] = 1;
  }
  tot_cand = warp_sum(tot_cand);
  if (lane == 0) {
    atomicAdd(C.stats, static_cast<unsigned long long>(tot_cand));
    atomicAdd(C.stats + 1, static_cast<unsigned long long>(tot_hits));
  }
}

// Exact, order-independent accumulation (symmetric mode): a contribution v is
// rounded once to the integer q = round(v * 2^48) and added as two 64-bit
// words, q mod 2^32 (unsigned) to a[0] and floor(q / 2^32) (signed) to a[1],
// with fire-and-forget atomics (no returned value on the critical path). The
// low word has 32 bits of headroom, so the exact sum a[1] * 2^32 + a[0] does
// not depend on the order the pairs arrive in.
__device__ __forceinline__ void fix_add(unsigned long long* a, double v, int* err) {
  if (v == 0.0) return;
  if (!(fabs(v) < 0x1.0p46)) {  // beyond the exact range (or not finite): the call reruns unpaired
    atomicOr(err, kErrFixRange);
    return;
  }
  const double sc = v * 0x1.0p48;
  long long hi;
  unsigned long long lo;
  if (fabs(sc) < 0x1.0p62) {
    const long long q = __double2ll_rn(sc);
    lo = static_cast<unsigned long long>(q) & 0xFFFFFFFFull;
    hi = q >> 32;  // arithmetic shift: floor
  } else {  // |v| >= 2^14
    const double qh = floor(sc * 0x1.0p-32);
    hi = static_cast<long long>(qh);
    lo = __double2ull_rn(sc - qh * 0x1.0p32);
  }
  if (lo) atomicAdd(a, lo);
  if (hi) atomicAdd(a + 1, static_cast<unsigned long long>(hi));
}

__device__ __forceinline__ double fix_value(const unsigned long long* a) {
  const long long hi = static_cast<long long>(a[1]);
  const unsigned long long lo = a[0];
  if (hi > -(1ll << 30) && hi < (1ll << 30))  // |sum * 2^48| < 2^62: exact in 64 bits, one rounding
    return static_cast<double>(static_cast<long long>((static_cast<unsigned long long>(hi) << 32) + lo)) *
           0x1.0p-48;
  return static_cast<double>(hi) * 0x1.0p-16 + static_cast<double>(lo) * 0x1.0p-48;
}

#ifndef QVMC_EVAL_MINB
#define QVMC_EVAL_MINB 3  // 80 registers (measured best, r01z)
#endif
#ifndef QVMC_EVAL_HITS
#define QVMC_EVAL_HITS 1  // hits per lane with records in flight together (2+: fewer warps, slower)
#endif

// Split evaluation, part 2: one warp per hit chunk (one row's hits in walk
// order). Row context once per chunk, then QVMC_JOIN_DRAIN_HITS hits per lane
// with all their records in flight; the chunk's sum goes to part[chunk].
template <int W>
__global__ void __launch_bounds__(kThreads, QVMC_EVAL_MINB)
    k_eval_chunks(const __grid_constant__ HamView H, const __grid_constant__ JoinView J,
                  const uint64_t* __restrict__ keys, const uint4* __restrict__ chunk,
                  const unsigned long long* __restrict__ n_chunks, const uint32_t* __restrict__ hy,
                  const uint32_t* __restrict__ hg, const uint32_t* __restrict__ hk, int side, int s,
                  const int* __restrict__ exp_flag, const uint8_t* __restrict__ rowpos, double2* __restrict__ part,
                  uint64_t chunk_cap, unsigned long long* __restrict__ fix, int* __restrict__ fix_err) {
  // fix != null (symmetric mode): the search walked only partners y > x, so every
  // hit also adds H_yx psi(x)/psi(y) = conj(H_xy) psi(x)/psi(y) to row y, exactly
  constexpr int DH = QVMC_EVAL_HITS;
  __shared__ uint16_t s_pos[kWarps][32];
  const int lane = threadIdx.x & 31;
  uint16_t* spos = s_pos[threadIdx.x >> 5];
  const uint64_t nc = min(static_cast<uint64_t>(*n_chunks), chunk_cap);  // an overflowed batch is rerun
  const bool mag = *exp_flag == 0;  // amplitude magnitudes from the records (k_gather_records)
  const uint64_t n_warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t c = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; c < nc; c += n_warps) {
    const uint4 ch = __ldg(chunk + c);
    const int64_t row = ch.x;
    Key<W> xrow;
#pragma unroll
    for (int w = 0; w < W; ++w) xrow.w[w] = __ldg(keys + row * W + w);
    const U64x4 sr = ldg256(J.rec + row * 4);
    const double la_i = __longlong_as_double(static_cast<long long>(sr.a));
    const double2 cs_i = make_double2(__longlong_as_double(static_cast<long long>(sr.b)),
                                      __longlong_as_double(static_cast<long long>(sr.c)));
    const double inv_ai = mag ? 1.0 / __longlong_as_double(static_cast<long long>(sr.d)) : 0.0;
    // minority orbitals of the row (kind B elements), as the search kernel listed them
    __syncwarp();
    if (lane < s) spos[lane] = __ldg(rowpos + row * 32 + lane);
    __syncwarp();
    double2 acc = make_double2(0.0, 0.0);
    const unsigned n_hits = ch.z;
    for (unsigned k0 = 0; k0 < n_hits; k0 += 32 * DH) {
      JoinHit h[DH];
#pragma unroll
      for (int d = 0; d < DH; ++d) {
        const unsigned k = k0 + 32 * d + lane;
        JoinHit& q = h[d];
        q.valid = k < n_hits;
        q.key = kNoKey;
        q.y = 0;
        q.sr = U64x4{0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < kGrecWords; ++i) q.r[i] = 0;
        if (q.valid) {
          const uint64_t at = static_cast<uint64_t>(ch.y) + k;
          const uint32_t y = __ldcs(hy + at), g = __ldcs(hg + at);  // streaming, see the search's flush
          q.key = __ldcs(hk + at);
          q.y = y;
          q.sr = ldg256(J.rec + static_cast<int64_t>(y) * 4);
          const U64x4 g0 = ldg256(J.grec + static_cast<int64_t>(g) * kGrecWords);
          const U64x4 g1 = ldg256(J.grec + static_cast<int64_t>(g) * kGrecWords + 4);
          q.r[0] = g0.a; q.r[1] = g0.b; q.r[2] = g0.c; q.r[3] = g0.d;
          q.r[4] = g1.a; q.r[5] = g1.b; q.r[6] = g1.c; q.r[7] = g1.d;
        }
      }
#pragma unroll
      for (int d = 0; d < DH; ++d) {
        if (!fix) {
          eval_hit<W>(H, J, spos, h[d], xrow, la_i, cs_i, lane, s, side, acc, inv_ai);
          continue;
        }
        double hr, hi;
        hit_element<W>(H, J, spos, h[d], xrow, lane, s, side, hr, hi);
        if (h[d].valid) {
          const double la_j = __longlong_as_double(static_cast<long long>(h[d].sr.a));
          const double2 cs_j = make_double2(__longlong_as_double(static_cast<long long>(h[d].sr.b)),
                                            __longlong_as_double(static_cast<long long>(h[d].sr.c)));
          double2 m = make_double2(0.0, 0.0);
          if (mag) {
            const double ej = __longlong_as_double(static_cast<long long>(h[d].sr.d));
            add_ratio_mag(ej * inv_ai, cs_j, cs_i, hr, hi, acc);
            add_ratio_mag(__longlong_as_double(static_cast<long long>(sr.d)) * (1.0 / ej), cs_i, cs_j, hr, -hi, m);
          } else {
            add_ratio(la_j, cs_j, la_i, cs_i, hr, hi, acc);
            add_ratio(la_i, cs_i, la_j, cs_j, hr, -hi, m);
          }
          unsigned long long* fy = fix + 4 * static_cast<uint64_t>(h[d].y);
          fix_add(fy, m.x, fix_err);
          fix_add(fy + 2, m.y, fix_err);
        }
      }
    }
    const double re = warp_sum(acc.x);
    const double im = warp_sum(acc.y);
    if (lane == 0) part[c] = make_double2(re, im);
  }
}

// Sharded symmetric mode: the rank's rows get the mirrored sums of every rank
// (all-reduced fixed point) after their own evaluation has finished.
__global__ void k_add_fix(const RowSet R, const unsigned long long* __restrict__ fix, double2* __restrict__ eloc) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < R.n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = R.list ? static_cast<int64_t>(__ldg(R.list + r)) : R.base + r;
    const int64_t i = (R.perm ? static_cast<int64_t>(__ldg(R.perm + row)) : row) - R.out_base;
    double2 e = eloc[i];
    e.x += fix_value(fix + 4 * row);
    e.y += fix_value(fix + 4 * row + 2);
    eloc[i] = e;
  }
}

// Split evaluation, part 3: E_loc = base + the row's chunk sums, newest chunk
// first (a fixed order: deterministic). Rows of one batch (RowSet).
__global__ void k_finalize_rows(const uint32_t* __restrict__ row_last, const uint4* __restrict__ chunk,
                                const double2* __restrict__ part, const double2* __restrict__ base, const RowSet R,
                                double2* __restrict__ eloc, const unsigned long long* __restrict__ fix) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < R.n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = R.list ? static_cast<int64_t>(__ldg(R.list + r)) : R.base + r;
    const int64_t i = (R.perm ? static_cast<int64_t>(__ldg(R.perm + row)) : row) - R.out_base;
    double2 e = base[i];
    for (uint32_t c = row_last[i]; c != ~0u; c = __ldg(chunk + c).w) {
      const double2 p = part[c];
      e.x += p.x;
      e.y += p.y;
    }
    if (fix) {  // symmetric mode: the partners y < x, exactly accumulated
      e.x += fix_value(fix + 4 * row);
      e.y += fix_value(fix + 4 * row + 2);
    }
    eloc[i] = e;
  }
}

}  // namespace qvmc_b200
