// Exact autoregressive sampling without replacement on the device: the
// ancestral Gumbel top-K beam of sample_without_replacement
// (/root/reference/proj/src/sampler.cpp:37-102), so the sampled keys never
// leave HBM between sampling, amplitudes and the local energies (SURVEY §8f
// item 3).
//
// Per qudit level (host loop, one level at a time):
//   1. k_log_psi_part(only_j = level, cond): the amplitude head's conditional
//      log-probability table of every beam prefix (model.cpp:203-252);
//   2. k_expand: one warp per beam entry b. Each allowed child value v gets
//      log p = parent + cond[b][v] and the Gumbel draw of the counter
//      (iteration, level, b, v) (Philox4x32-10, rng.cpp / rng.hpp), the
//      warp max z, then condition_max (sampler.cpp:15-23); children are
//      appended to the candidate list (warp-aggregated atomics);
//   3. CUB radix sort of the candidates by conditioned value, descending;
//      runs of equal values (rare) are ordered by child prefix (k_ties) —
//      together exactly ChildLess (sampler.cpp:27-33);
//   4. k_gather_beam: the first min(K, candidates) become the next beam,
//      in that order (the beam slot b feeds the next level's counters).
#pragma once

#include <cstdint>

namespace qvmc_sampler {

// Philox4x32-10 (rng.cpp:15-44)
__device__ __forceinline__ void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

// CounterRng(seed, stream).gumbel(c0, c1, c2, c3) (rng.hpp:38-63)
__device__ __forceinline__ double counter_gumbel(uint64_t seed, uint32_t stream, uint32_t c0, uint32_t c1,
                                                 uint32_t c2, uint32_t c3) {
  uint32_t c[4] = {c0, c1, c2, c3};
  philox(c, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32) ^ stream);
  const uint64_t b = (static_cast<uint64_t>(c[1]) << 32) | c[0];
  double u = static_cast<double>(b >> 11) * 0x1.0p-53;
  if (u < 1e-300) u = 1e-300;
  if (u > 1.0 - 1e-16) u = 1.0 - 1e-16;
  return -log(-log(u));
}

// condition_max (sampler.cpp:15-23)
__device__ __forceinline__ double condition_max(double parent, double z, double child) {
  if (child == z) return parent;
  const double m = fmax(-parent, -child);
  const double v = exp(-parent - m) - exp(-z - m) + exp(-child - m);
  if (!(v > 0.0)) return parent;
  const double r = -(m + log(v));
  return fmin(r, parent);
}

// sort key: ascending order of the key = descending conditioned value
__device__ __forceinline__ uint64_t desc_key(double d) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(d));
  const uint64_t asc = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  return ~asc;
}

struct Candidates {
  uint64_t* key;   // desc_key(conditioned perturbed value)
  uint32_t* slot;  // 0..n-1 (sort payload)
  uint32_t* bv;    // beam entry << 6 | value
  double* lp;      // child log-probability
  double* pert;    // conditioned perturbed value
  unsigned long long* count;
};

// one warp per beam entry (sampler.cpp:53-74); the 8 warps of a block take 8
// consecutive entries per step and reserve their children's output slots with
// one atomic per block step (a block-level scan of the warps' counts), not one
// per warp: a single global counter hit by every warp serialised the kernel
__global__ void __launch_bounds__(256)
    k_expand(const double* __restrict__ cond, const double* __restrict__ beam_lp, const double* __restrict__ beam_pert,
             int64_t B, int n_out, uint64_t seed, uint32_t stream, uint32_t iteration, uint32_t level, Candidates C) {
  __shared__ unsigned s_cnt[2][8];
  __shared__ unsigned long long s_base[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int ph = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * 8;
  // the entry's conditional row and parent values, loaded one step ahead (the kernel waits on them)
  auto fetch = [&](int64_t e, double& a0, double& a1, double& lp, double& pt) {
    const bool lv = e < B;
    a0 = (lv && lane < n_out) ? cond[e * 64 + lane] : -CUDART_INF;
    a1 = (lv && lane + 32 < n_out) ? cond[e * 64 + 32 + lane] : -CUDART_INF;
    lp = lv ? beam_lp[e] : 0.0;
    pt = lv ? beam_pert[e] : 0.0;
  };
  double n0c, n1c, nlp, npt;
  fetch(static_cast<int64_t>(blockIdx.x) * 8 + warp, n0c, n1c, nlp, npt);
  for (int64_t b0 = static_cast<int64_t>(blockIdx.x) * 8; b0 < B; b0 += stride) {
    const int64_t b = b0 + warp;  // b >= B: the fetch gave -inf rows, so no children
    const double c0 = n0c, c1 = n1c, plp = nlp, ppert = npt;
    fetch(b + stride, n0c, n1c, nlp, npt);
    // the entry's allowed values (cond > -inf), compacted onto lanes in value order: the k-th
    // allowed value goes to lane k % 32 of pass k / 32 (one pass unless more than 32 are allowed)
    const unsigned m0 = __ballot_sync(0xffffffffu, c0 != -CUDART_INF);
    const unsigned m1 = __ballot_sync(0xffffffffu, c1 != -CUDART_INF);
    const int n0 = __popc(m0), n = n0 + __popc(m1);
    double clp[2], u[2];
    int vv[2];
    double z = -CUDART_INF;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      u[h] = -CUDART_INF;
      clp[h] = 0.0;
      vv[h] = 0;
      if (32 * h >= n) continue;  // warp-uniform
      const int k = 32 * h + lane;
      int v = 0;
      if (k < n) v = k < n0 ? static_cast<int>(__fns(m0, 0, k + 1)) : 32 + static_cast<int>(__fns(m1, 0, k - n0 + 1));
      const double s0 = __shfl_sync(0xffffffffu, c0, v & 31), s1 = __shfl_sync(0xffffffffu, c1, v & 31);
      if (k < n) {
        vv[h] = v;
        clp[h] = plp + (v < 32 ? s0 : s1);
        u[h] = clp[h] + counter_gumbel(seed, stream, iteration, level, static_cast<uint32_t>(b),
                                       static_cast<uint32_t>(v));
        z = fmax(z, u[h]);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) z = fmax(z, __shfl_xor_sync(0xffffffffu, z, o));
    if (lane == 0) s_cnt[ph][warp] = static_cast<unsigned>(n);
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned tot = 0;
      for (int w = 0; w < 8; ++w) tot += s_cnt[ph][w];
      s_base[ph] = tot ? atomicAdd(C.count, static_cast<unsigned long long>(tot)) : 0ull;
    }
    __syncthreads();
    unsigned long long base = s_base[ph];
    for (int w = 0; w < warp; ++w) base += s_cnt[ph][w];
    ph ^= 1;  // the next step writes the other buffers: one barrier per step suffices
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = 32 * h + lane;
      if (k < n) {
        const uint64_t s = base + static_cast<uint64_t>(k);
        const double cp = condition_max(ppert, z, u[h]);
        C.key[s] = desc_key(cp);
        C.slot[s] = static_cast<uint32_t>(s);
        C.bv[s] = static_cast<uint32_t>(b) << 6 | static_cast<uint32_t>(vv[h]);
        C.lp[s] = clp[h];
        C.pert[s] = cp;
      }
    }
  }
}

// child prefix: the parent's key with value v deposited at [off, off + k)
// (deposit_bits, basis_vector.cpp:47-50: qubit off+t <- bit k-1-t of v)
template <int W>
__device__ __forceinline__ void child_key(const uint64_t* __restrict__ beam_keys, uint32_t bv, int off, int k,
                                          uint64_t* out) {
  const uint32_t b = bv >> 6, v = bv & 63u;
#pragma unroll
  for (int w = 0; w < W; ++w) out[w] = beam_keys[static_cast<int64_t>(b) * W + w];
  for (int t = 0; t < k; ++t)
    if ((v >> (k - 1 - t)) & 1u) {
      const int q = off + t;
      out[q >> 6] |= 1ull << (q & 63);
    }
}

template <int W>
__device__ __forceinline__ bool key_less(const uint64_t* a, const uint64_t* b) {  // std::array words_ order
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (a[w] != b[w]) return a[w] < b[w];
  return false;
}

// runs of equal conditioned values that start inside the kept prefix [0, keep):
// order them by child prefix (ChildLess ties, sampler.cpp:31). One thread per run.
template <int W>
__global__ void k_ties(const uint64_t* __restrict__ skey, uint32_t* __restrict__ sslot, int64_t n, int64_t keep,
                       const uint32_t* __restrict__ bv, const uint64_t* __restrict__ beam_keys, int off, int k) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < keep;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (i + 1 >= n || skey[i + 1] != skey[i] || (i > 0 && skey[i - 1] == skey[i])) continue;
    int64_t e = i + 1;
    while (e < n && skey[e] == skey[i]) ++e;
    for (int64_t a = i + 1; a < e; ++a) {  // insertion sort by prefix
      const uint32_t s = sslot[a];
      uint64_t ks[W], kb[W];
      child_key<W>(beam_keys, bv[s], off, k, ks);
      int64_t c = a;
      while (c > i) {
        child_key<W>(beam_keys, bv[sslot[c - 1]], off, k, kb);
        if (!key_less<W>(ks, kb)) break;
        sslot[c] = sslot[c - 1];
        --c;
      }
      sslot[c] = s;
    }
  }
}

template <int W>
__global__ void k_gather_beam(const uint32_t* __restrict__ sslot, int64_t keep, const Candidates C,
                              const uint64_t* __restrict__ beam_keys, int off, int k, uint64_t* __restrict__ out_keys,
                              double* __restrict__ out_lp, double* __restrict__ out_pert) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < keep;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s = sslot[i];
    uint64_t kk[W];
    child_key<W>(beam_keys, C.bv[s], off, k, kk);
#pragma unroll
    for (int w = 0; w < W; ++w) out_keys[i * W + w] = kk[w];
    out_lp[i] = C.lp[s];
    out_pert[i] = C.pert[s];
  }
}

}  // namespace qvmc_sampler
