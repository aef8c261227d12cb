// Amplitude evaluation on the device: AnqsModel::log_psi over a batch of
// sampled determinants and fill_amplitudes (the stage that
// produces the (log ψ, φ) the local-energy path consumes).
//
// Reference: /root/reference/proj/src/model.cpp
//   parameter blocks    :65-80   (per qudit: amplitude block, then phase block;
//                                 W1 [hidden][n] row-major, b1, W2, b2, W3 [2^k][hidden], b3)
//   QuditInfo           :82-93
//   allowed_values      :129-151
//   encode_prefix       :153-158 (+1/-1 on the prefix bits, 0 after them)
//   mlp_forward         :160-175 (h1 = tanh(W1 e + b1), h2 = tanh(W2 h1 + b2 + h1), out = W3 h2 + b3)
//   conditional         :203-252 (mean shift; log-softmax of 2*amp over the allowed values)
//   in_sector, log_psi  :254-271
// and fill_amplitudes, /root/reference/proj/src/sampler.cpp:104-120.
//
// Design (B200, fp64 on the CUDA cores — the reference computes in double and
// tcgen05 has no fp64 kind):
//  * one CTA of 256 threads owns a tile of 64 samples and walks every qudit
//    in order, so log ψ and φ are summed in the reference's qudit order
//    without a second pass;
//  * layer 1 never multiplies by the ±1 encoding: W1 e = 2 Σ_{ones} W1[:,i] − c
//    = c − 2 Σ_{zeros} W1[:,i] with c = Σ_{i<offset} W1[:,i] precomputed per
//    qudit, summed over the minority of the prefix (≤ 8 holes per sample at
//    118 qubits / 110 electrons instead of 118 products);
//  * layers 2 and 3 are 64×64×64 register-tiled GEMMs (4 samples × 4 outputs
//    per thread) out of shared memory; activations are stored k-major with a
//    32-byte-chunk XOR swizzle so both the transposed writes and the GEMM
//    reads are conflict-free; the next weight matrix streams into a second
//    buffer with cp.async while the current GEMM runs;
//  * the phase head's output layer is a single dot product per sample
//    (only out[v] of the sampled value is used);
//  * the amplitude softmax reduces across the 16 lanes that hold one sample's
//    64 outputs with shuffles.
// Parameters are re-laid out once per set_params (W1ᵀ, W2ᵀ, W3ᵀ, prefix
// column sums) so every load in the kernel is contiguous.

#include <cuda_pipeline_primitives.h>

namespace qvmc_model {

constexpr int kHid = 64;      // hidden width of the device path (the reference's default, model.hpp:61)
constexpr int kMaxK = 6;      // bits per qudit (2^k ≤ 64 outputs; the reference's default, model.hpp:24)
constexpr int kTile = 64;     // samples per CTA
constexpr int kMThreads = 256;

// per (qudit, head) block of the device parameter layout, in doubles
struct BlockLayout {
  int n;
  __host__ __device__ int w1t() const { return 0; }                 // [n][64]
  __host__ __device__ int b1() const { return n * kHid; }           // [64]
  __host__ __device__ int csum() const { return n * kHid + 64; }    // [64] Σ_{i<offset} W1[h][i]
  __host__ __device__ int w2t() const { return n * kHid + 128; }    // [64 k][64 h]
  __host__ __device__ int b2() const { return n * kHid + 128 + 4096; }
  __host__ __device__ int w3t() const { return n * kHid + 192 + 4096; }  // [64 k][64 v], v ≥ 2^k zero
  __host__ __device__ int b3() const { return n * kHid + 192 + 8192; }   // [64], v ≥ 2^k zero
  __host__ __device__ int size() const { return n * kHid + 256 + 8192; }
};

struct ModelView {
  const double* P;      // [n_qudits][2][BlockLayout::size()]
  int n, n_qudits, bits;
  int n_e, spin, n_up;
};

// swizzled k-major activation tile: element (k, s) of a [64][64] tile
__device__ __forceinline__ int act_idx(int k, int s) { return k * kTile + (((s >> 2) ^ ((k >> 2) & 15)) << 2) + (s & 3); }

__device__ __forceinline__ void stage_64x64(double* dst, const double* src, int tid) {
  // 32 KB, 16 B per cp.async, 8 per thread
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int e = (r * kMThreads + tid) * 2;
    __pipeline_memcpy_async(dst + e, src + e, 16);
  }
  __pipeline_commit();
}

// a thread's 4 samples × 4 features <-> the swizzled tile, as 16-byte pairs of samples
__device__ __forceinline__ void store_tile(double* act, const double v[4][4], int sg, int hg) {
#pragma unroll
  for (int hi = 0; hi < 4; ++hi) {
    double2* p = reinterpret_cast<double2*>(act + act_idx(hg * 4 + hi, sg * 4));
    p[0] = make_double2(v[0][hi], v[1][hi]);
    p[1] = make_double2(v[2][hi], v[3][hi]);
  }
}
__device__ __forceinline__ void load_tile(const double* act, double v[4][4], int sg, int hg) {
#pragma unroll
  for (int hi = 0; hi < 4; ++hi) {
    const double2* p = reinterpret_cast<const double2*>(act + act_idx(hg * 4 + hi, sg * 4));
    const double2 a = p[0], b = p[1];
    v[0][hi] = a.x;
    v[1][hi] = a.y;
    v[2][hi] = b.x;
    v[3][hi] = b.y;
  }
}

// acc[si][hi] = Σ_k act[k][sg*4+si] · w[k][hg*4+hi]
__device__ __forceinline__ void gemm_64(const double* __restrict__ act, const double* __restrict__ w, int sg, int hg,
                                        double acc[4][4]) {
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
#pragma unroll 8
  for (int k = 0; k < kHid; ++k) {
    const double2* ap = reinterpret_cast<const double2*>(act + act_idx(k, sg * 4));
    const double2 a01 = ap[0], a23 = ap[1];
    const double2* wp = reinterpret_cast<const double2*>(w + k * kHid + hg * 4);
    const double2 w01 = wp[0], w23 = wp[1];
    const double av[4] = {a01.x, a01.y, a23.x, a23.y};
    const double wv[4] = {w01.x, w01.y, w23.x, w23.y};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], wv[b], acc[a][b]);
  }
}

template <int W>
__global__ void __launch_bounds__(kMThreads, 2)
    k_log_psi(const ModelView M, const uint64_t* __restrict__ keys, int64_t N, double* __restrict__ out_la,
              double* __restrict__ out_ph) {
  extern __shared__ __align__(16) double smem[];
  double* act = smem;                     // [64][64] swizzled activations
  double* wA = smem + kHid * kTile;       // W2ᵀ of the current head
  double* wB = wA + kHid * kHid;          // W3ᵀ of the amplitude head
  __shared__ uint64_t s_key[kTile][W];
  __shared__ double s_la[kTile], s_ph[kTile];

  const int tid = threadIdx.x;
  const int hg = tid & 15, sg = tid >> 4;
  const int64_t s0 = static_cast<int64_t>(blockIdx.x) * kTile;
  for (int e = tid; e < kTile * W; e += kMThreads) {
    const int s = e / W, w = e % W;
    s_key[s][w] = (s0 + s < N) ? __ldg(keys + (s0 + s) * W + w) : 0ull;
  }
  if (tid < kTile) {
    s_la[tid] = 0.0;
    s_ph[tid] = 0.0;
  }
  __syncthreads();

  const BlockLayout L{M.n};
  const int bsize = L.size();
  for (int j = 0; j < M.n_qudits; ++j) {
    const int off = j * M.bits;
    const int k = min(M.bits, M.n - off);
    const int n_out = 1 << k;
    // QuditInfo (model.cpp:82-93)
    const int rem_after = M.n - off - k;
    int rem_up_after = 0;
    for (int i = off + k; i < M.n; ++i) rem_up_after += (i % 2 == 0);
    uint32_t up_value_mask = 0;
    for (int t = 0; t < k; ++t)
      if ((off + t) % 2 == 0) up_value_mask |= 1u << (k - 1 - t);

    // per-sample prefix facts for this thread's 4 samples
    int pw[4], pu[4], val[4];
#pragma unroll
    for (int si = 0; si < 4; ++si) {
      const int s = sg * 4 + si;
      int c = 0, cu = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const int lo = 64 * w;
        if (off <= lo) break;
        const uint64_t m = (off - lo >= 64) ? ~0ull : ((1ull << (off - lo)) - 1);
        const uint64_t x = s_key[s][w] & m;
        c += __popcll(x);
        cu += __popcll(x & 0x5555555555555555ull);
      }
      pw[si] = c;
      pu[si] = cu;
      uint32_t v = 0;  // extract_bits (basis_vector.cpp:40-45): qubit off+t -> bit k-1-t
      for (int t = 0; t < k; ++t) {
        const int q = off + t;
        v |= static_cast<uint32_t>((s_key[s][q >> 6] >> (q & 63)) & 1ull) << (k - 1 - t);
      }
      val[si] = static_cast<int>(v);
    }

    for (int hd = 0; hd < 2; ++hd) {
      const double* B = M.P + static_cast<int64_t>(2 * j + hd) * bsize;
      stage_64x64(wA, B + L.w2t(), tid);
      if (hd == 0) stage_64x64(wB, B + L.w3t(), tid);

      // layer 1: pre1 = b1 + W1 e over the prefix minority (model.cpp:153-158, :171)
      {
        const double2* cp = reinterpret_cast<const double2*>(B + L.csum() + hg * 4);
        const double2 c01 = __ldg(cp), c23 = __ldg(cp + 1);
        const double2* bp = reinterpret_cast<const double2*>(B + L.b1() + hg * 4);
        const double2 b01 = __ldg(bp), b23 = __ldg(bp + 1);
        const double cs[4] = {c01.x, c01.y, c23.x, c23.y}, bb[4] = {b01.x, b01.y, b23.x, b23.y};
        double h1[4][4];
#pragma unroll
        for (int si = 0; si < 4; ++si) {
          const int s = sg * 4 + si;
          const bool ones = 2 * pw[si] <= off;  // sum over the smaller of ones / zeros
          double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const int lo = 64 * w;
            if (off <= lo) break;
            const uint64_t m = (off - lo >= 64) ? ~0ull : ((1ull << (off - lo)) - 1);
            uint64_t x = (ones ? s_key[s][w] : ~s_key[s][w]) & m;
            while (x) {
              const int i = lo + __ffsll(static_cast<long long>(x)) - 1;
              x &= x - 1;
              const double2* wp = reinterpret_cast<const double2*>(B + L.w1t() + i * kHid + hg * 4);
              const double2 w01 = __ldg(wp), w23 = __ldg(wp + 1);
              a[0] += w01.x;
              a[1] += w01.y;
              a[2] += w23.x;
              a[3] += w23.y;
            }
          }
#pragma unroll
          for (int hi = 0; hi < 4; ++hi) {
            const double we = ones ? 2.0 * a[hi] - cs[hi] : cs[hi] - 2.0 * a[hi];
            h1[si][hi] = tanh(we + bb[hi]);
          }
        }
        store_tile(act, h1, sg, hg);
      }
      if (hd == 0) __pipeline_wait_prior(1);  // W2ᵀ landed (W3ᵀ may still be in flight)
      else __pipeline_wait_prior(0);
      __syncthreads();

      // layer 2: h2 = tanh(W2 h1 + b2 + h1) (model.cpp:172)
      double acc[4][4];
      gemm_64(act, wA, sg, hg, acc);
      {
        const double2* bp = reinterpret_cast<const double2*>(B + L.b2() + hg * 4);
        const double2 b01 = __ldg(bp), b23 = __ldg(bp + 1);
        const double bb[4] = {b01.x, b01.y, b23.x, b23.y};
        double res[4][4];
        load_tile(act, res, sg, hg);
#pragma unroll
        for (int si = 0; si < 4; ++si)
#pragma unroll
          for (int hi = 0; hi < 4; ++hi) acc[si][hi] = tanh(acc[si][hi] + bb[hi] + res[si][hi]);
      }
      __syncthreads();
      store_tile(act, acc, sg, hg);
      __pipeline_wait_prior(0);
      __syncthreads();

      if (hd == 0) {
        // amplitude head: out = W3 h2 + b3, mean shift, log-softmax of 2*out over
        // the allowed values (model.cpp:173-174, :218-249)
        gemm_64(act, wB, sg, hg, acc);
        const double2* bp = reinterpret_cast<const double2*>(B + L.b3() + hg * 4);
        const double2 b01 = __ldg(bp), b23 = __ldg(bp + 1);
        const double bb[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int si = 0; si < 4; ++si) {
          double sum = 0.0;
#pragma unroll
          for (int vi = 0; vi < 4; ++vi) {
            acc[si][vi] += bb[vi];
            sum += acc[si][vi];  // v ≥ 2^k: W3ᵀ and b3 are zero-padded, out = 0
          }
#pragma unroll
          for (int o = 8; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
          const double mean = sum / static_cast<double>(n_out);
          double two[4];
          bool ok[4];
          double mx = -CUDART_INF;
#pragma unroll
          for (int vi = 0; vi < 4; ++vi) {
            const int v = hg * 4 + vi;
            two[vi] = 2.0 * (acc[si][vi] - mean);
            // allowed_values (model.cpp:129-151)
            const int w = pw[si] + __popc(v);
            bool a = v < n_out && w <= M.n_e && w + rem_after >= M.n_e;
            if (a && M.spin) {
              const int wu = pu[si] + __popc(static_cast<uint32_t>(v) & up_value_mask);
              const int wd = w - wu;
              const int n_down = M.n_e - M.n_up;
              const int rem_down = rem_after - rem_up_after;
              a = wu <= M.n_up && wu + rem_up_after >= M.n_up && wd <= n_down && wd + rem_down >= n_down;
            }
            ok[vi] = a;
            if (a) mx = fmax(mx, two[vi]);
          }
#pragma unroll
          for (int o = 8; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
          double se = 0.0;
#pragma unroll
          for (int vi = 0; vi < 4; ++vi)
            if (ok[vi]) se += exp(two[vi] - mx);
#pragma unroll
          for (int o = 8; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
          const int v = val[si];
          if ((v >> 2) == hg) {  // the lane holding out[v]: log_amp[v] = (2 out[v] - lse) / 2
            const double lse = mx + log(se);
            const int q = v & 3;
            const double tv = q == 0 ? two[0] : q == 1 ? two[1] : q == 2 ? two[2] : two[3];
            s_la[sg * 4 + si] += 0.5 * (tv - lse);
          }
        }
      } else {
        // phase head: only out[v] of the sampled value (model.cpp:173-174, :250)
        double part[4];
#pragma unroll
        for (int si = 0; si < 4; ++si) {
          const int s = sg * 4 + si;
          const int v = val[si];
          double d = 0.0;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const int kx = hg * 4 + kk;
            d = fma(act[act_idx(kx, s)], __ldg(B + L.w3t() + kx * kHid + v), d);
          }
          part[si] = d;
        }
#pragma unroll
        for (int si = 0; si < 4; ++si) {
#pragma unroll
          for (int o = 8; o; o >>= 1) part[si] += __shfl_xor_sync(0xffffffffu, part[si], o);
          if (hg == 0) s_ph[sg * 4 + si] += part[si] + __ldg(B + L.b3() + val[si]);
        }
      }
      __syncthreads();
    }
  }

  if (tid < kTile && s0 + tid < N) {
    // in_sector (model.cpp:254-259): masked states get (-inf, 0) (model.cpp:263)
    int pc = 0, pe = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      pc += __popcll(s_key[tid][w]);
      pe += __popcll(s_key[tid][w] & 0x5555555555555555ull);
    }
    const bool ins = pc == M.n_e && (!M.spin || pe == M.n_up);
    out_la[s0 + tid] = ins ? s_la[tid] : -CUDART_INF;
    out_ph[s0 + tid] = ins ? s_ph[tid] : 0.0;
  }
}

// log_norm = logsumexp(log_probs) (sampler.cpp:114-119), deterministic:
// fixed grid, per-block online (max, scaled sum), merged in block order.
constexpr int kLseBlocks = 296;

__global__ void __launch_bounds__(256) k_lse_partial(const double* __restrict__ lp, int64_t n, double2* part) {
  __shared__ double2 red[256];
  double m = -CUDART_INF, s = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x; i < n; i += static_cast<int64_t>(gridDim.x) * 256) {
    const double x = __ldg(lp + i);
    if (x == -CUDART_INF) continue;  // exp(-inf - m) = 0
    if (x > m) {
      s = s * exp(m - x) + 1.0;
      m = x;
    } else {
      s += exp(x - m);
    }
  }
  red[threadIdx.x] = make_double2(m, s);
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if (threadIdx.x < w) {
      const double2 a = red[threadIdx.x], b = red[threadIdx.x + w];
      const double mm = fmax(a.x, b.x);
      red[threadIdx.x] = mm == -CUDART_INF ? make_double2(mm, 0.0)
                                           : make_double2(mm, a.y * exp(a.x - mm) + b.y * exp(b.x - mm));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_lse_final(const double2* __restrict__ part, int nb, double* out2) {
  if (threadIdx.x != 0) return;
  double m = -CUDART_INF, s = 0.0;
  for (int b = 0; b < nb; ++b) {
    const double2 p = part[b];
    const double mm = fmax(m, p.x);
    if (mm == -CUDART_INF) continue;
    s = s * exp(m - mm) + p.y * exp(p.x - mm);
    m = mm;
  }
  const double ln = m + log(s);
  out2[0] = exp(ln);  // norm
  out2[1] = ln;       // log_norm
}

}  // namespace qvmc_model
