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
#ifndef QVMC_MODEL_MINB
#define QVMC_MODEL_MINB 3  // CTAs per SM (measured: 3 with one weight buffer beats 2 with a W3ᵀ prefetch buffer)
#endif
constexpr int kWBufs = QVMC_MODEL_MINB >= 3 ? 1 : 2;  // 3+ CTAs/SM: W3ᵀ reuses the W2ᵀ buffer (64 KB smem)

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

// e^x for x ≤ 0 in ~17 instructions: x = k ln2 + r (magic-number rounding, two-part ln2),
// Taylor degree 12 on |r| ≤ ln2/2, 2^k added to the exponent field. Relative error
// ≲ 1e-14 over [-700, 0] (vs 1 ulp for the libdevice exp, which costs ~3× more).
__device__ __forceinline__ double exp_core(double x);  // x in [-700, 0], no clamp
__device__ __forceinline__ double exp_nonpos(double x) {
  return exp_core(x < -700.0 ? -700.0 : x);  // a select, not fmax (no NaN handling needed)
}
__device__ __forceinline__ double exp_core(double x) {
  const double t = fma(x, 1.4426950408889634, 6755399441055744.0);  // 1.5·2^52: k in the low word
  const int k = __double2loint(t);
  const double kf = t - 6755399441055744.0;
  double r = fma(kf, -6.93147180559945286227e-01, x);
  r = fma(kf, -2.31904681384629955842e-17, r);
  double p = 2.08767569878680989792e-09;  // 1/12!
  p = fma(p, r, 2.50521083854417187751e-08);
  p = fma(p, r, 2.75573192239858906526e-07);
  p = fma(p, r, 2.75573192239858906526e-06);
  p = fma(p, r, 2.48015873015873015873e-05);
  p = fma(p, r, 1.98412698412698412698e-04);
  p = fma(p, r, 1.38888888888888888889e-03);
  p = fma(p, r, 8.33333333333333333333e-03);
  p = fma(p, r, 4.16666666666666666667e-02);
  p = fma(p, r, 1.66666666666666666667e-01);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  return __hiloint2double(__double2hiint(p) + (k << 20), __double2loint(p));
}

// tanh(x) = sign(x) (1 − e)/(1 + e), e = e^{−2|x|}; the reciprocal from the
// MUFU.RCP64H seed plus two Newton steps. Absolute error ≲ 5e-15 (the
// activations feed linear layers, so absolute error is what propagates).
__device__ __forceinline__ double tanh_fast(double x) {
  const double ax = fabs(x);
  const double e = exp_core(-2.0 * (ax < 40.0 ? ax : 40.0));  // tanh(40) = 1 in fp64
  const double d = 1.0 + e;
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  y = fma(y, fma(-d, y, 1.0), y);
  y = fma(y, fma(-d, y, 1.0), y);
  return copysign((1.0 - e) * y, x);
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
__global__ void __launch_bounds__(kMThreads, QVMC_MODEL_MINB)
    k_log_psi(const ModelView M, const uint64_t* __restrict__ keys, int64_t N, double* __restrict__ out_la,
              double* __restrict__ out_ph) {
  extern __shared__ __align__(16) double smem[];
  double* act = smem;                     // [64][64] swizzled activations
  double* wA = smem + kHid * kTile;       // W2ᵀ of the current head
  double* wB = kWBufs == 2 ? wA + kHid * kHid : wA;  // W3ᵀ of the amplitude head
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
      if (hd == 0 && kWBufs == 2) stage_64x64(wB, B + L.w3t(), tid);

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
            h1[si][hi] = tanh_fast(we + bb[hi]);
          }
        }
        store_tile(act, h1, sg, hg);
      }
      if (hd == 0 && kWBufs == 2) __pipeline_wait_prior(1);  // W2ᵀ landed (W3ᵀ may still be in flight)
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
          for (int hi = 0; hi < 4; ++hi) acc[si][hi] = tanh_fast(acc[si][hi] + bb[hi] + res[si][hi]);
      }
      __syncthreads();
      store_tile(act, acc, sg, hg);
      if (hd == 0 && kWBufs == 1) stage_64x64(wB, B + L.w3t(), tid);  // W2ᵀ reads are done
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
            if (ok[vi]) se += exp_nonpos(two[vi] - mx);
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

// ---------------------------------------------------------------------------
// Warp-tiled variant (default): one CTA of 16 warps owns ONE (qudit, head)
// block of the model and a chunk of samples. The block's W2ᵀ / W3ᵀ are staged
// into shared memory once; every warp then runs its own 16-sample tiles
// through layer 1, the layer-2 GEMM and the output layer with only
// __syncwarp — no CTA barrier inside the sample loop, so the 16 warps hide
// each other's gather / transcendental / shuffle latency. A lane holds 4
// samples × 8 features (32 fp64 accumulators): per k it loads 4 activations
// and 8 weights (6 LDS.128, one wavefront each) for 32 DFMA. Each (sample,
// qudit, head) writes its conditional log-amplitude / phase to
// part[2j+hd][s]; k_sum_qudits adds them in qudit order (the reference's
// summation order, model.cpp:264-270) and applies in_sector.
constexpr int kWT = 16;        // samples per warp tile
constexpr int kPWarps = 16;    // warps per CTA
constexpr int kPThreads = kPWarps * 32;

// warp activation tile [64 k][16 s]: 32-byte chunk swizzled by (k >> 3), the
// 16-byte half by (k >> 1), so stores of rows 16m+2hq+b by the 8 hq lanes and
// the GEMM's row reads are both conflict-free
__device__ __forceinline__ int pidx(int k, int s) {
  return k * kWT + ((((s >> 2) ^ (k >> 3)) & 3) << 2) + (((((s >> 1) ^ (k >> 1)) & 1)) << 1) + (s & 1);
}

template <int W>
__global__ void __launch_bounds__(kPThreads, 1)
    k_log_psi_part(const ModelView M, const uint64_t* __restrict__ keys, int64_t N, int64_t chunk,
                   double* __restrict__ part, int only_j = -1, double* __restrict__ cond = nullptr,
                   int phase_only = 0, double* __restrict__ hcache = nullptr) {
  // hcache (phase_only): the phase heads' activations per sample, [qudit][N][h1 64 | h2 64], kept for
  // the energy gradient of the same batch (k_grad_fwd copies them instead of recomputing)
  // only_j >= 0 (the sampler, sampler.cpp:53-55): the amplitude head of qudit only_j
  // for every key (a beam prefix), writing the whole conditional log-probability
  // table cond[s][64] (model.cpp:226-249; -inf for disallowed values) instead of part
  extern __shared__ __align__(16) double smem[];
  double* w2 = smem;                   // [64 k][64 h]
  double* w3 = smem + 4096;            // [64 k][64 v]
  double* bias = smem + 8192;          // b1 | csum | b2 | b3, 64 each
  double* acts = smem + 8448;          // [16 warps][64][16]
  uint64_t* skeys = reinterpret_cast<uint64_t*>(acts + kPWarps * 64 * kWT);  // [16 warps][16][W]

  // phase_only: the phase heads alone (a freshly sampled batch's log|psi| is half its log p)
  const int n_jh = only_j >= 0 ? 1 : (phase_only ? M.n_qudits : 2 * M.n_qudits);
  const int jh = only_j >= 0 ? 2 * only_j
                             : (phase_only ? 2 * static_cast<int>(blockIdx.x % n_jh) + 1
                                           : static_cast<int>(blockIdx.x % n_jh)),
            j = jh >> 1, hd = jh & 1;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x / n_jh) * chunk;
  const int64_t c1 = min(N, c0 + chunk);
  const BlockLayout L{M.n};
  const double* B = M.P + static_cast<int64_t>(jh) * L.size();
  for (int e = threadIdx.x * 2; e < 4096; e += kPThreads * 2) {
    *reinterpret_cast<double2*>(w2 + e) = __ldg(reinterpret_cast<const double2*>(B + L.w2t() + e));
    *reinterpret_cast<double2*>(w3 + e) = __ldg(reinterpret_cast<const double2*>(B + L.w3t() + e));  // both heads
  }
  if (threadIdx.x < 64) {
    bias[threadIdx.x] = __ldg(B + L.b1() + threadIdx.x);
    bias[64 + threadIdx.x] = __ldg(B + L.csum() + threadIdx.x);
    bias[128 + threadIdx.x] = __ldg(B + L.b2() + threadIdx.x);
    bias[192 + threadIdx.x] = __ldg(B + L.b3() + threadIdx.x);
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sq = lane >> 3, hq = lane & 7;  // samples sq*4..+3; features 16m + 2hq + b
  double* act = acts + warp * 64 * kWT;
  uint64_t* sk = skeys + warp * kWT * W;
  const int off = j * M.bits;
  const int k = min(M.bits, M.n - off);
  const int n_out = 1 << k;
  const int rem_after = M.n - off - k;  // QuditInfo (model.cpp:82-93)
  int rem_up_after = 0;
  for (int i = off + k; i < M.n; ++i) rem_up_after += (i % 2 == 0);
  uint32_t up_value_mask = 0;
  for (int t = 0; t < k; ++t)
    if ((off + t) % 2 == 0) up_value_mask |= 1u << (k - 1 - t);
  double* out = part + static_cast<int64_t>(jh) * N;

  for (int64_t t0 = c0 + static_cast<int64_t>(warp) * kWT; t0 < c1; t0 += static_cast<int64_t>(kWT) * kPWarps) {
    __syncwarp();
    for (int e = lane; e < kWT * W; e += 32) {
      const int64_t g = t0 + e / W;
      sk[e] = g < c1 ? __ldg(keys + g * W + (e % W)) : 0ull;
    }
    __syncwarp();
    int pw[4], pu[4], val[4];
#pragma unroll
    for (int si = 0; si < 4; ++si) {
      const uint64_t* x = sk + (sq * 4 + si) * W;
      int c = 0, cu = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const int lo = 64 * w;
        if (off > lo) {
          const uint64_t msk = (off - lo >= 64) ? ~0ull : ((1ull << (off - lo)) - 1);
          c += __popcll(x[w] & msk);
          cu += __popcll(x[w] & msk & 0x5555555555555555ull);
        }
      }
      pw[si] = c;
      pu[si] = cu;
      // extract_bits (basis_vector.cpp:40-45): qubit off+t -> bit k-1-t, i.e. the
      // k-bit field at off (spanning at most two words) bit-reversed
      const int wq = off >> 6, bq = off & 63;
      uint64_t fld = x[wq] >> bq;
      if (bq + k > 64 && wq + 1 < W) fld |= x[wq + 1] << (64 - bq);
      val[si] = static_cast<int>(__brev(static_cast<uint32_t>(fld)) >> (32 - k));
    }

    // layer 1 over the prefix minority, two samples at a time (model.cpp:153-158, :171)
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      double a[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int si = 2 * p + u;
        const uint64_t* x = sk + (sq * 4 + si) * W;
        const bool ones = 2 * pw[si] <= off;
#pragma unroll
        for (int f = 0; f < 8; ++f) a[u][f] = 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const int lo = 64 * w;
          if (off <= lo) break;
          const uint64_t msk = (off - lo >= 64) ? ~0ull : ((1ull << (off - lo)) - 1);
          uint64_t xm = (ones ? x[w] : ~x[w]) & msk;
          while (xm) {
            const int i = lo + __ffsll(static_cast<long long>(xm)) - 1;
            xm &= xm - 1;
            const double* row = B + L.w1t() + i * kHid + 2 * hq;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const double2 wv = __ldg(reinterpret_cast<const double2*>(row + 16 * m));
              a[u][2 * m] += wv.x;
              a[u][2 * m + 1] += wv.y;
            }
          }
        }
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          const int h = 16 * (f >> 1) + 2 * hq + (f & 1);
          const double cs = bias[64 + h];
          a[u][f] = tanh_fast((ones ? 2.0 * a[u][f] - cs : cs - 2.0 * a[u][f]) + bias[h]);
        }
      }
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        const int h = 16 * (f >> 1) + 2 * hq + (f & 1);
        *reinterpret_cast<double2*>(act + pidx(h, sq * 4 + 2 * p)) = make_double2(a[0][f], a[1][f]);
      }
      if (hcache) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int64_t g = t0 + sq * 4 + 2 * p + u;
          if (g < c1)
#pragma unroll
            for (int f = 0; f < 8; f += 2)
              *reinterpret_cast<double2*>(hcache + (static_cast<int64_t>(j) * N + g) * 128 + 16 * (f >> 1) + 2 * hq) =
                  make_double2(a[u][f], a[u][f + 1]);
        }
      }
    }
    __syncwarp();

    // layer 2 GEMM: acc[si][f] = Σ_k h1[s][k] W2[h][k] (model.cpp:172)
    double acc[4][8];
    auto gemm = [&](const double* wm) {
#pragma unroll
      for (int si = 0; si < 4; ++si)
#pragma unroll
        for (int f = 0; f < 8; ++f) acc[si][f] = 0.0;
#pragma unroll 4
      for (int kk = 0; kk < kHid; ++kk) {
        const double2 a01 = *reinterpret_cast<const double2*>(act + pidx(kk, sq * 4));
        const double2 a23 = *reinterpret_cast<const double2*>(act + pidx(kk, sq * 4 + 2));
        const double av[4] = {a01.x, a01.y, a23.x, a23.y};
        double wv[8];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const double2 t = *reinterpret_cast<const double2*>(wm + kk * kHid + 16 * m + 2 * hq);
          wv[2 * m] = t.x;
          wv[2 * m + 1] = t.y;
        }
#pragma unroll
        for (int si = 0; si < 4; ++si)
#pragma unroll
          for (int f = 0; f < 8; ++f) acc[si][f] = fma(av[si], wv[f], acc[si][f]);
      }
    };
    gemm(w2);
    // h2 = tanh(W2 h1 + b2 + h1): the residual h1 is read at this lane's own positions
#pragma unroll
    for (int f = 0; f < 8; ++f) {
      const int h = 16 * (f >> 1) + 2 * hq + (f & 1);
      const double2 r01 = *reinterpret_cast<const double2*>(act + pidx(h, sq * 4));
      const double2 r23 = *reinterpret_cast<const double2*>(act + pidx(h, sq * 4 + 2));
      const double b2 = bias[128 + h];
      acc[0][f] = tanh_fast(acc[0][f] + b2 + r01.x);
      acc[1][f] = tanh_fast(acc[1][f] + b2 + r01.y);
      acc[2][f] = tanh_fast(acc[2][f] + b2 + r23.x);
      acc[3][f] = tanh_fast(acc[3][f] + b2 + r23.y);
    }

    if (hd == 1) {
      if (hcache) {
#pragma unroll
        for (int si = 0; si < 4; ++si) {
          const int64_t g = t0 + sq * 4 + si;
          if (g < c1)
#pragma unroll
            for (int f = 0; f < 8; f += 2)
              *reinterpret_cast<double2*>(hcache + (static_cast<int64_t>(j) * N + g) * 128 + 64 + 16 * (f >> 1) +
                                          2 * hq) = make_double2(acc[si][f], acc[si][f + 1]);
        }
      }
      // phase head: only out[v] of the sampled value (model.cpp:173-174, :250)
#pragma unroll
      for (int si = 0; si < 4; ++si) {
        const int v = val[si];
        double d = 0.0;
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          const int h = 16 * (f >> 1) + 2 * hq + (f & 1);
          d = fma(acc[si][f], w3[h * kHid + v], d);
        }
#pragma unroll
        for (int o = 4; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        const int64_t g = t0 + sq * 4 + si;
        if (hq == 0 && g < c1) out[g] = d + bias[192 + v];
      }
      continue;
    }

    // amplitude head: h2 -> act, out = W3 h2 + b3, mean shift, log-softmax of
    // 2*out over the allowed values (model.cpp:173-174, :218-249)
    __syncwarp();
#pragma unroll
    for (int f = 0; f < 8; ++f) {
      const int h = 16 * (f >> 1) + 2 * hq + (f & 1);
      *reinterpret_cast<double2*>(act + pidx(h, sq * 4)) = make_double2(acc[0][f], acc[1][f]);
      *reinterpret_cast<double2*>(act + pidx(h, sq * 4 + 2)) = make_double2(acc[2][f], acc[3][f]);
    }
    __syncwarp();
    gemm(w3);
#pragma unroll
    for (int si = 0; si < 4; ++si) {
      double sum = 0.0;
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        acc[si][f] += bias[192 + 16 * (f >> 1) + 2 * hq + (f & 1)];
        sum += acc[si][f];  // v ≥ 2^k: zero-padded weights and bias, out = 0
      }
#pragma unroll
      for (int o = 4; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const double mean = sum / static_cast<double>(n_out);
      double mx = -CUDART_INF;
      uint32_t okm = 0;
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        const int v = 16 * (f >> 1) + 2 * hq + (f & 1);
        acc[si][f] = 2.0 * (acc[si][f] - mean);
        const int w = pw[si] + __popc(v);  // allowed_values (model.cpp:129-151)
        bool a = v < n_out && w <= M.n_e && w + rem_after >= M.n_e;
        if (a && M.spin) {
          const int wu = pu[si] + __popc(static_cast<uint32_t>(v) & up_value_mask);
          const int wd = w - wu;
          const int n_down = M.n_e - M.n_up;
          const int rem_down = rem_after - rem_up_after;
          a = wu <= M.n_up && wu + rem_up_after >= M.n_up && wd <= n_down && wd + rem_down >= n_down;
        }
        if (a) {
          okm |= 1u << f;
          mx = fmax(mx, acc[si][f]);
        }
      }
#pragma unroll
      for (int o = 4; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      double se = 0.0;
#pragma unroll
      for (int f = 0; f < 8; ++f)
        if (okm >> f & 1u) se += exp_nonpos(acc[si][f] - mx);
#pragma unroll
      for (int o = 4; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
      const int v = val[si];
      const int64_t g = t0 + sq * 4 + si;
      if (cond) {  // sampler: every value's log-probability (model.cpp:236-247)
        if (g < c1) {
          const double lse = mx + log(se);
#pragma unroll
          for (int f = 0; f < 8; ++f)
            cond[g * 64 + 16 * (f >> 1) + 2 * hq + (f & 1)] = (okm >> f & 1u) ? acc[si][f] - lse : -CUDART_INF;
        }
        continue;
      }
      if (((v >> 1) & 7) == hq && g < c1) {  // the lane holding out[v]
        const int fv = 2 * (v >> 4) + (v & 1);
        double tv = acc[si][0];
#pragma unroll
        for (int f = 1; f < 8; ++f)
          if (f == fv) tv = acc[si][f];
        out[g] = 0.5 * (tv - (mx + log(se)));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Gradient of log ψ (grad_log_psi, model.cpp:273-325, mlp_backward :177-201)
// contracted with per-sample coefficients, for energy_gradient (energy.cpp:80-107):
//   grad = Σ_i 2 Re{c_i O_i},  c_i = w_i (E_i − Ē),  O_i = [d log|ψ| ; −i d φ].
// The amplitude blocks collect 2 Re c_i · (d log|ψ|), the phase blocks
// 2 Im c_i · (d φ). Every weight gradient is an outer product summed over
// samples, so k_grad_fwd / k_grad_bwd write, per (qudit, head) block and
// sample, the forward activations h1, h2 and the coefficient-scaled backward
// vectors g (output), gz2, gz1 (64 doubles each) to chunk buffers, and the host
// sums them with strided-batched DGEMMs (gW1 = Σ gz1 eᵀ, gW2 = Σ gz2 h1ᵀ,
// gW3 = Σ g h2ᵀ; biases = Σ of the vectors). Same warp tiling as
// k_log_psi_part (16-sample tiles, lane = 4 samples × 8 features); the
// backward GEMMs read W3 / W2 in their original (v, h) / (h, k) layouts.
// row stride of the W2 / W3 gradient accumulators [block][out][kHS]: 64 inputs,
// the bias gradient (row 64 of each output's column) and a zero pad. The h1 / h2
// chunk rows are 64 wide: the GEMMs run at M = 64 (whole 32-row tiles) and the
// bias rows come from the kernels' per-warp sums (k_bias_rows)
constexpr int kHS = 66;

// the forward / backward split of the gradient kernels: 16 warps per CTA each
#ifndef QVMC_G2_WARPS
#define QVMC_G2_WARPS 16
#endif
constexpr int kG2Warps = QVMC_G2_WARPS;
constexpr int kG2Threads = kG2Warps * 32;

// bias sums: a warp adds its tile's 4 samples x 8 features per lane, summed over the
// 4 sample groups, into its own shared row (lanes 0-7 hold distinct features)
// (samples past the chunk end are masked: their softmax can be 0/0)
__device__ __forceinline__ void add_tile_sums(const double (&v)[4][8], unsigned valid, double* row, int lane) {
  const int hq = lane & 7;
#pragma unroll
  for (int f = 0; f < 8; ++f) {
    double t = ((valid & 1u) ? v[0][f] : 0.0) + ((valid & 2u) ? v[1][f] : 0.0);
    t += ((valid & 4u) ? v[2][f] : 0.0) + ((valid & 8u) ? v[3][f] : 0.0);
    t += __shfl_xor_sync(0xffffffffu, t, 8);
    t += __shfl_xor_sync(0xffffffffu, t, 16);
    if (lane < 8) row[16 * (f >> 1) + 2 * hq + (f & 1)] += t;
  }
}

// the CTA's sums, warps in order, to out[jh][cta][64] (summed over CTAs by k_bias_rows)
__device__ __forceinline__ void write_cta_sums(const double* bsum, double* out, int jh, int cta, int n_cta) {
  __syncthreads();
  if (threadIdx.x < 64) {
    double t = 0.0;
    for (int w = 0; w < kG2Warps; ++w) t += bsum[w * 64 + threadIdx.x];
    out[(static_cast<int64_t>(jh) * n_cta + cta) * 64 + threadIdx.x] = t;
  }
}

template <int W>
__global__ void __launch_bounds__(kG2Threads, 1)
    k_grad_fwd(const ModelView M, const uint64_t* __restrict__ keys, int64_t N, int64_t chunk,
                const double2* __restrict__ coef, double* __restrict__ H1, double* __restrict__ H2,
                double* __restrict__ G, int64_t N_blk, double* __restrict__ GSUM,
                const double* __restrict__ HC = nullptr, int64_t hc_rows = 0) {
  // HC (phase blocks): this chunk's cached activations [qudit][hc_rows][h1 | h2] from the sampled-batch
  // fill (bit-identical to recomputing them): copied to the chunk rows, only the one-hot g formed
  // N: samples of this call; N_blk: rows per block in the buffers (>= N, padded for split-K)
  extern __shared__ __align__(16) double smem[];
  double* w2 = smem;            // [64 k][64 h]  (W2 transposed)
  double* w3 = smem + 4096;     // [64 k][64 v]  (W3 transposed)
  double* bias = smem + 8192;   // b1 | csum | b2 | b3
  double* acts = smem + 8448;   // [warps][64][16]
  double* bsum = acts + kG2Warps * 64 * kWT;  // [warps][64]: Σ g of the warp's tiles (gb3)
  uint64_t* skeys = reinterpret_cast<uint64_t*>(bsum + kG2Warps * 64);

  const int n_jh = 2 * M.n_qudits;
  const int jh = static_cast<int>(blockIdx.x % n_jh), j = jh >> 1, hd = jh & 1;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x / n_jh) * chunk;
  const int64_t c1 = min(N, c0 + chunk);
  const BlockLayout L{M.n};
  const double* B = M.P + static_cast<int64_t>(jh) * L.size();
  for (int e = threadIdx.x; e < 4096; e += kG2Threads) {
    w2[e] = __ldg(B + L.w2t() + e);
    w3[e] = __ldg(B + L.w3t() + e);
  }
  for (int e = threadIdx.x; e < kG2Warps * 64; e += kG2Threads) bsum[e] = 0.0;
  if (threadIdx.x < 64) {
    bias[threadIdx.x] = __ldg(B + L.b1() + threadIdx.x);
    bias[64 + threadIdx.x] = __ldg(B + L.csum() + threadIdx.x);
    bias[128 + threadIdx.x] = __ldg(B + L.b2() + threadIdx.x);
    bias[192 + threadIdx.x] = __ldg(B + L.b3() + threadIdx.x);
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sq = lane >> 3, hq = lane & 7;
  double* act = acts + warp * 64 * kWT;
  uint64_t* sk = skeys + warp * kWT * W;
  const int off = j * M.bits;
  const int k = min(M.bits, M.n - off);
  const int n_out = 1 << k;
  const int rem_after = M.n - off - k;
  int rem_up_after = 0;
  for (int i = off + k; i < M.n; ++i) rem_up_after += (i % 2 == 0);
  uint32_t up_value_mask = 0;
  for (int t = 0; t < k; ++t)
    if ((off + t) % 2 == 0) up_value_mask |= 1u << (k - 1 - t);
  const int64_t blk = static_cast<int64_t>(jh) * N_blk * 64;
  double *h1o = H1 + blk, *h2o = H2 + blk, *go = G + blk;
  auto feat = [&](int f) { return 16 * (f >> 1) + 2 * hq + (f & 1); };

  for (int64_t t0 = c0 + static_cast<int64_t>(warp) * kWT; t0 < c1; t0 += static_cast<int64_t>(kWT) * kG2Warps) {
    __syncwarp();
    for (int e = lane; e < kWT * W; e += 32) {
      const int64_t g = t0 + e / W;
      sk[e] = g < c1 ? __ldg(keys + g * W + (e % W)) : 0ull;
    }
    __syncwarp();
    int pw[4], pu[4], val[4];
    double cf[4];
#pragma unroll
    for (int si = 0; si < 4; ++si) {
      const uint64_t* x = sk + (sq * 4 + si) * W;
      int c = 0, cu = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const int lo = 64 * w;
        if (off > lo) {
          const uint64_t msk = (off - lo >= 64) ? ~0ull : ((1ull << (off - lo)) - 1);
          c += __popcll(x[w] & msk);
          cu += __popcll(x[w] & msk & 0x5555555555555555ull);
        }
      }
      pw[si] = c;
      pu[si] = cu;
      const int wq = off >> 6, bq = off & 63;
      uint64_t fld = x[wq] >> bq;
      if (bq + k > 64 && wq + 1 < W) fld |= x[wq + 1] << (64 - bq);
      val[si] = static_cast<int>(__brev(static_cast<uint32_t>(fld)) >> (32 - k));
      const int64_t g = t0 + sq * 4 + si;
      const double2 c2 = g < c1 ? coef[g] : make_double2(0.0, 0.0);
      cf[si] = hd ? c2.y : c2.x;
    }
    auto row = [&](int si) { return t0 + sq * 4 + si; };
    auto put = [&](double* o, int si, int f, double v0, double v1, int ld = 64) {  // features f, f+1 of sample si
      if (row(si) < c1) *reinterpret_cast<double2*>(o + row(si) * ld + feat(f)) = make_double2(v0, v1);
    };

    double g[4][8];
    if (HC != nullptr && hd) {  // phase block of the sampled batch: cached h1 / h2, one-hot g
#pragma unroll
      for (int si = 0; si < 4; ++si)
        if (row(si) < c1) {
          const double* hr = HC + (static_cast<int64_t>(j) * hc_rows + row(si)) * 128;
#pragma unroll
          for (int f = 0; f < 8; f += 2) {
            const double2 x1 = *reinterpret_cast<const double2*>(hr + feat(f));
            const double2 x2 = *reinterpret_cast<const double2*>(hr + 64 + feat(f));
            put(h1o, si, f, x1.x, x1.y);
            put(h2o, si, f, x2.x, x2.y);
          }
        }
#pragma unroll
      for (int si = 0; si < 4; ++si)
#pragma unroll
        for (int f = 0; f < 8; ++f) g[si][f] = feat(f) == val[si] ? cf[si] : 0.0;
    } else {
    // layer 1 -> h1 (model.cpp:171), as in k_log_psi_part
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      double a[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int si = 2 * p + u;
        const uint64_t* x = sk + (sq * 4 + si) * W;
        const bool ones = 2 * pw[si] <= off;
#pragma unroll
        for (int f = 0; f < 8; ++f) a[u][f] = 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const int lo = 64 * w;
          if (off <= lo) break;
          const uint64_t msk = (off - lo >= 64) ? ~0ull : ((1ull << (off - lo)) - 1);
          uint64_t xm = (ones ? x[w] : ~x[w]) & msk;
          while (xm) {
            const int i = lo + __ffsll(static_cast<long long>(xm)) - 1;
            xm &= xm - 1;
            const double* rw = B + L.w1t() + i * kHid + 2 * hq;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const double2 wv = __ldg(reinterpret_cast<const double2*>(rw + 16 * m));
              a[u][2 * m] += wv.x;
              a[u][2 * m + 1] += wv.y;
            }
          }
        }
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          const double cs = bias[64 + feat(f)];
          a[u][f] = tanh_fast((ones ? 2.0 * a[u][f] - cs : cs - 2.0 * a[u][f]) + bias[feat(f)]);
        }
#pragma unroll
        for (int f = 0; f < 8; f += 2) put(h1o, si, f, a[u][f], a[u][f + 1]);
      }
#pragma unroll
      for (int f = 0; f < 8; ++f)
        *reinterpret_cast<double2*>(act + pidx(feat(f), sq * 4 + 2 * p)) = make_double2(a[0][f], a[1][f]);
    }
    __syncwarp();

    double acc[4][8];
    auto gemm = [&](const double* wm) {
#pragma unroll
      for (int si = 0; si < 4; ++si)
#pragma unroll
        for (int f = 0; f < 8; ++f) acc[si][f] = 0.0;
#pragma unroll 4
      for (int kk = 0; kk < kHid; ++kk) {
        const double2 a01 = *reinterpret_cast<const double2*>(act + pidx(kk, sq * 4));
        const double2 a23 = *reinterpret_cast<const double2*>(act + pidx(kk, sq * 4 + 2));
        const double av[4] = {a01.x, a01.y, a23.x, a23.y};
        double wv[8];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const double2 t = *reinterpret_cast<const double2*>(wm + kk * kHid + 16 * m + 2 * hq);
          wv[2 * m] = t.x;
          wv[2 * m + 1] = t.y;
        }
#pragma unroll
        for (int si = 0; si < 4; ++si)
#pragma unroll
          for (int f = 0; f < 8; ++f) acc[si][f] = fma(av[si], wv[f], acc[si][f]);
      }
    };
    // acc tile -> act (k-major) for the next GEMM
    auto to_act = [&](double (*v)[8]) {
      __syncwarp();
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        *reinterpret_cast<double2*>(act + pidx(feat(f), sq * 4)) = make_double2(v[0][f], v[1][f]);
        *reinterpret_cast<double2*>(act + pidx(feat(f), sq * 4 + 2)) = make_double2(v[2][f], v[3][f]);
      }
      __syncwarp();
    };

    // layer 2: h2 = tanh(W2 h1 + b2 + h1) (model.cpp:172)
    gemm(w2);
    double h2[4][8];
#pragma unroll
    for (int f = 0; f < 8; ++f) {
      const int h = feat(f);
      const double2 r01 = *reinterpret_cast<const double2*>(act + pidx(h, sq * 4));
      const double2 r23 = *reinterpret_cast<const double2*>(act + pidx(h, sq * 4 + 2));
      const double b2 = bias[128 + h];
      h2[0][f] = tanh_fast(acc[0][f] + b2 + r01.x);
      h2[1][f] = tanh_fast(acc[1][f] + b2 + r01.y);
      h2[2][f] = tanh_fast(acc[2][f] + b2 + r23.x);
      h2[3][f] = tanh_fast(acc[3][f] + b2 + r23.y);
    }
#pragma unroll
    for (int si = 0; si < 4; ++si)
#pragma unroll
      for (int f = 0; f < 8; f += 2) put(h2o, si, f, h2[si][f], h2[si][f + 1]);

    // output gradient g (d/d raw output), scaled by the sample's coefficient
    if (hd == 0) {
      // amplitude head: onehot(v) - softmax(2 out) over allowed, minus its mean (model.cpp:288-310)
      to_act(h2);
      gemm(w3);
#pragma unroll
      for (int si = 0; si < 4; ++si) {
        double sum = 0.0;
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          acc[si][f] += bias[192 + feat(f)];
          sum += acc[si][f];
        }
#pragma unroll
        for (int o = 4; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const double mean = sum / static_cast<double>(n_out);
        double mx = -CUDART_INF;
        uint32_t okm = 0;
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          const int v = feat(f);
          acc[si][f] = 2.0 * (acc[si][f] - mean);
          const int w = pw[si] + __popc(v);
          bool a = v < n_out && w <= M.n_e && w + rem_after >= M.n_e;
          if (a && M.spin) {
            const int wu = pu[si] + __popc(static_cast<uint32_t>(v) & up_value_mask);
            const int wd = w - wu;
            const int n_down = M.n_e - M.n_up;
            const int rem_down = rem_after - rem_up_after;
            a = wu <= M.n_up && wu + rem_up_after >= M.n_up && wd <= n_down && wd + rem_down >= n_down;
          }
          if (a) {
            okm |= 1u << f;
            mx = fmax(mx, acc[si][f]);
          }
        }
#pragma unroll
        for (int o = 4; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        double se = 0.0;
        double ex[8];
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          ex[f] = (okm >> f & 1u) ? exp(acc[si][f] - mx) : 0.0;
          se += ex[f];
        }
#pragma unroll
        for (int o = 4; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
        double gs = 0.0;
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          const int v = feat(f);
          g[si][f] = (v == val[si] ? 1.0 : 0.0) - ex[f] / se;
          gs += g[si][f];  // v >= n_out: 0
        }
#pragma unroll
        for (int o = 4; o; o >>= 1) gs += __shfl_xor_sync(0xffffffffu, gs, o);
        const double gm = gs / static_cast<double>(n_out);
#pragma unroll
        for (int f = 0; f < 8; ++f) g[si][f] = feat(f) < n_out ? (g[si][f] - gm) * cf[si] : 0.0;
      }
    } else {
      // phase head: d phase / d raw = onehot(v) (model.cpp:316-320)
#pragma unroll
      for (int si = 0; si < 4; ++si)
#pragma unroll
        for (int f = 0; f < 8; ++f) g[si][f] = feat(f) == val[si] ? cf[si] : 0.0;
    }
    }
#pragma unroll
    for (int si = 0; si < 4; ++si)
#pragma unroll
      for (int f = 0; f < 8; f += 2) put(go, si, f, g[si][f], g[si][f + 1]);
    add_tile_sums(g, (row(0) < c1) | (row(1) < c1) << 1 | (row(2) < c1) << 2 | (row(3) < c1) << 3, bsum + warp * 64,
                  lane);
  }
  write_cta_sums(bsum, GSUM, jh, static_cast<int>(blockIdx.x / n_jh), static_cast<int>(gridDim.x / n_jh));
}

// Backward half (mlp_backward, model.cpp:177-201) of the gradient vectors:
// gz2 = (W3ᵀ g) ⊙ (1 − h2²), gz1 = (W2ᵀ gz2 + gz2) ⊙ (1 − h1²) from the g,
// h1, h2 rows k_grad_fwd wrote; W3 and W2 staged in their original (v, h) /
// (h, k) orientation, the same warp tiling and GEMM as the forward kernels.
template <int W>
__global__ void __launch_bounds__(kG2Threads, 1)
    k_grad_bwd(const ModelView M, const uint64_t* __restrict__ keys, int64_t N, int64_t chunk,
               const double* __restrict__ H1, const double* __restrict__ H2, const double* __restrict__ G,
               double* __restrict__ GZ2, double* __restrict__ GZ1, int64_t N_blk, double* __restrict__ GZ2SUM) {
  extern __shared__ __align__(16) double smem[];
  double* w2o = smem;           // [64 h][64 k]  (W2)
  double* w3o = smem + 4096;    // [64 v][64 h]  (W3)
  double* acts = smem + 8192;   // [warps][64][16]
  double* bsum = acts + kG2Warps * 64 * kWT;  // [warps][64]: Σ gz2 of the warp's tiles (gb2)
  const int n_jh = 2 * M.n_qudits;
  const int jh = static_cast<int>(blockIdx.x % n_jh), hd = jh & 1;
  const int off = (jh >> 1) * M.bits, kb = min(M.bits, M.n - off);
  const int64_t c0 = static_cast<int64_t>(blockIdx.x / n_jh) * chunk;
  const int64_t c1 = min(N, c0 + chunk);
  const BlockLayout L{M.n};
  const double* B = M.P + static_cast<int64_t>(jh) * L.size();
  for (int e = threadIdx.x; e < 4096; e += kG2Threads) {
    const int r = e >> 6, c = e & 63;  // (k, h) -> (h, k)
    w2o[c * 64 + r] = __ldg(B + L.w2t() + e);
    w3o[c * 64 + r] = __ldg(B + L.w3t() + e);
  }
  for (int e = threadIdx.x; e < kG2Warps * 64; e += kG2Threads) bsum[e] = 0.0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sq = lane >> 3, hq = lane & 7;
  double* act = acts + warp * 64 * kWT;
  const int64_t blk = static_cast<int64_t>(jh) * N_blk * 64;
  const double *h1i = H1 + blk, *h2i = H2 + blk, *gi = G + blk;
  double *gz2o = GZ2 + blk, *gz1o = GZ1 + blk;
  auto feat = [&](int f) { return 16 * (f >> 1) + 2 * hq + (f & 1); };
  for (int64_t t0 = c0 + static_cast<int64_t>(warp) * kWT; t0 < c1; t0 += static_cast<int64_t>(kWT) * kG2Warps) {
    auto row = [&](int si) { return t0 + sq * 4 + si; };
    double acc[4][8], v[4][8];
    auto load = [&](const double* src, int ld) {
#pragma unroll
      for (int si = 0; si < 4; ++si)
#pragma unroll
        for (int f = 0; f < 8; f += 2) {
          double2 x = make_double2(0.0, 0.0);
          if (row(si) < c1) x = *reinterpret_cast<const double2*>(src + row(si) * ld + feat(f));
          v[si][f] = x.x;
          v[si][f + 1] = x.y;
        }
    };
    auto to_act = [&]() {
      __syncwarp();
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        *reinterpret_cast<double2*>(act + pidx(feat(f), sq * 4)) = make_double2(v[0][f], v[1][f]);
        *reinterpret_cast<double2*>(act + pidx(feat(f), sq * 4 + 2)) = make_double2(v[2][f], v[3][f]);
      }
      __syncwarp();
    };
    auto gemm = [&](const double* wm) {
#pragma unroll
      for (int si = 0; si < 4; ++si)
#pragma unroll
        for (int f = 0; f < 8; ++f) acc[si][f] = 0.0;
#pragma unroll 4
      for (int kk = 0; kk < kHid; ++kk) {
        const double2 a01 = *reinterpret_cast<const double2*>(act + pidx(kk, sq * 4));
        const double2 a23 = *reinterpret_cast<const double2*>(act + pidx(kk, sq * 4 + 2));
        const double av[4] = {a01.x, a01.y, a23.x, a23.y};
        double wv[8];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const double2 t = *reinterpret_cast<const double2*>(wm + kk * kHid + 16 * m + 2 * hq);
          wv[2 * m] = t.x;
          wv[2 * m + 1] = t.y;
        }
#pragma unroll
        for (int si = 0; si < 4; ++si)
#pragma unroll
          for (int f = 0; f < 8; ++f) acc[si][f] = fma(av[si], wv[f], acc[si][f]);
      }
    };
    if (hd) {  // phase head: g = coefficient * onehot(v), so W3ᵀ g = g[v] * row v of W3
#pragma unroll
      for (int si = 0; si < 4; ++si) {
        int val = 0;
        double gv = 0.0;
        if (row(si) < c1) {  // the sampled value of this qudit (extract_bits, basis_vector.cpp:40-45)
          const uint64_t* x = keys + row(si) * W;
          const int wq = off >> 6, bq = off & 63;
          uint64_t fld = __ldg(x + wq) >> bq;
          if (bq + kb > 64 && wq + 1 < W) fld |= __ldg(x + wq + 1) << (64 - bq);
          val = static_cast<int>(__brev(static_cast<uint32_t>(fld)) >> (32 - kb));
          gv = gi[row(si) * 64 + val];
        }
#pragma unroll
        for (int f = 0; f < 8; ++f) acc[si][f] = gv * w3o[val * 64 + feat(f)];
      }
    } else {
      load(gi, 64);  // g -> act
      to_act();
      gemm(w3o);     // W3ᵀ g
    }
    load(h2i, 64);
#pragma unroll
    for (int si = 0; si < 4; ++si)
#pragma unroll
      for (int f = 0; f < 8; ++f) v[si][f] = acc[si][f] * (1.0 - v[si][f] * v[si][f]);  // gz2
#pragma unroll
    for (int si = 0; si < 4; ++si)
      if (row(si) < c1)
#pragma unroll
        for (int f = 0; f < 8; f += 2)
          *reinterpret_cast<double2*>(gz2o + row(si) * 64 + feat(f)) = make_double2(v[si][f], v[si][f + 1]);
    add_tile_sums(v, (row(0) < c1) | (row(1) < c1) << 1 | (row(2) < c1) << 2 | (row(3) < c1) << 3, bsum + warp * 64,
                  lane);
    to_act();
    gemm(w2o);     // W2ᵀ gz2; v still holds gz2 (the residual)
#pragma unroll
    for (int si = 0; si < 4; ++si)
#pragma unroll
      for (int f = 0; f < 8; ++f) acc[si][f] += v[si][f];
    load(h1i, 64);
#pragma unroll
    for (int si = 0; si < 4; ++si)
      if (row(si) < c1)
#pragma unroll
        for (int f = 0; f < 8; f += 2)
          *reinterpret_cast<double2*>(gz1o + row(si) * 64 + feat(f)) =
              make_double2(acc[si][f] * (1.0 - v[si][f] * v[si][f]), acc[si][f + 1] * (1.0 - v[si][f + 1] * v[si][f + 1]));
  }
  write_cta_sums(bsum, GZ2SUM, jh, static_cast<int>(blockIdx.x / n_jh), static_cast<int>(gridDim.x / n_jh));
}

// bias rows of the W2 / W3 split-K partials (row 64 of every output column, ld kHS):
// part 0 gets the CTA sums of this chunk in CTA order, the other parts 0 (the
// GEMMs write rows 0-63 only); row 65 is the zero pad
__global__ void k_bias_rows(const double* __restrict__ sums, int nb, int n_cta, int parts, int64_t len,
                            double* __restrict__ part) {
  const int total = nb * parts * 64;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int o = e & 63, bq = e >> 6, jh = bq / parts, q = bq - jh * parts;
    double t = 0.0;
    if (q == 0)
      for (int c = 0; c < n_cta; ++c) t += sums[(static_cast<int64_t>(jh) * n_cta + c) * 64 + o];
    double* col = part + static_cast<int64_t>(bq) * len + static_cast<int64_t>(o) * kHS;
    col[64] = t;
    col[65] = 0.0;
  }
}

// ±1 encoding of every qubit of a chunk's keys: X[s][i] (model.cpp:153-158
// before the prefix cut; gW1 of qudit j keeps only columns i < offset_j)
// row stride n + 2: column n is a constant 1 (the gW1 GEMM then also yields gb1), n + 1 a zero pad
template <int W>
__global__ void k_pm_bits(const uint64_t* __restrict__ keys, int64_t N, int n, double* __restrict__ X) {
  const int ld = n + 2;
  const int64_t total = N * ld;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = e / ld;
    const int i = static_cast<int>(e - s * ld);
    X[e] = i == n ? 1.0 : i > n ? 0.0 : ((__ldg(keys + s * W + (i >> 6)) >> (i & 63)) & 1ull ? 1.0 : -1.0);
  }
}

// split-K partial sums [nb][parts][len] -> acc [nb][len] in part order (deterministic); first = overwrite
__global__ void k_sum_parts(const double* __restrict__ part, int nb, int parts, int64_t len, int first,
                            double* __restrict__ acc) {
  const int64_t total = static_cast<int64_t>(nb) * len;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t jh = e / len, t = e - jh * len;
    double sum = 0.0;
    for (int q = 0; q < parts; ++q) sum += part[(jh * parts + q) * len + t];
    acc[e] = first ? sum : acc[e] + sum;
  }
}

// per-sample coefficients (2 Re c_i, 2 Im c_i), c_i = w_i (E_i − Ē) (energy.cpp:84-88)
__global__ void k_grad_coef(const double* __restrict__ w, const double2* __restrict__ loc, int64_t N,
                            const double2* __restrict__ mean, double2* __restrict__ coef) {
  const double2 m = *mean;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double2 e = loc[i];
    coef[i] = make_double2(2.0 * w[i] * (e.x - m.x), 2.0 * w[i] * (e.y - m.y));
  }
}

// Ē = Σ_i w_i E_i, fixed grid + fixed merge order (deterministic)
__global__ void __launch_bounds__(256) k_wmean_partial(const double* __restrict__ w, const double2* __restrict__ loc,
                                                       int64_t N, double2* __restrict__ part) {
  __shared__ double2 red[256];
  double2 s = make_double2(0.0, 0.0);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * 256) {
    s.x += w[i] * loc[i].x;
    s.y += w[i] * loc[i].y;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) {
      red[threadIdx.x].x += red[threadIdx.x + o].x;
      red[threadIdx.x].y += red[threadIdx.x + o].y;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_wmean_final(const double2* __restrict__ part, int nb, double2* __restrict__ out) {
  if (threadIdx.x) return;
  double2 s = make_double2(0.0, 0.0);
  for (int b = 0; b < nb; ++b) {
    s.x += part[b].x;
    s.y += part[b].y;
  }
  *out = s;
}

// accumulated block sums -> the reference's flat parameter layout (model.cpp:65-80)
//   gw1 [jh][64 h][n] (columns >= offset zeroed), gw2 [jh][64 h][64 k], gw3 [jh][64 v][64 h], gb [jh][3][64]
//   acc1 [jh][64 h][n + 2] (column n = gb1), acc2 [jh][64 h][66] (row... column 64 = gb2),
//   acc3 [jh][64 v][66] (column 64 = gb3)
__global__ void k_grad_scatter(const ModelView M, const double* __restrict__ gw1, const double* __restrict__ gw2,
                               const double* __restrict__ gw3, double* __restrict__ out) {
  const int jh = blockIdx.x, j = jh >> 1;
  const int n = M.n, off = j * M.bits, k = min(M.bits, n - off), n_out = 1 << k;
  int64_t base = 0;  // flat offset of block jh
  for (int q = 0; q < jh; ++q) {
    const int kq = min(M.bits, n - (q >> 1) * M.bits);
    base += static_cast<int64_t>(kHid) * n + kHid + kHid * kHid + kHid + (1 << kq) * kHid + (1 << kq);
  }
  double* o = out + base;
  const int nx = n + 2;
  const double* a1 = gw1 + static_cast<int64_t>(jh) * kHid * nx;
  const double* a2 = gw2 + static_cast<int64_t>(jh) * kHid * kHS;
  const double* a3 = gw3 + static_cast<int64_t>(jh) * kHid * kHS;
  for (int e = threadIdx.x; e < kHid * n; e += blockDim.x) {
    const int h = e / n, i = e - h * n;
    o[e] = i < off ? a1[h * nx + i] : 0.0;
  }
  o += kHid * n;
  for (int e = threadIdx.x; e < kHid; e += blockDim.x) o[e] = a1[e * nx + n];
  o += kHid;
  for (int e = threadIdx.x; e < kHid * kHid; e += blockDim.x) o[e] = a2[(e >> 6) * kHS + (e & 63)];
  o += kHid * kHid;
  for (int e = threadIdx.x; e < kHid; e += blockDim.x) o[e] = a2[e * kHS + 64];
  o += kHid;
  for (int e = threadIdx.x; e < n_out * kHid; e += blockDim.x) o[e] = a3[(e >> 6) * kHS + (e & 63)];
  o += n_out * kHid;
  for (int e = threadIdx.x; e < n_out; e += blockDim.x) o[e] = a3[e * kHS + 64];
}

// Jacobian rows of selected samples (grad_log_psi, model.cpp:273-325) from
// the gradient kernels' buffers run with coefficients (1, 1): R[i][t] = d log|ψ| / dθ_t
// for amplitude-block parameters and d φ / dθ_t for phase-block ones (the
// complex row is R on the amplitude blocks and -i R on the phase blocks).
// Block jh of the flat layout starts at boff[jh]. One CTA per (row, block).
__global__ void k_jac_real(const ModelView M, const int64_t* __restrict__ boff, int64_t N, const double* __restrict__ H1,
                           const double* __restrict__ H2, const double* __restrict__ G, const double* __restrict__ GZ2,
                           const double* __restrict__ GZ1, const double* __restrict__ X, int64_t ld,
                           double* __restrict__ R) {
  const int64_t i = blockIdx.x;
  const int jh = blockIdx.y, j = jh >> 1;
  const int n = M.n, off = j * M.bits, k = min(M.bits, n - off), n_out = 1 << k;
  const int64_t v0 = (static_cast<int64_t>(jh) * N + i) * 64;
  const double *h1 = H1 + v0, *h2 = H2 + v0, *g = G + v0, *gz2 = GZ2 + v0, *gz1 = GZ1 + v0, *x = X + i * (n + 2);
  double* o = R + i * ld + boff[jh];
  for (int e = threadIdx.x; e < kHid * n; e += blockDim.x) {  // W1[h][c] = gz1[h] e[c], e = ±1 before the offset
    const int h = e / n, c = e - h * n;
    o[e] = c < off ? gz1[h] * x[c] : 0.0;
  }
  o += kHid * n;
  for (int e = threadIdx.x; e < kHid; e += blockDim.x) o[e] = gz1[e];
  o += kHid;
  for (int e = threadIdx.x; e < kHid * kHid; e += blockDim.x) o[e] = gz2[e >> 6] * h1[e & 63];
  o += kHid * kHid;
  for (int e = threadIdx.x; e < kHid; e += blockDim.x) o[e] = gz2[e];
  o += kHid;
  for (int e = threadIdx.x; e < n_out * kHid; e += blockDim.x) o[e] = g[e >> 6] * h2[e & 63];
  o += n_out * kHid;
  for (int e = threadIdx.x; e < n_out; e += blockDim.x) o[e] = g[e];
}

// build_sr_context (sr.cpp:25-72) rows: stacked[i] = Re(sqrt(w_i)(row_i - mean)),
// stacked[n+i] = Im(...). The row is real on the amplitude blocks and -i R on
// the phase blocks, so stacked[i] holds only amplitude columns and
// stacked[n+i] only phase columns (negated). One CTA per (row, block).
__global__ void k_sr_stack(const ModelView M, const int64_t* __restrict__ boff, int64_t n_sr,
                           const double* __restrict__ R, const double* __restrict__ mean,
                           const double* __restrict__ sw, int64_t ld, double* __restrict__ S) {
  const int64_t i = blockIdx.x;
  const int jh = blockIdx.y, hd = jh & 1;
  const int64_t b0 = boff[jh], b1 = boff[jh + 1];
  const double si = sw[i];
  double* re = S + i * ld;
  double* im = S + (n_sr + i) * ld;
  for (int64_t t = b0 + threadIdx.x; t < b1; t += blockDim.x) {
    const double c = si * (R[i * ld + t] - mean[t]);
    re[t] = hd ? 0.0 : c;
    im[t] = hd ? -c : 0.0;
  }
}

// adam_step (optimizer.cpp:17-31) on the device-resident flat parameters;
// c1, c2 = bias corrections of this step. A non-finite direction entry sets *bad
// and leaves everything unchanged (the reference throws before updating).
__global__ void k_adam_check(const double* __restrict__ d, int64_t n, int* __restrict__ bad) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (!isfinite(d[i])) atomicOr(bad, 1);
}

__global__ void k_adam(const double* __restrict__ d, int64_t n, double lr, double b1, double b2, double eps, double c1,
                       double c2, const int* __restrict__ bad, double* __restrict__ m, double* __restrict__ v,
                       double* __restrict__ theta) {
  if (*bad) return;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double g = d[i];
    const double mi = b1 * m[i] + (1.0 - b1) * g;
    const double vi = b2 * v[i] + (1.0 - b2) * (g * g);
    m[i] = mi;
    v[i] = vi;
    theta[i] -= lr * (mi / c1) / (sqrt(vi / c2) + eps);
  }
}

// set_params on the device: the flat layout (model.cpp:65-80) -> the kernels'
// block layout (BlockLayout: W1ᵀ, prefix column sums, W2ᵀ, W3ᵀ zero-padded),
// the same arithmetic as the host re-layout (column sums in i order). One CTA per block.
__global__ void k_params_relayout(const ModelView M, const int64_t* __restrict__ boff, const double* __restrict__ theta,
                                  double* __restrict__ P) {
  const int jh = blockIdx.x, j = jh >> 1;
  const int n = M.n, off = j * M.bits, k = min(M.bits, n - off), n_out = 1 << k;
  const BlockLayout L{n};
  const double* w1 = theta + boff[jh];
  const double* b1 = w1 + kHid * n;
  const double* w2 = b1 + kHid;
  const double* b2 = w2 + kHid * kHid;
  const double* w3 = b2 + kHid;
  const double* b3 = w3 + n_out * kHid;
  double* B = P + static_cast<int64_t>(jh) * L.size();
  for (int e = threadIdx.x; e < kHid * n; e += blockDim.x) {
    const int h = e / n, i = e - h * n;
    B[L.w1t() + i * kHid + h] = w1[e];
  }
  for (int h = threadIdx.x; h < kHid; h += blockDim.x) {
    double c = 0.0;
    for (int i = 0; i < off; ++i) c += w1[h * n + i];
    B[L.csum() + h] = c;
    B[L.b1() + h] = b1[h];
    B[L.b2() + h] = b2[h];
    B[L.b3() + h] = h < n_out ? b3[h] : 0.0;
  }
  for (int e = threadIdx.x; e < kHid * kHid; e += blockDim.x) {
    const int h = e >> 6, kk = e & 63;
    B[L.w2t() + kk * kHid + h] = w2[e];
    const int v = e >> 6;  // W3[v][kk]
    B[L.w3t() + kk * kHid + v] = v < n_out ? w3[v * kHid + kk] : 0.0;
  }
}

// log ψ = Σ_j log_amp_j[v_j], φ = Σ_j phase_j[v_j] in qudit order; masked
// states (-inf, 0) (model.cpp:254-271)
template <int W>
__global__ void k_sum_qudits(const ModelView M, const uint64_t* __restrict__ keys, int64_t N,
                             const double* __restrict__ part, double* __restrict__ out_la,
                             double* __restrict__ out_ph) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= N) return;
  int pc = 0, pe = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const uint64_t x = __ldg(keys + s * W + w);
    pc += __popcll(x);
    pe += __popcll(x & 0x5555555555555555ull);
  }
  double la = 0.0, ph = 0.0;
  for (int j = 0; j < M.n_qudits; ++j) {
    la += __ldcs(part + static_cast<int64_t>(2 * j) * N + s);
    ph += __ldcs(part + static_cast<int64_t>(2 * j + 1) * N + s);
  }
  const bool ins = pc == M.n_e && (!M.spin || pe == M.n_up);
  out_la[s] = ins ? la : -CUDART_INF;
  out_ph[s] = ins ? ph : 0.0;
}

// fill_amplitudes of a batch qvmc_cuda_sample just produced with the current
// parameters: the sampler accumulated log p = Σ_j c_j in qudit order from the
// same amplitude-head arithmetic whose halves 0.5 c_j k_sum_qudits would add in
// that order, so log|ψ| = 0.5 log p exactly (scaling by 2^-1 commutes with the
// rounded sums); φ from the phase heads as in k_sum_qudits
template <int W>
__global__ void k_sum_phases(const ModelView M, const uint64_t* __restrict__ keys, int64_t N,
                             const double* __restrict__ part, const double* __restrict__ lp,
                             double* __restrict__ out_la, double* __restrict__ out_ph) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= N) return;
  int pc = 0, pe = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const uint64_t x = __ldg(keys + s * W + w);
    pc += __popcll(x);
    pe += __popcll(x & 0x5555555555555555ull);
  }
  double ph = 0.0;
  for (int j = 0; j < M.n_qudits; ++j) ph += __ldcs(part + static_cast<int64_t>(2 * j + 1) * N + s);
  const bool ins = pc == M.n_e && (!M.spin || pe == M.n_up);
  out_la[s] = ins ? 0.5 * lp[s] : -CUDART_INF;
  out_ph[s] = ins ? ph : 0.0;
}

// order-independent fingerprint of a batch (keys, log p): wrapping sum of mixed
// (index, words, bits) per sample, for recognising the sampler's own output
template <int W>
__global__ void k_fingerprint(const uint64_t* __restrict__ keys, const double* __restrict__ lp, int64_t N,
                              unsigned long long* __restrict__ out) {
  unsigned long long acc = 0;
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < N;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t z = static_cast<uint64_t>(s) * 0x9E3779B97F4A7C15ull ^
                 (lp ? static_cast<uint64_t>(__double_as_longlong(lp[s])) : 0ull);  // lp null: keys only
#pragma unroll
    for (int w = 0; w < W; ++w) {
      z ^= keys[s * W + w] + 0x632BE59BD9B4E019ull * (w + 1);
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
    }
    acc += z;
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
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
