// Integer-pipe rates and load latencies of the B200 SM (CC 10.0), measured on
// the box: the peaks the search kernel's roofline is taken against (SURVEY.md
// §8d asks for them; the CC 9.0 table is not a B200 measurement).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o int_rates int_rates.cu
//   ./int_rates > profiles/int_rates_b200.json
//
// Throughput kernels: every thread runs 8 independent dependency chains of
// one instruction (inline PTX so SASS is exactly that opcode; checked with
// cuobjdump -sass), 32 warps per SM, all SMs. Rate = warp instructions per
// SM-clock (clock64 brackets per CTA, CTAs resident together). "issue" mixes
// an alu-pipe op (LOP3) with an fma-pipe op (IMAD) so both pipes fill: the
// per-SM instruction issue ceiling (4 schedulers x 1 warp-inst/clk).
//
// Latency kernels: one thread chases a random pointer cycle; ns per hop
// from clock64 / SM clock. L2: a 32 MiB cycle (L2-resident after a warm
// pass, L1 bypassed with ld.global.cg); HBM: a 2 GiB cycle.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

enum Op { kLop3 = 0, kIadd3 = 1, kPopc = 2, kShf = 3, kImad = 4, kIssue = 5, kFlo = 6 };

constexpr int kIters = 65536;
constexpr int kChains = 8;

template <int OP>
__device__ __forceinline__ uint32_t step(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  if (OP == kLop3) {
    asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  } else if (OP == kIadd3) {
    asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  } else if (OP == kPopc) {
    asm volatile("popc.b32 %0, %1;" : "=r"(r) : "r"(a));
  } else if (OP == kShf) {
    asm volatile("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  } else if (OP == kImad) {
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  } else if (OP == kFlo) {
    asm volatile("bfind.u32 %0, %1;" : "=r"(r) : "r"(a));
  }
  return r;
}

template <int OP>
__global__ void __launch_bounds__(1024) k_rate(uint32_t seed, uint32_t* sink, unsigned long long* cycles) {
  uint32_t x[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) x[k] = seed * (threadIdx.x + 1 + k) ^ (k * 0x9e3779b9u);
  const uint32_t b = seed | 1u, c = seed >> 3;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) {
      if (OP == kIssue) {  // alu + fma pipes interleaved
        if (k & 1) x[k] = step<kImad>(x[k], b, c);
        else x[k] = step<kLop3>(x[k], b, c);
      } else {
        x[k] = step<OP>(x[k], b, c);
      }
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s ^= x[k];
  if (s == 0x12345678u) sink[blockIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

__global__ void k_chase(const uint64_t* __restrict__ next, uint64_t start, int hops, uint64_t* out,
                        unsigned long long* cycles) {
  uint64_t p = start;
  for (int i = 0; i < 1024; ++i) {  // warm (L2 case) / TLB
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(p) : "l"(next + p));
  }
  const unsigned long long t0 = clock64();
  for (int i = 0; i < hops; ++i) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(p) : "l"(next + p));
  const unsigned long long t1 = clock64();
  out[0] = p;
  cycles[0] = t1 - t0;
}

__global__ void k_touch(const uint64_t* __restrict__ a, size_t n, uint64_t* out) {
  uint64_t s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    s += __ldcg(a + i);
  if (s == 42) out[0] = s;
}

template <int OP>
int run_rate(const char* name, int sms, int threads, int ctas_per_sm, double clk_mhz, bool last) {
  const int grid = sms * ctas_per_sm;
  uint32_t* sink;
  unsigned long long* cyc;
  CK(cudaMalloc(&sink, grid * 4));
  CK(cudaMalloc(&cyc, grid * 8));
  k_rate<OP><<<grid, threads>>>(12345u, sink, cyc);  // warm
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_rate<OP><<<grid, threads>>>(12345u, sink, cyc);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> c(grid);
  CK(cudaMemcpy(c.data(), cyc, grid * 8, cudaMemcpyDeviceToHost));
  const double cmax = static_cast<double>(*std::max_element(c.begin(), c.end()));
  const double cmed = [&] { auto v = c; std::nth_element(v.begin(), v.begin() + grid / 2, v.end()); return (double)v[grid / 2]; }();
  const int insts_per_op = OP == kIadd3 ? 2 : 1;  // ptxas fuses two dependent adds into one IADD3 (SASS-checked)
  const double warp_inst_per_cta = (double)kIters * kChains * (threads / 32) / insts_per_op;
  // CTAs of one SM run concurrently: per-SM rate = ctas_per_sm * per-CTA instructions / CTA cycles
  // chip rate from the CUDA events around the launch (all CTAs, launch overhead included: a lower bound);
  // per-SM per-clock = chip rate / SMs / SM clock, with the clock implied by the slowest CTA's clock64 span
  const double per_s_chip_event = warp_inst_per_cta * grid / (ms * 1e-3);
  const double implied_mhz = cmax / (ms * 1e3);
  const double per_clk_sm = per_s_chip_event / sms / (implied_mhz * 1e6);
  const double per_clk_sm_attr = per_s_chip_event / sms / (clk_mhz * 1e6);
  std::printf("  \"%s\": {\"warp_inst_per_clk_per_sm\": %.4f, \"warp_inst_per_clk_per_sm_at_attr_clock\": %.4f, "
              "\"lane_ops_per_clk_per_sm\": %.2f, \"warp_inst_per_s_chip\": %.5e, \"lane_ops_per_s_chip\": %.5e, "
              "\"implied_clock_mhz\": %.1f, \"cycles_median\": %.0f, \"cycles_max\": %.0f, \"ms\": %.4f}%s\n",
              name, per_clk_sm, per_clk_sm_attr, 32 * per_clk_sm, per_s_chip_event, 32 * per_s_chip_event,
              implied_mhz, cmed, cmax, ms, last ? "" : ",");
  cudaFree(sink);
  cudaFree(cyc);
  return 0;
}

int chase(const char* name, size_t bytes, int hops, double clk_mhz, bool last) {
  const size_t n = bytes / 8;
  std::vector<uint64_t> perm(n);
  std::iota(perm.begin(), perm.end(), 0);
  // one random cycle over 128-byte-spaced slots (distinct lines)
  const size_t stride = 16;
  const size_t m = n / stride;
  std::vector<uint64_t> order(m);
  std::iota(order.begin(), order.end(), 0);
  std::mt19937_64 rng(7);
  std::shuffle(order.begin(), order.end(), rng);
  std::vector<uint64_t> next(n, 0);
  for (size_t i = 0; i < m; ++i) next[order[i] * stride] = order[(i + 1) % m] * stride;
  uint64_t *d, *out;
  unsigned long long* cyc;
  CK(cudaMalloc(&d, bytes));
  CK(cudaMalloc(&out, 8));
  CK(cudaMalloc(&cyc, 8));
  CK(cudaMemcpy(d, next.data(), bytes, cudaMemcpyHostToDevice));
  if (bytes <= (64ull << 20)) {
    k_touch<<<1184, 256>>>(d, n, out);
    k_touch<<<1184, 256>>>(d, n, out);
  }
  k_chase<<<1, 1>>>(d, order[0] * stride, hops, out, cyc);
  CK(cudaDeviceSynchronize());
  unsigned long long c = 0;
  CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
  const double cyc_per = (double)c / hops;
  std::printf("  \"%s\": {\"bytes\": %zu, \"cycles_per_hop\": %.1f, \"ns_per_hop_at_clock\": %.1f}%s\n", name, bytes,
              cyc_per, cyc_per / clk_mhz * 1e3, last ? "" : ",");
  cudaFree(d);
  cudaFree(out);
  cudaFree(cyc);
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double clk_mhz = clk_khz / 1e3;
  const int sms = p.multiProcessorCount;
  std::printf("{\n  \"gpu\": \"%s\", \"sm_count\": %d, \"cc\": \"%d.%d\", \"attr_clock_mhz\": %.0f,\n", p.name, sms,
              p.major, p.minor, clk_mhz);
  std::printf("  \"method\": \"8 independent chains/thread of one inline-PTX op (SASS-checked), 4 CTAs x 256 "
              "threads per SM, 65536 iterations; chip rate = warp instructions / CUDA-event time of the launch; per SM "
              "clock = chip rate / SMs / clock implied by the longest CTA clock64 span\",\n");
  int rc = 0;
  rc |= run_rate<kLop3>("lop3", sms, 256, 4, clk_mhz, false);
  rc |= run_rate<kIadd3>("iadd3", sms, 256, 4, clk_mhz, false);
  rc |= run_rate<kShf>("shf", sms, 256, 4, clk_mhz, false);
  rc |= run_rate<kPopc>("popc", sms, 256, 4, clk_mhz, false);
  rc |= run_rate<kFlo>("flo", sms, 256, 4, clk_mhz, false);
  rc |= run_rate<kImad>("imad", sms, 256, 4, clk_mhz, false);
  rc |= run_rate<kIssue>("issue_lop3_imad", sms, 256, 4, clk_mhz, false);
  rc |= chase("latency_l2_32MiB", 32ull << 20, 20000, clk_mhz, false);
  rc |= chase("latency_hbm_2GiB", 2ull << 30, 20000, clk_mhz, true);
  std::printf("}\n");
  return rc;
}
