// fp64 issue-rate microbenchmark on the B200: DFMA vs DMMA (mma.sync m8n8k4 f64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_rates fp64_rates.cu && ./fp64_rates
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
  double a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-9 + i;
  const double b = 1.0000001, c = 1e-7;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmma(double* out, int iters) {
  double acc[8][2];
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-9;
  const double a = 1.0000001 + threadIdx.x * 1e-12, b = 0.9999999;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// even warps DFMA, odd warps DMMA in the same CTAs: do the two share one pipe?
__global__ void k_mixed(double* out, int iters) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp & 1) {
    double acc[8][2];
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-9;
    const double a = 1.0000001 + threadIdx.x * 1e-12, b = 0.9999999;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  } else {
    double a[16];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-9 + i;
    const double b = 1.0000001, c = 1e-7;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
    for (int i = 0; i < 16; ++i) s += a[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps = 8; warps <= 32; warps *= 2) {
    const int blocks = sms * 2, threads = warps * 16;  // warps per SM = 2 blocks x threads/32
    float ms;
    k_dfma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double f1 = 2.0 * 16 * iters * double(blocks) * threads / (ms * 1e-3) / 1e12;
    k_dmma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double f2 = 2.0 * 256 * 8 * iters * double(blocks) * (threads / 32) / (ms * 1e-3) / 1e12;
    k_mixed<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0);
    k_mixed<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms3;
    cudaEventElapsedTime(&ms3, e0, e1);
    // half the warps do DFMA work (16 FMA per thread-iteration), half DMMA (8 x 256 per warp-iteration)
    const double fm = (2.0 * 16 * iters * double(blocks) * threads / 2 +
                       2.0 * 256 * 8 * iters * double(blocks) * (threads / 64)) / (ms3 * 1e-3) / 1e12;
    printf("warps/SM %2d: DFMA %.1f TFLOP/s, DMMA m8n8k4 %.1f TFLOP/s, half/half mixed %.1f TFLOP/s (%s)\n",
           warps, f1, f2, fm, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
