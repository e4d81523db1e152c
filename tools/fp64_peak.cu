// FP64 roofline probe: DMMA (mma.sync f64 -> DMMA.8x8x4) and DFMA issue rates,
// measured with CUDA events. Used once to pin the FP64 denominator that
// MEASURED_PEAKS.json does not carry (roofline section).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double d[4][4] = {};
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, b0 = a0 * 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(d[r][0]), "+d"(d[r][1]), "+d"(d[r][2]), "+d"(d[r][3]) : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0;
  for (int r = 0; r < 4; ++r) s += d[r][0] + d[r][1] + d[r][2] + d[r][3];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  const double a = 0.999999, b = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    dim3 grid(sms * 2), block(32 * warps / 2);
    dmma_loop<<<grid, block>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<grid, block>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // m16n8k4 = 16*8*4 FMA = 1024 flop per warp-instruction, 4 per iter
    double flops = double(grid.x) * (block.x / 32) * iters * 4 * 16 * 8 * 4 * 2.0;
    printf("{\"probe\": \"dmma_m16n8k4\", \"warps_per_sm\": %d, \"tflops\": %.2f}\n", warps, flops / ms / 1e9);
  }
  for (int warps : {8, 16, 32}) {
    dim3 grid(sms * 2), block(32 * warps / 2);
    dfma_loop<<<grid, block>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<grid, block>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = double(grid.x) * block.x * iters * 8 * 2.0;
    printf("{\"probe\": \"dfma\", \"warps_per_sm\": %d, \"tflops\": %.2f}\n", warps, flops / ms / 1e9);
  }
  return 0;
}
