// Probe: FP64 DFMA peak and HBM copy bandwidth on the B200 box (roofline denominators
// for the FP64-bound element kernel; HBM peak comes from MEASURED_PEAKS.json).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-7, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void copyk(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096; float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); dfma_loop<<<sms * 8, 256>>>(out, iters, 0.999999, 1e-9); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * 8 * (double)iters * sms * 8 * 256;
  printf("{\"fp64_dfma_tflops\": %.2f, ", flops / best / 1e9);
  size_t n = (size_t)1 << 27;  // 4 GiB per buffer
  double4 *a, *b; cudaMalloc(&a, n * sizeof(double4)); cudaMalloc(&b, n * sizeof(double4));
  cudaMemset(a, 0, n * sizeof(double4)); best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); copyk<<<sms * 16, 256>>>(a, b, n); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("\"copy_gbs\": %.1f, \"sms\": %d}\n", 2.0 * n * sizeof(double4) / best / 1e6, sms);
  return 0;
}
