// FP64 throughput probe on the B200 (sm_100a): the two FP64 pipes the solver
// uses.
//   * DMMA: mma.sync.aligned.m8n8k4.row.col.f64 (the tensor-pipe FP64 MMA;
//     there is no tcgen05 kind for f64), 2*8*8*4 = 512 flop per warp-instruction;
//   * DFMA: fma.rn.f64 on the CUDA cores, 2 flop per thread-instruction.
// Each warp runs 8 independent accumulator chains so the pipe, not the
// dependency latency, is the limit; grid = 148 SMs x 8 CTAs x 256 threads.
// Prints one JSON line; nvcc -gencode arch=compute_100a,code=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

__global__ void __launch_bounds__(256) k_dmma(double* out, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5 + threadIdx.x * 1e-10;
  double c[kChains][2];
#pragma unroll
  for (int k = 0; k < kChains; ++k) c[k][0] = c[k][1] = 0.0;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < kChains; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[threadIdx.x] = s;  // keep the work alive
}

__global__ void __launch_bounds__(256) k_dfma(double* out, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
  double c[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) c[k] = k * 1e-3;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) c[k] = fma(c[k], b, a);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += c[k];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <class K>
static double time_kernel(K kern, double flop_per_thread_iter, int grid, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<grid, 256>>>(out, 1.0);  // warm-up
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) kern<<<grid, 256>>>(out, 1.0 + r);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = flop_per_thread_iter * kIters * kChains * 256.0 * grid * reps;
  return flop / (ms * 1e-3) / 1e12;
}

int main() {
  int sms = 0, mhz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 256 * sizeof(double));
  const int grid = sms * 8;
  // DMMA: 512 flop per warp-instruction = 16 per thread per instruction
  const double dmma = time_kernel(k_dmma, 16.0, grid, out);
  const double dfma = time_kernel(k_dfma, 2.0, grid, out);
  const cudaError_t e = cudaDeviceSynchronize();
  printf("{\"dmma_tflops\": %.3f, \"dfma_tflops\": %.3f, \"sms\": %d, \"clock_mhz\": %d, \"status\": \"%s\", "
         "\"how\": \"tools/probes/fp64_peak.cu: %d CTAs x 256 threads, 8 independent chains per thread, "
         "%d iterations, 5 timed launches (CUDA events)\"}\n",
         dmma, dfma, sms, mhz / 1000, cudaGetErrorString(e), grid, kIters);
  return e == cudaSuccess ? 0 : 1;
}
