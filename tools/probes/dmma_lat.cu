// DMMA m8n8k4 f64 latency and per-SM throughput probe (dependent chain vs independent chains).
#include <cstdio>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, long long* cyc, int iters) {
  double d[CH][2];
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-3;
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CH>
void run(int warps, int blocks) {
  double* o; long long* c; cudaMalloc(&o, 8 << 20); cudaMalloc(&c, 8 * 1024);
  int it = 4096;
  k<CH><<<blocks, 32 * warps>>>(o, c, it);
  k<CH><<<blocks, 32 * warps>>>(o, c, it);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double per = double(h) / it;
  printf("chains=%d warps/CTA=%2d blocks=%3d: %.1f cyc per iteration -> %.1f cyc per DMMA per warp, SM rate %.2f cyc/DMMA\n",
         CH, warps, blocks, per, per / CH, per / (CH * warps) * (blocks > 148 ? 1.0 : 1.0));
  cudaFree(o); cudaFree(c);
}
int main() {
  run<1>(1, 1); run<2>(1, 1); run<4>(1, 1); run<8>(1, 1);
  run<1>(4, 1); run<4>(4, 1); run<1>(8, 1); run<4>(8, 1); run<4>(16, 1); run<8>(16, 1);
  return 0;
}
