// FP64 latency probe (B200): dependent-chain cycles of DFMA, DADD, 64-bit
// warp shuffle, DMMA m8n8k4, LDS, named barrier.  nvcc -arch sm_100a -O3
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x, int n) {
  __shared__ double sh[1024];
  sh[threadIdx.x] = threadIdx.x * 0.5;
  __syncthreads();
  double a = x + threadIdx.x, b = 1.0000001, c = 1e-9;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = a + c;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / n;
  // shfl 64 chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_down_sync(0xffffffffu, a, 1) + c;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / n;
  // dmma chain
  double d0 = a, d1 = c;
  t0 = clock64();
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1) : "d"(b), "d"(c));
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / n;
  // LDS chain (pointer chase through index)
  int idx = threadIdx.x & 31;
  t0 = clock64();
  for (int i = 0; i < n; ++i) idx = static_cast<int>(sh[idx]) & 511;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / n;
  // named barrier round (all threads)
  t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("bar.sync 3, %0;" ::"r"(blockDim.x) : "memory");
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / n;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = a * b;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0) / n;
  out[threadIdx.x] = a + d0 + d1 + idx;
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 8192);
  cudaMalloc(&c, 64);
  long long h[8];
  for (int bs : {32, 512}) {
    k<<<1, bs>>>(o, c, 1.0, 4096);
    cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    printf("block %d: dfma %lld dadd %lld shfl64+dadd %lld dmma %lld lds %lld bar %lld dmul %lld cycles\n", bs, h[0], h[1],
           h[2], h[3], h[4], h[5], h[6]);
  }
  return 0;
}
