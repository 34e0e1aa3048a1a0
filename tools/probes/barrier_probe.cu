// Grid-barrier latency probe (B200): cycles per barrier round for the flag,
// atomic and neighbour-only schemes used by k_gauss_path, with and without
// per-round slab stores.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_release(unsigned* a, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* a) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

// mode 0: flag barrier, all CTAs polled by warp 0 (release store / acquire polls)
// mode 1: atomic counter barrier (one thread)
// mode 2: neighbour flags only (|r - s| <= 3)
// mode 3: flag barrier with relaxed polls + one fence.acq_rel after
// mode 4: flag barrier, fence.acq_rel.gpu + relaxed store instead of st.release
__global__ void k_probe(int mode, int rounds, int nstore, int fs, unsigned* flags, unsigned* bar, double* data,
                        long long* out) {
  const int s = blockIdx.x, nb = gridDim.x, lane = threadIdx.x & 31;
  __syncthreads();
  long long t0 = clock64();
  for (int k = 1; k <= rounds; ++k) {
    for (int e = threadIdx.x; e < nstore; e += blockDim.x) data[(long long)s * nstore + e] = k + e;
    __syncthreads();
    if (threadIdx.x < 32) {
      if (mode == 1) {
        if (lane == 0) {
          unsigned g = ld_relaxed(bar + 1), old;
          asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
          if (old == nb - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
          } else {
            while (ld_acquire(bar + 1) == g) {
            }
          }
        }
        __syncwarp();
      } else {
        if (lane == 0) {
          if (mode == 4) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(flags + s * fs), "r"(k) : "memory");
          } else {
            st_release(flags + s * fs, k);
          }
        }
        for (;;) {
          bool mine = true;
          for (int r = lane; r < nb; r += 32) {
            if ((mode == 2 || mode >= 5) && (r < s - 3 || r > s + 3)) continue;
            const unsigned f = (mode == 3 || mode == 6) ? ld_relaxed(flags + r * fs) : ld_acquire(flags + r * fs);
            mine = mine && f >= (unsigned)k;
          }
          if (__all_sync(0xffffffffu, mine)) break;
          if (mode == 5) __nanosleep(100);
        }
        if (mode == 3 || mode == 6) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[s] = (t1 - t0) / rounds;
}

int main() {
  unsigned *flags, *bar;
  double* data;
  long long* out;
  cudaMalloc(&flags, 4096 * 4 * 32);
  cudaMalloc(&bar, 64);
  cudaMalloc(&data, 64 << 20);
  cudaMalloc(&out, 4096 * 8);
  long long h[4096];
  const int grids[] = {10, 120, 148};
  const int stores[] = {0, 900};
  for (int fs : {32})
  for (int nst : {900})
    for (int g : {10, 30, 60, 90, 120})
      for (int mode : {1, 2, 5, 6}) {
        cudaMemset(flags, 0, 4096 * 4 * 32);
        cudaMemset(bar, 0, 64);
        k_probe<<<g, 544>>>(mode, 2000, nst, fs, flags, bar, data, out);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, out, g * 8, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < g; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("stride %2d stores %4d grid %3d mode %d: %6lld cycles/round %s\n", fs, nst, g, mode, mx,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
