// Microbenchmark: CTA barrier and dependent shared-memory load latency on
// one SM (1024 threads), to size the per-phase floor of the single-CTA
// local-search kernels.  nvcc -arch=sm_100a -O3 bar_lat.cu -o /tmp/bar_lat
#include <cstdio>
__global__ void k(long long* out, int iters, int* gbuf, int use_s) {
  __shared__ int a[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) a[i] = (i * 97 + 13) & 4095;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  int acc = 0;
  for (int i = 0; i < iters; ++i) acc += __syncthreads_or(i == threadIdx.x);
  long long t2 = clock64();
  int p = threadIdx.x & 4095;
  for (int i = 0; i < iters; ++i) p = a[p] & 4095;
  long long t3 = clock64();
  int q = threadIdx.x;
  for (int i = 0; i < iters; ++i) q += __shfl_xor_sync(0xffffffffu, q, 1);
  long long t4 = clock64();
  unsigned long long c = 0;
  for (int i = 0; i < iters; ++i) c += atomicAdd(reinterpret_cast<unsigned*>(&a[(p + i) & 4095]), 1u);
  long long t5 = clock64();
  const int* gp = use_s ? a : gbuf;  // generic pointer, shared at run time
  int r = threadIdx.x & 4095;
  for (int i = 0; i < iters; ++i) r = gp[r] & 4095;
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; out[2] = (t3 - t2) / iters;
    out[3] = (t4 - t3) / iters; out[4] = (t5 - t4) / iters; out[5] = acc + p + q + c + r; out[6] = (t6 - t5) / iters;
  }
}
int main() {
  long long* d; cudaMalloc(&d, 64);
  long long h[7]; int* gb; cudaMalloc(&gb, 4 * 4096); cudaMemset(gb, 0, 4 * 4096);
  for (int threads : {32, 256, 1024}) {
    k<<<1, threads>>>(d, 1000, gb, 1);
    k<<<1, threads>>>(d, 1000, gb, 1);
    cudaMemcpy(h, d, 56, cudaMemcpyDeviceToHost);
    printf("threads %d: syncthreads %lld, syncthreads_or %lld, dep LDS %lld, shfl %lld, atoms %lld, dep generic->shared %lld cycles\n",
           threads, h[0], h[1], h[2], h[3], h[4], h[6]);
  }
  return 0;
}
