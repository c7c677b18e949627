// L2 read bandwidth on one B200: every CTA streams a buffer that fits L2
// (after one warming pass), 16-byte loads, four in flight per thread, grid = 148 x 8 CTAs of
// 512 threads; best of 20.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 l2_bw.cu -o l2_bw
#include <cstdio>
__global__ void k_read(const int4* __restrict__ a, long long n, int reps, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
      int4 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)  // four independent 16-byte loads in flight, L2 only
        v[q] = i + q * stride < n ? __ldcg(a + i + q * stride) : make_int4(0, 0, 0, 0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc.x ^= v[q].x; acc.y ^= v[q].y; acc.z ^= v[q].z; acc.w ^= v[q].w;
      }
    }
  if (acc.x == 0x12345678) sink[0] = acc;
}
int main() {
  for (long long mb : {16LL, 32LL, 64LL, 96LL, 512LL}) {
    const long long n = mb * (1 << 20) / 16;
    int4 *a, *s;
    cudaMalloc(&a, n * 16);
    cudaMalloc(&s, 16);
    cudaMemset(a, 1, n * 16);
    const int reps = 32;
    k_read<<<148 * 8, 512>>>(a, n, 1, s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int t = 0; t < 20; ++t) {
      cudaEventRecord(e0);
      k_read<<<148 * 8, 512>>>(a, n, reps, s);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("buffer %lld MB: %.0f GB/s\n", mb, double(n) * 16 * reps / (best * 1e-3) / 1e9);
    cudaFree(a);
    cudaFree(s);
  }
  return 0;
}
