// Which SM each CTA of a persistent 2-CTA-per-SM grid lands on (block -> SM
// map of the zpipe passes: 296 CTAs of 256 threads, ~105 KB of shared memory).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int *sm, long long *t0) {
  extern __shared__ char s[];
  if (threadIdx.x == 0) {
    unsigned id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    sm[blockIdx.x] = id;
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    t0[blockIdx.x] = t;
    s[0] = 1;
  }
  // linger so every CTA is resident at once
  long long a, b;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b)); } while (b - a < 200000);
}
int main() {
  int G = 296, smem = 105 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int *d; long long *dt;
  cudaMalloc(&d, G * 4); cudaMalloc(&dt, G * 8);
  int h[296], ref[296];
  for (int rep = 0; rep < 5; rep++) {
    probe<<<G, 256, smem>>>(d, dt);
    cudaMemcpy(h, d, G * 4, cudaMemcpyDeviceToHost);
    if (rep == 0) {
      for (int i = 0; i < G; i++) ref[i] = h[i];
      printf("block: sm\n");
      for (int i = 0; i < G; i++) printf("%d:%d%s", i, h[i], (i % 16 == 15) ? "\n" : " ");
      printf("\n");
      // partner of block b (other block on the same SM)
      int same_plus148 = 0, same_plus1 = 0;
      for (int b = 0; b < 148; b++) same_plus148 += h[b] == h[b + 148];
      for (int b = 0; b + 1 < G; b += 2) same_plus1 += h[b] == h[b + 1];
      printf("pairs (b, b+148) on one SM: %d / 148; (2i, 2i+1): %d / 148\n", same_plus148, same_plus1);
    } else {
      int diff = 0;
      for (int i = 0; i < G; i++) diff += h[i] != ref[i];
      printf("rep %d: %d blocks on a different SM than rep 0\n", rep, diff);
    }
  }
  return 0;
}
