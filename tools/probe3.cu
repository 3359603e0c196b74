// probe3.cu -- bisect TMA kernel parameters (debug tool)
#include <cstdio>
#include <vector>
#include "../paper_math_9907190_b200/csrc/tma.cuh"
using namespace mg;

struct P2 { CUtensorMap tu, tf; double *out; int a, b, c; };

__global__ void kA(const __grid_constant__ P2 P, int x0, int y0) {   // struct param
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) { mbar_expect_tx(&bar, 36 * 68 * 8); tma_load_2d(smem, &P.tu, x0, y0, &bar); }
  mbar_wait(&bar, 0);
  if (threadIdx.x == 0) P.out[0] = ((const double *)smem)[3 * 68 + 5];
}
__global__ void kB(const __grid_constant__ CUtensorMap tm, double *out, int x0, int y0) {  // bare, big smem
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) { mbar_expect_tx(&bar[0], 36 * 68 * 8); tma_load_2d(smem, &tm, x0, y0, &bar[0]); }
  mbar_wait(&bar[0], 0);
  if (threadIdx.x == 0) out[0] = ((const double *)smem)[3 * 68 + 5];
}
__global__ void kC(const __grid_constant__ P2 P, int x0, int y0) {   // struct param, second map
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) { mbar_expect_tx(&bar, 36 * 68 * 8); tma_load_2d(smem, &P.tf, x0, y0, &bar); }
  mbar_wait(&bar, 0);
  if (threadIdx.x == 0) P.out[0] = ((const double *)smem)[3 * 68 + 5];
}

__global__ void kD(const __grid_constant__ P2 P, int x0, int y0) {   // two loads, one barrier
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, 2 * 36 * 68 * 8);
    tma_load_2d(smem, &P.tu, x0, y0, &bar);
    tma_load_2d(smem + 19584, &P.tf, x0 + 1, y0 + 1, &bar);
  }
  mbar_wait(&bar, 0);
  if (threadIdx.x == 0) P.out[0] = ((const double *)smem)[3 * 68 + 5] + ((const double *)(smem + 19584))[0];
}

template <int MODE>
__global__ void kE(const __grid_constant__ P2 P, int x0, int y0) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); }
  __syncthreads();
  const int off = (MODE & 4) ? 20480 : 19584;
  if (threadIdx.x == 0) {
    if (MODE & 2) {
      mbar_expect_tx(&bar[0], 36 * 68 * 8);
      tma_load_2d(smem, &P.tu, x0, y0, &bar[0]);
      mbar_expect_tx(&bar[1], 36 * 68 * 8);
      tma_load_2d(smem + off, (MODE & 1) ? &P.tf : &P.tu, x0 + 1, y0 + 1, &bar[1]);
    } else {
      mbar_expect_tx(&bar[0], 2 * 36 * 68 * 8);
      tma_load_2d(smem, &P.tu, x0, y0, &bar[0]);
      tma_load_2d(smem + off, (MODE & 1) ? &P.tf : &P.tu, x0 + 1, y0 + 1, &bar[0]);
    }
  }
  mbar_wait(&bar[0], 0);
  if (MODE & 2) mbar_wait(&bar[1], 0);
  if (threadIdx.x == 0) P.out[0] = ((const double *)smem)[3 * 68 + 5] + ((const double *)(smem + off))[0];
}

int main(int argc, char **argv) {
  int v = atoi(argv[1]);
  int n = 129; int64_t pitch = 144;
  std::vector<double> h(n * pitch);
  for (int j = 0; j < n; j++) for (int i = 0; i < pitch; i++) h[j * pitch + i] = j * 1000 + i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, 64);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  P2 P{};
  uint64_t dims[2] = {(uint64_t)n, (uint64_t)n}; uint32_t box[2] = {68, 36};
  encode_tmap(&P.tu, d, 8, 2, dims, pitch, 0, box);
  encode_tmap(&P.tf, d, 8, 2, dims, pitch, 0, box);
  P.out = o;
  int smem = (v == 1) ? 100000 : 40000;
  if (v == 0) { cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); kA<<<1, 256, smem>>>(P, -2, -2); }
  if (v == 1) { cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); kB<<<8, 256, smem>>>(P.tu, o, -2, -2); }
  if (v == 2) { cudaFuncSetAttribute(kC, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); kC<<<1, 256, smem>>>(P, -2, -2); }
  if (v == 3) { cudaFuncSetAttribute(kD, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); kD<<<1, 256, smem>>>(P, -2, -2); }
#define RUNE(M) if (v == 10 + M) { cudaFuncSetAttribute(kE<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 50000); kE<M><<<1, 256, 50000>>>(P, -2, -2); }
  RUNE(0) RUNE(1) RUNE(2) RUNE(3) RUNE(4) RUNE(5) RUNE(6) RUNE(7)
  cudaError_t e = cudaDeviceSynchronize();
  double r = -1; if (!e) cudaMemcpy(&r, o, 8, cudaMemcpyDeviceToHost);
  printf("v%d: %s  r=%g\n", v, cudaGetErrorString(e), r);
  return 0;
}
