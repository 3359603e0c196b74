// tma_probe.cu -- minimal TMA load check on the GPU (debug tool).
#include <cstdio>
#include <vector>
#include "../paper_math_9907190_b200/csrc/tma.cuh"
using namespace mg;

template <int VAR>
__global__ void probe(const __grid_constant__ CUtensorMap tm, double *out, int x0, int y0) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    if (VAR & 1) fence_mbar_init();
    if (VAR & 2) tma_prefetch_desc(&tm);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, 36 * 68 * 8);
    tma_load_2d(smem, &tm, x0, y0, &bar);
  }
  mbar_wait(&bar, 0);
  const double *s = (const double *)smem;
  for (int i = threadIdx.x; i < 36 * 68; i += blockDim.x) out[i] = s[i];
}

int main() {
  int n = 65; int64_t pitch = 80;
  std::vector<double> h(n * pitch);
  for (int j = 0; j < n; j++) for (int i = 0; i < pitch; i++) h[j * pitch + i] = j * 1000 + i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, 36 * 68 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  uint64_t dims[2] = {(uint64_t)n, (uint64_t)n}; uint32_t box[2] = {68, 36};
  bool ok = encode_tmap(&tm, d, 8, 2, dims, pitch, 0, box);
  printf("encode ok=%d\n", ok);
  printf("smem %p\n", nullptr);
  auto run = [&](auto kern, const char *name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    kern<<<1, 128, 40000>>>(tm, o, -2, -2);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s: %s\n", name, cudaGetErrorString(e));
    if (e == cudaSuccess) {
      std::vector<double> r(36 * 68);
      cudaMemcpy(r.data(), o, r.size() * 8, cudaMemcpyDeviceToHost);
      printf("  r[0]=%g r[2*68+2]=%g r[3*68+5]=%g\n", r[0], r[2 * 68 + 2], r[3 * 68 + 5]);
    }
    return e;
  };
  if (run(probe<0>, "plain")) return 1;
  if (run(probe<1>, "fence_init")) return 1;
  if (run(probe<2>, "prefetch")) return 1;
  return 0;
}
