// tile_probe.cu -- run one TMA tile kernel standalone (debug tool).
#include <cstdio>
#include <vector>
#include "../paper_math_9907190_b200/csrc/kernels.h"
using namespace mg;
int main(int argc, char **argv) {
  int n = argc > 1 ? atoi(argv[1]) : 129;
  int M = n - 1;
  int64_t pitch = (n + 15) / 16 * 16;
  std::vector<double> h(n * pitch, 0.0);
  for (int j = 1; j < M; j++) for (int i = 1; i < M; i++) h[j * pitch + i] = 0.001 * ((i * 7 + j * 13) % 17);
  double *u, *f, *e, *o; unsigned long long *hist; int *cnt;
  cudaMalloc(&u, h.size() * 8); cudaMalloc(&f, h.size() * 8);
  int H = M / 2 + 1; int64_t ph = (H + 15) / 16 * 16;
  cudaMalloc(&e, H * ph * 8); cudaMalloc(&o, H * ph * 8);
  cudaMemset(e, 0, H * ph * 8); cudaMemset(o, 0, H * ph * 8);
  cudaMalloc(&hist, 64); cudaMalloc(&cnt, 4); cudaMemset(hist, 0, 64); cudaMemset(cnt, 0, 4);
  cudaMemcpy(u, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(f, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  Coef<double> k{(double)M * M, (double)M * M / 6.0};
  S2<double> d{e, o, ph};
  NormSink ns{hist, cnt, 8};
  cudaError_t r = fast2_desc_fine<double>(u, f, pitch, d, M, 2, k, ns, 0);
  printf("launch: %s\n", cudaGetErrorString(r));
  r = cudaDeviceSynchronize();
  printf("sync: %s\n", cudaGetErrorString(r));
  return r != cudaSuccess;
}
