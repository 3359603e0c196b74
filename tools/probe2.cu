// probe2.cu -- bisect the tile pipeline (debug tool)
#include <cstdio>
#include "../paper_math_9907190_b200/csrc/k2f.cu"
using namespace mg;

template <int V>
struct OpT {
  static constexpr int NT = 256;
  static constexpr int UW = 68, UH = 36, FW = 66, FH = 34;
  static constexpr int U_BYTES = UW * UH * 8, F_BYTES = FW * FH * 8;
  static constexpr int U_OFF = 0, F_OFF = al128(U_BYTES);
  static constexpr int STAGE = al128(F_OFF + F_BYTES);
  static constexpr int SMEM = 2 * STAGE + 20000;
  struct Params { CUtensorMap tu, tf; double *out; int M, ntx, ntiles; NormSink ns; };
  struct Acc { double mx; };
  static __device__ void prefetch(const Params &P) { if (V & 1) { tma_prefetch_desc(&P.tu); tma_prefetch_desc(&P.tf); } }
  static __device__ void init(Acc &a) { a.mx = 0; }
  static __device__ void issue(const Params &P, int t, unsigned char *st, uint64_t *bar) {
    int x0 = (t % P.ntx) * 64, y0 = (t / P.ntx) * 32;
    mbar_expect_tx(bar, U_BYTES + F_BYTES);
    tma_load_2d(st + U_OFF, &P.tu, x0 - 2, y0 - 2, bar);
    tma_load_2d(st + F_OFF, &P.tf, x0 - 1, y0 - 1, bar);
  }
  static __device__ void compute(const Params &P, int t, unsigned char *st, unsigned char *, Acc &acc) {
    const double *U = (const double *)st;
    if (threadIdx.x == 0) P.out[t] = U[3 * 68 + 5];
    acc.mx = nmax(acc.mx, U[threadIdx.x]);
  }
  static __device__ void finish(const Params &P, Acc &acc) { if (V & 2) block_norm_push<NT>(P.ns, acc.mx); }
};

template <class Op>
int runit(int n) {
  int M = n - 1; int64_t pitch = (n + 15) / 16 * 16;
  double *u, *out; unsigned long long *hist; int *cnt;
  cudaMalloc(&u, n * pitch * 8); cudaMemset(u, 0, n * pitch * 8);
  cudaMalloc(&out, 1 << 20); cudaMalloc(&hist, 64); cudaMalloc(&cnt, 4); cudaMemset(hist, 0, 64); cudaMemset(cnt, 0, 4);
  typename Op::Params P{};
  tm2<double>(&P.tu, u, n, n, pitch, Op::UW, Op::UH);
  tm2<double>(&P.tf, u, n, n, pitch, Op::FW, Op::FH);
  P.out = out; P.M = M; P.ntx = (M + 63) / 64; P.ntiles = P.ntx * ((M + 31) / 32); P.ns = NormSink{hist, cnt, 8};
  cudaError_t r = run_op<Op>(P, 0);
  printf("launch %s\n", cudaGetErrorString(r));
  r = cudaDeviceSynchronize();
  printf("sync %s\n", cudaGetErrorString(r));
  return r != cudaSuccess;
}

int main(int argc, char **argv) {
  int v = atoi(argv[1]);
  int n = 129;
  switch (v) {
    case 0: return runit<OpT<0>>(n);
    case 1: return runit<OpT<1>>(n);
    case 2: return runit<OpT<2>>(n);
    case 3: return runit<OpT<3>>(n);
  }
  return 0;
}
