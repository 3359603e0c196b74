// tma_host.cu -- host-side tensor-map encoding (cuTensorMapEncodeTiled via the
// runtime's driver entry point; no link dependency on libcuda).
#include <cudaTypedefs.h>

#include <cstdlib>

#include "tma.cuh"

namespace mg {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// L2 sector promotion of the TMA loads (MG_L2_PROMO = 0 / 64 / 128 / 256).  Default none:
// measured on B200 (interleaved A/B, tools/ab.py) 256 B promotion cost 1.2 % (3D) and 0.8 %
// (2D) per cycle -- the halo boxes' edges pulled in sectors nobody reads.
static CUtensorMapL2promotion l2_promotion() {
  static const CUtensorMapL2promotion p = [] {
    const char *e = getenv("MG_L2_PROMO");
    const int v = e ? atoi(e) : 0;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                  : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                            : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  return p;
}

bool encode_tmap(CUtensorMap *tm, const void *base, int esz, int rank, const uint64_t *dims, uint64_t pitch,
                 uint64_t plane, const uint32_t *box) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t gdim[3] = {dims[0], dims[1], rank > 2 ? dims[2] : 1};
  cuuint64_t gstr[2] = {pitch * (uint64_t)esz, plane * (uint64_t)esz};
  cuuint32_t bdim[3] = {box[0], box[1], rank > 2 ? box[2] : 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(tm, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank,
                  const_cast<void *>(base), gdim, gstr, bdim, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Off by default: measured on B200 it gained nothing (the next pass's CTAs
// cannot become resident before the previous pass's 200 KB-smem CTAs exit).
bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("MG_PDL");
    return e && *e && *e != '0';
  }();
  return on;
}

}  // namespace mg
