// K1 instantiations for degree k = 2 (split per degree for parallel compilation).
#include "stage_apply.cuh"

cudaError_t spk_launch_apply_k2(int Q, bool block_mode, int epi, const SpkApplyArgs& a, cudaStream_t s,
                                int* nctas_out) {
  return dispatch_k<2>(Q, block_mode, epi, a, s, nctas_out);
}

int spk_apply_geo_k2(int Q, int what) {
  switch (Q) {
#define SPK_GEO(q) \
  case q: return what == 0 ? (int)(sizeof(double) * Geo<2, q>::SMEM_DOUBLES) \
               : what == 1 ? Geo<2, q>::NT : what == 2 ? Geo<2, q>::TYE : Geo<2, q>::TZE;
    SPK_GEO(1) SPK_GEO(2) SPK_GEO(3) SPK_GEO(4)
#undef SPK_GEO
  }
  return -1;
}
