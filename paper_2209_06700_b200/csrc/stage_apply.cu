// K1 dispatch over the polynomial degree (kernels: stage_apply.cuh, instantiated per degree in
// stage_apply_k{1,2,3,4}.cu).
#include "spk_internal.cuh"

cudaError_t spk_launch_apply_k1(int, bool, int, const SpkApplyArgs&, cudaStream_t, int*);
cudaError_t spk_launch_apply_k2(int, bool, int, const SpkApplyArgs&, cudaStream_t, int*);
cudaError_t spk_launch_apply_k3(int, bool, int, const SpkApplyArgs&, cudaStream_t, int*);
cudaError_t spk_launch_apply_k4(int, bool, int, const SpkApplyArgs&, cudaStream_t, int*);
int spk_apply_geo_k1(int, int);
int spk_apply_geo_k2(int, int);
int spk_apply_geo_k3(int, int);
int spk_apply_geo_k4(int, int);

cudaError_t spk_launch_apply(int K, int Q, bool block_mode, int epi, const SpkApplyArgs& a,
                             cudaStream_t s, int* nctas_out) {
  switch (K) {
    case 1: return spk_launch_apply_k1(Q, block_mode, epi, a, s, nctas_out);
    case 2: return spk_launch_apply_k2(Q, block_mode, epi, a, s, nctas_out);
    case 3: return spk_launch_apply_k3(Q, block_mode, epi, a, s, nctas_out);
    case 4: return spk_launch_apply_k4(Q, block_mode, epi, a, s, nctas_out);
  }
  return cudaErrorInvalidValue;
}

int spk_apply_geo(int K, int Q, int what) {
  switch (K) {
    case 1: return spk_apply_geo_k1(Q, what);
    case 2: return spk_apply_geo_k2(Q, what);
    case 3: return spk_apply_geo_k3(Q, what);
    case 4: return spk_apply_geo_k4(Q, what);
  }
  return -1;
}

int spk_apply_smem_bytes(int K, int Q) { return spk_apply_geo(K, Q, 0); }
int spk_apply_threads(int K, int Q) { return spk_apply_geo(K, Q, 1); }
